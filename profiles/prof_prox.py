"""C5 driver (1024 scenes, prox_eps = 1e-2) for one ncu --set full capture of the
k_sweep launch running the NEXT f4 dual Newton pair solver."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07048_b200 as ca, scenes
sc = scenes.make_c5(n_scenes=1024)
g = ca.Problem(sc, prox_eps=1e-2)
g.admm_iterate(3, hist=False)
print("ok")
