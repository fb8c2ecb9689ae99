"""Full-size C5 (4096 scenes) driver for one ncu --set full capture of k_sweep."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07048_b200 as ca, scenes
sc = scenes.make_c5()
g = ca.Problem(sc)
g.admm_iterate(3, hist=False)
print("ok")
