"""Build k_sweep tuning variants (compile-time -D switches) and time them on the GPU.

    python profiles/tune.py build NAME=DEF1,DEF2 NAME2= ...   # here (no GPU): libs in scratch/libs/
    python profiles/tune.py time [n_scenes] [iters]          # on the B200: times every built variant

Each variant is a full libca.so built with extra -D flags into scratch/libs/<NAME>.so;
`time` runs profiles/time_sweep.py against each with CA_LIBRARY pointing at it.
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = os.path.join(ROOT, "scratch", "libs")


def main():
    cmd = sys.argv[1]
    if cmd == "build":
        sys.path.insert(0, ROOT)
        from paper_2406_07048_b200 import build

        os.makedirs(LIBS, exist_ok=True)
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            defines = tuple(d for d in defs.split(",") if d)
            out = build.build(out=os.path.join(LIBS, name + ".so"), defines=defines)
            log = open(out + ".log").read()
            i = log.find("k_sweepILi2ELi13ELb1")
            print(name, defines, log[i:i + 400].split("\n")[2:4] if i >= 0 else "")
    else:
        args = sys.argv[2:] or ["1024", "10"]
        for lib in sorted(glob.glob(os.path.join(LIBS, "*.so"))):
            env = dict(os.environ, CA_LIBRARY=lib)
            r = subprocess.run([sys.executable, os.path.join(ROOT, "profiles", "time_sweep.py"), *args], env=env,
                               capture_output=True, text=True, timeout=600)
            print(os.path.basename(lib), (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1])


if __name__ == "__main__":
    main()
