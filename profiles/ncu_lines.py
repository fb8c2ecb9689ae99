"""Per-source-line instruction / stall attribution of an ncu capture (needs -lineinfo).

    python profiles/ncu_lines.py <report.ncu-rep> <object.o> <mangled-kernel-name> [top]

Maps ncu's per-SASS-address counters to CUDA source lines using nvdisasm -g on the
cubin extracted from the object file.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def addr_lines(obj, fun):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = glob.glob(os.path.join(d, "*.cubin"))[0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    secs = re.split(r"\n\s*\.section\s+\.text\.", txt)
    sec = [s for s in secs if s.startswith(fun)][0]
    cur, m2l = None, {}
    for line in sec.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m and cur:
            m2l[int(m.group(1), 16)] = cur
    return m2l


def main():
    rep, obj, fun = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    m2l = addr_lines(obj, fun)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isamp, ith = (hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"),
                      hdr.index("Avg. Threads Executed"))
    data = [(int(r[0], 16), int(r[ia]), int(r[isamp]), float(r[ith] or 0)) for r in rows[2:] if r[0].startswith("0x")]
    base = data[0][0]
    inst, stall, thr = collections.Counter(), collections.Counter(), collections.Counter()
    for a, n, s, th in data:
        k = m2l.get(a - base, ("?", 0))
        inst[k] += n
        stall[k] += s
        thr[k] += n * th
    tot, tots = sum(inst.values()), max(1, sum(stall.values()))
    srcs = {}
    for f in glob.glob(os.path.join(ROOT, "paper_2406_07048_b200", "csrc", "*")):
        srcs[os.path.basename(f)] = open(f).read().split("\n")
    print(f"total warp-instructions {tot}")
    for k, n in inst.most_common(top):
        txt = srcs.get(k[0], [""] * (k[1] + 1))[k[1] - 1].strip()[:72] if k[1] else ""
        print(f"{100 * n / tot:5.1f}% inst {100 * stall[k] / tots:5.1f}% stall thr {thr[k] / max(n, 1):4.1f} "
              f"{k[0]}:{k[1]} {txt}")


if __name__ == "__main__":
    main()
