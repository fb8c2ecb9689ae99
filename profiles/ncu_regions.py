"""Per-region stall-reason breakdown of a k_sweep ncu capture (needs -lineinfo).

    python profiles/ncu_regions.py <report.ncu-rep> <object.o> <mangled-kernel-name>

Regions are source-line ranges of ca_sweep.cuh / ca_lemke.cuh (setup, pivot loop,
structural solve, epilogue ...); prints instruction share and the stall samples
of each reason per region.
"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import addr_lines  # noqa: E402

REASONS = ["stall_long_sb", "stall_no_inst", "stall_wait", "stall_short_sb", "stall_branch_resolving",
           "stall_selected", "stall_not_selected", "stall_mio", "stall_lg", "stall_math", "stall_dispatch"]


def region(k):
    f, l = k
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2406_07048_b200", "csrc", f)
    marks = REG.get(f)
    if not marks:
        return f
    name = f
    for ln, nm in marks:
        if l >= ln:
            name = nm
    return name


def marks_of(f):
    """Region boundaries: lines containing '// @region <name>' markers."""
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2406_07048_b200", "csrc", f)
    out = [(0, f)]
    for i, line in enumerate(open(p).read().split("\n"), 1):
        if "@region" in line:
            out.append((i, line.split("@region", 1)[1].strip().split()[0]))
    return out


REG = {f: marks_of(f) for f in ("ca_sweep.cuh", "ca_lemke.cuh", "ca_kernels.cuh")}


def main():
    rep, obj, fun = sys.argv[1:4]
    m2l = addr_lines(obj, fun)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    ir = {r: hdr.index(r) for r in REASONS}
    data = [r for r in rows[2:] if r[0].startswith("0x")]
    base = int(data[0][0], 16)
    inst = collections.Counter()
    st = collections.defaultdict(collections.Counter)
    for r in data:
        k = m2l.get(int(r[0], 16) - base, ("?", 0))
        g = region(k) if k[0] != "?" else "?"
        inst[g] += int(r[ia])
        for s, i in ir.items():
            st[g][s] += int(r[i] or 0)
    tot = sum(inst.values())
    stot = sum(sum(c.values()) for c in st.values())
    print(f"{'region':16s} {'inst%':>6s} {'stall%':>6s} " + " ".join(f"{s[6:]:>8s}" for s in REASONS))
    for g, n in inst.most_common():
        ss = sum(st[g].values())
        print(f"{g:16s} {100 * n / tot:6.1f} {100 * ss / stot:6.1f} " +
              " ".join(f"{100 * st[g][s] / stot:8.1f}" for s in REASONS))
    print(f"{'TOTAL':16s} {100.0:6.1f} {100.0:6.1f} " +
          " ".join(f"{100 * sum(st[g][s] for g in st) / stot:8.1f}" for s in REASONS))


if __name__ == "__main__":
    main()
