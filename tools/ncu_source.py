"""Summarise an ncu --set full report's SASS source page: totals, instructions and
stall samples by execution-count class, the top stalls and (optionally) the
stall-reason mix of an instruction-index range.
   python tools/ncu_source.py report.ncu-rep [lo hi]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
I, S, SRC = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
W = hdr.index("L1 Wavefronts Shared")
WI = hdr.index("L1 Wavefronts Shared Ideal")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) > W]
num = lambda r, i: int(r[i] or 0)  # noqa: E731
print("warp instr %.3g  samples %d  smem wavefronts %.3g (ideal %.3g)" % (
    sum(num(r, I) for r in data), sum(num(r, S) for r in data), sum(num(r, W) for r in data),
    sum(num(r, WI) for r in data)))
cls = collections.defaultdict(lambda: [0, 0, 0, 0])
for r in data:
    c = cls[num(r, I)]
    c[0] += 1
    c[1] += num(r, I)
    c[2] += num(r, S)
    c[3] += num(r, W)
for k, v in sorted(cls.items(), key=lambda x: -x[1][1])[:6]:
    print(f"  exec {k:>12}: {v[0]:4d} instrs {v[1]:.3g} warp-instr {v[2]} samples {v[3]:.3g} wf")
print("top stalls (index, exec, samples, wavefronts, sass):")
for i, r in sorted(enumerate(data), key=lambda x: -num(x[1], S))[:14]:
    print(f"  {i:5d} {num(r, I):>12} {num(r, S):>7} {num(r, W):>10} {r[SRC].strip()[:70]}")
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    agg = collections.Counter()
    for r in data[lo:hi]:
        for i in stall_cols:
            agg[hdr[i]] += num(r, i)
    print("stall reasons in", lo, hi, agg.most_common(10))
