"""Per-kernel summary of an ncu launch list (time, DRAM bytes per launch):
   python tools/summarize_launches.py launches.csv [--last K]
Prints, per kernel name, launches, mean ms, mean read/write GB and GB/s, for the
launches of the timed steps (the last K launches of the step kernels; the input
generator and warm-up are listed separately by name)."""
import collections
import csv
import io
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

path = sys.argv[1]
txt = open(path).read()
i = txt.index('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[i:])))
per = collections.OrderedDict()
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    d = per.setdefault(key, {})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0}[unit]
    d[r["Metric Name"]] = v * scale
agg = collections.OrderedDict()
for (kid, name), d in per.items():
    short = name.split("(")[0].replace("void ", "").replace("skh::", "").replace("(anonymous namespace)::", "")
    a = agg.setdefault(short, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0)
    a[3] += d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'n':>4s} {'ms/launch':>10s} {'share':>6s} {'rd GB/l':>9s} {'wr GB/l':>9s} {'GB/s':>8s}")
for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {n:4d} {1e3 * t / n:10.4f} {t / tot:6.1%} {rd / n / 1e9:9.3f} {wr / n / 1e9:9.3f} "
          f"{(rd + wr) / t / 1e9:8.1f}")
