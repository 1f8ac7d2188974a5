"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]; cnt[name] += 1
T = sum(tot.values())
import signal; signal.signal(signal.SIGPIPE, signal.SIG_DFL)
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:44s} n={cnt[k]:5d} {v/1e3:9.2f} ms {100*v/T:5.1f}%  avg {v/cnt[k]:9.1f} us")
print(f"total serialized {T/1e3:.2f} ms")
