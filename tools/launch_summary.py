"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch
list (cold-cache, serialised launches: compare shares, not absolutes)."""
import csv, sys, collections
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if len(r) <= vi or not r[vi]:
        continue
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("hykkt::dev::", "")
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
for k, v in tot.most_common():
    print(f"{k:24s} launches={cnt[k]:3d} total={v:9.3f} ms share={v / T:.3f}")
print(f"total {T:.3f} ms")
