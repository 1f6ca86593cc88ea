"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export per
CUDA source line: warp-stall samples, instructions executed, top stall
reasons.  Usage: python tools/ncu_lines.py export.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.defaultdict(lambda: collections.Counter())
src_text = {}
file = None
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    ln, src = r[0], r[1]
    if ln:
        cur_line = (file, int(ln))
        src_text[cur_line] = src
    if cur_line is None or not r[2]:
        continue
    def num(name):
        try:
            return float(r[hdr.index(name)] or 0)
        except (ValueError, IndexError):
            return 0.0
    c = agg[cur_line]
    c["samples"] += num("Warp Stall Sampling (All Samples)")
    c["inst"] += num("Instructions Executed")
    for name in hdr:
        if name.startswith("stall_") and "Not Issued" not in name:
            c[name] += num(name)
tot = sum(c["samples"] for c in agg.values())
tot_i = sum(c["inst"] for c in agg.values())
print(f"total samples {tot:.0f}  instructions {tot_i:.3e}")
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    stalls = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    s = " ".join(f"{n}:{v/max(c['samples'],1):.2f}" for v, n in stalls)
    print(f"{key[0]}:{key[1]:4d} {100*c['samples']/tot:5.1f}% inst {100*c['inst']/tot_i:5.1f}%  {s}  | {src_text.get(key,'').strip()[:70]}")
