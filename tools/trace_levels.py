"""Per-level timeline of one traced H^-1 pass (from tools/trace_trsv.py's
TRACE_NPZ dump): per supernode level, task count, first claim, last end, and
the median claim-to-end time, forward and backward."""
import sys
import numpy as np

d = np.load(sys.argv[1])
par = d["parent"]; ns = len(par)
lev = np.zeros(ns, int)
for k in range(ns):  # children precede parents in the supernode numbering
    p = par[k]
    if p >= 0: lev[p] = max(lev[p], lev[k] + 1)
for tag in ("f", "b"):
    st, en = d[tag + "start"], d[tag + "end"]
    print(f"{'forward' if tag == 'f' else 'backward'}: lev n first_claim last_claim last_end med_hold p90_hold")
    for l in range(lev.max() + 1):
        m = (lev == l) & (st > -1e6) & (en > -1e6) & (st < 1e7) & (en < 1e7)
        if m.sum() == 0: continue
        hold = en[m] - st[m]
        print(f"  {l:3d} {m.sum():6d} {st[m].min():8.1f} {st[m].max():8.1f} {en[m].max():8.1f} {np.median(hold):6.2f} {np.percentile(hold, 90):6.2f}")
