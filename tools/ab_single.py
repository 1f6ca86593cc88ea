"""A/B of single-system solve variants (env settings read at analysis time).
usage: ab_single.py C1,C2 'HYKKT_TRSV_BINS=0' 'HYKKT_TRSV_BINS=1' ...
Prints per config and variant: total / factor / CG ms, CG us per iteration,
and the solution's max relative deviation from the first variant."""
import json, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf

cfgs = sys.argv[1].split(",")
variants = sys.argv[2:] or [""]
for name in cfgs:
    s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
    perm = None
    base = None
    for v in variants:
        keys = []
        for kv in v.split():
            k, val = kv.split("=")
            os.environ[k] = val
            keys.append(k)
        dev = Device(0)
        dev.analyze(s, perm)
        if perm is None:
            perm = dev.perm()
        dev.upload(s)
        cfg = SolverConfig()
        best = None
        for rep in range(5):
            r = dev.solve_resident(cfg, timing=True)
            tm = dev.timing()
            if best is None or tm["total_ms"] < best["total_ms"]:
                best = tm
        sol = dev.download().stacked()
        err = 0.0 if base is None else float(np.max(np.abs(sol - base)) / np.max(np.abs(base)))
        if base is None:
            base = sol
        its = r.cg_iterations
        print(json.dumps(dict(cfg=name, variant=v, cg_its=its, status=int(r.status),
                              total_ms=round(best["total_ms"], 3), factor_ms=round(best["factor_ms"], 3),
                              cg_ms=round(best["cg_ms"], 3), cg_us_it=round(1e3 * best["cg_ms"] / max(its, 1), 1),
                              dev_vs_first=err)), flush=True)
        for k in keys:
            del os.environ[k]
        dev.close()
