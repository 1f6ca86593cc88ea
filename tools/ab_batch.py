"""A/B of batched-solve variants (env is read when the context and the plan
are built): AB_B systems of ACTIVSg2000 shape, 4 drifted value sets cycled as
in bench.py; per variant: device ms per step (sum of the per-call device
totals) and the phase split.  usage: ab_batch.py 'VAR=1 VAR2=x' ..."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
from paper_2110_03636_b200 import Device, SolverConfig
from paper_2110_03636_b200.solver import Batch, stack_values

B = int(os.environ.get("AB_B", "256"))
steps = int(os.environ.get("AB_STEPS", "6"))
sets = bench.value_sets(2000, list(range(7, 7 + B)))
stacked = [stack_values(s) for s in sets]
cfg = SolverConfig()
for v in sys.argv[1:] or [""]:
    keys = []
    for kv in v.split():
        k, val = kv.split("=")
        os.environ[k] = val
        keys.append(k)
    dev = Device(0)
    dev.analyze(sets[0][0])
    bt = Batch(dev)
    acc = {}
    for st in range(3 + steps):
        bt.upload(stacked[st % len(stacked)])
        reps = bt.solve_resident(cfg, timing=True)
        t = dev.timing()
        if st >= 3:
            for k in ("total_ms", "assemble_ms", "factor_ms", "cg_ms"):
                acc[k] = acc.get(k, 0.0) + t[k] / steps
    print(json.dumps(dict(variant=v, B=B, **{k: round(x, 3) for k, x in acc.items()},
                          solves_per_s=round(B / acc["total_ms"] * 1e3, 1),
                          bad=sum(1 for r in reps if r.status > 1))), flush=True)
    for k in keys:
        del os.environ[k]
    dev.close()
