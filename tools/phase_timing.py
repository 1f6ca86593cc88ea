"""Per-phase device timings of the single-system path on configs C1-C4."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf

cfgs = sys.argv[1:] or ["C1", "C2", "C3", "C4"]
for name in cfgs:
    nb = acopf.CONFIG_BUSES[name]
    s = acopf.generate(nb, 7, 7)
    dev = Device(0)
    t = time.time(); dev.analyze(s); ta = time.time() - t
    info = dev.info()
    dev.upload(s)
    cfg = SolverConfig()
    for rep in range(4):
        r = dev.solve_resident(cfg, timing=True)
    tm = dev.timing()
    print(json.dumps(dict(cfg=name, analyze_s=round(ta, 2), nnz_l=info["nnz_l"], nsup=info["n_supernodes"],
                          levels=info["n_levels"], cg_its=r.cg_iterations, status=int(r.status),
                          **{k: round(v, 3) if isinstance(v, float) else v for k, v in tm.items()})))
    dev.close()
