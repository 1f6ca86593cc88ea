"""Single-system solve of config C1-C4 with per-phase device timing; saves the
solution to /tmp/<tag>_<cfg>.npz so two factor variants (HYKKT_FACTOR=ll vs
the default multifrontal) can be compared with --diff."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

if sys.argv[1] == "--diff":
    for cfg in sys.argv[4:]:
        a, b = np.load(f"/tmp/{sys.argv[2]}_{cfg}.npz"), np.load(f"/tmp/{sys.argv[3]}_{cfg}.npz")
        x = np.concatenate([a[k] for k in ("dx", "dy", "ds", "dyd")])
        y = np.concatenate([b[k] for k in ("dx", "dy", "ds", "dyd")])
        print(cfg, "its", int(a["its"]), int(b["its"]), "rel diff", np.linalg.norm(x - y) / np.linalg.norm(y))
    sys.exit(0)
from paper_2110_03636_b200 import Device, SolverConfig, acopf
tag = sys.argv[1]
for name in sys.argv[2:]:
    s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
    dev = Device(0)
    dev.analyze(s)
    dev.upload(s)
    for rep in range(3):
        r = dev.solve_resident(SolverConfig(), timing=True)
    tm = dev.timing()
    sol = dev.download()
    print(tag, name, json.dumps({k: round(v, 3) if isinstance(v, float) else v for k, v in tm.items()}),
          "its", r.cg_iterations, "status", int(r.status), flush=True)
    np.savez(f"/tmp/{tag}_{name}.npz", its=r.cg_iterations, dx=sol.dx, dy=sol.dy, ds=sol.ds, dyd=sol.dyd)
    dev.close()
