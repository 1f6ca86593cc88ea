"""Protocol-cost experiment: ks_solve with the step compute skipped
(HYKKT_KS_DEBUG=3; CG counts forced by max_iter) vs the real run at the same
iteration count."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values
systems = acopf.batch(2000, 256, seed=7)
dev = Device(0)
dev.analyze(systems[0])
bt = Batch(dev)
bt.upload(stack_values(systems))
cfg = SolverConfig(cg_max_iter=22, cg_tol=1e-300)
for _ in range(2):
    bt.solve_resident(cfg, timing=True)
print(os.environ.get("HYKKT_KS_DEBUG", "0"), {k: round(v, 3) for k, v in dev.timing().items() if k in ("cg_ms", "factor_ms")})
