import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values
nb, B = int(sys.argv[1]), int(sys.argv[2])
systems = acopf.batch(nb, B, seed=7)
dev = Device(0)
dev.analyze(systems[0])
bt = Batch(dev)
bt.upload(stack_values(systems))
cfg = SolverConfig(cg_max_iter=22, cg_tol=1e-300)
bt.solve_resident(cfg, timing=True)
print(os.environ.get("HYKKT_KS_DEBUG", "0"), dev.timing()["cg_ms"])
