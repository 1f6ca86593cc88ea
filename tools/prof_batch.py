"""One batched solve_full of B ACTIVSg2000-shaped systems (profiling driver:
run under ncu with -k regex:<kernel>)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
systems = acopf.batch(nb, B, seed=7)
dev = Device(0)
dev.analyze(systems[0])
bt = Batch(dev)
bt.upload(stack_values(systems))
for _ in range(reps):
    r = bt.solve_resident(SolverConfig(), timing=True)
print({k: round(v, 3) for k, v in dev.timing().items()})
print("cg its max", max(x.cg_iterations for x in r), "mean", sum(x.cg_iterations for x in r) / len(r))
