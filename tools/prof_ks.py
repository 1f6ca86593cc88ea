"""One batched solve_full (system-per-CTA path) of B ACTIVSg2000-shaped
systems: profiling driver for ncu -k regex:ks_solve."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
systems = acopf.batch(nb, B, seed=7)
dev = Device(0)
dev.analyze(systems[0])
bt = Batch(dev)
bt.upload(stack_values(systems))
for _ in range(reps):
    bt.solve_resident(SolverConfig())
print("done")
