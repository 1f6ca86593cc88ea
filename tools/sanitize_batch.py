"""Small batched solve for compute-sanitizer runs (both batch paths)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values
for path in ("default", "lane"):
    os.environ.pop("HYKKT_BATCH_PATH", None)
    if path == "lane":
        os.environ["HYKKT_BATCH_PATH"] = "lane"
    systems = acopf.batch(200, 40, seed=7)
    d = Device(0); d.analyze(systems[0])
    b = Batch(d); b.upload(stack_values(systems))
    reps = b.solve_resident(SolverConfig())
    print(path, sorted(set(int(r.status) for r in reps)), max(r.cg_iterations for r in reps), flush=True)
    d.close()
