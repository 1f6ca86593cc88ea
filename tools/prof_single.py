"""One single-system solve (ncu target): analyze, upload, solve twice."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
dev = Device(0); dev.analyze(s); dev.upload(s)
for _ in range(2):
    r = dev.solve_resident(SolverConfig())
print(name, int(r.status), r.cg_iterations)
