import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values
def log(*a): print(*a, flush=True)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
bad_at = int(sys.argv[2]) if len(sys.argv) > 2 else 17
good = acopf.batch(60, n - 1, seed=11)
bad = acopf.generate(60, 7, 999)
bad.h = bad.h.with_values(bad.h.values.copy())
diag = np.flatnonzero(bad.h.rowidx == bad.h.col_of_entries())
bad.h.values[diag[5]] = -1e6
systems = good[:bad_at] + [bad] + good[bad_at:] if bad_at >= 0 else good + [good[0]]
dev = Device(0); dev.analyze(systems[0]); log("analyzed")
b = Batch(dev); b.upload(stack_values(systems)); log("uploaded")
t = time.time(); reps = b.solve_resident(SolverConfig(), timing=True); log("solved", time.time() - t, dev.timing())
log([int(r.status) for r in reps]); log([r.cg_iterations for r in reps])
single = Device(0); single.analyze(systems[0], dev.perm()); log("single analyzed")
for k, s in enumerate(systems):
    t = time.time(); r1 = single.solve_full(s, SolverConfig()); log(k, int(r1.report.status), r1.report.cg_iterations, "%.3f" % (time.time() - t))
