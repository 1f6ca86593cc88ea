import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf
good = acopf.generate(60, 7, 11)
bad = acopf.generate(60, 7, 999)
bad.h = bad.h.with_values(bad.h.values.copy())
diag = np.flatnonzero(bad.h.rowidx == bad.h.col_of_entries())
bad.h.values[diag[5]] = -1e6
d = Device(0); d.analyze(good); print("analyzed", flush=True)
r = d.solve_full(good, SolverConfig()); print("good", r.report.status, r.report.cg_iterations, flush=True)
r = d.solve_full(bad, SolverConfig()); print(r.report.status, flush=True)
