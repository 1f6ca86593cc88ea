import sys; sys.path.insert(0, '.')
import numpy as np
from oracle import ref
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values
systems = acopf.batch(120, 4, seed=7)
cfg = SolverConfig()
perm = ref.hgamma_amd(systems[0], cfg)
dev = Device(0); dev.analyze(systems[0], perm)
b = Batch(dev); b.upload(stack_values(systems)); reps = b.solve_resident(cfg); out = b.download()
for k, s in enumerate(systems):
    want = ref.solve_full(s, cfg, perm)
    single = Device(0); single.analyze(s, perm); g1 = single.solve_full(s, cfg)
    for name in ["dx", "ds", "dy", "dyd"]:
        w = getattr(want, name); got = out[name][k]; sg = getattr(g1.solution, name)
        print(k, name, "batch err %.2e" % (np.linalg.norm(got - w) / np.linalg.norm(w)), "single err %.2e" % (np.linalg.norm(sg - w) / np.linalg.norm(w)))
    print(k, reps[k].status, reps[k].cg_iterations, want.report["cg_iterations"], reps[k].ruiz_iterations, want.report["ruiz_iterations"], reps[k].factorization_attempts)
