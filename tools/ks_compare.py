"""Batched solve of B ACOPF-shaped systems with per-phase device timing;
saves reports + solutions to /tmp/<tag>.npz so the lane-per-system
(HYKKT_BATCH_PATH=lane) and system-per-CTA paths can be compared."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf
from paper_2110_03636_b200.solver import Batch, stack_values

nb, B, reps, tag = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
systems = acopf.batch(nb, B, seed=7)
dev = Device(0)
dev.analyze(systems[0])
bt = Batch(dev)
bt.upload(stack_values(systems))
for i in range(reps):
    r = bt.solve_resident(SolverConfig(), timing=True)
    print(tag, {k: round(v, 3) for k, v in dev.timing().items()}, flush=True)
sol = bt.download()
its = np.array([x.cg_iterations for x in r])
st = np.array([int(x.status) for x in r])
print(tag, "cg its max", its.max(), "mean", its.mean(), "status", np.bincount(st))
np.savez(f"/tmp/{tag}.npz", its=its, status=st, **sol)
import ctypes as C, os
if os.environ.get("HYKKT_KS_PROF"):
    from paper_2110_03636_b200 import _lib
    L = _lib.lib()
    n = C.c_int64(0)
    buf = np.zeros(1024 * 16, np.uint64)
    tr = np.zeros(100000, np.uint64)
    L.hykkt_debug_ks_prof.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
    _lib.check(L.hykkt_debug_ks_prof(dev.h, buf.ctypes.data, C.byref(n), tr.ctypes.data))
    ns_ = C.c_int64(0)
    L.hykkt_debug_ks_program.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    _lib.check(L.hykkt_debug_ks_program(dev.h, None, C.byref(ns_)))
    steps = np.zeros(8 * ns_.value, np.int32)
    _lib.check(L.hykkt_debug_ks_program(dev.h, steps.ctypes.data, C.byref(ns_)))
    steps = steps.reshape(-1, 8)
    t = tr[:ns_.value + 1].astype(np.int64)
    print("step trace (CTA 0, first CG operator): k kind ilen vlen h3 h4 h5 h6 maxw ns")
    prev = None
    for k in range(ns_.value):
        dt = t[k] - prev if prev is not None and t[k] and prev else 0
        prev = t[k] if t[k] else prev
        print("  %4d %d %6d %6d %5d %5d %5d %d %3d %8d" % (k, *steps[k], dt))
    pr = buf[:16 * n.value].reshape(-1, 16).astype(np.float64)
    names = ["JT", "wait", "A", "B", "prod", "sum2", "upd", "pupd", "recover", "steps", "solves", "iters", "J", "sync"]
    tot = pr[:, :4].sum(1) + pr[:, 5:9].sum(1) + pr[:, 12] + pr[:, 13]
    print("CTAs", n.value, "mean busy ms", tot.mean() / 1e6, "max", tot.max() / 1e6)
    for i, nm in enumerate(names):
        col = pr[:, i]
        if i < 9 or i >= 12:
            print(f"  {nm:8s} mean ms {col.mean()/1e6:8.3f}  share {col.sum()/tot.sum():.3f}")
        else:
            print(f"  {nm:8s} mean {col.mean():10.1f}")
    it = pr[:, 11].sum(); so = pr[:, 10].sum(); stp = pr[:, 9].sum()
    print("  per solve us: wait %.2f A %.2f B %.2f sync %.2f (producer busy %.2f); per step ns: %.0f" % (
        pr[:, 1].sum() / so / 1e3, pr[:, 2].sum() / so / 1e3, pr[:, 3].sum() / so / 1e3, pr[:, 13].sum() / so / 1e3,
        pr[:, 4].sum() / so / 1e3, (pr[:, 1:4].sum() + pr[:, 13].sum() + pr[:, 0].sum() + pr[:, 12].sum()) / stp))
    print("  per CG iteration us: JT %.2f J %.2f sum2 %.2f upd %.2f pupd %.2f" % tuple(pr[:, i].sum() / it / 1e3 for i in (0, 12, 5, 6, 7)))
