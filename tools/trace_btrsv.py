"""Trace one batched H^-1 pass (diagnostics): where does the time go?"""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib
from paper_2110_03636_b200.solver import Batch, stack_values

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
systems = acopf.batch(nb, B, seed=7)
dev = Device(0); dev.analyze(systems[0])
bt = Batch(dev); bt.upload(stack_values(systems)); bt.solve_resident(SolverConfig(), timing=True)
print("batch timing", {k: round(v, 2) for k, v in dev.timing().items()})
info = dev.info(); ns = info["n_supernodes"]; T = max(1, (1 << (max(B, 32) - 1).bit_length()) // 32)
L = _lib.lib(); I32P = C.POINTER(C.c_int32)
L.hykkt_debug_btrsv_trace.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
L.hykkt_debug_plan.argtypes = [C.c_void_p, I32P, I32P, I32P, I32P]
order = np.zeros(ns, np.int32); first = np.zeros(ns + 1, np.int32); nrows = np.zeros(ns, np.int32); parent = np.zeros(ns, np.int32)
_lib.check(L.hykkt_debug_plan(dev.h, *[a.ctypes.data_as(I32P) for a in (order, first, nrows, parent)]))
nt = ns * T
out = np.zeros(4 * nt, np.uint64)
for _ in range(2):
    _lib.check(L.hykkt_debug_btrsv_trace(dev.h, out.ctypes.data_as(C.POINTER(C.c_uint64))))
end, start = out[:2 * nt].astype(np.int64), out[2 * nt:].astype(np.int64)
t0 = start.min(); end = (end - t0) / 1e3; start = (start - t0) / 1e3
dur = end - start
width = np.diff(first)
print("pass us %.1f  fwd done %.1f" % (end.max(), end[:nt].max()))
sn_of_task = np.concatenate([order[np.arange(nt) // T], order[(2 * nt - 1 - np.arange(nt, 2 * nt)) // T]])
work = (width * nrows)[sn_of_task]
for lo, hi in [(0, 64), (64, 256), (256, 1024), (1024, 4096), (4096, 1 << 30)]:
    m = (work >= lo) & (work < hi)
    if m.any():
        print("w*nr in [%d,%d): tasks %d  dur us mean %.1f max %.1f  sum %.0f" % (lo, hi, m.sum(), dur[m].mean(), dur[m].max(), dur[m].sum()))
q = np.linspace(0, nt - 1, 10).astype(int)
print("fwd end at order quantiles:", [round(end[i], 1) for i in q])
print("bwd end at order quantiles:", [round(end[nt + i], 1) for i in q])
print("task start max %.1f" % start.max())
# forward critical path for tile 0 (root first)
fend = np.zeros(ns); fstart = np.zeros(ns)
for t in range(nt):
    if t % T == 0:
        fend[order[t // T]] = end[t]; fstart[order[t // T]] = start[t]
kids = [[] for _ in range(ns)]
for k in range(ns):
    if parent[k] >= 0: kids[parent[k]].append(k)
node = int(np.argmax(fend)); path = []
while True:
    path.append(node)
    if not kids[node]: break
    node = max(kids[node], key=lambda c: fend[c])
print("tile0 fwd critical path: sn w nr nchild start childend end own_us")
tot = 0
for k in path[:14]:
    ce = max([fend[c] for c in kids[k]], default=fstart[k])
    tot += fend[k] - ce
    print("  %6d %4d %4d %3d %9.1f %9.1f %9.1f %8.1f" % (k, width[k], nrows[k], len(kids[k]), fstart[k], ce, fend[k], fend[k] - ce))
