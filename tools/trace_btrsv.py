"""Trace one batched H^-1 pass (diagnostics): per CTA job start/end times."""
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
bt = Batch(dev); bt.upload(stack_values(systems))
for _ in range(2):
    bt.solve_resident(SolverConfig(), timing=True)
print("batch timing", {k: round(v, 2) for k, v in dev.timing().items()})
info = dev.info(); ns = info["n_supernodes"]
Bp = max(32, 1 << (B - 1).bit_length()); T = Bp // 32
L = _lib.lib(); I32P = C.POINTER(C.c_int32)
L.hykkt_debug_btrsv_trace.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
L.hykkt_debug_batch_jobs.argtypes = [C.c_void_p, I32P, I32P, C.POINTER(C.c_uint8), I32P]
L.hykkt_debug_plan.argtypes = [C.c_void_p, I32P, I32P, I32P, I32P]
nj = C.c_int64(0)
_lib.check(L.hykkt_debug_btrsv_trace(dev.h, None, C.byref(nj)))
nj = nj.value
jp = np.zeros(nj + 1, np.int32); kind = np.zeros(nj, np.uint8); mode = np.zeros(ns, np.int32)
_lib.check(L.hykkt_debug_batch_jobs(dev.h, jp.ctypes.data_as(I32P), None, kind.ctypes.data_as(C.POINTER(C.c_uint8)), mode.ctypes.data_as(I32P)))
items = np.zeros(jp[-1], np.int32)
_lib.check(L.hykkt_debug_batch_jobs(dev.h, None, items.ctypes.data_as(I32P), None, None))
order = np.zeros(ns, np.int32); first = np.zeros(ns + 1, np.int32); nrows = np.zeros(ns, np.int32); parent = np.zeros(ns, np.int32)
_lib.check(L.hykkt_debug_plan(dev.h, *[a.ctypes.data_as(I32P) for a in (order, first, nrows, parent)]))
out = np.zeros(2 * nj, np.uint64)
for _ in range(3):
    _lib.check(L.hykkt_debug_btrsv_trace(dev.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), None))
end, start = out[:nj].astype(np.int64), out[nj:].astype(np.int64)
t0 = start.min(); end = (end - t0) / 1e3; start = (start - t0) / 1e3
dur = end - start
w = np.diff(first)
print(f"jobs {nj}: lane {int((kind==0).sum())} wide-fwd {int((kind==1).sum())} wide-bwd {int((kind==2).sum())}; wide supernodes {int(mode.sum())} of {ns}")
print("pass us %.1f" % end.max())
for k, name in [(0, "lane"), (1, "wide fwd"), (2, "wide bwd")]:
    m = kind == k
    if m.any():
        print(f"{name:9s}: start {start[m].min():8.1f}..{start[m].max():8.1f}  end max {end[m].max():8.1f}  dur mean {dur[m].mean():6.1f} max {dur[m].max():7.1f}")
nlane_f = None
# lane forward jobs = kind 0 jobs whose first item < ns*T
lf = (kind == 0) & (items[jp[:-1]] < ns * T)
print("lane fwd end %.1f  lane bwd start %.1f" % (end[lf].max(), start[(kind == 0) & ~lf].min() if ((kind == 0) & ~lf).any() else -1))
# per wide supernode: mean fwd / bwd duration
for k, name in [(1, "fwd"), (2, "bwd")]:
    m = np.flatnonzero(kind == k)
    sn = items[jp[m]] // Bp
    rows = []
    for s in np.unique(sn):
        mm = m[sn == s]
        rows.append((dur[mm].mean(), s, start[mm].min(), end[mm].max()))
    rows.sort(reverse=True)
    print(f"wide {name} supernodes by mean job us: sn w nr mean first_start last_end")
    for d, s, a, e in rows[:10]:
        print(f"  {s:6d} {w[s]:4d} {nrows[s]:4d} {d:7.1f} {a:8.1f} {e:8.1f}")
