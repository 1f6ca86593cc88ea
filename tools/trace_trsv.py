"""Critical-path trace of one sync-free H^-1 pass (diagnostics)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
dev = Device(0); dev.analyze(s); dev.upload(s); dev.solve_resident(SolverConfig())
info = dev.info(); ns = info["n_supernodes"]
L = _lib.lib()
I32P = C.POINTER(C.c_int32)
L.hykkt_debug_trsv_trace.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
L.hykkt_debug_plan.argtypes = [C.c_void_p, I32P, I32P, I32P, I32P]
order = np.zeros(ns, np.int32); first = np.zeros(ns + 1, np.int32)
nrows = np.zeros(ns, np.int32); parent = np.zeros(ns, np.int32)
_lib.check(L.hykkt_debug_plan(dev.h, *[a.ctypes.data_as(I32P) for a in (order, first, nrows, parent)]))
out = np.zeros(6 * ns, np.uint64)
for _ in range(3):
    _lib.check(L.hykkt_debug_trsv_trace(dev.h, out.ctypes.data_as(C.POINTER(C.c_uint64))))
end, start, ready = out[:2 * ns].astype(np.int64), out[2 * ns:4 * ns].astype(np.int64), out[4 * ns:].astype(np.int64)
t0 = start[start > 0].min(); end = (end - t0) / 1e3; start = (start - t0) / 1e3; ready = np.where(ready > 0, (ready - t0) / 1e3, np.nan)
width = np.diff(first)
fend = np.zeros(ns); fstart = np.zeros(ns); bend = np.zeros(ns); bstart = np.zeros(ns); fready = np.zeros(ns); bready = np.zeros(ns)
fend[order] = end[:ns]; fstart[order] = start[:ns]; fready[order] = ready[:ns]; bready[order[::-1]] = ready[ns:]
bend[order[::-1]] = end[ns:]; bstart[order[::-1]] = start[ns:]
print(name, "nsup", ns, "pass us %.1f" % end.max(), "fwd done %.1f" % fend.max())
# walk the critical path of the forward pass from the root downward
root = int(np.argmax(fend))
kids = [[] for _ in range(ns)]
for k in range(ns):
    if parent[k] >= 0: kids[parent[k]].append(k)
node = root; path = []
while True:
    path.append(node)
    if not kids[node]: break
    node = max(kids[node], key=lambda c: fend[c])
print("forward critical path (root first): sn w nr start ready end dur detect(ready-childend) compute(end-ready)")
for k in path[:25]:
    ce = max([fend[c] for c in kids[k]], default=0)
    print("  %6d %4d %4d %8.1f %8.1f %8.1f %7.1f %7.2f %7.2f" % (k, width[k], nrows[k], fstart[k], fready[k], fend[k], fend[k] - max(fstart[k], ce), fready[k] - ce, fend[k] - fready[k]))
print("backward: root bwd start %.1f end %.1f; last bwd end %.1f" % (bstart[root], bend[root], bend.max()))
leaf = int(np.argmax(bend)); node = leaf; chain = []
while node >= 0: chain.append(node); node = parent[node]
print("backward chain of the last finisher (leaf first): sn w nr end dur_after_parent")
for k in chain[:25]:
    p = parent[k]
    pe = bend[p] if p >= 0 else fend[k]
    print("  %6d %4d %4d %8.1f %7.1f detect %7.2f compute %7.2f" % (k, width[k], nrows[k], bend[k], bend[k] - pe, bready[k] - pe, bend[k] - bready[k]))
# raw per-supernode times for offline analysis (tools/trace_levels.py)
import os
if os.environ.get("TRACE_NPZ"):
    np.savez_compressed(os.environ["TRACE_NPZ"], fstart=fstart, fready=fready, fend=fend, bstart=bstart,
                        bready=bready, bend=bend, width=width, nrows=nrows, parent=parent, order=order)
