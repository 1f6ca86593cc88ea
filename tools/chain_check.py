"""Compare one H^-1 pass with and without the chains' register hand-off
(first differing supernode in y / x)."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib
from paper_2110_03636_b200._lib import i64, ip

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
L = _lib.lib()
L.hykkt_debug_trsv_vectors.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
res = {}
for regs in ("0", "1"):
    os.environ["HYKKT_TRSV_CHAINS"] = "1"
    os.environ["HYKKT_TRSV_CHAIN_REGS"] = regs
    dev = Device(0); dev.analyze(s); dev.upload(s)
    try:
        dev.solve_resident(SolverConfig())
    except Exception as e:
        print("solve", regs, e)
    y = np.zeros(s.n_x); x = np.zeros(s.n_x)
    _lib.check(L.hykkt_debug_trsv_vectors(dev.h, y.ctypes.data, x.ctypes.data))
    res[regs] = (y, x)
    ns = dev.info()["n_supernodes"]
    I32P = C.POINTER(C.c_int32)
    L.hykkt_debug_plan.argtypes = [C.c_void_p, I32P, I32P, I32P, I32P]
    order = np.zeros(ns, np.int32); first = np.zeros(ns + 1, np.int32); nrows = np.zeros(ns, np.int32); parent = np.zeros(ns, np.int32)
    _lib.check(L.hykkt_debug_plan(dev.h, *[a.ctypes.data_as(I32P) for a in (order, first, nrows, parent)]))
    dev.close()
for k, nm in ((0, "y"), (1, "x")):
    a, b = res["0"][k], res["1"][k]
    bad = np.where(~np.isclose(a, b, rtol=1e-10, atol=1e-14))[0]
    print(nm, "differing entries", len(bad))
    if len(bad):
        cols = set(bad.tolist())
        col2sn = np.searchsorted(first, np.arange(s.n_x), side="right") - 1
        sns = sorted(set(col2sn[bad].tolist()), key=lambda t: list(order).index(t) if k == 0 else -list(order).index(t))
        for t in sns[:8]:
            w = first[t + 1] - first[t]
            print(f"  sn {t} w {w} nr {nrows[t]} parent {parent[t]} a {a[first[t]:first[t+1]]} b {b[first[t]:first[t+1]]}")
