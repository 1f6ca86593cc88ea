"""Phase breakdown of the single-system CG kernel (k_cg): per-CTA stamps of
the last iteration of one run on the factored system (hykkt_debug_cg_phases):
pass (bottom levels, task loop, backward bottom), J product + dots, x / r
update, and the grid barriers between them.  usage: cg_phases.py C4[,C2...]"""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib

for name in sys.argv[1].split(","):
    s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
    dev = Device(0); dev.analyze(s); dev.upload(s)
    dev.solve_resident(SolverConfig())
    L = _lib.lib()
    L.hykkt_debug_cg_phases.argtypes = [C.c_void_p, C.POINTER(_lib.Config), C.c_void_p, C.c_int64,
                                        C.POINTER(C.c_int64)]
    cfg = _lib.Config(); L.hykkt_config_default(C.byref(cfg))
    nb = C.c_int64(0)
    out = np.zeros(16 * 4096, np.uint64)
    for rep in range(3):
        _lib.check(L.hykkt_debug_cg_phases(dev.h, C.byref(cfg), out.ctypes.data, out.size, C.byref(nb)))
    n = nb.value
    t = np.hstack([out[:8 * n].astype(np.int64).reshape(n, 8), out[8 * n:16 * n].astype(np.int64).reshape(n, 8)])
    t0 = t[:, 8].min()
    r = (t - t0) / 1e3
    def st(col): return f"min {r[:, col].min():8.1f} med {np.median(r[:, col]):8.1f} max {r[:, col].max():8.1f}"
    print(f"{name}: blocks {nb.value} (last CG iteration, us from its start)")
    for col, nm in ((8, "iteration start"), (2, "fwd bottom done"), (3, "task loop exit"), (5, "bwd bottom done"),
                    (9, "pass end"), (10, "barrier"), (11, "J product + dots"), (12, "barrier"),
                    (13, "rearm + x, r"), (14, "barrier")):
        print(f"  {nm:18s} {st(col)}")
    dev.close()
