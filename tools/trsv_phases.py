"""Phase breakdown of one grid-wide H^-1 pass (k_trsv) on C1-C4."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib

for name in sys.argv[1].split(","):
    s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
    dev = Device(0); dev.analyze(s); dev.upload(s)
    dev.solve_resident(SolverConfig())
    L = _lib.lib()
    L.hykkt_debug_trsv_phases.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    nb = C.c_int64(0)
    out = np.zeros(8 * 4096, np.uint64)
    for rep in range(3):
        _lib.check(L.hykkt_debug_trsv_phases(dev.h, out.ctypes.data, out.size, C.byref(nb)))
    t = out[:8 * nb.value].astype(np.int64).reshape(-1, 8)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    def st(col): return f"min {r[:, col].min():8.1f} med {np.median(r[:, col]):8.1f} max {r[:, col].max():8.1f}"
    print(f"{name}: blocks {nb.value}")
    for col, nm in ((0, "start"), (1, "rearm+sync"), (2, "fwd bottom/bins"), (3, "task loop exit"),
                    (4, "bwd bottom sync"), (5, "bwd bottom/bins"), (7, "end")):
        print(f"  {nm:18s} {st(col)}")
    dev.close()
