"""Per-level times of the cluster solve's last H^-1 pass (HYKKT_CL_STAMPS)."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["HYKKT_CLUSTER"] = "1"
os.environ["HYKKT_CL_STAMPS"] = "1"
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib

for name in sys.argv[1].split(","):
    s = acopf.generate(acopf.CONFIG_BUSES[name], 7, 7)
    dev = Device(0); dev.analyze(s); dev.upload(s)
    dev.solve_resident(SolverConfig())
    L = _lib.lib()
    L.hykkt_debug_cluster_stamps.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    nl = C.c_int64(0)
    out = np.zeros(8192, np.uint64); sz = np.zeros(8192, np.int32)
    _lib.check(L.hykkt_debug_cluster_stamps(dev.h, out.ctypes.data, sz.ctypes.data, 8192, C.byref(nl)))
    n = nl.value
    t = out[:2 * n].astype(np.int64)
    dt = np.diff(t) / 1e3
    sz = sz[:4 * n].reshape(n, 4)
    print(f"{name}: levels {n} fwd {(t[n-1]-t[0])/1e3:.1f} us  bwd {(t[2*n-1]-t[n-1])/1e3:.1f} us")
    for i in range(1, 2 * n):
        l = i if i < n else 2 * n - 1 - i
        print(f"  {'F' if i < n else 'B'} lev {l:3d} thr {sz[l,0]:6d} warp {sz[l,1]:5d} cta {sz[l,2]:3d}  {dt[i-1]:7.2f} us")
    ws = out[2 * n:2 * n + 768].astype(np.int64).reshape(2, 64, 6)
    for d, nm in ((0, "fwd"), (1, "bwd")):
        print(f"  warp 0 tasks ({nm}): issue, wait, gathers, chain, end, gap to next start (ns)")
        for i in range(64):
            r = ws[d, i]
            if r[0] == 0: break
            nxt = ws[d, i + 1, 0] - r[5] if i + 1 < 64 and ws[d, i + 1, 0] else 0
            print(f"    {i:3d} " + " ".join(f"{r[j+1]-r[j]:6d}" for j in range(5)) + f" {nxt:7d}")
    dev.close()
