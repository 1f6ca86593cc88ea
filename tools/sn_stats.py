"""Per-supernode work of the analysed plan (host only, no GPU)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import acopf, _lib
from paper_2110_03636_b200._lib import i64, ip

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
s = acopf.generate(nb, 7, 7)
L = _lib.lib()
a = [i64(x) for x in (s.h.colptr, s.h.rowidx, s.j.colptr, s.j.rowidx, s.j_d.colptr, s.j_d.rowidx)]
ns = C.c_int64(0)
out = np.zeros(6 * s.n_x)
L.hykkt_debug_host_sn_stats.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 7 + [C.POINTER(C.c_int64), C.c_void_p]
_lib.check(L.hykkt_debug_host_sn_stats(s.n_x, s.m_c, s.m_d, *[ip(x) for x in a], None, C.byref(ns), out.ctypes.data))
st = out[:6 * ns.value].reshape(-1, 6)
w, nr, lev, nu, uf, df = st.T
print(f"nsup {ns.value} levels {int(lev.max())+1} total update FMAs {uf.sum():.3e} dense {df.sum():.3e}")
top = np.argsort(-(uf + df))[:15]
print("top supernodes by work: w nr level nupd upd_fma dense_fma")
for k in top:
    print(f"  {k:6d} {int(w[k]):4d} {int(nr[k]):4d} {int(lev[k]):3d} {int(nu[k]):5d} {uf[k]:10.0f} {df[k]:9.0f}")
# critical path by work (sum along root path of max child)
par = None
