"""Per-level work of the analysed supernode tree (host only): how many
supernodes, widths, forward row-gather entries and panel sizes per level --
the input for choosing the per-system solve's task modes."""
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
out = np.zeros(8 * s.n_x)
L.hykkt_debug_host_sn_stats.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 7 + [C.POINTER(C.c_int64), C.c_void_p]
_lib.check(L.hykkt_debug_host_sn_stats(s.n_x, s.m_c, s.m_d, *[ip(x) for x in a], None, C.byref(ns), out.ctypes.data))
st = out[:8 * ns.value].reshape(-1, 8)
w, nr, lev, nu, uf, df, ge, par = st.T
tri = w * (w + 1) / 2
pan = w * nr
print(f"n {s.n_x} nsup {ns.value} nnzL {int(pan.sum() - (w*(w-1)/2).sum())} fwd-gather {int(ge.sum())} tri {int(tri.sum())}")
print("lev  nsup  sum_w max_w  max_nr  gather  max_gather_per_sn  tri  panel  nsn(w>4)")
for l in range(int(lev.max()) + 1):
    m = lev == l
    print(f"{l:3d} {m.sum():5d} {int(w[m].sum()):6d} {int(w[m].max()):4d} {int(nr[m].max()):5d} {int(ge[m].sum()):7d} "
          f"{int(ge[m].max()):6d} {int(tri[m].sum()):6d} {int(pan[m].sum()):7d} {int((w[m]>4).sum()):4d}")
