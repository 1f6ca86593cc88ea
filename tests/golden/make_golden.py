"""Regenerates tests/golden/*.npz from the compiled reference (oracle/_ref,
built from /root/reference by oracle/Makefile).  Run in the build container
(where /root/reference exists):  python tests/golden/make_golden.py

Each fixture holds the inputs of one block-4x4 system, the reference AMD
ordering of its H_gamma pattern, and the reference solve_full outputs and
report — the known answers the GPU path and the C restatement are checked
against when the reference itself is not available (GPU box)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_2110_03636_b200 import SolverConfig, acopf  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, builder, config overrides) — reference test instances
# (tests/test_hybrid_solver.cpp seeds) plus small ACOPF-shaped ones.
CASES = [
    ("ref_n240_s23", lambda: ref.generate(240, 60, 50, seed=23)[0], {}),           # :335-342
    ("ref_n60_s31", lambda: ref.generate(60, 15, 12, seed=31)[0], {}),             # :363-379
    ("ref_n40_s37", lambda: ref.generate(40, 10, 8, seed=37)[0], {}),              # :381-392
    ("ref_rankdef_s7", lambda: ref.generate(30, 8, 6, klass=2, seed=7)[0], {}),    # :291-305
    ("ref_inconsistent_s8", lambda: ref.generate(30, 8, 6, klass=3, seed=8)[0], {}),  # :307-315
    ("ref_indefinite_s44", lambda: ref.generate(40, 10, 8, klass=1, seed=44)[0], {}),  # :415-440
    ("ref_cgcap_s59", lambda: ref.generate(40, 10, 8, seed=59)[0],
     {"cg_max_iter": 1, "cg_tol": 1e-15, "gamma": 1.0}),                              # :485-496
    ("acopf_nb60", lambda: acopf.generate(60, 7, 7), {}),
    ("acopf_nb120_g1e2", lambda: acopf.generate(120, 7, 7), {"gamma": 1e2}),
    ("acopf_nb120_g1e8", lambda: acopf.generate(120, 7, 7), {"gamma": 1e8}),
]


def main():
    for name, build, over in CASES:
        s = build()
        cfg = SolverConfig(**over)
        perm = ref.hgamma_amd(s, cfg)
        r = ref.solve_full(s, cfg, perm)
        rep = {k: np.array(v) for k, v in r.report.items()}
        np.savez_compressed(
            OUT / f"{name}.npz",
            n_x=s.n_x, m_c=s.m_c, m_d=s.m_d,
            h_cp=s.h.colptr, h_ri=s.h.rowidx, h_v=s.h.values,
            j_cp=s.j.colptr, j_ri=s.j.rowidx, j_v=s.j.values,
            jd_cp=s.j_d.colptr, jd_ri=s.j_d.rowidx, jd_v=s.j_d.values,
            d_x=s.d_x, d_s=s.d_s, r_tilde_x=s.r_tilde_x, r_s=s.r_s, r_y=s.r_y, r_yd=s.r_yd,
            perm=perm, dx=r.dx, ds=r.ds, dy=r.dy, dyd=r.dyd,
            cfg_keys=np.array(list(over.keys()), dtype="U32"),
            cfg_vals=np.array(list(over.values()), dtype=np.float64),
            **{"rep_" + k: v for k, v in rep.items()})
        print(name, r.report["status"], r.report["cg_iterations"])


if __name__ == "__main__":
    main()
