"""Loads tests/golden/*.npz fixtures (inputs + reference outputs)."""
from pathlib import Path

import numpy as np

from paper_2110_03636_b200 import SolverConfig
from paper_2110_03636_b200.kkt import BlockKkt4x4, CscMatrix

GOLDEN = Path(__file__).resolve().parent / "golden"
NAMES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    nx, mc, md = int(z["n_x"]), int(z["m_c"]), int(z["m_d"])
    s = BlockKkt4x4(
        h=CscMatrix(nx, nx, z["h_cp"], z["h_ri"], z["h_v"]),
        j=CscMatrix(mc, nx, z["j_cp"], z["j_ri"], z["j_v"]),
        j_d=CscMatrix(md, nx, z["jd_cp"], z["jd_ri"], z["jd_v"]),
        d_x=z["d_x"], d_s=z["d_s"], r_tilde_x=z["r_tilde_x"], r_s=z["r_s"], r_y=z["r_y"], r_yd=z["r_yd"])
    cfg = SolverConfig()
    for k, v in zip(z["cfg_keys"], z["cfg_vals"]):
        setattr(cfg, str(k), int(v) if str(k) in ("cg_max_iter", "ruiz_max_iters") else float(v))
    want = dict(dx=z["dx"], ds=z["ds"], dy=z["dy"], dyd=z["dyd"],
                report={k[4:]: z[k].item() for k in z.files if k.startswith("rep_")})
    return s, cfg, z["perm"], want


def stacked(w):
    return np.concatenate([w["dx"], w["ds"], w["dy"], w["dyd"]])
