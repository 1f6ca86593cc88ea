"""Synthetic ACOPF-shaped ("ACTIVSg-grid sparsity") block-4x4 KKT systems.

The reference generator (proj/core/src/generator.cpp:46-82) draws random
expander graphs whose Cholesky fill explodes with size (SURVEY.md finding 2),
so the benchmark configs use this grid-shaped construction instead
(SURVEY.md Appendix B):

* nb buses on a ceil(sqrt(nb))-wide lattice; branches = a random spanning
  tree over lattice-neighbour edges plus further shuffled lattice edges until
  nbr = round(1.3 nb); ng = nb // 5 generators at buses 5g.
* primal variables (n_x = 2 nb + 4 nbr + 2 ng): (V_m, V_a) per bus,
  (P_f, Q_f, P_t, Q_t) per branch, (P_g, Q_g) per generator.
* J (m_c = 2 nb + 4 nbr): 4 flow-definition rows per branch (+1 on the flow,
  U(-1,1) on the 4 end-bus voltages); 2 balance rows per bus (-1 on incident
  flows, +1 on the bus generator).
* J_d (m_d = 2 nbr): 2 thermal-limit rows per branch, U(-1,1) on (P_f, Q_f)
  and on (P_t, Q_t).
* H: a 4x4 block of U(-1,1) over each branch's end-bus voltages (coinciding
  entries summed), U(-0.1, 0.1) couplings inside (P_f,Q_f) and (P_t,Q_t);
  diagonal = row sum of |off-diagonals| (bus variables) + U(0.1, 1.0).
* D_x, D_s ~ U(0.1, 1.1); right-hand sides ~ U(-1, 1).
* sequences drift values by `drift` per step with the semantics of
  generator.cpp:197-210 (x *= 1 + drift U(-1,1); diagonals clamped at 1e-6).

Topology depends only on `topo_seed`; values only on `value_seed`, so a
batch of systems on one shared pattern is `value_seed = seed + b`
(SURVEY.md §8(d)).  Sizes: nb = 500 / 2000 / 10000 / 70000 give the configs
C1-C4 (N = 10k / 40k / 200k / 1.4M).
"""
from __future__ import annotations

import functools
import math

import numpy as np

from .kkt import BlockKkt4x4, CscMatrix

CONFIG_BUSES = {"C1": 500, "C2": 2000, "C3": 10000, "C4": 70000}


@functools.lru_cache(maxsize=8)
def _topology(nb: int, seed: int, branch_ratio: float):
    rng = np.random.default_rng(seed)
    w = int(math.ceil(math.sqrt(nb)))
    b = np.arange(nb)
    right = b[((b % w) + 1 < w) & (b + 1 < nb)]
    down = b[b + w < nb]
    cand = np.concatenate([np.stack([right, right + 1], 1), np.stack([down, down + w], 1)])
    cand = cand[rng.permutation(len(cand))]
    parent = list(range(nb))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    tree, rest = [], []
    for e, (u, v) in enumerate(cand.tolist()):
        ru, rv = find(u), find(v)
        if ru != rv:
            parent[ru] = rv
            tree.append(e)
        else:
            rest.append(e)
    nbr_target = max(len(tree), int(round(branch_ratio * nb)))
    chosen = tree + rest[: max(0, nbr_target - len(tree))]
    br = cand[np.sort(np.array(chosen, dtype=np.int64))]
    br = br[np.lexsort((br[:, 1], br[:, 0]))]
    return br[:, 0].astype(np.int64), br[:, 1].astype(np.int64)


def generate(nb: int, topo_seed: int = 7, value_seed: int | None = None,
             branch_ratio: float = 1.3) -> BlockKkt4x4:
    if nb < 4:
        raise ValueError("need at least 4 buses")
    fb, tb = _topology(nb, topo_seed, branch_ratio)
    nbr = fb.size
    ng = nb // 5
    gbus = 5 * np.arange(ng, dtype=np.int64)
    n_x = 2 * nb + 4 * nbr + 2 * ng
    m_c = 2 * nb + 4 * nbr
    m_d = 2 * nbr
    rng = np.random.default_rng(topo_seed * 1_000_003 + 11 if value_seed is None else value_seed)
    U = rng.uniform

    vm = lambda bus: 2 * bus
    va = lambda bus: 2 * bus + 1
    e = np.arange(nbr, dtype=np.int64)
    pf, qf, pt, qt = 2 * nb + 4 * e, 2 * nb + 4 * e + 1, 2 * nb + 4 * e + 2, 2 * nb + 4 * e + 3
    pg, qg = 2 * nb + 4 * nbr + 2 * np.arange(ng), 2 * nb + 4 * nbr + 2 * np.arange(ng) + 1

    # ---- H (lower) ----------------------------------------------------------
    blk_r = np.stack([va(fb), vm(tb), vm(tb), va(tb), va(tb), va(tb)], 1)
    blk_c = np.stack([vm(fb), vm(fb), va(fb), vm(fb), va(fb), vm(tb)], 1)
    blk_v = U(-1.0, 1.0, size=(nbr, 6))
    cpl_r = np.stack([qf, qt], 1)
    cpl_c = np.stack([pf, pt], 1)
    cpl_v = U(-0.1, 0.1, size=(nbr, 2))
    off = CscMatrix.from_triplets(n_x, n_x, np.concatenate([blk_r.ravel(), cpl_r.ravel()]),
                                  np.concatenate([blk_c.ravel(), cpl_c.ravel()]),
                                  np.concatenate([blk_v.ravel(), cpl_v.ravel()]))
    absrow = np.zeros(n_x)
    oc = off.col_of_entries()
    np.add.at(absrow, off.rowidx, np.abs(off.values))
    np.add.at(absrow, oc, np.abs(off.values))
    absrow[2 * nb:] = 0.0  # flow / generator variables: only the U(0.1, 1) term
    diag = absrow + U(0.1, 1.0, size=n_x)
    h = CscMatrix.from_triplets(n_x, n_x, np.concatenate([off.rowidx, np.arange(n_x)]),
                                np.concatenate([oc, np.arange(n_x)]),
                                np.concatenate([off.values, diag]))

    # ---- J --------------------------------------------------------------------
    rows, cols, vals = [], [], []
    flows = np.stack([pf, qf, pt, qt], 1)              # nbr x 4
    volt = np.stack([vm(fb), va(fb), vm(tb), va(tb)], 1)  # nbr x 4
    fr = 4 * e[:, None] + np.arange(4)[None, :]          # flow rows
    rows += [fr.ravel()]
    cols += [flows.ravel()]
    vals += [np.ones(4 * nbr)]
    rows += [np.repeat(fr.ravel(), 4)]
    cols += [np.repeat(volt, 4, axis=0).ravel()]
    vals += [U(-1.0, 1.0, size=16 * nbr)]
    base = 4 * nbr
    rows += [base + 2 * fb, base + 2 * fb + 1, base + 2 * tb, base + 2 * tb + 1]
    cols += [pf, qf, pt, qt]
    vals += [-np.ones(nbr)] * 4
    rows += [base + 2 * gbus, base + 2 * gbus + 1]
    cols += [pg, qg]
    vals += [np.ones(ng)] * 2
    j = CscMatrix.from_triplets(m_c, n_x, np.concatenate(rows), np.concatenate(cols),
                                np.concatenate(vals))

    # ---- J_d ------------------------------------------------------------------
    jd = CscMatrix.from_triplets(m_d, n_x,
                                 np.concatenate([2 * e, 2 * e, 2 * e + 1, 2 * e + 1]),
                                 np.concatenate([pf, qf, pt, qt]),
                                 U(-1.0, 1.0, size=4 * nbr))

    return BlockKkt4x4(
        h=h, j=j, j_d=jd,
        d_x=U(0.1, 1.1, size=n_x), d_s=U(0.1, 1.1, size=m_d),
        r_tilde_x=U(-1.0, 1.0, size=n_x), r_s=U(-1.0, 1.0, size=m_d),
        r_y=U(-1.0, 1.0, size=m_c), r_yd=U(-1.0, 1.0, size=m_d))


def drift(sys: BlockKkt4x4, amount: float, seed: int) -> BlockKkt4x4:
    """Next matrix of an IPM-like sequence: same pattern, values perturbed
    (generator.cpp:197-210, :383-404)."""
    rng = np.random.default_rng(seed)

    def d(v, clamp=0.0):
        out = v * (1.0 + amount * rng.uniform(-1.0, 1.0, size=v.shape))
        if clamp > 0.0:
            out = np.maximum(out, clamp)
        return out

    return BlockKkt4x4(
        h=sys.h.with_values(d(sys.h.values)), j=sys.j.with_values(d(sys.j.values)),
        j_d=sys.j_d.with_values(d(sys.j_d.values)), d_x=d(sys.d_x, 1e-6), d_s=d(sys.d_s, 1e-6),
        r_tilde_x=d(sys.r_tilde_x), r_s=d(sys.r_s), r_y=d(sys.r_y), r_yd=d(sys.r_yd))


def sequence(nb: int, length: int, seed: int = 7, amount: float = 0.01) -> list[BlockKkt4x4]:
    out = [generate(nb, seed, seed)]
    for k in range(1, length):
        out.append(drift(out[-1], amount, seed * 7919 + k))
    return out


def batch(nb: int, count: int, seed: int = 7) -> list[BlockKkt4x4]:
    """`count` independent systems on one pattern (value seed = seed + b)."""
    return [generate(nb, seed, seed + b) for b in range(count)]
