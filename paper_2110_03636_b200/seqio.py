"""Sequence IO surface of the reference: the JSON
sequence manifest with Matrix Market blocks and vector files, the solve /
gamma-sweep CSV reports and the JSON run manifest, with the GPU path doing
the solves.  Files are byte-compatible with the reference's writers
(proj/docs/formats.md):

  read_matrix_market / write_matrix_market   proj/core/src/matrix_market.cpp
  load_sequence / save_sequence              proj/core/src/manifest.cpp
  cmd_solve / cmd_sweep_gamma                proj/core/src/driver.cpp:182-279
  RunManifest (to_json / from_json)          proj/core/src/driver.cpp:39-129, 141-180

Exit codes as proj/core/include/hkkt/driver.hpp:27-29: 0 all solved, 1 solve
failures present, 2 usage or input errors.  Command line:

  python -m paper_2110_03636_b200.seqio solve MANIFEST OUT_DIR [--gamma G]
  python -m paper_2110_03636_b200.seqio sweep-gamma MANIFEST OUT_DIR --gammas 1e2,1e4,...
"""
from __future__ import annotations

import json
import math
import os
import sys
from dataclasses import dataclass, field, fields
from pathlib import Path

import numpy as np

from .kkt import BlockKkt4x4, CscMatrix
from .solver import SequenceStats, SolveReport, SolverConfig, SolveStatus, is_success

EXIT_OK, EXIT_SOLVE_FAILURE, EXIT_USAGE = 0, 1, 2
SOLVE_CSV_SCHEMA = "# schema: hybrid-kkt-solve-v1"
SOLVE_CSV_HEADER = "k,delta1,delta2,cg_iterations,be_4x4,rr_4x4,be_2x2,rr_2x2,nnz_fac,ratio,status"
SWEEP_CSV_SCHEMA = "# schema: hybrid-kkt-sweep-v1"
SWEEP_CSV_HEADER = "gamma,k,cg_iterations,be_4x4,rr_4x4,delta1"

_STATUS_NAMES = {SolveStatus.kSolved: "solved", SolveStatus.kSolvedWithDelta2: "solved_delta2",
                 SolveStatus.kFailedDeltaMaxExceeded: "failed_delta_max",
                 SolveStatus.kFailedCgNoConvergence: "failed_cg"}
_STATUS_OF = {v: k for k, v in _STATUS_NAMES.items()}


class MatrixMarketError(ValueError):
    pass


class ManifestError(RuntimeError):
    pass


def fmt(v: float) -> str:
    """17 significant digits, as the reference's snprintf("%.17g")."""
    return "%.17g" % float(v)


def _dump(obj) -> str:
    """nlohmann::json::dump(1) layout: one-space indent, keys sorted, NaN as null."""
    def clean(o):
        if isinstance(o, float) and not math.isfinite(o):
            return None
        if isinstance(o, dict):
            return {k: clean(v) for k, v in o.items()}
        if isinstance(o, list):
            return [clean(v) for v in o]
        return o
    return json.dumps(clean(obj), indent=1, sort_keys=True, allow_nan=False) + "\n"


# ---- Matrix Market (matrix_market.cpp) -------------------------------------

def read_matrix_market(path) -> tuple[CscMatrix, bool]:
    """Coordinate / real / general or symmetric (lower triangle on disk),
    1-based on disk, duplicates summed.  Returns (matrix, symmetric)."""
    path = Path(path)
    try:
        lines = path.read_text().splitlines()
    except OSError as e:
        raise MatrixMarketError(f"cannot open {path}") from e
    if not lines:
        raise MatrixMarketError(f"{path}:1: empty file")
    head = lines[0].split()
    if len(head) < 5 or head[0] != "%%MatrixMarket":
        raise MatrixMarketError(f"{path}:1: missing banner")
    if head[1].lower() != "matrix" or head[2].lower() != "coordinate" or head[3].lower() != "real":
        raise MatrixMarketError(f"{path}:1: only 'matrix coordinate real' is supported")
    qual = head[4].lower()
    if qual not in ("general", "symmetric"):
        raise MatrixMarketError(f"{path}:1: unsupported qualifier {head[4]}")
    symmetric = qual == "symmetric"
    k = 1
    while k < len(lines) and (not lines[k].strip() or lines[k].lstrip().startswith("%")):
        k += 1
    if k >= len(lines):
        raise MatrixMarketError(f"{path}:{k + 1}: missing size line")
    try:
        nrows, ncols, nnz = (int(t) for t in lines[k].split()[:3])
    except ValueError as e:
        raise MatrixMarketError(f"{path}:{k + 1}: bad size line") from e
    if nrows < 0 or ncols < 0 or nnz < 0 or (symmetric and nrows != ncols):
        raise MatrixMarketError(f"{path}:{k + 1}: bad dimensions")
    rows = np.empty(nnz, np.int64)
    cols = np.empty(nnz, np.int64)
    vals = np.empty(nnz, np.float64)
    e = 0
    for ln in range(k + 1, len(lines)):
        s = lines[ln].strip()
        if not s or s.startswith("%"):
            continue
        if e == nnz:
            raise MatrixMarketError(f"{path}:{ln + 1}: more entries than declared")
        t = s.split()
        try:
            i, j, v = int(t[0]) - 1, int(t[1]) - 1, float(t[2])
        except (ValueError, IndexError) as err:
            raise MatrixMarketError(f"{path}:{ln + 1}: bad entry") from err
        if not (0 <= i < nrows and 0 <= j < ncols):
            raise MatrixMarketError(f"{path}:{ln + 1}: index out of range")
        if symmetric and i < j:
            raise MatrixMarketError(f"{path}:{ln + 1}: symmetric file stores an upper-triangle entry")
        rows[e], cols[e], vals[e] = i, j, v
        e += 1
    if e != nnz:
        raise MatrixMarketError(f"{path}: {e} entries, {nnz} declared")
    return CscMatrix.from_triplets(nrows, ncols, rows, cols, vals), symmetric


def write_matrix_market(path, a: CscMatrix, symmetric: bool) -> None:
    cols = a.col_of_entries()
    if symmetric and np.any(a.rowidx < cols):
        raise MatrixMarketError("symmetric write requires lower-triangle storage")
    out = [f"%%MatrixMarket matrix coordinate real {'symmetric' if symmetric else 'general'}",
           f"{a.nrows} {a.ncols} {a.nnz}"]
    out += [f"{i + 1} {j + 1} {fmt(v)}" for i, j, v in zip(a.rowidx.tolist(), cols.tolist(), a.values.tolist())]
    Path(path).write_text("\n".join(out) + "\n")


# ---- sequence manifest (manifest.cpp) ---------------------------------------

_VECTORS = (("D_x", "d_x"), ("D_s", "d_s"), ("r_tilde_x", "r_tilde_x"), ("r_s", "r_s"),
            ("r_y", "r_y"), ("r_yd", "r_yd"))


def load_sequence(manifest_path) -> tuple[list[BlockKkt4x4], bool]:
    """Systems listed by a manifest (paths relative to its directory) and
    whether they share the first system's block patterns."""
    manifest_path = Path(manifest_path)
    try:
        m = json.loads(manifest_path.read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise ManifestError(f"manifest {manifest_path}: {e}") from e
    if m.get("version") != 1 or not isinstance(m.get("systems"), list):
        raise ManifestError(f"manifest {manifest_path}: unsupported version or no systems list")
    base = manifest_path.parent
    systems = []
    for k, ent in enumerate(m["systems"]):
        try:
            n_x, m_c, m_d = int(ent["n_x"]), int(ent["m_c"]), int(ent["m_d"])
            h, hsym = read_matrix_market(base / ent["H"])
            j, _ = read_matrix_market(base / ent["J"])
            jd, _ = read_matrix_market(base / ent["J_d"])
            vec = json.loads((base / ent["vectors"]).read_text())
        except (KeyError, OSError, json.JSONDecodeError, MatrixMarketError) as e:
            raise ManifestError(f"system {k}: {e}") from e
        if not hsym:
            raise ManifestError(f"system {k}: H must use the symmetric qualifier")
        if (h.nrows, h.ncols) != (n_x, n_x) or (j.nrows, j.ncols) != (m_c, n_x) or (jd.nrows, jd.ncols) != (m_d, n_x):
            raise ManifestError(f"system {k}: block dimensions do not match the manifest")
        arrs = {}
        for key, attr in _VECTORS:
            if key not in vec:
                raise ManifestError(f"system {k}: vector {key} missing")
            arrs[attr] = np.asarray(vec[key], np.float64)
        want = {"d_x": n_x, "d_s": m_d, "r_tilde_x": n_x, "r_s": m_d, "r_y": m_c, "r_yd": m_d}
        for attr, n in want.items():
            if arrs[attr].shape != (n,):
                raise ManifestError(f"system {k}: vector {attr} has the wrong length")
        systems.append(BlockKkt4x4(h, j, jd, **arrs))
    uniform = all(s.same_pattern_as(systems[0]) for s in systems[1:])
    return systems, uniform


def save_sequence(out_dir, systems) -> Path:
    """Writes sys<k>_{H,J,Jd}.mtx, sys<k>_vectors.json and manifest.json."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    entries = []
    for k, s in enumerate(systems):
        stem = f"sys{k}"
        write_matrix_market(out_dir / f"{stem}_H.mtx", s.h, True)
        write_matrix_market(out_dir / f"{stem}_J.mtx", s.j, False)
        write_matrix_market(out_dir / f"{stem}_Jd.mtx", s.j_d, False)
        vec = {key: [float(x) for x in getattr(s, attr)] for key, attr in _VECTORS}
        (out_dir / f"{stem}_vectors.json").write_text(_dump(vec))
        entries.append({"n_x": s.n_x, "m_c": s.m_c, "m_d": s.m_d, "H": f"{stem}_H.mtx",
                        "J": f"{stem}_J.mtx", "J_d": f"{stem}_Jd.mtx", "vectors": f"{stem}_vectors.json"})
    path = out_dir / "manifest.json"
    path.write_text(_dump({"version": 1, "systems": entries}))
    return path


# ---- run manifest and CSV reports (driver.cpp) ------------------------------

def config_to_json(cfg: SolverConfig) -> dict:
    d = {f.name: getattr(cfg, f.name) for f in fields(cfg)}
    for k in ("gamma", "delta_min", "delta_max", "delta2", "cg_tol", "small_quadratic_threshold",
              "pivot_floor", "ruiz_tol"):
        d[k] = float(d[k])
    d["cg_max_iter"] = int(d["cg_max_iter"])
    d["ruiz_max_iters"] = int(d["ruiz_max_iters"])
    d["parallel_sequence"] = False  # the batch path replaces the thread pool
    return d


def config_from_json(d: dict) -> SolverConfig:
    return SolverConfig(**{f.name: d[f.name] for f in fields(SolverConfig)})


def report_to_json(r: SolveReport) -> dict:
    return {"status": _STATUS_NAMES[SolveStatus(r.status)], "delta1": float(r.delta1_final),
            "delta2": float(r.delta2_used), "cg_iterations": int(r.cg_iterations),
            "factorization_attempts": int(r.factorization_attempts), "be_4x4": float(r.be_4x4),
            "rr_4x4": float(r.rr_4x4), "be_2x2": float(r.be_2x2), "rr_2x2": float(r.rr_2x2),
            "be_2x2_scaled": float(r.be_2x2_scaled), "rr_2x2_scaled": float(r.rr_2x2_scaled),
            "symbolic_reused": bool(r.symbolic_reused), "ruiz_iterations": int(r.ruiz_iterations),
            "density": {"rho_c": float(r.rho_c), "nnz_op": int(r.nnz_op), "nnz_fac": int(r.nnz_fac),
                        "ratio": float(r.density_ratio)},
            "failure_detail": r.failure_detail}


def report_from_json(d: dict) -> SolveReport:
    nan = float("nan")
    g = lambda k: nan if d[k] is None else float(d[k])  # noqa: E731  (null = NaN)
    dens = d["density"]
    return SolveReport(status=_STATUS_OF[d["status"]], delta1_final=g("delta1"), delta2_used=g("delta2"),
                       cg_iterations=int(d["cg_iterations"]), factorization_attempts=int(d["factorization_attempts"]),
                       be_4x4=g("be_4x4"), rr_4x4=g("rr_4x4"), be_2x2=g("be_2x2"), rr_2x2=g("rr_2x2"),
                       be_2x2_scaled=g("be_2x2_scaled"), rr_2x2_scaled=g("rr_2x2_scaled"),
                       symbolic_reused=bool(d["symbolic_reused"]), ruiz_iterations=int(d["ruiz_iterations"]),
                       rho_c=nan if dens["rho_c"] is None else float(dens["rho_c"]), nnz_op=int(dens["nnz_op"]),
                       nnz_fac=int(dens["nnz_fac"]),
                       density_ratio=nan if dens["ratio"] is None else float(dens["ratio"]),
                       failure_detail=d["failure_detail"])


@dataclass
class Run:
    gamma: float
    reports: list
    stats: SequenceStats


@dataclass
class RunManifest:
    kind: str
    config: SolverConfig
    input_manifest: str
    csv_path: str
    runs: list = field(default_factory=list)
    version: int = 1

    def to_json_string(self) -> str:
        return _dump({"version": self.version, "kind": self.kind, "config": config_to_json(self.config),
                      "input_manifest": self.input_manifest, "csv": self.csv_path,
                      "runs": [{"gamma": float(r.gamma), "reports": [report_to_json(x) for x in r.reports],
                                "stats": {"symbolic_analyses": int(r.stats.symbolic_analyses),
                                          "numeric_factorizations": int(r.stats.numeric_factorizations),
                                          "factorization_attempts": int(r.stats.factorization_attempts)}}
                               for r in self.runs]})[:-1]

    @staticmethod
    def from_json_string(text: str) -> "RunManifest":
        try:
            j = json.loads(text)
        except json.JSONDecodeError as e:
            raise ManifestError(f"run manifest: {e}") from e
        runs = [Run(float(r["gamma"]), [report_from_json(x) for x in r["reports"]],
                    SequenceStats(**{k: int(v) for k, v in r["stats"].items()})) for r in j["runs"]]
        return RunManifest(j["kind"], config_from_json(j["config"]), j["input_manifest"], j["csv"], runs,
                           int(j["version"]))


def solve_csv_row(k: int, r: SolveReport) -> str:
    return (f"{k},{fmt(r.delta1_final)},{fmt(r.delta2_used)},{r.cg_iterations},{fmt(r.be_4x4)},"
            f"{fmt(r.rr_4x4)},{fmt(r.be_2x2)},{fmt(r.rr_2x2)},{r.nnz_fac},{fmt(r.density_ratio)},"
            f"{_STATUS_NAMES[SolveStatus(r.status)]}")


def sweep_csv_row(gamma: float, k: int, r: SolveReport) -> str:
    return f"{fmt(gamma)},{k},{r.cg_iterations},{fmt(r.be_4x4)},{fmt(r.rr_4x4)},{fmt(r.delta1_final)}"


def csv_text(m: RunManifest) -> str:
    if m.kind == "solve":
        rows = [SOLVE_CSV_SCHEMA, SOLVE_CSV_HEADER]
        rows += [solve_csv_row(k, r) for run in m.runs for k, r in enumerate(run.reports)]
    else:
        rows = [SWEEP_CSV_SCHEMA, SWEEP_CSV_HEADER]
        rows += [sweep_csv_row(run.gamma, k, r) for run in m.runs for k, r in enumerate(run.reports)]
    return "\n".join(rows) + "\n"


def _run_over_sequence(manifest_path, cfg: SolverConfig, out_dir, gammas, sweep: bool, err=sys.stderr,
                       device: int = 0, perm=None) -> int:
    from .solver import solve_sequence  # the GPU path
    tag = "sweep-gamma" if sweep else "solve"
    try:
        if not (cfg.gamma >= 0 and 0 < cfg.delta_min <= cfg.delta_max):
            raise ManifestError("invalid solver configuration")
        systems, _ = load_sequence(manifest_path)
    except (ManifestError, MatrixMarketError) as e:
        print(f"{tag}: {e}", file=err)
        return EXIT_USAGE
    if not systems:
        print(f"{tag}: manifest lists no systems: {manifest_path}", file=err)
        return EXIT_USAGE
    os.makedirs(str(out_dir), exist_ok=True)
    csv_path = os.path.join(str(out_dir), "sweep.csv" if sweep else "solve.csv")
    m = RunManifest("sweep" if sweep else "solve", cfg, str(manifest_path), csv_path)
    failed = False
    for g in (gammas if sweep else [cfg.gamma]):
        run_cfg = SolverConfig(**{f.name: getattr(cfg, f.name) for f in fields(cfg)})
        run_cfg.gamma = float(g)
        res = solve_sequence(systems, run_cfg, device=device, perm=perm)
        m.runs.append(Run(float(g), list(res.reports), res.stats))
        failed = failed or not all(is_success(r.status) for r in res.reports)
    Path(csv_path).write_text(csv_text(m))
    Path(os.path.join(str(out_dir), "run_manifest.json")).write_text(m.to_json_string() + "\n")
    return EXIT_SOLVE_FAILURE if failed else EXIT_OK


def cmd_solve(manifest_path, cfg: SolverConfig, out_dir, err=sys.stderr, device: int = 0, perm=None) -> int:
    """hkkt::cmd_solve (driver.cpp): solve_sequence over the manifest,
    solve.csv + run_manifest.json in out_dir."""
    return _run_over_sequence(manifest_path, cfg, out_dir, None, False, err, device, perm)


def cmd_sweep_gamma(manifest_path, gammas, cfg: SolverConfig, out_dir, err=sys.stderr, device: int = 0,
                    perm=None) -> int:
    """hkkt::cmd_sweep_gamma (driver.cpp): one solve_sequence per gamma,
    sweep.csv + run_manifest.json in out_dir."""
    return _run_over_sequence(manifest_path, cfg, out_dir, list(gammas), True, err, device, perm)


def main(argv=None) -> int:
    import argparse
    p = argparse.ArgumentParser(prog="python -m paper_2110_03636_b200.seqio")
    sub = p.add_subparsers(dest="cmd", required=True)
    s1 = sub.add_parser("solve")
    s1.add_argument("manifest")
    s1.add_argument("out_dir")
    s1.add_argument("--gamma", type=float, default=SolverConfig().gamma)
    s2 = sub.add_parser("sweep-gamma")
    s2.add_argument("manifest")
    s2.add_argument("out_dir")
    s2.add_argument("--gammas", required=True)
    try:
        a = p.parse_args(argv)
    except SystemExit:
        return EXIT_USAGE
    if a.cmd == "solve":
        return cmd_solve(a.manifest, SolverConfig(gamma=a.gamma), a.out_dir)
    try:
        gammas = [float(x) for x in a.gammas.split(",") if x]
    except ValueError:
        print("sweep-gamma: bad --gammas", file=sys.stderr)
        return EXIT_USAGE
    return cmd_sweep_gamma(a.manifest, gammas, SolverConfig(), a.out_dir)


if __name__ == "__main__":
    sys.exit(main())
