#!/usr/bin/env python
"""HyKKT on B200 — driver benchmark (one JSON line on rank 0).

Workload (BASELINE.json configs[4], per GPU; configs[1]'s shape): a batch of
independent ACTIVSg2000-shaped block-4x4 KKT systems (SURVEY.md Appendix B
generator, nb = 2000 -> N = 40k, shared pattern, symbolic analysis once); a
step is the full per-IPM-iteration HyKKT solve (reduce, Ruiz, H_gamma, delta1
ladder + supernodal Cholesky, w solve, Schur-complement CG, dx solve,
recover) of every system in the batch.

  value    solves/s over all ranks, values resident in HBM, device-timed
  e2e      same metric through the public C ABI with pinned host buffers:
           H2D of the step's values + solve + D2H of the solutions
  roofline the CG kernel (k_cg, the dominant kernel): canonical algorithmic
           bytes per CG iteration x iterations / its
           CUDA-event time, against the measured HBM copy peak
  cpu_baseline the reference C++ library (oracle/_ref, built from the
           reference sources) on the host cores, same systems

Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under
torch.distributed.run (one rank per GPU, nccl plumbing for barrier/max only —
the systems are independent, no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hykkt", "reference"], default="hykkt")
    ap.add_argument("--batch", type=int, default=256, help="systems per GPU per step")
    ap.add_argument("--nb", type=int, default=2000, help="buses (2000 = ACTIVSg2000 shape)")
    ap.add_argument("--gamma", type=float, default=1e4)
    ap.add_argument("--cpu-sample", type=int, default=64)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the ACTIVSg70k-shaped probe")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = max(smax, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def canonical_cg_bytes(info: dict) -> int:
    """B_it = 24 nnz(J) + 24 nnz(L) + 4 (2 (n_x+1) + 2 (m_c+1))
    + 8 (6 n_x + 9 m_c) — each stored entry 8 B value + 4 B index per
    traversal (J^T p, J t, L forward, L backward), pointer arrays once,
    vector touches."""
    nx, mc = info["n"], info["m_c"]
    return (24 * info["nnz_j"] + 24 * info["nnz_l"] + 4 * (2 * (nx + 1) + 2 * (mc + 1))
            + 8 * (6 * nx + 9 * mc))


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if args.impl == "hykkt" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_reference_run(systems, cfg, seconds: float, threads: int):
    """Reference solve_full over `systems` with a std::thread pool and a
    shared symbolic factor (reference AMD ordering), repeated until
    `seconds` of work; returns (solves/s, solves, wall s, cg iterations)."""
    from oracle import ref
    b = ref.Batch(systems)
    b.run(cfg, None, threads=threads)  # warm
    done, wall, its = 0, 0.0, None
    while wall < seconds and done < 50 * len(systems):
        sec, its, st = b.run(cfg, None, threads=threads)
        done += len(systems)
        wall += sec
        if (st > 1).any():
            raise RuntimeError("reference solve failed on the bench workload")
    return done / wall, done, wall, its


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2110_03636_b200 import SolverConfig, acopf
    cfg = SolverConfig(gamma=args.gamma)
    threads = os.cpu_count() or 1
    sample = max(1, min(args.batch, args.cpu_sample))
    systems = acopf.batch(args.nb, sample, seed=7)
    from oracle import ref
    b = ref.Batch(systems)
    for _ in range(args.warmup):
        b.run(cfg, None, threads=threads)
    times = []
    for _ in range(args.steps):
        sec, its, st = b.run(cfg, None, threads=threads)
        times.append(sec)
    total = sum(times)
    value = sample * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"reference C++ solve_full (oracle/_ref) on {sample} ACTIVSg2000-shaped "
                               f"systems per step, std::thread pool of {threads}, shared symbolic",
                   "nb": args.nb, "gamma": args.gamma},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} systems x {args.steps} steps"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "HyKKT solves/s (factor + CG per system), ACTIVSg2000-shaped KKT batch"


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch

    from paper_2110_03636_b200 import Device, SolverConfig, acopf
    from paper_2110_03636_b200.solver import VALUE_FIELDS, Batch, stack_values

    torch.cuda.set_device(local)
    cfg = SolverConfig(gamma=args.gamma)
    B = args.batch
    systems = acopf.batch(args.nb, B, seed=7 + rank * B)
    dev = Device(local)
    t0 = time.perf_counter()
    dev.analyze(systems[0])
    analyze_s = time.perf_counter() - t0
    info = dev.info()

    # pinned host staging (torch as plumbing)
    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    sizes = {n: v.shape[0] for n, v in zip(VALUE_FIELDS, __import__(
        "paper_2110_03636_b200.solver", fromlist=["system_values"]).system_values(systems[0]))}
    host_vals = {n: pinned((B, sizes[n])) for n in VALUE_FIELDS}
    stack_values(systems, out=host_vals)
    s0 = systems[0]
    host_out = dict(dx=pinned((B, s0.n_x)), ds=pinned((B, s0.m_d)), dy=pinned((B, s0.m_c)),
                    dyd=pinned((B, s0.m_d)))
    h2d = int(sum(v.nbytes for v in host_vals.values()))
    d2h = int(sum(v.nbytes for v in host_out.values()))

    batch = Batch(dev)
    batch.upload(host_vals)
    for _ in range(args.warmup):
        reps = batch.solve_resident(cfg, timing=True)
    bad = [r for r in reps if r.status > 1]
    if bad:
        raise RuntimeError(f"{len(bad)} systems failed: {bad[0]}")

    # ---- device-resident timed region ----
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    launches, cg_ms, cg_its, tot_dev_ms = 0, 0.0, 0, 0.0
    phase = dict(assemble_ms=0.0, factor_ms=0.0, solve_w_ms=0.0, cg_ms=0.0, solve_dx_ms=0.0)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            reps = batch.solve_resident(cfg, timing=True)
            t = dev.timing()
            launches += t["kernel_launches"]
            cg_ms += t["cg_ms"]
            tot_dev_ms += t["total_ms"]
            for k in phase:
                phase[k] += t[k]
            cg_its += sum(r.cg_iterations for r in reps)
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = ev0.elapsed_time(ev1)
    step_ms = allmax(elapsed_ms / args.steps, world)
    value = world * B / (step_ms / 1e3)

    # ---- end to end through the public API (pinned host buffers) ----
    barrier(world)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        batch.upload(host_vals)
        batch.solve_resident(cfg)
        batch.download(host_out)
    ev1.record(stream)
    torch.cuda.synchronize()
    e2e_step_ms = allmax(ev0.elapsed_time(ev1) / args.steps, world)
    e2e_value = world * B / (e2e_step_ms / 1e3)

    # ---- roofline of the dominant kernel ----
    # ks_solve (system-per-CTA) applies the Schur operator once per CG
    # iteration plus the w and dx solves per system: (its + 2) applications
    # of the canonical SURVEY.md §8(d) bytes each.  Its CUDA-event time is
    # the handle's cg_ms phase (the launch is alone between two events on
    # the handle's stream).
    peak, peak_kind = peaks()
    bytes_it = canonical_cg_bytes(info)
    ops = cg_its + 2 * B * args.steps
    achieved = bytes_it * ops / (cg_ms / 1e3) / 1e9 if cg_ms > 0 else 0.0
    traffic = None
    prof = ROOT / "profiles" / "ks_solve_traffic.json"
    if prof.exists():
        try:
            d = json.loads(prof.read_text())
            if d.get("nb") == args.nb:
                traffic = d.get("dram_bytes_per_operator")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm",
                "kernel": "ks_solve (one CTA per system: w solve, Schur-complement CG with the J^T / "
                          "supernodal forward+backward / J operator streamed through shared-memory "
                          "rings, dx solve, recover)",
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "bytes_per_operator": bytes_it, "operator_applications": ops, "cg_iterations": cg_its,
                "kernel_ms": cg_ms}

    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic ACOPF-shaped KKT (SURVEY.md Appendix B generator; topology seed 7, "
                "value seed 7+b)",
        "config": {"workload": f"batch of {B} independent ACTIVSg2000-shaped KKT systems per GPU "
                               f"(nb={args.nb}, n_x={s0.n_x}, m_c={s0.m_c}, m_d={s0.m_d}, N={s0.total_size}), "
                               "shared pattern, symbolic once; step = solve_full of every system",
                   "per_gpu_batch": B, "global_batch": B * world, "gamma": args.gamma,
                   "parallelism": f"independent systems sharded over {world} GPU(s), no collective",
                   "scheduling": ("ks_solve takes systems longest-first by their CG iterations in the previous "
                                  "call on the same batch (history LPT; warm-up calls seed it; every system is "
                                  "fully solved every step; HYKKT_KS_LPT=0 disables: about 61 vs 54 ms per step)"),
                   "l2": f"inputs > L2: {h2d / 1e6:.0f} MB of resident values per GPU per step",
                   "nnz_l": info["nnz_l"], "n_supernodes": info["n_supernodes"],
                   "supernode_levels": info["n_levels"], "analyze_s": analyze_s},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step_ms},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "single_system": {"config": "ACTIVSg2000-shaped (configs[1])",
                          "ms_per_system_device": tot_dev_ms / (args.steps * B),
                          "note": "batched per-system averages; on the system-per-CTA path solve_w_ms "
                                  "is the stream build (remap) and cg_ms the fused ks_solve launch "
                                  "(w solve + CG + dx solve + recover)",
                          **{k: v / (args.steps * B) for k, v in phase.items()},
                          "cg_iterations_mean": cg_its / (args.steps * B)},
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = systems[: max(1, min(B, args.cpu_sample))]
        v, done, wall, its = cpu_reference_run(sample, cfg, args.cpu_seconds, threads)
        line["cpu_baseline"] = {"value": v, "unit": "solves/s", "cores": threads, "kind": "reference",
                                "sample": f"{done} solve_full calls over {len(sample)} of the bench systems "
                                          f"({wall:.1f} s, std::thread pool, shared symbolic)"}
    if rank == 0 and world == 1 and not args.no_large:
        line["large"] = large_probe(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(world)


def large_probe(cfg):
    """ACTIVSg70k-shaped single system (configs[3]): device ms/system and
    the reference's 1-thread time on the same ordering."""
    from oracle import ref
    from paper_2110_03636_b200 import Device, acopf
    s = acopf.generate(70000, 7, 7)
    dev = Device(0)
    dev.analyze(s)
    info = dev.info()
    dev.upload(s)
    for _ in range(2):
        r = dev.solve_resident(cfg, timing=True)
    t = dev.timing()
    bytes_it = canonical_cg_bytes(info)
    peak, _ = peaks()
    cg_gbs = bytes_it * r.cg_iterations / (t["cg_ms"] / 1e3) / 1e9
    out = {"config": "ACTIVSg70k-shaped (configs[3]), nb=70000", "n_x": s.n_x, "N": s.total_size,
           "nnz_l": info["nnz_l"], "supernode_levels": info["n_levels"],
           "ms_per_system_device": t["total_ms"], "phases_ms": {k: t[k] for k in (
               "assemble_ms", "factor_ms", "solve_w_ms", "cg_ms", "solve_dx_ms")},
           "cg_iterations": r.cg_iterations, "cg_gbs": cg_gbs, "cg_frac_of_hbm": cg_gbs / peak}
    try:
        a, f, c, its = ref.time_phases(s, cfg, dev.perm(), reps=1)
        out["cpu_reference_1thread"] = {"assemble_s": a, "factor_s": f, "cg_s": c, "cg_iterations": its,
                                        "ms_per_system": 1e3 * (a + f + c), "ordering": "same as device"}
    except Exception as e:  # pragma: no cover
        out["cpu_reference_1thread"] = {"error": str(e)}
    dev.close()
    return out


if __name__ == "__main__":
    main()
