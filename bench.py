#!/usr/bin/env python
"""HyKKT on B200 — driver benchmark (one JSON line on rank 0).

Workload (BASELINE.json configs[4]): a batch of 256 independent
ACTIVSg2000-shaped block-4x4 KKT systems (SURVEY.md Appendix B generator,
nb = 2000 -> N = 40k, one shared pattern, symbolic analysis once, value seed
7 + b for system b), sharded across the job's GPUs in contiguous blocks of
256/G (strong scaling; --scaling weak gives every GPU its own
256).  A step is the full per-interior-point-iteration HyKKT solve of every
system (reduce, Ruiz, H_gamma, delta1 ladder + supernodal Cholesky, w solve,
Schur-complement CG, dx solve, recover).  The timed loop cycles through four
IPM-like value sets (each the previous one drifted by 0.01, generator.cpp
197-210 semantics), so no step sees the values of the step before and the
history longest-first system order works from the previous set's CG counts.

  value     solves/s over all ranks, values resident in HBM when the step
            starts (the step's device-to-device copy of its value set into
            the handle's batch buffers is inside the timed region)
  e2e       the same through the public C ABI with pinned host buffers:
            H2D of the step's values + solve + D2H of the solutions
  roofline  ks_solve (the dominant kernel): SURVEY.md §8(d) canonical bytes
            per Schur-operator application under the C5 rule (values per
            system, index arrays once per 32-system tile) x applications /
            its CUDA-event time, against the measured HBM copy peak
  cpu_baseline  the reference C++ library (oracle/_ref, built from the
            reference sources) on all host cores, a bounded sample of the
            same systems

Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under
torch.distributed.run (one rank per GPU; nccl only for barrier / max / gather).
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
METRIC = "HyKKT solves/s (factor + CG per system), ACTIVSg2000-shaped KKT batch"
N_SETS = 4
DRIFT = 0.01


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", choices=["hykkt", "reference"], default="hykkt")
    ap.add_argument("--global-batch", type=int, default=256, help="systems in the whole job (strong)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--nb", type=int, default=2000, help="buses (2000 = ACTIVSg2000 shape)")
    ap.add_argument("--gamma", type=float, default=1e4)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the single-system / batch-size / ACTIVSg70k probes")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


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


def canonical_bytes(info: dict) -> dict:
    """SURVEY.md §8(d) canonical bytes of one Schur-operator application
    (J^T p, L forward, L backward, J t): each stored entry 8 B value + 4 B
    int32 index per traversal, pointer arrays once per traversal, vector
    touches t (n_x: 6) and p / q / x / r (m_c: 9).  Split into the value
    part (per system) and the index part (per pattern)."""
    nx, mc, nj, nl = info["n"], info["m_c"], info["nnz_j"], info["nnz_l"]
    values = 8 * (2 * nj + 2 * nl) + 8 * (6 * nx + 9 * mc)
    index = 4 * (2 * nj + 2 * nl) + 4 * (2 * (nx + 1) + 2 * (mc + 1))
    return {"single": values + index, "values": values, "index": index,
            "c5": values + index / 32.0}


def value_sets(nb: int, seeds: list[int], n_sets: int = N_SETS):
    """n_sets IPM-like value sets of the same systems: set k = set k-1
    drifted by DRIFT (acopf.drift, generator.cpp:197-210 semantics)."""
    from paper_2110_03636_b200 import acopf
    sets = [[acopf.generate(nb, 7, s) for s in seeds]]
    for k in range(1, n_sets):
        sets.append([acopf.drift(x, DRIFT, s * 7919 + k) for x, s in zip(sets[-1], seeds)])
    return sets


def run_reference(args, world, rank):
    """The reference arm: the reference's own CPU implementation
    (oracle/_ref, the unmodified reference library) on all host cores, on
    the whole job's systems, cycling the same value sets; rank 0 only."""
    if rank != 0:
        return
    from oracle import ref
    from paper_2110_03636_b200 import SolverConfig
    from paper_2110_03636_b200 import dist as hd
    cfg = SolverConfig(gamma=args.gamma)
    threads = os.cpu_count() or 1
    if args.scaling == "strong":
        seeds = hd.shard_seeds(args.global_batch, 1, 0)
    else:
        seeds = [s for r in range(world) for s in hd.shard_seeds(args.global_batch, world, r, scaling="weak")]
    sets = value_sets(args.nb, seeds)
    batches = [ref.Batch(s) for s in sets]
    for w in range(args.warmup):
        batches[w % N_SETS].run(cfg, None, threads=threads)
    total = 0.0
    for st in range(args.steps):
        sec, its, status = batches[(args.warmup + st) % N_SETS].run(cfg, None, threads=threads)
        if (status > 1).any():
            raise RuntimeError("reference solve failed on the bench workload")
        total += sec
    n = len(seeds)
    value = n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"reference C++ solve_full (oracle/_ref, the unmodified reference library) on "
                               f"the job's {n} ACTIVSg2000-shaped systems per step, {N_SETS} drifted value sets "
                               f"cycled, std::thread pool of {threads}, shared symbolic (reference AMD)",
                   "nb": args.nb, "gamma": args.gamma, "global_batch": n},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": "reference",
                         "sample": f"{n} systems x {args.steps} steps"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_reference_run(systems, cfg, seconds: float, threads: int):
    """Reference solve_full over `systems` with a std::thread pool and a
    shared symbolic factor, repeated until `seconds` of work."""
    from oracle import ref
    b = ref.Batch(systems)
    b.run(cfg, None, threads=threads)  # warm
    done, wall = 0, 0.0
    while wall < seconds and done < 50 * len(systems):
        sec, its, st = b.run(cfg, None, threads=threads)
        done += len(systems)
        wall += sec
        if (st > 1).any():
            raise RuntimeError("reference solve failed on the bench workload")
    return done / wall, done, wall


def main():
    args = parse()
    from paper_2110_03636_b200 import dist as hd
    world, rank, local = hd.setup("nccl" if args.impl == "hykkt" else "gloo")
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch

    from paper_2110_03636_b200 import Device, SolverConfig
    from paper_2110_03636_b200.solver import VALUE_FIELDS, Batch, stack_values, system_values

    torch.cuda.set_device(local)
    cfg = SolverConfig(gamma=args.gamma)
    seeds = hd.shard_seeds(args.global_batch, world, rank, scaling=args.scaling)
    B = len(seeds)
    sets = value_sets(args.nb, seeds)
    s0 = sets[0][0]
    dev = Device(local)
    t0 = time.perf_counter()
    dev.analyze(s0)
    analyze_s = time.perf_counter() - t0
    info = dev.info()

    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    sizes = {n: v.shape[0] for n, v in zip(VALUE_FIELDS, system_values(s0))}
    host_sets = []
    for s in sets:
        hv = {n: pinned((B, sizes[n])) for n in VALUE_FIELDS}
        stack_values(s, out=hv)
        host_sets.append(hv)
    dev_sets = [{n: torch.from_numpy(hv[n]).to(f"cuda:{local}") for n in VALUE_FIELDS} for hv in host_sets]
    dev_ptrs = [{n: t[n].data_ptr() for n in VALUE_FIELDS} for t in dev_sets]
    host_out = dict(dx=pinned((B, s0.n_x)), ds=pinned((B, s0.m_d)), dy=pinned((B, s0.m_c)),
                    dyd=pinned((B, s0.m_d)))
    h2d = int(sum(v.nbytes for v in host_sets[0].values()))
    d2h = int(sum(v.nbytes for v in host_out.values()))
    upload_launches = sum(1 for n in VALUE_FIELDS if sizes[n] > 0)  # kb_interleave per field
    torch.cuda.synchronize()

    batch = Batch(dev)

    def device_loop(steps, offset, timing=True):
        acc = dict(launches=0, cg_ms=0.0, total_ms=0.0, cg_its=0, assemble_ms=0.0, factor_ms=0.0,
                   solve_w_ms=0.0, solve_dx_ms=0.0)
        for st in range(steps):
            batch.upload_device(dev_ptrs[(offset + st) % N_SETS], B)
            reps = batch.solve_resident(cfg, timing=timing)
            bad = [r for r in reps if r.status > 1]
            if bad:
                raise RuntimeError(f"{len(bad)} systems failed: {bad[0]}")
            t = dev.timing()
            acc["launches"] += t["kernel_launches"] + upload_launches
            for k in ("cg_ms", "total_ms", "assemble_ms", "factor_ms", "solve_w_ms", "solve_dx_ms"):
                acc[k] += t[k]
            acc["cg_its"] += sum(r.cg_iterations for r in reps)
        return acc

    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        hd.barrier(world)
        torch.cuda.synchronize()
        ev0.record(stream)
        out = fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), out

    # ---- device-resident timed region (history-LPT order, the default) ----
    device_loop(args.warmup, 0)
    with ClockSampler(local) as clk:
        elapsed_ms, acc = timed(lambda: device_loop(args.steps, args.warmup))
    step_ms = hd.allmax(elapsed_ms / args.steps, world, f"cuda:{local}")
    value = hd.allsum(B, world, f"cuda:{local}") / (step_ms / 1e3)

    # ---- the same with natural system order (LPT off) ----
    dev.set_option("ks_lpt", 0)
    device_loop(1, 0)
    nat_ms, _ = timed(lambda: device_loop(args.steps, args.warmup))
    dev.set_option("ks_lpt", 1)
    nat_step_ms = hd.allmax(nat_ms / args.steps, world, f"cuda:{local}")

    # ---- end to end through the public API (pinned host buffers) ----
    # sequential: upload (H2D) -> solve -> download (D2H) per step
    def e2e_loop():
        for st in range(args.steps):
            batch.upload(host_sets[st % N_SETS])
            batch.solve_resident(cfg)
            batch.download(host_out)

    e2e_seq_ms, _ = timed(e2e_loop)
    e2e_seq_step_ms = hd.allmax(e2e_seq_ms / args.steps, world, f"cuda:{local}")
    e2e_seq_value = hd.allsum(B, world, f"cuda:{local}") / (e2e_seq_step_ms / 1e3)

    # pipelined (the reported e2e): hykkt_batch_upload_async of step k+1's
    # inputs is issued before the solve of step k, and step k's outputs come
    # back with hykkt_batch_download_async (double-buffered pinned host
    # outputs); every step's H2D and D2H still happen inside the timed region
    host_outs = [host_out, {n: pinned(a.shape) for n, a in host_out.items()}]

    def e2e_pipe():
        batch.upload_async(host_sets[0])
        for st in range(args.steps):
            if st + 1 < args.steps:
                batch.upload_async(host_sets[(st + 1) % N_SETS])
            batch.solve_resident(cfg)
            batch.download_async(host_outs[st % 2])
        batch.sync()

    e2e_pipe()  # warm the staging buffers
    e2e_ms, _ = timed(e2e_pipe)
    e2e_step_ms = hd.allmax(e2e_ms / args.steps, world, f"cuda:{local}")
    e2e_value = hd.allsum(B, world, f"cuda:{local}") / (e2e_step_ms / 1e3)

    # ---- roofline of the dominant kernel (ks_solve) ----
    peak, peak_kind = peaks()
    cb = canonical_bytes(info)
    ops = acc["cg_its"] + 2 * B * args.steps  # (CG its + w solve + dx solve) per system
    ks_s = acc["cg_ms"] / 1e3
    achieved = cb["c5"] * ops / ks_s / 1e9 if ks_s > 0 else 0.0
    traffic, ncu_frac = None, None
    prof = ROOT / "profiles" / "ks_solve_traffic.json"
    if prof.exists():
        try:
            d = json.loads(prof.read_text())
            if d.get("nb") == args.nb:
                traffic = d.get("dram_bytes_per_operator")
                ncu_frac = traffic * ops / ks_s / 1e9 / peak if traffic and ks_s > 0 else None
        except Exception:
            traffic = None
    roofline = {"bound": "hbm",
                "kernel": "ks_solve (one CTA per system: w solve, Schur-complement CG with the J^T / "
                          "supernodal forward+backward / J operator streamed through shared-memory rings, "
                          "dx solve, recover)",
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "bytes_rule": "SURVEY.md §8(d) C5: per operator application values 8(2 nnzJ + 2 nnzL) + "
                              "8(6 n_x + 9 m_c) per system + index 4(2 nnzJ + 2 nnzL) + 4(2(n_x+1) + 2(m_c+1)) "
                              "once per 32-system tile",
                "bytes_per_operator_c5": cb["c5"], "bytes_per_operator_single": cb["single"],
                "operator_applications": ops, "cg_iterations": acc["cg_its"], "kernel_ms": acc["cg_ms"],
                "frac_ncu_dram": ncu_frac,
                "frac_single_system_rule": cb["single"] * ops / ks_s / 1e9 / peak if ks_s > 0 else None}

    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic ACOPF-shaped KKT (SURVEY.md Appendix B generator; topology seed 7, value seed 7+b, "
                f"{N_SETS} value sets drifted by {DRIFT} cycled through the steps)",
        "config": {"workload": f"batch of {args.global_batch} independent ACTIVSg2000-shaped KKT systems "
                               f"(nb={args.nb}, n_x={s0.n_x}, m_c={s0.m_c}, m_d={s0.m_d}, N={s0.total_size}), "
                               f"{'split over' if args.scaling == 'strong' else 'per GPU on'} {world} GPU(s), "
                               "shared pattern, symbolic once; step = solve_full of every system",
                   "per_gpu_batch": B, "global_batch": args.global_batch * (world if args.scaling == "weak" else 1),
                   "gamma": args.gamma,
                   "parallelism": f"contiguous blocks of independent systems on {world} GPU(s), no collective",
                   "value_sets": f"{N_SETS} IPM-like sets (drift {DRIFT}) cycled: each step solves values the "
                                 "previous step did not see",
                   "scheduling": "ks_solve takes systems longest-first by the previous call's CG iterations "
                                 "(history LPT, from the previous value set)",
                   "ms_per_step_natural_order": nat_step_ms,
                   "l2": f"inputs > L2: {h2d / 1e6:.0f} MB of per-step values per GPU (126 MB L2)",
                   "nnz_l": info["nnz_l"], "n_supernodes": info["n_supernodes"],
                   "supernode_levels": info["n_levels"], "analyze_s": analyze_s},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step_ms,
                "protocol": "pipelined public API: hykkt_batch_upload_async (pinned host -> device, next "
                            "step's inputs issued before this step's solve) + hykkt_batch_solve_resident + "
                            "hykkt_batch_download_async (device -> pinned host), hykkt_batch_sync at the end",
                "sequential": {"value": e2e_seq_value, "ms_per_step": e2e_seq_step_ms,
                               "protocol": "hykkt_batch_upload -> hykkt_batch_solve_resident -> "
                                           "hykkt_batch_download per step"}},
        "gpu_launches": acc["launches"],
        "clocks": clk.summary(),
        "batch_phases_ms_per_step": {k: acc[k] / args.steps for k in (
            "assemble_ms", "factor_ms", "solve_w_ms", "cg_ms", "solve_dx_ms", "total_ms")},
        "cg_iterations_mean": acc["cg_its"] / (args.steps * B),
    }
    del dev_sets
    if rank == 0 and world == 1 and not args.no_extras:
        line["batch_size_sweep"] = batch_size_sweep(args, cfg, sets, local)
        line["single_system"] = single_system_probe(cfg)
        line["large"] = large_probe(cfg)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, done, wall = cpu_reference_run(sets[0], cfg, args.cpu_seconds, threads)
        line["cpu_baseline"] = {"value": v, "unit": "solves/s", "cores": threads, "kind": "reference",
                                "sample": f"{done} solve_full calls over the {len(sets[0])} bench systems of value "
                                          f"set 0 ({wall:.1f} s, std::thread pool, shared symbolic)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    hd.barrier(world)


def batch_size_sweep(args, cfg, sets, local):
    """Device-resident solves/s on one GPU at the per-GPU batch sizes of the
    strong-scaling split (256/G for G = 8, 4, 2): the first B systems of each
    value set, cycled."""
    import torch

    from paper_2110_03636_b200 import Device
    from paper_2110_03636_b200.solver import Batch, stack_values
    out = {}
    for B in (32, 64, 128):
        dev = Device(local)
        dev.analyze(sets[0][0])
        bt = Batch(dev)
        vals = [stack_values(s[:B]) for s in sets]
        for w in range(3):
            bt.upload(vals[w % N_SETS])
            bt.solve_resident(cfg)
        torch.cuda.synchronize()
        ms = 0.0
        steps = 4
        for st in range(steps):
            bt.upload(vals[(3 + st) % N_SETS])
            bt.solve_resident(cfg, timing=True)
            ms += dev.timing()["total_ms"]
        out[str(B)] = {"solves_per_s": B * steps / (ms / 1e3), "ms_per_step": ms / steps,
                       "note": "device time of the solve (values uploaded before each step)"}
        dev.close()
    return out


def single_system_probe(cfg):
    """configs[0]-[2] single-system latency (values resident, device events)
    next to the reference on ONE host thread with the same ordering."""
    from oracle import ref
    from paper_2110_03636_b200 import Device, acopf
    out = {}
    for name, nb in (("C1", 500), ("C2", 2000), ("C3", 10000)):
        s = acopf.generate(nb, 7, 7)
        dev = Device(0)
        dev.analyze(s)
        dev.upload(s)
        runs = []
        for k in range(8):
            r = dev.solve_resident(cfg, timing=True)
            if k >= 3:
                runs.append(dev.timing())
        t = sorted(runs, key=lambda x: x["total_ms"])[len(runs) // 2]
        a, f, c, its = ref.time_phases(s, cfg, dev.perm(), reps=3)
        out[name] = {"nb": nb, "n_x": s.n_x, "N": s.total_size, "ms_per_system_device": t["total_ms"],
                     "phases_ms": {k: t[k] for k in ("assemble_ms", "factor_ms", "solve_w_ms", "cg_ms",
                                                     "solve_dx_ms")},
                     "cg_iterations": r.cg_iterations,
                     "cg_us_per_iteration": 1e3 * t["cg_ms"] / max(1, r.cg_iterations),
                     "cpu_reference_1thread_ms": 1e3 * (a + f + c),
                     "cpu_reference_1thread_phases_ms": {"assemble": 1e3 * a, "factor": 1e3 * f, "cg": 1e3 * c},
                     "cpu_reference_cg_iterations": its}
        dev.close()
    return out


def large_probe(cfg):
    """ACTIVSg70k-shaped single system (configs[3], the roofline config):
    device ms/system, the CG phase against the HBM roofline (canonical
    bytes per iteration), and the reference's 1-thread time on the same
    ordering."""
    from oracle import ref
    from paper_2110_03636_b200 import Device, acopf
    s = acopf.generate(70000, 7, 7)
    dev = Device(0)
    t0 = time.perf_counter()
    dev.analyze(s)
    analyze_s = time.perf_counter() - t0
    info = dev.info()
    dev.upload(s)
    runs = []
    for k in range(5):
        r = dev.solve_resident(cfg, timing=True)
        if k >= 2:
            runs.append(dev.timing())
    t = sorted(runs, key=lambda x: x["total_ms"])[len(runs) // 2]
    bytes_it = canonical_bytes(info)["single"]
    peak, _ = peaks()
    cg_gbs = bytes_it * r.cg_iterations / (t["cg_ms"] / 1e3) / 1e9
    out = {"config": "ACTIVSg70k-shaped (configs[3]), nb=70000", "n_x": s.n_x, "N": s.total_size,
           "nnz_l": info["nnz_l"], "n_supernodes": info["n_supernodes"], "supernode_levels": info["n_levels"],
           "analyze_s": analyze_s, "ms_per_system_device": t["total_ms"],
           "phases_ms": {k: t[k] for k in ("assemble_ms", "factor_ms", "solve_w_ms", "cg_ms", "solve_dx_ms")},
           "cg_iterations": r.cg_iterations, "cg_us_per_iteration": 1e3 * t["cg_ms"] / r.cg_iterations,
           "cg_bytes_per_iteration": bytes_it, "cg_gbs": cg_gbs, "cg_frac_of_hbm": cg_gbs / peak}
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
