"""Relaxed-amalgamation sweep (B200): per (width, zeros) the supernode count,
tree levels, explicit zeros, single-system phase times at C1-C4 and the
256-system batched step, written as JSON lines."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_03636_b200 import Device, SolverConfig, acopf  # noqa: E402
from paper_2110_03636_b200.solver import Batch, stack_values  # noqa: E402

cfg = SolverConfig()
widths = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16,32,64").split(",")]
zeros = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "60").split(",")]
configs = (sys.argv[3] if len(sys.argv) > 3 else "C1,C2,C3,C4,B").split(",")
systems = {c: acopf.generate(acopf.CONFIG_BUSES[c], 7, 7) for c in configs if c != "B"}
batch = stack_values(acopf.batch(2000, 256, seed=7)) if "B" in configs else None
for wd in widths:
    for z in zeros:
        row = {"amalg_width": wd, "amalg_zeros_pct": z}
        for c, s in systems.items():
            dev = Device(0)
            dev.set_option("amalg_width", wd)
            dev.set_option("amalg_zeros_pct", z)
            dev.analyze(s)
            info = dev.info()
            dev.upload(s)
            ts = []
            for k in range(5):
                r = dev.solve_resident(cfg, timing=True)
                if k >= 2:
                    ts.append(dev.timing())
            t = sorted(ts, key=lambda x: x["total_ms"])[1]
            row[c] = {"nsup": info["n_supernodes"], "levels": info["n_levels"], "zeros": info["explicit_zeros"],
                      "total_ms": round(t["total_ms"], 3), "factor_ms": round(t["factor_ms"], 3),
                      "cg_ms": round(t["cg_ms"], 3), "cg_its": r.cg_iterations,
                      "cg_us_per_it": round(1e3 * t["cg_ms"] / max(1, r.cg_iterations), 1)}
            dev.close()
        if batch is not None:
            dev = Device(0)
            dev.set_option("amalg_width", wd)
            dev.set_option("amalg_zeros_pct", z)
            dev.analyze(acopf.generate(2000, 7, 7))
            bt = Batch(dev)
            bt.upload(batch)
            ts = []
            for k in range(4):
                bt.solve_resident(cfg, timing=True)
                if k >= 1:
                    ts.append(dev.timing())
            t = sorted(ts, key=lambda x: x["total_ms"])[1]
            row["B256"] = {k: round(t[k], 3) for k in ("total_ms", "factor_ms", "cg_ms", "assemble_ms")}
            dev.close()
        print(json.dumps(row), flush=True)
