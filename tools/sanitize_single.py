"""Small single-system solves under each kernel variant, for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2110_03636_b200 import Device, SolverConfig, acopf
for env in ({}, {"HYKKT_MF_BIG": "1", "HYKKT_TRSV_WIDE": "1"}, {"HYKKT_TRSV_BOTTOM_MIN": "1"}):
    for k in ("HYKKT_MF_BIG", "HYKKT_TRSV_WIDE", "HYKKT_TRSV_BOTTOM_MIN"):
        os.environ.pop(k, None)
    os.environ.update(env)
    s = acopf.generate(200, 7, 7)
    d = Device(0); d.analyze(s); r = d.solve_full(s, SolverConfig())
    print(env, int(r.report.status), r.report.cg_iterations, flush=True)
    d.close()
