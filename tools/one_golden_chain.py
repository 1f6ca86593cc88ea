import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
os.environ["HYKKT_TRSV_CHAINS"] = "1"
from golden_util import load
from paper_2110_03636_b200 import Device
s, cfg, perm, want = load("acopf_nb120_g1e2")
dev = Device(0); dev.analyze(s, perm)
r = dev.solve_full(s, cfg)
print("ok", r.report.cg_iterations)
