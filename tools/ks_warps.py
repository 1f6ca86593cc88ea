"""Per-warp timeline of CTA 0's first CG operator run (HYKKT_KS_PROF=1):
for each step, when each warp left the barrier, finished issuing, read the
header, finished phase A and arrived at the closing barrier."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2110_03636_b200 import Device, SolverConfig, acopf, _lib
from paper_2110_03636_b200.solver import Batch, stack_values
nb, B = int(sys.argv[1]), int(sys.argv[2])
systems = acopf.batch(nb, B, seed=7)
dev = Device(0)
dev.analyze(systems[0])
bt = Batch(dev)
bt.upload(stack_values(systems))
bt.solve_resident(SolverConfig())
L = _lib.lib()
ns_ = C.c_int64(0)
L.hykkt_debug_ks_program.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
_lib.check(L.hykkt_debug_ks_program(dev.h, None, C.byref(ns_)))
ns = ns_.value
steps = np.zeros(8 * ns, np.int32)
_lib.check(L.hykkt_debug_ks_program(dev.h, steps.ctypes.data, C.byref(ns_)))
steps = steps.reshape(-1, 8)
buf = np.zeros(1024 * 16, np.uint64)
tr = np.zeros((ns + 1) * 81, np.uint64)
n = C.c_int64(0)
L.hykkt_debug_ks_prof.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
_lib.check(L.hykkt_debug_ks_prof(dev.h, buf.ctypes.data, C.byref(n), tr.ctypes.data))
w = tr[ns + 1:ns + 1 + ns * 80].reshape(ns, 16, 5).astype(np.int64)
w[:, :, 2] &= (1 << 60) - 1
print("step kind vlen ilen | per warp: [issue, header, phaseA_end(rel), arrive(rel)] ns; last warp; span ns")
tot = np.zeros(4)
for k in range(ns):
    if w[k, 0, 0] == 0:
        continue
    t0 = w[k, :, 0].min()
    rel = w[k] - t0
    arrive = rel[:, 4]
    last = int(np.argmax(arrive))
    nxt = w[k + 1, :, 0].min() - t0 if k + 1 < ns and w[k + 1, 0, 0] else 0
    tot += [rel[:, 1].max(), rel[:, 2].max(), arrive.max(), nxt]
    if k < 40 or k % 10 == 0:
        print(f"{k:4d} {steps[k][0]} {steps[k][2]:5d} {steps[k][1]:5d} | issue {rel[:,1].max():5d} hdr {rel[:,2].max():5d} "
              f"arrive min {arrive.min():5d} med {int(np.median(arrive)):5d} max {arrive.max():6d} (warp {last:2d}) next {nxt:6d}")
print("sums over steps (us): max issue %.1f, max header %.1f, max arrive %.1f, step span %.1f" % tuple(tot / 1e3))
# producer-bound steps: how much the step would shrink if the producer
# arrived with the slowest compute warp
ex, cnt, comp = 0, 0, 0
for k in range(ns):
    if w[k, 0, 0] == 0:
        continue
    t0 = w[k, :, 0].min()
    rel = w[k] - t0
    pc = rel[15, 4]
    cm = rel[:15, 4].max()
    comp += cm
    if pc > cm:
        ex += pc - cm
        cnt += 1
print("producer last in %d steps; excess %.1f us; compute-only arrive sum %.1f us; compute issue-wait sum %.1f us" % (
    cnt, ex / 1e3, comp / 1e3, sum((w[k, :15, 1] - w[k, :, 0].min()).max() for k in range(ns) if w[k, 0, 0]) / 1e3))
# phase split per L step (compute warps; warps [0, ww) hold the warp tasks)
sa = sb_w = sb_t = 0.0
nstep = 0
crit_w = crit_t = 0.0
print("L-step phases: k kind nseg nw nt ww | A_end  B_end(warp-task warps)  B_end(thread warps) ns")
for k in range(ns):
    if w[k, 0, 0] == 0 or steps[k][0] not in (0, 1):
        continue
    t0 = w[k, :, 0].min()
    rel = w[k, :15] - t0
    ww = int(steps[k][7])
    a_end = rel[:, 3].max()
    bw = rel[:ww, 4].max() if ww > 0 else 0
    bt = rel[ww:, 4].max()
    nstep += 1
    sa += a_end
    if bw >= bt:
        crit_w += bw - a_end
    else:
        crit_t += bt - a_end
    if k % 4 == 0:
        print(f"  {k:4d} {steps[k][0]} {steps[k][3]:4d} {steps[k][4]:3d} {steps[k][5]:4d} {ww:2d} | {a_end:6d} {bw:6d} {bt:6d}")
print("L steps %d: sum A_end %.1f us; phase B critical: warp-task bound %.1f us, thread-task bound %.1f us" % (
    nstep, sa / 1e3, crit_w / 1e3, crit_t / 1e3))
