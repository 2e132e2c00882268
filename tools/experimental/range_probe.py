"""Developer probe of the range-pipelined sweeps on one workload: device
time of both stand-alone sweeps (CUDA events) and, with PCLAB_RANGE_TRACE
set, a per-range summary of the step trace (range start lag, step time,
time waiting for the staged stream)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_118"
w = P.workloads.by_name(name)
a, b, model = P.workloads.build(w)
pc = P.Precond(a, "ic0")
x = torch.randn(a.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)


def dev_ms(f, reps=10):
    f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tr = os.environ.pop("PCLAB_RANGE_TRACE", None)
lo = dev_ms(lambda: pc.trsv_device(False, x.data_ptr(), y.data_ptr()))
up = dev_ms(lambda: pc.trsv_device(True, x.data_ptr(), y.data_ptr()))
print(f"R={os.environ.get('PCLAB_RANGE_NODES', 'auto')} lower {lo:.3f} ms upper {up:.3f} ms (incl. pad copies)",
      flush=True)
if tr:
    os.environ["PCLAB_RANGE_TRACE"] = tr
    pc.trsv_device(False, x.data_ptr(), y.data_ptr())
    with open(tr + ".lo", "rb") as f:
        ns, nr, R = np.frombuffer(f.read(24), np.int64)
        t8 = np.frombuffer(f.read(64 * ns), np.int64).reshape(ns, 8)
        t = t8[:, [0, 0, 2]]
        st = np.frombuffer(f.read(16 * ns), np.int32).reshape(ns, 4)
        rs = np.frombuffer(f.read(8 * (nr + 1)), np.int64)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3  # us
    print(f"steps {ns} ranges {nr} R {R} span {t[:, 2].max():.1f} us")
    starts = np.array([t[rs[r], 1] for r in range(nr)])
    ends = np.array([t[rs[r + 1] - 1, 2] for r in range(nr)])
    nst = np.diff(rs)
    dur = t[:, 2] - t[:, 1]
    wait = t[:, 1] - t[:, 0]
    print("range start lag (us): median %.2f  p90 %.2f" % (np.median(np.diff(starts)), np.percentile(np.diff(starts), 90)))
    print("range busy (us): median %.1f  steps/range median %d" % (np.median(ends - starts), np.median(nst)))
    print("step time (us): median %.3f p90 %.3f  stage wait (us): median %.3f p90 %.3f  nodes/step median %d" %
          (np.median(dur), np.percentile(dur, 90), np.median(wait), np.percentile(wait, 90), np.median(st[:, 2])))
    d = np.diff(t8[:, :3], axis=1) / 1e3
    print("warp0 phases (us, median): finish %.3f  prefetch+bar %.3f" % tuple(np.median(d, axis=0)))
    for r in (0, 1, nr // 2, nr - 1):
        sl = slice(rs[r], rs[r + 1])
        print(f" range {r}: start {starts[r]:.1f} end {ends[r]:.1f} steps {nst[r]} step-time med "
              f"{np.median(dur[sl]):.3f} wait med {np.median(wait[sl]):.3f}")
