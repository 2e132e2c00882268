"""Developer probe: device time of the stand-alone sweeps and SpMV on one
workload (knobs come from the PCLAB_* environment of the process)."""
import os
import sys

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


lo = dev_ms(lambda: pc.trsv_device(False, x.data_ptr(), y.data_ptr()))
up = dev_ms(lambda: pc.trsv_device(True, x.data_ptr(), y.data_ptr()))
bt = torch.from_numpy(b).cuda()
xt = torch.zeros_like(bt)
try:
    prof = pc.profile_device(bt.data_ptr(), xt.data_ptr(), 10)
    prof = {k: round(float(v), 4) for k, v in prof.items()}
except P.PclabError as e:  # probe builds with wrong numerics
    prof = repr(e)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("PCLAB_"))
print(f"[{env}] lower {lo:.3f} upper {up:.3f} profile {prof}", flush=True)
