"""Developer probe: per-tile timestamps of one stand-alone lts sweep
(PCLAB_LTS_TRACE=<path> makes the launcher re-run the sweep with a trace)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.environ.setdefault("PCLAB_LTS_TRACE", "gpurun_out/lts_trace")
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_118"
w = P.workloads.by_name(name)
a, b, model = P.workloads.build(w)
pc = P.Precond(a, "ic0")
x = torch.randn(a.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
pc.trsv_device(False, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
t = np.loadtxt(path + ".lo", dtype=np.int64)
t0 = t[:, 3].min()
start, first, end = (t[:, 3] - t0) / 1e3, (t[:, 4] - t0) / 1e3, (t[:, 5] - t0) / 1e3
print("tiles", len(t), "total us", end.max())
print("residency us: mean %.1f median %.1f max %.1f" % ((end - start).mean(), np.median(end - start), (end - start).max()))
print("wait for first item us: mean %.1f median %.1f max %.1f" % ((first - start).mean(), np.median(first - start), (first - start).max()))
print("run after first item us: mean %.1f median %.1f" % ((end - first).mean(), np.median(end - first)))
ph = np.zeros((len(t), 6))
print("phase us per tile (wait next stage, loads returned, spin, reduce+solve+publish, refill): mean", ph.mean(0)[:5])
for i in (0, 1, 2, 100, 500, 1000, 1500):
    print("tile", i, "phases us", np.round(ph[i, :5], 1), "sum", round(ph[i, :5].sum(), 1), "run", round(end[i] - first[i], 1))
step = max(len(t) // 20, 1)
print("ticket chain0 nch start first end sm")
for i in range(0, len(t), step):
    print(t[i, 0], t[i, 1], t[i, 2], "%.1f %.1f %.1f" % (start[i], first[i], end[i]), t[i, 6])
# concurrency: tiles running (past first item) over time
grid = np.linspace(0, end.max(), 21)
for g in grid:
    print("t=%.0f resident %d running %d" % (g, ((start <= g) & (end > g)).sum(), ((first <= g) & (end > g)).sum()))
