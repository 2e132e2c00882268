"""Developer trace of the node-blocked sweep (build with -DBSS_TRACE, load via
PCLAB_LIB): per node {item start, dependencies seen, published, last
dependency}; walks the critical path back from the last node published and
splits it into hop (producer's publish -> consumer saw it), chain (seen ->
published) and late starts (the warp reached the item after its dependencies)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_118"
upper = len(sys.argv) > 2 and sys.argv[2] == "upper"
w = P.workloads.by_name(name)
a, b, model = P.workloads.build(w)
pc = P.Precond(a, "ic0")
bsz = 3 if w.family == "elasticity" else 2
nb = a.n // bsz
x = torch.randn(a.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
tr = torch.zeros(4 * nb, dtype=torch.int64, device="cuda")
L = P.lib()
L.pclab_debug_bss_trace.argtypes = [C.c_void_p]
for _ in range(3):
    pc.trsv_device(upper, x.data_ptr(), y.data_ptr())
assert L.pclab_debug_bss_trace(tr.data_ptr()) == 0
pc.trsv_device(upper, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
L.pclab_debug_bss_trace(None)
t = tr.cpu().numpy().reshape(nb, 4)
t0, t1, t2 = t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), t[:, 2].astype(np.int64)
cnt = ((t[:, 3].view(np.uint64) >> np.uint64(32)) & np.uint64(0xFFFF)).astype(np.int64)
gap = (t[:, 3].view(np.uint64) >> np.uint64(48)).astype(np.int64)  # record sweep only: loop top of the item
dep = (t[:, 3].view(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
dep[dep == 0xFFFFFFFF] = -1
base = t0[t0 > 0].min()
t0, t1, t2 = t0 - base, t1 - base, t2 - base
print(f"nodes {nb} span {t2.max() / 1e3:.1f} us; timer step {np.min(np.diff(np.unique(t2))[:1000])} ns")
waited = dep >= 0
print(f"items that re-polled: {waited.mean() * 100:.1f} %, re-polls per waiting node: mean {cnt[waited].mean():.1f} median {np.median(cnt[waited])}")
hop = t1[waited] - t2[dep[waited]]
chain = t2 - t1
front = t1[~waited] - t0[~waited]
q = lambda v: "p10 %.0f p50 %.0f p90 %.0f mean %.0f" % (*np.percentile(v, [10, 50, 90]), v.mean())
print("hop   ns (publish of the last dependency -> all seen):", q(hop))
print("chain ns (all seen -> published):", q(chain))
print("front ns (item start -> all seen, nodes that never re-polled):", q(front))
print("wait  ns (item start -> all seen, nodes that re-polled):", q(t1[waited] - t0[waited]))
if gap.max() > 0:
    print("gap   ns (previous item's end -> item start, same warp):", q(gap))
    print("  of which up to the issue of the record loads two items ahead (record sweep: field reused):", q(cnt))
late = t0[waited] - t2[dep[waited]]
print("late  ns (item start - publish of its last dependency; > 0: the warp arrived after it):", q(late),
      "; late starts %.1f %%" % (100.0 * (late > 0).mean()))
ontime = late <= 0
print("hop   ns, items whose warp was already waiting:", q(hop[ontime]))
# critical path: back from the last publication
cur = int(np.argmax(t2))
hops = chains = late = 0
nh = nl = steps = 0
while True:
    steps += 1
    chains += t2[cur] - t1[cur]
    if dep[cur] >= 0:
        hops += t1[cur] - t2[dep[cur]]
        nh += 1
        cur = int(dep[cur])
    else:
        # dependencies were there when the warp arrived: the warp's previous work bounds it
        late += t1[cur] - t0[cur]
        nl += 1
        break
print(f"critical path back from the last node: {steps} nodes; hops {hops / 1e3:.1f} us over {nh} ({hops / max(nh, 1):.0f} ns each); "
      f"chains {chains / 1e3:.1f} us ({chains / steps:.0f} ns each); stopped at a node that never waited (start {t0[cur] / 1e3:.1f} us)")
