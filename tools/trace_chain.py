"""Developer probe: per-block stamps of the chain sweep (PCLAB_TRSV_TRACE):
[operands issued, published, item, in-chain] for every block."""
import sys

import numpy as np

for suf in (".lo", ".up"):
    base = sys.argv[1] + suf
    lv = np.fromfile(base + ".lev", dtype=np.int32)
    t = np.fromfile(base, dtype=np.int64)
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else None
    t = t.reshape(-1, 4)
    pub = t[:, 1]
    ok = pub > 0
    t = t[ok]
    t0 = t[:, 0].min()
    iss, pubt = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    step = pubt - iss
    chain = t[:, 3] == 1
    print(suf, "blocks", ok.sum(), "span us %.1f" % pubt.max())
    print("  issue->publish: median %.2f p10 %.2f p90 %.2f us; in-chain %.2f, segment start %.2f"
          % (np.median(step), np.percentile(step, 10), np.percentile(step, 90), np.median(step[chain]),
             np.median(step[~chain])))
    busy = np.array([((iss <= x) & (pubt >= x)).sum() for x in np.linspace(0, pubt.max(), 9)[1:-1]])
    print("  blocks in flight at 1/8..7/8:", busy)
