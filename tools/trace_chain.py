"""Developer probe: per-block stamps of the chain sweep (PCLAB_TRSV_TRACE):
[step start, dependencies in hand, published, in-chain | re-polls << 1]."""
import sys

import numpy as np

for suf in (".lo", ".up"):
    t = np.fromfile(sys.argv[1] + suf, dtype=np.int64).reshape(-1, 4)
    ok = t[:, 1] > 0
    t = t[ok]
    t0 = t[:, 0].min()
    st, rd, pb = (t[:, 0] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    chain = (t[:, 3] & 1) == 1
    rp = t[:, 3] >> 1
    print(suf, "blocks", ok.sum(), "span us %.1f" % pb.max())
    for name, m in (("all", np.ones_like(chain)), ("no re-poll", rp == 0), ("re-polled", rp > 0)):
        if m.sum() == 0:
            continue
        print("  %-10s share %.2f  start->ready %.2f  ready->pub %.2f  (median us)"
              % (name, m.mean(), np.median(rd[m] - st[m]), np.median(pb[m] - rd[m])))
    print("  re-poll rounds when re-polled: median %d" % (np.median(rp[rp > 0]) if np.any(rp > 0) else 0))
