"""Developer probe: per-chunk timeline of the chunked sweep (PCLAB_TRSV_TRACE)."""
import sys
import numpy as np
for suf in (".lo", ".up"):
    t = np.fromfile(sys.argv[1] + suf, dtype=np.int64).reshape(-1, 4)
    nch = int(sys.argv[2])
    t = t[:nch]
    t0 = t[:, 0].min()
    s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    print(suf, "chunks", nch, "span us %.1f" % e.max(), "chunk dur median %.1f us max %.1f" % (np.median(e - s), (e - s).max()))
    order = np.argsort(t[:, 3])
    for k in list(order[:6]) + list(order[nch // 2: nch // 2 + 4]):
        print(f"   chunk {k} claim {t[k,3]} sm {t[k,2]} start {s[k]:.1f} end {e[k]:.1f}")
