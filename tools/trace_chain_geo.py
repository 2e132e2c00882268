"""Developer probe: chain-sweep trace on the structured elasticity mesh
(nodes m x m x (m-1) after clamping z = 0): for every block, the time from
its latest cross-pencil dependency's publication to its own publication,
and from its in-pencil predecessor's publication."""
import sys

import numpy as np

m = int(sys.argv[2]) if len(sys.argv) > 2 else 119
for suf in (".lo",):
    t = np.fromfile(sys.argv[1] + suf, dtype=np.int64).reshape(-1, 4)
    nb = m * m * (m - 1)
    t = t[:nb]
    pub = t[:, 1].astype(np.float64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    pub = (pub - t0) / 1e3
    idx = np.arange(nb)
    i = idx % m
    j = (idx // m) % m
    k = idx // (m * m)
    # lower neighbours across pencils: (di, dj, dk) with dk = -1 (any di, dj) or dk = 0, dj = -1
    cross = np.full(nb, -1.0)
    for dk in (-1, 0):
        for dj in (-1, 0, 1):
            if dk == 0 and dj != -1:
                continue
            for di in (-1, 0, 1):
                ii, jj, kk = i + di, j + dj, k + dk
                ok = (ii >= 0) & (ii < m) & (jj >= 0) & (jj < m) & (kk >= 0)
                nbr = np.where(ok, (kk * m + jj) * m + ii, 0)
                cross = np.where(ok, np.maximum(cross, pub[nbr]), cross)
    prev = np.where(i > 0, pub[np.maximum(idx - 1, 0)], -1.0)
    has_c = cross >= 0
    has_p = i > 0
    dc = pub - cross
    dp = pub - prev
    bind_c = has_c & has_p & (cross > prev)
    print(suf, "span %.1f us" % pub.max())
    print("  after latest cross dep: median %.2f p10 %.2f us" % (np.median(dc[has_c]), np.percentile(dc[has_c], 10)))
    print("  after in-pencil predecessor: median %.2f p10 %.2f us" % (np.median(dp[has_p]), np.percentile(dp[has_p], 10)))
    print("  cross dep published after the predecessor (binding) for %.2f of blocks" % bind_c.mean())
    print("  when cross binds: pub - cross median %.2f; when predecessor binds: pub - prev median %.2f"
          % (np.median(dc[bind_c]), np.median(dp[has_p & has_c & ~bind_c])))
