"""Developer probe: analyse PCLAB_TRSV_TRACE dumps of one sweep."""
import sys
import numpy as np
for suf in (".lo", ".up"):
    lv = np.fromfile(sys.argv[1] + suf + ".lev", dtype=np.int32)
    t = np.fromfile(sys.argv[1] + suf, dtype=np.int64)[: 4 * len(lv)].reshape(-1, 4)
    t0 = t[:, 0].min()
    s, c, d = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    print(suf, "items", len(t), "span us", d.max(), "levels", lv.max() + 1)
    print("  per item: start->crit %.2f us, crit->done %.2f us (median)" % (np.median(c - s), np.median(d - c)))
    nl = lv.max() + 1
    fin = np.array([d[lv == l].max() for l in range(nl)])
    rdy = np.array([c[lv == l].max() for l in range(nl)])
    st = np.array([s[lv == l].min() for l in range(nl)])
    print("  level finish deltas (us): median %.2f  p90 %.2f" % (np.median(np.diff(fin)), np.percentile(np.diff(fin), 90)))
    busy = np.array([((s <= x) & (d >= x)).sum() for x in np.linspace(0, d.max(), 9)[1:-1]])
    print("  items in flight at 1/8..7/8 of the span:", busy)
    for l in list(range(0, 6)) + list(range(nl // 2, nl // 2 + 6)):
        m = lv == l
        print(f"   L{l}: n={m.sum()} start[{s[m].min():.1f},{s[m].max():.1f}] crit[{c[m].min():.1f},{c[m].max():.1f}] done[{d[m].min():.1f},{d[m].max():.1f}]")
