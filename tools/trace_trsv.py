"""Developer probe: analyse PCLAB_TRSV_TRACE dumps of one sweep.

Per item: [start, values-ready, published, extra] globaltimer stamps; with
the schedule's slots and critical predecessors, the handoff latency (ready
of an item minus publication of its critical predecessor's item) and the
share of items that started only after that publication (too few warps)."""
import sys

import numpy as np

for suf in (".lo", ".up"):
    base = sys.argv[1] + suf
    lv = np.fromfile(base + ".lev", dtype=np.int32)
    t = np.fromfile(base, dtype=np.int64)[: 4 * len(lv)].reshape(-1, 4)
    t0 = t[:, 0].min()
    s, c, d = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    print(suf, "items", len(t), "span us", d.max(), "levels", lv.max() + 1)
    print("  per item: start->ready %.2f us, ready->done %.2f us (median)" % (np.median(c - s), np.median(d - c)))
    g = (t[:, 3] // 1024) / 1e3
    rr = t[:, 3] % 1024
    print("  gather after crit %.2f us median; poll rounds median %d p90 %d"
          % (np.median(g), np.median(rr), np.percentile(rr, 90)))
    try:
        sl = np.fromfile(base + ".slots", dtype=np.int32)
        cr = np.fromfile(base + ".crit", dtype=np.int32)
    except FileNotFoundError:
        sl = None
    if sl is not None and len(sl):
        G = len(sl) // len(lv)
        bs = 3 if cr.max() % 3 == 2 else 1
        nb = len(cr)
        item_of = np.full(nb, -1, dtype=np.int64)
        idx = np.nonzero(sl >= 0)[0]
        item_of[sl[idx]] = idx // G
        blk = sl[idx]
        it = idx // G
        cb = cr[blk]
        ok = cb >= 0
        pi = item_of[cb[ok] // max(bs, 1)]
        ho = c[it[ok]] - d[pi]
        late = s[it[ok]] - d[pi]
        print("  handoff crit-published -> ready: median %.2f p10 %.2f p90 %.2f us"
              % (np.median(ho), np.percentile(ho, 10), np.percentile(ho, 90)))
        print("  items started after their crit was published: %.3f (median lateness %.2f us)"
              % (np.mean(late > 0), np.median(late[late > 0]) if np.any(late > 0) else 0))
    nl = lv.max() + 1
    fin = np.array([d[lv == l].max() for l in range(nl)])
    print("  level finish deltas (us): median %.2f  p90 %.2f" % (np.median(np.diff(fin)), np.percentile(np.diff(fin), 90)))
    busy = np.array([((s <= x) & (d >= x)).sum() for x in np.linspace(0, d.max(), 9)[1:-1]])
    print("  items in flight at 1/8..7/8 of the span:", busy)
    for l in list(range(0, 4)) + list(range(nl // 2, nl // 2 + 4)):
        m = lv == l
        print(f"   L{l}: n={m.sum()} start[{s[m].min():.1f},{s[m].max():.1f}] ready[{c[m].min():.1f},{c[m].max():.1f}] done[{d[m].min():.1f},{d[m].max():.1f}]")
