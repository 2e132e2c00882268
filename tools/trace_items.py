"""Developer probe: item timeline of chunk 0 of the chunked sweep."""
import sys
import numpy as np
nch = int(sys.argv[2])
t = np.fromfile(sys.argv[1] + ".lo", dtype=np.int64)
ch = t[: 4 * nch].reshape(-1, 4)
items = t[4 * nch:].reshape(-1, 4)
t0 = ch[0, 0]
n0 = int(sys.argv[3])  # items in chunk 0
it = items[:n0]
s, r, d = (it[:, 0] - t0) / 1e3, (it[:, 1] - t0) / 1e3, (it[:, 2] - t0) / 1e3
print("chunk0 end", (ch[0, 1] - t0) / 1e3)
print("median start->ready %.2f ready->done %.2f" % (np.median(r - s), np.median(d - r)))
for k in list(range(0, 40)) + list(range(400, 420)):
    print(f" item {k:4d} warp {it[k,3]:2d} start {s[k]:8.2f} ready {r[k]:8.2f} done {d[k]:8.2f}")
