"""Developer probe: wall time of each device stage (warm, synchronous C-ABI
calls) on one workload, plus the per-kernel device times of an iteration."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402


def timeit(f, reps=3):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return min(ts) * 1e3


def main(name, m=None, iters=30):
    w = P.workloads.by_name(name)
    if m:
        w = w.scaled(m)
    t = time.perf_counter()
    a, b, model = P.workloads.build(w)
    print(f"[{w.name}] n={a.n} nnz={a.nnz} build {time.perf_counter()-t:.2f}s", flush=True)
    t = time.perf_counter()
    ic = P.Precond(a, "ic0")
    print(f"  first ic0 build {time.perf_counter()-t:.3f}s timings {ic.timings()} info {ic.info()}", flush=True)
    print(f"  ic0 build warm {timeit(lambda: P.Precond(a, 'ic0')):.2f} ms", flush=True)
    print(f"  gnnic build warm {timeit(lambda: P.Precond(a, 'gnnic', model)):.2f} ms", flush=True)
    g = P.Precond(a, "gnnic", model)
    print(f"  gnnic timings {g.timings()}", flush=True)
    n = a.n
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ms = timeit(lambda: a.spmv_device(x.data_ptr(), y.data_ptr()), 10)
    nb = a.nnz * 12 + (n + 1) * 8 + 2 * n * 8
    print(f"  spmv {ms:.3f} ms  {nb/ms/1e6:.0f} GB/s (algorithmic {nb/1e9:.2f} GB)", flush=True)
    lnnz = ic.info()["nnz_lower"]
    lb = lnnz * 12 + (n + 1) * 8 + 2 * n * 8
    for up in (False, True):
        ms = timeit(lambda: ic.trsv_device(up, x.data_ptr(), y.data_ptr()), 10)
        print(f"  trsv {'upper' if up else 'lower'} {ms:.3f} ms  {lb/ms/1e6:.0f} GB/s", flush=True)
    bt = torch.from_numpy(b).cuda()
    xt = torch.zeros_like(bt)
    for kind, pc in (("ic0", ic), ("gnnic", g)):
        for _ in range(2):
            rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=w.rel_tol, max_iters=iters)
        print(f"  pcg[{kind}] {rep['iterations']} its cg {rep['cg_time']*1e3:.2f} ms "
              f"-> {rep['cg_time']/max(rep['iterations'],1)*1e3:.3f} ms/it conv {rep['converged']}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 30)
