#!/usr/bin/env python
"""PCG time-to-tolerance and iterations/s on the BASELINE workload.

One step = the full device path of pclab_pcg_solve on a resident system:
symbolic analysis (L/U patterns, level sets, schedules) + IC(0)
factorisation + PCG to rel_tol 1e-8 (BASELINE.json configs[2]: Q1
elasticity, 118^3 elements, 5.01M dofs, 4.1e8 nnz). `value` = PCG
iterations per second of PCG-loop time (device events) summed over ranks;
`ms_per_step` = the whole step (analysis + factor + loop). `e2e` is the same
metric through the host C-ABI call (pinned host CSR and b in, x out, every
copy inside the timed region). `--impl reference` times the reference's own
pcg() (oracle/_ref, compiled from /root/reference) on the host cores.

Multi-GPU: the path does not shard (BASELINE north star: one GPU, no
collectives), so --gpus N runs N independent replicas ("replicas only").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="elasticity_q1_118")
    ap.add_argument("--kind", default="ic0")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-iters", type=int, default=2, help="PCG iterations per reference step")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def combine_ranks(ms: float, cg_s: float, iters: int, world: int, device: str):
    """Whole-job numbers over replicas: step time and loop time are the MAX
    over ranks, iterations the SUM (value = all ranks' iterations / slowest
    rank's loop time)."""
    if world <= 1:
        return ms, cg_s, float(iters)
    import torch
    import torch.distributed as dist

    t = torch.tensor([ms, cg_s], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = torch.tensor([float(iters)], dtype=torch.float64, device=device)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return t[0].item(), t[1].item(), s[0].item()


# ------------------------------------------------------------ CPU reference
def reference_sample(w, iters: int, steps: int, warmup: int):
    """The reference's pcg() (krylov.cpp:114, compiled from /root/reference
    into oracle/_ref) on the full system with its IC(0) factor (computed once
    by the C oracle, bit-identical to the reference's ic0). Returns
    (iterations, cg seconds, wall seconds per step) per timed step."""
    from oracle import oracle as O
    import paper_2412_07127_b200.workloads as WL

    t0 = time.perf_counter()
    a, b, _ = WL.build_oracle(w)
    lvals, _ = O.ic0(a)
    setup = time.perf_counter() - t0
    out = []
    for s in range(warmup + steps):
        t = time.perf_counter()
        _, rep = O.ref_pcg_factor(a, lvals, b, w.rel_tol, iters)
        if s >= warmup:
            out.append((rep["iterations"], rep["cg_time"], time.perf_counter() - t))
    return out, setup, a


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    res, setup, a = reference_sample(w, args.ref_iters, args.steps, args.warmup)
    its = sum(r[0] for r in res)
    cg = sum(r[1] for r in res)
    wall = sum(r[2] for r in res)
    v = its / cg
    line = {
        "metric": "pcg_iters_per_s", "value": v, "unit": "iter/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / len(res) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)", "impl": "reference",
        "config": {"workload": w.name, "n": a.n, "nnz": a.nnz, "kind": "ic0", "rel_tol": w.rel_tol,
                   "sample": f"{args.ref_iters} PCG iterations per step"},
        "cpu_baseline": {"value": v, "unit": "iter/s", "cores": 1, "kind": "reference",
                         "sample": f"{args.ref_iters} iterations of the reference pcg() per step on the "
                                   f"full {a.n}-dof system, IC(0) factor, single thread"},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup,
    }
    print(json.dumps(line))


# --------------------------------------------------------------- B200 arm
def run_b200(args, w):
    import torch
    import torch.distributed as dist
    import paper_2412_07127_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    P.set_stream(stream.cuda_stream)

    a, b_host, model = P.workloads.build(w)
    n, _, nnz = a.shape()
    bt = torch.from_numpy(b_host).cuda()
    xt = torch.zeros_like(bt)
    need_model = args.kind in ("nic", "gnnic")

    def step():
        a.drop_analysis()
        pc = P.Precond(a, args.kind, model if need_model else None)
        rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=w.rel_tol, max_iters=w.max_iters,
                              stream=stream.cuda_stream)
        return pc, rep

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    reps = []
    l0 = P.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            pc, rep = step()
            reps.append(rep)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = P.launch_count() - l0
    ms = e0.elapsed_time(e1)
    its = sum(r["iterations"] for r in reps)
    cg = sum(r["cg_time"] for r in reps)
    ms, cg, its_all = combine_ranks(ms, cg, its, world, "cuda")
    value = its_all / cg

    # per-kernel device times of the loop (eager iterations, events between kernels)
    prof = pc.profile_device(bt.data_ptr(), xt.data_ptr(), 20)
    info = pc.info()
    hbm, peak_kind = peaks()
    nl = info["nnz_lower"]
    lay = pc.layout()
    # algorithmic HBM bytes per launch of each kernel, for the layout it runs on
    if lay["node_blocked"]:
        # node-blocked sweep: L values once, one column index per 3x3 block,
        # the slot schedule (4-byte slot + 32-byte row record), rhs, 1/l_ii,
        # solution write and the re-arm write of the other sweep vector
        def sweep_bytes_of(bc, slots):
            return 8 * nl + 4 * bc + 36 * slots + 4 * 8 * n
        sweep_lo = sweep_bytes_of(lay["block_cols_lower"], lay["slots_lower"])
        sweep_up = sweep_bytes_of(lay["block_cols_upper"], lay["slots_upper"])
        sweep_name = "bsr_trsv_kernel (node-blocked sweep)"
    else:
        sweep_lo = sweep_up = 12 * nl + 8 * (n + 1) + 4 * 8 * n  # L vals+cols, row_ptr, rhs, x, 1/l_ii, reset
        sweep_name = "trsv_kernel (lower sweep)"
    if lay["a_node_blocked"]:
        # p <- z + beta p (24n) then q = A p: A values, block columns, row and
        # block pointers, p gathered once, q written
        spmv_bytes = 24 * n + 8 * nnz + 4 * lay["block_cols_a"] + 8 * n + 8 * (n // 3 + 1) + 2 * 8 * n
    else:
        spmv_bytes = 24 * n + 12 * nnz + 8 * (n + 1) + 2 * 8 * n
    # reference format (scalar CSR, int32 columns): two sweeps, p update +
    # product, axpy + norm, dot
    csr_bytes = (2 * (12 * nl + 8 * (n + 1) + 4 * 8 * n) + (24 * n + 12 * nnz + 8 * (n + 1) + 2 * 8 * n)
                 + 6 * 8 * n + 2 * 8 * n)
    if prof["fused"]:
        fused_bytes = sweep_up + spmv_bytes - 24 * n
        kern = {
            "sweep_lower": {"ms": prof["sweep_lower_ms"], "bytes": sweep_lo},
            "sweep_upper_spmv": {"ms": prof["sweep_upper_ms"], "bytes": fused_bytes},
            "pq_update": {"ms": prof["spmv_ms"], "bytes": 6 * 8 * n},
            "axpy_norm": {"ms": prof["axpy_ms"], "bytes": 6 * 8 * n},
            "dot": {"ms": prof["dot_ms"], "bytes": 2 * 8 * n},
        }
        top, top_name = "sweep_upper_spmv", "bsr_upper_mv_kernel (fused sweep + product)"
    else:
        kern = {
            "sweep_lower": {"ms": prof["sweep_lower_ms"], "bytes": sweep_lo},
            "sweep_upper": {"ms": prof["sweep_upper_ms"], "bytes": sweep_up},
            "spmv_p": {"ms": prof["spmv_ms"], "bytes": spmv_bytes},
            "axpy_norm": {"ms": prof["axpy_ms"], "bytes": 6 * 8 * n},
            "dot": {"ms": prof["dot_ms"], "bytes": 2 * 8 * n},
        }
        top, top_name = "sweep_lower", sweep_name
    for k in kern.values():
        k["gbs"] = k["bytes"] / k["ms"] / 1e6
    iter_bytes = sum(k["bytes"] for k in kern.values())
    iter_ms = sum(k["ms"] for k in kern.values())
    achieved = kern[top]["gbs"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "kernel": top_name,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "iteration": {"bytes": iter_bytes, "ms": iter_ms, "gbs": iter_bytes / iter_ms / 1e6,
                              "frac": iter_bytes / iter_ms / 1e6 / hbm,
                              # the same iteration in the reference's scalar CSR format
                              "csr_equivalent_bytes": csr_bytes,
                              "csr_equivalent_gbs": csr_bytes / iter_ms / 1e6,
                              "csr_equivalent_frac": csr_bytes / iter_ms / 1e6 / hbm}}

    # end to end through the host C-ABI: pinned CSR + b in, x out
    rp, cols, vals = a.csr()
    rp_p = torch.from_numpy(rp).pin_memory()
    cols_p = torch.from_numpy(cols).pin_memory()
    vals_p = torch.from_numpy(vals).pin_memory()
    b_p = torch.from_numpy(b_host).pin_memory()
    x_p = torch.empty_like(b_p).pin_memory()
    e2e_rates = []
    for k in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ah = P.Matrix.from_csr_device(n, nnz, rp_p.data_ptr(), cols_p.data_ptr(), vals_p.data_ptr())
        x_np, rep = P.pcg_solve(ah, b_p.numpy(), args.kind, model if need_model else None,
                                rel_tol=w.rel_tol, max_iters=w.max_iters)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        del ah
        if k > 0:
            e2e_rates.append(rep["iterations"] / dt)
    e2e_v = float(np.mean(e2e_rates)) * (world if world > 1 else 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            if O.ref_available():
                res, _, _ = reference_sample(w, args.ref_iters, 1, 0)
                cpu = {"value": res[0][0] / res[0][1], "unit": "iter/s", "cores": 1, "kind": "reference",
                       "sample": f"{args.ref_iters} iterations of the reference pcg() (oracle/_ref) on the "
                                 f"full {n}-dof system with its IC(0) factor, single thread"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "iter/s", "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}"}

    if rank == 0:
        r0 = reps[-1]
        line = {
            "metric": "pcg_iters_per_s", "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, device-assembled)",
            "config": {"workload": w.name, "n": n, "nnz": nnz, "kind": args.kind, "rel_tol": w.rel_tol,
                       "parallelism": f"replicas{world}", "l2": "inputs (4.9 GB CSR) larger than L2",
                       "iterations": r0["iterations"], "converged": r0["converged"],
                       "time_to_tol_s": ms / args.steps / 1e3, "p_time_s": r0["p_time"],
                       "analysis_s": r0["analysis_time"], "ic0_s": r0["ic0_time"], "cg_s": r0["cg_time"],
                       "true_rel_residual": r0["true_rel_residual"], "block_size": info["block_size"],
                       "levels": [info["block_levels_lower"], info["block_levels_upper"]]},
            "roofline": roofline,
            "kernels": kern,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_v, "unit": "iter/s",
                    "h2d_bytes_per_step": int(8 * (n + 1) + 4 * nnz + 8 * nnz + 8 * n),
                    "d2h_bytes_per_step": int(8 * n)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    import paper_2412_07127_b200.workloads as WL
    w = WL.by_name(args.config)
    if w is None:
        raise SystemExit(f"unknown config {args.config}")
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_b200(args, w)


if __name__ == "__main__":
    main()
