#!/usr/bin/env python
"""bench.py -- TSQR factor GFLOP/s (2mn^2 model) and roofline fraction on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is the config's workload (BASELINE.json): c1/c2/c4 = factor + form Q,
c5 = factor + apply Q^T to C (k = 128).  `value` = 2 m n^2 / t_factor with
t_factor the device time of tsqr_factor (CUDA events on its stream, mean over
the K timed steps, max over ranks); ms_per_step covers the whole step.  The
factor is in place, so the pristine input is restored (device copy, outside
the events) before every step; every config's A is larger than the 126 MB L2.

N > 1: launched with torchrun, one rank per GPU, NCCL butterfly between ranks
(paper_0808_2664_b200.dist); the matrix is the config's global one (strong
scaling).  --impl reference times the CPU oracle (oracle/, plain C) on a
bounded sample of the same workload on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (block rows b from the config; tile rows s: the leaves of the
# binary tree, each factored as a flat chain of register-resident chunks)
CONFIGS = {
    "c1": dict(m=4096, n=16, b=512, s=512, kind="gauss", op="form_q", k=0,
               desc="fp64 A 4096x16 N(0,1) seed 0, row blocks 512 (8-leaf binary tree): factor + form Q"),
    "c2": dict(m=1_000_000, n=50, b=4096, s=1366, kind="gauss", op="form_q", k=0,
               desc="fp64 A 1,000,000x50 N(0,1), row blocks 4096, binary tree: factor + form Q"),
    "c3": dict(m=100_000, n=200, b=2048, s=400, kind="gauss", op="apply_qt", k=64,
               desc="fp64 A 100,000x200 N(0,1), row blocks 2048 (blocked compact-WY leaves): factor + apply Q^T "
                    "to C 100,000x64"),
    "c4": dict(m=16_777_216, n=64, b=4096, s=4096, kind="cond", op="form_q", k=0,
               desc="fp64 A 16,777,216x64 = G diag(sigma) V^T, sigma 1..1e-10: factor + form Q"),
    "c5": dict(m=33_554_432, n=32, b=4096, s=4096, kind="gauss", op="apply_qt", k=128,
               desc="fp64 A 33,554,432x32 N(0,1): factor + apply Q^T to C 33,554,432x128"),
}
DEFAULT_CONFIG = "c2"   # configs[1]: the workload BASELINE.json's metric is quoted on that fits one GPU

# FP64 peak for the roofline: B200 has no FP64 tensor multiplier
# (tcgen05 has no f64 kind; DMMA = DFMA rate), so the path is bound by the FP64 ALU:
# 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz = 37.23 TFLOP/s (tools/peaks.cu measured
# DMMA 37.18, DFMA 34.2 TFLOP/s on this pool).
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def kernel_launches(info, n, op, world):
    """Kernels of this repo launched per step (tsqr_api.cu's dispatch): factor, then the second op."""
    multi = info["ntiles"] > 1
    rounds = info["cross_rounds"] if world > 1 else 0
    if n <= 64:
        fac = 1 + 1                                   # chain leaves + pipelined tree (or R extraction)
        second = (1 + multi) if op == "apply_qt" else (info["depth"] + 2)   # leaves+nodes | identity+node steps+leaves
    else:
        fac = 1 + multi + 1                           # leaves + pipelined tree + R extraction
        second = (1 + info["depth"]) if op == "apply_qt" else (info["depth"] + 4)
    # butterfly rounds: pack + combine per round on the factor; apply exchanges the head per round
    cross = 2 * rounds + (1 if rounds else 0) + (2 * rounds if op == "apply_qt" else 0)
    return fac + second + cross


def max_over_ranks(vals, dev):
    """Element-wise max over the process group (device tensor for NCCL, host for gloo)."""
    import torch
    import torch.distributed as dist
    x = torch.tensor(vals, dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return x.tolist()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0, period=0.05):
        self.samples, self.reasons, self.period, self.index = [], set(), period, index
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.nv:
            self._stop.set()
            self.t.join()
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# -------------------------------------------------------------- input recipe
def make_slab(cfg, row0, rows, device):
    from paper_0808_2664_b200 import inputs
    if cfg["kind"] == "gauss":
        return inputs.gaussian_rows(row0, rows, cfg["n"], 0, device)
    return inputs.conditioned_rows(row0, rows, cfg["n"], 0, 1e10, 2, device)


def make_c_slab(cfg, row0, rows, device):
    from paper_0808_2664_b200 import inputs
    return inputs.gaussian_rows(row0, rows, cfg["k"], 1, device)


# -------------------------------------------------------------- CPU baseline
def oracle_sample(cfg, rows_budget_flops=1.2e10):
    """Time the CPU oracle (as it stands, 1 thread) on a bounded sample of the workload:
    the first whole row blocks of the config (same tile plan), factor only."""
    import numpy as np
    import oracle as orc
    from paper_0808_2664_b200 import inputs
    m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
    blocks = max(1, min(m // b, int(rows_budget_flops / (2.0 * b * n * n))))
    rows = blocks * b if m >= b else m
    At = make_slab(cfg, 0, rows, "cpu")
    A = inputs.to_numpy_colmajor(At)
    p = orc.plan(rows, n, b, s, 1)
    t0 = time.perf_counter()
    orc.tsqr_factor(A, p)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * rows * n * n / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle tsqr_factor on rows 0..{rows} ({blocks} row blocks of {b}) x {n}, same plan, 1 thread",
            "seconds": dt}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    budget = 2.0e9 / max(1, K + W) * 4
    for _ in range(W):
        oracle_sample(cfg, budget)
    vals, secs = [], []
    for _ in range(K):
        r = oracle_sample(cfg, budget)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * statistics.mean(secs), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "sample": r["sample"]},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


METRIC = "TSQR factor GFLOP/s (2mn^2 model) and fraction of HBM/FP64 roofline"


# -------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_0808_2664_b200 as T
    from paper_0808_2664_b200 import dist as tdist

    N = args.gpus
    rank, world = 0, 1
    if N > 1:
        # TSQR_BENCH_BACKEND=gloo + TSQR_BENCH_ONE_GPU=1: a functional check of the multi-rank
        # path with every rank on one GPU (the butterfly's messages staged through the host);
        # never a scaling measurement
        backend = os.environ.get("TSQR_BENCH_BACKEND", "nccl")
        local = 0 if os.environ.get("TSQR_BENCH_ONE_GPU") else int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", "0")))
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(backend)
        rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    m, n, b, s, k = cfg["m"], cfg["n"], cfg["b"], cfg["s"], cfg["k"]
    row0, ml = T.slab(m, n, b, world, rank)
    A0 = make_slab(cfg, row0, ml, dev)                  # pristine slab (column-major (n, ml))
    A = torch.empty_like(A0)
    C0 = make_c_slab(cfg, row0, ml, dev) if cfg["op"] == "apply_qt" else None
    C = torch.empty_like(C0) if C0 is not None else None
    Q = torch.empty((n, ml), dtype=torch.float64, device=dev) if cfg["op"] == "form_q" else None
    R = torch.empty((n, n), dtype=torch.float64, device=dev)
    info = T.plan_info(ml, n, block_rows=b, tile_rows=s, nranks=world, rank=rank)
    stream = torch.cuda.current_stream()
    tree = None
    st = None

    engine = tdist.CudaEngine(stage_timing=True) if world > 1 else None

    def step():
        nonlocal tree, st
        if world == 1:
            _, tree = T.factor(A, b, s, R=R, tree=tree, stage_timing=True)
        else:
            st = tdist.factor(A, b, s, engine=engine, tree=tree, cross=args.cross)   # workspace reused
            tree = st.tree
        ev_f.record(stream)
        if cfg["op"] == "form_q":
            T.form_q(tree, Q)
        else:
            if world == 1:
                T.apply_qt(tree, C)
            else:
                tdist.apply_qt(st, C)

    def restore():
        A.copy_(A0)
        if C is not None:
            C.copy_(C0)

    ev_s, ev_f, ev_e = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    for _ in range(args.warmup):
        restore()
        ev_s.record(stream)
        step()
        ev_e.record(stream)
    torch.cuda.synchronize()

    clocks = ClockSampler(dev.index)
    clocks.start()
    t_factor, t_step, t_leaf, t_tree = [], [], [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        restore()
        ev_s.record(stream)
        step()
        ev_e.record(stream)
        ev_e.synchronize()
        t_factor.append(ev_s.elapsed_time(ev_f))
        t_step.append(ev_s.elapsed_time(ev_e))
        lm, tm = tree.stage_ms()                          # the leaf kernel's own launch (device events)
        t_leaf.append(lm)
        t_tree.append(tm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    tf, ts = statistics.mean(t_factor), statistics.mean(t_step)
    tl, tt = statistics.mean(t_leaf), statistics.mean(t_tree)
    if world > 1:
        tf, ts, tl, tt = max_over_ranks([tf, ts, tl, tt], dev)

    # ---- e2e through the public API with pinned host buffers (host <-> device inside);
    # every rank copies its own slab, the time is the max over ranks
    A_h = A0.cpu().pin_memory()
    R_h = torch.empty((n, n), dtype=torch.float64).pin_memory()
    out_h = torch.empty((n, ml) if cfg["op"] == "form_q" else (k, ml), dtype=torch.float64).pin_memory()
    C_h = C0.cpu().pin_memory() if C0 is not None else None
    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    te = []
    for it in range(max(2, min(args.steps, 10)) + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_s.record(stream)
        A.copy_(A_h, non_blocking=True)
        if C_h is not None:
            C.copy_(C_h, non_blocking=True)
        if world == 1:
            _, tree = T.factor(A, b, s, R=R, tree=tree)
            Rr = R
        else:
            st = tdist.factor(A, b, s, engine=engine, tree=tree, cross=args.cross)
            tree, Rr = st.tree, st.R
        if cfg["op"] == "form_q":
            T.form_q(tree, Q)                            # no communication (butterfly replication)
            out_h.copy_(Q, non_blocking=True)
        else:
            if world == 1:
                T.apply_qt(tree, C)
            else:
                tdist.apply_qt(st, C)
            out_h.copy_(C, non_blocking=True)
        R_h.copy_(Rr, non_blocking=True)
        e_e.record(stream)
        e_e.synchronize()
        if it > 0:
            te.append(e_s.elapsed_time(e_e))
    t_e2e = statistics.mean(te)
    if world > 1:
        t_e2e = max_over_ranks([t_e2e], dev)[0]
    h2d = 8 * m * n + (8 * m * k if C_h is not None else 0)                 # all ranks' slabs
    d2h = 8 * n * n * world + (8 * m * n if cfg["op"] == "form_q" else 8 * m * k)
    e2e = {"value": 2.0 * m * n * n / (t_e2e * 1e-3) / 1e9, "unit": "GFLOP/s (2mn^2 over the whole e2e step)",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e}

    if rank != 0:
        dist.destroy_process_group()
        return 0

    flops = 2.0 * m * n * n
    # dominant kernel = the leaf stage (a2+a3), one launch per step: its algorithmic flops are
    # the Householder QR flops of every local tile, sum(2 h n^2 - 2 n^3/3),
    # over its own launch time from device events on the factor's stream (tsqr_tree_stage_ms)
    tiles = T.plan_export(ml, n, block_rows=b, tile_rows=s, nranks=world, rank=rank)["tile_rows"]
    leaf_flops = float(sum(2.0 * h * n * n - 2.0 * n ** 3 / 3 for h in tiles)) * world
    achieved = leaf_flops / (tl * 1e-3) / 1e12      # TFLOP/s of the leaf kernel (all ranks)
    peak = FP64_PEAK_TFLOPS * world
    pk = measured_peaks()
    bw = pk.get("hbm_gbs", 6555.8)
    t_roof = max(flops / (peak * 1e12), 8.0 * m * n / (bw * 1e9 * world))
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{args.config}_factor")
        except Exception:
            traffic = None
    launches_per_step = kernel_launches(info, n, cfg["op"], world)
    cpu = oracle_sample(cfg) if (world == 1 and not args.no_cpu_baseline) else None
    line = {
        "metric": METRIC, "value": flops / (tf * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ts, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "m": m, "n": n, "block_rows": b,
                   "tile_rows": info["tile_rows"], "ntiles_per_rank": info["ntiles"], "tree_depth": info["depth"],
                   "cross_rounds": info["cross_rounds"], "cross": args.cross if world > 1 else None, "second_op": cfg["op"], "k": k,
                   "l2": "inputs larger than L2 (A = %.0f MB > 126 MB), pristine A restored before each step"
                         % (8e-6 * m * n),
                   "value_timing": "CUDA events around tsqr_factor (leaf kernel + tree kernel) per step, mean of K, "
                                   "max over ranks"},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md); measured DMMA 37.18",
                     "kernel": "leaf stage (k_chain_factor n<=64 / k_wide_leaves n>64), one launch per step",
                     "kernel_ms": tl, "kernel_flops_per_launch": leaf_flops / world, "tree_ms": tt,
                     "frac_of_max_roofline": t_roof / (tf * 1e-3)},
        "ms_factor": tf, "second_op_ms": ts - tf,
        "second_op_gflops": (2.0 * m * n * n - 2.0 * n ** 3 / 3 if cfg["op"] == "form_q" else 4.0 * m * n * k)
        / ((ts - tf) * 1e-3) / 1e9 if ts > tf else None,
        "timed_region_wall_ms": wall * 1e3,
        "clocks": clk, "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cross", default="butterfly", choices=["butterfly", "allgather"],
                    help="N > 1: the cross-GPU R-combine as log2 N pairwise rounds or one all-gather")
    args = ap.parse_args()
    if args.config is None:
        args.config = DEFAULT_CONFIG
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
