#!/usr/bin/env python
"""bench.py -- TSQR factor GFLOP/s (2mn^2 model) and roofline fraction on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Workload (BASELINE.json): the default is config 4 (16,777,216 x 64, kappa = 1e10:
factor + form Q), the largest configuration BASELINE.json quotes the metric on that
fits one GPU; c1/c2/c3/c5 are selectable.  A step is the config's workload
(c1/c2/c4 factor + form Q, c3/c5 factor + apply Q^T to C).

  value        2 m n^2 / t_factor, t_factor the device time of the factor (CUDA events
               on its stream), MEDIAN of the K timed steps, max over ranks
  roofline     the dominant kernel (the leaf stage, one launch per step): its
               algorithmic flops sum(2 h n^2 - 2n^3/3) over its own launch time (events
               on the factor's stream, tsqr_tree_stage_ms) against the FP64 pipe peak
  e2e          the same metric through the public C-ABI with HOST buffers
               (tsqr_qr_host: H2D of A, factor, second op, D2H of R and Q / Q^T C)
  cpu_baseline the CPU oracle (oracle/, plain C, leaves in parallel) on the box's host
               cores, T = all cores and T = 1, on a bounded sample of the same workload

The factor is in place, so the pristine input is restored (device copy, outside the
events) before every step; every config's A but C1's exceeds the 126 MB L2.
N > 1: torchrun, one rank per GPU; the C library's communicator layer runs the
butterfly rounds over NCCL inside one call (tsqr_ctx_factor); the matrix is the
config's global one (strong scaling).  --impl reference times the CPU oracle alone.
"""
from __future__ import annotations

import argparse
import json
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
# configs[3]: the largest configuration BASELINE.json's metric is quoted on that fits one GPU
# (8.6 GB of A; C5 is quoted at 2/4/8 GPUs only)
DEFAULT_CONFIG = "c4"

# FP64 peak for the roofline: B200 has no FP64 tcgen05 kind; DMMA runs at
# the DFMA rate, so the path is bound by the FP64 pipe: 148 SMs x 64 FP64 FMA/clk x 2 flop x
# 1.965 GHz = 37.22 TFLOP/s (derived; MEASURED_PEAKS.json has no FP64 entry).  The bench also
# measures DMMA and DFMA peaks in the run (tsqr_measure_fp64_peak) and reports them beside it.
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
METRIC = "TSQR factor GFLOP/s (2mn^2 model) and fraction of HBM/FP64 roofline"
UNIT = "GFLOP/s"


def kernel_launches(info, n, op, world):
    """Kernels of this repo launched per step (tsqr_api.cu's dispatch): factor, then the second op."""
    multi = info["ntiles"] > 1
    rounds = info["cross_rounds"] if world > 1 else 0
    # the node stages of apply / form Q are one pipelined launch for n <= 224 (else one per step)
    nodes = (1 if multi else 0) if n <= 224 else info["depth"]
    if n <= 64:
        fac = 1 + 1                                   # chain leaves + pipelined tree (or R extraction)
        second = (1 + nodes) if op == "apply_qt" else (2 + nodes)   # leaves+nodes | identity+nodes+leaves
    else:
        fac = 1 + multi + 1                           # leaves + pipelined tree + R extraction
        second = (1 + nodes) if op == "apply_qt" else (3 + nodes)   # | identity+nodes+[X;0]+leaves
    # butterfly rounds: pack + combine per round on the factor; apply: one combine per round + top copy
    cross = 2 * rounds + (2 * rounds if op == "apply_qt" else 0)
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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi's clocks line via NVML, every `period` s on a thread, over the timed region."""

    NAMES = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
             "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0, period=0.005):
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
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.NAMES.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def stop(self):
        if self.nv:
            self._stop.set()
            self.t.join()
        s = self.samples
        return {"sm_mhz": statistics.median(s) if s else None, "sm_min_mhz": min(s) if s else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(s),
                "period_ms": 1e3 * self.period}


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
ORACLE_GFLOPS_PER_THREAD = 2.5       # plain unblocked Householder leaf, long-double sums
SAMPLE_BYTES = 2 << 30               # host copy of the sample: at most 2 GiB of A


def oracle_sample(cfg, seconds, threads, A_dev=None):
    """Time the CPU oracle (as it stands; leaves in parallel on `threads` host threads) on a
    bounded sample of the workload: the first whole row blocks of the config, the same tile
    plan, factor only, sized for about `seconds` of work.  The bytes are the device's (D2H)
    when A_dev is given, else the recipe on the CPU generator."""
    import oracle as orc
    from paper_0808_2664_b200 import api, inputs
    m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
    c = api.plan_info(min(m, b), n, block_rows=b, tile_rows=s)["chunk_rows"]
    per_block = 2.0 * b * n * n
    budget = seconds * ORACLE_GFLOPS_PER_THREAD * 1e9 * threads
    blocks = max(threads, int(budget / per_block)) if m >= b else 1
    blocks = min(blocks, max(1, m // b), max(1, SAMPLE_BYTES // (8 * b * n)))
    rows = blocks * b if m >= b else m
    if A_dev is not None:
        A = A_dev[:, :rows].contiguous().cpu().numpy().T
    else:
        A = inputs.to_numpy_colmajor(make_slab(cfg, 0, rows, "cpu"))
    p = orc.plan(rows, n, b, s, 1, c)
    t0 = time.perf_counter()
    orc.tsqr_factor(A, p, threads=threads, overwrite=True, keep_y1=False)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * rows * n * n / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"oracle tsqr_factor (plain C, long-double sums) on rows 0..{rows} ({blocks} row blocks of "
                      f"{b}, {p.ntiles} leaves, chunk rows {c}) x {n} of the {cfg['desc'].split(':')[0]}, "
                      f"same plan, leaves over {threads} threads",
            "seconds": dt, "cpu_model": cpu_model()}


def cpu_baselines(cfg, A_dev=None, seconds=6.0):
    nproc = host_cores()
    allc = oracle_sample(cfg, seconds, nproc, A_dev)
    one = oracle_sample(cfg, seconds, 1, A_dev) if nproc > 1 else allc
    out = dict(allc)
    out["single_core"] = {k: one[k] for k in ("value", "unit", "cores", "sample", "seconds")}
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    nproc = host_cores()
    per_step = max(1.0, 120.0 / max(1, K + W))          # the whole run within about two minutes
    for _ in range(W):
        oracle_sample(cfg, per_step, nproc)
    vals, secs = [], []
    r = None
    for _ in range(K):
        r = oracle_sample(cfg, per_step, nproc)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "sample": r["sample"]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nproc, "kind": "oracle", "sample": r["sample"],
                             "cpu_model": r["cpu_model"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_0808_2664_b200 as T
    from paper_0808_2664_b200 import dist as tdist

    N = args.gpus
    rank, world = 0, 1
    if N > 1:
        # the communicator's NCCL init lines (rank count, transport) go to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
    dmma_pk, dfma_pk = T.measure_fp64_peak()              # this GPU, now (outside the timed region)
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

    t_factor, t_step, t_leaf, t_tree = [], [], [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index).start()
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
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    med = statistics.median
    tf, ts, tl, tt = med(t_factor), med(t_step), med(t_leaf), med(t_tree)
    tf_min, tf_mean = min(t_factor), statistics.mean(t_factor)
    if world > 1:
        tf, ts, tl, tt, tf_min, tf_mean = max_over_ranks([tf, ts, tl, tt, tf_min, tf_mean], dev)

    # ---- e2e through the public C-ABI with HOST buffers (pinned): copies inside the timed region
    A_h = A0.cpu().pin_memory()
    out_h = torch.empty((n, ml) if cfg["op"] == "form_q" else (k, ml), dtype=torch.float64).pin_memory()
    C_h = C0.cpu().pin_memory() if C0 is not None else None
    R_h = torch.empty((n, n), dtype=torch.float64).pin_memory()
    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    te = []
    hq = T.HostQR() if world == 1 else None
    for it in range(max(2, min(args.steps, 5)) + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if C_h is not None:
            out_h.copy_(C_h)                              # apply Q^T overwrites its C (outside the events)
        e_s.record(stream)
        if world == 1:                                    # one C call: H2D, factor, second op, D2H
            if cfg["op"] == "form_q":
                hq(A_h, b, s, R_host=R_h, Q_host=out_h)
            else:
                hq(A_h, b, s, R_host=R_h, C_host=out_h, want_q=False)
        else:                                             # the collective calls on the rank's slab
            A.copy_(A_h, non_blocking=True)
            if C is not None:
                C.copy_(out_h, non_blocking=True)
            st = tdist.factor(A, b, s, engine=engine, tree=tree, cross=args.cross)
            tree = st.tree
            if cfg["op"] == "form_q":
                T.form_q(tree, Q)                        # communication-free
                out_h.copy_(Q, non_blocking=True)
            else:
                tdist.apply_qt(st, C)
                out_h.copy_(C, non_blocking=True)
            R_h.copy_(st.R, non_blocking=True)
        e_e.record(stream)
        e_e.synchronize()
        if it > 0:
            te.append(e_s.elapsed_time(e_e))
    if hq is not None:
        hq.free()
    del A_h, out_h, C_h, R_h                              # pinned host memory back before the CPU baseline
    t_e2e = med(te)
    if world > 1:
        t_e2e = max_over_ranks([t_e2e], dev)[0]
    h2d = 8 * m * n + (8 * m * k if C0 is not None else 0)                 # all ranks' slabs
    d2h = 8 * n * n * world + (8 * m * n if cfg["op"] == "form_q" else 8 * m * k)
    e2e = {"value": 2.0 * m * n * n / (t_e2e * 1e-3) / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e,
           "path": ("tsqr_qr_host (one C-ABI call: H2D of A%s, factor, %s, D2H of R and %s from pinned host "
                    "memory), median of %d, CUDA events on its stream") % (
               " and C" if C0 is not None else "", cfg["op"], "Q" if cfg["op"] == "form_q" else "Q^T C", len(te))
           if world == 1 else "torch H2D of the slab + tsqr_ctx_* collective calls + D2H, max over ranks"}

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
    bw = measured_peaks().get("hbm_gbs", 6534.5)
    t_roof8 = max(flops / (peak * 1e12), 8.0 * m * n / (bw * 1e9 * world))
    t_roof16 = max(flops / (peak * 1e12), 16.0 * m * n / (bw * 1e9 * world))
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            traffic = tj.get(f"{args.config}_factor")
            traffic_src = tj.get("source")
        except Exception:
            traffic = None
    # the second op against its own roofline: form Q at DORGQR's count 2mn^2 - 2n^3/3 with Y read
    # and Q written (16mn bytes), Q^T C at 4mnk with Y read and C read and written (8m(n + 2k))
    t2 = ts - tf
    second_roof = None
    if t2 > 0:
        if cfg["op"] == "form_q":
            f2, b2 = 2.0 * m * n * n - 2.0 * n ** 3 / 3, 16.0 * m * n
            models = ("2mn^2 - 2n^3/3", "16mn (Y in, Q out)")
        else:
            f2, b2 = 4.0 * m * n * k, 8.0 * m * (n + 2 * k)
            models = ("4mnk", "8m(n + 2k) (Y in, C in and out)")
        tf2, tb2 = f2 / (peak * 1e12), b2 / (bw * 1e9 * world)
        second_roof = {"op": cfg["op"], "ms": t2, "flops_model": models[0], "bytes_model": models[1],
                       "achieved_tflops": f2 / (t2 * 1e-3) / 1e12, "achieved_gbs": b2 / (t2 * 1e-3) / 1e9,
                       "bound": "alu" if tf2 >= tb2 else "hbm", "frac": max(tf2, tb2) / (t2 * 1e-3),
                       "timing": "median step minus median factor (CUDA events on the step's stream)"}
    launches_per_step = kernel_launches(info, n, cfg["op"], world)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baselines(cfg, A0)
    l2 = ("A = %.0f MB > 126 MB L2 (inputs larger than L2); the pristine A is restored before each step"
          % (8e-6 * m * n)) if 8 * m * n > 126e6 else \
         ("A = %.2f MB fits the 126 MB L2: C1 is a correctness (latency-bound) config; the pristine A is "
          "restored before each step" % (8e-6 * m * n))
    line = {
        "metric": METRIC, "value": flops / (tf * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ts, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "m": m, "n": n, "block_rows": b,
                   "tile_rows": info["tile_rows"], "chunk_rows": info["chunk_rows"],
                   "ntiles_per_rank": info["ntiles"], "tree_depth": info["depth"],
                   "cross_rounds": info["cross_rounds"], "cross": args.cross if world > 1 else None,
                   "second_op": cfg["op"], "k": k, "l2": l2,
                   "value_timing": "CUDA events around tsqr_factor (leaf kernel + tree kernel%s) per step, "
                                   "median of K (min and mean beside), max over ranks"
                                   % (" + butterfly rounds" if world > 1 else "")},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md 8); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "peak_measured_now": {"dmma_tflops": dmma_pk, "dfma_tflops": dfma_pk},
                     "kernel": "leaf stage (k_chain_factor n<=64 / k_wide_leaves n>64), one launch per step",
                     "kernel_ms": tl, "kernel_flops_per_launch": leaf_flops / world,
                     "kernel_frac_of_measured_dmma": achieved / (dmma_pk * world) if dmma_pk else None,
                     "tree_ms": tt,
                     "factor_frac_8mn_roofline": t_roof8 / (tf * 1e-3),
                     "factor_frac_16mn_roofline": t_roof16 / (tf * 1e-3)},
        "ms_factor": tf, "ms_factor_min": tf_min, "ms_factor_mean": tf_mean, "second_op_ms": ts - tf,
        "second_op_gflops": (2.0 * m * n * n - 2.0 * n ** 3 / 3 if cfg["op"] == "form_q" else 4.0 * m * n * k)
        / ((ts - tf) * 1e-3) / 1e9 if ts > tf else None,
        "second_op_roofline": second_roof,
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
