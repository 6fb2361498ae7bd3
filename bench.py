#!/usr/bin/env python
"""Benchmark: theta-instantiations/s of a parametric H^2 matrix at n = 2^18 (3D)
(BASELINE.json configs[2], "C3"), one step = instantiate(theta) + one MVM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (rows sharded, NCCL all-gather of y)

Data: seeded synthetic (points U[0,1)^3, theta draws of harness.cpp:254-260,
x ~ N(0,1)); random-free otherwise. The near-field stream (113 GB at C3) is
far larger than the 126 MB L2, so no L2 flush is needed between steps.

`--impl reference` times the reference's CPU path (the oracle port of
proj/src/phmatrix.cpp:168-269; the reference itself needs Eigen3 and cannot
be built here) on a bounded sample of the same workload, extrapolated.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[2] (the metric's n = 2^18, 3D configuration)
    "c3": dict(n=262144, d=3, family="e", box=(0.05, 0.5), l_max=4, p_s=4, p_theta=8, eta=1.0, fmt="h2",
               points="uniform"),
    # BASELINE.json configs[1]
    "c2": dict(n=65536, d=2, family="m32", box=(0.05, 0.5), l_max=5, p_s=8, p_theta=10, eta=1.0, fmt="h2",
               points="uniform"),
    # BASELINE.json configs[0] (CPU-runnable PR1 case; param-H)
    "c1": dict(n=4096, d=2, family="gauss", box=(0.1, 1.0), l_max=3, p_s=6, p_theta=8, eta=1.0, fmt="h",
               points="uniform"),
    # BASELINE.json configs[4] (C5): the C3 matrix, 4096 thetas sharded over
    # GPUs with no communication, each instantiated and applied to 10 vectors
    "c5": dict(n=262144, d=3, family="e", box=(0.05, 0.5), l_max=4, p_s=4, p_theta=8, eta=1.0, fmt="h2",
               points="uniform", sweep=True, rhs=10, n_theta=4096, theta_batch=16),
    # BASELINE.json configs[3] (C4, the 8-GPU DMMA case): n = 2^20 points from
    # a 16-Gaussian mixture, leaf 32, Matern-5/2 with theta = (l, sigma^2) on
    # an 8 x 6 grid, 64 right-hand sides. Fits 8 x B200 only with symmetric
    # near storage sharded over the ranks (about 150 GB of snapshots + D per
    # rank); run under torchrun --nproc-per-node 8.
    "c4": dict(n=1048576, d=3, family="m52", box=(0.05, 0.5), boxes=[(0.05, 0.5), (0.5, 2.0)], amplitude=True,
               l_max=5, p_s=4, p_theta=[8, 6], eta=1.0, fmt="h2", points="mixture", rhs=64),
    # profiling proxy of C4's near field on one GPU (not a BASELINE config):
    # the same mixture and kernel at n = 2^18, l_max 4 -- clustered leaves of
    # up to a few thousand rows, as in C4 -- small enough for ncu replays
    "c4p": dict(n=262144, d=3, family="m52", box=(0.05, 0.5), boxes=[(0.05, 0.5), (0.5, 2.0)], amplitude=True,
                l_max=4, p_s=4, p_theta=[8, 6], eta=1.0, fmt="h2", points="mixture", rhs=64),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=16, help="1/f of near/far blocks timed on the CPU")
    ap.add_argument("--rhs", type=int, default=0, help="right-hand sides per MVM (default: the config's)")
    ap.add_argument("--theta-batch", type=int, default=0,
                    help="sweeps: thetas instantiated per snapshot pass (default: the config's; 1 = one at a time)")
    return ap.parse_args()


def theta_draws(lo, hi, count, seed):
    # harness.cpp:254-260: Rng(mix_seed(seed, 0x74686574)).uniform(lo, hi)
    import paper_2511_03109_b200 as ph

    return ph.theta_draws(lo, hi, count, seed)


def make_points(ph, c, seed):
    if c["points"] == "uniform":
        return ph.generate_points(c["n"], c["d"], seed)
    return ph.generate_mixture_points(c["n"], c["d"], 16, 0.05, seed)


def theta_vectors(c, count, seed, draws=None):
    """count theta vectors: harness draws per parameter (harness.cpp:254-260),
    the k-th parameter from seed + k. `draws` replaces the product's
    generator (the reference arm uses the reference's own Rng)."""
    boxes = c.get("boxes", [c["box"]])
    draws = draws or theta_draws
    cols = [draws(lo, hi, count, seed + k) for k, (lo, hi) in enumerate(boxes)]
    return [[float(col[i]) for col in cols] for i in range(count)]


def make_cfg(ph, c, rank=0, world=1, near_mode=None):
    spec = ph.KernelSpec(ph.Family.from_id(c["family"]), c.get("boxes", [c["box"]]), amplitude=c.get("amplitude", False))
    return ph.PHConfig(spec=spec, l_max=c["l_max"],
                       p_s=c["p_s"], p_theta=c["p_theta"], eta=c["eta"], eps=1e-5, seed=0,
                       near_mode=ph.NearMode.SNAPSHOT if near_mode is None else near_mode,
                       shard_rank=rank, shard_count=world)


def algorithmic_bytes(info, c, n_classes_bytes):
    """per-theta instantiate and per-vector H^2 MVM bytes."""
    P = info["P"]
    b_inst = 8 * info["near_stream_elems"] + n_classes_bytes
    n = c["n"]
    # near term: the D entries actually stored and streamed (symmetric storage
    # reads each sigma <= tau block once for both products)
    b_mvm = 8 * (info["near_stored"] + 2 * n + c["d"] * c["p_s"] * n + c["d"] * c["p_s"] ** 2 * info["nodes"]
                 + info["n_classes"] * P * P + 2 * P * info["nodes"])
    return b_inst, b_mvm


class Clocks:
    """SM clock / throttle-reason sampling during the timed region
    (B200_PROFILING.md clocks line): NVML polled every 5 ms from a thread
    (the device found by PCI bus id), nvidia-smi -lms as the fallback. The
    sampler is running before the warm-up starts, so short timed regions
    still get samples."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        self.window = (0.0, float("inf"))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.device)
            bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _poll(self):
        nv, h = self.nvml
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                row = [str(sm), str(mx), "%.1f" % pw, hex(rs)] + ["Active" if rs & b else "Not Active" for b in bits]
                self.rows.append((time.time(), row))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "50"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except FileNotFoundError:
                self.proc = None
        # wait (bounded) for the first sample so the timed region is covered
        t_end = time.time() + 3.0
        while (self.nvml or self.proc) and not self.rows and time.time() < t_end:
            time.sleep(0.01)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append((time.time(), parts))

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.nvml or self.proc:
            self.t.join(timeout=5)

    def summary(self):
        inside = [r for t, r in self.rows if self.window[0] <= t <= self.window[1]]
        rows = inside or [r for _, r in self.rows]
        self.rows_used = rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return self._summ(rows, in_window=bool(inside))

    def _summ(self, rows, in_window):
        self.rows = rows
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "in_timed_window": in_window,
                "source": "nvml" if self.nvml else "nvidia-smi"}


def measured_traffic(kernel, config, world):
    """DRAM bytes (read + write) per launch of `kernel` and where they come
    from: the committed ncu --set full capture of this bench's c3 step at
    N=1 (dram__bytes_read.sum + dram__bytes_write.sum; the newest
    profiles/r*_traffic.json). ncu cannot run inside the timed bench, so this
    is the captured number, not a live one; None for other workloads."""
    prof = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    files = sorted(f for f in os.listdir(prof) if f.endswith("_traffic.json")) if os.path.isdir(prof) else []
    if config != "c3" or world != 1 or not files:
        return None, None
    rec = json.load(open(os.path.join(prof, files[-1]))).get(kernel)
    return (rec["traffic_bytes_per_launch"], f"ncu --set full capture, profiles/{files[-1]}") if rec else (None, None)


def dmma_peak_tflops():
    """Measured fp64 tensor-core (mma.sync f64) peak of this part."""
    try:
        with open(os.path.join(ROOT, "profiles", "dmma_peak.json")) as f:
            return float(json.load(f)["dmma_f64_tflops"])
    except Exception:
        return None


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------ CPU baseline
def reference_cpu(c, steps, warmup, stride, seed, m=1, budget_s=None):
    """The REFERENCE ITSELF (oracle/_ref/libphmat_ref.so: the unmodified
    proj/src compiled against oracle/eigen_shim) on this host's cores, with no
    product code loaded: the reference generates the points
    (harness.cpp:174-181), builds its own parametric matrix (offline_h /
    offline_h2 with its TT-cross; snapshot-mode TTs by near_oracle for a
    seeded 1/stride sample of near blocks) and times its own instantiate
    (parallel_for over PHMAT_THREADS = all cores) + apply (single-threaded by
    design, phmatrix.cpp:227-269) per step. Each step is a bounded sample:
    the sampled matrix (1/stride of the near and far blocks, every class) and
    a fixed-cost matrix (every class, one far block per sigma, so the basis
    passes run in full) are both timed, and the per-theta cost is
    fixed + (sample - fixed) * stride. m right-hand sides cost m applies (the
    reference's apply takes one vector, phmatrix.hpp:95-100)."""
    from oracle import pyref as pr

    cores = os.cpu_count() or 1
    os.environ["PHMAT_THREADS"] = str(cores)
    if c["family"] not in pr.RefBench.FAMILIES or c.get("points", "uniform") != "uniform" or "boxes" in c:
        return None
    t0 = time.time()
    rb = pr.RefBench(c["n"], c["d"], seed, c["fmt"] == "h2", c["family"], c["box"], c["l_max"], c["p_s"],
                     c["p_theta"], c["eta"], 1e-5, stride, cores)
    setup_s = time.time() - t0
    thetas = theta_vectors(c, max(steps + warmup, 1), seed, draws=pr.theta_draws)
    X = np.stack([pr.generate_normal(c["n"], seed + 1 + j) for j in range(m)], axis=1)
    per, wall = [], []
    for s in range(warmup + steps):
        w0 = time.time()
        ti, ta = rb.step(0, thetas[s % len(thetas)], X)
        fi, fa = rb.step(1, thetas[s % len(thetas)], X)
        w1 = time.time()
        if s >= warmup:
            fixed, sample = fi + fa, ti + ta
            per.append(fixed + max(0.0, sample - fixed) * stride)
            wall.append(w1 - w0)
    t = float(np.median(per))
    return {"value": 1.0 / t, "unit": "theta/s", "cores": cores, "kind": "reference",
            "steps_timed": steps, "ms_per_sampled_step": 1000.0 * float(np.mean(wall)),
            "setup_s": setup_s,
            "sample": f"the reference itself (unmodified proj/src, g++ -O3, Eigen API shim): instantiate over all "
                      f"classes + 1/{stride} of near blocks ({rb.near_frac:.4f} of near entries, {rb.near_blocks} "
                      f"blocks) and 1/{stride} of far blocks ({rb.far_blocks}), {cores} threads; {m} apply(s), "
                      f"single-threaded as the reference; per theta = fixed + (sample - fixed) x {stride}, "
                      f"fixed = every class + one far block per sigma (full basis passes); median of {steps} "
                      f"thetas"}


# --------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2511_03109_b200 as ph

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the multi-rank path on a one-GPU box: every rank on
    # cuda:0, gloo for the exchange (never a performance number)
    same_gpu = os.environ.get("PHM_BENCH_FUNCTIONAL_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[args.config]
    sweep = c.get("sweep", False)          # C5: thetas sharded over ranks, no communication
    m = args.rhs or c.get("rhs", 1)        # right-hand sides per MVM
    row_shard = world > 1 and not sweep    # C3 at N GPUs: leaf rows sharded, y all-gathered
    ctx = ph.Context(local)
    # A real (non-legacy) stream shared by torch (events, NCCL ordering) and
    # every kernel the library launches.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    pts = make_points(ph, c, args.seed)
    cfg = make_cfg(ph, c, rank if row_shard else 0, world if row_shard else 1)
    t0 = time.time()
    pm = ph.offline_h2(pts, cfg, ctx) if c["fmt"] == "h2" else ph.offline_h(pts, cfg, ctx)
    build_s = time.time() - t0
    info = pm.info()
    n = c["n"]
    thetas = theta_vectors(c, c.get("n_theta", 32), args.seed)
    xs = np.stack([ph.generate_normal(n, args.seed + 1 + j) for j in range(m)])  # (m, n) = column-major n x m
    x_host = torch.from_numpy(xs).pin_memory()
    x_dev = x_host.cuda()
    y_dev = torch.empty((m, n), dtype=torch.float64, device="cuda")
    rows = info["row_end"] - info["row_begin"]
    if row_shard:
        # the library's own communicator: the sharded step runs its x-hat and
        # y all-reduces inside phm_instantiate_apply_sharded (NCCL over
        # NVLink; gloo on host copies for the one-GPU functional check)
        from paper_2511_03109_b200.dist import host_allreduce_comm, nccl_comm

        comm = host_allreduce_comm() if same_gpu else nccl_comm(ctx)
    inst = ph.instantiate(pm, thetas[0])
    # sweeps: tb thetas per step, instantiated by one snapshot pass (K1 batch)
    tb = (args.theta_batch or c.get("theta_batch", 1)) if sweep else 1
    binsts = ph.instantiate_batch(pm, [thetas[b] for b in range(tb)]) if tb > 1 else None

    def theta_of(s):
        return thetas[(s * world + rank) % len(thetas)] if sweep else thetas[s % len(thetas)]

    def step(s):
        if binsts is not None:
            ph.reinstantiate_batch(binsts, [theta_of(s * tb + b) for b in range(tb)])
            for b in range(tb):
                binsts[b].apply_device(x_dev.data_ptr(), y_dev.data_ptr(), m)
            return
        if not row_shard:
            # instantiate(theta_s) + MVM as one overlapped schedule
            inst.instantiate_apply_device(theta_of(s), x_dev.data_ptr(), y_dev.data_ptr(), m)
        else:
            # this rank's shard of the step (its owner leaves' near pairs,
            # both ways; its rows' far field; its share of the forward pass)
            # with both exchanges, one library call
            inst.instantiate_apply_sharded_device(comm, theta_of(s), x_dev.data_ptr(), y_dev.data_ptr(), m)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        for s in range(args.warmup):
            step(s)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # `value`: per-kernel timers off, so the step replays as one CUDA graph
        ctx.enable_timing(False)
        launches0 = ctx.launches
        torch.cuda.synchronize()
        tw0 = time.time()
        ev0.record(stream)
        for s in range(args.steps):
            step(args.warmup + s)
        ev1.record(stream)
        torch.cuda.synchronize()
        tw1 = time.time()
        time.sleep(0.05)  # the sampler's last row of the window
        clk.mark(tw0, tw1)
        launches = ctx.launches - launches0
        ms = ev0.elapsed_time(ev1)
        # the same K steps again with a CUDA event pair around every kernel
        # launch (direct launches): the per-kernel times the roofline uses
        ctx.enable_timing(True)
        ctx.reset_timers()
        ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ek0.record(stream)
        for s in range(args.steps):
            step(args.warmup + s)
        ek1.record(stream)
        torch.cuda.synchronize()
        ms_timed_loop = ek0.elapsed_time(ek1)
    # dominant kernel: the fused near-field pass (instantiate + GEMV) when the
    # step runs it, else the plain K1 instantiate stream
    k1_name, k1_desc = "near_inst_mvm", "k_near_tma (K1+K6 fused TMA pass: forms, stores and applies D)"
    k1_ms, k1_n = ctx.timer(k1_name)
    if k1_n == 0:
        k1_name = "near_inst"
        k1_desc = ("k_inst_tma (K1 near instantiate over TMA)" if 8 * info["near_stream_elems"] > 1.1e9 and
                   os.environ.get("PHM_K1_TMA", "1") != "0" else "k_inst_flat (K1 near instantiate)")
        k1_ms, k1_n = ctx.timer(k1_name)
    timers = {}
    for name in ("near_inst_mvm", "near_inst", "class_inst", "near_w", "near_mvm", "near_gather", "near_mrhs", "coupling",
                 "coupling_reduce", "leaf_fwd", "up", "down", "leaf_bwd", "gather", "scatter", "far_h"):
        t, cnt = ctx.timer(name)
        if cnt:
            timers[name] = {"ms_per_launch": t / cnt, "launches": cnt}
    ctx.enable_timing(False)

    def time_loop(fn):
        # warm first: the first call of a launch sequence runs directly and the
        # second captures its CUDA graph (host time that would stall the stream)
        for s in range(3):
            fn(s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for s in range(args.steps):
            fn(s)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    # phase split of the same step (same stream, CUDA events)
    inst_ms = time_loop(lambda s: inst.reinstantiate(theta_of(s)))
    # The MVM phase starts after 1 s of idle GPU: right behind the step and
    # instantiate loops it inherits their transient sw_power_cap clock dips
    # (C3: 1.94 ms per apply straight after 25 fused steps, 1.69 ms after a
    # 1 s pause, the same as a fresh process; tools/apply_probe.py --idle).
    if not row_shard:
        torch.cuda.synchronize()
        time.sleep(1.0)
    apply_ms = (time_loop(lambda s: inst.apply_device(x_dev.data_ptr(), y_dev.data_ptr(), m))
                if not row_shard else None)
    # per-kernel split of the apply phase (separate loop: the timers add events)
    apply_timers = {}
    if not row_shard:
        ctx.enable_timing(True)
        ctx.reset_timers()
        time_loop(lambda s: inst.apply_device(x_dev.data_ptr(), y_dev.data_ptr(), m))
        for name in ("near_mvm", "near_gather", "near_mrhs", "coupling", "coupling_reduce", "leaf_fwd", "up", "down",
                     "leaf_bwd", "gather", "scatter", "far_h"):
            t, cnt = ctx.timer(name)
            if cnt:
                apply_timers[name] = {"ms_per_launch": t / cnt, "launches": cnt}
        ctx.enable_timing(False)
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())

    # e2e through the public API with host buffers (rank-local)
    e2e = None
    if True:
        y_host = torch.empty((m, n), dtype=torch.float64).pin_memory()
        xh, yh = x_host.numpy(), y_host.numpy()
        from ctypes import POINTER, c_double

        def e2e_step(s):
            if binsts is not None:
                ph.reinstantiate_batch(binsts, [theta_of(s * tb + b) for b in range(tb)])
                for b in range(tb):
                    ph._check(ph.lib().phm_apply(binsts[b]._h, xh.ctypes.data_as(POINTER(c_double)), n,
                                                 yh.ctypes.data_as(POINTER(c_double)), m))
                return
            if row_shard:
                # host x -> every rank, sharded step + all-reduce, y -> host
                x_dev.copy_(x_host, non_blocking=True)
                step(s)
                y_host.copy_(y_dev, non_blocking=True)
                stream.synchronize()
                return
            th = np.array(theta_of(s))
            ph._check(ph.lib().phm_instantiate_apply(inst._h, th.ctypes.data_as(POINTER(c_double)), th.size,
                                                     xh.ctypes.data_as(POINTER(c_double)), n,
                                                     yh.ctypes.data_as(POINTER(c_double)), m))

        for s in range(args.warmup):
            e2e_step(s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s in range(args.steps):
            e2e_step(s)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": (world if sweep else 1) * tb * args.steps * 1000.0 / e_ms, "unit": "theta/s",
               "h2d_bytes_per_step": tb * (8 * n * m + 8), "d2h_bytes_per_step": tb * 8 * n * m}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = reference_cpu(c, 3, 1, args.cpu_sample, args.seed, m)

    if rank == 0:
        peak, peak_kind = measured_peak()
        ncls = info["n_classes"]
        cls_bytes = 0
        for k in range(ncls):  # middle cores + L/R read, H and C written, per class
            cores = pm.coupling_cores(k)
            mid = cores[c["d"]]
            rl, rr = mid.shape[0], mid.shape[2]
            cls_bytes += 8 * (mid.size + info["P"] * (rl + rr) + rl * rr + info["P"] ** 2)
        b_inst, b_mvm = algorithmic_bytes(info, c, cls_bytes)
        k1_avg = k1_ms / max(1, k1_n)
        traffic, traffic_src = measured_traffic(k1_desc.split()[0], args.config, world)
        k1_bytes = 8 * info["near_stream_elems"]  # R slab reads + 1 write per stored near entry
        if binsts is not None:  # batched K1: R slab reads + one write per theta of the batch
            k1_desc = "k_inst_flat_batch (K1 for %d thetas per snapshot pass)" % min(tb, 16)
            r_snap = round(info["near_stream_elems"] / max(1, info["near_stored"])) - 1
            k1_bytes = 8 * info["near_stored"] * (r_snap + min(tb, 16))
        achieved = k1_bytes / (k1_avg * 1e-3) / 1e9 if k1_avg > 0 else float("nan")
        mvm_ms = apply_ms
        # the near-field GEMV kernel of apply alone: reads every stored entry once
        nm = apply_timers.get("near_mvm")
        near_gemv = None
        if nm and m == 1:
            gb = 8 * info["near_stored"] / (nm["ms_per_launch"] * 1e-3) / 1e9
            near_gemv = {"kernel": ("k_near_tma_apply (K6 over TMA)" if os.environ.get("PHM_NEAR_GEMV", "1") == "0" else
                                    "k_near_gemv_lean (K6 over TMA, two 5-warp CTAs per SM beside the coupling)"),
                         "ms": nm["ms_per_launch"],
                         "bytes": 8 * info["near_stored"], "GB_s": gb, "frac": gb / peak}
        # fp64 tensor-core (DMMA) work of the MVM: coupling GEMMs and, for
        # block right-hand sides, the near-field contraction
        cp = timers.get("coupling")
        k9 = timers.get("near_mrhs")
        dmma_peak = dmma_peak_tflops()
        cp_tf = (2.0 * info["n_far"] * info["P"] ** 2 * m / (cp["ms_per_launch"] * 1e-3) / 1e12) if cp else None
        k9_tf = (2.0 * info["near_entries"] * m / (k9["ms_per_launch"] * 1e-3) / 1e12) if k9 else None
        mvm_gflop = ((2.0 * info["n_far"] * info["P"] ** 2 if c["fmt"] == "h2" else 0.0)
                     + 2.0 * info["near_entries"]) * m / 1e9
        dmma = {
            "note": ("useful fp64 flop over each kernel's event-timed duration inside the step, where it "
                     "time-shares the SMs with the near pass (the fused step's coupling is a capped grid "
                     "resident beside it); DMMA pipe utilisation of the kernels alone: profiles/r0*_full_summary.txt"),
            "peak_tflops": dmma_peak, "peak_source": "profiles/dmma_peak.json (tools/dmma_probe.cu)",
            "coupling_tflops_in_step": cp_tf,
            "coupling_frac_of_peak": cp_tf / dmma_peak if cp_tf and dmma_peak else None,
            "near_mrhs_tflops_in_step": k9_tf,
            "near_mrhs_frac_of_peak": k9_tf / dmma_peak if k9_tf and dmma_peak else None,
        }
        timing_note = ("kernel launch times from CUDA events around each launch, over a second pass "
                       "of the same K steps (value's pass runs without them, as CUDA graphs)")
        roofline = {"bound": "hbm", "kernel": k1_desc, "achieved": achieved,
                    "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                    "traffic_source": traffic_src, "peak_kind": peak_kind, "bytes_per_launch": k1_bytes,
                    "avg_launch_ms": k1_avg, "timing": timing_note,
                    "ms_per_step_event_pass": ms_timed_loop / args.steps}
        extra = {}
        if cp and dmma_peak and cp["ms_per_launch"] * cp["launches"] > k1_ms:
            # block right-hand sides (C5): the coupling's fp64 DMMA GEMMs outweigh the snapshot
            # stream, so the dominant kernel is tensor-bound; the HBM line of K1 stays beside it
            cp_flop = 2.0 * info["n_far"] * info["P"] ** 2 * m
            extra["roofline_hbm"] = roofline
            roofline = {"bound": "tensor", "kernel": "k_coupling_mma (K5: C_k x-hat on fp64 mma.sync m16n8k4)",
                        "achieved": cp_tf, "peak": dmma_peak, "unit": "TFLOP/s", "frac": cp_tf / dmma_peak,
                        "traffic": None,
                        "peak_kind": "measured fp64 DMMA peak, profiles/dmma_peak.json (tools/dmma_probe.cu); "
                                     "MEASURED_PEAKS.json holds bf16 only, and sm_100 has no tcgen05 f64 kind",
                        "flops_per_launch": cp_flop, "avg_launch_ms": cp["ms_per_launch"], "timing": timing_note,
                        "ms_per_step_event_pass": ms_timed_loop / args.steps}
        what, config = describe(args, c, m, tb, world)
        line = {
            "metric": what,
            "value": (world if sweep else 1) * tb * args.steps * 1000.0 / ms,
            "unit": "theta/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "thetas_per_step": tb,
            "higher_is_better": True,
            "scaling": "weak" if sweep else "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded uniform points, harness theta draws, x~N(0,1))",
            "config": config,
            "roofline": roofline,
            "phases": {"instantiate_ms": inst_ms, "apply_ms": apply_ms,
                       "instantiate_GB_s": b_inst / (inst_ms * 1e-3) / 1e9},
            "mvm": {"ms": mvm_ms, "algorithmic_bytes": b_mvm,
                    "GB_s": b_mvm / (mvm_ms * 1e-3) / 1e9 if mvm_ms else None,
                    "frac_of_hbm": (b_mvm / (mvm_ms * 1e-3) / 1e9) / peak if mvm_ms else None,
                    # the MVM's second resource: fp64 flop of the coupling (2 |far| P^2 m, only for
                    # H^2) and of the near product (2 per entry and RHS), against the measured
                    # fp64 peak (DMMA and DFMA share one pipe on this part)
                    "fp64_gflop": mvm_gflop,
                    "fp64_ms_at_peak": (mvm_gflop / dmma_peak) if dmma_peak else None,
                    "hbm_ms_at_peak": b_mvm / peak / 1e6},
            **extra,
            "near_gemv": near_gemv,
            "apply_kernels": apply_timers,
            "dmma": dmma,
            "instantiate_algorithmic_bytes": b_inst,
            "kernels": timers,
            "gpu_launches": launches,
            "build_s": build_s,
            "structure": {k: info[k] for k in ("n_near", "n_far", "n_classes", "c_sp", "near_entries", "near_stored",
                                               "device_bytes")},
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def describe(args, c, m, tb, world):
    """The metric name and config dict both arms print (same workload)."""
    n = c["n"]
    sweep = c.get("sweep", False)
    where = "n=2^%d, %dD" % (n.bit_length() - 1, c["d"]) if n & (n - 1) == 0 else "n=%d, %dD" % (n, c["d"])
    fmt_name = "H2" if c["fmt"] == "h2" else "H"
    what = ("theta/s (instantiate + %d-RHS %s MVM per theta) at %s, theta sweep sharded over GPUs"
            % (m, fmt_name, where) if sweep else
            "theta-instantiations/s (instantiate + %s MVM per theta) at %s" % (fmt_name, where) if m == 1 else
            "theta/s (instantiate + %d-RHS %s MVM per theta) at %s" % (m, fmt_name, where))
    config = {"workload": f"{args.config}: n={n} d={c['d']} {c['fmt']} kernel={c['family']} "
                          f"l_max={c['l_max']} p_s={c['p_s']} p_theta={c['p_theta']} eta={c['eta']} "
                          f"near=snapshot rhs={m}" + (f" theta_batch={tb}" if tb > 1 else ""),
              "parallelism": ("theta-sharded replicas" if sweep else f"rows sharded over {world}"),
              "l2": "inputs (near snapshots) larger than L2; no flush needed"}
    return what, config


def run_reference(args):
    """--impl reference: the reference's own CPU path (compiled from the
    unmodified sources, oracle/_ref) on rank 0's host cores; no product code
    is imported. Other ranks exit without work."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    c = CONFIGS[args.config]
    steps = max(1, args.steps)
    m = args.rhs or c.get("rhs", 1)
    tb = (args.theta_batch or c.get("theta_batch", 1)) if c.get("sweep", False) else 1
    what, config = describe(args, c, m, tb, world)
    cpu = reference_cpu(c, steps, args.warmup, args.cpu_sample, args.seed, m)
    if cpu is None:
        print(json.dumps({"impl": "reference", "unavailable": f"config {args.config} is outside the reference's "
                          "kernel families / point generators (SURVEY.md Appendix A)"}))
        return
    config["parallelism"] = "reference CPU path on the host cores of rank 0"
    line = {
        "impl": "reference",
        "metric": what,
        "value": cpu["value"], "unit": "theta/s", "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": cpu["ms_per_sampled_step"], "higher_is_better": True,
        "scaling": "weak" if c.get("sweep", False) else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded uniform points, harness theta draws, x~N(0,1))",
        "config": config,
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "theta/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "ms_per_step is the wall time of one bounded sampled step (sampled + fixed-cost reference runs); "
                "value is the per-theta rate of the whole workload from that sample (cpu_baseline.sample)",
    }
    print(json.dumps(line))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
