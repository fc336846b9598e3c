#!/usr/bin/env python3
"""Benchmark: hybrid-dealiased convolution on B200 (BASELINE.json metric:
"hybrid-dealiased conv output samples/s and % HBM roofline, 2D 4096^2 c128").

Workload (BASELINE.json configs[2]): complex128
4096x4096 image (re ~ U[0,1), im = 0) convolved with a 255x255 Gaussian kernel
(sigma 40) plus 1e-3 uniform noise; full linear output 4350x4350.  A step is one
complete hybrid-dealiased convolution (all three passes) through the C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3] [--no-tune] [--no-cpu]

N > 1: one process per GPU (bench.py spawns them with torch.distributed.run when
it is not already under torchrun).  The headline is ONE problem slab-decomposed
over the ranks (strong scaling; the NCCL all-to-alls run inside libhdconv,
hd_conv2d_dist / hd_conv3d_dist, overlapped chunk by chunk with the passes);
`weak_scaling` reports every rank convolving its own whole problem.  Timing is
the max over ranks of CUDA-event time.  `--impl reference` times the CPU
oracle (oracle/, plain direct convolution) on the host cores on a bounded
sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "hybrid-dealiased conv output samples/s and % HBM roofline, 2D 4096² c128"
UNIT = "output samples/s"
FALLBACK_HBM = 6650.0


# ---------------------------------------------------------------------------
def workload(cfg: int):
    d = synth.config_inputs(cfg)
    f, g = d["f"], d["g"]
    nd = d["ndim"]
    Lf, Lg = list(f[0].shape[-nd:]), list(g[0].shape[-nd:])
    Lout = [a + b - 1 for a, b in zip(Lf, Lg)]
    name = {1: "config1_1d_c128_64x40", 2: "config2_1d_c128_batch4096_8192x3000",
            3: "config3_2d_c128_4096sq_x_255sq_gauss", 4: "config4_3d_c64_512cube_x_129cube",
            5: "config5_2d_c128_multiconv6_2048sq_x_1024x1536"}[cfg]
    return d, f, g, Lf, Lg, Lout, name


def alg_bytes(ndim, N, Lf, Lg, Lout, eb, batch=1):
    """Algorithmic bytes per pass at minimal padding: each pass reads
    its inputs once and writes its outputs once; intermediates sized by L_out."""
    P = {}
    if ndim == 1:
        P["conv1d"] = batch * eb * N * (Lf[0] + Lg[0]) + batch * eb * Lout[0]
    elif ndim == 2:
        Xf = N * Lf[0] * Lout[1]
        Xg = N * Lg[0] * Lout[1]
        P["fwd_x_f"] = eb * (N * Lf[0] * Lf[1] + Xf)
        P["fwd_x_g"] = eb * (N * Lg[0] * Lg[1] + Xg)
        # (one launch "fwd_x" carries both families when the library merges them;
        # its bytes are fwd_x_f + fwd_x_g -- not a separate entry in the step total)
        P["conv_y"] = eb * (Xf + Xg + Lout[0] * Lout[1])
        P["inv_x"] = eb * 2 * Lout[0] * Lout[1]
    else:
        X1f = N * Lf[0] * Lf[1] * Lout[2]
        X1g = N * Lg[0] * Lg[1] * Lout[2]
        XYf = N * Lf[0] * Lout[1] * Lout[2]
        XYg = N * Lg[0] * Lout[1] * Lout[2]
        O3 = Lout[0] * Lout[1] * Lout[2]
        P["fwd_x_f"] = eb * (N * np.prod(Lf) + X1f)
        P["fwd_x_g"] = eb * (N * np.prod(Lg) + X1g)
        P["fwd_y_f"] = eb * (X1f + XYf)
        P["fwd_y_g"] = eb * (X1g + XYg)
        P["conv_z"] = eb * (XYf + XYg + O3)
        P["inv_y"] = eb * 2 * O3
        P["inv_x"] = eb * 2 * O3
    return {k: int(v) for k, v in P.items()}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak():
    """FP64 FMA throughput measured on this GPU model by tools/micro/fp64_peak.cu
    (profiles/fp64_peak.json, committed); the derived 64 lanes/clk/SM figure only
    if that file is missing (and then labelled as such)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            d = json.load(fh)
        return float(d["fp64_fma_tflops"]), "measured (profiles/fp64_peak.json: tools/micro/fp64_peak.cu DFMA chains)"
    except Exception:
        return 2 * 64 * 148 * 1.965e9 / 1e12, "derived: 64 FP64 FMA lanes/clk/SM x 2 x 148 SMs x 1.965 GHz"


def conv_flops(ndim, N, Lf, Lg, Lout, batch=1):
    """Plan-independent algorithmic flops of the convolution pass (SURVEY.md 8(d),
    VERDICT r01 item 2): per line of the convolution axis (axis 0) at minimal
    padding M = L_out, (2N + 1) transforms of nominal 5 M log2 M flops (N forward f,
    N forward g, one inverse) plus the N-pair product 6 M N; the lines are the
    L_out extents of the other axes (minimal padding there too).  A worse plan
    (more padding, naive folds) cannot raise it."""
    M = Lout[0]
    per_line = (2 * N + 1) * 5 * M * np.log2(M) + 6 * M * N
    lines = batch
    for i in range(1, ndim):
        lines *= Lout[i]
    return float(per_line * lines)


def ncu_traffic(kernel_name):
    """dram read+write bytes per launch of the kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get("traffic_bytes_per_launch", {}).get(kernel_name)
    except Exception:
        return None


def ncu_pipe(kernel_name):
    """FP64 (c128) / FMA pipe utilisation of the kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get("fp_pipe_pct", {}).get(kernel_name)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms in the background."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self, which):
        if which == 0:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.tmp.flush()
        self.tmp.seek(0)
        rows = [r.strip().split(", ") for r in self.tmp.read().splitlines() if r.strip()]
        os.unlink(self.tmp.name)
        sm, mx, reasons = [], [], set()
        for r in rows:
            try:
                ts = time.mktime(time.strptime(r[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
            except Exception:
                ts = None
            if ts is not None and self.t0 is not None and not (self.t0 - 1.0 <= ts <= self.t1 + 1.0):
                continue
            try:
                sm.append(float(r[2]))
                mx.append(float(r[3]))
            except Exception:
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_oracle_rate(f, g, Lout, target_s=12.0, seed=4242):
    """Oracle (as it stands) on host cores: output samples/s on a bounded random
    sample of output indices of the same workload."""
    import oracle
    # calibration: large enough that thread start-up does not dominate (a 256-sample
    # probe underestimated the rate 3x and the measured sample ran 4 s, not target_s)
    n = 8192
    idx = synth.sample_indices(Lout, n_random=n, seed=seed, edge=0)
    t = time.perf_counter()
    oracle.multiconv_sampled(f, g, idx)
    dt = time.perf_counter() - t
    n2 = int(min(8_000_000, max(n, len(idx) * target_s / max(dt, 1e-6))))
    idx = synth.sample_indices(Lout, n_random=n2, seed=seed + 1, edge=0)
    t = time.perf_counter()
    oracle.multiconv_sampled(f, g, idx)
    dt = time.perf_counter() - t
    return len(idx) / dt, len(idx), dt, oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    d, f, g, Lf, Lg, Lout, name = workload(args.config)
    if d["batch"] > 1:  # independent pairs: time the oracle on pair 0 (same per-sample cost)
        f, g = [f[0][0]], [g[0][0]]
    import oracle
    per_step = []
    nsamp = None
    # size each step to ~1/steps of a bounded budget
    budget = max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    rate0, n0, _, cores = cpu_oracle_rate(f, g, Lout, target_s=budget)
    nsamp = n0
    for s in range(args.warmup + args.steps):
        idx = synth.sample_indices(Lout, n_random=nsamp, seed=9000 + s, edge=0)
        t = time.perf_counter()
        oracle.multiconv_sampled(f, g, idx)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            per_step.append((len(idx), dt))
    tot_n = sum(n for n, _ in per_step)
    tot_t = sum(t for _, t in per_step)
    value = tot_n / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / len(per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": name, "sample": f"{nsamp} random output indices per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{nsamp} random output samples per step of the {name} "
                                   f"output (direct O(L_f L_g) sum per sample)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def pick_mode(world, ndim, npairs, batch):
    """--mode auto: one GPU -> the single-GPU pipeline ("independent"); N > 1 -> one
    problem over all ranks: 2-D / 3-D single pairs by slabs, 1-D batches by pairs
    (strong scaling); anything else -> every rank its own problem (weak)."""
    if world <= 1:
        return "independent"
    if ndim >= 2 and npairs == 1 and batch == 1:
        return "slab"
    if ndim == 1 and npairs == 1 and batch > 1:
        return "batch"
    return "independent"


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2306_10016_b200 import hdconv as H

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    d, f, g, Lf, Lg, Lout, name = workload(args.config)
    ndim = d["ndim"]
    N = len(f)
    npdt = f[0].dtype
    eb = 16 if npdt == np.complex128 else 8
    dtc = H.HD_C128 if eb == 16 else H.HD_C64
    batch = d["batch"] if ndim == 1 else 1
    ctx = H.Context(local_rank)
    fh = [torch.from_numpy(a).pin_memory() for a in f]
    gh = [torch.from_numpy(a).pin_memory() for a in g]
    fd = [t.to(dev) for t in fh]
    gd = [t.to(dev) for t in gh]
    out_shape = ([batch] if (ndim == 1 and batch > 1) else []) + Lout
    hd_ = torch.empty(out_shape, dtype=fd[0].dtype, device=dev)
    stream = torch.cuda.current_stream(dev)

    tune_s = 0.0
    plan = None
    if d.get("plan"):
        plan = H.Plan.make(ndim, [d["plan"]])
    elif not args.no_tune:
        t = time.perf_counter()
        plan = ctx.tune(dtc, Lf, Lg, N=N, batch=batch, reps=3)
        tune_s = time.perf_counter() - t
    if plan is None:
        plan = ctx.default_plan(dtc, Lf, Lg, npairs=N)
    plan = H.hd_plan_complete(dtc, Lf, Lg, plan, npairs=N)
    if dist:  # one plan for every rank (the slab exchange layouts depend on it): rank 0's
        obj = [bytes(plan)]
        dist.broadcast_object_list(obj, src=0)
        plan = H.Plan.from_buffer_copy(obj[0])

    slab = None
    shard = None  # 1-D batch sharding: (lo, hi) pairs of this rank
    mode = args.mode if args.mode != "auto" else pick_mode(world, ndim, N, batch)
    if mode == "slab":
        if ndim < 2 or N != 1 or batch != 1:
            raise SystemExit("--mode slab: 2D/3D single-pair configs only")
        # one problem over all ranks (strong scaling): libhdconv's NCCL slab path
        # (hd_conv2d_dist / hd_conv3d_dist); Python only broadcasts the NCCL id
        ctx.dist_init()
        slab = ctx.slab(dtc, Lf, Lg, 0, plan)
        f_local = fd[0][slab.in_lo:slab.in_hi].contiguous()
        h_local = torch.empty([slab.out_hi - slab.out_lo] + Lout[1:], dtype=fd[0].dtype, device=dev)
    elif mode == "batch":
        if ndim != 1 or N != 1 or batch < 2:
            raise SystemExit("--mode batch: 1-D batched single-pair configs only")
        # one batch over all ranks (strong scaling): hd_conv1d_dist with HD_SHARD_BATCH,
        # B / N pairs per rank, no data-path collective (the pairs are independent)
        ctx.dist_init()
        shard = H.dist_partition(batch, world, rank)
        f_local = fd[0][shard[0]:shard[1]].contiguous()
        g_local = gd[0][shard[0]:shard[1]].contiguous()
        h_local = torch.empty([shard[1] - shard[0], Lout[0]], dtype=fd[0].dtype, device=dev)

    def step():
        if shard is not None:
            ctx.conv1d_dist(f_local, g_local, batch, shard=H.HD_SHARD_BATCH, plan=plan, h=h_local)
        elif slab is not None:
            if ndim == 2:
                ctx.conv2d_dist(f_local, gd[0], Lf, plan=plan, h=h_local)
            else:
                ctx.conv3d_dist(f_local, gd[0], Lf, plan=plan, h=h_local)
        elif N > 1:
            ctx.multiconv(fd, gd, plan=plan, h=hd_)
        else:
            ctx.conv(fd[0], gd[0], plan=plan, h=hd_, batch=(ndim == 1 and batch > 1))

    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(args.warmup):
        step()
    # keep the clock sampler fed: >= 1 s of untimed load before timing
    torch.cuda.synchronize()
    t_end = time.time() + 1.0
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.mark(0)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(1)
    launches = ctx.launch_count() - l0
    ms = e0.elapsed_time(e1)
    # per-pass device times for the roofline: the same K steps again with CUDA events
    # around every launch on the launch stream (hd_profile_*).  The events cost ~20 us
    # per step, so they stay out of the headline timing above.
    ctx.profile_reset()
    ctx.profile_enable(True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    prof = ctx.profile_read()
    ms_profiled = e0.elapsed_time(e1)
    if dist:
        dist.barrier()
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    clk = clocks.stop()
    samples_per_step = batch * int(np.prod(Lout))
    # weak: every rank convolves its own problem; strong (slab): one problem over all ranks
    strong = slab is not None or shard is not None
    value = (1 if strong else world) * samples_per_step * args.steps / (ms * 1e-3)

    # N > 1 in slab mode: also the weak-scaling figure (every rank its own whole problem
    # on the single-GPU pipeline, no collective), max over ranks
    weak = None
    if strong and world > 1:
        def step_weak():
            ctx.conv(fd[0], gd[0], plan=plan, h=hd_, batch=(ndim == 1 and batch > 1))
        for _ in range(args.warmup):
            step_weak()
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step_weak()
        e1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wms = float(tt.item())
        weak = {"value": world * samples_per_step * args.steps / (wms * 1e-3), "unit": UNIT,
                "ms_per_step": wms / args.steps, "scaling": "weak",
                "what": "every rank convolves its own whole problem (single-GPU pipeline), no collective"}

    # roofline of the dominant kernel (largest share of the step)
    peak, peak_src = peaks()
    ab = alg_bytes(ndim, N, Lf, Lg, Lout, eb, batch)
    if slab is not None:
        # slab mode: each rank's one "pass_conv" launch convolves 1/world of the
        # spectral lines of the pipeline's convolution pass
        ab = dict(ab, pass_conv=ab["conv_y" if ndim == 2 else "conv_z"] // world)
    if shard is not None:  # batch mode: this rank's launch convolves its pairs only
        ab = {k: v * (shard[1] - shard[0]) // batch for k, v in ab.items()}
    dom = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
    roof = None
    if dom:
        dms, dl = prof[dom]
        avg = dms / dl
        ab_dom = ab.get(dom, ab.get(dom + "_f", 0) + ab.get(dom + "_g", 0))
        achieved = ab_dom / (avg * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom), "peak_source": peak_src,
                "alg_bytes_per_launch": ab_dom, "avg_launch_ms": avg,
                "share_of_step": dms / sum(v[0] for v in prof.values())}
        fl = None
        if dom.startswith("conv") or dom == "pass_conv":
            fl = conv_flops(ndim, N, Lf, Lg, Lout, batch) / (world if dom == "pass_conv" else 1)
            if shard is not None:
                fl = fl * (shard[1] - shard[0]) / batch
        if fl:
            # the convolution pass's arithmetic beside its HBM roofline: plan-independent
            # flops against the measured FP64 (FP32 for c64: nominal 2x FP64 is NOT
            # assumed -- the FP32 peak is the microbenchmark's FFMA figure) FMA peak
            fpk, fsrc = fp64_peak()
            if eb == 8:
                try:
                    with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fp:
                        fpk, fsrc = float(json.load(fp)["fp32_fma_tflops"]), "measured FFMA (profiles/fp64_peak.json)"
                except Exception:
                    fpk, fsrc = 2 * 128 * 148 * 1.965e9 / 1e12, "derived: 128 FP32 lanes/clk/SM x 2 x 148 x 1.965 GHz"
            ach = fl / (avg * 1e-3) / 1e12
            roof["alu"] = {"achieved": ach, "peak": fpk, "unit": "TFLOP/s", "frac": ach / fpk,
                           "peak_source": fsrc, "alg_flops_per_launch": fl,
                           "pipe_util_ncu": ncu_pipe(dom),
                           "flops": "(2N+1) x 5 M log2 M + 6 M N per line, M = L_out of the conv axis, "
                                    "lines = L_out of the other axes (plan-independent)"}
    total_ab = sum(v for k, v in ab.items() if k != "pass_conv")
    # compulsory bytes (stricter): the inputs read once, the output written once
    nb_local = (shard[1] - shard[0]) if shard is not None else batch
    comp = eb * nb_local * (N * (int(np.prod(Lf)) + int(np.prod(Lg))) + int(np.prod(Lout)))
    step_s = ms * 1e-3 / args.steps
    whole = {"alg_bytes_per_step": total_ab,
             "compulsory_bytes_per_step": comp,
             "compulsory_frac_of_hbm": comp / step_s / 1e9 / peak,
             "achieved_gbs": total_ab / (ms * 1e-3 / args.steps) / 1e9,
             "frac_of_hbm": total_ab / (ms * 1e-3 / args.steps) / 1e9 / peak,
             "per_kernel_ms": {k: v[0] / v[1] for k, v in prof.items()},
             "profiled_ms_per_step": ms_profiled / args.steps}

    # end to end through the host-buffer C-ABI entry point (copies inside)
    e2e = None
    if not args.no_e2e and slab is not None:
        # end to end at N ranks: this rank's f slab and g from pinned host memory, the
        # distributed call, its h slab back to pinned host memory, every step
        fh_l = fh[0][slab.in_lo:slab.in_hi].contiguous().pin_memory()
        hh_l = torch.empty(list(h_local.shape), dtype=h_local.dtype).pin_memory()
        k2 = max(4, min(args.steps, 20))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(k2):
            f_local.copy_(fh_l, non_blocking=True)
            gd[0].copy_(gh[0], non_blocking=True)
            step()
            hh_l.copy_(h_local, non_blocking=True)
        torch.cuda.synchronize()
        te = time.perf_counter() - t
        if dist:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": samples_per_step * k2 / te, "unit": UNIT,
               "h2d_bytes_per_step": int(fh_l.numel() * eb + sum(a.nbytes for a in g)),
               "d2h_bytes_per_step": int(hh_l.numel() * eb), "steps": k2, "per": "rank (max over ranks)"}
    if not args.no_e2e and shard is not None:
        # end to end at N ranks: this rank's pairs from pinned host memory, the sharded
        # call, its rows back to pinned host memory, every step
        fh_l = fh[0][shard[0]:shard[1]].contiguous().pin_memory()
        gh_l = gh[0][shard[0]:shard[1]].contiguous().pin_memory()
        hh_l = torch.empty(list(h_local.shape), dtype=h_local.dtype).pin_memory()
        k2 = max(4, min(args.steps, 20))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(k2):
            f_local.copy_(fh_l, non_blocking=True)
            g_local.copy_(gh_l, non_blocking=True)
            step()
            hh_l.copy_(h_local, non_blocking=True)
        torch.cuda.synchronize()
        te = time.perf_counter() - t
        if dist:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": samples_per_step * k2 / te, "unit": UNIT,
               "h2d_bytes_per_step": int((fh_l.numel() + gh_l.numel()) * eb),
               "d2h_bytes_per_step": int(hh_l.numel() * eb), "steps": k2, "per": "rank (max over ranks)"}
    if not args.no_e2e and slab is None and shard is None:
        # three result buffers: step k writes hh[k % 3] (asynchronous, triple-buffered
        # entry point: copy-in k+2 | convolution k+1 | copy-out k)
        hh = [torch.empty(out_shape, dtype=fd[0].dtype).pin_memory() for _ in range(3)]
        k2 = max(4, min(args.steps, 20))
        ctx.hd_conv_host(fh, gh, hh[0], ndim=ndim, batch=batch, plan=plan)
        if dist:
            dist.barrier()
        t = time.perf_counter()
        for k in range(k2):
            ctx.hd_conv_host_async(fh, gh, hh[k % 3], ndim=ndim, batch=batch, plan=plan)
        ctx.host_sync()
        te = time.perf_counter() - t
        if dist:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": world * samples_per_step * k2 / te, "unit": UNIT,
               "h2d_bytes_per_step": int(sum(a.nbytes for a in f) + sum(a.nbytes for a in g)),
               "d2h_bytes_per_step": int(samples_per_step * eb), "steps": k2}

    # explicit-padding GPU variant from the same kernels (context)
    explicit = None
    if not args.no_explicit and ndim >= 2 and slab is None:
        try:
            # the explicit variant with ITS OWN tuned plan (hd_tune_explicit; untimed), so the
            # comparison is hybrid vs explicit padding on equal terms
            t = time.perf_counter()
            xplan = ctx.tune_explicit(dtc, Lf, Lg, N=N, reps=3)
            xtune_s = time.perf_counter() - t
            ctx.hd_conv_explicit(fd, gd, h=hd_)
            torch.cuda.synchronize()
            k3 = max(2, min(args.steps, 20))
            e0.record(stream)
            for _ in range(k3):
                ctx.hd_conv_explicit(fd, gd, h=hd_)
            e1.record(stream)
            torch.cuda.synchronize()
            xms = e0.elapsed_time(e1) / k3
            m_exp = [1 << int(np.ceil(np.log2(o))) for o in Lout]
            predicted = float(np.prod(m_exp) / np.prod([a["M1"] for a in plan.as_dict()["axis"]]))
            explicit = {"value": samples_per_step / (xms * 1e-3), "ms_per_step": xms,
                        "hybrid_speedup": xms / (ms / args.steps),
                        "predicted_work_ratio": predicted,
                        "padded_extents": m_exp, "tune_seconds": xtune_s,
                        "plan": [{k: a[k] for k in ("m", "C", "S", "D", "q")} for a in xplan.as_dict()["axis"]]}
        except Exception as ex:  # report, never hide
            explicit = {"error": str(ex)}

    # real-input path on the same data when it is real-valued (config 3:
    # image and kernel have zero imaginary parts): context, not the metric
    real = None
    if not args.no_explicit and slab is None and N == 1 and batch == 1 and eb == 16 and \
            all(not np.any(np.imag(x)) for x in list(f) + list(g)):
        try:
            fr = torch.from_numpy(np.ascontiguousarray(np.real(f[0]))).to(dev)
            gr = torch.from_numpy(np.ascontiguousarray(np.real(g[0]))).to(dev)
            Lz = [(Lf[0] + 1) // 2] + list(Lf[1:])
            rplan = ctx.tune(dtc, Lz, Lg, reps=3) if not args.no_tune else None
            hr = ctx.conv_real(fr, gr, plan=rplan)
            torch.cuda.synchronize()
            k4 = max(2, min(args.steps, 50))
            e0.record(stream)
            for _ in range(k4):
                ctx.conv_real(fr, gr, plan=rplan, h=hr)
            e1.record(stream)
            torch.cuda.synchronize()
            rms = e0.elapsed_time(e1) / k4
            real = {"value": samples_per_step / (rms * 1e-3), "unit": UNIT, "ms_per_step": rms,
                    "speedup_vs_complex": (ms / args.steps) / rms,
                    "method": "halves of f along axis 0 packed as re/im of one complex problem (hd_conv_real)"}
            if not args.no_e2e:
                # end to end: real f and g from pinned host memory, real h back, every
                # step; two streams so the copy-in of step k+1 overlaps the copy-out of
                # step k (the calls themselves are ordered on the context scratch)
                fh_r = torch.from_numpy(np.ascontiguousarray(np.real(f[0]))).pin_memory()
                gh_r = torch.from_numpy(np.ascontiguousarray(np.real(g[0]))).pin_memory()
                sts = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
                fr2 = [torch.empty_like(fr), torch.empty_like(fr)]
                gr2 = [torch.empty_like(gr), torch.empty_like(gr)]
                hr2 = [torch.empty_like(hr), torch.empty_like(hr)]
                hh_r = [torch.empty(list(hr.shape), dtype=hr.dtype).pin_memory() for _ in range(2)]
                k5 = max(4, min(args.steps, 20))
                torch.cuda.synchronize()
                t = time.perf_counter()
                for k in range(k5):
                    i = k % 2
                    with torch.cuda.stream(sts[i]):
                        fr2[i].copy_(fh_r, non_blocking=True)
                        gr2[i].copy_(gh_r, non_blocking=True)
                        ctx.conv_real(fr2[i], gr2[i], plan=rplan, h=hr2[i], stream=sts[i])
                        hh_r[i].copy_(hr2[i], non_blocking=True)
                torch.cuda.synchronize()
                te = time.perf_counter() - t
                real["e2e"] = {"value": samples_per_step * k5 / te, "unit": UNIT,
                               "h2d_bytes_per_step": int(fh_r.numel() * 8 + gh_r.numel() * 8),
                               "d2h_bytes_per_step": int(hh_r[0].numel() * 8), "steps": k5}
        except Exception as ex:  # report, never hide
            real = {"error": str(ex)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        fo, go = (f, g) if batch == 1 else ([f[0][0]], [g[0][0]])
        rate, n, dt, cores = cpu_oracle_rate(fo, go, Lout, target_s=args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{n} random output samples of {name} (direct sum per sample), {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f64" if eb == 16 else "f32",
            "data": "synthetic",
            "config": {"workload": name, "Lf": Lf, "Lg": Lg, "Lout": Lout, "pairs": N, "batch": batch,
                       "plan": [{k: v for k, v in a.items()} for a in plan.as_dict()["axis"]],
                       "tune_seconds": tune_s,
                       "parallelism": (f"slab x{world} ({'rows' if ndim == 2 else 'z-planes'}; NCCL all-to-all "
                                       "transposes)" if slab is not None
                                       else f"batch x{world} (B/N pairs per rank, no collective)"
                                       if shard is not None
                                       else f"weak x{world} (independent problems)"),
                       "l2": "inputs larger than L2 (image 268 MB > 126 MB L2); no flush needed"},
            "roofline": roof, "whole_step": whole, "cpu_baseline": cpu, "e2e": e2e,
            "explicit_variant": explicit, "real_input_variant": real, "gpu_launches": int(launches), "clocks": clk,
        }
        if slab is not None:
            line["slab"] = {k: getattr(slab, k) for k in ("nchunks", "R", "Ro", "Ks", "block1", "block2",
                                                          "bytes_sent")}
        if strong:
            line["weak_scaling"] = weak
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


def spawn(args):
    """--gpus N > 1 without a torchrun environment: launch N ranks of this script with
    torch.distributed.run on this node (127.0.0.1) and pass its exit code through
    (rank 0 prints the JSON line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")   # communicator lines on stderr (NVLS / rings)
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """--dry-run: the multi-rank launch plumbing without a GPU (gloo, one all_reduce)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        n = int(t.item())
        dist.destroy_process_group()
    else:
        n = 1
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": n, "gpus_flag": args.gpus}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-explicit", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--mode", default="auto", choices=["auto", "independent", "slab", "batch"],
                    help="auto: N = 1 single-GPU pipeline; N > 1 one problem over the ranks (strong "
                         "scaling: 2-D/3-D slabs with NCCL exchanges in libhdconv, 1-D batches by "
                         "pairs) with weak scaling as an extra key; independent: each rank its own "
                         "problem (weak); slab / batch: those paths at any N")
    ap.add_argument("--dry-run", action="store_true", help="launch plumbing only (gloo, no GPU work)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.dry_run:
        return run_dry(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
