#!/usr/bin/env python
"""Benchmark of the DiffServe hot path on B200 (BASELINE.json metric:
"images scored+routed/sec and planner candidates/sec at 1/2/4/8 B200 vs CPU").

One STEP (the headline `value`, SURVEY.md 8(d) config 2 "Cascade 2"):
  5,000 synthetic 512x512x3 u8 images resident in HBM per GPU
  -> fused tcgen05 discriminator (K5-K7) -> confidences
  -> route at the 101 grid thresholds k/100 (K2: ordered heavy-queue ids)
  -> deferral-curve replay of the 5,000 confidences in id order (K3, decay 0.999)
  -> (N > 1) NCCL all-gather of the per-GPU routed counts + exclusive scan
     (global heavy-queue offsets; SURVEY 8(e), config 5 scale-out).
Per-GPU work is fixed (weak scaling). Inputs (3.9 GB) exceed L2 (126 MB), so
no flush is needed between steps.

Secondary legs in the same JSON line:
  planner : K1 over 4,096 config-4 problems (fitted 32x32 tables, 101 thresholds,
            S in {16,32,64,128}); unit = one (problem, t, b1, b2) candidate.
  latent  : the reference's own scorer (sample_query, bit-parity mode, K4) +
            route at t = 0.5 + curve replay over 1M queries per GPU (config 5).
  workload: generate_arrivals over a 1M-arrival Poisson trace (K8, bit-exact)
            + the Query records at those arrivals (K4 records); replicas per GPU.
  csv     : queries.csv bytes of 1M QueryRecords (K9, byte-identical to write_csv).
CPU baselines run on this box's host cores on bounded samples (rank 0, N=1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images scored+routed/sec and planner candidates/sec at 1/2/4/8 B200 vs CPU"
N_IMG = 5000
H = W = 512
IMG_SEED = 1
WEIGHT_SEED = 2024
DISC_FLOP_PER_IMG = 2 * (768 * 256 + 256 * 1024 + 1024 * 256) * ((H // 16) * (W // 16))
# Layer 1 runs on the int8 tensor path (u8 x s8 -> s32), whose rate is twice the
# bf16 rate per FLOP (an M128 N256 K32 kind::i8 MMA takes the same 128 cycles
# as an M128 N256 K16 kind::f16 one: tools/i8_rate_probe.cu). The roofline
# therefore counts layer-1 FLOPs at half weight: bf16-equivalent FLOP/image.
DISC_FLOP_L1 = 2 * 768 * 256 * ((H // 16) * (W // 16))
DISC_FLOP_BF16_EQ = DISC_FLOP_PER_IMG - DISC_FLOP_L1 // 2
N_PLAN = 4096
CANDS_PER_PROBLEM = 101 * 32 * 32
N_LATENT = 1_000_000
DECAY = 0.999
CPU_DISC_SAMPLE = 256         # images for the CPU port of the discriminator
CPU_PLAN_SAMPLE = 256         # problems for the CPU reference planner
CPU_LATENT_SAMPLE = 200_000   # queries for the CPU reference scorer
WL_RATES = [2500.0] * 400     # 400 s at 2,500 qps: 1,000,811 arrivals at seed 3
WL_SEED = 3
N_CSV = 1_000_000
N_SCALE = 1_000_000           # config 5: queries over the whole world
WORKLOAD = ("cascade2: 5K synthetic 512x512 images/GPU, discriminator score + route at 101 "
            "thresholds + curve replay")
CPU_CSV_SAMPLE = 200_000      # records through the reference's write_csv


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class ClockSampler:
    """SM clock, power and throttle reasons sampled DURING the timed region:
    NVML polled every 2 ms from a thread (nvidia-smi's 100 ms cadence misses
    most of a ~0.1 s timed region); nvidia-smi as the fallback."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []     # (sm_mhz, max_mhz, power_w, set of reason names)
        self.stop_flag = False
        self.thread = None
        self.err = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def run():
                while not self.stop_flag:
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), pw,
                                          {k for k, b in bits.items() if rs & b}))
                    except Exception as e:   # keep sampling
                        self.err = str(e)
                    time.sleep(0.002)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception as e:
            self.err = str(e)
            self.thread = None

    def stop(self):
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": [f"no clock samples ({self.err})"]}
        try:   # raw samples for inspection (not part of the JSON line)
            with open(os.path.join(ROOT, "gpurun_out", "clocks_raw.csv"), "w") as f:
                for r in self.rows:
                    f.write(f"{r[0]},{r[1]},{r[2]},{'|'.join(sorted(r[3]))}\n")
        except Exception:
            pass
        pmax = max(r[2] for r in self.rows)
        # samples taken while the GPU was busy (power >= half the peak seen)
        busy = [r for r in self.rows if r[2] >= 0.5 * pmax] or self.rows
        reasons = set()
        for r in busy:
            reasons |= r[3]
        return {"sm_mhz": statistics.median(r[0] for r in busy),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": sorted(reasons),
                "power_w_max": pmax, "samples_under_load": len(busy),
                "samples": len(self.rows), "source": "nvml, 2 ms"}


def in_kernel_clock(L, disc, images, conf, ctx):
    """The SM clock the discriminator actually ran at: one traced launch of the
    step's disc_kernel right after the timed region (GPU still at its load
    state), every CTA stamping clock64 and globaltimer at its start and end.
    NVML's clock/power readings are averaged over a longer window than a
    4.7 ms launch, so they can read max clock while the kernel is power-capped;
    this is the direct measurement (and a clock-independent cycles per pair
    tile over the whole launch)."""
    import ctypes

    import torch

    from paper_2411_15381_b200 import native
    L.ds_disc_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                                                ctypes.c_int32] + [ctypes.c_void_p] * 3
    nt = 8 * 8 * 16
    tr = torch.zeros(nt + 5 * 160, dtype=torch.int64, device=images.device)
    native.check(L.ds_disc_trace_device(disc.handle, native.c_p(images.data_ptr()), N_IMG, H, W,
                                        native.c_p(conf.data_ptr()), native.c_p(tr.data_ptr()),
                                        native.c_p(ctx.stream)))
    ctx.synchronize()
    t = tr.cpu().numpy()
    ns = t[nt:nt + 480].reshape(160, 3)
    cyc = t[nt + 480:nt + 800].reshape(160, 2)
    used = (ns[:, 0] > 0) & (ns[:, 1] > ns[:, 0]) & (cyc[:, 1] > cyc[:, 0])
    if not used.any():
        return None
    mhz = (cyc[used, 1] - cyc[used, 0]) / ((ns[used, 1] - ns[used, 0]) / 1e3)
    pair_tiles = (N_IMG * (H // 16) * (W // 16) // 128 + 1) // 2
    per_sm_tiles = pair_tiles / (int(used.sum()) // 2)
    return {"sm_mhz_median": float(np.median(mhz)), "sm_mhz_min": float(mhz.min()),
            "sm_mhz_max": float(mhz.max()), "ctas": int(used.sum()),
            "launch_us": float((ns[used, 1].max() - ns[used, 0].min()) / 1e3),
            "cycles_per_pair_tile": float(np.median(cyc[used, 1] - cyc[used, 0]) / per_sm_tiles),
            "how": "clock64 / globaltimer at every CTA's start and end, one traced disc_kernel "
                   "launch of the step's images right after the timed region"}


def tensor_pipe_frac(ik):
    """Clock-independent view of the discriminator: the MMA cycles a 256-token
    pair tile needs at the tensor pipe's rate (152 MMAs x 128 cycles: GEMM1 24
    i8 K=32, GEMM2 64 and GEMM3 64 bf16 K=16, each M=256 N=256 on an SM pair)
    over the cycles a pair tile took (in-kernel clock64, whole launch)."""
    if not ik or not ik.get("cycles_per_pair_tile"):
        return None
    mma = 152 * 128
    return {"mma_cycles_per_pair_tile": mma,
            "cycles_per_pair_tile": ik["cycles_per_pair_tile"],
            "frac": mma / ik["cycles_per_pair_tile"],
            "note": "tensor-pipe utilisation per cycle; TFLOP/s also depends on the SM clock "
                    "the 1 kW cap allows (see clocks.in_kernel)"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the same path on the host cores
# ---------------------------------------------------------------------------

def cpu_images_leg(n_img: int):
    """The CPU port of the discriminator (oracle/disc_oracle.disc_forward_fast:
    fp32 BLAS with the exact centred layer 1, one image per BLAS call, images
    spread over every host thread) + the reference's own route loop (oracle/_ref, cluster.cpp:290-306)
    at all 101 thresholds over the same confidences."""
    from oracle import disc_oracle, lib
    from paper_2411_15381_b200 import abi, workloads
    # weights: the same deterministic network as the GPU (export needs no GPU
    # compute beyond creation, so regenerate on the host from the seed)
    wts = host_weights()
    imgs = disc_oracle.synth_images(IMG_SEED, 0, n_img, H, W)
    grid = workloads.make_grid(0.01)
    prior = np.zeros((), abi.CURVE)
    s = np.asarray(workloads.SHIPPED_PRIOR_SAMPLES, np.float64)
    t0 = time.perf_counter()
    conf = disc_oracle.disc_forward_fast(imgs, wts).astype(np.float64)
    idx = np.zeros(n_img, np.int64)
    cnt = np.zeros(1, np.int64)
    if lib.ref_available():
        r = lib.ref()
        for k, t in enumerate(grid):
            curve = prior.copy()
            r.dsref_curve_from_samples(abi.ptr(s), len(s), abi.ptr(curve))
            r.dsref_route_loop(abi.ptr(conf), n_img, float(t), 1 if k == 0 else 0, DECAY,
                               abi.ptr(curve), abi.ptr(idx), abi.ptr(cnt))
        kind = "port"   # discriminator is this repo's port; route loop is the reference's
    else:
        p = lib.port()
        for k, t in enumerate(grid):
            curve = prior.copy()
            p.dso_route_loop(abi.ptr(conf), n_img, float(t), 1 if k == 0 else 0, DECAY,
                             abi.ptr(curve), abi.ptr(idx), abi.ptr(cnt))
        kind = "port"
    dt = time.perf_counter() - t0
    return n_img / dt, kind, conf


def cpu_planner_leg(problems, cascades, grid, offs, threads):
    from oracle import lib
    from paper_2411_15381_b200 import abi
    out = np.zeros(len(problems), abi.PLAN)
    t0 = time.perf_counter()
    if lib.ref_available():
        lib.ref().dsref_plan_batch(abi.ptr(problems), len(problems), abi.ptr(cascades),
                                   len(cascades), abi.ptr(grid), abi.ptr(offs), 1, abi.ptr(out),
                                   threads)
        kind = "reference"
    else:
        st = np.zeros(len(problems), np.int32)
        lib.port().dso_plan_batch(abi.ptr(problems), len(problems), abi.ptr(cascades),
                                  abi.ptr(grid), abi.ptr(offs), abi.ptr(out), abi.ptr(st),
                                  threads)
        kind = "port"
    dt = time.perf_counter() - t0
    return len(problems) * CANDS_PER_PROBLEM / dt, kind, out, dt


def cpu_latent_leg(n, threads):
    """sample_query over ids (all cores) then the sequential observe+defers loop."""
    from oracle import lib
    from paper_2411_15381_b200 import abi, workloads
    m = workloads.query_model()
    conf = np.zeros(n)
    idx = np.zeros(n, np.int64)
    cnt = np.zeros(1, np.int64)
    curve = workloads.uniform_prior()
    t0 = time.perf_counter()
    if lib.ref_available():
        lib.ref().dsref_sample_queries(abi.ptr(m), 0, n, 5.0, abi.ptr(conf), None, threads)
        lib.ref().dsref_route_loop(abi.ptr(conf), n, 0.5, 1, DECAY, abi.ptr(curve), abi.ptr(idx),
                                   abi.ptr(cnt))
        kind = "reference"
    else:
        lib.port().dso_sample_queries(abi.ptr(m), 0, n, abi.ptr(conf), None, threads)
        lib.port().dso_route_loop(abi.ptr(conf), n, 0.5, 1, DECAY, abi.ptr(curve), abi.ptr(idx),
                                  abi.ptr(cnt))
        kind = "port"
    return n / (time.perf_counter() - t0), kind, conf, idx[:int(cnt[0])]


def cpu_workload_leg(threads):
    """The reference's generate_arrivals (sequential by construction) + the
    run_experiment sample_query loop, here on all cores."""
    from oracle import lib
    from paper_2411_15381_b200 import abi, workloads
    rates = np.asarray(WL_RATES, np.float64)
    m = workloads.query_model()
    use_ref = lib.ref_available()
    gen = lib.ref().dsref_generate_arrivals if use_ref else lib.port().dso_generate_arrivals
    t0 = time.perf_counter()
    n = gen(abi.ptr(rates), len(rates), 1.0, WL_SEED, 0, None, 0)
    a = np.zeros(n)
    t0 = time.perf_counter()
    gen(abi.ptr(rates), len(rates), 1.0, WL_SEED, 0, abi.ptr(a), n)
    t_arr = time.perf_counter() - t0
    conf = np.zeros(n)
    t0 = time.perf_counter()
    if use_ref:
        lib.ref().dsref_sample_queries(abi.ptr(m), 0, n, 5.0, abi.ptr(conf), None, threads)
    else:
        lib.port().dso_sample_queries(abi.ptr(m), 0, n, abi.ptr(conf), None, threads)
    t_q = time.perf_counter() - t0
    return n / (t_arr + t_q), n / t_arr, ("reference" if use_ref else "port"), a


def csv_records(n, seed=12):
    from tests import helpers
    return helpers.random_query_records(np.random.default_rng(seed), n)


def cpu_csv_leg(records):
    """The reference's write_csv (metrics.cpp:91-127) on the records, into a
    temporary directory (the port's snprintf formatter where it is absent)."""
    import tempfile
    from oracle import lib
    from paper_2411_15381_b200 import abi
    iv = np.zeros(0, abi.INTERVAL_SNAPSHOT)
    pl = np.zeros(0, abi.PLAN_LOG_ENTRY)
    if lib.ref_available():
        with tempfile.TemporaryDirectory() as tmp:
            t0 = time.perf_counter()
            lib.ref().dsref_write_csv(tmp.encode(), abi.ptr(iv), 0, abi.ptr(records),
                                      len(records), abi.ptr(pl), 0)
            return len(records) / (time.perf_counter() - t0), "reference"
    n = lib.port().dso_format_queries_csv(abi.ptr(records), len(records), None, 0)
    out = np.zeros(n, np.uint8)
    t0 = time.perf_counter()
    lib.port().dso_format_queries_csv(abi.ptr(records), len(records), abi.ptr(out), n)
    return len(records) / (time.perf_counter() - t0), "port"


def host_weights():
    """The discriminator weights exactly as ds_disc_create makes them: the
    committed export (profiles/, bit-identical when present) else the host
    restatement oracle/disc_oracle.gen_weights (no GPU needed)."""
    from oracle import disc_oracle
    cache = os.path.join(ROOT, "profiles", f"disc_weights_seed{WEIGHT_SEED}.npz")
    if os.path.exists(cache):
        d = dict(np.load(cache))
        ref = disc_oracle.gen_weights(WEIGHT_SEED, calibrate=False)
        if all(k in d and np.array_equal(d[k], ref[k]) for k in ("q1", "w2", "w3")):
            d["head_b"] = float(d["head_b"])
            return d
    return disc_oracle.gen_weights(WEIGHT_SEED, calibrate=True)


def planner_inputs():
    """BASELINE.md's planner batch: 4,096 acceptance-C2-recipe problems
    (mt19937_64(7)) over the three fitted 32x32 cascades x S in {16..128},
    grid k/100 -- generated by the reference itself (oracle/make_golden.py
    gen_config4_bench) and committed as a fixture with the reference's plans;
    the CPU arm times diffserve::solve on exactly these problems."""
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "config4_bench.npz")))
    return (g["problems"], g["cascades"].copy(), g["grid_values"], g["grid_offsets"],
            g["want_solve"])


def product_curves(ctx, cas):
    """Each planner cascade's deferral curve = DeferralCurve::from_samples of
    the 5K sample_query confidences (cascade cfg, seed 1)
    built by the PRODUCT: K4 scores, K3 replays at decay 1 from the empty
    curve. Returns whether they equal the fixture's (reference-built) curves."""
    from paper_2411_15381_b200 import abi, workloads
    conf = ctx.score_latent(workloads.query_model(), 0, 5000)
    curve = ctx.curve_observe(np.zeros((), abi.CURVE), conf, 1.0)
    same = all(cas[i]["deferral"].tobytes() == curve.tobytes() for i in range(len(cas)))
    for i in range(len(cas)):
        cas[i]["deferral"] = curve
    return same


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    kind = None
    for i in range(args.warmup + args.steps):
        v, kind, _ = cpu_images_leg(max(4, CPU_DISC_SAMPLE // 4))
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * max(4, CPU_DISC_SAMPLE // 4) / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": WORKLOAD, "global_batch": N_IMG,
                                        "image_hw": [H, W], "thresholds": 101,
                                        "sample_images": max(4, CPU_DISC_SAMPLE // 4)},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": kind,
                         "sample": f"{max(4, CPU_DISC_SAMPLE // 4)} images 512x512 per step"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2411_15381_b200 import abi, native, workloads
    from paper_2411_15381_b200 import dist as ddist

    ws, rank, local = dist_env()
    # Test hooks for the multi-rank path on a 1-GPU box: BENCH_DIST_BACKEND=gloo
    # and BENCH_SHARE_DEVICE=1 run every rank on cuda:0 with the library's host
    # transport (NCCL refuses two ranks on one device). The driver uses NCCL,
    # one rank per GPU.
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if os.environ.get("BENCH_SHARE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def allmax(vals):
        """Max over ranks (the contract: timings are the max over ranks)."""
        t = torch.tensor(vals, dtype=torch.float64)
        if ws > 1:
            t = t if backend == "gloo" else t.to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]

    def barrier():
        if ws > 1:
            dist.barrier()

    ctx = native.Context(local)
    L = native.lib()
    stream = torch.cuda.ExternalStream(ctx.stream)
    sp = native.c_p(ctx.stream)
    disc = native.Discriminator(ctx, WEIGHT_SEED)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    # The sharded hot path's collectives (include/ds_gpu.h "multi-GPU"): NCCL
    # from the library itself, one communicator per rank
    comm = None
    if ws > 1:
        comm = (ddist.nccl_comm(ctx) if backend == "nccl"
                else native.Comm.host(ctx, ws, rank, ddist.TorchHostOps()))

    # ---- inputs resident in HBM ---------------------------------------------
    id0 = rank * N_IMG
    NTOT = ws * N_IMG
    images = torch.empty(N_IMG * H * W * 3, dtype=torch.uint8, device=dev)
    native.check(L.ds_synth_images_device(ctx.handle, IMG_SEED, id0, N_IMG, H, W,
                                          native.c_p(images.data_ptr()), sp))
    grid_np = workloads.make_grid(0.01)
    grid_t = torch.tensor(grid_np, dtype=torch.float64, device=dev)
    NT = grid_t.numel()
    conf = torch.empty(N_IMG, dtype=torch.float32, device=dev)
    heavy = torch.empty(NT * N_IMG, dtype=torch.int64, device=dev)
    counts = torch.empty(NT, dtype=torch.int64, device=dev)
    offs = torch.empty(NT, dtype=torch.int64, device=dev)
    totals = torch.empty(NT, dtype=torch.int64, device=dev)
    # global heavy queues (rank 0, the load balancer's side) at N > 1
    gq = torch.empty(NT * NTOT if (ws > 1 and rank == 0) else 1, dtype=torch.int64, device=dev)
    gc = torch.empty(NT, dtype=torch.int64, device=dev)
    # prior = DeferralCurve::from_samples(shipped samples) (cascades.profiles:20)
    # through the product's K3 (observe at decay 1 from the empty curve)
    prior = ctx.curve_observe(np.zeros((), abi.CURVE),
                              np.asarray(workloads.SHIPPED_PRIOR_SAMPLES, np.float64), 1.0)
    prior_t = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).to(dev)
    curve_t = torch.empty_like(prior_t)
    torch.cuda.synchronize()

    def step(ev=None):
        with torch.cuda.stream(stream):
            if ev is not None:
                ev[0].record(stream)
            native.check(L.ds_disc_score_device(disc.handle, native.c_p(images.data_ptr()),
                                                N_IMG, H, W, native.c_p(conf.data_ptr()), sp))
            if ev is not None:
                ev[1].record(stream)
            curve_t.copy_(prior_t)
            if comm is None:
                native.check(L.ds_route_device(ctx.handle, native.c_p(conf.data_ptr()),
                                               abi.CONF_F32, N_IMG, native.c_p(grid_t.data_ptr()),
                                               NT, id0, native.c_p(heavy.data_ptr()),
                                               native.c_p(counts.data_ptr()), sp))
                native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(curve_t.data_ptr()),
                                                       native.c_p(conf.data_ptr()), abi.CONF_F32,
                                                       N_IMG, DECAY, sp))
            else:
                # route this shard + routed-count all-gather (each rank's
                # offset in every global queue), the ordered ids of every rank
                # assembled into the 101 global heavy queues at rank 0, and the
                # curve replayed over the GLOBAL id-ordered sequence on every
                # rank (cluster.cpp:288-307 order)
                comm.route(conf.data_ptr(), abi.CONF_F32, N_IMG, grid_t.data_ptr(), NT, id0,
                           heavy.data_ptr(), counts.data_ptr(), offs.data_ptr(),
                           totals.data_ptr(), stream=ctx.stream)
                comm.gather_queues(0, heavy.data_ptr(), N_IMG, counts.data_ptr(), NT,
                                   gq.data_ptr() if rank == 0 else 0, NTOT,
                                   gc.data_ptr() if rank == 0 else 0, stream=ctx.stream)
                comm.curve_observe(curve_t.data_ptr(), conf.data_ptr(), abi.CONF_F32,
                                   [N_IMG] * ws, DECAY, stream=ctx.stream)

    # ---- warmup + timed region -------------------------------------------------
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    n0 = ctx.launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - n0
    barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    clocks["in_kernel"] = in_kernel_clock(L, disc, images, conf, ctx)
    total_ms = t_start.elapsed_time(t_end)
    disc_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    total_ms, disc_ms = allmax([total_ms, disc_ms])
    ms_per_step = total_ms / args.steps
    value = ws * N_IMG / (ms_per_step / 1000.0)

    # ---- parity inside the benchmark -------------------------------------------
    # (1) this rank's routing vs its confidences (numpy)
    c_host = conf.cpu().numpy().astype(np.float64)
    cnt_host = counts.cpu().numpy()
    want_cnt = np.array([(c_host < t).sum() for t in grid_np])
    parity_ok = bool(np.array_equal(cnt_host, want_cnt))
    heavy50 = heavy[50 * N_IMG: 50 * N_IMG + int(cnt_host[50])].cpu().numpy()
    lists_ok = bool(np.array_equal(heavy50, np.flatnonzero(c_host < 0.5) + id0))
    # (2) N ranks == 1 GPU: rank 0 redoes the whole world's work on one GPU
    # (every rank's images scored here, routed in one call, one curve replay)
    # and compares the global queues, counts and curve bits
    parity_n1 = {}
    conf_all = None
    if rank == 0:
        conf_all = torch.empty(NTOT, dtype=torch.float32, device=dev)
        scratch_imgs = images if ws == 1 else torch.empty_like(images)
        with torch.cuda.stream(stream):
            for q in range(ws):
                if ws > 1:
                    native.check(L.ds_synth_images_device(
                        ctx.handle, IMG_SEED, q * N_IMG, N_IMG, H, W,
                        native.c_p(scratch_imgs.data_ptr()), sp))
                native.check(L.ds_disc_score_device(
                    disc.handle, native.c_p(scratch_imgs.data_ptr()), N_IMG, H, W,
                    native.c_p(conf_all.data_ptr() + 4 * q * N_IMG), sp))
            h1 = torch.empty(NT * NTOT, dtype=torch.int64, device=dev)
            c1 = torch.empty(NT, dtype=torch.int64, device=dev)
            native.check(L.ds_route_device(ctx.handle, native.c_p(conf_all.data_ptr()),
                                           abi.CONF_F32, NTOT, native.c_p(grid_t.data_ptr()), NT,
                                           0, native.c_p(h1.data_ptr()), native.c_p(c1.data_ptr()),
                                           sp))
            cur1 = prior_t.clone()
            native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(cur1.data_ptr()),
                                                   native.c_p(conf_all.data_ptr()), abi.CONF_F32,
                                                   NTOT, DECAY, sp))
        torch.cuda.synchronize()
        del scratch_imgs
        g_cnt = (gc if ws > 1 else counts).cpu().numpy()
        g_q = (gq if ws > 1 else heavy).cpu().numpy().reshape(NT, NTOT)
        w_cnt = c1.cpu().numpy()
        w_q = h1.cpu().numpy().reshape(NT, NTOT)
        parity_n1 = {
            "global_counts_equal_n1": bool(np.array_equal(g_cnt, w_cnt)),
            "global_queues_equal_n1": bool(np.array_equal(g_cnt, w_cnt) and all(
                np.array_equal(g_q[k, :w_cnt[k]], w_q[k, :w_cnt[k]]) for k in range(NT))),
            "global_curve_bits_equal_n1": curve_t.cpu().numpy().tobytes() ==
            cur1.cpu().numpy().tobytes(),
            "confidences_equal_n1": bool(torch.equal(conf_all[:N_IMG], conf)),
        }
        del h1
    step_curve = curve_t.cpu().numpy().view(abi.CURVE)[0].copy()
    take_err = ctx.take_error()   # no invalid confidence met by any device call
    barrier()

    # ---- e2e: the C-ABI calls with HOST buffers, copies inside the timed region
    pinned = torch.empty(N_IMG * H * W * 3, dtype=torch.uint8, pin_memory=True)
    pinned.copy_(images)
    host_imgs = pinned.numpy().reshape(N_IMG, H, W, 3)
    e2e_steps = max(2, min(args.steps, 5))

    def e2e_step():
        c = disc.score(host_imgs)
        cnts, _ = ctx.route(c, grid_np, index_base=id0, with_lists=True)
        ctx.curve_observe(prior, c, DECAY)
        return c, cnts

    e2e_step()
    barrier()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(e2e_steps):
        c, cnts = e2e_step()
        d2h = c.nbytes + int(cnts.sum()) * 8 + cnts.nbytes + abi.CURVE.itemsize
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_value = ws * N_IMG / allmax([e2e_s])[0]
    h2d = N_IMG * H * W * 3 + grid_np.nbytes + 2 * abi.CURVE.itemsize
    # what bounds e2e: the same pinned image bytes copied host -> device alone
    # (one cudaMemcpyAsync per step, CUDA events), i.e. the PCIe roofline
    pin_ms = []
    for _ in range(3):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a_.record(stream)
            images.copy_(pinned)   # blocking: no host-allocator event outlives the context
            b_.record(stream)
        torch.cuda.synchronize()
        pin_ms.append(a_.elapsed_time(b_))
    h2d_gbs = pinned.numel() / (min(pin_ms) / 1000.0) / 1e9
    e2e_gbs = N_IMG * H * W * 3 * (e2e_value / ws) / N_IMG / 1e9
    del pinned, host_imgs

    # ---- image legs for the other configs ------------------------
    def timed(fn, reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    # config 5 (scale-out): 1M queries over the world, contiguous id shards
    # scored in 5K chunks from each rank's resident pool (query i of rank q
    # uses pool image (i - lo_q) mod 5K), routed at t = 0.5 with global ids;
    # at N > 1 the routed-count all-gather and the global queue at rank 0
    lo5, hi5 = ddist.shard_range(N_SCALE, ws, rank)
    n5 = hi5 - lo5
    conf5 = torch.empty(n5, dtype=torch.float32, device=dev)
    heavy5 = torch.empty(n5, dtype=torch.int64, device=dev)
    count5 = torch.empty(1, dtype=torch.int64, device=dev)
    thr5 = torch.tensor([0.5], dtype=torch.float64, device=dev)
    gq5 = torch.empty(N_SCALE if (ws > 1 and rank == 0) else 1, dtype=torch.int64, device=dev)
    gc5 = torch.empty(1, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    def scale_step():
        with torch.cuda.stream(stream):
            for off in range(0, n5, N_IMG):
                m = min(N_IMG, n5 - off)
                native.check(L.ds_disc_score_device(
                    disc.handle, native.c_p(images.data_ptr()), m, H, W,
                    native.c_p(conf5.data_ptr() + 4 * off), sp))
            if comm is None:
                native.check(L.ds_route_device(ctx.handle, native.c_p(conf5.data_ptr()),
                                               abi.CONF_F32, n5, native.c_p(thr5.data_ptr()), 1,
                                               lo5, native.c_p(heavy5.data_ptr()),
                                               native.c_p(count5.data_ptr()), sp))
            else:
                comm.route(conf5.data_ptr(), abi.CONF_F32, n5, thr5.data_ptr(), 1, lo5,
                           heavy5.data_ptr(), count5.data_ptr(), stream=ctx.stream)
                comm.gather_queues(0, heavy5.data_ptr(), n5, count5.data_ptr(), 1,
                                   gq5.data_ptr() if rank == 0 else 0, N_SCALE,
                                   gc5.data_ptr() if rank == 0 else 0, stream=ctx.stream)
    scale_step()
    torch.cuda.synchronize()
    barrier()
    scale_ms = allmax([timed(scale_step, 1)])[0]
    scale_value = N_SCALE / (scale_ms / 1000.0)
    if rank == 0:
        # the 1M-query global queue vs one GPU's: pool confidences of every
        # rank (conf_all above), expanded over each rank's id range
        ca = conf_all.cpu().numpy().astype(np.float64)
        want = []
        for q in range(ws):
            qlo, qhi = ddist.shard_range(N_SCALE, ws, q)
            i = np.arange(qlo, qhi, dtype=np.int64)
            want.append(i[ca[q * N_IMG + (i - qlo) % N_IMG] < 0.5])
        want = np.concatenate(want)
        got_n = int((gc5 if ws > 1 else count5).item())
        got = (gq5 if ws > 1 else heavy5)[:got_n].cpu().numpy()
        parity_n1["config5_global_queue_equal_n1"] = bool(
            got_n == len(want) and np.array_equal(got, want))
        scale_routed = got_n
        del conf_all
    del conf5, heavy5, gq5

    # config 1 (cascade 1): the same pool in light batches of 32 -- per batch:
    # score, observe the 32 confidences into the curve, route at the plan's
    # threshold (cluster.cpp:288-307 order); independent per rank (each rank
    # serves its own light batches)
    B1 = 32
    NB1 = (N_IMG + B1 - 1) // B1
    conf1 = torch.empty(N_IMG, dtype=torch.float32, device=dev)
    heavy1 = torch.empty(N_IMG, dtype=torch.int64, device=dev)    # batch b's ids at its offset
    count1 = torch.empty(NB1, dtype=torch.int64, device=dev)      # one count per batch
    curve1 = torch.empty_like(prior_t)
    thr1 = torch.full((NB1,), 0.5, dtype=torch.float64, device=dev)   # the plan's t per batch
    offs1 = torch.tensor([min(b * B1, N_IMG) for b in range(NB1 + 1)], dtype=torch.int64,
                         device=dev)
    torch.cuda.synchronize()

    def batch32_step(spp=None):
        spp = sp if spp is None else spp
        curve1.copy_(prior_t)
        for b, off in enumerate(range(0, N_IMG, B1)):
            m = min(B1, N_IMG - off)
            native.check(L.ds_disc_batch_complete_device(
                disc.handle, native.c_p(images.data_ptr() + off * H * W * 3), m, H, W,
                native.c_p(conf1.data_ptr() + 4 * off), native.c_p(curve1.data_ptr()), DECAY,
                native.c_p(thr1.data_ptr() + 8 * b), 1, id0 + off,
                native.c_p(heavy1.data_ptr() + 8 * off), native.c_p(count1.data_ptr() + 8 * b),
                spp))

    def batch32_eager():
        with torch.cuda.stream(stream):
            batch32_step()
    batch32_eager()
    torch.cuda.synchronize()
    b32_ms = allmax([timed(batch32_eager, 2)])[0]
    b32_value = ws * N_IMG / (b32_ms / 1000.0)
    b32_batch_us = b32_ms * 1000.0 / NB1
    b32_parity = bool(torch.equal(conf1, conf))
    # the same 157 batches captured once into a CUDA graph (launch overhead off
    # the per-batch path, as a streaming server would run a fixed batch plan)
    g_stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(g_stream):
        batch32_step(native.c_p(g_stream.cuda_stream))   # warm-up on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=g_stream):
        batch32_step(native.c_p(g_stream.cuda_stream))
    conf1.fill_(-1.0)           # the replay must recompute every confidence
    ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(g_stream):
        graph.replay()
        g_stream.synchronize()
        b32g_parity = bool(torch.equal(conf1, conf))
        ga.record(g_stream)
        for _ in range(2):
            graph.replay()
        gb.record(g_stream)
    torch.cuda.synchronize()
    b32g_ms = allmax([ga.elapsed_time(gb) / 2])[0]
    del graph
    # batch by batch results (the reference: handle_batch_complete per batch)
    per_batch = (conf1.clone(), curve1.clone(), heavy1.clone(), count1.clone())
    # a backlog of the same 157 light batches in ONE call
    # (ds_disc_batches_complete_device): one discriminator launch streams all
    # their tiles, one curve replay, one segmented route (thresholds per batch)

    def backlog_step():
        with torch.cuda.stream(stream):
            curve1.copy_(prior_t)
            native.check(L.ds_disc_batches_complete_device(
                disc.handle, native.c_p(images.data_ptr()), N_IMG, native.c_p(offs1.data_ptr()),
                NB1, H, W, native.c_p(conf1.data_ptr()), native.c_p(curve1.data_ptr()), DECAY,
                native.c_p(thr1.data_ptr()), id0, native.c_p(heavy1.data_ptr()),
                native.c_p(count1.data_ptr()), sp))
    conf1.fill_(-1.0)
    heavy1.fill_(-1)
    count1.fill_(-1)
    backlog_step()
    torch.cuda.synchronize()
    bl_ms = allmax([timed(backlog_step, 3)])[0]
    pc, pcur, ph, pcnt = per_batch
    cnt_np = pcnt.cpu().numpy()
    h_new, h_old = heavy1.cpu().numpy(), ph.cpu().numpy()
    offs_np = offs1.cpu().numpy()
    bl_parity = bool(torch.equal(conf1, pc) and torch.equal(curve1, pcur) and
                     torch.equal(count1, pcnt) and all(
                         np.array_equal(h_new[offs_np[b]:offs_np[b] + cnt_np[b]],
                                        h_old[offs_np[b]:offs_np[b] + cnt_np[b]])
                         for b in range(NB1)))
    del conf1, per_batch

    # config 3 (cascade 3): 5K synthetic 1024x1024 images (15.7 GB) per GPU,
    # score + route at the 101 thresholds + curve replay
    N3, H3 = N_IMG, 1024
    images3 = torch.empty(N3 * H3 * H3 * 3, dtype=torch.uint8, device=dev)
    native.check(L.ds_synth_images_device(ctx.handle, 3, id0, N3, H3, H3,
                                          native.c_p(images3.data_ptr()), sp))
    conf3 = torch.empty(N3, dtype=torch.float32, device=dev)

    def c3_step():
        with torch.cuda.stream(stream):
            native.check(L.ds_disc_score_device(disc.handle, native.c_p(images3.data_ptr()), N3,
                                                H3, H3, native.c_p(conf3.data_ptr()), sp))
            native.check(L.ds_route_device(ctx.handle, native.c_p(conf3.data_ptr()), abi.CONF_F32,
                                           N3, native.c_p(grid_t.data_ptr()), NT, id0,
                                           native.c_p(heavy.data_ptr()),
                                           native.c_p(counts.data_ptr()), sp))
            curve_t.copy_(prior_t)
            native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(curve_t.data_ptr()),
                                                   native.c_p(conf3.data_ptr()), abi.CONF_F32,
                                                   N3, DECAY, sp))
    c3_step()
    torch.cuda.synchronize()
    c3_ms = allmax([timed(c3_step, 3)])[0]
    c3_value = ws * N3 / (c3_ms / 1000.0)
    c3_tflops = N3 * DISC_FLOP_BF16_EQ * 4 / (c3_ms / 1000.0) / 1e12
    del images3

    # ---- planner leg (config 4): BASELINE.md's 4,096-problem batch -------------
    # problem-sharded over the ranks (contiguous index ranges), plans gathered
    # at rank 0 (the controller) at N > 1
    pro, cas, grid, goffs, want_plans = planner_inputs()
    curves_ok = product_curves(ctx, cas)
    P_ALL = len(pro)
    plo, phi = ddist.shard_range(P_ALL, ws, rank)
    d_pro = torch.from_numpy(pro.view(np.uint8).copy()).to(dev)
    d_cas = torch.from_numpy(cas.view(np.uint8).copy()).to(dev)
    d_grid = torch.from_numpy(grid.copy()).to(dev)
    d_offs = torch.from_numpy(goffs.copy()).to(dev)
    PB = abi.PLAN.itemsize
    d_out = torch.empty(max(phi - plo, 1) * PB, dtype=torch.uint8, device=dev)
    d_all = torch.empty(P_ALL * PB, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def plan_step():
        native.check(L.ds_plan_batch_device(ctx.handle,
                                            native.c_p(d_pro.data_ptr() + plo * abi.PROBLEM.itemsize),
                                            phi - plo, native.c_p(d_cas.data_ptr()), len(cas),
                                            native.c_p(d_grid.data_ptr()),
                                            native.c_p(d_offs.data_ptr()), 1,
                                            native.c_p(d_out.data_ptr()), sp))
        if comm is not None:
            comm.gather(0, d_out.data_ptr(), (phi - plo) * PB,
                        d_all.data_ptr() if rank == 0 else 0, d_all.numel() if rank == 0 else 0,
                        stream=ctx.stream)
    for _ in range(args.warmup):
        plan_step()
    torch.cuda.synchronize()
    barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        plan_step()
    p1.record(stream)
    torch.cuda.synchronize()
    plan_ms = allmax([p0.elapsed_time(p1) / args.steps])[0]
    plan_value = P_ALL * CANDS_PER_PROBLEM / (plan_ms / 1000.0)
    plan_problems_s = P_ALL / (plan_ms / 1000.0)
    plans_host = (d_all if comm is not None else d_out).cpu().numpy().view(abi.PLAN)
    plans_ok = bool(rank != 0 or plans_host.tobytes() == want_plans.tobytes())
    # planner e2e through the host-buffer C-ABI call (this rank's problems)
    mine_pro = np.ascontiguousarray(pro[plo:phi])
    ctx.plan_batch(mine_pro, cas, grid, goffs)
    barrier()
    t0 = time.perf_counter()
    for _ in range(3):
        ctx.plan_batch(mine_pro, cas, grid, goffs)
    plan_e2e_s = allmax([(time.perf_counter() - t0) / 3])[0]
    plan_e2e = P_ALL * CANDS_PER_PROBLEM / plan_e2e_s

    # ---- planner, threshold-range sharded: every rank searches its slice of
    # the 101-point grid for the SAME problems, the packed selection keys are
    # MIN-all-reduced, every rank decodes (SURVEY 8(e) "by t-range";
    # ds_plan_sharded_device -- NCCL from the library at N > 1)
    G_T = int(grid.size)
    t_lo, t_hi = ddist.shard_range(G_T, ws, rank)
    d_keys = torch.empty(P_ALL, dtype=torch.int64, device=dev)
    d_out2 = torch.empty(P_ALL * PB, dtype=torch.uint8, device=dev)

    def tplan_step():
        with torch.cuda.stream(stream):
            if comm is not None:
                comm.plan(d_pro.data_ptr(), P_ALL, d_cas.data_ptr(), len(cas), d_grid.data_ptr(),
                          d_offs.data_ptr(), 1, t_lo, t_hi, d_out2.data_ptr(),
                          stream=ctx.stream)
                return
            args_ = (ctx.handle, native.c_p(d_pro.data_ptr()), P_ALL,
                     native.c_p(d_cas.data_ptr()), len(cas), native.c_p(d_grid.data_ptr()),
                     native.c_p(d_offs.data_ptr()), 1)
            native.check(L.ds_plan_keys_device(*args_, t_lo, t_hi,
                                               native.c_p(d_keys.data_ptr()), sp))
            native.check(L.ds_plan_from_keys_device(*args_, native.c_p(d_keys.data_ptr()),
                                                    native.c_p(d_out2.data_ptr()), sp))
    tplan_step()
    torch.cuda.synchronize()
    barrier()
    tplan_ms = allmax([timed(tplan_step, max(3, args.steps // 2))])[0]
    tplan_value = P_ALL * CANDS_PER_PROBLEM / (tplan_ms / 1000.0)
    tplan_parity = d_out2.cpu().numpy().tobytes() == want_plans.tobytes()

    # ---- latent leg (config 5 queries, the reference's own scorer): 1M per
    # rank (distinct id ranges), route at t = 0.5, curve over the global
    # sequence (at N > 1 the confidences all-gathered, every rank replays) ----
    lconf = torch.empty(N_LATENT, dtype=torch.float64, device=dev)
    lheavy = torch.empty(N_LATENT, dtype=torch.int64, device=dev)
    lcount = torch.empty(1, dtype=torch.int64, device=dev)
    lcurve = torch.empty_like(prior_t)
    thr = torch.tensor([0.5], dtype=torch.float64, device=dev)
    qm = workloads.query_model()
    lat_id0 = rank * N_LATENT
    levs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    uprior = torch.from_numpy(workloads.uniform_prior().reshape(1).view(np.uint8).copy()).to(dev)
    torch.cuda.synchronize()

    def latent_step(ev=False):
        with torch.cuda.stream(stream):
            if ev:
                levs[0].record(stream)
            native.check(L.ds_score_latent_device(ctx.handle, abi.ptr(qm), lat_id0, N_LATENT,
                                                  native.c_p(lconf.data_ptr()), native.c_p(0), sp))
            if ev:
                levs[1].record(stream)
            if comm is None:
                native.check(L.ds_route_device(ctx.handle, native.c_p(lconf.data_ptr()),
                                               abi.CONF_F64, N_LATENT, native.c_p(thr.data_ptr()),
                                               1, lat_id0, native.c_p(lheavy.data_ptr()),
                                               native.c_p(lcount.data_ptr()), sp))
            else:
                comm.route(lconf.data_ptr(), abi.CONF_F64, N_LATENT, thr.data_ptr(), 1, lat_id0,
                           lheavy.data_ptr(), lcount.data_ptr(), stream=ctx.stream)
            if ev:
                levs[2].record(stream)
            lcurve.copy_(uprior)
            if comm is None:
                native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(lcurve.data_ptr()),
                                                       native.c_p(lconf.data_ptr()), abi.CONF_F64,
                                                       N_LATENT, DECAY, sp))
            else:
                comm.curve_observe(lcurve.data_ptr(), lconf.data_ptr(), abi.CONF_F64,
                                   [N_LATENT] * ws, DECAY, stream=ctx.stream)
            if ev:
                levs[3].record(stream)
    latent_step()
    torch.cuda.synchronize()
    barrier()
    latent_step(ev=True)
    torch.cuda.synchronize()
    lat_ms = [levs[i].elapsed_time(levs[i + 1]) for i in range(3)]
    lconf_host = lconf.cpu().numpy()
    lheavy_host = lheavy[:int(lcount.item())].cpu().numpy()
    lcurve_host = lcurve.cpu().numpy().view(abi.CURVE)[0].copy()
    latent_value = ws * N_LATENT / (allmax([sum(lat_ms)])[0] / 1000.0)
    # K4 / K2 alone (kernel-level views for the rooflines below), timed as
    # CUDA-graph replays: GPU time, not the host's per-call enqueue rate
    def graph_ms(enqueue, reps):
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            enqueue(native.c_p(gs.cuda_stream))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(reps):
                enqueue(native.c_p(gs.cuda_stream))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(gs):
            g.replay()
            a.record(gs)
            g.replay()
            b.record(gs)
        torch.cuda.synchronize()
        del g
        return a.elapsed_time(b) / reps
    k4_ms = allmax([graph_ms(lambda s_: native.check(L.ds_score_latent_device(
        ctx.handle, abi.ptr(qm), lat_id0, N_LATENT, native.c_p(lconf.data_ptr()),
        native.c_p(0), s_)), 10)])[0]
    k2_ms = allmax([graph_ms(lambda s_: native.check(L.ds_route_device(
        ctx.handle, native.c_p(lconf.data_ptr()), abi.CONF_F64, N_LATENT,
        native.c_p(thr.data_ptr()), 1, lat_id0, native.c_p(lheavy.data_ptr()),
        native.c_p(lcount.data_ptr()), s_)), 20)])[0]
    k1_ms = allmax([graph_ms(lambda s_: native.check(L.ds_plan_batch_device(
        ctx.handle, native.c_p(d_pro.data_ptr()), P_ALL, native.c_p(d_cas.data_ptr()), len(cas),
        native.c_p(d_grid.data_ptr()), native.c_p(d_offs.data_ptr()), 1,
        native.c_p(d_out2.data_ptr()), s_)), 10)])[0]
    k2_check = lheavy[:int(lcount.item())].cpu().numpy()
    k2_ok = bool(np.array_equal(k2_check, lheavy_host))
    del lconf, lheavy

    # ---- workload leg: arrivals (K8) + Query records (K4); every rank its own
    # trace (seed WL_SEED + rank) and id range -- distinct work per rank -------
    wl_rates = np.asarray(WL_RATES, np.float64)
    wl_cap = 1_100_000
    wl_seed = WL_SEED + rank
    wl_arr = torch.empty(wl_cap, dtype=torch.float64, device=dev)
    wl_rec = torch.empty(wl_cap * 6, dtype=torch.float64, device=dev)   # ds_query = 48 B
    wl_n = native.i64(0)
    wevs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    def workload_step(ev=False):
        with torch.cuda.stream(stream):
            if ev:
                wevs[0].record(stream)
            native.check(L.ds_generate_arrivals_device(
                ctx.handle, abi.ptr(wl_rates), len(wl_rates), 1.0, wl_seed, abi.ARRIVALS_POISSON,
                native.c_p(wl_arr.data_ptr()), wl_cap, native.ctypes.byref(wl_n), sp))
            if ev:
                wevs[1].record(stream)
            native.check(L.ds_sample_queries_device(
                ctx.handle, abi.ptr(qm), rank * wl_cap, native.c_p(wl_arr.data_ptr()), wl_n.value,
                5.0, native.c_p(wl_rec.data_ptr()), sp))
            if ev:
                wevs[2].record(stream)
    for _ in range(2):
        workload_step()
    torch.cuda.synchronize()
    barrier()
    wl_ms = [0.0, 0.0]
    for _ in range(5):
        workload_step(ev=True)
        torch.cuda.synchronize()
        wl_ms[0] += wevs[0].elapsed_time(wevs[1]) / 5
        wl_ms[1] += wevs[1].elapsed_time(wevs[2]) / 5
    wl_count = wl_n.value
    wl_counts = torch.tensor([float(wl_count)], dtype=torch.float64)
    if ws > 1:
        wl_counts = wl_counts if backend == "gloo" else wl_counts.to(dev)
        dist.all_reduce(wl_counts)
    wl_total = float(wl_counts.cpu()[0])
    wl_value = wl_total / (allmax([sum(wl_ms)])[0] / 1000.0)
    wl_arr_value = wl_total / (allmax([wl_ms[0]])[0] / 1000.0)

    # ---- csv leg: queries.csv of 1M records per rank (distinct records) -------
    crec = csv_records(N_CSV, seed=12 + rank)
    drec = torch.from_numpy(crec.view(np.uint8).copy()).to(dev)
    csv_cap = N_CSV * 256 + 4096
    dcsv = torch.empty(csv_cap, dtype=torch.uint8, device=dev)
    csv_n = native.i64(0)
    cevs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()

    def csv_step(ev=False):
        with torch.cuda.stream(stream):
            if ev:
                cevs[0].record(stream)
            native.check(L.ds_format_queries_csv_device(
                ctx.handle, native.c_p(drec.data_ptr()), N_CSV, native.c_p(dcsv.data_ptr()),
                csv_cap, native.ctypes.byref(csv_n), sp))
            if ev:
                cevs[1].record(stream)
    csv_step()
    torch.cuda.synchronize()
    barrier()
    csv_ms = 0.0
    for _ in range(3):
        csv_step(ev=True)
        torch.cuda.synchronize()
        csv_ms += cevs[0].elapsed_time(cevs[1]) / 3
    csv_value = ws * N_CSV / (allmax([csv_ms])[0] / 1000.0)
    barrier()
    t0 = time.perf_counter()
    csv_bytes = ctx.format_queries_csv(crec)
    csv_e2e = ws * N_CSV / allmax([time.perf_counter() - t0])[0]
    csv_dev_ok = bool(dcsv[:csv_n.value].cpu().numpy().tobytes() == csv_bytes)

    if rank == 0:
        peaks, peak_src = load_peaks()
        achieved_tflops = N_IMG * DISC_FLOP_BF16_EQ / (disc_ms / 1000.0) / 1e12
        peak_burst = float(peaks["bf16_tflops"])
        peak_sus = float(peaks.get("bf16_tflops_sustained", peak_burst))
        hbm = float(peaks["hbm_gbs"])
        prof = load_profile_summaries()
        traffic = prof.get("disc", {}).get("dram_bytes_per_launch_5000img")
        # K2 at 1M f64 confidences, t = 0.5: algorithmic bytes = the confidences
        # read once + one 8-byte id per deferred query + the count
        k2_bytes = N_LATENT * 8 + int(lcount.item()) * 8 + 8
        k2_gbs = k2_bytes / (k2_ms / 1000.0) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8xs8->s32 (layer 1), bf16 x bf16 -> f32 (layers 2-3)",
            "data": "synthetic (device-generated 512x512 u8 images; seeded PatchDisc weights)",
            "config": {"workload": WORKLOAD,
                       "global_batch": ws * N_IMG, "image_hw": [H, W],
                       "thresholds": NT, "parallelism": f"dp{ws} (query shards)",
                       "collectives": ("none (1 GPU)" if ws == 1 else
                                       f"library {'NCCL' if backend == 'nccl' else 'host/gloo'}: "
                                       "count all-gather, queue gather at rank 0, confidence "
                                       "all-gather for the global curve"),
                       "l2": "inputs 3.9 GB/GPU > 126 MB L2, no flush"},
            "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": peak_burst,
                         "unit": "TFLOP/s (bf16-equivalent)", "frac": achieved_tflops / peak_burst,
                         "traffic": traffic, "kernel": "disc_kernel",
                         "peak_source": f"{peak_src} bf16_tflops (burst; the kernel runs at max "
                                        "SM clock, see clocks)",
                         "frac_of_sustained": achieved_tflops / peak_sus,
                         "disc_ms_per_step": disc_ms,
                         "flop_per_image": DISC_FLOP_PER_IMG,
                         "flop_per_image_bf16_equivalent": DISC_FLOP_BF16_EQ,
                         "note": "layer 1 (27% of FLOPs) is u8 x s8 on the int8 tensor path at "
                                 "2x the bf16 rate; its FLOPs count half",
                         "tensor_pipe": tensor_pipe_frac(clocks.get("in_kernel"))},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "bound": {"what": "host->device copy of the images (PCIe)",
                              "achieved_gbs": e2e_gbs, "h2d_copy_alone_gbs": h2d_gbs,
                              "frac": e2e_gbs / h2d_gbs}},
            "gpu_launches": launches,
            "clocks": clocks,
            "parity": {"route_counts_vs_confidences": parity_ok,
                       "route_ids_at_0.5_vs_confidences": lists_ok,
                       "device_errors": take_err == -1,
                       **parity_n1},
            "scaleout": {"value": scale_value, "unit": "images/s", "queries": N_SCALE,
                         "queries_per_gpu": n5, "ms": scale_ms, "routed_at_0.5": scale_routed,
                         "config": "config 5: 1M 512x512 queries, contiguous id shards, 5K "
                                   "resident pool per GPU, route t=0.5; N > 1: routed-count "
                                   "all-gather + global queue at rank 0"},
            "cascade1_batch32": {"value": b32_value, "unit": "images/s",
                                 "us_per_batch": b32_batch_us, "batch": B1,
                                 "parity_vs_full_batch": b32_parity,
                                 "cuda_graph": {"value": ws * N_IMG / (b32g_ms / 1000.0),
                                                "unit": "images/s",
                                                "us_per_batch": b32g_ms * 1000.0 / NB1,
                                                "roofline_us_per_batch": 1e6 * B1 *
                                                DISC_FLOP_BF16_EQ / (peak_burst * 1e12),
                                                "parity_vs_full_batch": b32g_parity},
                                 "backlog": {"value": ws * N_IMG / (bl_ms / 1000.0),
                                             "unit": "images/s",
                                             "us_per_batch": bl_ms * 1000.0 / NB1,
                                             "call": "ds_disc_batches_complete_device (all 157 "
                                                     "batches in one call)",
                                             "parity_vs_batch_by_batch": bl_parity},
                                 "config": "config 1: 5K 512x512 in light batches of 32 "
                                           "(ds_disc_batch_complete_device per batch): score, "
                                           "observe into the curve, route at the batch's t"},
            "cascade3": {"value": c3_value, "unit": "images/s", "image_hw": [H3, H3],
                         "images": N3, "ms_per_step": c3_ms,
                         "disc_bf16eq_tflops_step": c3_tflops,
                         "config": "config 3: 5K 1024x1024 (15.7 GB), score + route at 101 "
                                   "thresholds + curve replay"},
            "planner_t_sharded": {"value": tplan_value, "unit": "candidates/s",
                                  "problems": P_ALL, "grid_slice": [t_lo, t_hi],
                                  "ms_per_batch": tplan_ms, "scaling": "strong",
                                  "parity_vs_reference": bool(tplan_parity),
                                  "config": "config 4 batch, each rank a contiguous slice of "
                                            "the threshold grid, MIN all-reduce of the packed "
                                            "keys (ds_plan_sharded_device), decode"},
            "planner": {"value": plan_value, "unit": "candidates/s", "problems": P_ALL,
                        "problems_per_s": plan_problems_s,
                        "candidates_per_problem": CANDS_PER_PROBLEM, "ms_per_batch": plan_ms,
                        "scaling": "strong (one 4,096-problem batch split by problem index)",
                        "inputs": "tests/golden/config4_bench.npz: 4,096 acceptance-C2 "
                                  "problems (mt19937_64(7)) made by the reference",
                        "curves_from_product_equal_reference": bool(curves_ok),
                        "parity_vs_reference": plans_ok,
                        "roofline": issue_roofline(prof.get("plan_sweep"), k1_ms,
                                                   "plan_sweep_kernel (all 4,096 problems, one "
                                                   "GPU, CUDA-graph time)"),
                        "e2e": {"value": plan_e2e, "unit": "candidates/s",
                                "ms_per_batch": plan_e2e_s * 1000.0}},
            "latent": {"value": latent_value, "unit": "queries/s", "queries_per_gpu": N_LATENT,
                       "ms_score_route_curve": lat_ms,
                       "roofline": issue_roofline(prof.get("latent"), k4_ms,
                                                  "latent_kernel (1M queries, CUDA-graph time)"),
                       "route_roofline": {"bound": "hbm", "kernel": "K2 route (1M f64, t=0.5)",
                                          "achieved": k2_gbs, "peak": hbm, "unit": "GB/s",
                                          "frac": k2_gbs / hbm, "ms": k2_ms,
                                          "timing": "CUDA-graph replay of 20 launches",
                                          "lists_equal_leg": k2_ok,
                                          "algorithmic_bytes": k2_bytes,
                                          "traffic": prof.get("route", {}).get(
                                              "dram_bytes_per_launch")}},
            "workload": {"value": wl_value, "unit": "queries/s",
                         "arrivals_per_s": wl_arr_value, "arrivals_rank0": wl_count,
                         "arrivals_all_ranks": wl_total,
                         "ms_arrivals_records": wl_ms,
                         "trace": "400 intervals x 2500 qps, Poisson, seed 3 + rank"},
            "csv": {"value": csv_value, "unit": "rows/s", "rows_per_gpu": N_CSV,
                    "bytes": csv_n.value, "ms": csv_ms,
                    "e2e": {"value": csv_e2e, "unit": "rows/s",
                            "note": "host records in, host bytes out (ds_format_queries_csv)"},
                    "parity_device_vs_host": csv_dev_ok},
        }
        if ws == 1 and not args.no_cpu:
            cpu_legs(line, args, c_host, prior, step_curve, pro, cas, grid, goffs, plans_host,
                     lconf_host, lheavy_host, lcurve_host, wl_arr[:wl_count].cpu().numpy(), crec)
        print(json.dumps(line), flush=True)
        try:
            np.savez(os.path.join(ROOT, "gpurun_out", f"disc_weights_seed{WEIGHT_SEED}.npz"),
                     **disc.export())
        except Exception:
            pass
    barrier()
    if comm is not None:
        comm.close()
    disc.close()
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


def load_profile_summaries():
    """ncu per-launch figures committed under profiles/ (fixed for these
    inputs): dram bytes of disc_kernel and K2, executed warp-instructions of
    K1 and K4 (their issue roofline)."""
    out = {}
    for key, name in (("disc", "disc_ncu_summary.json"), ("route", "route_ncu_summary.json"),
                      ("plan_sweep", "plan_sweep_ncu_summary.json"),
                      ("latent", "latent_ncu_summary.json")):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            with open(p) as f:
                out[key] = json.load(f)
    return out


def issue_roofline(summary, ms, kernel):
    """Issue-bound kernels (no tensor or HBM bound): the launch's executed
    warp-instructions (ncu, fixed for these inputs) at the SMs' issue peak of
    4 warp-instructions per clock (148 SMs, max SM clock) is the floor;
    frac = floor / measured time."""
    if not summary or "warp_inst_per_launch" not in summary:
        return {"bound": "issue (int/fp64)", "kernel": kernel, "frac": None,
                "note": "no ncu instruction count committed"}
    peaks, _ = load_peaks()
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = int(summary.get("sms", 148))
    floor_ms = summary["warp_inst_per_launch"] / (sms * 4 * mhz * 1e6) * 1e3
    achieved = summary["warp_inst_per_launch"] / (ms / 1000.0) / 1e9
    peak = sms * 4 * mhz * 1e6 / 1e9
    return {"bound": "issue (int/fp64)", "kernel": kernel, "unit": "G warp-inst/s",
            "achieved": achieved, "peak": peak, "frac": floor_ms / ms, "ms": ms,
            "traffic": summary.get("dram_bytes_per_launch"),
            "source": summary.get("source")}


def cpu_legs(line, args, c_host, prior, gpu_curve, pro, cas, grid, goffs, gpu_plans, lconf_host,
             lheavy_host, lcurve_host, wl_arr, crec):
    """The CPU reference path on this box's host cores (rank 0, N = 1), and
    the parity checks that need it (the oracle/_ref checker)."""
    from oracle import lib
    from paper_2411_15381_b200 import abi, workloads
    threads = os.cpu_count() or 1
    cv, ck, cpu_conf = cpu_images_leg(CPU_DISC_SAMPLE)
    line["cpu_baseline"] = {"value": cv, "unit": "images/s", "cores": threads,
                            "kind": "port" if ck != "reference" else ck,
                            "sample": f"{CPU_DISC_SAMPLE} images 512x512: numpy fp32 port of "
                                      "the discriminator on every host thread (no reference network) + the "
                                      "reference route loop at 101 thresholds"}
    g = c_host[:len(cpu_conf)]
    rel = np.abs(g - cpu_conf) / np.maximum(np.abs(cpu_conf), 1e-2)
    line["parity"]["disc_vs_cpu_port"] = {"images": int(len(cpu_conf)),
                                          "max_rel_err": float(rel.max()),
                                          "within_1e-3": bool(rel.max() <= 1e-3)}
    # the step's curve vs the reference's observe loop on the same confidences
    use_ref = lib.ref_available()
    cw = prior.copy()
    idx = np.zeros(len(c_host), np.int64)
    cnt = np.zeros(1, np.int64)
    (lib.ref().dsref_route_loop if use_ref else lib.port().dso_route_loop)(
        abi.ptr(c_host), len(c_host), 0.5, 1, DECAY, abi.ptr(cw), abi.ptr(idx), abi.ptr(cnt))
    line["parity"]["curve_bits_vs_reference_loop"] = bool(cw.tobytes() == gpu_curve.tobytes())
    line["parity"]["route_ids_at_0.5_vs_reference_loop"] = bool(
        np.array_equal(idx[:int(cnt[0])], np.flatnonzero(c_host < 0.5)))
    # planner: diffserve::solve over the IDENTICAL 4,096-problem batch, all
    # threads and one thread
    pv, pk, cpu_plans, pt = cpu_planner_leg(pro, cas, grid, goffs, threads)
    pv1, _, _, pt1 = cpu_planner_leg(pro, cas, grid, goffs, 1)
    line["planner"]["cpu_baseline"] = {
        "value": pv, "unit": "candidates/s", "cores": threads, "kind": pk,
        "problems_per_s": len(pro) / pt, "seconds": pt,
        "one_thread": {"value": pv1, "problems_per_s": len(pro) / pt1, "seconds": pt1},
        "sample": f"the identical {len(pro)}-problem batch, diffserve::solve on "
                  f"{threads} threads and on 1"}
    line["planner"]["parity_cpu_vs_gpu"] = bool(cpu_plans.tobytes() == gpu_plans.tobytes())
    line["planner"]["speedup_vs_cpu_all_threads"] = pt / (line["planner"]["ms_per_batch"] / 1e3)
    lv, lk, lconf_cpu, lidx_cpu = cpu_latent_leg(CPU_LATENT_SAMPLE, threads)
    lv1, _, _, _ = cpu_latent_leg(CPU_LATENT_SAMPLE // 4, 1)
    line["latent"]["cpu_baseline"] = {
        "value": lv, "unit": "queries/s", "cores": threads, "kind": lk,
        "one_thread": {"value": lv1, "sample": f"{CPU_LATENT_SAMPLE // 4} queries"},
        "sample": f"{CPU_LATENT_SAMPLE} queries: sample_query on {threads} threads + "
                  "sequential observe/defers loop"}
    g = lconf_host[:CPU_LATENT_SAMPLE]
    rel = np.abs(g - lconf_cpu) / np.maximum(np.abs(lconf_cpu), 1e-2)
    gl = lheavy_host[lheavy_host < CPU_LATENT_SAMPLE]
    # the latent leg's curve (1M observations, uniform prior) vs the
    # reference's loop over the GPU's confidences
    cl = workloads.uniform_prior()
    li = np.zeros(len(lconf_host), np.int64)
    (lib.ref().dsref_route_loop if use_ref else lib.port().dso_route_loop)(
        abi.ptr(lconf_host), len(lconf_host), 0.5, 1, DECAY, abi.ptr(cl), abi.ptr(li),
        abi.ptr(cnt))
    line["latent"]["curve_bits_vs_reference_loop"] = bool(cl.tobytes() == lcurve_host.tobytes())
    line["latent"]["heavy_ids_vs_reference_loop"] = bool(
        np.array_equal(li[:int(cnt[0])], lheavy_host))
    line["latent"]["parity_vs_cpu"] = {
        "queries": CPU_LATENT_SAMPLE, "max_rel_err": float(rel.max()),
        "bit_identical": int((g.view(np.uint64) == lconf_cpu.view(np.uint64)).sum()),
        "all_bit_identical": bool(np.array_equal(g.view(np.uint64), lconf_cpu.view(np.uint64))),
        "heavy_ids_equal": bool(np.array_equal(gl, lidx_cpu))}
    wv, wav, wk, wa = cpu_workload_leg(threads)
    line["workload"]["cpu_baseline"] = {
        "value": wv, "unit": "queries/s", "arrivals_per_s": wav, "cores": threads,
        "kind": wk, "sample": f"the full {len(wa)}-arrival trace: generate_arrivals "
                              f"(sequential) + sample_query on {threads} threads"}
    line["workload"]["parity_vs_cpu"] = bool(len(wa) == len(wl_arr) and
                                             wl_arr.tobytes() == wa.tobytes())
    cv2, ck2 = cpu_csv_leg(np.ascontiguousarray(crec[:CPU_CSV_SAMPLE]))
    line["csv"]["cpu_baseline"] = {
        "value": cv2, "unit": "rows/s", "cores": 1, "kind": ck2,
        "sample": f"{CPU_CSV_SAMPLE} QueryRecords through write_csv (file in a tmp dir)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline legs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
