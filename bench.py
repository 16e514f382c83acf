#!/usr/bin/env python
"""Benchmark: rollout+BIC states scored per second (BASELINE.json metric), on
the configs[1] workload -- dubins (unicycle/car) reaching with obstacles,
N = 65,536 candidate initial states per GPU, H = 64 networks, gap x std score.

One step (metric 1) = for every candidate: a T-step
actor rollout with running + terminal cost (K1), critic V(x0) and std sigma(x0)
(K2, fused into the K1 launch), score sigma*|V - J|, a stable top-(N/10) select
(K3), and the kept 1/10's warm starts U (taken from the K1 controls).  `value` is device-resident
(inputs already in HBM); `e2e` goes through the public API with the candidate
states in pinned host memory and the kept indices + warm starts read back.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU (torchrun): each rank scores its own 65,536-candidate shard (weak
scaling), the shard winners are merged exactly with ONE NCCL all-gather, and
each rank returns the warm starts of its slice of the global kept set.

  --workload {dubins, pointmass, manipulator3, aliengo_lipm} selects the other
  BASELINE.json configs (N per GPU: 65,536 / 750 / 262,144 / 131,072 = the 1M
AlienGO set sharded 8 ways); the default is configs[1] (dubins).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "rollout+BIC states scored/sec"
CONFIG_NAME = "dubins"
N_PER_GPU = 65536
WORKLOADS = {"dubins": 65536, "pointmass": 750, "manipulator3": 262144, "aliengo_lipm": 1 << 17}
HIDDEN = 64
CAND_MULT = 10
SEED = 0


# ---------------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------------

def make_nets(spec, rng_seed=SEED):
    """TrainerState-style networks (trainer.py:96-118): Glorot init, output layer
    x0.1, workspace normalisation; the actor output layer is then scaled x10 so
    the synthetic policy produces non-trivial controls (declared in `data`)."""
    from paper_2602_19699_b200 import nets, specs
    rng = np.random.default_rng(np.random.SeedSequence([rng_seed, 0]))
    c, h = specs.normalisation(spec)
    d = spec.n + 1
    critic = nets.init_mlp([d, HIDDEN, HIDDEN, HIDDEN, 1], rng, in_center=c, in_half=h)
    actor = nets.init_mlp([d, HIDDEN, HIDDEN, HIDDEN, spec.m], rng, head="tanh", out_scale=spec.u_bound,
                          in_center=c, in_half=h)
    std = nets.init_mlp([d, HIDDEN, HIDDEN, HIDDEN, 1], rng, head="std", in_center=c, in_half=h)
    p = list(actor.flat_params())
    p[-2] = p[-2] * 10.0
    return actor.with_params(p), critic, std


def candidates(spec, lo_row, count, seed=SEED):
    """Rows [lo_row, lo_row+count) of sample_initial_states(spec, N_total, seed)
    (envs/__init__.py:112-122): uniform over the workspace, t = 0."""
    from paper_2602_19699_b200 import specs
    lo, hi = specs.region_box(spec)
    g = np.random.default_rng(seed)
    g.bit_generator.advance(lo_row * spec.n)
    return g.uniform(size=(count, spec.n)) * (hi - lo) + lo


def flops_per_candidate(spec, T):
    """GEMM FLOPs (2*MAC) per candidate: F_roll (1 + 1/cm) + 2 F_fwd."""
    d, H, m = spec.n + 1, HIDDEN, spec.m
    f_roll = T * 2 * (d * H + 2 * H * H + H * m)
    f_fwd = 2 * (d * H + 2 * H * H + H)
    return f_roll, f_roll * (1 + 1 / CAND_MULT) + 2 * f_fwd


# ---------------------------------------------------------------------------------
# clocks (NVML sampled during the timed region)
# ---------------------------------------------------------------------------------

class ClockSampler:
    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
               "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, device_index):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            uuid = "GPU-" + str(torch.cuda.get_device_properties(device_index).uuid)
            try:
                self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML missing
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()

    def stop(self):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        reasons = [k for k, bit in self.REASONS.items() if self.reasons & bit and k != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------------
# CPU baseline (the oracle port of the reference path, all host cores)
# ---------------------------------------------------------------------------------

_W = {}


def _worker_init(actor, spec, field):
    import threadpoolctl
    threadpoolctl.threadpool_limits(1)
    _W.update(actor=actor, spec=spec, field=field)


def _worker_rollouts(args):
    from oracle import nets as O_nets
    x0s, with_field = args
    out = []
    for x0 in x0s:
        X, U, sc = O_nets.actor_rollout(_W["actor"], _W["spec"], x0, 0, _W["spec"].t_max,
                                        _W["field"] if with_field else None)
        out.append(float(sc.sum()) if with_field else U.shape[0])
    return out


def cpu_pipeline(spec, field, actor, critic, std, x0, pool, cores):
    """The reference hot path on the host, per candidate exactly as trajrl runs it:
    per-start actor_rollout with costs (nets.py:403-423), critic / std forward
    (nets.py:165-173), stable argsort select (trainer.py:150-153) and the
    per-start warm-start rollouts of the kept starts (trainer.py:192-193)."""
    from oracle import nets as O_nets, select as O_select
    N = x0.shape[0]
    keep = max(1, N // CAND_MULT)
    chunks = [(x0[i::cores], True) for i in range(cores)]
    costs = np.empty(N)
    for i, res in enumerate(pool.map(_worker_rollouts, chunks)):
        costs[i::cores] = res
    xa = O_select.augmented(x0)
    s = O_select.std_scores(std, xa) * O_select.gap_scores(critic, xa, costs)
    order = O_select.select_order(s, keep)
    kept = x0[order]
    list(pool.map(_worker_rollouts, [(kept[i::cores], False) for i in range(cores)]))
    return order


def run_cpu(spec, field, actor, critic, std, sample, steps=1, warmup=0):
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores, initializer=_worker_init, initargs=(actor, spec, field)) as pool:
        x0 = candidates(spec, 0, sample)
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            cpu_pipeline(spec, field, actor, critic, std, x0, pool, cores)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
    return cores, times


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------

TF32_DENSE_TFLOPS = 1100.0   # /opt/skills/guides/B200_PROFILING.md peak table (dense tf32)


def measure_fp32_peak(torch, _lib, stream):
    """FFMA throughput of this B200 (roofline denominator of the SIMT kernels)."""
    blocks = 148 * 8
    iters = 4096
    out = torch.empty(blocks, device="cuda")
    flops = 2 * 16 * 8 * iters * blocks * 256
    for _ in range(2):
        _lib.call("cacto_fma_peak", _lib.F32, blocks, iters, out.data_ptr(), stream)
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("cacto_fma_peak", _lib.F32, blocks, iters, out.data_ptr(), stream)
        b.record()
        b.synchronize()
        best = max(best, flops / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cacto", choices=["cacto", "reference"])
    ap.add_argument("--n", type=int, default=0, help="candidates per GPU (0: the workload's)")
    ap.add_argument("--workload", default="dubins", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="CPU baseline sample (0 = auto)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    global CONFIG_NAME, N_PER_GPU
    CONFIG_NAME = args.workload
    N_PER_GPU = WORKLOADS[args.workload]
    if args.n <= 0:
        args.n = N_PER_GPU

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2602_19699_b200 import specs
    spec, field = specs.config(CONFIG_NAME)
    actor, critic, std = make_nets(spec)
    T = spec.t_max
    f_roll, f_cand = flops_per_candidate(spec, T)

    if args.impl == "reference":
        if rank != 0:
            return
        cores = len(os.sched_getaffinity(0))
        sample = min(args.cpu_sample or max(64, cores * 64), N_PER_GPU)    # ~0.6 s per step
        cores, times = run_cpu(spec, field, actor, critic, std, sample, args.steps, max(1, args.warmup))
        sec = float(np.mean(times))
        val = sample / sec
        line = {"metric": METRIC, "value": val, "unit": "states/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference",
                "config": {"workload": f"{CONFIG_NAME} rollout+BIC, {sample} candidates per step (bounded CPU "
                                       f"sample of the {N_PER_GPU}-candidate config), H={HIDDEN}, T={T}",
                           "candidates_per_step": sample, "keep_fraction": 1 / CAND_MULT},
                "cpu_baseline": {"value": val, "unit": "states/s", "cores": cores, "kind": "port",
                                 "sample": f"{sample} candidates/step, per-start NumPy rollouts on a {cores}-process "
                                           f"pool ({cpu_model()})"},
                "e2e": {"value": val, "unit": "states/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    import paper_2602_19699_b200 as P
    from paper_2602_19699_b200 import _lib, parallel, trainer
    P.set_precision(args.precision)
    stream = torch.cuda.current_stream().cuda_stream

    N = args.n
    keep_global = (N * world) // CAND_MULT
    base = rank * N
    x0_host = candidates(spec, base, N)
    x0_pinned = torch.from_numpy(x0_host).pin_memory()
    x0_dev = x0_pinned.to("cuda")
    pipe = trainer.BicPipeline(spec, field, actor, critic, std, mode="std_x_gap", precision=args.precision)
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")  # > 126 MB L2

    def step(x0):
        if world == 1:
            out = pipe.run(x0, keep_global)
            return out["order"], out["U"]
        # every global winner is among its own shard's top-keep, so each rank keeps the
        # warm starts of its local top-keep (taken from its cost rollout) and, after the
        # exact merge, a mask of which of them made the global cut -- no second rollout
        # and no control traffic between ranks
        out = pipe.run(x0, min(keep_global, N), warm_starts=True)
        rs, ro, rx = parallel.gather_winners(out["scores"], out["order"] + base,
                                             x0.index_select(0, out["order"]), keep_global)
        pos = parallel.merge_positions(rs, ro, keep_global, parallel.device_merge)
        gorder = ro.index_select(0, pos)
        kept = torch.isin(out["order"] + base, gorder)
        return gorder, (out["U"], kept)

    def timed(fn, K, W):
        for _ in range(W):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        total = 0.0
        for _ in range(K):
            flush.fill_(1.0)  # evict L2 between timed steps (outside the event pair)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            total += a.elapsed_time(b)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            t = torch.tensor([total], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return total / K  # ms per step

    # ---- device-resident value ----------------------------------------------------
    clocks = ClockSampler(local_rank)
    for _ in range(args.warmup):
        step(x0_dev)
    clocks.start()
    ms = timed(lambda: step(x0_dev), args.steps, 0)
    clk = clocks.stop()
    value = (N * world) / (ms * 1e-3)
    launches_per_step = pipe.kernel_launches

    # ---- e2e through the public API: pinned host -> device -> kept order + U back --
    keep_local_U = keep_global if world == 1 else min(keep_global, N)
    esz = 4 if args.precision == "fp32" else 8
    order_host = torch.empty(keep_global, dtype=torch.int64).pin_memory()
    U_host = torch.empty((keep_local_U, T, spec.m), dtype=torch.float32 if esz == 4 else torch.float64).pin_memory()
    mask_host = torch.empty(keep_local_U, dtype=torch.bool).pin_memory()

    def e2e_step():
        xd = x0_pinned.to("cuda", non_blocking=True)
        order, U = step(xd)
        order_host.copy_(order, non_blocking=True)
        if world == 1:
            U_host.copy_(U, non_blocking=True)
        else:
            U_host.copy_(U[0], non_blocking=True)
            mask_host.copy_(U[1], non_blocking=True)

    e2e_ms = timed(e2e_step, args.steps, args.warmup)
    e2e_value = (N * world) / (e2e_ms * 1e-3)
    h2d = N * spec.n * 8
    d2h = keep_global * 8 + keep_local_U * T * spec.m * esz + (keep_local_U if world > 1 else 0)

    # ---- roofline of the dominant kernel (K1 rollout over all candidates) ---------
    x0r = x0_dev
    for _ in range(2):
        pipe.rollout_costs(x0r, keep_controls=True)
    evs = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pipe.rollout_costs(x0r, keep_controls=True)
        b.record()
        b.synchronize()
        evs.append(a.elapsed_time(b))
    roll_ms = float(np.mean(evs))
    achieved = f_roll * N / (roll_ms * 1e-3) / 1e12
    ffma_peak = measure_fp32_peak(torch, _lib, stream)
    tc_path = args.precision == "fp32" and os.environ.get("CACTO_ROLLOUT_TC", "1") != "0"
    if tc_path:
        # K1 runs its policy layers on tcgen05 (kind::tf32, 3 MMA passes for fp32
        # accuracy): the roofline is the TF32 tensor pipe
        peak, bound = TF32_DENSE_TFLOPS, "tensor"
        peak_source = ("B200_PROFILING.md fallback: tf32 dense 1.1 PFLOP/s, the fp32-class tensor format "
                       "(MEASURED_PEAKS.json has no tf32 entry); algorithmic flops count each product once, the "
                       "3xFP16 split issues 3x the MMAs at twice tf32's per-K rate")
        kname = "rollout_tc_kernel (K1 on tcgen05, cost-only over all candidates)"
    else:
        peak, bound = ffma_peak, "fp32_simt"
        peak_source = "measured FFMA throughput on this GPU (cacto_fma_peak); MEASURED_PEAKS.json has no fp32 entry"
        kname = "rollout_kernel (K1 SIMT, cost-only over all candidates)"
    traffic = None
    prof = ROOT / "profiles" / "rollout_ncu_summary.json"
    if prof.exists() and args.workload == "dubins" and args.precision == "fp32":  # the captured launch
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": "states/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (uniform workspace starts, Glorot-init networks, actor output layer x10)",
        "config": {"workload": f"{CONFIG_NAME}: {N} candidate starts/GPU -> T={T} rollout with cost, "
                               f"sigma*|V-J| score, stable top-{keep_global} select, kept warm starts (controls of the cost rollout)",
                   "candidates_per_gpu": N, "keep": keep_global, "hidden": [HIDDEN] * 3,
                   "horizon": T, "score": "std_x_gap", "l2": "flushed between timed steps (256 MB write)",
                   "parallelism": f"shard-by-candidate x{world}"},
        "e2e": {"value": e2e_value, "unit": "states/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": kname + ", emitting every candidate's controls (the kept warm starts)", "kernel_ms": roll_ms, "flops_per_candidate_rollout": f_roll,
                     "peak_source": peak_source,
                     "mma_passes": 3 if tc_path else None,
                     "mma_issued_tflops": 3 * achieved if tc_path else None,
                     "mma_kind": "tcgen05 kind::f16, 3xFP16 split (fp16 dense peak 2250 TFLOP/s)" if tc_path else None,
                     "binding_resource": ("CUDA-core epilogue issue (ncu: issue active ~71 %, tensor pipe ~25 %; "
                                          "profiles/r01_ncu_rollout_tc.json)") if tc_path else None,
                     "fp32_ffma_peak": ffma_peak, "vs_ffma_peak": achieved / ffma_peak if ffma_peak else None},
        "clocks": clk,
        "flops_per_candidate": f_cand,
        "achieved_tflops_step": f_cand * N / (ms * 1e-3) / 1e12,
    }

    # ---- secondary: critic Sobolev samples/s (manipulator dims, B = 65536) ----------
    if not args.no_secondary:
        try:
            line["secondary"] = critic_bench(torch, P, stream, world=world, rank=rank,
                                             dist=dist if world > 1 else None)
        except Exception as e:  # keep the primary line alive
            line["secondary"] = {"error": str(e)[:200]}

    # ---- CPU baseline (rank 0, N = 1 only) ---------------------------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        sample = min(args.cpu_sample or max(128, cores * 128), N)   # ~10 core-seconds of work
        cores, times = run_cpu(spec, field, actor, critic, std, sample, 1, 1)
        line["cpu_baseline"] = {"value": sample / times[0], "unit": "states/s", "cores": cores, "kind": "port",
                                "sample": f"{sample} of the {N} candidates through the same pipeline: per-start "
                                          f"NumPy rollouts on a {cores}-process pool ({cpu_model()})"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def critic_bench(torch, P, stream, B=65536, world=1, rank=0, dist=None):
    """One Sobolev critic update per step (fused gather + target forward + Sobolev
    loss with double backprop + fold + Adam + Polyak), data-parallel over ranks:
    every rank draws the same global index stream and takes its B-row slice (weak
    scaling: B per GPU), losses divide by the global batch, and at world > 1 the
    folded gradient (+ loss) is summed with one NCCL all-reduce before Adam
    (north_star: "critic/actor minibatches are data-parallel with an NCCL gradient
    allreduce").  Device-timed, max over ranks."""
    import ctypes
    from paper_2602_19699_b200 import _lib, specs
    from paper_2602_19699_b200.device import DeviceNet
    from paper_2602_19699_b200.buffer import ReplayBuffer, SampleBatch
    spec, _ = specs.config("manipulator3")
    actor, critic, std = make_nets(spec)
    net = DeviceNet(critic)
    tgt = DeviceNet(critic)
    cap = 1 << 20
    buf = ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=cap)
    rng = np.random.default_rng(1)
    lo, hi = specs.region_box(spec)
    rows = 1 << 18
    xa = np.concatenate([rng.uniform(size=(rows, spec.n)) * (hi - lo) + lo,
                         rng.integers(0, spec.t_max, (rows, 1))], axis=1)
    xk = np.concatenate([rng.uniform(size=(rows, spec.n)) * (hi - lo) + lo,
                         rng.integers(1, spec.t_max + 1, (rows, 1))], axis=1)
    buf.push_many(SampleBatch(xa, rng.normal(size=(rows, spec.m)), rng.normal(size=rows),
                              rng.normal(size=(rows, spec.n)), xk, spec.t_max))
    idx_all = rng.integers(0, rows, B * world)           # the global stream, same on every rank
    idx = torch.as_tensor(idx_all[rank * B:(rank + 1) * B]).cuda()
    desc = buf.ring_desc(idx, rows=B)
    desc.denom = B * world                                 # mean over the global batch
    nbytes = _lib.load().cacto_loss_workspace_bytes(net.desc, B)
    ws = torch.empty(nbytes, device="cuda", dtype=torch.uint8)
    m = torch.zeros_like(net.params)
    v = torch.zeros_like(net.params)
    g = torch.empty(net.count + 1, device="cuda", dtype=net.params.dtype)  # grads + loss, one all-reduce
    npart = ctypes.c_int32(0)
    step_no = [0]

    def one():
        _lib.call("cacto_critic_loss", net.desc, tgt.desc, desc, 1.0, 1, ws.data_ptr(), nbytes, npart, stream)
        if world == 1:
            _lib.call("cacto_reduce_adam", net.desc.dtype, ws.data_ptr(), npart.value, net.count,
                      net.params.data_ptr(), m.data_ptr(), v.data_ptr(), step_no[0], 1e-3, 0.9, 0.999, 1e-8,
                      tgt.params.data_ptr(), 0.005, None, None, stream)
        else:
            _lib.call("cacto_reduce_grads", net.desc.dtype, ws.data_ptr(), npart.value, net.count, g.data_ptr(),
                      g[net.count:].data_ptr(), stream)
            dist.all_reduce(g)
            _lib.call("cacto_adam_step", net.desc.dtype, net.params.data_ptr(), m.data_ptr(), v.data_ptr(),
                      g.data_ptr(), net.count, step_no[0], 1e-3, 0.9, 0.999, 1e-8, stream)
            _lib.call("cacto_polyak", net.desc.dtype, tgt.params.data_ptr(), net.params.data_ptr(), net.count, 0.005,
                      stream)
        step_no[0] += 1

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    K = 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        one()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / K
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    H, d = HIDDEN, spec.n + 1
    f = 28 * H * H + 14 * d * H + 8 * H
    return {"metric": "critic Sobolev samples/sec", "value": B * world / (ms * 1e-3), "unit": "samples/s",
            "batch_per_gpu": B, "global_batch": B * world, "n_gpus": world, "hidden": [H] * 3,
            "ms_per_update": ms, "system": "manipulator3 (d=7)", "scaling": "weak",
            "achieved_tflops": f * B * world / (ms * 1e-3) / 1e12, "flops_per_sample": f,
            "includes": "fused gather + target forward + Sobolev fwd/double-backprop + fold + "
                        + ("Adam + Polyak" if world == 1 else "NCCL all-reduce of the gradient + Adam + Polyak"),
            "sweep": "profiles/critic_sweep.py (batch 4k-1M x hidden 64-512, 1 GPU)"}


if __name__ == "__main__":
    main()
