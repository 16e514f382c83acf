#!/usr/bin/env python
"""Benchmark: rollout+BIC states scored per second (BASELINE.json metric), on
the largest single-GPU config -- configs[2], the 3-DoF planar manipulator
reaching with obstacle avoidance, N = 262,144 candidate initial states per GPU,
H = 64 networks, gap x std score.

One step (metric 1) = for every candidate: a T-step
actor rollout with running + terminal cost (K1), critic V(x0) and std sigma(x0)
(K2, fused into the K1 launch), score sigma*|V - J|, a stable top-(N/10) select
(K3), and the kept 1/10's warm starts U (taken from the K1 controls).  `value` is device-resident
(inputs already in HBM); `e2e` goes through the public API with the candidate
states in pinned host memory (read zero-copy by the rollout kernel) and the kept
indices + warm starts returned to pinned host memory.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU (torchrun): each rank scores its own 262,144-candidate shard (weak
scaling); the global stable top-k is found by a distributed radix threshold
(4 all-reduces of a 2 KB histogram, one all-gather of 2 counts per rank, one
all-reduce of the keep winners -- parallel.DistributedSelect), and each rank
returns the warm starts of its OWN winners.

  --workload {dubins, pointmass, manipulator3, aliengo_lipm} selects the other
  BASELINE.json configs (N per GPU: 65,536 / 750 / 262,144 / 131,072 = the 1M
AlienGO set sharded 8 ways); the default is manipulator3 (configs[2]).

Reference arm (`--impl reference`): the UNMODIFIED reference `trajrl` from
baseline/_ref (nets.actor_rollout per start on a process pool over all host
cores, nets.mlp_forward scores, stable argsort, per-start warm-start rollouts --
trainer.py:183-193), on a bounded sample of the same workload.
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
CONFIG_NAME = "manipulator3"
N_PER_GPU = 262144
WORKLOADS = {"dubins": 65536, "pointmass": 750, "manipulator3": 262144, "aliengo_lipm": 1 << 17}
HIDDEN = 64
CAND_MULT = 10
SEED = 0
# e2e: the warm starts go to a pinned host buffer through the public call's u_out; the
# library takes them in chunks and copies each chunk with the copy engine while the next
# chunk's take runs (CACTO_WARM_ZEROCOPY=1: the take kernel writes the host buffer
# directly, measured slower -- SM stores over PCIe stream below the copy engine's rate)


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
    """GEMM FLOPs (2*MAC) per candidate actually executed: F_roll + 2 F_fwd.
    (SURVEY 8d's total adds F_roll / cm for re-rolling the kept starts; here the
    warm starts are the cost rollout's own controls, so that work is not done.)"""
    d, H, m = spec.n + 1, HIDDEN, spec.m
    f_roll = T * 2 * (d * H + 2 * H * H + H * m)
    f_fwd = 2 * (d * H + 2 * H * H + H)
    return f_roll, f_roll + 2 * f_fwd


def tensor_peak():
    """Dense 16-bit tensor peak (the pipe K1's kind::f16 MMAs and the critic's run
    on): MEASURED_PEAKS.json bf16 burst (kernels timed alone), else the fallback."""
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["bf16_tflops"]), "of measured (MEASURED_PEAKS.json bf16_tflops, cuBLAS bf16 burst)"
    except Exception:
        return 1590.0, "of fallback (B200_PROFILING.md: 1.59 PFLOP/s bf16 burst)"


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
    """Pool worker: single-threaded BLAS; the reference objects built once
    (the reference's own solve_batch pool pattern, ilqr.py:332-339)."""
    import threadpoolctl
    threadpoolctl.threadpool_limits(1)
    _W.update(actor=actor, spec=spec, field=field, ref=None)
    try:
        from oracle import refarm
        R = refarm.load()
        _W["ref"] = (R, refarm.mlp(actor), refarm.model(spec), refarm.field(field))
    except Exception as e:  # reference not installed: the oracle port
        _W["ref_error"] = str(e)


def _worker_rollouts(args):
    x0s, with_field = args
    out = []
    if _W.get("ref") is not None:
        R, ra, rm, rf = _W["ref"]
        for x0 in x0s:
            tr = R.nets.actor_rollout(ra, rm, R.envs.TimeState(x0, 0), rm.t_max, rf if with_field else None)
            out.append(float(tr.cost) if with_field else tr.U.shape[0])
        return out
    from oracle import nets as O_nets
    for x0 in x0s:
        X, U, sc = O_nets.actor_rollout(_W["actor"], _W["spec"], x0, 0, _W["spec"].t_max,
                                        _W["field"] if with_field else None)
        out.append(float(sc.sum()) if with_field else U.shape[0])
    return out


def _worker_kind(_):
    return "reference" if _W.get("ref") is not None else "port"


def cpu_pipeline(spec, field, actor, critic, std, x0, pool, cores):
    """The reference hot path on the host, per candidate exactly as trajrl runs it:
    per-start actor_rollout with costs (nets.py:403-423), critic / std forward
    (nets.py:165-173), stable argsort select (trainer.py:150-153) and the
    per-start warm-start rollouts of the kept starts (trainer.py:192-193)."""
    N = x0.shape[0]
    keep = max(1, N // CAND_MULT)
    chunks = [(x0[i::cores], True) for i in range(cores)]
    costs = np.empty(N)
    for i, res in enumerate(pool.map(_worker_rollouts, chunks)):
        costs[i::cores] = res
    xa = np.concatenate([x0, np.zeros((N, 1))], axis=1)
    try:
        from oracle import refarm
        R = refarm.load()
        sig = R.nets.mlp_forward(refarm.mlp(std), xa)[:, 0]
        V = R.nets.mlp_forward(refarm.mlp(critic), xa)[:, 0]
    except Exception:
        from oracle import nets as O_nets
        sig = O_nets.mlp_forward(std, xa)[:, 0]
        V = O_nets.mlp_forward(critic, xa)[:, 0]
    s = sig * np.abs(V - costs)
    order = np.argsort(-s, kind="stable")[:keep]
    kept = x0[order]
    list(pool.map(_worker_rollouts, [(kept[i::cores], False) for i in range(cores)]))
    return order


def run_cpu(spec, field, actor, critic, std, sample, steps=1, warmup=0):
    """(cores, per-step seconds, kind): kind "reference" when baseline/_ref loaded."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores, initializer=_worker_init, initargs=(actor, spec, field)) as pool:
        kind = "reference" if all(k == "reference" for k in pool.map(_worker_kind, range(cores))) else "port"
        x0 = candidates(spec, 0, sample)
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            cpu_pipeline(spec, field, actor, critic, std, x0, pool, cores)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
    return cores, times, kind


def critic_batch(spec, B, world=1, rank=0, seed=1):
    """The synthetic replay rows and the global index stream of metric 2."""
    from paper_2602_19699_b200 import specs
    rng = np.random.default_rng(seed)
    lo, hi = specs.region_box(spec)
    rows = 1 << 18
    xa = np.concatenate([rng.uniform(size=(rows, spec.n)) * (hi - lo) + lo,
                         rng.integers(0, spec.t_max, (rows, 1))], axis=1)
    xk = np.concatenate([rng.uniform(size=(rows, spec.n)) * (hi - lo) + lo,
                         rng.integers(1, spec.t_max + 1, (rows, 1))], axis=1)
    cols = (xa, rng.normal(size=(rows, spec.m)), rng.normal(size=rows), rng.normal(size=(rows, spec.n)), xk)
    idx_all = rng.integers(0, rows, B * world)
    return rows, cols, idx_all


def cpu_critic_baseline(B=65536, reps=2):
    """Metric 2 on the host: reference critic_loss (bootstrap on, k_s = 1) + adam_step
    + polyak (nets.py:233-290, 375-398) on the same B-row batch, best of 1 thread and
    all BLAS threads."""
    import threadpoolctl
    from paper_2602_19699_b200 import specs
    spec, _ = specs.config("manipulator3")
    _, critic, _ = make_nets(spec)
    rows, cols, idx = critic_batch(spec, B)
    kind = "reference"
    try:
        from oracle import refarm
        R = refarm.load()
        net, tgt = refarm.mlp(critic), refarm.mlp(critic)
        batch = R.buffer.SampleBatch(*(c[idx] for c in cols), t_max=spec.t_max)
        loss_fn, adam, polyak = R.nets.critic_loss, R.nets.adam_step, R.nets.polyak
        state = R.nets.AdamState.init(net.flat_params())

        def one():
            nonlocal net, tgt, state
            _, g = loss_fn(net, tgt, batch, 1.0, True)
            p, state = adam(net.flat_params(), state, g)
            net = net.with_params(p)
            tgt = polyak(tgt, net, 0.005)
    except Exception:
        from types import SimpleNamespace
        from oracle import nets as O_nets
        kind = "port"
        batch = SimpleNamespace(xa=cols[0][idx], u=cols[1][idx], v_bar=cols[2][idx], v_bar_x=cols[3][idx],
                                xa_plus_k=cols[4][idx], t_max=spec.t_max)
        p = list(critic.flat_params())
        m = [np.zeros_like(x) for x in p]
        v = [np.zeros_like(x) for x in p]

        def one():
            _, g = O_nets.critic_loss(critic, critic, batch, 1.0, True)
            O_nets.adam_step(p, m, v, g, 0, 1e-3)
    cores = len(os.sched_getaffinity(0))
    best, best_threads = None, 1
    for threads in sorted({1, cores}):
        with threadpoolctl.threadpool_limits(threads):
            one()  # warm-up
            for _ in range(reps):
                t0 = time.perf_counter()
                one()
                dt = time.perf_counter() - t0
                if best is None or dt < best:
                    best, best_threads = dt, threads
    return {"value": B / best, "unit": "samples/s", "cores": best_threads, "kind": kind,
            "sample": f"one critic update at B={B}, H=64, manipulator3 dims: trajrl critic_loss + adam_step + "
                      f"polyak, best of {reps} reps at 1 and {cores} BLAS threads (best: {best_threads}) "
                      f"({cpu_model()})"}


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

def measure_fp32_peak(torch, _lib, stream):
    """FFMA throughput of this B200 (the SIMT kernels' roofline, reported beside)."""
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


def ncu_traffic(kernel_prefix, workload):
    """dram bytes per launch of the kernel from the committed ncu --set full summary."""
    prof = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(prof.read_text())
        e = d.get(f"{kernel_prefix}:{workload}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def _max_over_ranks(v: float) -> float:
    """Device-side MAX over ranks (NCCL; a host tensor under the gloo test backend)."""
    import torch
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([v], device="cuda" if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reference_arm(args, spec, field, actor, critic, std, T, rank):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    # bounded per-step sample: ~64 candidates per core (~0.8 s per step on manipulator3)
    sample = min(args.cpu_sample or max(64, cores * 64), N_PER_GPU)
    cores, times, kind = run_cpu(spec, field, actor, critic, std, sample, args.steps, max(1, args.warmup))
    sec = float(np.mean(times))
    val = sample / sec
    what = ("trajrl (baseline/_ref, unmodified): nets.actor_rollout per start with the cost field, "
            "nets.mlp_forward std/critic scores, np.argsort stable select, per-start warm-start rollouts"
            if kind == "reference" else "oracle port of the reference path (baseline/_ref not importable)")
    line = {"metric": METRIC, "value": val, "unit": "states/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (same starts and networks as the GPU arm)",
            "impl": "reference",
            "config": {"workload": f"{CONFIG_NAME} rollout+BIC, {sample} candidates per step (bounded CPU "
                                   f"sample of the {N_PER_GPU}-candidate config), H={HIDDEN}, T={T}",
                       "candidates_per_step": sample, "keep_fraction": 1 / CAND_MULT},
            "cpu_baseline": {"value": val, "unit": "states/s", "cores": cores, "kind": kind,
                             "sample": f"{sample} candidates/step on a {cores}-process pool ({cpu_model()}): "
                                       + what},
            "e2e": {"value": val, "unit": "states/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cacto", choices=["cacto", "reference"])
    ap.add_argument("--n", type=int, default=0, help="candidates per GPU (0: the workload's)")
    ap.add_argument("--workload", default="manipulator3", choices=sorted(WORKLOADS))
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
        return reference_arm(args, spec, field, actor, critic, std, T, rank)

    import torch
    import torch.distributed as dist
    # CACTO_BENCH_BACKEND=gloo (tests only): the N > 1 code path on ONE GPU, every rank
    # on cuda:(local_rank % device_count), collectives through gloo
    backend = os.environ.get("CACTO_BENCH_BACKEND", "nccl")
    local_dev = local_rank % max(1, torch.cuda.device_count())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_dev))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local_dev)
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
    dsel = None
    if world > 1:
        dsel = parallel.DistributedSelect(N, keep_global, torch.float32 if args.precision == "fp32" else torch.float64)
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")  # > 126 MB L2

    def step(x0, u_out=None):
        if world == 1:
            out = pipe.run(x0, keep_global, u_out=u_out)
            return out["order"], out["U"]
        # shard-local K1+K2, the distributed exact select, and this rank's own
        # winners' warm starts (taken from its cost rollout): no states or controls
        # cross ranks, only the threshold histograms, counts and the keep winners
        out = pipe.run_sharded(x0, keep_global, base, dsel=dsel, u_out=u_out)
        return out["order"], out["U"]

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
            total = _max_over_ranks(total)
        return total / K  # ms per step

    # ---- device-resident value ----------------------------------------------------
    clocks = ClockSampler(local_dev)
    for _ in range(args.warmup):
        step(x0_dev)
    clocks.start()
    ms = timed(lambda: step(x0_dev), args.steps, 0)
    clk = clocks.stop()
    value = (N * world) / (ms * 1e-3)
    launches_per_step = pipe.kernel_launches

    # ---- e2e through the public API: pinned host -> device -> kept order + U back --
    esz = 4 if args.precision == "fp32" else 8
    order_host = torch.empty(keep_global, dtype=torch.int64).pin_memory()
    U_cap = keep_global if world == 1 else min(keep_global, N)
    U_host = torch.empty((U_cap, T, spec.m), dtype=torch.float32 if esz == 4 else torch.float64).pin_memory()
    d2h_rows = [0]

    def e2e_step():
        # the public call with HOST buffers: the rollout kernel reads the pinned x0
        # zero-copy and the take kernel writes the warm starts into pinned U_host
        # (both transfers cross PCIe inside the step, overlapped with the kernels)
        if world == 1:
            out = pipe.run(x0_pinned, keep_global, u_out=U_host)
        else:
            out = pipe.run_sharded(x0_pinned, keep_global, base, dsel=dsel, u_out=U_host)
        order_host.copy_(out["order"], non_blocking=True)
        k = out["U"].shape[0]
        if out["U"].is_cuda:
            U_host[:k].copy_(out["U"], non_blocking=True)
        d2h_rows[0] = k

    e2e_ms = timed(e2e_step, args.steps, args.warmup)
    e2e_value = (N * world) / (e2e_ms * 1e-3)
    h2d = N * spec.n * 8
    d2h = keep_global * 8 + d2h_rows[0] * T * spec.m * esz

    # ---- e2e with the candidates generated on the device (the reference's seeded
    #      sample_initial_states replayed bit-exactly, sampling.py): only the 32-byte
    #      PCG64 state goes in; the kept order + warm starts come back ------------------
    from paper_2602_19699_b200.sampling import sample_initial_states_device
    x0_seeded = torch.empty_like(x0_dev)

    def e2e_seeded_step():
        sample_initial_states_device(spec, N * world, SEED, first_row=base, rows=N, out=x0_seeded)
        order, U = step(x0_seeded, u_out=U_host)
        order_host.copy_(order, non_blocking=True)
        if U.is_cuda:
            U_host[:U.shape[0]].copy_(U, non_blocking=True)

    e2e_s_ms = timed(e2e_seeded_step, args.steps, args.warmup)
    if not torch.equal(x0_seeded, x0_dev):
        raise RuntimeError("device-sampled candidates differ from the host draw")

    # ---- roofline of the dominant kernel (the fused K1+K2 launch over all candidates) -
    for _ in range(2):
        pipe._scores(x0_dev, 0, True)
    evs = []
    for _ in range(5):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pipe._scores(x0_dev, 0, True)
        b.record()
        b.synchronize()
        evs.append(a.elapsed_time(b))
    k1_ms = float(np.mean(evs))
    f_k1 = f_cand  # rollout + the std / critic forwards fused into the same launch
    achieved = f_k1 * N / (k1_ms * 1e-3) / 1e12
    ffma_peak = measure_fp32_peak(torch, _lib, stream)
    tc_path = args.precision == "fp32" and os.environ.get("CACTO_ROLLOUT_TC", "1") != "0"
    if tc_path:
        peak, peak_source = tensor_peak()
        bound = "tensor"
        kname = ("rollout_tc_kernel: K1 rollout with cost + K2 std/critic forwards in one tcgen05 launch "
                 "(cacto_rollout_score), every candidate's controls kept for the warm starts")
    else:
        peak, bound = ffma_peak, "fp32_simt"
        peak_source = "measured FFMA throughput on this GPU (cacto_fma_peak)"
        kname = "rollout_kernel (K1 SIMT)"

    line = {
        "metric": METRIC, "value": value, "unit": "states/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (uniform workspace starts, Glorot-init networks, actor output layer x10)",
        "config": {"workload": f"{CONFIG_NAME}: {N} candidate starts/GPU -> T={T} rollout with cost, "
                               f"sigma*|V-J| score, stable top-{keep_global} select, kept warm starts (controls of "
                               f"the cost rollout)",
                   "candidates_per_gpu": N, "keep": keep_global, "hidden": [HIDDEN] * 3,
                   "horizon": T, "score": "std_x_gap", "l2": "flushed between timed steps (256 MB write)",
                   "parallelism": f"shard-by-candidate x{world}"},
        "e2e": {"value": e2e_value, "unit": "states/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "e2e_device_sampled": {"value": (N * world) / (e2e_s_ms * 1e-3), "unit": "states/s",
                               "h2d_bytes_per_step": 32, "d2h_bytes_per_step": d2h,
                               "note": "candidates = device PCG64 replay of sample_initial_states(seed) "
                                       "(bit-identical to the host draw, checked), as run_iteration uses"},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": ncu_traffic("rollout_tc_kernel", CONFIG_NAME) if tc_path else None,
                     "kernel": kname, "kernel_ms": k1_ms,
                     "flops_per_candidate": f_k1, "flops_rollout": f_roll,
                     "peak_source": peak_source,
                     "mma_passes": 3 if tc_path else None,
                     "mma_issued_tflops": 3 * achieved if tc_path else None,
                     "frac_of_3pass_ceiling": 3 * achieved / peak if tc_path else None,
                     "mma_kind": "tcgen05 kind::f16, 3xFP16 split (each fp32 product = 3 fp16 MMAs)" if tc_path
                     else None,
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
            if rank == 0 and world == 1 and not args.no_cpu:
                line["secondary"]["cpu_baseline"] = cpu_critic_baseline()
            # the config-5 grid (batch 4k-1M x hidden 64-512), device-timed, this GPU count
            grid = []
            for Hs in (64, 128, 256, 512):
                for Bs in (4096, 65536, 1 << 20):
                    r = critic_bench(torch, P, stream, B=Bs, world=world, rank=rank,
                                     dist=dist if world > 1 else None, H=Hs, K=3 if Bs >= (1 << 20) else 5)
                    grid.append({"hidden": Hs, "batch_per_gpu": Bs, "samples_per_s": r["value"],
                                 "ms_per_update": r["ms_per_update"], "tflops": r["achieved_tflops"],
                                 "frac": r["roofline"]["frac"]})
                    torch.cuda.empty_cache()
            line["secondary"]["sweep"] = grid
        except Exception as e:  # keep the primary line alive
            line["secondary"] = {"error": str(e)[:200]}

    # ---- per-iteration wall clock (north_star): the reference's
    #      run_iteration vs the installed hot path on pointmass.ini, TO on the CPU in
    #      both arms (bench_iteration.py) --------------------------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            import bench_iteration
            it = bench_iteration.measure(len(os.sched_getaffinity(0)))
            line["iteration_wallclock"] = {
                "unit": "s", "config": "pointmass.ini: 300 / 75 episodes, 750 candidates, M = 1000 cycles, B = 128",
                "reference_s": [r["wall_s"] for r in it["reference"]], "b200_s": [g["wall_s"] for g in it["b200"]],
                "reference_nets_s": [r["t_nets_s"] for r in it["reference"]],
                "b200_nets_s": [g["t_nets_s"] for g in it["b200"]],
                "to_cpu_s": [g["t_to_s"] for g in it["b200"]], "speedup_wall": it["speedup_wall"],
                "speedup_nets": it["speedup_nets"], "workers": it["workers"],
                "note": "iterations 2 and 3 (iteration 2 of the B200 arm includes engine set-up + graph capture)"}
        except Exception as e:
            line["iteration_wallclock"] = {"error": str(e)[:200]}

    # ---- CPU baseline (rank 0, N = 1 only) ---------------------------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        sample = min(args.cpu_sample or max(128, cores * 128), N)   # ~10-20 core-seconds of work
        cores, times, kind = run_cpu(spec, field, actor, critic, std, sample, 1, 1)
        line["cpu_baseline"] = {"value": sample / times[0], "unit": "states/s", "cores": cores, "kind": kind,
                                "sample": f"{sample} of the {N} candidates through the same pipeline: per-start "
                                          f"trajrl actor_rollout on a {cores}-process pool ({cpu_model()})"
                                          + ("" if kind == "reference" else " [oracle port]")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def critic_bench(torch, P, stream, B=65536, world=1, rank=0, dist=None, H=HIDDEN, K=10):
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
    if H == HIDDEN:
        actor, critic, std = make_nets(spec)
    else:
        from paper_2602_19699_b200 import nets as B_nets
        c, h = specs.normalisation(spec)
        critic = B_nets.init_mlp([spec.n + 1, H, H, H, 1], np.random.default_rng(np.random.SeedSequence([SEED, 0])),
                                 in_center=c, in_half=h)
    net = DeviceNet(critic)
    tgt = DeviceNet(critic)
    cap = 1 << 20
    buf = ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=cap)
    rows, cols, idx_all = critic_batch(spec, B, world, rank)   # the global stream, same on every rank
    buf.push_many(SampleBatch(*cols, spec.t_max))
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
            from paper_2602_19699_b200.parallel import all_reduce_sum
            all_reduce_sum(g)
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
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        one()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / K
    if world > 1:
        ms = _max_over_ranks(ms)
    d = spec.n + 1
    f = 28 * H * H + 14 * d * H + 8 * H
    peak, peak_source = tensor_peak()
    ach = f * B / (ms * 1e-3) / 1e12
    return {"metric": "critic Sobolev samples/sec", "value": B * world / (ms * 1e-3), "unit": "samples/s",
            "batch_per_gpu": B, "global_batch": B * world, "n_gpus": world, "hidden": [H] * 3,
            "ms_per_update": ms, "system": "manipulator3 (d=7)", "scaling": "weak",
            "achieved_tflops": ach, "flops_per_sample": f,
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                         "peak_source": peak_source,
                         "kernel": "the whole update (critic_tc_kernel per-sample stage on tcgen05 + reduction "
                                   "GEMMs + fold/Adam/Polyak), algorithmic F_critic = 28H^2+14dH+8H per sample"},
            "includes": "fused gather + target forward + Sobolev fwd/double-backprop + fold + "
                        + ("Adam + Polyak" if world == 1 else "NCCL all-reduce of the gradient + Adam + Polyak")}


if __name__ == "__main__":
    main()
