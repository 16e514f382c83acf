#!/usr/bin/env python
"""HBM-bound kernels of the hot path, timed alone against the measured copy
bandwidth (north_star: "achieved HBM GB/s for the rollout, scoring and gather
kernels").  Each launch is timed with CUDA events on the launching stream, with a
256 MB L2 flush between launches (inputs also exceed or approach the 126 MB L2).

  K4 gather   ReplayBuffer.sample_minibatch row gather (buffer.py:132-138):
              algorithmic bytes per sampled row = idx 8 B + row read + row write,
              row = (3n+m+3) values (manipulator3: 24 fp32 = 96 B).
  K4 push     ReplayBuffer.push_many FIFO append (buffer.py:108-130): 2 x row bytes.
  K3 select   stable top-keep of N scores (trainer.py:152): algorithmic bytes =
              one read of the scores + keep x (8 + 4) B written.
  K2 score    std sigma(x0) (trainer.py:150-151): one MLP forward per start; its
              bound is the FP32 pipe, reported as GFLOP/s and bytes both.

  python profiles/memkernels.py  -> one JSON line per kernel
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2602_19699_b200 import _lib, nets  # noqa: E402
from paper_2602_19699_b200.buffer import ReplayBuffer, SampleBatch  # noqa: E402
from paper_2602_19699_b200.device import device_net, set_precision  # noqa: E402
from paper_2602_19699_b200.trainer import score_device, select_topk_device  # noqa: E402


def peak_hbm():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 7700.0, "B200_PROFILING.md fallback"


def timed(fn, reps=10):
    flush = torch.empty(64 * 2 ** 20, device="cuda", dtype=torch.float32)
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ms = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def main():
    set_precision("fp32")
    peak, src = peak_hbm()
    n, m, t_max = 6, 3, 100
    W = 3 * n + m + 3
    cap = 1 << 22
    rng = np.random.default_rng(0)
    buf = ReplayBuffer(n, m, t_max, capacity=cap)
    # fill the ring on device (the contents do not matter for the byte count)
    for c in buf.cols:
        c.uniform_()
    buf._size = cap
    rows_bytes = W * 4
    for B in (65536, 1 << 20, 1 << 22):
        idx = torch.as_tensor(rng.integers(0, cap, size=B), dtype=torch.int64, device="cuda")
        ms = timed(lambda: buf.gather_device(idx))
        alg = B * (8 + 2 * rows_bytes)
        print(json.dumps({"kernel": "gather_kernel (K4)", "rows": B, "ring_rows": cap, "row_bytes": rows_bytes,
                          "ms": ms, "alg_bytes": alg, "achieved_gbs": alg / ms / 1e6, "peak_gbs": peak,
                          "frac": alg / ms / 1e6 / peak, "peak_source": src}))
    # ring push of 1M rows
    R = 1 << 20
    src_cols = [torch.rand((R,) + tuple(c.shape[1:]), device="cuda") for c in buf.cols]
    d = buf._desc(src_cols, R)
    st = torch.cuda.current_stream().cuda_stream
    ms = timed(lambda: _lib.call("cacto_ring_push", d, *[c.data_ptr() for c in buf.cols], cap, 12345, st))
    alg = R * 2 * rows_bytes
    print(json.dumps({"kernel": "ring_push_kernel (K4)", "rows": R, "ms": ms, "alg_bytes": alg,
                      "achieved_gbs": alg / ms / 1e6, "peak_gbs": peak, "frac": alg / ms / 1e6 / peak}))
    # select
    for N, keep in ((65536, 6553), (262144, 26214), (1 << 20, 104857), (1 << 22, 419430)):
        scores = torch.rand(N, device="cuda")
        ms = timed(lambda: select_topk_device(scores, keep))
        alg = N * 4 + keep * 12
        print(json.dumps({"kernel": "select_topk (K3: radix select + chunk sort + merge)", "N": N, "keep": keep,
                          "ms": ms, "alg_bytes": alg, "achieved_gbs": alg / ms / 1e6, "peak_gbs": peak,
                          "frac": alg / ms / 1e6 / peak, "candidates_per_s": N / ms * 1e3}))
    # std score (MLP forward per start)
    d_in = n + 1
    std = nets.init_mlp([d_in, 64, 64, 64, 1], np.random.default_rng(1), head="std")
    sn = device_net(std, "fp32")
    for N in (65536, 1 << 20):
        xa = torch.rand((N, d_in), device="cuda")
        ms = timed(lambda: score_device("std", xa, std_net=sn))
        flops = N * 2 * (d_in * 64 + 2 * 64 * 64 + 64)
        alg = N * (d_in * 4 + 4)
        print(json.dumps({"kernel": "score_kernel (K2, std)", "N": N, "ms": ms, "alg_bytes": alg,
                          "achieved_gbs": alg / ms / 1e6, "achieved_tflops": flops / ms / 1e9,
                          "starts_per_s": N / ms * 1e3}))


if __name__ == "__main__":
    main()
