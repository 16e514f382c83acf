#!/usr/bin/env python
"""Where the non-K1 time of one dubins BIC step goes: CUDA events between the
pipeline's stages (rollout+score, select, take_columns) on the launching stream,
and the host time to enqueue one step.  python profiles/step_timeline.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2602_19699_b200 import _lib, specs, trainer  # noqa: E402
from paper_2602_19699_b200.device import set_precision  # noqa: E402


def main():
    set_precision("fp32")
    bench.CONFIG_NAME = "dubins"
    spec, field = specs.config(bench.CONFIG_NAME)
    actor, critic, std = bench.make_nets(spec)
    N = 65536
    keep = N // 10
    x0 = torch.from_numpy(bench.candidates(spec, 0, N)).cuda()
    pipe = trainer.BicPipeline(spec, field, actor, critic, std, mode="std_x_gap", precision="fp32")
    flush = torch.empty(64 * 2 ** 20, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    res = []
    for it in range(13):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        ev[0].record()
        scores, cost = pipe._fused(x0, 0, True)
        ev[1].record()
        order, top = trainer.select_topk_device(scores, keep, 0, pipe.ws)
        ev[2].record()
        U = torch.empty((keep, spec.t_max, spec.m), device="cuda")
        _lib.call("cacto_take_columns", _lib.F32, pipe.u_all.data_ptr(), spec.t_max * spec.m, N, order.data_ptr(),
                  keep, U.data_ptr(), torch.cuda.current_stream().cuda_stream)
        ev[3].record()
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        if it >= 3:
            res.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                        ev[0].elapsed_time(ev[3]), (h1 - h0) * 1e3])
    m = np.median(np.array(res), axis=0)
    print(json.dumps({"rollout_score_ms": m[0], "select_ms": m[1], "take_ms": m[2], "step_ms": m[3],
                      "host_enqueue_ms": m[4]}))
    # whole pipe.run as bench times it
    t = []
    for it in range(13):
        flush.fill_(1.0)
        ev[0].record()
        pipe.run(x0, keep)
        ev[1].record()
        torch.cuda.synchronize()
        if it >= 3:
            t.append(ev[0].elapsed_time(ev[1]))
    print(json.dumps({"pipe_run_ms": float(np.median(t))}))


if __name__ == "__main__":
    main()
