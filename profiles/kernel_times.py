"""Warm, in-stream per-kernel device times (torch.profiler / CUPTI) of one critic
update (H = 64, B = 65,536) and of one bench step -- complements the cold,
serialised ncu launch lists.

  python profiles/kernel_times.py
"""
import collections
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def table(prof, reps):
    t = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            t[e.name[:90]].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    tot = sum(sum(v) for v in t.values()) / reps
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {len(v) / reps:5.1f} x {sum(v) / len(v):9.2f} us  {sum(v) / reps / tot * 100:5.1f}%  {k}")
    print(f"  total {tot:.1f} us per rep")


def main():
    import bench
    import paper_2602_19699_b200 as P
    from paper_2602_19699_b200 import specs, trainer
    P.set_precision("fp32")
    stream = torch.cuda.current_stream().cuda_stream
    # critic update
    import numpy as np
    reps = 10
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        r = bench.critic_bench(torch, P, stream, B=65536, K=reps)
        torch.cuda.synchronize()
    print("critic update (H=64, B=65,536):", r["ms_per_update"], "ms; kernels over 3 warm-up + reps updates:")
    table(prof, reps + 3)
    # bench step (manipulator3)
    spec, fld = specs.config("manipulator3")
    actor, critic, std = bench.make_nets(spec)
    x0 = torch.as_tensor(bench.candidates(spec, 0, 262144)).cuda()
    pipe = trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
    for _ in range(3):
        pipe.run(x0, 26214)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            pipe.run(x0, 26214)
        torch.cuda.synchronize()
    print("bench step (manipulator3, 262,144):")
    table(prof, reps)


if __name__ == "__main__":
    main()
