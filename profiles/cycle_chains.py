#!/usr/bin/env python
"""Per-chain time of the B = 128 update cycle (pointmass shapes): CUDA graphs of 16
critic-chain cycles alone (critic loss -> Adam/Polyak -> ring copy) and of 16
actor-chain cycles alone (actor loss on the ring's critic -> Adam), replayed and timed
with CUDA events -- which chain bounds the pipelined loop (engine.py _run_pipelined)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import engine_cycle  # noqa: E402


def main():
    eng = engine_cycle.build_engine()
    eng.run(1024, np.random.default_rng(1))  # index lists for 1024 cycles
    torch.cuda.synchronize()
    out = {}
    for name, fn in (("critic_chain", eng._cycle_critic), ("actor_chain", eng._cycle_actor)):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(16):
                fn()
        eng.cnt.zero_()  # <= 3 * 16 + 20 * 16 cycles of the 1024 drawn lists
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        b.synchronize()
        out[name + "_us_per_cycle"] = round(a.elapsed_time(b) * 1e3 / (20 * 16), 2)
    print(out)


if __name__ == "__main__":
    main()
