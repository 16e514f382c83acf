#!/usr/bin/env python
"""Per-stage latencies of K1's tile chain from the clock64 timeline variant
(CACTO_RTC_TIMELINE=1 build: variants/libtl.so; run with CACTO_B200_LIB pointing
at it).  CTA 10, passes 20..27, each tile's leader warp: epilogue end -> tile
joined (siblings' epilogues) -> MMAs issued -> MMA completion seen -> next
epilogue end.  Layers: 0 input, 1..2 hidden, 3 output."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_19699_b200 import _lib, specs as B_specs, trainer as B_trainer  # noqa: E402
from paper_2602_19699_b200.device import set_precision  # noqa: E402
from bench import make_nets, candidates, WORKLOADS  # noqa: E402


def main(name="manipulator3"):
    set_precision("fp32")
    N = WORKLOADS[name]
    spec, fld = B_specs.config(name)
    actor, critic, std = make_nets(spec)
    pipe = B_trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
    x0 = torch.as_tensor(candidates(spec, 0, N)).cuda()
    for _ in range(2):
        pipe._scores(x0, 0, True)
    torch.cuda.synchronize()
    lib = _lib.load()
    buf = (ctypes.c_ulonglong * (4 * 8 * 4 * 4))()
    assert lib.cacto_debug_rtc_timeline(buf) == 0
    t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(4, 8, 4, 4)
    names = ["input", "hidden1", "hidden2", "output"]
    out = {}
    for L in range(4):
        join = t[:, :, L, 1] - t[:, :, L, 0]
        issue = t[:, :, L, 2] - t[:, :, L, 1]
        mma = t[:, :, L, 3] - t[:, :, L, 2]
        out[names[L]] = dict(join=float(np.median(join)), issue=float(np.median(issue)), mma_wait=float(np.median(mma)))
    # epilogue after layer L's MMAs: MMA seen (L, 3) -> next handoff's epilogue end
    epi = {}
    for L in range(3):
        epi[names[L]] = float(np.median(t[:, :, L + 1, 0] - t[:, :, L, 3]))
    epi["output(+dynamics)"] = float(np.median(t[:, 1:, 0, 0] - t[:, :-1, 3, 3]))
    step = float(np.median(t[:, 1:, 0, 0] - t[:, :-1, 0, 0]))
    print({"workload": name, "cycles_per_step": step, "per_layer": out, "epilogue_after": epi})


if __name__ == "__main__":
    main(*(sys.argv[1:] or []))
