#!/usr/bin/env python
"""Rollout kernel alone (K1): the SIMT and tensor-core variants on the same
starts, timed with CUDA events on the launching stream, plus the fp32 result
difference between them.

  python profiles/rollout_ab.py [--system dubins] [--n 65536] [--t-hor 0] [--reps 5]
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2602_19699_b200 import _lib, specs  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets  # noqa: E402
from paper_2602_19699_b200.device import DeviceNet, set_precision  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="dubins")
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--t-hor", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    set_precision("fp32")
    spec, fld = specs.config(args.system)
    rng = np.random.default_rng(0)
    c, h = specs.normalisation(spec)
    d = spec.n + 1
    actor = B_nets.init_mlp([d, 64, 64, 64, spec.m], rng, head="tanh", out_scale=spec.u_bound, in_center=c,
                            in_half=h)
    actor = actor.with_params([q * (10.0 if i == 6 else 1.0) for i, q in enumerate(actor.flat_params())])
    dn = DeviceNet(actor)
    lo, hi = specs.region_box(spec)
    x0 = torch.as_tensor(rng.uniform(size=(args.n, spec.n)) * (hi - lo) + lo, device="cuda")
    T = args.t_hor or spec.t_max
    U = torch.empty(args.n, T, spec.m, device="cuda")
    C = torch.empty(args.n, device="cuda")
    sysd, costd = specs.system_struct(spec), specs.cost_struct(spec, fld)
    st = torch.cuda.current_stream()
    out = {}
    for mode in ("0", "1"):
        if args.only and mode != args.only:
            continue
        os.environ["CACTO_ROLLOUT_TC"] = mode
        lib = _lib.load()
        # the env switch is read once per process: re-read via a fresh variable
        def run():
            _lib.call("cacto_rollout", sysd, costd, dn.desc, x0.data_ptr(), None, 0, args.n, args.t_hor,
                      U.data_ptr(), None, None, C.data_ptr(), st.cuda_stream)
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.reps):
            run()
        b.record(st)
        b.synchronize()
        ms = a.elapsed_time(b) / args.reps
        flops = T * 2 * (d * 64 + 2 * 64 * 64 + 64 * spec.m) * args.n
        out[mode] = {"ms": ms, "tflops": flops / ms / 1e9, "cost": C.cpu().numpy().copy()}
        del lib
    line = {k: {"ms": v["ms"], "tflops": v["tflops"], "nonfinite": int((~np.isfinite(v["cost"])).sum())}
            for k, v in out.items()}
    if len(out) == 2:
        c0, c1 = out["0"]["cost"], out["1"]["cost"]
        ok = np.isfinite(c0) & np.isfinite(c1)
        err = np.abs(c0 - c1)[ok] / np.maximum(1.0, np.abs(c0[ok]))
        line["cost_rel_diff"] = {"median": float(np.median(err)), "p99": float(np.quantile(err, 0.99)),
                                 "max": float(err.max())}
    line.update(system=args.system, n=args.n, horizon=T)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
