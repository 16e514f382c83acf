#!/usr/bin/env python
"""Wall clock of one CACTO-BIC iteration: reference CPU vs the B200 hot path.

North_star: "wall-clock per CACTO-BIC iteration reported against the CPU
reference".  Config: pkg/configs/pointmass.ini values (N = 300 episodes, 25 %
later batches, 10 candidates per kept start, M = 1000 update cycles, B = 128,
3x64 networks) with the TO iteration caps fixed (max_iter 20 / 10, no
calibration) and evaluation without TO refinement, so the run is bounded.  The
TO solve runs on the reference CPU solver in BOTH arms (same worker count).

Both arms start from the same state after iteration 1 (reference) and run
iterations 2 and 3; iteration 2 of the B200 arm includes the one-off engine set-up
and CUDA-graph capture, iteration 3 is steady state.  Needs the reference package
(`trajrl`): pip-installed into baseline/_ref (git-ignored) or on PYTHONPATH.

  python bench_iteration.py [--workers W] [--m-updates M]
"""

from __future__ import annotations

import argparse
import copy
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if p.exists():
        sys.path.insert(0, str(p))
        break


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--m-updates", type=int, default=1000)
    ap.add_argument("--max-iter-first", type=int, default=20)
    ap.add_argument("--max-iter-later", type=int, default=10)
    ap.add_argument("--precision", default="fp32")
    args = ap.parse_args()
    print(json.dumps(measure(args.workers, args.m_updates, args.max_iter_first, args.max_iter_later,
                             args.precision)), flush=True)


def measure(workers, m_updates=1000, max_iter_first=20, max_iter_later=10, precision="fp32"):
    """The iteration wall-clock line (also embedded by bench.py as `iteration_wallclock`)."""
    from types import SimpleNamespace
    args = SimpleNamespace(workers=workers, m_updates=m_updates, max_iter_first=max_iter_first,
                           max_iter_later=max_iter_later, precision=precision)
    import trajrl
    import trajrl.trainer as T
    import paper_2602_19699_b200 as P
    from paper_2602_19699_b200 import iteration, specs

    P.set_precision(args.precision)
    spec, fld = specs.config("pointmass")
    model = trajrl.envs.ModelSpec(**{k: getattr(spec, k) for k in ("name", "n", "m", "dt", "t_max", "u_max",
                                                                   "workspace", "hard_region", "extra")})
    field = trajrl.envs.CostField(target=fld.target, obstacles=tuple(
        trajrl.envs.Ellipse(o.center, o.semi_axes, o.angle) for o in fld.obstacles),
        obstacle_weight=fld.obstacle_weight, target_reward_weight=fld.target_reward_weight,
        target_reward_radius=fld.target_reward_radius, control_weight=fld.control_weight,
        distance_weight=fld.distance_weight)
    # pointmass.ini [trainer]/[nets]/[solver] values; iteration caps fixed (see docstring)
    cfg = T.TrainConfig(model=model, field=field, n_episodes=300, episode_fraction=0.25, candidate_multiplier=10,
                        m_updates=args.m_updates, k_lookahead=10, minibatch=128, iterations=3, seed=0, bic=True,
                        eval_count=100, eval_use_to=False, buffer_capacity=1 << 20, reg_eps=1e-6, tol=1e-6,
                        max_iter_first=args.max_iter_first, max_iter_later=args.max_iter_later,
                        workers=args.workers)
    state = T.TrainerState(cfg)
    t = time.perf_counter()
    state, rep1 = T.run_iteration(state, 1)
    it1 = time.perf_counter() - t

    def arm(run):
        st = copy.deepcopy(state)
        out = []
        for j in (2, 3):
            t0 = time.perf_counter()
            st, rep = run(st, j)
            out.append({"iteration": j, "wall_s": time.perf_counter() - t0, "t_to_s": rep.t_to_s,
                        "t_nets_s": rep.t_nets_s, "critic_loss_mean": rep.critic_loss_mean,
                        "std_loss_mean": rep.std_loss_mean, "eval_mean_cost": rep.eval_mean_cost,
                        "episodes_cum": rep.episodes_cum})
        return out

    ref = arm(T.run_iteration)
    gpu = arm(lambda st, j: iteration.run_iteration(st, j, trajrl))
    line = {"metric": "CACTO-BIC iteration wall clock (pointmass.ini, TO on CPU in both arms)",
            "unit": "s", "workers": args.workers, "cpu_cores": len(os.sched_getaffinity(0)),
            "iteration1_reference_s": it1, "reference": ref, "b200": gpu,
            "speedup_wall": [r["wall_s"] / g["wall_s"] for r, g in zip(ref, gpu)],
            "speedup_nets": [r["t_nets_s"] / g["t_nets_s"] for r, g in zip(ref, gpu)],
            "precision": args.precision,
            "config": {"n_episodes": 300, "later_batch": 75, "candidates": 750, "m_updates": args.m_updates,
                       "minibatch": 128, "hidden": [64, 64, 64], "max_iter": [args.max_iter_first,
                                                                           args.max_iter_later],
                       "eval_use_to": False}}
    return line


if __name__ == "__main__":
    main()
