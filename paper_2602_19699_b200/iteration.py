"""One CACTO-BIC iteration with the hot path on the B200 (reference
`trajrl.trainer.run_iteration`, trainer.py:168-255).

Same control flow and the same random streams as the reference; the TO solve
(`solve_batch`) and the reports stay on the reference's CPU code, while
  * k-step targets + replay push (the producer)    -> cacto_kstep_push (200-201)
  * BIC candidate scoring + stable selection      -> K2/K3 (trainer.py:183-186)
  * warm-start actor rollouts of the kept starts   -> K1, one batched launch (192-193)
  * the M critic/actor + M std update cycles       -> UpdateEngine graphs (208-234)
  * the evaluation rollouts                        -> K1, one batched launch (267-268)
run on the GPU.  The reference `TrainerState` stays the source of truth for the
host side: after the update loop its networks and Adam states are refreshed from
the device.  Requires the reference package (`trajrl`) to be importable.
"""

from __future__ import annotations

import time
from dataclasses import replace

import numpy as np
import torch

from . import nets as B_nets
from . import trainer as B_trainer
from .buffer import ReplayBuffer
from .device import get_precision
from .engine import UpdateEngine


def _host_buffer_to_device(hb, precision):
    """Mirror a reference ReplayBuffer (buffer.py:85-106) into a device ring."""
    db = ReplayBuffer(hb.n, hb.m, hb.t_max, capacity=hb.capacity, model_name=hb.model_name,
                      k_lookahead=hb.k_lookahead, precision=precision)
    if len(hb):
        cols = (hb._xa, hb._u, hb._v, hb._vx, hb._xk)
        for dst, src in zip(db.cols, cols):
            dst.copy_(torch.as_tensor(src).to(dst.device, dst.dtype))
        db._size, db._cursor = hb._size, hb._cursor
    return db


def _engine(state):
    eng = getattr(state, "_cacto_engine", None)
    if eng is None:
        cfg = state.config
        dbuf = _host_buffer_to_device(state.buffer, get_precision())
        eng = UpdateEngine(cfg.model, cfg.field, state.actor, state.critic, state.critic_target, state.std, dbuf,
                           minibatch=cfg.minibatch, k_s=cfg.k_s, bootstrap=cfg.bootstrap, tau=cfg.tau,
                           lr_actor=cfg.lr_actor, lr_critic=cfg.lr_critic, lr_std=cfg.lr_std,
                           adam_states=(state.adam_actor, state.adam_critic, state.adam_std))
        state._cacto_engine = eng
        state.buffer = dbuf  # same API as the reference ring (push_many / sample_minibatch / dump)
    return eng


def _sync_state(state, eng):
    """Refresh the reference-side networks and Adam states from the device."""
    actor, critic, target, std = eng.networks()
    state.actor, state.critic, state.critic_target, state.std = actor, critic, target, std
    for name, net in (("adam_actor", eng.actor), ("adam_critic", eng.critic), ("adam_std", eng.std)):
        m, v, step = eng.adam_host(net)
        setattr(state, name, replace(getattr(state, name), m=tuple(m), v=tuple(v), step=step))


def warm_starts(actor, model, starts):
    """`[actor_rollout(actor, model, s, t_max - s.t).U for s in starts]` in one launch."""
    x0 = np.stack([s.x for s in starts])
    t0 = np.array([s.t for s in starts])
    U = B_nets.actor_rollout_batch(actor, model, x0, t0, None, None, emit=("U",))["U"]
    return [U[i, :model.t_max - s.t] for i, s in enumerate(starts)]


def run_iteration(state, iter_idx: int, trajrl):
    """Drop-in for trajrl.trainer.run_iteration (trainer.py:168-255)."""
    T = trajrl.trainer
    cfg = state.config
    model, fld = cfg.model, cfg.field
    eng = _engine(state)

    t0 = time.perf_counter()
    if iter_idx == 1:
        starts = T.sample_initial_states(model, cfg.n_episodes, T._seed_int(cfg.seed, 1, iter_idx),
                                         T.Region.WORKSPACE)
        starts = T._assign_start_times(starts, model, cfg, iter_idx)
        warms = [T._naive_warmstart(model, s) for s in starts]
        max_iter = state.max_iter_first
    else:
        n_sel = cfg.later_batch
        if cfg.bic:
            # candidates generated on the device (bit-exact PCG64 replay of
            # sample_initial_states, envs/__init__.py:112-122), scored and selected
            # there; only the kept starts come back (trainer.py:183-186)
            kept, _ = B_trainer.sample_select_bic(model, cfg.candidate_multiplier * n_sel,
                                                  T._seed_int(cfg.seed, 1, iter_idx), state.std, n_sel,
                                                  T.Region.WORKSPACE)
            starts = [T.TimeState(x=row, t=0) for row in kept]
        else:
            starts = T.sample_initial_states(model, n_sel, T._seed_int(cfg.seed, 1, iter_idx), T.Region.WORKSPACE)
        starts = T._assign_start_times(starts, model, cfg, iter_idx)
        warms = warm_starts(state.actor, model, starts)
        max_iter = state.max_iter_later
    if max_iter is None:
        raise RuntimeError("iteration cap not resolved; run via train()")

    results = T.solve_batch(model, fld, starts, warms, max_iter, state.reg, cfg.tol, cfg.workers)
    # replay producer on the device: k-step targets of every solution + FIFO push,
    # one H2D copy and one launch (trainer.py:200-201); state.buffer is the device ring
    eng.buffer.push_kstep(results, cfg.k_lookahead)
    state.episodes_cum += len(results)
    costs = np.array([r.cost for r in results])
    conv = float(np.mean([r.converged for r in results]))
    t_to = time.perf_counter() - t0

    t1 = time.perf_counter()
    critic_losses, std_losses = eng.run(cfg.m_updates, state.rng_batches)
    _sync_state(state, eng)
    torch.cuda.synchronize()
    t_nets = time.perf_counter() - t1

    t2 = time.perf_counter()
    x0 = np.stack([s.x for s in state.eval_starts])
    t0s = np.array([s.t for s in state.eval_starts])
    roll = B_nets.actor_rollout_batch(state.actor, model, x0, t0s, None, fld, emit=("U", "cost"))
    if cfg.eval_use_to:
        Us = [roll["U"][i, :model.t_max - s.t] for i, s in enumerate(state.eval_starts)]
        res = T.solve_batch(model, fld, state.eval_starts, Us, cfg.eval_max_iter, state.reg, cfg.tol, cfg.workers)
        eval_mean = float(np.array([r.cost for r in res]).mean())
    else:
        eval_mean = float(roll["cost"].mean())
    t_to += time.perf_counter() - t2

    report = T.IterationReport(
        iteration=iter_idx, episodes_cum=state.episodes_cum, to_cost_mean=float(costs.mean()),
        to_cost_median=float(np.median(costs)), converged_frac=conv,
        critic_loss_mean=float(critic_losses.mean()), std_loss_mean=float(std_losses.mean()),
        eval_mean_cost=eval_mean, t_to_s=t_to, t_nets_s=t_nets)
    return state, report
