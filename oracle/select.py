"""Oracle: BIC scoring and stable top-k selection (float64 scores, int64 order).

Restates `trainer.select_initial_states_bic` (trainer.py:141-153) and the
north_star `gap` score (no reference function -- composition of
nets.mlp_forward and nets.actor_rollout(...).cost).  Test infrastructure only.
"""

from __future__ import annotations

import numpy as np

from . import nets


def augmented(x, t=0):
    """[x, t] rows (envs/base.py:37-40)."""
    x = np.asarray(x, dtype=float)
    tcol = np.broadcast_to(np.asarray(t, dtype=float).reshape(-1, 1) if np.ndim(t) else float(t),
                           (x.shape[0], 1))
    return np.concatenate([x, tcol], axis=1)


def std_scores(std_net, xa):
    """trainer.py:150-151."""
    return nets.mlp_forward(std_net, xa)[:, 0]


def gap_scores(critic, xa, rollout_cost):
    """|V(x0) - J_rollout(x0)| (north_star; PAPER.md:141-157 variant)."""
    return np.abs(nets.mlp_forward(critic, xa)[:, 0] - np.asarray(rollout_cost, dtype=float))


def select_order(scores, keep):
    """Indices of the `keep` largest scores, descending, ties -> lower index,
    NaN last, -0.0 == +0.0; exactly np.argsort(-s, kind='stable')[:keep]
    (trainer.py:148-153)."""
    scores = np.asarray(scores)
    if keep > scores.shape[0]:
        raise ValueError(f"keep={keep} exceeds {scores.shape[0]} candidates")
    return np.argsort(-scores, kind="stable")[:keep]
