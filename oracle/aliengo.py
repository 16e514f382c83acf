"""Oracle: synthetic AlienGO-like quadruped (nonlinear LIPM, x in R^15, u in R^6).

The reference has NO AlienGO system.  The paper gives only the
state / control layout and, in a commented appendix, the
LIPM contact-phase update.  This module defines the
synthetic high-dimensional system used for BASELINE config 4; the CUDA kernel
implements the same equations.  It is registered into the reference through its
own plug-in API (`register_system`, envs/base.py:153-157; `register_cost`,
envs/costs.py:182-187) by `tests/golden/make_golden.py`, so the reference's
`actor_rollout` / `actor_loss` machinery runs on it -- parity of the system
itself is unpinned by any reference test.

State  x = (dp_f[2], dp_r[2], c[2], cdot[2], s_idx, c_obs[2], walls[4])
Control u = (dp_f+[2], dp_r+[2], a~, d~) with CoP weight alpha = 0.5 + a~ and
contact-phase duration delta = DELTA0 + d~ (both kept in range by u_max).

Per contact phase (rotation-free, diagonal pairs alternate
through sigma = cos(pi * s_idx)); the CoP carries a capture-point feedback term
cdot/omega (a low-level balance reflex) so that open-loop / random policies keep
the state bounded over 100 phases (the bare LIPM diverges like e^{omega delta}):
    du_cop = alpha (S_f - dp_f) + (1 - alpha) (S_r - dp_r) + cdot / omega
    c+    = c + sinh(w d)/w * cdot + (1 - cosh(w d)) du_cop
    cdot+ = cosh(w d) cdot - w sinh(w d) du_cop
    dp+   = u[0:4],  s_idx+ = s_idx + 1,  c_obs, walls constant
with shoulders S_f = (SX, sigma SY), S_r = (-SX, -sigma SY).
Stage cost on the CoM (target = origin), see `stage_cost`.
"""

from __future__ import annotations

import numpy as np

NAME = "aliengo_lipm"

OMEGA = float(np.sqrt(9.81 / 0.35))   # LIPM frequency sqrt(g / z_com)
SX, SY = 0.24, 0.13                   # shoulder offsets w.r.t. the CoM [m]
DELTA0 = 0.375                        # nominal contact-phase duration
SHARP = 10.0                          # barrier slope, as costs.py:16

DEFAULTS = dict(
    n=15, m=6, dt=DELTA0, t_max=100,
    u_max=(0.15, 0.15, 0.15, 0.15, 0.5, 0.125),
    workspace=((-0.1, 0.1),) * 4 + ((-4.0, 4.0),) * 2 + ((-1.0, 1.0),) * 2
    + ((0.0, 100.0),) + ((-2.0, 2.0),) * 2
    + ((-6.0, -4.5), (4.5, 6.0), (-6.0, -4.5), (4.5, 6.0)),
    hard_region=((0.0, 0.0),) * 4 + ((2.0, 3.5), (-1.0, 1.0)) + ((0.0, 0.0),) * 2
    + ((0.0, 0.0),) + ((1.0, 1.0), (0.0, 0.0))
    + ((-5.0, -5.0), (5.0, 5.0), (-5.0, -5.0), (5.0, 5.0)),
)

# cost weights (read from CostField where the field has them)
W_VEL = 0.05          # |cdot|^2
W_VBAR = 1.0          # velocity barrier weight
V_MAX2 = 1.5 ** 2     # velocity bound squared
OBS_R2 = 0.5 ** 2     # obstacle (sphere of radius 0.5 m)
W_WALL = 5.0          # wall barrier weight


def _phase(x, u):
    a = 0.5 + u[..., 4]
    d = DELTA0 + u[..., 5]
    sig = np.cos(np.pi * x[..., 8])
    sfx, sfy = SX, sig * SY
    srx, sry = -SX, -sig * SY
    # CoP offset from the CoM: feet term + capture-point feedback cdot / omega
    ux = a * (sfx - x[..., 0]) + (1.0 - a) * (srx - x[..., 2]) + x[..., 6] / OMEGA
    uy = a * (sfy - x[..., 1]) + (1.0 - a) * (sry - x[..., 3]) + x[..., 7] / OMEGA
    ch = np.cosh(OMEGA * d)
    sh = np.sinh(OMEGA * d)
    return a, d, ux, uy, ch, sh, (sfx - x[..., 0]) - (srx - x[..., 2]), (sfy - x[..., 1]) - (sry - x[..., 3])


def step_x(spec, x, u):
    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    _, _, ux, uy, ch, sh, _, _ = _phase(x, u)
    out = np.array(x, copy=True)
    out[..., 0:4] = u[..., 0:4]
    out[..., 4] = x[..., 4] + (sh / OMEGA) * x[..., 6] + (1.0 - ch) * ux
    out[..., 5] = x[..., 5] + (sh / OMEGA) * x[..., 7] + (1.0 - ch) * uy
    out[..., 6] = ch * x[..., 6] - OMEGA * sh * ux
    out[..., 7] = ch * x[..., 7] - OMEGA * sh * uy
    out[..., 8] = x[..., 8] + 1.0
    return out


def control_jacobian(spec, x, u):
    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    _, _, ux, uy, ch, sh, gx, gy = _phase(x, u)
    fu = np.zeros(x.shape[:-1] + (15, 6))
    for i in range(4):
        fu[..., i, i] = 1.0
    # d/d a~ (alpha)
    fu[..., 4, 4] = (1.0 - ch) * gx
    fu[..., 5, 4] = (1.0 - ch) * gy
    fu[..., 6, 4] = -OMEGA * sh * gx
    fu[..., 7, 4] = -OMEGA * sh * gy
    # d/d d~ (delta)
    fu[..., 4, 5] = ch * x[..., 6] - OMEGA * sh * ux
    fu[..., 5, 5] = ch * x[..., 7] - OMEGA * sh * uy
    fu[..., 6, 5] = OMEGA * sh * x[..., 6] - OMEGA * OMEGA * ch * ux
    fu[..., 7, 5] = OMEGA * sh * x[..., 7] - OMEGA * OMEGA * ch * uy
    return fu


def _softplus(z):
    return np.logaddexp(0.0, z)


def terminal_cost(spec, field, x):
    x = np.asarray(x, dtype=float)
    cx, cy = x[..., 4], x[..., 5]
    vx, vy = x[..., 6], x[..., 7]
    q = cx * cx + cy * cy
    v2 = vx * vx + vy * vy
    val = field.distance_weight * q
    val -= field.target_reward_weight * np.exp(-q / field.target_reward_radius ** 2)
    val += W_VEL * v2
    val += W_VBAR * _softplus(SHARP * (v2 - V_MAX2))
    ox, oy = cx - x[..., 9], cy - x[..., 10]
    val += field.obstacle_weight * _softplus(SHARP * (1.0 - (ox * ox + oy * oy) / OBS_R2))
    val += W_WALL * _softplus(SHARP * (x[..., 11] - cx))
    val += W_WALL * _softplus(SHARP * (cx - x[..., 12]))
    val += W_WALL * _softplus(SHARP * (x[..., 13] - cy))
    val += W_WALL * _softplus(SHARP * (cy - x[..., 14]))
    return val


def stage_cost(spec, field, x, u):
    u = np.asarray(u, dtype=float)
    return terminal_cost(spec, field, x) + field.control_weight * (u ** 2).sum(axis=-1)


def default_field():
    """Cost weights used for config 4 (no obstacles tuple: the obstacle is in the state)."""
    from types import SimpleNamespace
    return SimpleNamespace(target=(0.0, 0.0), obstacles=(), obstacle_weight=10.0,
                           target_reward_weight=15.0, target_reward_radius=1.0,
                           control_weight=0.01, distance_weight=0.05)
