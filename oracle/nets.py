"""Oracle: MLP forward / input gradient / Sobolev critic, actor and std losses,
Adam, Polyak and the closed-loop actor rollout (float64 NumPy).

Restates `nets.py` of the reference.  `mlp` arguments are duck-typed on the
reference `Mlp` fields (weights, biases, activation, head, out_scale,
sigma_min, in_center, in_half).  Batch arguments are duck-typed on the
reference `SampleBatch` (xa, u, v_bar, v_bar_x, xa_plus_k, t_max).
Test infrastructure only -- see `oracle/__init__.py`.
"""

from __future__ import annotations

import numpy as np

from . import envs


# -- activations: value, first and second derivative (nets.py:27-52) ---------

def _act(name):
    if name == "elu":
        return (lambda z: np.where(z > 0.0, z, np.expm1(np.minimum(z, 0.0))),
                lambda z: np.where(z > 0.0, 1.0, np.exp(np.minimum(z, 0.0))),
                lambda z: np.where(z > 0.0, 0.0, np.exp(np.minimum(z, 0.0))))
    if name == "tanh":
        return (np.tanh,
                lambda z: 1.0 - np.tanh(z) ** 2,
                lambda z: -2.0 * np.tanh(z) * (1.0 - np.tanh(z) ** 2))
    raise KeyError(name)


def _norm_in(mlp, xa):
    """nets.py:126-129."""
    if mlp.in_center is None:
        return xa
    return (xa - mlp.in_center) / mlp.in_half


def forward_caches(mlp, xa):
    """Pre-activations z_i, layer inputs a_i and raw output o; nets.py:132-141."""
    f = _act(mlp.activation)[0]
    acts = [_norm_in(mlp, xa)]
    pre = []
    nl = len(mlp.weights)
    for i in range(nl - 1):
        pre.append(acts[-1] @ mlp.weights[i].T + mlp.biases[i])
        acts.append(f(pre[-1]))
    return pre, acts, acts[-1] @ mlp.weights[nl - 1].T + mlp.biases[nl - 1]


def head_value(mlp, o):
    """nets.py:144-151."""
    if mlp.head == "linear":
        return o
    if mlp.head == "tanh":
        return mlp.out_scale * np.tanh(o)
    if mlp.head == "std":
        return mlp.sigma_min + envs.softplus(o)
    raise ValueError(f"unknown head '{mlp.head}'")


def head_chain(mlp, o):
    """Diagonal dY/dO; nets.py:154-162."""
    if mlp.head == "linear":
        return np.ones_like(o)
    if mlp.head == "tanh":
        return mlp.out_scale * (1.0 - np.tanh(o) ** 2)
    if mlp.head == "std":
        return envs.sigmoid(o)
    raise ValueError(f"unknown head '{mlp.head}'")


def mlp_forward(mlp, xa):
    """nets.py:165-173 (single (d,) or batched (B, d) input)."""
    xa = np.asarray(xa, dtype=float)
    if xa.shape[-1] != mlp.weights[0].shape[1]:
        raise ValueError(f"input dim {xa.shape[-1]} != {mlp.weights[0].shape[1]}")
    one = xa.ndim == 1
    _, _, o = forward_caches(mlp, xa[None, :] if one else xa)
    y = head_value(mlp, o)
    return y[0] if one else y


def mlp_input_gradient(mlp, xa):
    """Per-sample (out, in) Jacobian w.r.t. the raw input; nets.py:176-192."""
    xa = np.asarray(xa, dtype=float)
    one = xa.ndim == 1
    xb = xa[None, :] if one else xa
    if xb.shape[-1] != mlp.weights[0].shape[1]:
        raise ValueError("input dim mismatch")
    pre, _, o = forward_caches(mlp, xb)
    d1 = _act(mlp.activation)[1]
    jac = np.repeat(mlp.weights[-1][None], xb.shape[0], axis=0)
    for i in reversed(range(len(mlp.weights) - 1)):
        jac = (jac * d1(pre[i])[:, None, :]) @ mlp.weights[i]
    jac = jac * head_chain(mlp, o)[:, :, None]
    if mlp.in_center is not None:
        jac = jac / mlp.in_half
    return jac[0] if one else jac


def value_and_state_grad(mlp, xa):
    """(V (B,), dV/d raw input (B, in)) for a scalar linear head; nets.py:195-206."""
    xa = np.asarray(xa, dtype=float)
    pre, _, o = forward_caches(mlp, xa)
    d1 = _act(mlp.activation)[1]
    sens = np.repeat(mlp.weights[-1][0][None], xa.shape[0], axis=0)
    for i in reversed(range(len(mlp.weights) - 1)):
        sens = (d1(pre[i]) * sens) @ mlp.weights[i]
    if mlp.in_center is not None:
        sens = sens / mlp.in_half
    return o[:, 0], sens


def flat_params(mlp):
    """[W0, b0, W1, b1, ...]; nets.py:93-98."""
    out = []
    for w, b in zip(mlp.weights, mlp.biases):
        out += [w, b]
    return out


def _backprop(mlp, pre, acts, delta, grads, inject=None):
    """Value-path reverse sweep with optional injected pre-activation cotangents;
    nets.py:215-230."""
    d1 = _act(mlp.activation)[1]
    last = len(mlp.weights) - 1
    grads[2 * last] += delta.T @ acts[last]
    grads[2 * last + 1] += delta.sum(axis=0)
    up = delta @ mlp.weights[last]
    for i in reversed(range(last)):
        zbar = d1(pre[i]) * up
        if inject is not None:
            zbar = zbar + inject[i]
        grads[2 * i] += zbar.T @ acts[i]
        grads[2 * i + 1] += zbar.sum(axis=0)
        up = zbar @ mlp.weights[i]


def critic_loss(critic, critic_target, batch, k_s, gamma_bootstrap):
    """Sobolev value + state-gradient regression with exact double backprop;
    nets.py:233-290.  Returns (loss, grads in flat_params order)."""
    bsz = len(batch.xa)
    if bsz == 0:
        raise ValueError("empty batch")
    n = batch.xa.shape[1] - 1
    y = np.array(batch.v_bar, dtype=float, copy=True)
    if gamma_bootstrap and critic_target is not None:           # nets.py:247-251
        v_next = mlp_forward(critic_target, batch.xa_plus_k)[:, 0]
        y = y + np.where(batch.xa_plus_k[:, -1] < batch.t_max, v_next, 0.0)

    pre, acts, o = forward_caches(critic, batch.xa)
    _, d1, d2 = _act(critic.activation)
    last = len(critic.weights) - 1

    # sensitivities s_i = dV/d a_i, kept per layer (nets.py:258-266)
    sens = [None] * (last + 1)
    sens[last] = np.repeat(critic.weights[last][0][None], bsz, axis=0)
    for i in reversed(range(last)):
        sens[i] = (d1(pre[i]) * sens[i + 1]) @ critic.weights[i]
    half = critic.in_half if critic.in_center is not None else np.ones(critic.weights[0].shape[1])
    grad_x = sens[0] / half

    e_v = y - o[:, 0]
    e_g = batch.v_bar_x - grad_x[:, :n]
    loss = float((e_v ** 2).mean() + k_s * (e_g ** 2).sum(axis=1).mean())   # nets.py:271

    grads = [np.zeros_like(p) for p in flat_params(critic)]
    # gradient-path cotangent (nets.py:276-284)
    u = np.zeros((bsz, critic.weights[0].shape[1]))
    u[:, :n] = (-2.0 * k_s / bsz) * e_g / half[:n]
    inject = []
    for i in range(last):
        rbar = u @ critic.weights[i].T
        grads[2 * i] += (d1(pre[i]) * sens[i + 1]).T @ u
        inject.append(d2(pre[i]) * sens[i + 1] * rbar)
        u = d1(pre[i]) * rbar
    grads[2 * last] += u.sum(axis=0, keepdims=True)
    # value path plus the injected terms (nets.py:287-289)
    _backprop(critic, pre, acts, (-2.0 / bsz) * e_v[:, None], grads,
              inject if last > 0 else None)
    return loss, grads


def actor_loss(actor, critic, spec, field, xa):
    """One-step Q objective mean[l(x, mu) + V(f(x, mu), t+1)]; nets.py:293-334.

    `xa` is an (B, n+1) array of augmented states.  Returns (loss, grads, skipped).
    """
    xa = np.asarray(xa, dtype=float)
    if xa.shape[0] == 0:
        raise ValueError("empty batch")
    live = xa[:, -1] < spec.t_max
    skipped = int((~live).sum())
    xa = xa[live]
    if xa.shape[0] == 0:
        raise ValueError("all states are at the horizon")
    bsz = xa.shape[0]
    x = xa[:, :-1]
    pre, acts, o = forward_caches(actor, xa)
    u = head_value(actor, o)
    l_stage = envs.stage_cost(spec, field, x, u)
    lu = envs.stage_cost_du(spec, field, x, u)
    x_next = envs.step_x(spec, x, u)
    fu = envs.control_jacobian(spec, x, u)
    v_next, g_next = value_and_state_grad(critic, np.concatenate([x_next, xa[:, -1:] + 1.0], axis=1))
    loss = float((l_stage + v_next).mean())
    dq_du = lu + np.einsum("bnm,bn->bm", fu, g_next[:, :-1])
    grads = [np.zeros_like(p) for p in flat_params(actor)]
    _backprop(actor, pre, acts, (dq_du / bsz) * head_chain(actor, o), grads)
    return loss, grads, skipped


def std_critic_loss(std_net, critic, batch):
    """Gaussian NLL of the critic error; nets.py:337-353."""
    bsz = len(batch.xa)
    if bsz == 0:
        raise ValueError("empty batch")
    err = batch.v_bar - mlp_forward(critic, batch.xa)[:, 0]
    pre, acts, o = forward_caches(std_net, batch.xa)
    sigma = head_value(std_net, o)[:, 0]
    loss = float((np.log(sigma) + 0.5 * err ** 2 / sigma ** 2).mean())
    dl_dsigma = (1.0 / sigma - err ** 2 / sigma ** 3) / bsz
    grads = [np.zeros_like(p) for p in flat_params(std_net)]
    _backprop(std_net, pre, acts, (dl_dsigma * envs.sigmoid(o[:, 0]))[:, None], grads)
    return loss, grads


# -- optimizer (nets.py:375-398) ---------------------------------------------------

def adam_step(params, m, v, grads, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Bias-corrected Adam; `step` is the count BEFORE this update.
    Returns (params, m, v) as new lists."""
    t = step + 1
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    out_p, out_m, out_v = [], [], []
    for p, g, mm, vv in zip(params, grads, m, v):
        if p.shape != g.shape:
            raise ValueError(f"grad shape {g.shape} != param shape {p.shape}")
        mm = beta1 * mm + (1.0 - beta1) * g
        vv = beta2 * vv + (1.0 - beta2) * (g * g)
        out_p.append(p - lr * (mm / bc1) / (np.sqrt(vv / bc2) + eps))
        out_m.append(mm)
        out_v.append(vv)
    return out_p, out_m, out_v


def polyak(target_params, online_params, tau):
    return [(1.0 - tau) * pt + tau * po for pt, po in zip(target_params, online_params)]


# -- closed-loop rollout (nets.py:403-423) -------------------------------------------

def actor_rollout(actor, spec, x0, t0, t_hor, field=None):
    """Per-start rollout exactly as the reference loops it: one (d,) network
    call and one single-state step per time index.  Returns (X, U, step_costs)."""
    if t_hor > spec.t_max - t0:
        raise ValueError(f"rollout of {t_hor} steps exceeds horizon from t={t0}")
    X = np.empty((t_hor + 1, int(spec.n)))
    U = np.empty((t_hor, int(spec.m)))
    X[0] = x0
    for k in range(t_hor):
        U[k] = mlp_forward(actor, np.concatenate([X[k], [float(t0 + k)]]))
        X[k + 1] = envs.step_x(spec, X[k], U[k])
    sc = envs.trajectory_costs(spec, field, X, U) if field is not None else np.zeros(t_hor + 1)
    return X, U, sc


def actor_rollout_batch(actor, spec, x0, t0, t_hor, field=None):
    """Vectorised over starts (same arithmetic, batched BLAS calls): used by the
    tests to check large batches quickly.  x0 (N, n); t0 scalar.
    Returns X (N, T+1, n), U (N, T, m), step_costs (N, T+1), cost (N,)."""
    x0 = np.asarray(x0, dtype=float)
    N = x0.shape[0]
    X = np.empty((N, t_hor + 1, int(spec.n)))
    U = np.empty((N, t_hor, int(spec.m)))
    X[:, 0] = x0
    tcol = np.empty((N, 1))
    for k in range(t_hor):
        tcol[:] = float(t0 + k)
        U[:, k] = mlp_forward(actor, np.concatenate([X[:, k], tcol], axis=1))
        X[:, k + 1] = envs.step_x(spec, X[:, k], U[:, k])
    if field is None:
        sc = np.zeros((N, t_hor + 1))
    else:
        sc = np.empty((N, t_hor + 1))
        sc[:, :-1] = envs.stage_cost(spec, field, X[:, :-1], U)
        sc[:, -1] = envs.terminal_cost(spec, field, X[:, -1])
    return X, U, sc, sc.sum(axis=1)
