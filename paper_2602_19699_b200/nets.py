"""Drop-in replacements for the hot functions of `trajrl.nets` on the B200.

Same names, argument order, return types and exceptions as the reference
(`nets.py` line ranges cited per function); every computation runs in the
sm_100a kernels of libcacto_b200 -- there is no CPU fallback.  Inputs/outputs
are float64 NumPy like the reference; the arithmetic precision is the package
precision (`set_precision`, default fp32; fp64 reproduces the reference to
~1e-12).  Batched / device-resident entry points (`actor_rollout_batch`,
`engine.*`) avoid the per-call host round trips.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field as dc_field, replace
from typing import Optional

import numpy as np
import torch

from . import _lib, specs
from .device import (DeviceNet, abi_dtype, device, device_net, get_precision, to_device,
                     torch_dtype)


# ---- containers (mirrors of the reference types) -------------------------------------

@dataclass(frozen=True)
class Mlp:
    """nets.py:63-103."""

    weights: tuple
    biases: tuple
    activation: str = "elu"
    head: str = "linear"
    out_scale: Optional[np.ndarray] = None
    sigma_min: float = 1e-3
    in_center: Optional[np.ndarray] = None
    in_half: Optional[np.ndarray] = None

    @property
    def in_dim(self) -> int:
        return self.weights[0].shape[1]

    @property
    def out_dim(self) -> int:
        return self.weights[-1].shape[0]

    @property
    def layer_sizes(self) -> list:
        return [self.in_dim] + [w.shape[0] for w in self.weights]

    def flat_params(self) -> list:
        out = []
        for w, b in zip(self.weights, self.biases):
            out += [w, b]
        return out

    def with_params(self, params) -> "Mlp":
        L = len(self.weights)
        return replace(self, weights=tuple(params[2 * i] for i in range(L)),
                       biases=tuple(params[2 * i + 1] for i in range(L)))


def init_mlp(sizes, rng, activation="elu", head="linear", out_scale=None, sigma_min=1e-3,
             in_center=None, in_half=None) -> Mlp:
    """Glorot normal, output layer x0.1, zero biases (nets.py:106-123); host-side
    parameter setup drawing from the same NumPy stream as the reference."""
    ws, bs = [], []
    for i in range(len(sizes) - 1):
        fan_in, fan_out = sizes[i], sizes[i + 1]
        scale = math.sqrt(2.0 / (fan_in + fan_out))
        if i == len(sizes) - 2:
            scale *= 0.1
        ws.append(rng.normal(0.0, scale, size=(fan_out, fan_in)))
        bs.append(np.zeros(fan_out))
    arr = lambda v: None if v is None else np.asarray(v, float)  # noqa: E731
    return Mlp(tuple(ws), tuple(bs), activation, head, arr(out_scale), sigma_min, arr(in_center), arr(in_half))


@dataclass
class Trajectory:
    """ilqr.py:59-81."""

    X: np.ndarray
    U: np.ndarray
    step_costs: np.ndarray
    t0: int = 0

    @property
    def horizon(self) -> int:
        return self.U.shape[0]

    @property
    def cost(self) -> float:
        return float(self.step_costs.sum())

    def state_at(self, k: int) -> specs.TimeState:
        return specs.TimeState(self.X[k], self.t0 + k)


@dataclass(frozen=True)
class AdamState:
    """nets.py:358-372 (moments kept host-side as NumPy for API parity)."""

    m: tuple
    v: tuple
    step: int = 0
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps_adam: float = 1e-8

    @classmethod
    def init(cls, params, lr=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8):
        return cls(m=tuple(np.zeros_like(p) for p in params), v=tuple(np.zeros_like(p) for p in params),
                   step=0, lr=lr, beta1=beta1, beta2=beta2, eps_adam=eps_adam)


def _stream():
    return torch.cuda.current_stream().cuda_stream


# ---- forward / input gradient ------------------------------------------------------

def mlp_forward(mlp, xa) -> np.ndarray:
    """nets.py:165-173."""
    xa = np.asarray(xa, dtype=float)
    single = xa.ndim == 1
    if xa.shape[-1] != mlp.weights[0].shape[1]:
        raise ValueError(f"input dim {xa.shape[-1]} != {mlp.weights[0].shape[1]}")
    xb = xa[None, :] if single else xa
    y = mlp_forward_device(device_net(mlp), to_device(xb))
    out = y.to("cpu", torch.float64).numpy()
    return out[0] if single else out


def mlp_forward_device(net: DeviceNet, xa: torch.Tensor) -> torch.Tensor:
    """Device fast path: xa [B, in] tensor in the net's precision -> [B, out]."""
    B = xa.shape[0]
    y = torch.empty((B, net.sizes[-1]), device=xa.device, dtype=xa.dtype)
    _lib.call("cacto_mlp_forward", net.desc, xa.data_ptr(), B, y.data_ptr(), _stream())
    return y


def _jacobian(mlp, xb):
    net = device_net(mlp)
    x = to_device(xb)
    B = x.shape[0]
    val = torch.empty((B, net.sizes[-1]), device=x.device, dtype=x.dtype)
    jac = torch.empty((B, net.sizes[-1], net.sizes[0]), device=x.device, dtype=x.dtype)
    _lib.call("cacto_mlp_jacobian", net.desc, x.data_ptr(), B, val.data_ptr(), jac.data_ptr(), _stream())
    return val.to("cpu", torch.float64).numpy(), jac.to("cpu", torch.float64).numpy()


def mlp_input_gradient(mlp, xa) -> np.ndarray:
    """nets.py:176-192."""
    xa = np.asarray(xa, dtype=float)
    single = xa.ndim == 1
    xb = xa[None, :] if single else xa
    if xb.shape[-1] != mlp.weights[0].shape[1]:
        raise ValueError(f"input dim {xb.shape[-1]} != {mlp.weights[0].shape[1]}")
    _, jac = _jacobian(mlp, xb)
    return jac[0] if single else jac


def value_and_state_grad(mlp, xa):
    """nets.py:195-206."""
    assert mlp.head == "linear" and mlp.weights[-1].shape[0] == 1
    val, jac = _jacobian(mlp, np.asarray(xa, dtype=float))
    return val[:, 0], jac[:, 0, :]


# ---- losses ----------------------------------------------------------------------------

class _Batch:
    """Device copy of a SampleBatch (buffer.py:39-55) + its cacto_batch_t."""

    def __init__(self, batch=None, xa=None, n=None, m=None, t_max=None, denom=0):
        dev = device()
        if batch is not None:
            xa = batch.xa
            self.cols = [to_device(batch.xa), to_device(batch.u), to_device(batch.v_bar),
                         to_device(batch.v_bar_x), to_device(batch.xa_plus_k)]
            n = batch.xa.shape[1] - 1
            m = batch.u.shape[1]
            t_max = batch.t_max
        else:
            B = xa.shape[0]
            z = torch.zeros(1, device=dev, dtype=torch_dtype())
            self.cols = [to_device(xa), z, z, z, z]
        self.desc = _lib.CactoBatch()
        self.desc.dtype = abi_dtype()
        self.desc.n, self.desc.m, self.desc.t_max = int(n), int(m), int(t_max)
        self.desc.rows = int(xa.shape[0])
        self.desc.denom = int(denom)
        self.desc.idx = None
        self.desc.xa, self.desc.u, self.desc.v_bar, self.desc.v_bar_x, self.desc.xa_plus_k = \
            [c.data_ptr() for c in self.cols]


def _run_loss(net: DeviceNet, launch, also=()):
    """Allocate the workspace, run the loss launcher, fold the partials.  `also`:
    nets evaluated inside the loss whose workspace is added (the critic of the
    actor loss, include/cacto_b200.h)."""
    dev = device()
    rows = launch.rows
    L = _lib.load()
    nbytes = L.cacto_loss_workspace_bytes(net.desc, rows) + sum(L.cacto_loss_workspace_bytes(n.desc, rows)
                                                                 for n in also)
    ws = torch.empty(nbytes, device=dev, dtype=torch.uint8)
    import ctypes
    npart = ctypes.c_int32(0)
    launch(ws, nbytes, npart)
    grad = torch.empty(net.count, device=dev, dtype=torch_dtype(net.precision))
    loss = torch.empty(1, device=dev, dtype=torch_dtype(net.precision))
    _lib.call("cacto_reduce_grads", net.desc.dtype, ws.data_ptr(), npart.value, net.count,
              grad.data_ptr(), loss.data_ptr(), _stream())
    return float(loss.item()), net.unpack(grad)


def critic_loss(critic, critic_target, batch, k_s: float, gamma_bootstrap: bool):
    """nets.py:233-290."""
    if len(batch.xa) == 0:
        raise ValueError("empty batch")
    net = device_net(critic)
    tgt = device_net(critic_target) if (gamma_bootstrap and critic_target is not None) else None
    b = _Batch(batch)

    def launch(ws, nbytes, npart):
        _lib.call("cacto_critic_loss", net.desc, tgt.desc if tgt else None, b.desc, float(k_s),
                  int(bool(gamma_bootstrap and tgt is not None)), ws.data_ptr(), nbytes, npart, _stream())
    launch.rows = b.desc.rows
    return _run_loss(net, launch)


def std_critic_loss(std_net, critic, batch):
    """nets.py:337-353."""
    if len(batch.xa) == 0:
        raise ValueError("empty batch")
    net = device_net(std_net)
    cn = device_net(critic)
    b = _Batch(batch)

    def launch(ws, nbytes, npart):
        _lib.call("cacto_std_loss", net.desc, cn.desc, b.desc, ws.data_ptr(), nbytes, npart, _stream())
    launch.rows = b.desc.rows
    return _run_loss(net, launch)


def actor_loss(actor, critic, model, field, states):
    """nets.py:293-334: returns (loss, grads, skipped)."""
    if hasattr(states, "xa") and not isinstance(states, (list, tuple)):
        xa = np.asarray(states.xa, dtype=float)
    else:
        states = list(states)
        if not states:
            raise ValueError("empty batch")
        xa = np.stack([s.augmented for s in states])
    if xa.shape[0] == 0:
        raise ValueError("empty batch")
    live = int((xa[:, -1] < model.t_max).sum())
    skipped = xa.shape[0] - live
    if live == 0:
        raise ValueError("all states are at the horizon")
    net = device_net(actor)
    cn = device_net(critic)
    sysd = specs.system_struct(model)
    costd = specs.cost_struct(model, field)
    b = _Batch(xa=xa, n=model.n, m=model.m, t_max=model.t_max)
    live_t = torch.tensor([live], device=device(), dtype=torch.int64)

    def launch(ws, nbytes, npart):
        _lib.call("cacto_actor_loss", net.desc, cn.desc, sysd, costd, b.desc, live_t.data_ptr(),
                  ws.data_ptr(), nbytes, npart, _stream())
    launch.rows = b.desc.rows
    loss, grads = _run_loss(net, launch, also=(cn,))
    return loss, grads, skipped


# ---- optimizer --------------------------------------------------------------------------

def adam_step(params, state: AdamState, grads):
    """nets.py:375-392 (fused device update; bit-identical to NumPy in fp64)."""
    if len(params) != len(grads):
        raise ValueError("params/grads length mismatch")
    for p, g in zip(params, grads):
        if np.shape(p) != np.shape(g):
            raise ValueError(f"grad shape {np.shape(g)} != param shape {np.shape(p)}")
    shapes = [np.shape(p) for p in params]
    cat = lambda xs: to_device(np.concatenate([np.asarray(x, float).reshape(-1) for x in xs]))  # noqa: E731
    p, m, v, g = cat(params), cat(state.m), cat(state.v), cat(grads)
    P = p.numel()
    _lib.call("cacto_adam_step", abi_dtype(), p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), P,
              int(state.step), float(state.lr), float(state.beta1), float(state.beta2),
              float(state.eps_adam), _stream())

    def split(t):
        a = t.to("cpu", torch.float64).numpy()
        out, off = [], 0
        for s in shapes:
            k = int(np.prod(s)) if len(s) else 1
            out.append(a[off:off + k].reshape(s))
            off += k
        return out
    return split(p), replace(state, m=tuple(split(m)), v=tuple(split(v)), step=state.step + 1)


def polyak(target, online, tau: float):
    """nets.py:395-398."""
    tp = target.flat_params()
    shapes = [np.shape(x) for x in tp]
    cat = lambda xs: to_device(np.concatenate([np.asarray(x, float).reshape(-1) for x in xs]))  # noqa: E731
    t, o = cat(tp), cat(online.flat_params())
    _lib.call("cacto_polyak", abi_dtype(), t.data_ptr(), o.data_ptr(), t.numel(), float(tau), _stream())
    a = t.to("cpu", torch.float64).numpy()
    out, off = [], 0
    for s in shapes:
        k = int(np.prod(s))
        out.append(a[off:off + k].reshape(s))
        off += k
    return target.with_params(out)


# ---- rollouts ----------------------------------------------------------------------------

def actor_rollout_batch(actor, model, x0, t0=0, t_hor: Optional[int] = None, field=None,
                        emit=("U", "X", "step_costs", "cost"), as_numpy=True):
    """Batched closed-loop rollouts (nets.py:403-423 for N starts at once).

    x0 (N, n) starts; t0 scalar or (N,) start times; t_hor None -> every start
    runs to the horizon (t_max - t0_i, the warm-start / eval call sites
    trainer.py:192-193, 267-268).  Returns a dict with the requested outputs
    (`U` (N, T, m), `X` (N, T+1, n), `step_costs` (N, T+1), `cost` (N,)), rows
    beyond a start's horizon being NaN.
    """
    dev = device()
    x0 = np.asarray(x0, dtype=float)
    N = x0.shape[0]
    t0a = np.broadcast_to(np.asarray(t0, dtype=np.int64), (N,))
    if t_hor is not None:
        if N and t_hor > model.t_max - int(t0a.max()):
            raise ValueError(f"rollout of {t_hor} steps exceeds horizon from t={int(t0a.max())}")
        T = int(t_hor)
    else:
        T = int(model.t_max - (t0a.min() if N else 0))
    net = device_net(actor)
    sysd = specs.system_struct(model)
    costd = specs.cost_struct(model, field) if field is not None else None
    dt = torch_dtype(net.precision)
    stride = T if t_hor is not None else model.t_max
    out = {}
    if "U" in emit:
        out["U"] = torch.full((N, stride, model.m), float("nan"), device=dev, dtype=dt)
    if "X" in emit:
        out["X"] = torch.full((N, stride + 1, model.n), float("nan"), device=dev, dtype=dt)
    if "step_costs" in emit:
        out["step_costs"] = torch.full((N, stride + 1), float("nan"), device=dev, dtype=dt)
    if "cost" in emit:
        out["cost"] = torch.empty((N,), device=dev, dtype=dt)
    x0d = torch.as_tensor(x0).to(dev)
    uniform = bool(N == 0 or (t0a == t0a[0]).all())
    t0d = None if uniform else torch.as_tensor(t0a.astype(np.int32)).to(dev)
    t0s = int(t0a[0]) if N else 0
    _lib.call("cacto_rollout", sysd, costd, net.desc, x0d.data_ptr(),
              t0d.data_ptr() if t0d is not None else None, t0s, N, T if t_hor is not None else _lib.FULL_HORIZON,
              *(out[k].data_ptr() if k in out else None for k in ("U", "X", "step_costs", "cost")),
              _stream())
    if as_numpy:
        out = {k: v.to("cpu", torch.float64).numpy() for k, v in out.items()}
    return out


def actor_rollout(actor, model, x0, t_hor: int, field=None) -> Trajectory:
    """nets.py:403-423 (one start; same checks and outputs)."""
    if t_hor > model.t_max - x0.t:
        raise ValueError(f"rollout of {t_hor} steps exceeds horizon from t={x0.t}")
    r = actor_rollout_batch(actor, model, np.asarray(x0.x, dtype=float)[None, :], x0.t, t_hor, field,
                            emit=("U", "X", "step_costs"))
    sc = r["step_costs"][0] if field is not None else np.zeros(t_hor + 1)
    return Trajectory(X=r["X"][0], U=r["U"][0], step_costs=sc, t0=x0.t)


# ---- checkpoints (nets.py:428-464; interchange format, host I/O) ---------------------------

def save_checkpoint(path, mlp, kind: str, model_name: str, config_hash: str):
    doc = {"kind": kind, "model": model_name, "layer_sizes": [int(mlp.weights[0].shape[1])] +
           [int(w.shape[0]) for w in mlp.weights], "activation": mlp.activation, "head": mlp.head,
           "out_scale": None if mlp.out_scale is None else np.asarray(mlp.out_scale).tolist(),
           "sigma_min": mlp.sigma_min,
           "norm_center": None if mlp.in_center is None else np.asarray(mlp.in_center).tolist(),
           "norm_half": None if mlp.in_half is None else np.asarray(mlp.in_half).tolist(),
           "weights": [np.asarray(w).reshape(-1).tolist() for w in mlp.weights],
           "biases": [np.asarray(b).tolist() for b in mlp.biases], "config_hash": config_hash}
    with open(path, "w") as fh:
        json.dump(doc, fh)


def load_checkpoint(path):
    with open(path) as fh:
        doc = json.load(fh)
    sizes = doc["layer_sizes"]
    arr = lambda v: None if v is None else np.asarray(v, float)  # noqa: E731
    mlp = Mlp(weights=tuple(np.asarray(doc["weights"][i], float).reshape(sizes[i + 1], sizes[i])
                            for i in range(len(sizes) - 1)),
              biases=tuple(np.asarray(b, float) for b in doc["biases"]), activation=doc["activation"],
              head=doc["head"], out_scale=arr(doc["out_scale"]), sigma_min=doc["sigma_min"],
              in_center=arr(doc["norm_center"]), in_half=arr(doc["norm_half"]))
    return mlp, {k: doc[k] for k in ("kind", "model", "config_hash")}
