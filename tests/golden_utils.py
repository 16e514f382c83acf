"""Load the committed golden fixtures (tests/golden/*.npz) into plain objects.

The fixtures were produced by the real reference (tests/golden/make_golden.py);
nothing here imports the reference, so these helpers work on the GPU box.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field as dc_field
from pathlib import Path
from types import SimpleNamespace
from typing import Optional

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
_CACHE: dict = {}


def load(name: str):
    if name not in _CACHE:
        _CACHE[name] = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
    return _CACHE[name]


@dataclass(frozen=True)
class Ellipse:
    center: tuple
    semi_axes: tuple
    angle: float = 0.0


@dataclass(frozen=True)
class Field:
    target: tuple = (-7.0, 0.0)
    obstacles: tuple = ()
    obstacle_weight: float = 0.0
    target_reward_weight: float = 0.0
    target_reward_radius: float = 1.0
    control_weight: float = 0.0
    distance_weight: float = 1.0


@dataclass(frozen=True)
class Spec:
    name: str
    n: int
    m: int
    dt: float
    t_max: int
    u_max: tuple
    workspace: tuple
    hard_region: tuple
    extra: tuple = dc_field(default=())


@dataclass(frozen=True, eq=False)
class Net:
    weights: tuple
    biases: tuple
    activation: str = "elu"
    head: str = "linear"
    out_scale: Optional[np.ndarray] = None
    sigma_min: float = 1e-3
    in_center: Optional[np.ndarray] = None
    in_half: Optional[np.ndarray] = None

    def flat_params(self):
        out = []
        for w, b in zip(self.weights, self.biases):
            out += [w, b]
        return out


def spec(data, key) -> Spec:
    d = json.loads(str(data[key]))
    return Spec(name=d["name"], n=d["n"], m=d["m"], dt=d["dt"], t_max=d["t_max"],
                u_max=tuple(d["u_max"]), workspace=tuple(tuple(b) for b in d["workspace"]),
                hard_region=tuple(tuple(b) for b in d["hard_region"]),
                extra=tuple(tuple(e) for e in d["extra"]))


def field(data, key) -> Field:
    d = json.loads(str(data[key]))
    obs = tuple(Ellipse(tuple(o["center"]), tuple(o["semi_axes"]), o["angle"]) for o in d["obstacles"])
    return Field(target=tuple(d["target"]), obstacles=obs, obstacle_weight=d["obstacle_weight"],
                 target_reward_weight=d["target_reward_weight"],
                 target_reward_radius=d["target_reward_radius"],
                 control_weight=d["control_weight"], distance_weight=d["distance_weight"])


def net(data, prefix) -> Net:
    meta = json.loads(str(data[f"{prefix}_meta"]))
    L = meta["n_layers"]
    arr = lambda v: None if v is None else np.asarray(v, dtype=float)  # noqa: E731
    return Net(weights=tuple(data[f"{prefix}_W{i}"] for i in range(L)),
               biases=tuple(data[f"{prefix}_b{i}"] for i in range(L)),
               activation=meta["activation"], head=meta["head"], sigma_min=meta["sigma_min"],
               out_scale=arr(meta["out_scale"]), in_center=arr(meta["in_center"]),
               in_half=arr(meta["in_half"]))


def grads(data, prefix, count):
    return [data[f"{prefix}_g{i}"] for i in range(count)]


def batch(data, prefix):
    return SimpleNamespace(xa=data[f"{prefix}_xa"], u=data[f"{prefix}_u"],
                           v_bar=data[f"{prefix}_v_bar"], v_bar_x=data[f"{prefix}_v_bar_x"],
                           xa_plus_k=data[f"{prefix}_xa_plus_k"],
                           t_max=int(data[f"{prefix}_t_max"]))


SYSTEMS = ("toy1d", "pointmass", "dubins", "manipulator3", "aliengo_lipm")


KSTEP_SETS = ("pointmass", "dubins", "synthetic")


def solutions(d, name):
    """The iLQR solutions of a kstep fixture set, as reference-shaped objects
    (`SolveResult` with `.traj.X/.U/.step_costs/.t0`, `.V_bar`, `.V_bar_x`)."""
    out = []
    for i in range(int(d[f"ks_{name}_count"])):
        p = f"ks_{name}_{i}"
        traj = SimpleNamespace(X=d[f"{p}_X"], U=d[f"{p}_U"], step_costs=d[f"{p}_sc"], t0=int(d[f"{p}_t0"]))
        out.append(SimpleNamespace(traj=traj, V_bar=d[f"{p}_Vb"], V_bar_x=d[f"{p}_Vbx"]))
    return out
