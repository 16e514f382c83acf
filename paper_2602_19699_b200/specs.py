"""Host-side problem descriptions, mirroring the reference `trajrl.envs` types.

`TimeState`, `Region`, `Ellipse`, `CostField`, `ModelSpec` and `default_model`
have the reference's field names and validation (envs/base.py:18-119,
envs/__init__.py:24-57), so reference objects and these mirrors are
interchangeable everywhere in this package (duck typing).  The functions at
the bottom translate a (spec, field) pair into the C-ABI descriptors
`cacto_system_t` / `cacto_cost_t`.  Only systems compiled into the CUDA
library are accepted -- a system registered in Python alone raises, per the
"no CPU fallback" rule.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib

Bounds = tuple


class Region(enum.Enum):
    WORKSPACE = "workspace"
    HARD_REGION = "hard_region"


@dataclass(frozen=True)
class TimeState:
    """Augmented state [x, t] (envs/base.py:23-40)."""

    x: np.ndarray
    t: int = 0

    def __post_init__(self):
        object.__setattr__(self, "x", np.asarray(self.x, dtype=float))
        if self.x.ndim != 1:
            raise ValueError(f"state must be a 1-d vector, got shape {self.x.shape}")
        if self.t < 0:
            raise ValueError(f"time index must be >= 0, got {self.t}")

    @property
    def augmented(self) -> np.ndarray:
        return np.concatenate([self.x, [float(self.t)]])


@dataclass(frozen=True)
class Ellipse:
    center: tuple
    semi_axes: tuple
    angle: float = 0.0

    def __post_init__(self):
        if min(self.semi_axes) <= 0.0:
            raise ValueError(f"semi-axes must be positive, got {self.semi_axes}")

    def quadratic_form(self) -> np.ndarray:
        """E with (p-c)^T E (p-c) = 1 on the boundary (envs/base.py:53-58)."""
        c, s = np.cos(self.angle), np.sin(self.angle)
        rot = np.array([[c, s], [-s, c]])
        d = np.diag([1.0 / self.semi_axes[0] ** 2, 1.0 / self.semi_axes[1] ** 2])
        return rot.T @ d @ rot


@dataclass(frozen=True)
class CostField:
    target: tuple = (-7.0, 0.0)
    obstacles: tuple = ()
    obstacle_weight: float = 0.0
    target_reward_weight: float = 0.0
    target_reward_radius: float = 1.0
    control_weight: float = 0.0
    distance_weight: float = 1.0

    def __post_init__(self):
        for w in (self.obstacle_weight, self.target_reward_weight, self.control_weight,
                  self.distance_weight):
            if w < 0.0:
                raise ValueError("cost weights must be non-negative")
        if self.target_reward_radius <= 0.0:
            raise ValueError("target_reward_radius must be positive")


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n: int
    m: int
    dt: float
    t_max: int
    u_max: tuple
    workspace: tuple
    hard_region: tuple
    extra: tuple = dc_field(default=())

    def __post_init__(self):
        if self.dt <= 0.0 or self.t_max < 1:
            raise ValueError("need dt > 0 and t_max >= 1")
        if len(self.u_max) != self.m or any(b <= 0.0 for b in self.u_max):
            raise ValueError("u_max must have m positive components")
        for bounds, label in ((self.workspace, "workspace"), (self.hard_region, "hard_region")):
            if len(bounds) != self.n:
                raise ValueError(f"{label} must cover all {self.n} state dims")

    @property
    def u_bound(self) -> np.ndarray:
        return np.asarray(self.u_max, dtype=float)

    def region_box(self, region) -> tuple:
        return region_box(self, region)

    def extra_params(self) -> dict:
        return dict(self.extra)


def region_box(spec, region=Region.WORKSPACE):
    region = getattr(region, "value", region)
    bounds = spec.workspace if region == "workspace" else spec.hard_region
    lo = np.array([float(b[0]) for b in bounds])
    hi = np.array([float(b[1]) for b in bounds])
    if np.any(lo > hi):
        raise ValueError(f"empty {region} box: lo > hi")
    return lo, hi


_PI = float(np.pi)

# ---- synthetic AlienGO-like quadruped (equations in DESIGN.md) ----
ALIENGO = "aliengo_lipm"
LIPM_OMEGA = math.sqrt(9.81 / 0.35)
LIPM_SX, LIPM_SY = 0.24, 0.13
LIPM_DELTA0 = 0.375
LIPM_W_VEL, LIPM_W_VBAR, LIPM_V_MAX2, LIPM_OBS_R2, LIPM_W_WALL = 0.05, 1.0, 1.5 ** 2, 0.5 ** 2, 5.0

DEFAULTS = {
    "toy1d": dict(n=1, m=1, dt=0.05, t_max=60, u_max=(2.0,), workspace=((-2.0, 2.0),),
                  hard_region=((0.3, 1.9),)),
    "pointmass": dict(n=4, m=2, dt=0.05, t_max=60, u_max=(20.0, 20.0),
                      workspace=((-15.0, 15.0), (-15.0, 15.0), (-6.0, 6.0), (-6.0, 6.0)),
                      hard_region=((5.0, 12.0), (-3.0, 3.0), (0.0, 0.0), (0.0, 0.0))),
    "dubins": dict(n=5, m=2, dt=0.05, t_max=100, u_max=(3.0, 6.0),
                   workspace=((-15.0, 15.0), (-15.0, 15.0), (-_PI, _PI), (-8.0, 8.0), (-4.0, 4.0)),
                   hard_region=((5.0, 12.0), (-3.0, 3.0), (-_PI, _PI), (0.0, 0.0), (0.0, 0.0))),
    "manipulator3": dict(n=6, m=3, dt=0.05, t_max=100, u_max=(100.0, 60.0, 25.0),
                         workspace=((-_PI, _PI),) * 3 + ((-2.0, 2.0),) * 3,
                         hard_region=((-0.4, 0.4),) * 3 + ((0.0, 0.0),) * 3),
    ALIENGO: dict(n=15, m=6, dt=LIPM_DELTA0, t_max=100, u_max=(0.15, 0.15, 0.15, 0.15, 0.5, 0.125),
                  workspace=((-0.1, 0.1),) * 4 + ((-4.0, 4.0),) * 2 + ((-1.0, 1.0),) * 2 + ((0.0, 100.0),)
                  + ((-2.0, 2.0),) * 2 + ((-6.0, -4.5), (4.5, 6.0), (-6.0, -4.5), (4.5, 6.0)),
                  hard_region=((0.0, 0.0),) * 4 + ((2.0, 3.5), (-1.0, 1.0)) + ((0.0, 0.0),) * 2
                  + ((0.0, 0.0),) + ((1.0, 1.0), (0.0, 0.0))
                  + ((-5.0, -5.0), (5.0, 5.0), (-5.0, -5.0), (5.0, 5.0))),
}


def default_model(name: str, **overrides) -> ModelSpec:
    """envs/__init__.py:52-57."""
    if name not in DEFAULTS:
        raise ValueError(f"unknown system '{name}' (known: {sorted(DEFAULTS)})")
    kw = dict(DEFAULTS[name])
    kw.update(overrides)
    return ModelSpec(name=name, **kw)


# ---- the reference experiment configs (pkg/configs/*.ini) ------------------------
_PI_INI = 3.14159265
_WALL = (Ellipse((0.0, 3.5), (1.8, 3.2)), Ellipse((0.0, -3.5), (1.8, 3.2)), Ellipse((1.2, 0.0), (2.2, 1.4)))


def config(name: str):
    """(ModelSpec, CostField) of the reference INI configs: pointmass.ini:3-21,
    dubins.ini:3-20, manipulator.ini:3-29 (param_* extras), toy1d.ini:3-14, plus
    the synthetic quadruped."""
    if name == "pointmass":
        return (default_model("pointmass"),
                CostField((-7.0, 0.0), _WALL, 10.0, 15.0, 2.0, 0.005, 0.02))
    if name == "dubins":
        ws = ((-15.0, 15.0), (-15.0, 15.0), (-_PI_INI, _PI_INI), (-8.0, 8.0), (-4.0, 4.0))
        hr = ((5.0, 12.0), (-3.0, 3.0), (-_PI_INI, _PI_INI), (0.0, 0.0), (0.0, 0.0))
        return (default_model("dubins", workspace=ws, hard_region=hr),
                CostField((-7.0, 0.0), _WALL, 10.0, 15.0, 2.0, 0.005, 0.02))
    if name in ("manipulator", "manipulator3"):
        ws = ((-_PI_INI, _PI_INI),) * 3 + ((-2.0, 2.0),) * 3
        extra = tuple(sorted({"l1": 4.0, "l2": 3.5, "l3": 2.5, "m1": 1.5, "m2": 1.0, "m3": 0.6}.items()))
        obst = (Ellipse((0.0, 5.75), (2.0, 5.25)), Ellipse((0.0, -5.75), (2.0, 5.25)),
                Ellipse((1.2, 0.0), (2.5, 1.6)))
        return (default_model("manipulator3", workspace=ws, extra=extra),
                CostField((-7.0, 0.0), obst, 10.0, 15.0, 2.0, 0.0001, 0.02))
    if name == "toy1d":
        return default_model("toy1d"), CostField(control_weight=0.01)
    if name == ALIENGO:
        return (default_model(ALIENGO),
                CostField((0.0, 0.0), (), 10.0, 15.0, 1.0, 0.01, 0.05))
    raise ValueError(f"unknown config '{name}'")


# ---- C-ABI descriptors -------------------------------------------------------------
_MANIP_DEFAULT = {"l1": 4.0, "l2": 3.5, "l3": 2.5, "m1": 1.5, "m2": 1.0, "m3": 0.6}


def system_struct(spec) -> _lib.CactoSystem:
    if spec.name not in _lib.SYS:
        raise ValueError(f"system '{spec.name}' has no CUDA implementation in libcacto_b200 "
                         f"(built: {sorted(_lib.SYS)})")
    s = _lib.CactoSystem()
    s.kind = _lib.SYS[spec.name]
    s.n, s.m, s.t_max = int(spec.n), int(spec.m), int(spec.t_max)
    s.dt = float(spec.dt)
    for j, b in enumerate(spec.u_max):
        s.u_max[j] = float(b)
    if spec.name == "manipulator3":
        p = dict(_MANIP_DEFAULT)
        p.update(dict(getattr(spec, "extra", ()) or ()))
        for i, k in enumerate(("l1", "l2", "l3", "m1", "m2", "m3")):
            s.p[i] = float(p[k])
    if spec.name == ALIENGO:
        s.p[0], s.p[1], s.p[2], s.p[3] = LIPM_OMEGA, LIPM_SX, LIPM_SY, LIPM_DELTA0
    return s


def cost_struct(spec, field) -> _lib.CactoCost:
    c = _lib.CactoCost()
    if spec.name == "toy1d":
        c.kind = _lib.COST_TOY1D
    elif spec.name == ALIENGO:
        c.kind = _lib.COST_LIPM
        c.extra[0], c.extra[1], c.extra[2], c.extra[3], c.extra[4] = (
            LIPM_W_VEL, LIPM_W_VBAR, LIPM_V_MAX2, LIPM_OBS_R2, LIPM_W_WALL)
    else:
        c.kind = _lib.COST_TASK
        if len(field.obstacles) != 3:   # costs.py:197-199
            raise ValueError(f"{spec.name} expects exactly 3 obstacles, got {len(field.obstacles)}")
    obs = tuple(field.obstacles)
    if len(obs) > _lib.MAX_OBST:
        raise ValueError("too many obstacles")
    c.n_obstacles = len(obs) if c.kind == _lib.COST_TASK else 0
    c.target[0], c.target[1] = float(field.target[0]), float(field.target[1])
    for i, ob in enumerate(obs):
        E = Ellipse(tuple(ob.center), tuple(ob.semi_axes), float(ob.angle)).quadratic_form()
        c.obs_center[i][0], c.obs_center[i][1] = float(ob.center[0]), float(ob.center[1])
        for q, v in enumerate(E.reshape(-1)):
            c.obs_form[i][q] = float(v)
    c.w_obstacle = float(field.obstacle_weight)
    c.w_reward = float(field.target_reward_weight)
    c.reward_radius = float(field.target_reward_radius)
    c.w_control = float(field.control_weight)
    c.w_distance = float(field.distance_weight)
    return c


def normalisation(spec):
    """(in_center, in_half) used by the trainer's networks (trainer.py:96-99)."""
    lo, hi = region_box(spec, Region.WORKSPACE)
    center = np.concatenate([(lo + hi) / 2.0, [0.0]])
    half = np.concatenate([np.maximum((hi - lo) / 2.0, 1e-9), [float(spec.t_max)]])
    return center, half
