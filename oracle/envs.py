"""Oracle: discrete dynamics, task costs and start sampling (float64, NumPy).

Restates `envs/systems.py`, `envs/manipulator.py`, `envs/costs.py`,
`envs/base.py` and `envs/__init__.py` of the reference.  Specs are duck-typed:
anything with the reference `ModelSpec` / `CostField` / `Ellipse` attributes
works (the reference's own objects, the product's mirrors, or plain
namespaces).  Test infrastructure only -- see `oracle/__init__.py`.
"""

from __future__ import annotations

import numpy as np

from . import aliengo

SHARPNESS = 10.0   # envs/costs.py:16  BARRIER_SHARPNESS
TOY_TILT = 0.3     # envs/costs.py:19

_PI = float(np.pi)

# envs/__init__.py:24-49 -- per-system defaults (plus the synthetic quadruped)
DEFAULTS = {
    "toy1d": dict(n=1, m=1, dt=0.05, t_max=60, u_max=(2.0,),
                  workspace=((-2.0, 2.0),), hard_region=((0.3, 1.9),)),
    "pointmass": dict(n=4, m=2, dt=0.05, t_max=60, u_max=(20.0, 20.0),
                      workspace=((-15.0, 15.0), (-15.0, 15.0), (-6.0, 6.0), (-6.0, 6.0)),
                      hard_region=((5.0, 12.0), (-3.0, 3.0), (0.0, 0.0), (0.0, 0.0))),
    "dubins": dict(n=5, m=2, dt=0.05, t_max=100, u_max=(3.0, 6.0),
                   workspace=((-15.0, 15.0), (-15.0, 15.0), (-_PI, _PI), (-8.0, 8.0), (-4.0, 4.0)),
                   hard_region=((5.0, 12.0), (-3.0, 3.0), (-_PI, _PI), (0.0, 0.0), (0.0, 0.0))),
    "manipulator3": dict(n=6, m=3, dt=0.05, t_max=100, u_max=(100.0, 60.0, 25.0),
                         workspace=((-_PI, _PI),) * 3 + ((-2.0, 2.0),) * 3,
                         hard_region=((-0.4, 0.4),) * 3 + ((0.0, 0.0),) * 3),
    aliengo.NAME: aliengo.DEFAULTS,
}

# envs/manipulator.py:19 -- default link lengths and masses
MANIP_LINKS = {"l1": 4.0, "l2": 3.5, "l3": 2.5, "m1": 1.5, "m2": 1.0, "m3": 0.6}


def extra_params(spec) -> dict:
    return dict(getattr(spec, "extra", ()) or ())


def region_box(spec, region="workspace"):
    """envs/base.py:110-116."""
    region = getattr(region, "value", region)
    bounds = spec.workspace if region == "workspace" else spec.hard_region
    lo = np.array([float(b[0]) for b in bounds])
    hi = np.array([float(b[1]) for b in bounds])
    if np.any(lo > hi):
        raise ValueError(f"empty {region} box: lo > hi")
    return lo, hi


# -- manipulator rigid-body constants (envs/manipulator.py:25-47) -------------

def manipulator_constants(spec):
    p = dict(MANIP_LINKS)
    p.update(extra_params(spec))
    l1, l2, l3 = p["l1"], p["l2"], p["l3"]
    m1, m2, m3 = p["m1"], p["m2"], p["m3"]
    r = (l1 / 2, l2 / 2, l3 / 2)
    inert = (m1 * l1 ** 2 / 12, m2 * l2 ** 2 / 12, m3 * l3 ** 2 / 12)
    a1 = inert[0] + m1 * r[0] ** 2 + (m2 + m3) * l1 ** 2
    a2 = inert[1] + m2 * r[1] ** 2 + m3 * l2 ** 2
    a3 = inert[2] + m3 * r[2] ** 2
    b12 = (m2 * r[1] + m3 * l2) * l1
    b13 = m3 * r[2] * l1
    b23 = m3 * r[2] * l2
    A0 = np.array([[a1 + a2 + a3, a2 + a3, a3], [a2 + a3, a2 + a3, a3], [a3, a3, a3]])
    B12 = b12 * np.array([[2.0, 1, 0], [1, 0, 0], [0, 0, 0]])
    B13 = b13 * np.array([[2.0, 1, 1], [1, 0, 0], [1, 0, 0]])
    B23 = b23 * np.array([[2.0, 2, 1], [2, 2, 1], [1, 1, 0]])
    return dict(lengths=np.array([l1, l2, l3]), A0=A0, B12=B12, B13=B13, B23=B23)


def _manip_mass(k, q):
    """M(q) and dM/dq_l (leading derivative index), envs/manipulator.py:51-65."""
    c2, s2 = np.cos(q[..., 1]), np.sin(q[..., 1])
    c3, s3 = np.cos(q[..., 2]), np.sin(q[..., 2])
    q23 = q[..., 1] + q[..., 2]
    c23, s23 = np.cos(q23), np.sin(q23)
    sc = lambda a, mat: a[..., None, None] * mat  # noqa: E731
    M = k["A0"] + sc(c2, k["B12"]) + sc(c23, k["B13"]) + sc(c3, k["B23"])
    dM = np.zeros(q.shape[:-1] + (3, 3, 3))
    dM[..., 1, :, :] = -sc(s2, k["B12"]) - sc(s23, k["B13"])
    dM[..., 2, :, :] = -sc(s23, k["B13"]) - sc(s3, k["B23"])
    return M, dM


def manipulator_accel(k, q, dq, tau):
    """qdd = M^-1 (tau - C(q)[dq, dq]); envs/manipulator.py:73-84."""
    M, dM = _manip_mass(k, q)
    # Christoffel symbols of the first kind, c[i,j,k] (manipulator.py:73-78)
    d_k_ij = np.moveaxis(dM, -3, -1)
    chris = 0.5 * (d_k_ij + np.swapaxes(d_k_ij, -2, -1) - dM)
    h = np.einsum("...ijk,...j,...k->...i", chris, dq, dq)
    return np.linalg.solve(M, (tau - h)[..., None])[..., 0], M


# -- dynamics -----------------------------------------------------------------

def step_x(spec, x, u):
    """One explicit-Euler step x+ = f(x, u), batched over leading axes.

    toy1d systems.py:26-27, pointmass systems.py:47-48, dubins systems.py:72-80,
    manipulator3 manipulator.py:88-91, aliengo_lipm oracle/aliengo.py.
    """
    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    dt = float(spec.dt)
    name = spec.name
    if name == "toy1d":
        return x + dt * u
    if name == "pointmass":
        out = np.empty_like(x)
        out[..., 0] = x[..., 0] + dt * x[..., 2]
        out[..., 1] = x[..., 1] + dt * x[..., 3]
        out[..., 2] = x[..., 2] + dt * u[..., 0]
        out[..., 3] = x[..., 3] + dt * u[..., 1]
        return out
    if name == "dubins":
        th, v, a = x[..., 2], x[..., 3], x[..., 4]
        out = np.empty_like(x)
        out[..., 0] = x[..., 0] + dt * v * np.cos(th)
        out[..., 1] = x[..., 1] + dt * v * np.sin(th)
        out[..., 2] = th + dt * u[..., 0]
        out[..., 3] = v + dt * a
        out[..., 4] = a + dt * u[..., 1]
        return out
    if name == "manipulator3":
        k = manipulator_constants(spec)
        q, dq = x[..., :3], x[..., 3:]
        qdd, _ = manipulator_accel(k, q, dq, u)
        return np.concatenate([q + dt * dq, dq + dt * qdd], axis=-1)
    if name == aliengo.NAME:
        return aliengo.step_x(spec, x, u)
    raise ValueError(f"unknown system '{name}'")


def control_jacobian(spec, x, u):
    """f_u = d x+/d u, shape (..., n, m).

    pointmass systems.py:50-54, dubins systems.py:82-94 (fu part),
    manipulator3 manipulator.py:109-122 (fu = dt*M^-1), toy1d systems.py:29-33.
    """
    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    dt = float(spec.dt)
    batch = x.shape[:-1]
    n, m = int(spec.n), int(spec.m)
    name = spec.name
    fu = np.zeros(batch + (n, m))
    if name == "toy1d":
        fu[..., 0, 0] = dt
    elif name == "pointmass":
        fu[..., 2, 0] = dt
        fu[..., 3, 1] = dt
    elif name == "dubins":
        fu[..., 2, 0] = dt
        fu[..., 4, 1] = dt
    elif name == "manipulator3":
        k = manipulator_constants(spec)
        M, _ = _manip_mass(k, x[..., :3])
        fu[..., 3:, :] = dt * np.linalg.inv(M)
    elif name == aliengo.NAME:
        return aliengo.control_jacobian(spec, x, u)
    else:
        raise ValueError(f"unknown system '{name}'")
    return fu


def position(spec, x):
    """Task-space point p(x): systems.py:56-57, 96-97, manipulator.py:130-133."""
    x = np.asarray(x, dtype=float)
    if spec.name in ("pointmass", "dubins"):
        return x[..., :2]
    if spec.name == "manipulator3":
        lengths = manipulator_constants(spec)["lengths"]
        ang = np.cumsum(x[..., :3], axis=-1)
        return np.stack([(lengths * np.cos(ang)).sum(axis=-1),
                         (lengths * np.sin(ang)).sum(axis=-1)], axis=-1)
    if spec.name == aliengo.NAME:
        return x[..., 4:6]
    raise ValueError(f"system '{spec.name}' has no task point")


# -- costs ----------------------------------------------------------------------

def softplus(z):
    """costs.py:22-23 (np.logaddexp(0, z))."""
    return np.logaddexp(0.0, z)


def sigmoid(z):
    """costs.py:26-29 / nets.py:59-60."""
    z = np.asarray(z, dtype=float)
    return np.exp(z - np.logaddexp(0.0, z))


def ellipse_form(ob) -> np.ndarray:
    """E with (p-c)^T E (p-c) = 1 on the boundary; envs/base.py:53-58."""
    ca, sa = np.cos(ob.angle), np.sin(ob.angle)
    rot = np.array([[ca, sa], [-sa, ca]])
    scale = np.diag([1.0 / ob.semi_axes[0] ** 2, 1.0 / ob.semi_axes[1] ** 2])
    return rot.T @ scale @ rot


def _check_field(spec, field):
    """costs.py:190-200 -- the task cost needs exactly three obstacles."""
    if spec.name in ("toy1d", aliengo.NAME):
        return
    if len(field.obstacles) != 3:
        raise ValueError(f"{spec.name} expects exactly 3 obstacles, got {len(field.obstacles)}")


def point_value(field, p):
    """Reach/avoid scalar field over the task point; costs.py:97-107."""
    rel = p - np.asarray(field.target, dtype=float)
    q = (rel ** 2).sum(axis=-1)
    val = field.distance_weight * q
    val -= field.target_reward_weight * np.exp(-q / field.target_reward_radius ** 2)
    for ob in field.obstacles:
        d = p - np.asarray(ob.center, dtype=float)
        e = np.einsum("...i,ij,...j->...", d, ellipse_form(ob), d)
        val += field.obstacle_weight * softplus(SHARPNESS * (1.0 - e))
    return val


def _toy_base(x):
    s = x[..., 0]
    return (s ** 2 - 1.0) ** 2 + TOY_TILT * s          # costs.py:59-64


def terminal_cost(spec, field, x):
    """l_T(x): costs.py:78-79 (toy), 167-168 (task)."""
    x = np.asarray(x, dtype=float)
    _check_field(spec, field)
    if spec.name == "toy1d":
        return _toy_base(x)
    if spec.name == aliengo.NAME:
        return aliengo.terminal_cost(spec, field, x)
    return point_value(field, position(spec, x))


def stage_cost(spec, field, x, u):
    """l(x, u): costs.py:66-67 (toy), 147-149 (task)."""
    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    _check_field(spec, field)
    w_u = field.control_weight
    if spec.name == "toy1d":
        return _toy_base(x) + w_u * (u[..., 0] ** 2)
    if spec.name == aliengo.NAME:
        return aliengo.stage_cost(spec, field, x, u)
    return point_value(field, position(spec, x)) + w_u * (u ** 2).sum(axis=-1)


def stage_cost_du(spec, field, x, u):
    """l_u = 2 w_u u for every system (costs.py:71, 162; aliengo likewise)."""
    return 2.0 * field.control_weight * np.asarray(u, dtype=float)


def trajectory_costs(spec, field, X, U):
    """step costs [stage(X[:-1], U), terminal(X[-1])]; ilqr.py:210-214."""
    sc = np.empty(U.shape[-2] + 1)
    sc[:-1] = stage_cost(spec, field, X[:-1], U)
    sc[-1] = terminal_cost(spec, field, X[-1])
    return sc


# -- start sampling ---------------------------------------------------------------

def sample_initial_states(spec, count, rng_seed, region="workspace"):
    """Uniform i.i.d. starts at t=0 as an (count, n) array; envs/__init__.py:112-122."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    lo, hi = region_box(spec, region)
    draws = np.random.default_rng(rng_seed).uniform(size=(count, int(spec.n)))
    return draws * (hi - lo) + lo


def seed_int(seed, *tags) -> int:
    """trainer.py:133-138."""
    seq = np.random.SeedSequence([int(seed)] + [int(t) for t in tags])
    return int(seq.generate_state(1)[0])


def normalisation(spec):
    """(in_center, in_half) of the trainer's networks; trainer.py:96-99."""
    lo, hi = region_box(spec, "workspace")
    center = np.concatenate([(lo + hi) / 2.0, [0.0]])
    half = np.concatenate([np.maximum((hi - lo) / 2.0, 1e-9), [float(spec.t_max)]])
    return center, half
