"""Reference-arm adapter (bench / test infrastructure, never the product).

Loads the UNMODIFIED reference package `trajrl` installed in `baseline/_ref`
 and converts this repo's spec / field / network objects into
the reference's own types, so `bench.py --impl reference` and the CPU baselines
time the reference's public functions themselves:
  nets.actor_rollout (nets.py:403-423), nets.mlp_forward (nets.py:165-173),
  nets.critic_loss (nets.py:233-290), nets.adam_step (nets.py:375-392),
  nets.polyak (nets.py:395-398).
The synthetic AlienGO system (no reference counterpart) is registered
through the reference's own plug-in API (register_system, envs/base.py:153-157;
register_cost, envs/costs.py:182-187), as tests/golden/make_golden.py does.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

from . import aliengo as O_aliengo

_R = None


def load(root=None):
    """Import trajrl from baseline/_ref (raises ImportError if it is not installed)."""
    global _R
    if _R is not None:
        return _R
    root = Path(root) if root else Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if not (root / "trajrl").is_dir():
        raise ImportError(f"reference not installed at {root}")
    sys.path.insert(0, str(root))
    import trajrl
    from trajrl import nets, envs
    from trajrl.envs.base import System, register_system
    from trajrl.envs.costs import Cost, register_cost
    if not str(Path(trajrl.__file__).resolve()).startswith(str(root.resolve())):
        raise ImportError(f"trajrl resolved to {trajrl.__file__}, not {root}")

    if O_aliengo.NAME not in getattr(envs.base, "_REGISTRY", {}):
        try:
            @register_system(O_aliengo.NAME)
            class _AlienGoLipm(System):
                def step_x(self, x, u):
                    return O_aliengo.step_x(self.spec, x, u)

                def jacobians(self, x, u):
                    fu = O_aliengo.control_jacobian(self.spec, x, u)
                    return np.zeros(fu.shape[:-2] + (self.n, self.n)), fu

                def position(self, x):
                    return x[..., 4:6]

            class _AlienGoCost(Cost):
                def __init__(self, spec, field, system):
                    self.spec, self.field = spec, field

                def stage(self, x, u):
                    return O_aliengo.stage_cost(self.spec, self.field, x, u)

                def terminal(self, x):
                    return O_aliengo.terminal_cost(self.spec, self.field, x)

            register_cost(O_aliengo.NAME)(lambda spec, field, system: _AlienGoCost(spec, field, system))
        except ValueError:  # already registered in this process
            pass
    _R = trajrl
    return trajrl


def model(spec):
    R = load()
    return R.envs.ModelSpec(name=spec.name, n=int(spec.n), m=int(spec.m), dt=float(spec.dt), t_max=int(spec.t_max),
                            u_max=tuple(float(v) for v in spec.u_max), workspace=tuple(spec.workspace),
                            hard_region=tuple(spec.hard_region), extra=tuple(spec.extra))


def field(fld):
    R = load()
    obst = tuple(R.envs.Ellipse(tuple(o.center), tuple(o.semi_axes), float(o.angle)) for o in fld.obstacles)
    return R.envs.CostField(target=tuple(fld.target), obstacles=obst, obstacle_weight=fld.obstacle_weight,
                            target_reward_weight=fld.target_reward_weight,
                            target_reward_radius=fld.target_reward_radius, control_weight=fld.control_weight,
                            distance_weight=fld.distance_weight)


def mlp(net):
    R = load()
    arr = lambda v: None if v is None else np.asarray(v, dtype=float)  # noqa: E731
    return R.nets.Mlp(weights=tuple(np.asarray(w, float) for w in net.weights),
                      biases=tuple(np.asarray(b, float) for b in net.biases), activation=net.activation,
                      head=net.head, out_scale=arr(net.out_scale), sigma_min=net.sigma_min,
                      in_center=arr(net.in_center), in_half=arr(net.in_half))
