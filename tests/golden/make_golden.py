"""Generate the golden fixtures for the hot path by running the REAL reference.

Run in the build container (where /root/reference exists), never on the GPU box:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [fixture ...]

It imports `trajrl` read-only from /root/reference/pkg/src, evaluates the hot
path functions on seeded inputs and writes `tests/golden/*.npz`.  The fixtures
carry everything needed to rebuild the inputs (specs / fields as JSON, network
parameters, batches), so the oracle tests and the GPU parity tests never read
the reference at run time.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path(os.environ.get("CACTO_REFERENCE", "/root/reference")) / "pkg"
sys.path.insert(0, str(REF / "src"))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from trajrl import envs as R_envs, ilqr as R_ilqr, nets as R_nets, trainer as R_trainer  # noqa: E402
from trajrl.buffer import ReplayBuffer, SampleBatch, TOSample  # noqa: E402
from trajrl.config import load_config  # noqa: E402
from trajrl.envs import TimeState  # noqa: E402
from trajrl.envs.base import System, register_system  # noqa: E402
from trajrl.envs.costs import Cost, register_cost  # noqa: E402

from oracle import aliengo as O_aliengo  # noqa: E402  (system definition only)


# -- register the synthetic quadruped through the reference plug-in API --------

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

    def stage_derivs(self, x, u):
        l = self.stage(x, u)
        lu = 2.0 * self.field.control_weight * u
        return l, None, lu, None, None, None


register_cost(O_aliengo.NAME)(lambda spec, field, system: _AlienGoCost(spec, field, system))


def aliengo_spec():
    return R_envs.ModelSpec(name=O_aliengo.NAME, **O_aliengo.DEFAULTS)


def aliengo_field():
    return R_envs.CostField(target=(0.0, 0.0), obstacles=(), obstacle_weight=10.0,
                            target_reward_weight=15.0, target_reward_radius=1.0,
                            control_weight=0.01, distance_weight=0.05)


# -- helpers -------------------------------------------------------------------

def spec_json(spec):
    return json.dumps(dict(name=spec.name, n=spec.n, m=spec.m, dt=spec.dt, t_max=spec.t_max,
                           u_max=list(spec.u_max), workspace=[list(b) for b in spec.workspace],
                           hard_region=[list(b) for b in spec.hard_region],
                           extra=[list(e) for e in spec.extra]))


def field_json(field):
    return json.dumps(dict(target=list(field.target),
                           obstacles=[dict(center=list(o.center), semi_axes=list(o.semi_axes),
                                           angle=o.angle) for o in field.obstacles],
                           obstacle_weight=field.obstacle_weight,
                           target_reward_weight=field.target_reward_weight,
                           target_reward_radius=field.target_reward_radius,
                           control_weight=field.control_weight,
                           distance_weight=field.distance_weight))


def mlp_dict(prefix, mlp):
    d = {f"{prefix}_meta": json.dumps(dict(
        activation=mlp.activation, head=mlp.head, sigma_min=mlp.sigma_min,
        n_layers=len(mlp.weights),
        out_scale=None if mlp.out_scale is None else list(map(float, mlp.out_scale)),
        in_center=None if mlp.in_center is None else list(map(float, mlp.in_center)),
        in_half=None if mlp.in_half is None else list(map(float, mlp.in_half))))}
    for i, (w, b) in enumerate(zip(mlp.weights, mlp.biases)):
        d[f"{prefix}_W{i}"] = w
        d[f"{prefix}_b{i}"] = b
    return d


def grads_dict(prefix, grads):
    return {f"{prefix}_g{i}": g for i, g in enumerate(grads)}


def trainer_nets(spec, seed, hidden=(64, 64, 64)):
    cfg = R_trainer.TrainConfig(model=spec, field=R_envs.CostField(), hidden=hidden, seed=seed)
    st = R_trainer.TrainerState(cfg)
    return st.actor, st.critic, st.std


def scale_output(mlp, factor):
    p = list(mlp.flat_params())
    p[-2] = p[-2] * factor
    return mlp.with_params(p)


def rand_batch(rng, spec, bsz, t_lo=0):
    """Workspace-uniform replay rows."""
    lo, hi = spec.region_box(R_envs.Region.WORKSPACE)
    n, m = spec.n, spec.m
    xa = np.empty((bsz, n + 1))
    xa[:, :n] = rng.uniform(size=(bsz, n)) * (hi - lo) + lo
    xa[:, n] = rng.integers(t_lo, spec.t_max, bsz)
    xk = np.empty((bsz, n + 1))
    xk[:, :n] = rng.uniform(size=(bsz, n)) * (hi - lo) + lo
    xk[:, n] = rng.integers(1, spec.t_max + 1, bsz)
    return SampleBatch(xa, rng.normal(0.0, 1.0, (bsz, m)), rng.normal(0.0, 1.0, bsz),
                       rng.normal(0.0, 1.0, (bsz, n)), xk, t_max=spec.t_max)


def batch_dict(prefix, b):
    return {f"{prefix}_xa": b.xa, f"{prefix}_u": b.u, f"{prefix}_v_bar": b.v_bar,
            f"{prefix}_v_bar_x": b.v_bar_x, f"{prefix}_xa_plus_k": b.xa_plus_k,
            f"{prefix}_t_max": np.array(b.t_max)}


def configs():
    rc = {name: load_config(REF / "configs" / f"{name}.ini")
          for name in ("pointmass", "dubins", "manipulator", "toy1d")}
    out = {"pointmass": (rc["pointmass"].model, rc["pointmass"].field),
           "dubins": (rc["dubins"].model, rc["dubins"].field),
           "manipulator3": (rc["manipulator"].model, rc["manipulator"].field),
           "toy1d": (rc["toy1d"].model, rc["toy1d"].field),
           O_aliengo.NAME: (aliengo_spec(), aliengo_field())}
    return out


# -- fixture builders -----------------------------------------------------------

def make_rollouts(cfgs):
    data = {}
    for name, (spec, field) in cfgs.items():
        actor, _, _ = trainer_nets(spec, seed=3)
        for tag, net in (("init", actor), ("trained", scale_output(actor, 10.0))):
            starts = R_envs.sample_initial_states(spec, 12, 1000 + len(name), R_envs.Region.WORKSPACE)
            # two starts mid-horizon, rolled out to the end (t0 > 0)
            t0s = [0] * 10 + [spec.t_max // 3, spec.t_max - 5]
            X, U, SC, C = [], [], [], []
            for s, t0 in zip(starts, t0s):
                st = TimeState(s.x, t0)
                tr = R_nets.actor_rollout(net, spec, st, spec.t_max - t0, field)
                pad = spec.t_max - t0
                Xp = np.full((spec.t_max + 1, spec.n), np.nan)
                Up = np.full((spec.t_max, spec.m), np.nan)
                Sp = np.full(spec.t_max + 1, np.nan)
                Xp[:pad + 1], Up[:pad], Sp[:pad + 1] = tr.X, tr.U, tr.step_costs
                X.append(Xp), U.append(Up), SC.append(Sp), C.append(tr.cost)
            key = f"{name}_{tag}"
            data.update(mlp_dict(f"{key}_actor", net))
            data[f"{key}_x0"] = np.stack([s.x for s in starts])
            data[f"{key}_t0"] = np.array(t0s)
            data[f"{key}_X"] = np.stack(X)
            data[f"{key}_U"] = np.stack(U)
            data[f"{key}_step_costs"] = np.stack(SC)
            data[f"{key}_cost"] = np.array(C)
        data[f"{name}_spec"] = spec_json(spec)
        data[f"{name}_field"] = field_json(field)
        # no-field rollout (warm-start call site trainer.py:192-193): zero costs
        tr = R_nets.actor_rollout(actor, spec, TimeState(starts[0].x, 0), spec.t_max)
        data[f"{name}_nofield_U"] = tr.U
        data[f"{name}_nofield_step_costs"] = tr.step_costs
    return data


def make_nets():
    rng = np.random.default_rng(2024)
    data = {}
    # forward / input gradient for all heads and odd shapes (test_nets.py:81-93 style)
    cases = [("lin3", [7, 64, 64, 64, 1], "linear", None),
             ("tanh", [6, 12, 8, 2], "tanh", np.array([2.0, 1.5])),
             ("std", [4, 10, 6, 1], "std", None),
             ("lin1", [4, 16, 1], "linear", None),
             ("tanh3", [16, 64, 64, 64, 6], "tanh", np.linspace(0.2, 1.2, 6))]
    for key, sizes, head, scale in cases:
        d = sizes[0]
        net = R_nets.init_mlp(sizes, rng, head=head, out_scale=scale,
                              in_center=rng.normal(0, 1, d), in_half=rng.uniform(0.5, 3.0, d))
        net = net.with_params([p + rng.normal(0, 0.05, p.shape) for p in net.flat_params()])
        xa = rng.normal(0.0, 2.0, (33, d))
        data.update(mlp_dict(f"fwd_{key}", net))
        data[f"fwd_{key}_x"] = xa
        data[f"fwd_{key}_y"] = R_nets.mlp_forward(net, xa)
        data[f"fwd_{key}_jac"] = R_nets.mlp_input_gradient(net, xa)
        if head == "linear":
            v, g = R_nets.value_and_state_grad(net, xa)
            data[f"fwd_{key}_v"], data[f"fwd_{key}_g"] = v, g
    # a single linear layer (test_nets.py:54-65) and the BIC stub (test_trainer.py:40-43)
    net = R_nets.Mlp(weights=(rng.normal(0, 1, (3, 4)),), biases=(rng.normal(0, 1, 3),))
    data.update(mlp_dict("fwd_single", net))
    data["fwd_single_x"] = rng.normal(0, 1, (5, 4))
    data["fwd_single_y"] = R_nets.mlp_forward(net, data["fwd_single_x"])
    data["fwd_single_jac"] = R_nets.mlp_input_gradient(net, data["fwd_single_x"])
    return data


def make_losses(cfgs):
    rng = np.random.default_rng(77)
    data = {}
    # critic: trainer-shaped nets on manipulator dims, plus an odd small shape
    spec, field = cfgs["manipulator3"]
    actor, critic, std = trainer_nets(spec, seed=11)
    _, target, _ = trainer_nets(spec, seed=12)
    critic = critic.with_params([p + rng.normal(0, 0.05, p.shape) for p in critic.flat_params()])
    for key, bsz in (("b64", 64), ("b200", 200)):
        batch = rand_batch(rng, spec, bsz)
        batch.xa_plus_k[: bsz // 4, -1] = spec.t_max          # bootstrap gate at the horizon
        data.update(batch_dict(f"critic_{key}", batch))
        for boot in (True, False):
            loss, grads = R_nets.critic_loss(critic, target if boot else None, batch, 0.7, boot)
            data[f"critic_{key}_boot{int(boot)}_loss"] = np.array(loss)
            data.update(grads_dict(f"critic_{key}_boot{int(boot)}", grads))
        sloss, sgrads = R_nets.std_critic_loss(std, critic, batch)
        data[f"std_{key}_loss"] = np.array(sloss)
        data.update(grads_dict(f"std_{key}", sgrads))
    data.update(mlp_dict("critic_net", critic))
    data.update(mlp_dict("critic_target", target))
    data.update(mlp_dict("std_net", std))
    data["critic_spec"] = spec_json(spec)

    small_c = R_nets.init_mlp([4, 10, 8, 1], rng, in_center=np.zeros(4),
                              in_half=np.array([2.0, 1.0, 3.0, 50.0]))
    small_t = R_nets.init_mlp([4, 10, 8, 1], rng)
    xa = rng.normal(0.0, 1.0, (12, 4)); xa[:, -1] = rng.integers(0, 50, 12)
    xk = rng.normal(0.0, 1.0, (12, 4)); xk[:, -1] = rng.integers(1, 51, 12)
    sb = SampleBatch(xa, rng.normal(0, 1, (12, 2)), rng.normal(0, 1, 12),
                     rng.normal(0, 1, (12, 3)), xk, t_max=50)
    loss, grads = R_nets.critic_loss(small_c, small_t, sb, 0.5, True)
    data.update(mlp_dict("critic_small_net", small_c))
    data.update(mlp_dict("critic_small_target", small_t))
    data.update(batch_dict("critic_small", sb))
    data["critic_small_loss"] = np.array(loss)
    data.update(grads_dict("critic_small", grads))

    # actor loss on every system (states incl. some at the horizon)
    for name, (spec, field) in cfgs.items():
        if name == "toy1d":
            continue
        actor, critic, _ = trainer_nets(spec, seed=21)
        actor = scale_output(actor, 5.0)
        critic = critic.with_params([p + rng.normal(0, 0.05, p.shape) for p in critic.flat_params()])
        batch = rand_batch(rng, spec, 96)
        batch.xa[:5, -1] = spec.t_max                      # skipped rows (nets.py:308-312)
        loss, grads, skipped = R_nets.actor_loss(actor, critic, spec, field, batch)
        data.update(mlp_dict(f"actor_{name}_actor", actor))
        data.update(mlp_dict(f"actor_{name}_critic", critic))
        data[f"actor_{name}_xa"] = batch.xa
        data[f"actor_{name}_loss"] = np.array(loss)
        data[f"actor_{name}_skipped"] = np.array(skipped)
        data.update(grads_dict(f"actor_{name}", grads))
    return data


def make_optim():
    rng = np.random.default_rng(5)
    params = [rng.normal(0, 1, (7, 5)), rng.normal(0, 1, 7)]
    state = R_nets.AdamState.init(params, lr=3e-3)
    data = {"adam_p0_0": params[0], "adam_p0_1": params[1]}
    for k in range(5):
        grads = [rng.normal(0, 1, p.shape) for p in params]
        if k == 2:
            grads[1][:] = 0.0
        data[f"adam_g{k}_0"], data[f"adam_g{k}_1"] = grads
        params, state = R_nets.adam_step(params, state, grads)
        data[f"adam_p{k + 1}_0"], data[f"adam_p{k + 1}_1"] = params
    a = R_nets.init_mlp([3, 4, 1], rng)
    b = R_nets.init_mlp([3, 4, 1], rng)
    data.update(mlp_dict("polyak_a", a))
    data.update(mlp_dict("polyak_b", b))
    data.update(grads_dict("polyak_mix", R_nets.polyak(a, b, 0.25).flat_params()))
    return data


def make_select(cfgs):
    data = {}
    for name in ("pointmass", "dubins", "manipulator3"):
        spec, _ = cfgs[name]
        _, _, std = trainer_nets(spec, seed=31)
        std = std.with_params([p * 3.0 for p in std.flat_params()])
        seed = R_trainer._seed_int(0, 1, 2)
        cands = R_envs.sample_initial_states(spec, 750, seed, R_envs.Region.WORKSPACE)
        kept = R_trainer.select_initial_states_bic(cands, std, 75)
        idx = {id(c): i for i, c in enumerate(cands)}
        data.update(mlp_dict(f"select_{name}_std", std))
        data[f"select_{name}_seed"] = np.array(seed, dtype=np.uint64)
        data[f"select_{name}_cands"] = np.stack([c.x for c in cands])
        data[f"select_{name}_order"] = np.array([idx[id(c)] for c in kept])
        data[f"select_{name}_scores"] = R_nets.mlp_forward(std, np.stack([c.augmented for c in cands]))[:, 0]
    # ties / signed zero / NaN via the one-layer stub (test_trainer.py:40-60)
    stub = R_nets.Mlp(weights=(np.array([[1.0, 0.0]]),), biases=(np.zeros(1),), head="linear")
    vals = np.array([0.5, -0.0, 0.0, 2.0, np.nan, 0.5, -1.0, 0.0, np.nan, 2.0, -0.0, 0.5])
    cands = [TimeState(np.array([v]), 0) for v in vals]
    kept = R_trainer.select_initial_states_bic(cands, stub, 12)
    data["select_ties_vals"] = vals
    data["select_ties_order"] = np.array([next(i for i, c in enumerate(cands) if c is k) for k in kept])
    return data


def make_buffer():
    data = {}
    buf = ReplayBuffer(n=3, m=2, t_max=60, capacity=50, model_name="pointmass", k_lookahead=5)
    rng = np.random.default_rng(9)
    rows = []
    for i in range(83):                                    # wraps the ring
        rows.append(TOSample(TimeState(rng.normal(0, 1, 3), int(rng.integers(0, 60))),
                             rng.normal(0, 1, 2), float(rng.normal()), rng.normal(0, 1, 3),
                             TimeState(rng.normal(0, 1, 3), int(rng.integers(1, 61)))))
    buf.push_many(rows[:40])
    buf.push_many(rows[40:])
    g = np.random.default_rng(123)
    b1 = buf.sample_minibatch(64, g)
    b2 = buf.sample_minibatch(7, g)
    allb = SampleBatch.from_samples(rows, 60)
    data.update(batch_dict("buf_rows", allb))
    data.update(batch_dict("buf_mb1", b1))
    data.update(batch_dict("buf_mb2", b2))
    data["buf_capacity"] = np.array(50)
    data["buf_rng_seed"] = np.array(123)
    return data


def make_sampling(cfgs):
    data = {}
    for name, (spec, _) in cfgs.items():
        seed = R_trainer._seed_int(0, 1, 3)
        st = R_envs.sample_initial_states(spec, 40, seed, R_envs.Region.WORKSPACE)
        data[f"sample_{name}_seed"] = np.array(seed, dtype=np.uint64)
        data[f"sample_{name}_x"] = np.stack([s.x for s in st])
    return data


def _solution_dict(prefix, res):
    tr = res.traj
    return {f"{prefix}_X": tr.X, f"{prefix}_U": tr.U, f"{prefix}_sc": tr.step_costs,
            f"{prefix}_t0": np.array(tr.t0), f"{prefix}_Vb": np.asarray(res.V_bar, float),
            f"{prefix}_Vbx": np.asarray(res.V_bar_x, float)}


def make_kstep(cfgs):
    """Replay producer: kstep_targets (ilqr.py:358-407) on real
    iLQR solutions (pointmass, dubins; t0 = 0 and t0 > 0) and on synthetic
    solutions with long horizons (windows past NumPy's 128-term pairwise block),
    each pushed through ReplayBuffer.push_many into a small ring that wraps, and
    the TRLB dump of that ring (buffer.py:142-152)."""
    from trajrl.ilqr import SolveResult, Trajectory, solve_batch
    import tempfile
    from types import SimpleNamespace
    data = {}
    results = {}
    for name in ("pointmass", "dubins"):
        spec, fld = cfgs[name]
        st = R_envs.sample_initial_states(spec, 3, 11, R_envs.Region.WORKSPACE)
        st = [st[0], TimeState(st[1].x, 7), TimeState(st[2].x, spec.t_max - 3)]
        warms = [np.zeros((spec.t_max - s.t, spec.m)) for s in st]
        results[name] = (spec, solve_batch(spec, fld, st, warms, 4))
    rng = np.random.default_rng(21)
    syn = []
    for T, t0 in ((150, 0), (9, 2), (1, 0), (300, 5)):
        n, m = 3, 2
        tr = Trajectory(rng.normal(size=(T + 1, n)), rng.normal(size=(T, m)), rng.normal(size=T + 1) ** 2 * 10, t0)
        syn.append(SolveResult(tr, tr.cost, np.cumsum(rng.normal(size=T + 1)), rng.normal(size=(T + 1, n)), 1, True,
                               model=SimpleNamespace(m=m)))
    results["synthetic"] = (None, syn)
    for name, (spec, res) in results.items():
        data[f"ks_{name}_count"] = np.array(len(res))
        for i, r in enumerate(res):
            data.update(_solution_dict(f"ks_{name}_{i}", r))
        Ks = (1, 4, 10, 140, 400) if name == "synthetic" else (1, 5, 10, 1000)
        data[f"ks_{name}_Ks"] = np.array(Ks)
        for K in Ks:
            rows = [s for r in res for s in R_ilqr.kstep_targets(r, K)]
            data.update(batch_dict(f"ks_{name}_K{K}", SampleBatch.from_samples(rows, 0)))
        n, m = res[0].traj.X.shape[1], res[0].traj.U.shape[1]
        cap = 37
        buf = ReplayBuffer(n=n, m=m, t_max=0, capacity=cap, model_name=name, k_lookahead=10)
        for r in res:
            buf.push_many(R_ilqr.kstep_targets(r, 10))
        with tempfile.TemporaryDirectory() as td:
            buf.dump(Path(td) / "b.trlb")
            data[f"ks_{name}_dump"] = np.frombuffer((Path(td) / "b.trlb").read_bytes(), dtype=np.uint8)
        data[f"ks_{name}_cap"] = np.array(cap)
    return data


def main():
    cfgs = configs()
    only = sys.argv[1:]
    builders = {"rollout": lambda: make_rollouts(cfgs), "nets": make_nets, "losses": lambda: make_losses(cfgs),
                "optim": make_optim, "select": lambda: make_select(cfgs), "buffer": make_buffer,
                "sampling": lambda: make_sampling(cfgs), "kstep": lambda: make_kstep(cfgs)}
    out = {name: fn() for name, fn in builders.items() if not only or name in only}
    for name, data in out.items():
        np.savez_compressed(HERE / f"{name}.npz", **data)
        print(name, len(data), "arrays", (HERE / f"{name}.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
