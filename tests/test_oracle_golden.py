"""Pin the CPU oracle against the golden fixtures produced by the real reference.

Tolerances: the oracle restates the reference in float64 with the same
operation order except for BLAS/einsum blocking, so agreement is ~1e-12
relative (manipulator3 rollouts allow 1e-8: chaotic amplification of
last-bit differences between LAPACK `solve` paths).
"""

import numpy as np
import pytest

import golden_utils as G
from oracle import buffer as O_buffer
from oracle import envs as O_envs
from oracle import nets as O_nets
from oracle import rng as O_rng
from oracle import select as O_select


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


# -- rollouts ----------------------------------------------------------------

@pytest.mark.parametrize("name", G.SYSTEMS)
@pytest.mark.parametrize("tag", ["init", "trained"])
def test_rollout_matches_reference(name, tag):
    d = G.load("rollout")
    spec, fld = G.spec(d, f"{name}_spec"), G.field(d, f"{name}_field")
    key = f"{name}_{tag}"
    actor = G.net(d, f"{key}_actor")
    tol = 1e-8 if name == "manipulator3" else 1e-11
    for i, (x0, t0) in enumerate(zip(d[f"{key}_x0"], d[f"{key}_t0"])):
        T = spec.t_max - int(t0)
        X, U, sc = O_nets.actor_rollout(actor, spec, x0, int(t0), T, fld)
        assert _rel(X, d[f"{key}_X"][i, :T + 1]) < tol
        assert _rel(U, d[f"{key}_U"][i, :T]) < tol
        assert _rel(sc, d[f"{key}_step_costs"][i, :T + 1]) < tol
        assert abs(sc.sum() - d[f"{key}_cost"][i]) <= tol * max(1.0, abs(d[f"{key}_cost"][i]))


@pytest.mark.parametrize("name", ["pointmass", "dubins"])
def test_batched_rollout_matches_per_start(name):
    d = G.load("rollout")
    spec, fld = G.spec(d, f"{name}_spec"), G.field(d, f"{name}_field")
    key = f"{name}_trained"
    x0 = d[f"{key}_x0"][:10]
    X, U, sc, cost = O_nets.actor_rollout_batch(G.net(d, f"{key}_actor"), spec, x0, 0, spec.t_max, fld)
    assert _rel(X, d[f"{key}_X"][:10]) < 1e-11
    assert _rel(cost, d[f"{key}_cost"][:10]) < 1e-11


def test_rollout_without_field_has_zero_costs():
    d = G.load("rollout")
    spec = G.spec(d, "dubins_spec")
    X, U, sc = O_nets.actor_rollout(G.net(d, "dubins_init_actor"), spec, d["dubins_init_x0"][0],
                                    0, spec.t_max)
    np.testing.assert_array_equal(sc, d["dubins_nofield_step_costs"])
    assert _rel(U, d["dubins_nofield_U"]) < 1e-12


def test_rollout_rejects_horizon_overflow():
    d = G.load("rollout")
    spec = G.spec(d, "pointmass_spec")
    with pytest.raises(ValueError):
        O_nets.actor_rollout(G.net(d, "pointmass_init_actor"), spec, np.zeros(4), 30, 31)


# -- forward / input gradient -----------------------------------------------------

@pytest.mark.parametrize("key", ["lin3", "tanh", "std", "lin1", "tanh3", "single"])
def test_forward_and_jacobian(key):
    d = G.load("nets")
    net = G.net(d, f"fwd_{key}")
    x = d[f"fwd_{key}_x"]
    assert _rel(O_nets.mlp_forward(net, x), d[f"fwd_{key}_y"]) < 1e-13
    assert _rel(O_nets.mlp_input_gradient(net, x), d[f"fwd_{key}_jac"]) < 1e-12
    if f"fwd_{key}_v" in d:
        v, g = O_nets.value_and_state_grad(net, x)
        assert _rel(v, d[f"fwd_{key}_v"]) < 1e-13
        assert _rel(g, d[f"fwd_{key}_g"]) < 1e-12


# -- losses ---------------------------------------------------------------------

@pytest.mark.parametrize("key", ["b64", "b200"])
@pytest.mark.parametrize("boot", [0, 1])
def test_critic_loss(key, boot):
    d = G.load("losses")
    critic, target = G.net(d, "critic_net"), G.net(d, "critic_target")
    batch = G.batch(d, f"critic_{key}")
    loss, grads = O_nets.critic_loss(critic, target if boot else None, batch, 0.7, bool(boot))
    assert loss == pytest.approx(float(d[f"critic_{key}_boot{boot}_loss"]), rel=1e-12)
    for g, ref in zip(grads, G.grads(d, f"critic_{key}_boot{boot}", 8)):
        assert _rel(g, ref) < 1e-10


def test_critic_loss_small_odd_shape():
    d = G.load("losses")
    loss, grads = O_nets.critic_loss(G.net(d, "critic_small_net"), G.net(d, "critic_small_target"),
                                     G.batch(d, "critic_small"), 0.5, True)
    assert loss == pytest.approx(float(d["critic_small_loss"]), rel=1e-12)
    for g, ref in zip(grads, G.grads(d, "critic_small", 6)):
        assert _rel(g, ref) < 1e-10


@pytest.mark.parametrize("key", ["b64", "b200"])
def test_std_loss(key):
    d = G.load("losses")
    loss, grads = O_nets.std_critic_loss(G.net(d, "std_net"), G.net(d, "critic_net"),
                                         G.batch(d, f"critic_{key}"))
    assert loss == pytest.approx(float(d[f"std_{key}_loss"]), rel=1e-12)
    for g, ref in zip(grads, G.grads(d, f"std_{key}", 8)):
        assert _rel(g, ref) < 1e-10


@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3", "aliengo_lipm"])
def test_actor_loss(name):
    d = G.load("losses")
    r = G.load("rollout")
    spec, fld = G.spec(r, f"{name}_spec"), G.field(r, f"{name}_field")
    loss, grads, skipped = O_nets.actor_loss(G.net(d, f"actor_{name}_actor"),
                                             G.net(d, f"actor_{name}_critic"), spec, fld,
                                             d[f"actor_{name}_xa"])
    assert skipped == int(d[f"actor_{name}_skipped"])
    assert loss == pytest.approx(float(d[f"actor_{name}_loss"]), rel=1e-11)
    for g, ref in zip(grads, G.grads(d, f"actor_{name}", 8)):
        assert _rel(g, ref) < 1e-9


# -- optimizer --------------------------------------------------------------------

def test_adam_sequence_bitwise():
    d = G.load("optim")
    p = [d["adam_p0_0"], d["adam_p0_1"]]
    m = [np.zeros_like(x) for x in p]
    v = [np.zeros_like(x) for x in p]
    for k in range(5):
        p, m, v = O_nets.adam_step(p, m, v, [d[f"adam_g{k}_0"], d[f"adam_g{k}_1"]], k, 3e-3)
        np.testing.assert_array_equal(p[0], d[f"adam_p{k + 1}_0"])
        np.testing.assert_array_equal(p[1], d[f"adam_p{k + 1}_1"])


def test_polyak_bitwise():
    d = G.load("optim")
    mix = O_nets.polyak(G.net(d, "polyak_a").flat_params(), G.net(d, "polyak_b").flat_params(), 0.25)
    for a, b in zip(mix, G.grads(d, "polyak_mix", 4)):
        np.testing.assert_array_equal(a, b)


# -- select / sampling / buffer ------------------------------------------------------

@pytest.mark.parametrize("name", ["pointmass", "dubins", "manipulator3"])
def test_select_order_bitwise(name):
    d = G.load("select")
    cands = d[f"select_{name}_cands"]
    scores = O_select.std_scores(G.net(d, f"select_{name}_std"), O_select.augmented(cands))
    assert _rel(scores, d[f"select_{name}_scores"]) < 1e-13
    np.testing.assert_array_equal(O_select.select_order(d[f"select_{name}_scores"], 75),
                                  d[f"select_{name}_order"])


def test_select_ties_nan_signed_zero():
    d = G.load("select")
    np.testing.assert_array_equal(O_select.select_order(d["select_ties_vals"], 12),
                                  d["select_ties_order"])


def test_select_rejects_keep_too_large():
    with pytest.raises(ValueError):
        O_select.select_order(np.zeros(3), 4)


@pytest.mark.parametrize("name", G.SYSTEMS)
def test_sample_initial_states_bitwise(name):
    d, r = G.load("sampling"), G.load("rollout")
    spec = G.spec(r, f"{name}_spec")
    x = O_envs.sample_initial_states(spec, 40, int(d[f"sample_{name}_seed"]))
    np.testing.assert_array_equal(x, d[f"sample_{name}_x"])


def test_pcg64_uniform_recipe():
    d, r = G.load("sampling"), G.load("rollout")
    spec = G.spec(r, "dubins_spec")
    lo, hi = O_envs.region_box(spec)
    u = O_rng.uniform(int(d["sample_dubins_seed"]), 40 * 5).reshape(40, 5)
    np.testing.assert_array_equal(u * (hi - lo) + lo, d["sample_dubins_x"])


def test_buffer_ring_and_minibatches_bitwise():
    d = G.load("buffer")
    rows = G.batch(d, "buf_rows")
    ring = O_buffer.Ring(3, 2, int(d["buf_capacity"]))
    cols = {k: getattr(rows, k) for k in O_buffer.COLUMNS}
    ring.push_many({k: v[:40] for k, v in cols.items()})
    ring.push_many({k: v[40:] for k, v in cols.items()})
    g = np.random.default_rng(int(d["buf_rng_seed"]))
    for mb, bsz in (("buf_mb1", 64), ("buf_mb2", 7)):
        got = ring.gather(ring.draw_indices(bsz, g))
        ref = G.batch(d, mb)
        for k in O_buffer.COLUMNS:
            np.testing.assert_array_equal(got[k], getattr(ref, k))


def test_lemire_replay_matches_generator():
    d = G.load("buffer")
    seed = int(d["buf_rng_seed"])
    raws = O_rng.raw_stream(seed, 64)
    idx = O_rng.lemire_indices(raws, 50, 64)
    np.testing.assert_array_equal(idx, np.random.default_rng(seed).integers(0, 50, 64))


# -- replay producer: kstep_targets + push_many + TRLB dump -------

@pytest.mark.parametrize("name", G.KSTEP_SETS)
def test_kstep_rows_bitwise(name):
    d = G.load("kstep")
    sols = G.solutions(d, name)
    for K in d[f"ks_{name}_Ks"]:
        got = O_buffer.concat_rows([O_buffer.kstep_rows(s.traj.X, s.traj.U, s.traj.step_costs, s.traj.t0,
                                                        s.V_bar, s.V_bar_x, int(K)) for s in sols])
        ref = G.batch(d, f"ks_{name}_K{K}")
        for k in O_buffer.COLUMNS:
            np.testing.assert_array_equal(got[k], getattr(ref, k), err_msg=f"K={K} {k}")


@pytest.mark.parametrize("name", G.KSTEP_SETS)
def test_kstep_ring_dump_bitwise(name):
    d = G.load("kstep")
    sols = G.solutions(d, name)
    n, m = sols[0].traj.X.shape[1], sols[0].traj.U.shape[1]
    ring = O_buffer.Ring(n, m, int(d[f"ks_{name}_cap"]))
    for s in sols:
        ring.push_many(O_buffer.kstep_rows(s.traj.X, s.traj.U, s.traj.step_costs, s.traj.t0, s.V_bar, s.V_bar_x, 10))
    blob = O_buffer.dump_bytes(ring, name, 10)
    assert blob == d[f"ks_{name}_dump"].tobytes()
    got_name, gn, gm, gk, rows = O_buffer.parse_dump(blob)
    assert (got_name, gn, gm, gk) == (name, n, m, 10)
    assert rows["v_bar"].shape[0] == ring.size


def test_kstep_rejects_bad_window():
    with pytest.raises(ValueError):
        O_buffer.kstep_rows(np.zeros((3, 2)), np.zeros((2, 1)), np.zeros(3), 0, np.zeros(3), np.zeros((3, 2)), 0)
    with pytest.raises(ValueError):
        O_buffer.parse_dump(b"XXXX" + bytes(40))
