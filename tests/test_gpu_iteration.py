"""One CACTO-BIC iteration end to end (iteration.run_iteration, the drop-in for
trajrl.trainer.run_iteration trainer.py:168-255) against the reference's own
iteration on a small pointmass config, in fp64 mode.

Iteration 1 has naive (zero) warm starts, so the TO solutions -- and therefore
the replay rows the device producer (cacto_kstep_push) writes -- must be
bit-identical to the reference's host ring; the update losses agree to 1e-9.
Iteration 2 runs BIC selection, warm-start rollouts, TO, the producer and the
update loop on top: replay rows and losses agree to 1e-6 (the rollouts differ
from NumPy's in the last bits, and iLQR amplifies that a little).

Needs the reference package (baseline/_ref, installed by DESIGN.md's recipe, or
/root/reference in the build container); skipped without it.
"""

import copy
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (p / "trajrl").exists():
        sys.path.insert(0, str(p))
        break
trajrl = pytest.importorskip("trajrl")
import trajrl.trainer as T  # noqa: E402

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import iteration, specs  # noqa: E402


@pytest.fixture(autouse=True)
def fp64():
    old = P.get_precision()
    P.set_precision("fp64")
    yield
    P.set_precision(old)


def small_cfg():
    spec, fld = specs.config("pointmass")
    model = trajrl.envs.ModelSpec(**{k: getattr(spec, k) for k in ("name", "n", "m", "dt", "t_max", "u_max",
                                                                   "workspace", "hard_region", "extra")})
    field = trajrl.envs.CostField(target=fld.target, obstacles=tuple(
        trajrl.envs.Ellipse(o.center, o.semi_axes, o.angle) for o in fld.obstacles),
        obstacle_weight=fld.obstacle_weight, target_reward_weight=fld.target_reward_weight,
        target_reward_radius=fld.target_reward_radius, control_weight=fld.control_weight,
        distance_weight=fld.distance_weight)
    return T.TrainConfig(model=model, field=field, n_episodes=8, episode_fraction=0.5, candidate_multiplier=4,
                         m_updates=6, k_lookahead=10, minibatch=16, iterations=2, seed=3, bic=True, eval_count=4,
                         eval_use_to=False, buffer_capacity=1 << 12, reg_eps=1e-6, tol=1e-6, max_iter_first=3,
                         max_iter_later=2, workers=1)


def ring(buf):
    order = (np.arange(len(buf)) + (buf._cursor - len(buf))) % buf.capacity
    if hasattr(buf, "cols"):
        return [c.to("cpu", torch.float64).numpy()[order] for c in buf.cols]
    return [a[order] for a in (buf._xa, buf._u, buf._v, buf._vx, buf._xk)]


def test_iteration_matches_reference():
    state = T.TrainerState(small_cfg())
    ref = copy.deepcopy(state)
    ref, r1 = T.run_iteration(ref, 1)
    state, g1 = iteration.run_iteration(state, 1, trajrl)
    assert len(state.buffer) == len(ref.buffer) > 0
    for a, b in zip(ring(state.buffer), ring(ref.buffer)):
        np.testing.assert_array_equal(a, b)
    assert g1.episodes_cum == r1.episodes_cum
    assert g1.to_cost_mean == r1.to_cost_mean
    np.testing.assert_allclose(g1.critic_loss_mean, r1.critic_loss_mean, rtol=1e-9)
    np.testing.assert_allclose(g1.std_loss_mean, r1.std_loss_mean, rtol=1e-9)
    np.testing.assert_allclose(g1.eval_mean_cost, r1.eval_mean_cost, rtol=1e-9)

    ref, r2 = T.run_iteration(ref, 2)
    state, g2 = iteration.run_iteration(state, 2, trajrl)
    assert len(state.buffer) == len(ref.buffer)
    for a, b in zip(ring(state.buffer), ring(ref.buffer)):
        np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(g2.to_cost_mean, r2.to_cost_mean, rtol=1e-6)
    np.testing.assert_allclose(g2.critic_loss_mean, r2.critic_loss_mean, rtol=1e-6)
    np.testing.assert_allclose(g2.std_loss_mean, r2.std_loss_mean, rtol=1e-6)


def test_installed_train_matches_reference():
    # `install(trajrl)` rebinds the reference's hot functions and run_iteration;
    # trajrl.trainer.train (trainer.py:283-330: calibration, iterations, the
    # actor-warm-start calibration after iteration 1) then runs on the B200
    cfg = small_cfg()
    from dataclasses import replace
    cfg = replace(cfg, max_iter_first=None, max_iter_later=None, calibration_probes=10, calibration_cap=8)
    a_ref, c_ref, s_ref, reps_ref = T.train(cfg)
    uninstall = P.install(trajrl)
    try:
        a_gpu, c_gpu, s_gpu, reps_gpu = T.train(cfg)
    finally:
        uninstall()
    assert T.run_iteration is not None and T.run_iteration.__module__ == "trajrl.trainer"
    assert len(reps_gpu) == len(reps_ref) == cfg.iterations
    r1, g1 = reps_ref[0], reps_gpu[0]
    assert g1.to_cost_mean == r1.to_cost_mean   # naive warm starts: identical TO solutions
    for r, g in zip(reps_ref, reps_gpu):
        np.testing.assert_allclose(g.to_cost_mean, r.to_cost_mean, rtol=1e-6)
        np.testing.assert_allclose(g.critic_loss_mean, r.critic_loss_mean, rtol=1e-6)
        np.testing.assert_allclose(g.std_loss_mean, r.std_loss_mean, rtol=1e-6)
    for a, b in zip(a_gpu.weights + c_gpu.weights + s_gpu.weights, a_ref.weights + c_ref.weights + s_ref.weights):
        np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-8)
