"""Replay producer on the GPU: `ReplayBuffer.push_kstep`
(csrc/kstep.cu, kstep_targets ilqr.py:358-407 + push_many buffer.py:108-130 in
one launch) and the TRLB dump / restore (buffer.py:142-168), through the C ABI,
against the golden fixtures the reference produced (tests/golden/kstep.npz:
real iLQR solutions of pointmass / dubins with t0 = 0 and t0 > 0, synthetic
solutions with windows past NumPy's 128-term pairwise block) and the oracle.

Tolerance: bit-exact (fp64 ring); fp32 ring = the reference rows rounded once.
"""

import numpy as np
import pytest

import golden_utils as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2602_19699_b200 import buffer as B_buffer  # noqa: E402
from oracle import buffer as O_buffer  # noqa: E402

COLS = O_buffer.COLUMNS


def ring_rows(buf):
    """Ring contents oldest first, float64 host."""
    order = (np.arange(len(buf)) + (buf._cursor - len(buf))) % buf.capacity
    return {k: c.to("cpu", torch.float64).numpy()[order] for k, c in zip(COLS, buf.cols)}


def dims(sols):
    return sols[0].traj.X.shape[1], sols[0].traj.U.shape[1]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", G.KSTEP_SETS)
def test_push_kstep_rows_match_reference(name, precision):
    d = G.load("kstep")
    sols = G.solutions(d, name)
    n, m = dims(sols)
    for K in d[f"ks_{name}_Ks"]:
        ref = G.batch(d, f"ks_{name}_K{K}")
        buf = B_buffer.ReplayBuffer(n, m, 0, capacity=len(ref.v_bar) + 5, precision=precision)
        assert buf.push_kstep(sols, int(K)) == len(ref.v_bar)
        got = ring_rows(buf)
        for k in COLS:
            want = getattr(ref, k)
            if precision == "fp32":
                want = want.astype(np.float32).astype(np.float64)
            np.testing.assert_array_equal(got[k], want, err_msg=f"K={K} {k}")


@pytest.mark.parametrize("name", G.KSTEP_SETS)
def test_push_kstep_wrapping_ring_and_dump(name, tmp_path):
    # per-solution pushes into a 37-row ring (wraps several times), then the
    # TRLB dump must be byte-identical to the reference's
    d = G.load("kstep")
    sols = G.solutions(d, name)
    n, m = dims(sols)
    buf = B_buffer.ReplayBuffer(n, m, 0, capacity=int(d[f"ks_{name}_cap"]), model_name=name, k_lookahead=10,
                                precision="fp64")
    for s in sols:
        buf.push_kstep([s], 10)
    buf.dump(tmp_path / "b.trlb")
    assert (tmp_path / "b.trlb").read_bytes() == d[f"ks_{name}_dump"].tobytes()


@pytest.mark.parametrize("cap", [1, 5, 37, 10_000])
def test_push_kstep_batch_eviction_matches_oracle(cap):
    # one push of every solution: FIFO eviction inside a single batch keeps the newest
    d = G.load("kstep")
    sols = G.solutions(d, "synthetic")
    n, m = dims(sols)
    ring = O_buffer.Ring(n, m, cap)
    ring.push_many({"xa": np.zeros((3, n + 1)), "u": np.zeros((3, m)), "v_bar": np.arange(3.0),
                    "v_bar_x": np.zeros((3, n)), "xa_plus_k": np.zeros((3, n + 1))})
    ring.push_many(O_buffer.concat_rows([O_buffer.kstep_rows(s.traj.X, s.traj.U, s.traj.step_costs, s.traj.t0,
                                                             s.V_bar, s.V_bar_x, 4) for s in sols]))
    buf = B_buffer.ReplayBuffer(n, m, 0, capacity=cap, precision="fp64")
    buf.push_many(B_buffer.SampleBatch(np.zeros((3, n + 1)), np.zeros((3, m)), np.arange(3.0), np.zeros((3, n)),
                                       np.zeros((3, n + 1)), 0))
    buf.push_kstep(sols, 4)
    assert (len(buf), buf._cursor) == (ring.size, ring.cursor)
    for k, c in zip(COLS, buf.cols):
        np.testing.assert_array_equal(c.cpu().numpy(), ring.cols[k])


def test_restore_roundtrip_and_minibatch(tmp_path):
    d = G.load("kstep")
    blob = d["ks_dubins_dump"].tobytes()
    (tmp_path / "r.trlb").write_bytes(blob)
    buf = B_buffer.ReplayBuffer.restore(tmp_path / "r.trlb", capacity=64, t_max=100, precision="fp64")
    name, n, m, k, rows = O_buffer.parse_dump(blob)
    assert (buf.model_name, buf.n, buf.m, buf.k_lookahead, len(buf)) == (name, n, m, k, rows["v_bar"].shape[0])
    got = ring_rows(buf)
    for c in COLS:
        np.testing.assert_array_equal(got[c], rows[c])
    buf.dump(tmp_path / "again.trlb")
    assert (tmp_path / "again.trlb").read_bytes() == blob
    ring = O_buffer.Ring(n, m, 64)
    ring.push_many(rows)
    g1, g2 = np.random.default_rng(5), np.random.default_rng(5)
    mb = buf.sample_minibatch(50, g1)
    ref = ring.gather(ring.draw_indices(50, g2))
    for c in COLS:
        np.testing.assert_array_equal(getattr(mb, c), ref[c])


def test_kstep_targets_single_and_errors():
    d = G.load("kstep")
    sols = G.solutions(d, "pointmass")
    s = sols[1]
    b = B_buffer.kstep_targets(s, 5)
    ref = O_buffer.kstep_rows(s.traj.X, s.traj.U, s.traj.step_costs, s.traj.t0, s.V_bar, s.V_bar_x, 5)
    for c in COLS:
        np.testing.assert_array_equal(getattr(b, c), ref[c])
    n, m = dims(sols)
    buf = B_buffer.ReplayBuffer(n, m, 0, capacity=500, precision="fp64")
    with pytest.raises(ValueError):
        buf.push_kstep(sols, 0)
    with pytest.raises(NotImplementedError):
        B_buffer.kstep_targets(s, 5, critic_eval=lambda st: (0.0, np.zeros(n)))
    from types import SimpleNamespace
    sc = np.array(s.traj.step_costs, float)
    sc[3] = np.inf
    bad = SimpleNamespace(traj=SimpleNamespace(X=s.traj.X, U=s.traj.U, step_costs=sc, t0=s.traj.t0),
                          V_bar=s.V_bar, V_bar_x=s.V_bar_x)
    with pytest.raises(ValueError):
        buf.push_kstep([bad], 5)
    assert len(buf) == 0
    assert buf.push_kstep([], 5) == 0
