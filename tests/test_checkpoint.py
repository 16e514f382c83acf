"""Checkpoint interchange (nets.py:428-464), CPU: the repo's load_checkpoint reads
a file the reference wrote (tests/golden/checkpoint_actor.json, made by
tests/golden/make_checkpoint_golden.py) and save_checkpoint writes it back byte
for byte; the resume state round-trips through JSON exactly."""

import json
from pathlib import Path

import numpy as np

from paper_2602_19699_b200 import nets

GOLD = Path(__file__).resolve().parent / "golden" / "checkpoint_actor.json"


def test_load_reference_checkpoint_and_write_same_bytes(tmp_path):
    mlp, meta = nets.load_checkpoint(GOLD)
    assert meta == {"kind": "actor", "model": "pointmass", "config_hash": "abc123"}
    assert [w.shape for w in mlp.weights] == [(16, 5), (16, 16), (2, 16)]
    assert mlp.head == "tanh" and mlp.activation == "elu"
    out = tmp_path / "actor.json"
    nets.save_checkpoint(out, mlp, "actor", "pointmass", "abc123")
    assert out.read_bytes() == GOLD.read_bytes()


def test_checkpoint_values_exact():
    doc = json.loads(GOLD.read_text())
    mlp, _ = nets.load_checkpoint(GOLD)
    for i, w in enumerate(mlp.weights):
        np.testing.assert_array_equal(w.reshape(-1), np.asarray(doc["weights"][i]))
    np.testing.assert_array_equal(mlp.in_half, np.asarray(doc["norm_half"]))


def test_generator_state_roundtrips_through_json():
    rng = np.random.default_rng(5)
    rng.integers(0, 100, 17)
    st = json.loads(json.dumps(rng.bit_generator.state))
    r2 = np.random.Generator(np.random.PCG64())
    r2.bit_generator.state = st
    np.testing.assert_array_equal(rng.integers(0, 1 << 20, 64), r2.integers(0, 1 << 20, 64))
