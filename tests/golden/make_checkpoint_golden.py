"""Reference-written checkpoint fixture (run in the build container, where
/root/reference exists): trajrl.nets.save_checkpoint of a seeded actor ->
tests/golden/checkpoint_actor.json.  tests/test_checkpoint.py checks that this
repo's load_checkpoint reads it and save_checkpoint writes the same bytes."""
import os
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, str(Path(os.environ.get("CACTO_REFERENCE", "/root/reference")) / "pkg" / "src"))
from trajrl import nets as R_nets  # noqa: E402

rng = np.random.default_rng(11)
mlp = R_nets.init_mlp([5, 16, 16, 2], rng, head="tanh", out_scale=np.array([2.0, 1.5]),
                      in_center=np.array([0.1, 0.0, -0.2, 0.0, 0.0]), in_half=np.array([1.0, 2.0, 3.0, 4.0, 60.0]))
R_nets.save_checkpoint(Path(__file__).parent / "checkpoint_actor.json", mlp, "actor", "pointmass", "abc123")
