"""CPU oracle for the CACTO-BIC data-parallel hot path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 NumPy restatement of the reference `trajrl` algorithms
on the hot path (rollout, BIC select, Sobolev critic / actor / std losses,
Adam + Polyak, replay gather, start-state sampling).  Every function cites the
reference `file:line` it restates (paths relative to `pkg/src/trajrl/`).

It is the CHECKER, never the product:
  * only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
    `--impl reference` legs may import it;
  * `paper_2602_19699_b200` never imports it and has no CPU fallback.

Pinning: `tests/golden/make_golden.py` runs the real reference (importable
read-only in the build container) on seeded inputs and commits the outputs as
`tests/golden/*.npz`; `tests/test_oracle_golden.py` checks this oracle against
every fixture.  The synthetic AlienGO-like system (`oracle.aliengo`) has no
reference implementation: its rollouts/losses are pinned only through the
reference's own machinery running on the NumPy system registered via the
reference plug-in API (`register_system` / `register_cost`), see DESIGN.md.
"""

from . import envs, nets, select, buffer, rng  # noqa: F401
