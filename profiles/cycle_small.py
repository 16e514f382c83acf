"""A few B=128 update cycles (pointmass shapes) for ncu captures."""
import sys
sys.path.insert(0, "profiles")
import engine_cycle  # noqa: E402
engine_cycle.main(M=4)
