"""Seeded synthetic inputs + config registry, shared by the oracle and the CUDA path.

Holds no arithmetic of the method (see generators.py docstring)."""
from .configs import CONFIGS, Config, get  # noqa: F401
from .generators import (make_inputs, subsample, small_subsample, check_rows, uniform_test_weights,  # noqa: F401
                         shard_range)
