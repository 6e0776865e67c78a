"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no rates, pairs, scaling,
fits, ranking or scoring). It only draws the Tier-1 profiler-like inputs the
method consumes (counters, cycles, runtimes, optimization bit positions) and
the explicit train/test group sets of the paper's Table 2 experiments, so the
oracle (`oracle/`) and the GPU path (`paper_1910_07776_b200/`) are fed the
same bytes.  Random split hashing is part of the method and
is implemented independently on each side, not here.
"""
from .synth import Dataset, generate, OPT_NAMES_C2, BH_OPTS, NB_OPTS
from .configs import CONFIGS, make_config, table2_scenarios

__all__ = ["Dataset", "generate", "OPT_NAMES_C2", "BH_OPTS", "NB_OPTS",
           "CONFIGS", "make_config", "table2_scenarios"]
