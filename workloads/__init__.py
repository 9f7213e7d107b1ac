"""Seeded synthetic workloads shared by the oracle, the tests and bench.py.

This package holds ONLY input recipes: camera/volume geometry parameter sets and
seeded volumes/vectors.  It contains none of the method's arithmetic (no optics
composition, no transport entries, no rotation factors); both `oracle/` and the
CUDA path consume these plain numbers independently.  Recipes follow
SURVEY.md §8(d) and are restated in DESIGN.md §"Input recipe".
"""
from .geometry import (  # noqa: F401
    CONFIGS, make_config, plenoptic_camera, single_camera, pose_yaw, pose_pitch, pose_yaw_pitch,
)
from .volumes import flame_volume, uniform_volume, normal_vector, uniform_vector  # noqa: F401
