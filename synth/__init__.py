"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO cDMD arithmetic: it only draws videos (uint8, frame-major)
and names the BASELINE.json configurations.  Both sides of every parity test
receive the same bytes from here.
"""

from .scene import CONFIGS, Config, make_video, config_by_name  # noqa: F401
