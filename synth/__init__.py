"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no operator, no PaLS, no solve,
no Jacobian).  It only turns a workload description (BASELINE.json configs) into
plain arrays: grid sizes, physical constants, node indices of the point sources
and detectors, PaLS parameter vectors drawn from the stated distributions,
Rademacher sketch matrices and the Gaussian noise draws.  Every random number
the method consumes is drawn here and passed in as an input to both sides.
"""
from .configs import DOTConfig, CONFIGS, config_by_name  # noqa: F401
from .generate import (  # noqa: F401
    face_nodes,
    draw_params,
    rademacher,
    noise_draws,
    subspace_start,
    Workload,
    make_workload,
)
