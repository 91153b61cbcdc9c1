"""Seeded synthetic input generators shared by the tests, the oracle runs and bench.py.

This package holds NONE of the method's arithmetic (no blur, gradient, watershed or
waterfall step).  It only produces raw u8 images/volumes whose structure is shaped like the
paper's workloads; both the CUDA path and the oracle consume the same
bytes.  See DESIGN.md "Input recipe".
"""
from .generators import (  # noqa: F401
    CONFIGS,
    cameraman_like,
    disc_composite,
    knee_like,
    microct_like,
    hsi_batch,
    random_plateau_image,
    make_config_image,
)
