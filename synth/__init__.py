"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This package holds NO arithmetic of the SOMF method (no masks, no codes, no
surrogate statistics, no projections): only the data the method is run on.
Both the oracle (``oracle/``) and the CUDA path consume what it produces;
neither imports the other.  The recipes follow the paper's workloads
(§V-A) and BASELINE.json's configs; DESIGN.md §3
states them.
"""
from .generators import (  # noqa: F401
    tiny_dictionary_learning,
    fmri_voxel_grid,
    fmri_dictionary,
    fmri_codes,
    fmri_matrix,
    fmri_stream,
    hyperspectral_patches,
    nmf_matrix,
    random_state_for_step,
)
