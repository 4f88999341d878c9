"""B200-native subsampled online matrix factorisation (SOMF, arXiv 1701.05363).

The hot path (Alg. 3 + Alg. 4 of the paper) is hand-written CUDA for sm_100a
in ``csrc/``, compiled into ``libsomf.so`` and exposed through the C ABI of
``include/somf.h``.  ``somf`` is the thin Python binding (same names).
"""
from ._lib import build, LIB_PATH  # noqa: F401
from .somf import (Somf, SomfError, mask_rows, atom_permutation, column_ids,  # noqa: F401
                   project_columns, lib, dist_reducer, device_view)

__all__ = ["Somf", "SomfError", "mask_rows", "atom_permutation", "column_ids",
           "project_columns", "build", "lib", "LIB_PATH", "dist_reducer", "device_view"]
