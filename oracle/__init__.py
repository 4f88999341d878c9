"""SOMF float64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import, call or execute
anything under ``oracle/``.  The product path (``paper_1701_05363_b200``)
never imports it and fails loudly when its CUDA library is missing.

It is a plain, slow, obviously correct implementation of what the SOMF hot
path computes, written from PAPER.md (arXiv 1701.05363) in float64:

  * ``philox``   Philox4x32-10 counter-based generator (the randomness the
                 method draws is keyed by counters so both sides can share it)
  * ``streams``  row mask M_t (Eq. mt), atom permutation (Alg. 4
                 line "permutation([1,k])"), column stream
  * ``prox``     elastic-net value / atom norm (Eq. 2), projection
                 onto the elastic-net ball (Alg. 4), code
                 regression (Eq. somf_alpha)
  * ``somf``     Alg. 3 with estimator (a) and Alg. 4
                 (P:853-871); full-row objective (Eq. 3)
  * ``omf``      Alg. 1, written separately, the r=1 reference

It shares no code with the CUDA path.  Each function cites the passage it
follows; the DESIGN.md "readings" table lists every interpretation taken where
the paper is silent or garbled.  Parity pins live in tests/test_oracle_*.py.
Functions without an independent pin say "parity unpinned" in their
docstring (none at present; the trajectory itself has no printed values in the
paper and is only sanity-checked).
"""
from .philox import philox4x32_10, PHILOX_M0, PHILOX_M1, PHILOX_W0, PHILOX_W1  # noqa: F401
from .streams import mask_rows, mask_threshold, atom_permutation, column_ids  # noqa: F401
from .prox import enet_value, enet_projection, solve_codes  # noqa: F401
from .somf import SomfOracle, OracleConfig, objective, surrogate_value  # noqa: F401
from .omf import OmfOracle  # noqa: F401
