"""Random draws of the method: row mask, atom order, column stream.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Counter layout (reading R1): Philox4x32-10 with key = seed and
counter (c0, c1, c2, c3) = (block, t_or_epoch, STREAM, hi).  STREAM separates
the draws: 1 = row mask, 2 = atom permutation, 3 = column stream.
"""
import math

import numpy as np

from .philox import philox4x32_10

STREAM_MASK = 1
STREAM_PERM = 2
STREAM_COLS = 3


def mask_threshold(r: float) -> int:
    """T(r) = floor(2^32 / r), evaluated in IEEE double (reading R2).

    A row is selected iff its uniform 32-bit word u satisfies u < T(r), which
    happens with probability T(r)/2^32 ~= 1/r: Eq. (mt), P:559-566,
    "P[M_t[j,j] = r] = 1/r".  For r = 1, T = 2^32 and every row is selected.
    """
    if not (r >= 1.0):
        raise ValueError("reduction factor r must be >= 1 (P:553-555)")
    return int(math.floor(4294967296.0 / float(r)))


def mask_rows(seed: int, t: int, p: int, r: float, row_lo: int = 0,
              row_hi: int | None = None) -> np.ndarray:
    """Ascending global indices of the rows selected by M_t in [row_lo, row_hi).

    Eq. (mt): each diagonal entry of M_t is r with probability 1/r
    and 0 otherwise, independently per row; P_t keeps the selected rows
    (P:573-577).  Row i uses word (i & 3) of the Philox block with counter
    (i >> 2, t, 1, i >> 34): the draw is keyed by the global row index, so a
    row-sharded run selects exactly the same rows (reading R1).
    """
    if row_hi is None:
        row_hi = p
    T = mask_threshold(r)
    rows = np.arange(row_lo, row_hi, dtype=np.int64)
    if rows.size == 0:
        return rows
    blk = rows >> 2
    words = philox4x32_10(blk & 0xFFFFFFFF, t, STREAM_MASK, blk >> 32, seed)
    lane = (rows & 3).astype(np.int64)
    w = np.choose(lane, words)
    return rows[w.astype(np.uint64) < np.uint64(T)]


def atom_permutation(seed: int, t: int, k: int, cyclic: bool = False) -> np.ndarray:
    """Atom visiting order of Alg. 4 ("for j in permutation([1,k])").

    Fisher-Yates from the top (reading R13): for w = 0 .. k-2, i = k-1-w,
    draw the Philox word number w of stream 2 at iteration t (block w >> 2,
    lane w & 3) and swap positions i and j = floor(word * (i+1) / 2^32).
    ``cyclic`` gives the identity order.
    """
    perm = np.arange(k, dtype=np.int64)
    if cyclic or k <= 1:
        return perm
    nw = k - 1
    blocks = np.arange((nw + 3) // 4, dtype=np.int64)
    words = philox4x32_10(blocks, t, STREAM_PERM, 0, seed)
    flat = np.stack(words, axis=1).reshape(-1)
    for w in range(nw):
        i = k - 1 - w
        j = (int(flat[w]) * (i + 1)) >> 32
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def _feistel_bits(n: int) -> int:
    b = max(2, int(math.ceil(math.log2(max(n, 2)))))
    return b + (b & 1)


def column_ids(seed: int, n: int, s0: int, count: int) -> np.ndarray:
    """Sample ids for stream positions s0 .. s0+count-1.

    The experiments "cycle randomly" through the n columns:
    position s belongs to epoch e = s // n and takes column pi_e(s mod n),
    where pi_e is a keyed bijection of [0, n): a 6-round balanced Feistel
    network on b bits (b even, 2^b >= n) with round function
    F(R) = Philox((R, e, 3, round))[0] mod 2^(b/2), restricted to [0, n) by
    cycle walking (reading R16).  Mini-batch t takes positions
    [(t-1) eta, t eta).
    """
    if n <= 0:
        raise ValueError("n must be positive")
    s = np.arange(s0, s0 + count, dtype=np.int64)
    epoch = s // n
    x = (s % n).astype(np.int64)
    b = _feistel_bits(n)
    half = b // 2
    hmask = (1 << half) - 1
    out = np.empty_like(x)
    todo = np.ones(x.size, dtype=bool)
    cur = x.copy()
    while todo.any():
        L = cur[todo] >> half
        R = cur[todo] & hmask
        ep = epoch[todo]
        for rnd in range(6):
            F = philox4x32_10(R, ep & 0xFFFFFFFF, STREAM_COLS, rnd, seed)[0]
            F = (F & np.uint64(hmask)).astype(np.int64)
            L, R = R, L ^ F
        y = (L << half) | R
        idx = np.flatnonzero(todo)
        cur[idx] = y
        done = y < n
        out[idx[done]] = y[done]
        todo[idx[done]] = False
    return out
