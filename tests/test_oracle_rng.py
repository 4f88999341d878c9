"""Pins of the oracle's random draws (not gpu).

* Philox4x32-10 against cuRAND's own host-compiled curand_Philox4x32_10
  (library routine, independent of the oracle and of the CUDA path).
* Row mask: Eq. (mt) P:559-572 -- r = 1 selects all rows; E|S| = p/r within
  3 sigma; keyed by global row (sharding invariance); strictly ascending.
* Atom permutation (Alg. 4): a permutation; uniform over S_3.
* Column stream: each epoch is a bijection of [0, n).
"""
import subprocess

import numpy as np
import pytest

from oracle.philox import philox4x32_10
from oracle.streams import (mask_rows, mask_threshold, atom_permutation,
                            column_ids)


def test_philox_matches_curand_host(curand_philox_ref):
    rng = np.random.default_rng(123)
    n = 3000
    c = rng.integers(0, 2 ** 32, size=(n, 4), dtype=np.uint64)
    k = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64)
    # include structured counters the library actually uses
    c[:8] = [[0, 0, 0, 0], [1, 0, 0, 0], [0, 1, 1, 0], [5, 7, 1, 0],
             [2 ** 32 - 1] * 4, [0, 0, 2, 0], [3, 9, 3, 5], [2 ** 31, 1, 1, 1]]
    k[:8] = [[0, 0], [0, 0], [0, 0], [1, 0], [2 ** 32 - 1] * 2, [7, 9], [0, 1], [123, 456]]
    inp = "\n".join(" ".join(str(int(x)) for x in list(c[i]) + list(k[i]))
                    for i in range(n)) + "\n"
    res = subprocess.run([curand_philox_ref], input=inp, capture_output=True,
                         text=True, check=True)
    ref = np.array([[int(x) for x in line.split()] for line in res.stdout.splitlines()],
                   dtype=np.uint64)
    seeds = [int(k[i, 0]) | (int(k[i, 1]) << 32) for i in range(n)]
    for i in range(n):
        out = philox4x32_10(c[i, 0], c[i, 1], c[i, 2], c[i, 3], seeds[i])
        assert [int(o) for o in out] == [int(x) for x in ref[i]], i


def test_mask_threshold_values():
    assert mask_threshold(1.0) == 2 ** 32
    assert mask_threshold(2.0) == 2 ** 31
    assert mask_threshold(4.0) == 2 ** 30
    assert mask_threshold(12.0) == 357913941      # floor(4294967296/12)
    with pytest.raises(ValueError):
        mask_threshold(0.5)


def test_mask_r1_selects_everything():
    for t in (1, 2, 77):
        S = mask_rows(9, t, 1001, 1.0)
        assert np.array_equal(S, np.arange(1001))


def test_mask_expected_size_and_unbiasedness():
    p, r = 10000, 4.0
    sizes = np.array([mask_rows(3, t, p, r).size for t in range(1, 401)])
    sigma = np.sqrt(p * (1 / r) * (1 - 1 / r))
    # mean of 400 draws: standard error sigma / 20
    assert abs(sizes.mean() - p / r) < 3 * sigma / np.sqrt(sizes.size)
    # each row is selected with probability 1/r (E[M_t x] = x)
    counts = np.zeros(p)
    T = 300
    for t in range(1, T + 1):
        counts[mask_rows(11, t, p, r)] += 1
    freq = counts.sum() / (p * T)
    assert abs(freq - 1 / r) < 3 * np.sqrt((1 / r) * (1 - 1 / r) / (p * T))


def test_mask_sorted_and_shard_invariant():
    p, r = 5003, 3.0
    full = mask_rows(42, 17, p, r)
    assert np.all(np.diff(full) > 0)
    bounds = [0, 1000, 1001, 3333, p]
    parts = [mask_rows(42, 17, p, r, lo, hi) for lo, hi in zip(bounds[:-1], bounds[1:])]
    assert np.array_equal(np.concatenate(parts), full)


def test_mask_huge_r_can_be_empty():
    S = mask_rows(0, 1, 50, 1e9)
    assert S.size == 0


def test_atom_permutation_is_permutation_and_uniform():
    for k in (1, 2, 5, 70, 256):
        for t in (1, 2, 3):
            pi = atom_permutation(5, t, k)
            assert np.array_equal(np.sort(pi), np.arange(k))
    assert np.array_equal(atom_permutation(5, 1, 9, cyclic=True), np.arange(9))
    # uniform over the 6 permutations of 3 atoms
    counts = {}
    T = 6000
    for t in range(1, T + 1):
        key = tuple(atom_permutation(1, t, 3))
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 6
    exp = T / 6
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 20.5   # chi2(5) 0.999 quantile


def test_column_ids_bijection_per_epoch():
    for n in (1, 2, 7, 1000, 4097):
        ids = column_ids(8, n, 0, 3 * n)
        for e in range(3):
            assert np.array_equal(np.sort(ids[e * n:(e + 1) * n]), np.arange(n))
    a = column_ids(8, 1000, 0, 1000)
    b = column_ids(8, 1000, 1000, 1000)
    assert not np.array_equal(a, b)
    # offsets are consistent with a longer draw
    long = column_ids(8, 1000, 0, 2500)
    assert np.array_equal(long[1200:1300], column_ids(8, 1000, 1200, 100))
