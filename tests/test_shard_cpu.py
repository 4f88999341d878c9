"""Row sharding on the CPU: world_size-2 gloo process groups.

Covers the N > 1 host logic without a GPU:
  * the reducer the library calls at every exchange point
    (paper_1701_05363_b200.somf.dist_reducer: SUM / MIN / MAX, float64 and
    the int32 float-bit encoding of the per-atom min / max), and
  * the exchange schedule itself: an oracle step whose rows are split over
    the ranks, combining exactly the quantities the CUDA path reduces
    ([beta | G], the radius sums, the per-atom projection sums), equals the
    unsharded oracle step.  Masks are keyed by the global row (reading R1), so
    each rank draws its own rows of the same mask.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# the reducer
# ---------------------------------------------------------------------------
def _reducer_body(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1701_05363_b200 import _lib
    from paper_1701_05363_b200.somf import dist_reducer
    red = dist_reducer()
    x = torch.tensor([1.5, -2.0, 3.25], dtype=torch.float64) * (rank + 1)
    red(x, _lib.OP_SUM)
    assert torch.equal(x, torch.tensor([1.5, -2.0, 3.25], dtype=torch.float64) * 3)
    # per-atom min above / max below travel as int32 bit patterns of floats >= 0
    vals = [np.float32(0.25), np.float32(3.0)] if rank == 0 else [np.float32(0.5), np.float32(np.inf)]
    bits = torch.tensor(np.array(vals, np.float32).view(np.int32))
    red(bits, _lib.OP_MIN)
    got = bits.numpy().view(np.float32)
    assert got[0] == np.float32(0.25) and got[1] == np.float32(3.0)
    mx = torch.tensor(np.array([np.float32(rank + 1.0), 0.0], np.float32).view(np.int32))
    red(mx, _lib.OP_MAX)
    assert mx.numpy().view(np.float32)[0] == np.float32(world)


def test_dist_reducer_gloo_world2():
    _run(2, _reducer_body)


def test_float_bits_order_is_int_order():
    """The int32 MIN/MAX over ranks is the float MIN/MAX for values >= 0
    (including the +inf 'no element' sentinel the kernels use)."""
    rng = np.random.default_rng(0)
    v = np.concatenate([np.abs(rng.standard_normal(1000)).astype(np.float32),
                        np.array([0.0, np.inf, 1e-38, 3e38], np.float32)])
    b = v.view(np.int32)
    order_f = np.argsort(v, kind="stable")
    order_i = np.argsort(b, kind="stable")
    assert np.array_equal(v[order_f], v[order_i])
    assert (b >= 0).all()


# ---------------------------------------------------------------------------
# the exchange schedule: sharded oracle step == unsharded oracle step
# ---------------------------------------------------------------------------
def _allreduce_np(a, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.ascontiguousarray(a, np.float64))
    dist.all_reduce(t, op=op)
    return t.numpy()


def _sharded_step(rank, world, p, k, eta, kw, X, D, Bbar, Cbar, n, t, out_path):
    """One SOMF step on rows [lo, hi): every sum over masked rows is a local
    partial plus an allreduce (the CUDA path's exchange points)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.prox import enet_projection, enet_value, solve_codes
    from oracle.streams import atom_permutation, mask_rows
    lo, hi = p * rank // world, p * (rank + 1) // world
    seed, r, u, mu, lam, nu = kw["seed"], kw["r"], kw["u"], kw["mu"], kw["lam"], kw["nu"]
    t += 1
    w = float(t) ** (-u)
    S = mask_rows(seed, t, p, r, lo, hi)                       # global rows of my shard
    DS, XS = D[S], X[S]
    bg = np.concatenate([(r * DS.T @ XS).ravel(), (r * DS.T @ DS).ravel()])
    bg = _allreduce_np(bg)                                     # exchange 1: [beta | G]
    beta, G = bg[:k * eta].reshape(k, eta), bg[k * eta:].reshape(k, k)
    A = solve_codes(G, beta, lam, nu, False, tol=1e-12)       # replicated
    Cbar = (1.0 - w) * Cbar + (w / eta) * (A @ A.T)           # replicated
    Bbar = Bbar.copy()
    Bbar[S] = (1.0 - w) * Bbar[S] + (w / eta) * (XS @ A.T)
    D = D.copy()
    DS = D[S].copy()
    BS = Bbar[S]
    # exchange 2: radius sums of every atom
    rs = np.concatenate([np.abs(DS).sum(axis=0), (DS * DS).sum(axis=0)])
    rs = _allreduce_np(rs)
    n = n.copy()
    rho = np.maximum(0.0, n + (1 - mu) * rs[:k] + 0.5 * mu * rs[k:])
    dmax = max(1.0, float(np.max(np.diag(Cbar))))
    for j in atom_permutation(seed, t, k):
        if Cbar[j, j] <= 1e-12 * dmax:
            continue
        uj = DS[:, j] + (BS[:, j] - DS @ Cbar[:, j]) / Cbar[j, j]
        # exchange 3: the projection of the column needs its global threshold;
        # the reference here gathers the column (the kernels reduce sums)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([uj.size], dtype=torch.int64))
        mx = int(max(s.item() for s in sizes))
        buf = torch.zeros(mx, dtype=torch.float64)
        buf[:uj.size] = torch.from_numpy(uj)
        parts = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, buf)
        full = np.concatenate([parts[i][:int(sizes[i].item())].numpy() for i in range(world)])
        dfull = enet_projection(full, rho[j], mu, False)
        off = sum(int(sizes[i].item()) for i in range(rank))
        DS[:, j] = dfull[off:off + uj.size]
        n[j] = rho[j] - enet_value(dfull, mu)
    D[S] = DS
    np.savez(out_path + f".{rank}.npz", D=D[lo:hi], Bbar=Bbar[lo:hi], Cbar=Cbar, n=n, A=A)


@pytest.mark.parametrize("mu", [0.0, 1.0, 0.5])
def test_sharded_oracle_step_equals_unsharded(tmp_path, mu):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    from oracle.somf import SomfOracle, OracleConfig
    p, k, eta = 1201, 12, 16
    kw = dict(lam=0.05, nu=1.0, mu=mu, r=4.0, u=0.917, seed=5)
    X, _, _ = synth.tiny_dictionary_learning(p=p, n=k + 4 * eta, seed=2)
    ora = SomfOracle(OracleConfig(p=p, k=k, eta=eta, **kw))
    ora.set_components(X[:, :k])
    for s in range(3):
        ora.partial_fit(X[:, k + s * eta:k + (s + 1) * eta])
    state = (ora.D.copy(), ora.Bbar.copy(), ora.Cbar.copy(), ora.n.copy(), ora.t)
    batch = X[:, k + 3 * eta:k + 4 * eta]
    out = ora.partial_fit(batch)
    out_path = str(tmp_path / "step")
    _run(2, _sharded_step, p, k, eta, kw, batch, *state, out_path)
    parts = [np.load(out_path + f".{i}.npz") for i in range(2)]
    D = np.concatenate([q["D"] for q in parts])
    B = np.concatenate([q["Bbar"] for q in parts])
    np.testing.assert_allclose(D, ora.D, rtol=0, atol=1e-12)
    np.testing.assert_allclose(B, ora.Bbar, rtol=0, atol=1e-12)
    for q in parts:       # replicated state identical on every rank
        np.testing.assert_allclose(q["Cbar"], ora.Cbar, rtol=0, atol=1e-12)
        np.testing.assert_allclose(q["n"], ora.n, rtol=0, atol=1e-10)
        np.testing.assert_allclose(q["A"], out["A"], rtol=0, atol=1e-10)
    np.testing.assert_array_equal(parts[0]["Cbar"], parts[1]["Cbar"])
