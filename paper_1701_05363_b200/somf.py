"""Thin Python binding of the SOMF C ABI (include/somf.h): same names,
argument marshalling only.  PyTorch supplies device memory and the stream.

Every array crossing the ABI is a contiguous float32 (codes / data) or
float64 (Cbar, slack norms) torch tensor; data matrices are row-major
``rows x m`` (feature-major), exactly as the C ABI documents.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

_L = None


def lib():
    global _L
    if _L is None:
        _L = _lib.load()
    return _L


class SomfError(RuntimeError):
    pass


def _check(status: int, handle=None):
    if status != 0:
        msg = lib().somf_status_string(status).decode()
        if handle is not None:
            detail = lib().somf_last_error(handle).decode()
            if detail:
                msg += ": " + detail
        raise SomfError(msg)


def _ptr(t: torch.Tensor) -> C.c_void_p:
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


B_MODES = {"masked": 0, "unbiased": 1, "full": 2}
# kernel selection (somf_config *_kernel fields, include/somf.h)
CONTRACT_KERNELS = {"auto": 0, "tc": 1, "slice": 2, "tiled": 3, "generic": 4}
BBAR_KERNELS = {"auto": 0, "tc": 1, "slice": 2, "tiled": 3, "generic": 4}
CODES_KERNELS = {"auto": 0, "ridge": 1, "cd_jump": 2, "cd": 3}


class _CudaArray:
    """Zero-copy view of a device buffer (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


def device_view(ptr: int, n: int, dtype: int, device) -> torch.Tensor:
    """torch view of `n` float64 (dtype 0) or int32 (dtype 1) values at a device pointer."""
    return torch.as_tensor(_CudaArray(ptr, n, "<f8" if dtype == _lib.DT_F64 else "<i4"), device=device)


def dist_reducer(group=None):
    """Reducer over a torch.distributed process group (NCCL on GPUs, gloo on
    CPU tensors): the allreduce of the row-sharded step (somf_set_reducer)."""
    import torch.distributed as dist
    ops = {_lib.OP_SUM: dist.ReduceOp.SUM, _lib.OP_MIN: dist.ReduceOp.MIN, _lib.OP_MAX: dist.ReduceOp.MAX}

    def reduce(buf: torch.Tensor, op: int):
        dist.all_reduce(buf, op=ops[op], group=group)
    return reduce


class Somf:
    """One SOMF learner (a handle of the C ABI) owning rows [row_lo, row_hi)."""

    def __init__(self, p: int, k: int, eta: int, lam: float = 0.1, nu: float = 1.0,
                 pos_code: bool = False, mu: float = 0.0, pos_dict: bool = False,
                 r: float = 1.0, u: float = 0.917, b_mode: str = "masked",
                 perm_cyclic: bool = False, cd_tol: float = 1e-7, cd_max_sweeps: int = 4000,
                 seed: int = 0, row_lo: int = 0, row_hi: int = 0, device: int = 0,
                 stream=None, debug: bool = False, bcd_kernel: str = "auto",
                 contract_kernel: str = "auto", bbar_kernel: str = "auto", codes_kernel: str = "auto",
                 bcd_lam_tol: float = 0.0, bcd_copies: int = 0,
                 estimator: str = "a", n_samples: int = 0, v: float = 0.751, bcd_tile_rows: int = 0,
                 bcd_group: int = 0):
        L = lib()
        cfg = _lib.SomfConfig()
        L.somf_config_default(C.byref(cfg))
        cfg.p, cfg.k, cfg.eta = p, k, eta
        cfg.lambda_, cfg.nu, cfg.pos_code = lam, nu, int(pos_code)
        cfg.mu, cfg.pos_dict = mu, int(pos_dict)
        cfg.r, cfg.u = r, u
        cfg.b_mode = B_MODES[b_mode]
        cfg.perm_cyclic = int(perm_cyclic)
        cfg.cd_tol, cfg.cd_max_sweeps = cd_tol, cd_max_sweeps
        cfg.seed = seed
        cfg.row_lo, cfg.row_hi = row_lo, row_hi
        cfg.device = device
        self.device = torch.device("cuda", device)
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        cfg.stream = _stream_ptr(self.stream)
        cfg.debug = int(debug)
        cfg.bcd_kernel = {"auto": 0, "global": 1, "onchip": 2, "newton": 3, "big": 4}[bcd_kernel]
        cfg.contract_kernel = CONTRACT_KERNELS[contract_kernel]
        cfg.bbar_kernel = BBAR_KERNELS[bbar_kernel]
        cfg.codes_kernel = CODES_KERNELS[codes_kernel]
        cfg.bcd_lam_tol = bcd_lam_tol
        cfg.bcd_copies = bcd_copies
        cfg.estimator = {"a": 0, "b": 1, "c": 2}[estimator]
        cfg.n_samples = n_samples
        cfg.v = v
        cfg.bcd_tile_rows = bcd_tile_rows
        cfg.bcd_group = bcd_group
        h = C.c_void_p()
        st = L.somf_create(C.byref(cfg), C.byref(h))
        if st != 0:
            msg = L.somf_last_error(h).decode() if h.value else ""
            if h.value:
                L.somf_destroy(h)
            raise SomfError(f"somf_create: {L.somf_status_string(st).decode()} {msg}")
        self._h = h
        self.cfg = cfg
        self.p, self.k, self.eta = p, k, eta
        self.rows = (row_hi or p) - row_lo

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _L is not None:
            _L.somf_destroy(h)
            self._h = None

    # -- checks -------------------------------------------------------------
    def _dev_f32(self, X: torch.Tensor, rows: int, name: str) -> torch.Tensor:
        if X.dtype != torch.float32 or X.dim() != 2 or X.shape[0] != rows:
            raise ValueError(f"{name} must be a float32 {rows} x m tensor")
        if X.stride(1) != 1:
            raise ValueError(f"{name} must be row-major")
        if not X.is_cuda and not X.is_pinned():
            raise ValueError(f"{name} must live on the GPU or in pinned host memory")
        return X

    # -- C ABI --------------------------------------------------------------------
    def set_components(self, D0: torch.Tensor):
        D0 = self._dev_f32(D0, self.rows, "D0")
        _check(lib().somf_set_components(self._h, C.c_void_p(D0.data_ptr()), D0.stride(0)), self._h)

    def partial_fit(self, X: torch.Tensor):
        X = self._dev_f32(X, self.rows, "X")
        if X.shape[1] != self.eta:
            raise ValueError("X must have eta columns")
        _check(lib().somf_partial_fit(self._h, C.c_void_p(X.data_ptr()), X.stride(0)), self._h)

    def partial_fit_ids(self, X: torch.Tensor, ids):
        """Estimators (b) / (c): X's columns are the samples ``ids`` (int64,
        host array or CUDA tensor, distinct within the batch)."""
        X = self._dev_f32(X, self.rows, "X")
        if X.shape[1] != self.eta:
            raise ValueError("X must have eta columns")
        if isinstance(ids, torch.Tensor):
            ids_t = ids.to(torch.int64).contiguous()
            ptr = C.c_void_p(ids_t.data_ptr())
        else:
            ids_t = np.ascontiguousarray(ids, dtype=np.int64)
            ptr = ids_t.ctypes.data_as(C.c_void_p)
        if ids_t.shape[0] != self.eta:
            raise ValueError("ids must hold eta sample ids")
        _check(lib().somf_partial_fit_ids(self._h, C.c_void_p(X.data_ptr()), X.stride(0), ptr), self._h)

    def next_mask(self, want_indices: bool = True):
        q = C.c_int64()
        buf = np.empty(self.rows, dtype=np.int32) if want_indices else None
        _check(lib().somf_next_mask(self._h, C.byref(q),
                                    buf.ctypes.data_as(C.c_void_p) if want_indices else None), self._h)
        return (q.value, buf[:q.value].copy()) if want_indices else (q.value, None)

    def partial_fit_masked(self, X_M: torch.Tensor):
        if X_M.dtype != torch.float32 or X_M.dim() != 2 or X_M.stride(1) != 1:
            raise ValueError("X_M must be a row-major float32 q x eta tensor")
        _check(lib().somf_partial_fit_masked(self._h, C.c_void_p(X_M.data_ptr()), X_M.stride(0)), self._h)

    def get_codes(self, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self.k, self.eta), dtype=torch.float32, device=self.device)
        _check(lib().somf_get_codes(self._h, _ptr(out)), self._h)
        return out

    def transform(self, X: torch.Tensor) -> torch.Tensor:
        X = self._dev_f32(X, self.rows, "X")
        m = X.shape[1]
        out = torch.empty((self.k, m), dtype=torch.float32, device=self.device)
        _check(lib().somf_transform(self._h, C.c_void_p(X.data_ptr()), X.stride(0), m, _ptr(out)), self._h)
        return out

    def objective(self, X: torch.Tensor) -> float:
        X = self._dev_f32(X, self.rows, "X")
        v = C.c_double()
        _check(lib().somf_objective(self._h, C.c_void_p(X.data_ptr()), X.stride(0), X.shape[1],
                                    C.byref(v)), self._h)
        return v.value

    def components(self) -> torch.Tensor:
        out = torch.empty((self.rows, self.k), dtype=torch.float32, device=self.device)
        _check(lib().somf_components(self._h, _ptr(out), self.k), self._h)
        return out

    def get_state(self):
        D = np.empty((self.rows, self.k), np.float32)
        B = np.empty((self.rows, self.k), np.float32)
        Cb = np.empty((self.k, self.k), np.float64)
        n = np.empty(self.k, np.float64)
        t = C.c_int64()
        _check(lib().somf_get_state(self._h, D.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
                                    Cb.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p),
                                    C.byref(t)), self._h)
        return dict(D=D, Bbar=B, Cbar=Cb, n=n, t=t.value)

    def set_state(self, D, Bbar, Cbar, n, t: int):
        D = np.ascontiguousarray(D, np.float32)
        B = np.ascontiguousarray(Bbar, np.float32)
        Cb = np.ascontiguousarray(Cbar, np.float64)
        n = np.ascontiguousarray(n, np.float64)
        _check(lib().somf_set_state(self._h, D.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
                                    Cb.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p), int(t)),
               self._h)

    PHASES = ("stage", "mask", "contract", "codes", "cbar", "bbar", "bcd")

    def profile_enable(self, on: bool = True):
        _check(lib().somf_profile_enable(self._h, int(on)), self._h)

    def profile_read(self):
        ms = np.zeros(len(self.PHASES), np.float64)
        nl = np.zeros(len(self.PHASES), np.int64)
        steps = C.c_int64()
        _check(lib().somf_profile_read(self._h, ms.ctypes.data_as(C.c_void_p), nl.ctypes.data_as(C.c_void_p),
                                       C.byref(steps)), self._h)
        return dict(ms=dict(zip(self.PHASES, ms.tolist())), launches=dict(zip(self.PHASES, nl.tolist())),
                    steps=steps.value)

    BCD_PHASES = ("setup", "recurrence", "stats", "barrier", "update", "finish", "writeback")

    def bcd_phase_cycles(self):
        v = np.zeros(248, np.int64)       # SOMF_PROF_SLOTS
        _check(lib().somf_bcd_phase_cycles(self._h, v.ctypes.data_as(C.c_void_p)), self._h)
        out = dict(zip(self.BCD_PHASES, v[:7].tolist()), launches=int(v[7]))
        # slot 8 + r: (frozen prefix F << 16) + unconverged atoms, summed over launches
        out["unconverged_per_round"] = (v[8:72] & 0xFFFF).tolist()
        out["first_unconverged_per_round"] = (v[8:72] >> 16).tolist()
        out["frozen_prefix_per_round"] = (v[8:72] >> 16).tolist()
        out["ridge"] = dict(zip(("load", "factor", "solve", "cbar_partial"), v[72:76].tolist()), inverse=int(v[79]))
        out["setup_split"] = dict(zip(("params", "gather", "permute"), v[76:79].tolist()))
        out["update_split"] = dict(zip(("ring_reset", "record_read"), v[80:82].tolist()))
        out["raw"] = v.tolist()
        out["contract"] = dict(zip(("issue", "rows_wait", "mma_wait", "transpose_split", "epilogue", "barrier",
                                    "reduce"), v[224:231].tolist()), mma_issue=int(v[241]),
                               launches=int(v[231]))
        out["bbar"] = dict(zip(("x_stage", "solver_wait", "codes_stage", "mma_issue", "cbar", "mma_wait", "epilogue"),
                               v[232:239].tolist()), launches=int(v[239]))
        # lasso / nonneg CD with support jumps (cd_as.cuh): totals over its columns
        out["cd"] = dict(zip(("columns", "sweeps", "face_solves", "face_size_sum", "sweep_cycles", "jump_cycles",
                              "face_size_max", "jumps_accepted"), v[84:92].tolist()))
        return out

    def set_reducer(self, fn):
        """Row sharding: fn(buf, op) combines the tensor `buf` (a zero-copy view
        of the handle's device buffer) over the ranks in place, op in
        _lib.OP_SUM / OP_MIN / OP_MAX, on the current stream (the handle's).
        fn=None restores the single-GPU path."""
        if fn is None:
            self._reducer_cb = None
            _check(lib().somf_set_reducer(self._h, None, None), self._h)
            return
        dev = self.device

        def cb(user, buf, count, dtype, op, stream):
            try:
                t = device_view(buf, count, dtype, dev)
                s = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.default_stream(dev)
                with torch.cuda.stream(s):
                    fn(t, op)
                return 0
            except Exception:          # noqa: BLE001 -- reported to the C side as a failed collective
                import traceback
                traceback.print_exc()
                return 1
        self._reducer_cb = _lib.REDUCE_FN(cb)
        _check(lib().somf_set_reducer(self._h, self._reducer_cb, None), self._h)

    @property
    def bcd_variant(self) -> str:
        return {1: "global", 2: "onchip", 3: "newton", 5: "big"}.get(lib().somf_bcd_variant(self._h), "?")

    def last_kernels(self):
        """Kernel variants of the last partial_fit (somf_last_kernels): names
        as in CONTRACT_KERNELS / CODES_KERNELS / BBAR_KERNELS."""
        v = np.zeros(8, np.int32)
        _check(lib().somf_last_kernels(self._h, v.ctypes.data_as(C.c_void_p)), self._h)
        inv = lambda d, x: {i: n for n, i in d.items()}.get(int(x), "none")  # noqa: E731
        return dict(contract=inv(CONTRACT_KERNELS, v[0]), codes=inv(CODES_KERNELS, v[1]),
                    bbar=inv(BBAR_KERNELS, v[2]),
                    bcd={1: "global", 2: "onchip", 3: "newton", 4: "sharded", 5: "big"}.get(int(v[3]), "none"),
                    bbar_complement=bool(v[4]), bcd_group=(int(v[5]), int(v[6])), bcd_pdl=bool(v[7]))

    def last_step_info(self):
        q, nred, w = C.c_int64(), C.c_int64(), C.c_double()
        _check(lib().somf_last_step_info(self._h, C.byref(q), C.byref(nred), C.byref(w)), self._h)
        return dict(q=q.value, bcd_reductions=nred.value, w=w.value)


# ---- stateless kernels ------------------------------------------------------
def mask_rows(seed: int, t: int, row_lo: int, row_hi: int, r: float, device: int = 0) -> np.ndarray:
    idx = torch.empty(max(1, row_hi - row_lo), dtype=torch.int32, device=f"cuda:{device}")
    q = C.c_int64()
    _check(lib().somf_mask_rows(seed, t, row_lo, row_hi, r, _ptr(idx), C.byref(q), _stream_ptr(None)))
    return idx[:q.value].cpu().numpy().astype(np.int64)


def atom_permutation(seed: int, t: int, k: int, cyclic: bool = False, device: int = 0) -> np.ndarray:
    perm = torch.empty(k, dtype=torch.int32, device=f"cuda:{device}")
    _check(lib().somf_atom_permutation(seed, t, k, int(cyclic), _ptr(perm), _stream_ptr(None)))
    return perm.cpu().numpy().astype(np.int64)


def column_ids(seed: int, n: int, s0: int, count: int, device: int = 0) -> torch.Tensor:
    ids = torch.empty(max(1, count), dtype=torch.int64, device=f"cuda:{device}")
    _check(lib().somf_column_ids(seed, n, s0, count, _ptr(ids), _stream_ptr(None)))
    return ids[:count]


def project_columns(U: torch.Tensor, radius: torch.Tensor, mu: float, positive: bool = False) -> torch.Tensor:
    if U.dtype != torch.float32 or not U.is_cuda or U.dim() != 2 or not U.is_contiguous():
        raise ValueError("U must be a contiguous float32 CUDA matrix")
    radius = radius.to(device=U.device, dtype=torch.float64).contiguous()
    out = torch.empty_like(U)
    _check(lib().somf_project_columns(_ptr(U), U.shape[0], U.shape[1], U.shape[1], _ptr(radius), mu,
                                      int(positive), _ptr(out), _stream_ptr(None)))
    return out
