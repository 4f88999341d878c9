"""ctypes loader for libsomf.so (the C ABI declared in include/somf.h).

Argument marshalling only: every step of the SOMF path runs in the CUDA
kernels of ``csrc/``.  There is no fallback: if the shared library is missing
or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libsomf.so")
CSRC = os.path.join(HERE, "csrc")
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh"))) + [os.path.join(ROOT, "include", "somf.h")]


NT_KPTS = (16, 32, 48, 64, 72, 80, 96, 128)   # bcd_newton_inst.cu variants (one object each)
NB_KPTS = (72, 128, 192, 256)                  # bcd_big_inst.cu variants


def _units():
    """(name, source, extra flags) of every translation unit of libsomf.so."""
    units = [("somf_capi", os.path.join(CSRC, "somf_capi.cu"), []),
             ("bcd_onchip_inst", os.path.join(CSRC, "bcd_onchip_inst.cu"), [])]
    units += [(f"bcd_newton_k{k}", os.path.join(CSRC, "bcd_newton_inst.cu"), [f"-DNT_KPT={k}"])
              for k in NT_KPTS]
    units += [(f"bcd_big_k{k}", os.path.join(CSRC, "bcd_big_inst.cu"), [f"-DNB_KPT={k}"]) for k in NB_KPTS]
    return units


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/ into libsomf.so for sm_100a (in-tree): one object per
    translation unit, compiled in parallel, then linked with nvcc -shared."""
    from concurrent.futures import ThreadPoolExecutor
    newest = max(os.path.getmtime(s) for s in _sources())
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    base = [nvcc, "-O3", "-std=c++17", *NVCC_ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden"]
    if verbose:
        base.append("-Xptxas=-v")

    headers = [s for s in _sources() if not s.endswith(".cu")]
    newest_hdr = max(os.path.getmtime(s) for s in headers)

    def compile_one(unit):
        name, src, extra = unit
        obj = os.path.join(objdir, name + ".o")
        # an object is reused when it is newer than its source and every header
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(newest_hdr, os.path.getmtime(src))):
            return name, obj, subprocess.CompletedProcess([], 0, "", "")
        res = subprocess.run(base + extra + ["-c", src, "-o", obj], capture_output=True, text=True)
        return name, obj, res

    with ThreadPoolExecutor(max_workers=max(1, min(len(_units()), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, _units()))
    errs = [f"[{n}]\n{r.stdout}{r.stderr}" for n, _, r in results if r.returncode != 0]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    if verbose:
        for n, _, r in results:
            print(f"[{n}]\n{r.stderr}")
    tmp = LIB_PATH + ".tmp"
    res = subprocess.run([nvcc, *NVCC_ARCH, "-shared", "-o", tmp] + [o for _, o, _ in results],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class SomfConfig(C.Structure):
    _fields_ = [
        ("p", C.c_int64), ("k", C.c_int32), ("eta", C.c_int32),
        ("lambda_", C.c_double), ("nu", C.c_double), ("pos_code", C.c_int32),
        ("mu", C.c_double), ("pos_dict", C.c_int32),
        ("r", C.c_double), ("u", C.c_double),
        ("b_mode", C.c_int32), ("perm_cyclic", C.c_int32),
        ("cd_tol", C.c_double), ("cd_max_sweeps", C.c_int32),
        ("seed", C.c_uint64), ("row_lo", C.c_int64), ("row_hi", C.c_int64),
        ("device", C.c_int32), ("stream", C.c_void_p), ("debug", C.c_int32),
        ("bcd_kernel", C.c_int32),
        ("contract_kernel", C.c_int32), ("bbar_kernel", C.c_int32), ("codes_kernel", C.c_int32),
        ("bcd_lam_tol", C.c_double), ("bcd_copies", C.c_int32),
        ("estimator", C.c_int32), ("n_samples", C.c_int64), ("v", C.c_double),
        ("bcd_tile_rows", C.c_int32), ("bcd_group", C.c_int32),
    ]


# (name, restype, argtypes) of every symbol include/somf.h declares
P = C.c_void_p
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double
SIGNATURES = [
    ("somf_config_default", None, [C.POINTER(SomfConfig)]),
    ("somf_abi_version", I32, []),
    ("somf_config_size", I64, []),
    ("somf_status_string", C.c_char_p, [I32]),
    ("somf_last_error", C.c_char_p, [P]),
    ("somf_create", I32, [C.POINTER(SomfConfig), C.POINTER(P)]),
    ("somf_destroy", I32, [P]),
    ("somf_set_components", I32, [P, P, I64]),
    ("somf_partial_fit", I32, [P, P, I64]),
    ("somf_partial_fit_ids", I32, [P, P, I64, P]),
    ("somf_next_mask", I32, [P, C.POINTER(I64), P]),
    ("somf_partial_fit_masked", I32, [P, P, I64]),
    ("somf_get_codes", I32, [P, P]),
    ("somf_transform", I32, [P, P, I64, I64, P]),
    ("somf_objective", I32, [P, P, I64, I64, C.POINTER(D)]),
    ("somf_components", I32, [P, P, I64]),
    ("somf_get_state", I32, [P, P, P, P, P, C.POINTER(I64)]),
    ("somf_set_state", I32, [P, P, P, P, P, I64]),
    ("somf_last_step_info", I32, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(D)]),
    ("somf_bcd_variant", I32, [P]),
    ("somf_last_kernels", I32, [P, P]),
    ("somf_set_reducer", I32, [P, P, P]),
    ("somf_bcd_phase_cycles", I32, [P, P]),
    ("somf_profile_enable", I32, [P, I32]),
    ("somf_profile_read", I32, [P, P, P, C.POINTER(I64)]),
    ("somf_mask_rows", I32, [U64, I64, I64, I64, D, P, C.POINTER(I64), P]),
    ("somf_atom_permutation", I32, [U64, I64, I32, I32, P, P]),
    ("somf_column_ids", I32, [U64, I64, I64, I64, P, P]),
    ("somf_project_columns", I32, [P, I64, I32, I64, P, D, I32, P, P]),
]


# int32 reducer(void* user, void* buf, int64 count, int32 dtype, int32 op, void* stream)
REDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p)
DT_F64, DT_I32 = 0, 1
OP_SUM, OP_MIN, OP_MAX = 0, 1, 2


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                          "there is no CPU fallback")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.somf_config_size() != C.sizeof(SomfConfig):
        raise ImportError("somf_config layout mismatch between libsomf.so and the binding")
    return lib
