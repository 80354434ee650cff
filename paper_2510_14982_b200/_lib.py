"""Loader and builder for libapo_b200.so (the sm_100a kernels behind the C ABI).

The library is built in-tree with nvcc (``build()``), loaded with ctypes
and bound to the prototypes of include/apo_b200.h.  There is no CPU
fallback: if the library is missing or a CUDA device is absent, every entry
point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import threading
import time

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB_PATH = os.path.join(PKG_DIR, "libapo_b200.so")

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: oracle-exact arithmetic (the reference never fuses mul+add).
NVCC_FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-diag-suppress", "177"]
# One TU per kernel family so nvcc runs in parallel (the templates live in
# csrc/apo_kernels.cuh); linked into a single shared library.
SOURCES = ["apo_kernels.cu", "apo_update_sel.cu", "apo_update_dense.cu", "apo_batch.cu", "apo_batch_m1.cu",
           "apo_batch_m2.cu", "apo_batch_m4.cu", "apo_batch_m0.cu", "apo_batch_warp.cu", "apo_cec_eval.cu",
           "apo_cec_gemm.cu", "apo_prologue.cu", "apo_update_fused.cu",
           "apo_update_fused12.cu", "apo_update_scripted.cu"]

# CEC2022-only TUs (parity unpinned, checked at 1e-9 relative): FMA contraction allowed.  Every TU
# on the reference's bit-exact path keeps --fmad=false.
FMA_SOURCES = ("apo_cec_eval.cu", "apo_cec_gemm.cu")
# Hot-kernel TUs compiled a second time with -DAPO_PHILOX_VARIANT: the default objects read the keyed
# stream only (no Philox call site in their loops), these serve rng = "philox" runs.
PHILOX_VARIANTS = ("apo_update_sel.cu", "apo_update_dense.cu", "apo_batch_m1.cu", "apo_batch_m2.cu", "apo_batch_m4.cu",
                   "apo_batch_m0.cu", "apo_batch_warp.cu")


# Batch TUs compiled once more with -DAPO_MANY_PAIRS_VARIANT: keyed kernels for npairs > 1 (the default
# objects are built for npairs == 1 only).
MANY_PAIRS_VARIANTS = ("apo_batch_m1.cu", "apo_batch_m2.cu", "apo_batch_m4.cu", "apo_batch_m0.cu")


def _units():
    """(source, object name, extra nvcc flags) of every translation unit."""
    units = [(src, src.replace(".cu", ".o"), []) for src in SOURCES]
    units += [(src, src.replace(".cu", "_philox.o"), ["-DAPO_PHILOX_VARIANT"]) for src in PHILOX_VARIANTS]
    units += [(src, src.replace(".cu", "_many.o"), ["-DAPO_MANY_PAIRS_VARIANT"]) for src in MANY_PAIRS_VARIANTS]
    return units

_lock = threading.Lock()
_lib = None


class ApoError(RuntimeError):
    """A C-ABI call failed (CUDA error or rejected argument)."""


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise ApoError("nvcc not found; cannot build libapo_b200.so")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "apo_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libapo_b200.so for sm_100a (in-tree, so it travels with the repo).

    Each TU compiles to an object in parallel, then nvcc links the shared
    library."""
    from concurrent.futures import ThreadPoolExecutor

    with _lock:
        if not force and not _stale():
            return LIB_PATH
        objdir = os.path.join(PKG_DIR, "build")
        os.makedirs(objdir, exist_ok=True)
        flags = [f for f in NVCC_FLAGS if f != "-shared"]

        headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
        headers.append(os.path.join(INCLUDE, "apo_b200.h"))
        newest_header = max(os.path.getmtime(h) for h in headers)

        def compile_one(unit):
            src, oname, extra = unit
            obj = os.path.join(objdir, oname)
            if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(
                    newest_header, os.path.getmtime(os.path.join(CSRC, src))):
                return obj, subprocess.CompletedProcess([], 0, "", "")  # up to date (same flags)
            f = flags
            if src in FMA_SOURCES:  # no bit-exact reference there: let nvcc contract multiply-adds
                f = ["--fmad=true" if x == "--fmad=false" else x for x in flags]
            cmd = [nvcc(), *ARCH_FLAGS, *f, *extra, "-I", INCLUDE, "-I", CSRC, "-c", "-o", obj, os.path.join(CSRC, src)]
            if verbose:
                print(" ".join(cmd), flush=True)
            t0 = time.time()
            proc = subprocess.run(cmd, capture_output=True, text=True)
            if verbose:
                print(f"  {oname}: {time.time() - t0:.0f} s", flush=True)
            return obj, proc

        units = _units()
        with ThreadPoolExecutor(max_workers=len(units)) as ex:
            results = list(ex.map(compile_one, units))
        for obj, proc in results:
            if proc.returncode != 0:
                raise ApoError(f"nvcc failed for {obj} ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
        tmp = LIB_PATH + ".tmp"
        cmd = [nvcc(), *ARCH_FLAGS, "-shared", "-o", tmp, *[o for o, _ in results]]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise ApoError(f"nvcc link failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
        os.replace(tmp, LIB_PATH)
        return LIB_PATH


_P = C.c_void_p
_I = C.c_int64
_U = C.c_uint64
_D = C.c_double
_INT = C.c_int


class apo_objective(C.Structure):
    _fields_ = [("code", C.c_int32), ("table_len", C.c_int32), ("table", C.c_void_p), ("shift", C.c_void_p),
                ("rot_t", C.c_void_p), ("shuffle", C.c_void_p), ("rot_pad", C.c_void_p),
                ("rot_gemm", C.c_void_p), ("flags", C.c_int32)]


PROTOTYPES = {
    "apo_abi_version": (_INT, []),
    "apo_max_dim": (_I, []),
    "apo_last_error": (C.c_char_p, []),
    "apo_device_count": (_INT, []),
    "apo_run_updates": (_INT, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _U, _U, _I, _D, _D, _D, _D, _D, _D, _D, _I, _P,
                               _I, _P, _P, _P]),
    "apo_run_updates_obj": (_INT, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _U, _U, _I, _D, _D, _D, _D, _D, _D,
                                   C.POINTER(apo_objective), _P, _P, _P]),
    "apo_run_updates_range": (_INT, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _U, _U, _I, _D, _D, _D, _D, _D, _D,
                                     C.POINTER(apo_objective), _P, _P, _I, _I, _P]),
    "apo_run_updates_ordered": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _U, _U, _I, _D, _D, _D, _D, _D, _D,
                                       C.POINTER(apo_objective), _P, _P, _I, _I, _P]),
    "apo_run_updates_scripted": (_INT, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _I, _D, _D, _D, _D, _D, _D,
                                        C.POINTER(apo_objective), _P, _P, _P]),
    "apo_select_dr_scripted": (_INT, [_P, _I, _I, _P, _P]),
    "apo_evaluate": (_INT, [_P, _I, _I, _I, C.POINTER(apo_objective), _P, _P]),
    "apo_initialize": (_INT, [_U, _I, _I, _I, _D, _D, C.POINTER(apo_objective), _P, _P, _P]),
    "apo_sort_order": (_INT, [_P, _I, _P, _P]),
    "apo_select_dr": (_INT, [_U, _U, _I, _D, _P, C.POINTER(C.c_int64), _P]),
    "apo_histogram_u8": (_INT, [_P, _I, _P, _P]),
    "apo_threshold_tables": (_INT, [_P, _INT, _P, _P]),
    "apo_run_create": (_INT, [C.POINTER(C.c_void_p), _I, _I, _I, _U, _I, _D, _D, _D, _D, C.POINTER(apo_objective),
                              _P, _P, _INT, _P]),
    "apo_run_initialize": (_INT, [_P]),
    "apo_run_iterate": (_INT, [_P, _I]),
    "apo_run_load": (_INT, [_P, _P, _P, _INT, _I, _I]),
    "apo_run_trace": (_INT, [_P, _P, _I]),
    "apo_run_population": (_INT, [_P, _P, _P, _INT]),
    "apo_run_best": (_INT, [_P, _P, _P, C.POINTER(C.c_int64)]),
    "apo_run_counters": (_INT, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "apo_run_destroy": (_INT, [_P]),
    "apo_run_profile": (_INT, [_P, _INT]),
    "apo_run_profile_read": (_INT, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "apo_run_profile_split": (_INT, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "apo_run_update_path": (_INT, [_P, C.POINTER(_INT)]),
    "apo_run_batch": (_INT, [_I, _P, C.POINTER(apo_objective), _I, _I, _I, _I, _I, _D, _D, _D, _D, _P, _P, _P, _P,
                             _P, _P, _P, _P, _INT, _P]),
    "apo_run_batch_shaped": (_INT, [_I, _P, C.POINTER(apo_objective), _I, _I, _I, _I, _I, _D, _D, _D, _D, _P, _P,
                                    _P, _P, _P, _P, _P, _P, _INT, _INT, _P]),
    "apo_run_batch_max_elems": (_I, [_I, _I]),
    "apo_release_cached_memory": (_INT, []),
    "apo_run_batch_fits": (_INT, [_I, _I, C.POINTER(apo_objective), _I]),
    "apo_shard_create": (_INT, [C.POINTER(C.c_void_p), _I, _I, _I, _I, _U, _I, _D, _D, _D, _D,
                                C.POINTER(apo_objective), _P, _P, _INT, _P, _P, _P, _P, _P]),
    "apo_shard_initialize": (_INT, [_P]),
    "apo_shard_begin": (_INT, [_P]),
    "apo_shard_update_range": (_INT, [_P, _I, _I]),
    "apo_shard_end": (_INT, [_P]),
    "apo_shard_state": (_INT, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "apo_shard_counters": (_INT, [_P, _P, _I, C.POINTER(C.c_int64)]),
    "apo_shard_destroy": (_INT, [_P]),
    "apo_debug_exp": (_INT, [_P, _P, _I, _P]),
    "apo_debug_cos": (_INT, [_P, _P, _I, _P]),
    "apo_debug_cec_basic": (_INT, [_INT, _P, _I, _I, _P, _P, _INT, _P]),
    "apo_philox4x32_10": (None, [_P, _P, _P]),
    "apo_rng_uniform": (_D, [_INT, _U, _U, _U, _U]),
}


def load(path: str = None):
    """dlopen the library and bind every prototype (no device needed).

    APO_LIB overrides the path (used to A/B build variants; never set in tests)."""
    global _lib
    path = path or os.environ.get("APO_LIB") or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ApoError(f"{path} is missing: run __graft_entry__.build() (or paper_2510_14982_b200._lib.build())")
        lib = C.CDLL(path)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().apo_last_error().decode(errors="replace")
        raise ApoError(f"{what or 'libapo_b200'} failed (status {rc}): {msg}")


def require_cuda():
    """The CUDA path is the only path: fail loudly without a device."""
    import torch

    if not torch.cuda.is_available():
        raise ApoError("the cuda backend needs a CUDA device (no CPU fallback exists)")
    return load()


def stream_handle(stream=None) -> C.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t) -> C.c_void_p:
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())
