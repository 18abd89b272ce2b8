"""Loader for libskv_b200.so (the C ABI in include/skv_b200.h).

There is no CPU fallback: if the shared library is missing and cannot be
built, every entry point raises. The library is built in-tree (so it travels
with the repo snapshot to the GPU box) by ``build()``.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO_PATH = os.environ.get("SKV_LIB") or os.path.join(PKG, "libskv_b200.so")

_lock = threading.Lock()
_lib = None


class ContractViolation(Exception):
    """skv::ContractViolation (common.hpp:12)."""


class OutOfDeviceMemory(Exception):
    """skv::OutOfDeviceMemory (common.hpp:17)."""


class InfeasiblePlan(Exception):
    """skv::InfeasiblePlan (common.hpp:22)."""


class CudaError(RuntimeError):
    pass


class Unsupported(RuntimeError):
    pass


_STATUS = {1: ContractViolation, 2: OutOfDeviceMemory, 3: InfeasiblePlan, 4: CudaError, 5: Unsupported}


def build(force: bool = False) -> str:
    """Compile libskv_b200.so for sm_100a with nvcc (make in csrc/)."""
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    subprocess.run(["make", "-s", "-C", CSRC, "-j4", f"NVCC={nvcc}"], check=True)
    return SO_PATH


# skv_reduce_fn (include/skv_b200.h): sum `count` device fp64 values in place
# across the head shards, ordered on `stream`.
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


def _declare(lib):
    P, I, I64, U64, SZ, D = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_size_t, C.c_double
    sig = {
        "skv_last_error": (C.c_char_p, []),
        "skv_version": (C.c_char_p, []),
        "skv_launch_count": (U64, []),
        "skv_swa_window_k": (SZ, [SZ, D]),
        "skv_swa_keep_count": (SZ, [SZ, D]),
        "skv_cache_create": (I, [P, P]),
        "skv_cache_create_paged": (I, [P, U64, P]),
        "skv_cache_set_capacity": (I, [P, U64]),
        "skv_ledger_totals": (I, [P, P, P, P, P, P]),
        "skv_cache_storage": (I, [P, P, P, P]),
        "skv_ledger_counters": (I, [P, P, P]),
        "skv_profile_move": (I, [P, I, I, I, P, P]),
        "skv_cache_destroy": (I, [P]),
        "skv_cache_get_desc": (I, [P, P, P]),
        "skv_cache_write": (I, [P, I, I, I, I, I, P, P, P]),
        "skv_cache_read": (I, [P, I, I, I, I, I, P, P]),
        "skv_importance_set": (I, [P, I, I, I, I, P, P]),
        "skv_importance_get": (I, [P, I, I, I, I, P, P]),
        "skv_prefill_seed": (I, [P, I, I, P, P, P]),
        "skv_prefill_layer": (I, [P, I, I, P, P, P]),
        "skv_prefill_sparsity_get": (I, [P, I, P, P]),
        "skv_swa_decode_layer": (I, [P, I, I, D, P, P, P, P, P, P, P]),
        "skv_swa_decode_step": (I, [P, I, D, P, P, P, P, P]),
        "skv_swa_decode_step_host": (I, [P, I, D, P, P, P, P, P]),
        "skv_attend_over_indices": (I, [P, I, I, P, I, P, P, P, P]),
        "skv_swa_select": (I, [P, I, I64, I, D, P, P, P]),
        "skv_top_k_indices": (I, [P, I, I64, I, I, P, P]),
        "skv_quantize": (I, [P, SZ, C.c_uint32, SZ, P, P, P, P]),
        "skv_dequantize": (I, [P, SZ, SZ, P, P, P, P]),
        "skv_cache_set_plan": (I, [P, P]),
        "skv_cache_enable_host_tier": (I, [P, I]),
        "skv_cache_attach_recompute": (I, [P, I, P, P, P, P]),
        "skv_solve_plan": (I, [P, P, P]),
        "skv_predict_plan": (I, [P, P, P]),
        "skv_cache_set_variant": (I, [P, I, I]),
        "skv_cache_set_head_shard": (I, [P, I, I, REDUCE_FN, P]),
        "skv_selection_size": (I, [P, I, D, P, P]),
        "skv_sparsity_get": (I, [P, I, I, I, P, P]),
        "skv_pending_selection": (I, [P, I, I, D, P, P, P]),
        "skv_ledger_set": (I, [P, I, I, I, I, P, P]),
        "skv_ledger_get": (I, [P, I, I, I, I, P, P]),
        "skv_step_actions": (I, [P, I, I, P, I, I, I, P, P, P]),
        "skv_last_actions": (I, [P, I, P, P, P]),
        "skv_gemm_tn": (I, [P, P, P, I, I, I, I, P]),
        "skv_device_alloc": (I, [I, SZ, P]),
        "skv_device_free": (I, [P]),
        "skv_copy": (I, [P, P, SZ, P]),
        "skv_host_alloc": (I, [SZ, P]),
        "skv_host_free": (I, [P]),
        "skv_stream_synchronize": (I, [P]),
        "skv_profile_enable": (I, [P, I]),
        "skv_profile_read": (I, [P, P, P, P]),
        "skv_profile_attend_chain": (I, [P, I, D, P, P, P, P, I, P, P]),
        "skv_attend_config": (I, [P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded C ABI. Builds it first when absent (nvcc present here and on
    the GPU box); raises when that is impossible -- never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO_PATH):
                try:
                    build()
                except Exception as e:  # pragma: no cover - environment failure
                    raise RuntimeError(f"libskv_b200.so missing and build failed: {e}") from e
            _lib = _declare(C.CDLL(SO_PATH))
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().skv_last_error().decode(errors="replace")
        raise _STATUS.get(status, RuntimeError)(msg)
