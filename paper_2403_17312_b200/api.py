"""Python view of the reference `skv` API for the SWA decode hot path.

Same names, argument meaning and error classes as the reference C++
functions (cited per function); every call goes through the C ABI in
include/skv_b200.h into sm_100a kernels. torch tensors are only the device
memory and stream plumbing. There is no CPU path: CPU tensors are rejected.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from ._lib import (REDUCE_FN, ContractViolation, CudaError, InfeasiblePlan, OutOfDeviceMemory,  # noqa: F401
                   Unsupported, check, lib)

SKV_F32, SKV_F16, SKV_BF16, SKV_U8 = 0, 1, 2, 3
_DT = {torch.float32: SKV_F32, torch.float16: SKV_F16, torch.bfloat16: SKV_BF16, torch.uint8: SKV_U8}
_TORCH = {v: k for k, v in _DT.items()}
_NAMES = {"f32": SKV_F32, "fp32": SKV_F32, "f16": SKV_F16, "fp16": SKV_F16, "bf16": SKV_BF16,
          "u8": SKV_U8, "int8": SKV_U8}


def _code(dt) -> int:
    if isinstance(dt, str):
        return _NAMES[dt]
    return _DT[dt]


def _stream(t: torch.Tensor | None = None):
    # the raw cudaStream_t of the current stream (an int; ctypes passes it as void*)
    idx = t.device.index if t is not None else torch.cuda.current_device()
    return _raw_stream(torch.cuda.current_device() if idx is None else idx)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None) or (
    lambda i: torch.cuda.current_stream(i).cuda_stream)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ContractViolation("device tensor required (no CPU path)")
    if not t.is_contiguous():
        raise ContractViolation("contiguous tensor required")
    return C.c_void_p(t.data_ptr())


class _DeviceView:
    """A device fp64 buffer owned by the library, seen by torch through
    __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, count: int, device: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


# ---- attention.hpp:122-138 -------------------------------------------------
def swa_window_k(n: int, r: float) -> int:
    k = lib().skv_swa_window_k(n, r)
    if k == 0:
        raise ContractViolation(lib().skv_last_error().decode())
    return k


def swa_keep_count(n: int, r: float) -> int:
    return min(2 * swa_window_k(n, r), n)


# ---- matrix.hpp:162-176 ----------------------------------------------------
def top_k_indices(v: torch.Tensor, k: int) -> torch.Tensor:
    """k largest per row (ties -> lower index), ascending. v: fp64 [len] or [B, len]."""
    v2 = v.reshape(1, -1) if v.dim() == 1 else v
    if v2.dtype != torch.float64:
        raise ContractViolation("top_k_indices: fp64 input required")
    out = torch.empty((v2.shape[0], max(k, 1)), dtype=torch.int32, device=v2.device)
    check(lib().skv_top_k_indices(_ptr(v2.contiguous()), v2.shape[0], v2.stride(0), v2.shape[1], k,
                                  _ptr(out), _stream(v2)))
    out = out[:, :k]
    return out[0] if v.dim() == 1 else out


# ---- attention.hpp:142-171 -------------------------------------------------
@dataclass
class SparseSelection:
    """attention.hpp:26-39; `all` is SparseSelection::all() per row."""
    all: torch.Tensor  # int32 [B, m] ascending
    k: int


def swa_select(importance: torch.Tensor, n: int, r: float) -> SparseSelection:
    imp = importance.reshape(1, -1) if importance.dim() == 1 else importance
    k = swa_window_k(n, r)
    m = n if (n < 2 or 2 * k >= n) else 2 * k
    if not (n < 2 or 2 * k >= n) and imp.shape[1] < n - 1:
        raise ContractViolation("swa_select: importance length must be n-1")
    out = torch.empty((imp.shape[0], max(m, 1)), dtype=torch.int32, device=imp.device)
    mo = C.c_int32()
    check(lib().skv_swa_select(_ptr(imp.contiguous()), imp.shape[0], imp.stride(0), n, r, _ptr(out),
                               C.byref(mo), _stream(imp)))
    out = out[:, :mo.value]
    return SparseSelection(out[0] if importance.dim() == 1 else out, k)


# ---- quant.hpp:43-95 -------------------------------------------------------
def quantize(x: torch.Tensor, bits: int = 8, channel_size: int = 0):
    """-> (codes uint16, scales fp64 [groups], zero_points int64 [groups])."""
    if x.dtype != torch.float64:
        raise ContractViolation("quantize: fp64 input required")
    n = x.numel()
    cs = channel_size or max(n, 1)
    groups = max(n // cs, 1)
    codes = torch.empty(max(n, 1), dtype=torch.uint16, device=x.device)
    scales = torch.empty(groups, dtype=torch.float64, device=x.device)
    zps = torch.empty(groups, dtype=torch.int64, device=x.device)
    check(lib().skv_quantize(_ptr(x.contiguous()), n, bits, channel_size, _ptr(codes), _ptr(scales),
                             _ptr(zps), _stream(x)))
    return codes[:n], scales, zps


def dequantize(codes: torch.Tensor, channel_size: int, scales: torch.Tensor, zps: torch.Tensor):
    out = torch.empty(codes.numel(), dtype=torch.float64, device=codes.device)
    check(lib().skv_dequantize(_ptr(codes), codes.numel(), channel_size, _ptr(scales), _ptr(zps),
                               _ptr(out), _stream(codes)))
    return out


def quantize_roundtrip(x: torch.Tensor, bits: int, channel_size: int) -> torch.Tensor:
    """quant.hpp:98-101"""
    codes, scales, zps = quantize(x, bits, channel_size)
    return dequantize(codes, channel_size or x.numel(), scales, zps)


# ---- AttentionState x L layers x B sequences ---------------------------------
class _Desc(C.Structure):
    _fields_ = [("layers", C.c_int32), ("batch", C.c_int32), ("heads", C.c_int32),
                ("head_dim", C.c_int32), ("capacity", C.c_int32), ("kv_dtype", C.c_int32),
                ("q_dtype", C.c_int32), ("device", C.c_int32), ("out_f32", C.c_int32)]


class _Plan(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("p1", C.c_int64), ("p2", C.c_int64),
                ("recompute_enabled", C.c_int32), ("input_len", C.c_int64), ("output_len", C.c_int64)]


class _CostParams(C.Structure):
    _fields_ = [("hidden", C.c_int64), ("layers", C.c_int64), ("batch", C.c_int64), ("input_len", C.c_int64),
                ("output_len", C.c_int64), ("ratio", C.c_double), ("bandwidth", C.c_double),
                ("bytes_per_element", C.c_int32), ("device_capacity", C.c_uint64), ("mac_rate", C.c_double),
                ("recompute_overhead", C.c_double)]


class _Prediction(C.Structure):
    _fields_ = [("total_seconds", C.c_double), ("prefill_compute_seconds", C.c_double),
                ("phase_compute", C.c_double * 3), ("phase_transfer", C.c_double * 3),
                ("phase_recompute", C.c_double * 3), ("phase_steps", C.c_int64 * 3),
                ("peak_device_bytes", C.c_uint64), ("feasible", C.c_int32)]


def _cost(cost: dict) -> _CostParams:
    return _CostParams(cost["hidden"], cost["layers"], cost.get("batch", 1), cost["input_len"], cost["output_len"],
                       cost.get("ratio", 1.0), cost.get("bandwidth", 1.0), cost.get("bytes_per_element", 2),
                       cost.get("device_capacity", 0), cost.get("mac_rate", 1e9), cost.get("recompute_overhead", 1.0))


def _pred(p: _Prediction) -> dict:
    return {"total_seconds": p.total_seconds, "prefill_compute_seconds": p.prefill_compute_seconds,
            "phase_compute": list(p.phase_compute), "phase_transfer": list(p.phase_transfer),
            "phase_recompute": list(p.phase_recompute), "phase_steps": list(p.phase_steps),
            "peak_device_bytes": p.peak_device_bytes, "feasible": bool(p.feasible)}


def solve_plan(cost: dict):
    """solve_plan (scheduler.hpp:207-303) -> (plan dict, prediction dict).
    cost keys follow CostParams (memsim.hpp:15-38)."""
    pl, pr = _Plan(), _Prediction()
    check(lib().skv_solve_plan(C.byref(_cost(cost)), C.byref(pl), C.byref(pr)))
    plan = {"alpha": pl.alpha, "beta": pl.beta, "p1": pl.p1, "p2": pl.p2,
            "recompute_enabled": bool(pl.recompute_enabled)}
    return plan, _pred(pr)


def predict_plan(cost: dict, plan: dict) -> dict:
    """predict_plan (scheduler.hpp:174-186)."""
    pl = _Plan(plan["alpha"], plan["beta"], plan["p1"], plan["p2"], int(plan.get("recompute_enabled", True)), 0, 0)
    pr = _Prediction()
    check(lib().skv_predict_plan(C.byref(_cost(cost)), C.byref(pl), C.byref(pr)))
    return _pred(pr)


class SwaCache:
    """Device-resident decode state: the reference's AttentionState
    (attention.hpp:45-86) for `layers` x `batch` sequences, K/V token-major in
    HBM, fp64 head-summed importance accumulator."""

    def __init__(self, layers: int, batch: int, heads: int, head_dim: int, capacity: int,
                 kv_dtype="f16", q_dtype=None, device: int | None = None, out_f32: bool = False,
                 device_capacity: int | None = None):
        """device_capacity (bytes): a PAGED cache whose device K/V pool is
        bounded by the KvLedger capacity (skv_cache_create_paged); None: the
        dense [L][B][capacity] layout."""
        self.layers, self.batch, self.heads, self.head_dim, self.capacity = (
            layers, batch, heads, head_dim, capacity)
        self.kv_code = _code(kv_dtype)
        self.q_code = _code(q_dtype) if q_dtype is not None else (
            SKV_F16 if self.kv_code == SKV_U8 else self.kv_code)
        self.q_dtype = _TORCH[self.q_code]
        self.device = torch.cuda.current_device() if device is None else device
        self.dev = torch.device("cuda", self.device)
        self.out_dtype = torch.float32 if out_f32 else self.q_dtype
        d = _Desc(layers, batch, heads, head_dim, capacity, self.kv_code, self.q_code, self.device,
                  int(out_f32))
        h = C.c_void_p()
        if device_capacity is None:
            check(lib().skv_cache_create(C.byref(d), C.byref(h)))
        else:
            check(lib().skv_cache_create_paged(C.byref(d), int(device_capacity), C.byref(h)))
        self._h = h

    def set_head_shard(self, head_offset: int, total_heads: int, reduce=None):
        """Hold heads [head_offset, head_offset + heads) of a model with
        total_heads (SURVEY §8 e). `reduce(buf, stream)` gets a device fp64
        tensor viewing the library's exchange row and must sum it in place
        across the shards, ordered on `stream` (a torch.cuda.ExternalStream),
        e.g. shard.dist_reducer(). reduce=None: unsharded again."""
        if reduce is None:
            self._reduce_cb = None
            check(lib().skv_cache_set_head_shard(self._h, 0, 0, REDUCE_FN(), None))
            return
        dev = self.dev

        def _cb(ptr, count, stream, _user):
            try:
                buf = torch.as_tensor(_DeviceView(ptr, count, dev.index), device=dev)
                reduce(buf, torch.cuda.ExternalStream(stream or 0, device=dev))
                return 0
            except Exception as e:  # surfaces as the entry point's error
                import sys
                print(f"skv head-shard reduce failed: {e!r}", file=sys.stderr)
                return 4  # SKV_ERR_CUDA

        self._reduce_cb = REDUCE_FN(_cb)
        check(lib().skv_cache_set_head_shard(self._h, head_offset, total_heads, self._reduce_cb, None))

    def close(self):
        if getattr(self, "_h", None):
            lib().skv_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        b = C.c_uint64()
        check(lib().skv_cache_get_desc(self._h, None, C.byref(b)))
        return b.value

    # ---- KvLedger byte accounting (memsim.hpp:77-215)
    def set_capacity(self, device_capacity: int):
        check(lib().skv_cache_set_capacity(self._h, int(device_capacity)))

    def ledger_totals(self) -> dict:
        """device / host / peak device bytes and the capacity; raises the first
        failure a kernel reported (OutOfDeviceMemory, ContractViolation)."""
        v = [C.c_uint64() for _ in range(4)]
        check(lib().skv_ledger_totals(self._h, *[C.byref(x) for x in v], _stream()))
        return dict(zip(("device_bytes", "host_bytes", "peak_device_bytes", "capacity"), (x.value for x in v)))

    def ledger_counters(self) -> dict:
        rows = (C.c_uint64 * 5)()
        check(lib().skv_ledger_counters(self._h, rows, _stream()))
        return dict(zip(("offloaded", "deleted", "reloaded", "recomputed", "kept"), (int(x) for x in rows)))

    def profile_move(self, layer: int, rows: int, reps: int = 5) -> float:
        """ms per duplex movement launch of `rows` rows each way per sequence."""
        ms = C.c_double()
        check(lib().skv_profile_move(self._h, layer, rows, reps, C.byref(ms), _stream()))
        return ms.value

    def storage(self) -> dict:
        sl, pool, full = C.c_int32(), C.c_uint64(), C.c_uint64()
        check(lib().skv_cache_storage(self._h, C.byref(sl), C.byref(pool), C.byref(full)))
        return {"slots_per_sequence": sl.value, "kv_pool_bytes": pool.value, "full_kv_bytes": full.value}

    def _q(self, t: torch.Tensor, shape) -> torch.Tensor:
        if t.dtype != self.q_dtype or tuple(t.shape) != tuple(shape):
            raise ContractViolation(f"expected {self.q_dtype} {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")
        return t

    # AttentionState::append_token over a block of tokens (attention.hpp:65-74)
    def append_tokens(self, layer: int, b0: int, t0: int, k: torch.Tensor, v: torch.Tensor):
        nb, nt = k.shape[0], k.shape[1]
        shp = (nb, nt, self.heads, self.head_dim)
        check(lib().skv_cache_write(self._h, layer, b0, nb, t0, nt, _ptr(self._q(k, shp)),
                                    _ptr(self._q(v, shp)), _stream(k)))

    def read(self, layer: int, b0: int, nb: int, t0: int, nt: int) -> torch.Tensor:
        out = torch.empty((nb, nt, 2, self.heads, self.head_dim), dtype=torch.float32, device=self.dev)
        check(lib().skv_cache_read(self._h, layer, b0, nb, t0, nt, _ptr(out), _stream(out)))
        return out

    def set_importance(self, layer: int, imp: torch.Tensor, b0: int = 0):
        imp = imp.to(torch.float64).contiguous()
        check(lib().skv_importance_set(self._h, layer, b0, imp.shape[0], imp.shape[1], _ptr(imp),
                                       _stream(imp)))

    def importance(self, layer: int, length: int, b0: int = 0, nb: int | None = None) -> torch.Tensor:
        nb = self.batch - b0 if nb is None else nb
        out = torch.empty((nb, length), dtype=torch.float64, device=self.dev)
        check(lib().skv_importance_get(self._h, layer, b0, nb, length, _ptr(out), _stream(out)))
        return out

    # Engine::prefill accumulator seeding (engine.hpp:508-512)
    def prefill_seed(self, layer: int, n: int, q_last: torch.Tensor) -> torch.Tensor:
        out = torch.empty(self._q(q_last, (self.batch, self.heads, self.head_dim)).shape,
                          dtype=self.out_dtype, device=self.dev)
        check(lib().skv_prefill_seed(self._h, layer, n, _ptr(q_last), _ptr(out), _stream(q_last)))
        return out

    # Engine::prefill's attention (engine.hpp:485-529) on tensor cores: the
    # prompt's K/V must already be in the cache (append_tokens); returns the
    # causal attention output [B][s][H][D] and seeds the importance.
    def prefill_layer(self, layer: int, q: torch.Tensor) -> torch.Tensor:
        if q.dim() != 4 or q.shape[0] != self.batch or q.shape[2:] != (self.heads, self.head_dim):
            raise ContractViolation(f"prefill: q must be [B][s][H][D], got {tuple(q.shape)}")
        s = q.shape[1]
        self._q(q, (self.batch, s, self.heads, self.head_dim))
        out = torch.empty(q.shape, dtype=self.out_dtype, device=self.dev)
        check(lib().skv_prefill_layer(self._h, layer, s, _ptr(q), _ptr(out), _stream(q)))
        return out

    def prefill_sparsity(self, layer: int) -> torch.Tensor:
        # engine.hpp:513-518 per sequence: mean over heads of the causal sparsity
        out = torch.empty(self.batch, dtype=torch.float64, device=self.dev)
        check(lib().skv_prefill_sparsity_get(self._h, layer, _ptr(out), _stream(out)))
        return out

    # One decode step of one layer (engine.hpp:592-629 order; swa_attention)
    def swa_decode_layer(self, layer: int, n: int, r: float, q, k_new, v_new, out=None,
                         return_indices: bool = False, return_weights: bool = False):
        shp = (self.batch, self.heads, self.head_dim)
        for t in (q, k_new, v_new):
            self._q(t, shp)
        out = torch.empty(q.shape, dtype=self.out_dtype, device=self.dev) if out is None else out
        m = self.selection_size(n, r)[0]
        idx = torch.empty((self.batch, m), dtype=torch.int32, device=self.dev) if return_indices else None
        w = (torch.empty((self.batch, self.heads, m), dtype=torch.float32, device=self.dev)
             if return_weights else None)
        check(lib().skv_swa_decode_layer(self._h, layer, n, r, _ptr(q), _ptr(k_new), _ptr(v_new),
                                         _ptr(out), _ptr(idx), _ptr(w), _stream(q)))
        return out, idx, w

    def swa_decode_step(self, n: int, r: float, q, k_new, v_new, out=None):
        # per-step host cost matters at config 1 (one layer, b = 1): checks kept, object churn trimmed
        shp = (self.layers, self.batch, self.heads, self.head_dim)
        for t in (q, k_new, v_new):
            self._q(t, shp)
        out = torch.empty(q.shape, dtype=self.out_dtype, device=self.dev) if out is None else out
        st = _raw_stream(q.device.index) if q.is_cuda else None
        rc = lib().skv_swa_decode_step(self._h, n, r, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), st)
        if rc:
            check(rc)
        return out

    def swa_decode_step_host(self, n: int, r: float, q, k_new, v_new, out):
        """Host (CPU, ideally pinned) tensors in and out; enqueued on the
        current stream of this cache's device."""
        for t in (q, k_new, v_new, out):
            if t.is_cuda or not t.is_contiguous():
                raise ContractViolation("host contiguous tensors required")
        s = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        check(lib().skv_swa_decode_step_host(self._h, n, r, C.c_void_p(q.data_ptr()),
                                             C.c_void_p(k_new.data_ptr()), C.c_void_p(v_new.data_ptr()),
                                             C.c_void_p(out.data_ptr()), s))
        return out

    # attend_over_indices (attention.hpp:183-231): any order, duplicates allowed
    # (each occurrence is one softmax term and adds its weight, as in the reference)
    def attend_over_indices(self, layer: int, n: int, idx: torch.Tensor, q: torch.Tensor,
                            return_weights: bool = False):
        idx = idx.to(torch.int32).contiguous()
        if idx.dim() == 1:
            idx = idx.reshape(1, -1).expand(self.batch, -1).contiguous()
        m = idx.shape[1]
        out = torch.empty(self._q(q, (self.batch, self.heads, self.head_dim)).shape, dtype=self.out_dtype,
                          device=self.dev)
        w = (torch.empty((self.batch, self.heads, m), dtype=torch.float32, device=self.dev)
             if return_weights else None)
        check(lib().skv_attend_over_indices(self._h, layer, n, _ptr(idx), m, _ptr(q), _ptr(out), _ptr(w),
                                            _stream(q)))
        return out, w

    # ---- attention variants (attention.hpp:15-21, engine.hpp:531-569)
    VARIANTS = {"dense": 0, "swa": 1, "local": 2, "strided": 3}

    def set_variant(self, variant: str = "swa", stride: int = 0):
        check(lib().skv_cache_set_variant(self._h, self.VARIANTS[variant], stride))

    def selection_size(self, n: int, r: float):
        m, k = C.c_int32(), C.c_int32()
        check(lib().skv_selection_size(self._h, n, r, C.byref(m), C.byref(k)))
        return m.value, k.value

    def pending_selection(self, layer: int, n: int, r: float) -> torch.Tensor:
        """SparseSelection::all() the next decode step of `layer` attends at
        (n, r): int32 [B, m] ascending (selected one step ahead)."""
        m, _ = self.selection_size(n, r)
        out = torch.empty((self.batch, max(m, 1)), dtype=torch.int32, device=self.dev)
        mo = C.c_int32()
        check(lib().skv_pending_selection(self._h, layer, n, r, _ptr(out), C.byref(mo), _stream(out)))
        return out[:, :mo.value]

    def sparsity(self, layer: int) -> torch.Tensor:
        # attention_sparsity of each sequence's last step row (attention.hpp:275-310)
        out = torch.empty(self.batch, dtype=torch.float64, device=self.dev)
        check(lib().skv_sparsity_get(self._h, layer, 0, self.batch, _ptr(out), _stream(out)))
        return out

    # ---- three-phase schedule bookkeeping (memsim.hpp:77-215, scheduler.hpp:320-381)
    def set_plan(self, alpha: float, beta: float, p1: int, p2: int, input_len: int, output_len: int,
                 recompute_enabled: bool = True):
        pl = _Plan(alpha, beta, p1, p2, int(recompute_enabled), input_len, output_len)
        check(lib().skv_cache_set_plan(self._h, C.byref(pl)))

    def enable_host_tier(self, poison: bool = False):
        check(lib().skv_cache_enable_host_tier(self._h, int(poison)))

    def attach_recompute(self, layer: int, x_ln1: torch.Tensor, wk: torch.Tensor, wv: torch.Tensor):
        # recompute_kv sources (engine.hpp:718-737); x_ln1 [B, capacity, H*D] is kept by reference
        self._rec = getattr(self, "_rec", {})
        self._rec[layer] = x_ln1
        check(lib().skv_cache_attach_recompute(self._h, layer, _ptr(x_ln1), _ptr(wk.contiguous()),
                                               _ptr(wv.contiguous()), _stream(x_ln1)))
        torch.cuda.current_stream(self.dev).synchronize()

    def clear_plan(self):
        check(lib().skv_cache_set_plan(self._h, None))

    def set_tiers(self, layer: int, tiers: torch.Tensor, b0: int = 0):
        # tiers: uint8 [nb, len] (0 device, 1 host, 2 deleted, 255 absent)
        t = tiers.to(device=self.dev, dtype=torch.uint8).contiguous()
        check(lib().skv_ledger_set(self._h, layer, b0, t.shape[0], t.shape[1], _ptr(t), _stream(t)))

    def tiers(self, layer: int, length: int, b0: int = 0, nb: int | None = None) -> torch.Tensor:
        nb = self.batch - b0 if nb is None else nb
        out = torch.empty((nb, length), dtype=torch.uint8, device=self.dev)
        check(lib().skv_ledger_get(self._h, layer, b0, nb, length, _ptr(out), _stream(out)))
        return out

    def _lists(self, lists: torch.Tensor, counts: torch.Tensor):
        names = ("offload", "delete", "reload", "recompute")
        lists, counts = lists.cpu(), counts.cpu()
        return [{nm: lists[b, i, :counts[b, i]].tolist() for i, nm in enumerate(names)} for b in range(self.batch)]

    def step_actions(self, layer: int, j: int, selected: torch.Tensor, k: int, apply: bool = True):
        # step_actions for every sequence; selected: int32 [B, m] ascending
        sel = selected.to(device=self.dev, dtype=torch.int32).contiguous()
        lists = torch.empty((self.batch, 4, self.capacity), dtype=torch.int32, device=self.dev)
        counts = torch.empty((self.batch, 4), dtype=torch.int32, device=self.dev)
        check(lib().skv_step_actions(self._h, layer, j, _ptr(sel), sel.shape[1], k, int(apply), _ptr(lists),
                                     _ptr(counts), _stream(sel)))
        return self._lists(lists, counts)

    def last_actions(self, layer: int):
        lists = torch.empty((self.batch, 4, self.capacity), dtype=torch.int32, device=self.dev)
        counts = torch.empty((self.batch, 4), dtype=torch.int32, device=self.dev)
        check(lib().skv_last_actions(self._h, layer, _ptr(lists), _ptr(counts), _stream(lists)))
        return self._lists(lists, counts)

    # measurement hooks
    def profile(self, enable: bool):
        check(lib().skv_profile_enable(self._h, int(enable)))

    def attend_chain_ms(self, n: int, r: float, q, k_new, v_new, out, reps: int = 3) -> float:
        ms = C.c_double()
        check(lib().skv_profile_attend_chain(self._h, n, r, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), reps,
                                             C.byref(ms), _stream(q)))
        return ms.value

    def attend_config(self) -> dict:
        v = [C.c_int32() for _ in range(4)]
        check(lib().skv_attend_config(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("heads_per_cta", "grid", "smem_bytes", "ctas_per_sm"), (x.value for x in v)))

    def profile_read(self):
        ms, n, b = C.c_double(), C.c_int64(), C.c_uint64()
        check(lib().skv_profile_read(self._h, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value


# ---- attention.hpp:91-117 ---------------------------------------------------
def dense_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal: bool):
    """softmax(q k^T / sqrt(D)) v per query row -> (attn [sq, D], aw [sq, sk])
    fp32, like the reference's pair (attention.hpp:91-117). The causal mask is
    aligned to the bottom-right corner as in the reference (:98-103): row i
    sees keys j <= i + (sk - sq). Same checks and messages as the reference,
    in its order; a causal row with no visible key fails like softmax_rows
    (matrix.hpp:145). Each row is one attend over its key range on a one-head
    fp32 cache (head_dim 128); for the batched causal prefill of a cache use
    SwaCache.prefill_layer (tensor cores)."""
    sq, D = q.shape
    sk, Dk = k.shape
    if D != Dk or v.shape[1] != Dk:
        raise ContractViolation("dense_attention: head_dim mismatch")
    if v.shape[0] != sk:
        raise ContractViolation("dense_attention: key/value length mismatch")
    if sq == 0 or sk == 0:
        raise ContractViolation("dense_attention: empty input")
    off = sk - sq
    if causal and off < 0:
        raise ContractViolation("softmax_rows: row has no finite entry")
    dev = q.device
    cache = SwaCache(1, 1, 1, D, sk, kv_dtype="f32", device=dev.index, out_f32=True)
    f = lambda t: t.to(device=dev, dtype=torch.float32).contiguous()  # noqa: E731
    cache.append_tokens(0, 0, 0, f(k).reshape(1, sk, 1, D), f(v).reshape(1, sk, 1, D))
    idx = torch.arange(sk, dtype=torch.int32, device=dev)
    attn = torch.empty((sq, D), dtype=torch.float32, device=dev)
    aw = torch.zeros((sq, sk), dtype=torch.float32, device=dev)
    qf = f(q)
    for r in range(sq):
        n = r + 1 + off if causal else sk
        out, w = cache.attend_over_indices(0, n, idx[:n], qf[r].reshape(1, 1, D), return_weights=True)
        attn[r] = out[0, 0]
        aw[r, :n] = w[0, 0]
    cache.close()
    return attn, aw


def launch_count() -> int:
    return lib().skv_launch_count()
