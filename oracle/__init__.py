"""ctypes view of the CPU parity checker -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the CPU legs of ``bench.py``
may import this package; the product (``paper_2403_17312_b200``) never does.

Two interchangeable backends expose the same Python API:

* ``Oracle("port")``      -- ``build/liboracle.so``: the C restatement in
  ``skv_oracle.c`` (every function cites the reference file:line it follows).
* ``Oracle("reference")`` -- ``_ref/libskvref.so``: the unmodified reference
  headers (/root/reference/proj/include/skv) behind ``ref_harness.cpp``.
  Built only where /root/reference exists; the prebuilt .so travels with the
  repo snapshot.

Errors map to the reference exception classes (common.hpp:12-34).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libskvref.so")


class ContractViolation(Exception):
    """common.hpp:12 -- precondition / invariant breach by the caller."""


class OutOfDeviceMemory(Exception):
    """common.hpp:17 -- simulated device tier cannot hold the bytes."""


class InfeasiblePlan(Exception):
    """common.hpp:22 -- no schedule satisfies the capacity constraints."""


_ERR = {1: ContractViolation, 2: OutOfDeviceMemory, 3: InfeasiblePlan}


def build() -> None:
    """Compile the restatement (and the reference harness where possible)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class _Ledger(C.Structure):
    _fields_ = [
        ("layers", C.c_size_t), ("ntok_cap", C.c_size_t),
        ("capacity", C.c_uint64), ("device_bytes", C.c_uint64), ("host_bytes", C.c_uint64),
        ("row_len", C.POINTER(C.c_size_t)), ("present", C.POINTER(C.c_uint8)),
        ("tier", C.POINTER(C.c_uint8)), ("bytes", C.POINTER(C.c_uint64)),
    ]


class _Plan(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("p1", C.c_size_t),
                ("p2", C.c_size_t), ("recompute_enabled", C.c_int)]


class _Cost(C.Structure):
    _fields_ = [("hidden", C.c_size_t), ("layers", C.c_size_t), ("batch", C.c_size_t),
                ("input_len", C.c_size_t), ("output_len", C.c_size_t),
                ("ratio", C.c_double), ("bandwidth", C.c_double),
                ("bytes_per_element", C.c_size_t), ("device_capacity", C.c_uint64),
                ("mac_rate", C.c_double), ("recompute_overhead", C.c_double)]


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


_D, _I64, _U16, _SZ = C.c_double, C.c_int64, C.c_uint16, C.c_size_t


class RefLedger:
    """The reference's own KvLedger (memsim.hpp:77-215), compiled from the
    unmodified headers (oracle/_ref): driven with the engine's action order
    (engine.hpp:686-716 then store_new) it is the checker for the device
    ledger's byte totals and its OutOfDeviceMemory point and message."""

    OPS = {"store_new": 0, "offload": 1, "reload": 2, "erase": 3, "restore": 4}

    def __init__(self, layers: int, capacity: int):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"reference build missing: {REF_SO}")
        lib = self.lib = C.CDLL(REF_SO)
        lib.ref_ledger_new.restype = C.c_void_p
        lib.ref_ledger_new.argtypes = [_SZ, C.c_uint64]
        lib.ref_ledger_free.argtypes = [C.c_void_p]
        lib.ref_ledger_op.argtypes = [C.c_void_p, C.c_int, _SZ, C.POINTER(_I64), _SZ, C.c_uint64]
        lib.ref_ledger_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.ref_ledger_tiers.argtypes = [C.c_void_p, _SZ, _SZ, C.POINTER(C.c_int8)]
        lib.ref_last_error.restype = C.c_char_p
        self.h = lib.ref_ledger_new(layers, capacity)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_ledger_free(self.h)
            self.h = None

    def op(self, name: str, layer: int, tokens, nbytes: int = 0) -> None:
        t = np.ascontiguousarray(np.asarray(tokens, np.int64).reshape(-1))
        rc = self.lib.ref_ledger_op(self.h, self.OPS[name], layer, _p(t, _I64), t.size, nbytes)
        if rc:
            raise _ERR.get(rc, RuntimeError)(self.lib.ref_last_error().decode())

    def bytes(self):
        d, h = C.c_uint64(), C.c_uint64()
        self.lib.ref_ledger_bytes(self.h, C.byref(d), C.byref(h))
        return d.value, h.value

    def tiers(self, layer: int, ntok: int) -> np.ndarray:
        out = np.zeros(ntok, np.int8)
        self.lib.ref_ledger_tiers(self.h, layer, ntok, _p(out, C.c_int8))
        return out


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in ("port", "reference"):
            raise ValueError(kind)
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            if kind == "port":
                build()
            if not os.path.exists(path):
                raise FileNotFoundError(f"oracle backend missing: {path}")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = "oc_" if kind == "port" else "ref_"
        f = self._f
        f("last_error").restype = C.c_char_p
        f("round_half_even").restype = C.c_int64
        f("round_half_even").argtypes = [_D]
        f("swa_window_k").restype = _SZ
        f("swa_window_k").argtypes = [_SZ, _D]
        f("swa_keep_count").restype = _SZ
        f("swa_keep_count").argtypes = [_SZ, _D]
        f("fill_normal").restype = None
        f("fill_normal").argtypes = [C.c_uint64, _D, C.POINTER(_D), _SZ]
        f("bench_swa").restype = _D
        f("bench_swa").argtypes = [_SZ, _SZ, _SZ, _D, _SZ, _SZ, C.c_uint64]

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc:
            msg = self._f("last_error")().decode()
            raise _ERR.get(rc, RuntimeError)(msg)

    # ---- common / rng ---------------------------------------------------
    def round_half_even(self, x: float) -> int:
        return self._f("round_half_even")(x)

    def fill_normal(self, seed: int, n: int, gain: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._f("fill_normal")(seed, gain, _p(out, _D), n)
        return out

    # ---- attention.hpp -------------------------------------------------
    def swa_window_k(self, n: int, r: float) -> int:
        k = self._f("swa_window_k")(n, r)
        if k == 0:
            raise ContractViolation("swa_window_k: ratio out of (0,1]")
        return k

    def swa_keep_count(self, n: int, r: float) -> int:
        return min(2 * self.swa_window_k(n, r), n)

    def top_k_indices(self, v, k: int) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros(max(k, 1), np.int64)
        self._check(self._f("top_k_indices")(_p(v, _D), _SZ(v.size), _SZ(k), _p(out, _I64)))
        return out[:k]

    def swa_select(self, importance, n: int, r: float):
        """-> (all_ascending, k, local, global) as in SparseSelection."""
        imp = np.ascontiguousarray(importance, np.float64)
        cap = max(n, 1) + 1
        alls, loc, glo = (np.zeros(cap, np.int64) for _ in range(3))
        m, k, nl, ng = _SZ(), _SZ(), _SZ(), _SZ()
        self._check(self._f("swa_select")(
            _p(imp, _D), _SZ(imp.size), _SZ(n), _D(r), _p(alls, _I64), C.byref(m), C.byref(k),
            _p(loc, _I64), C.byref(nl), _p(glo, _I64), C.byref(ng)))
        return alls[:m.value], k.value, loc[:nl.value], glo[:ng.value]

    def attend_over_indices(self, keys, values, acc, acc_len: int, q, idx, n: int):
        """keys/values [H][ncap][D] f64, acc [H][ld] f64 (updated in place),
        q [H][D], idx ascending -> (attn [H][D], new_aw_row [n])."""
        H, ncap, D = keys.shape
        assert acc.flags.c_contiguous and acc.dtype == np.float64
        ld = acc.shape[1]
        idx = np.ascontiguousarray(idx, np.int64)
        q = np.ascontiguousarray(q, np.float64)
        attn = np.zeros((H, D), np.float64)
        aw = np.zeros(max(n, 1), np.float64)
        if self.kind == "port":
            acc[:, acc_len:n] = 0.0
            rc = self.lib.oc_attend_over_indices(
                _SZ(H), _SZ(D), _SZ(n), _SZ(ncap), _p(keys, _D), _p(values, _D), _p(acc, _D),
                _SZ(ld), _p(q, _D), _p(idx, _I64), _SZ(idx.size), _p(attn, _D), _p(aw, _D))
        else:
            rc = self.lib.ref_attend_over_indices(
                _SZ(H), _SZ(D), _SZ(n), _SZ(ncap), _p(keys, _D), _p(values, _D), _p(acc, _D),
                _SZ(ld), _SZ(acc_len), _p(q, _D), _p(idx, _I64), _SZ(idx.size), _p(attn, _D),
                _p(aw, _D))
        self._check(rc)
        return attn, aw[:n]

    def swa_attention(self, keys, values, acc, q, r: float, n: int):
        """State has n tokens appended, accumulators of length n-1."""
        H, ncap, D = keys.shape
        ld = acc.shape[1]
        q = np.ascontiguousarray(q, np.float64)
        attn = np.zeros((H, D), np.float64)
        aw = np.zeros(max(n, 1), np.float64)
        idx = np.zeros(max(n, 1), np.int64)
        m = _SZ()
        if self.kind == "port":
            acc[:, n - 1:n] = 0.0
        self._check(self._f("swa_attention")(
            _SZ(H), _SZ(D), _SZ(n), _SZ(ncap), _p(keys, _D), _p(values, _D), _p(acc, _D),
            _SZ(ld), _p(q, _D), _D(r), _p(attn, _D), _p(aw, _D), _p(idx, _I64), C.byref(m)))
        return attn, aw[:n], idx[:m.value]

    def softmax_rows(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros_like(x)
        self._check(self._f("softmax_rows")(_SZ(x.shape[0]), _SZ(x.shape[1]), _p(x, _D),
                                            _p(out, _D)))
        return out

    def dense_attention(self, q, k, v, causal: bool):
        q, k, v = (np.ascontiguousarray(a, np.float64) for a in (q, k, v))
        sq, D = q.shape
        sk = k.shape[0]
        attn = np.zeros((sq, D), np.float64)
        aw = np.zeros((sq, sk), np.float64)
        self._check(self._f("dense_attention")(_SZ(sq), _SZ(sk), _SZ(D), _p(q, _D), _p(k, _D),
                                               _p(v, _D), C.c_int(int(causal)), _p(attn, _D),
                                               _p(aw, _D)))
        return attn, aw

    def local_attention_mask(self, n: int, window: int) -> np.ndarray:
        f = self._f("local_attention_mask")
        f.restype = _SZ
        out = np.zeros(max(n, 1), np.int64)
        c = f(_SZ(n), _SZ(window), _p(out, _I64))
        if window < 1:
            raise ContractViolation("local_attention_mask: window must be >= 1")
        return out[:c]

    def strided_attention_mask(self, n: int, stride: int) -> np.ndarray:
        f = self._f("strided_attention_mask")
        f.restype = _SZ
        out = np.zeros(max(n, 1), np.int64)
        c = f(_SZ(n), _SZ(stride), _p(out, _I64))
        if stride < 1:
            raise ContractViolation("strided_attention_mask: stride must be >= 1")
        return out[:c]

    def variant_selection(self, variant: str, n: int, r: float, stride: int = 0):
        # engine.hpp:531-569 -> (all ascending, k); importance-free variants only
        if variant == "local":
            w = self.swa_keep_count(n, r)
            out = self.local_attention_mask(n, w)
            return out, out.size
        if stride == 0:
            budget = self.swa_keep_count(n, r)
            stride = max(1, (n + budget - 1) // budget)
        return self.strided_attention_mask(n, stride), 1

    def attention_sparsity(self, aw, rel: float = 0.01, causal: bool = False) -> float:
        aw = np.ascontiguousarray(np.atleast_2d(aw), np.float64)
        f = self._f("attention_sparsity")
        f.restype = _D
        return f(_SZ(aw.shape[0]), _SZ(aw.shape[1]), _p(aw, _D), _D(rel), C.c_int(int(causal)))

    # ---- quant.hpp ------------------------------------------------------
    def quantize(self, x, bits: int = 8, channel_size: int = 0):
        x = np.ascontiguousarray(x, np.float64)
        cs = channel_size or max(x.size, 1)
        groups = max(x.size // cs, 1)
        codes = np.zeros(max(x.size, 1), np.uint16)
        scales = np.zeros(groups, np.float64)
        zps = np.zeros(groups, np.int64)
        self._check(self._f("quantize")(_p(x, _D), _SZ(x.size), C.c_uint32(bits), _SZ(channel_size),
                                        _p(codes, _U16), _p(scales, _D), _p(zps, _I64)))
        return codes[:x.size], scales, zps

    def dequantize(self, codes, channel_size: int, scales, zps):
        codes = np.ascontiguousarray(codes, np.uint16)
        scales = np.ascontiguousarray(scales, np.float64)
        zps = np.ascontiguousarray(zps, np.int64)
        out = np.zeros(codes.size, np.float64)
        self._check(self._f("dequantize")(_p(codes, _U16), _SZ(codes.size), _SZ(channel_size),
                                          _p(scales, _D), _p(zps, _I64), _p(out, _D)))
        return out

    # ---- scheduler.hpp --------------------------------------------------
    def step_actions(self, plan: dict, j: int, selected, k: int, tiers, layers: int,
                     layer: int, input_len: int, output_len: int):
        """tiers: int8 per token of `layer` (-1 absent, 0 device, 1 host, 2 deleted).
        -> dict(phase, offload, delete, reload, recompute)."""
        sel = np.ascontiguousarray(selected, np.int64)
        tiers = np.ascontiguousarray(tiers, np.int8)
        ntok = tiers.size
        outs = [np.zeros(ntok + 1, np.int64) for _ in range(4)]
        cnt = [_SZ() for _ in range(4)]
        phase = C.c_int()
        if self.kind == "reference":
            rc = self.lib.ref_step_actions(
                _D(plan["alpha"]), _D(plan["beta"]), _SZ(plan["p1"]), _SZ(plan["p2"]),
                C.c_int(int(plan.get("recompute_enabled", True))), _SZ(j), _p(sel, _I64),
                _SZ(sel.size), _SZ(k), _p(tiers, C.c_int8), _SZ(ntok), _SZ(layers), _SZ(layer),
                _SZ(input_len), _SZ(output_len), C.byref(phase),
                _p(outs[0], _I64), C.byref(cnt[0]), _p(outs[1], _I64), C.byref(cnt[1]),
                _p(outs[2], _I64), C.byref(cnt[2]), _p(outs[3], _I64), C.byref(cnt[3]))
            self._check(rc)
        else:
            led = _Ledger()
            self._check(self.lib.oc_ledger_init(C.byref(led), _SZ(layers),
                                                C.c_uint64(2 ** 62), _SZ(ntok)))
            try:
                for t in range(ntok):
                    if tiers[t] < 0:
                        continue
                    self._check(self.lib.oc_ledger_store_new(C.byref(led), _SZ(layer), _SZ(t),
                                                             C.c_uint64(1)))
                    one = np.array([t], np.int64)
                    if tiers[t] == 1:
                        self._check(self.lib.oc_ledger_offload(C.byref(led), _SZ(layer),
                                                               _p(one, _I64), _SZ(1), None))
                    elif tiers[t] == 2:
                        self._check(self.lib.oc_ledger_erase(C.byref(led), _SZ(layer),
                                                             _p(one, _I64), _SZ(1), None))
                pl = _Plan(plan["alpha"], plan["beta"], plan["p1"], plan["p2"],
                           int(plan.get("recompute_enabled", True)))
                cost = _Cost(1, layers, 1, input_len, output_len, 1.0, 1.0, 2, 0, 1e9, 1.0)
                rc = self.lib.oc_step_actions(
                    C.byref(pl), _SZ(j), _p(sel, _I64), _SZ(sel.size), _SZ(k), C.byref(led),
                    _SZ(layer), C.byref(cost), C.byref(phase),
                    _p(outs[0], _I64), C.byref(cnt[0]), _p(outs[1], _I64), C.byref(cnt[1]),
                    _p(outs[2], _I64), C.byref(cnt[2]), _p(outs[3], _I64), C.byref(cnt[3]))
                self._check(rc)
            finally:
                self.lib.oc_ledger_free(C.byref(led))
        names = ("offload", "delete", "reload", "recompute")
        res = {nm: o[:c.value].copy() for nm, o, c in zip(names, outs, cnt)}
        res["phase"] = phase.value
        return res

    # ---- CPU timing leg -------------------------------------------------
    def bench_swa(self, H: int, D: int, n: int, r: float, items: int, threads: int,
                  seed: int = 1) -> float:
        return self._f("bench_swa")(H, D, n, r, items, threads, seed)
