"""Shared helpers for the parity tests: the oracle-side per-sequence state
(reference AttentionState in the engine's step order) and the tolerance /
tie rules from BASELINE.json's north_star."""
from __future__ import annotations

import numpy as np

# north_star: attention outputs within 1e-3 relative for fp16/bf16, 1e-5 for
# fp32. Relative to the row scale: |g - r| <= tol * (|r| + max|r|).
TOL = {"f32": 1e-5, "f16": 1e-3, "bf16": 1e-3, "u8": 1e-3}
# Selected indices are bit-exact except at importance ties within 1e-6 relative.
TIE_REL = 1e-6


def assert_close(got, ref, tol, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.abs(ref).max(axis=-1, keepdims=True) if ref.ndim else abs(ref)
    err = np.abs(got - ref)
    bound = tol * (np.abs(ref) + scale)
    bad = err > bound
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} elements out of tolerance {tol}; first at {tuple(i)}: "
                             f"got {got[tuple(i)]!r} ref {ref[tuple(i)]!r}; max err {err.max():.3e}")


def err_over_tol(got, ref, tol) -> float:
    """Worst |g - r| / (tol (|r| + max|r|)) over the elements (< 1 passes)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.abs(ref).max(axis=-1, keepdims=True) if ref.ndim else abs(ref)
    return float((np.abs(got - ref) / (tol * (np.abs(ref) + scale))).max())


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp64 data to the device storage dtype and back, so oracle and
    device see identical input values."""
    import torch

    t = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16, "u8": torch.float16}[dtype]
    return torch.from_numpy(np.ascontiguousarray(x)).to(t).to(torch.float64).numpy()


class OracleSeq:
    """One sequence's reference AttentionState (per-head fp64 K/V/accumulators)."""

    def __init__(self, port, H: int, D: int, ncap: int, quant: bool = False):
        self.port, self.H, self.D, self.quant = port, H, D, quant
        self.keys = np.zeros((H, ncap, D))
        self.vals = np.zeros((H, ncap, D))
        self.acc = np.zeros((H, ncap))

    def _store(self, x_hd: np.ndarray) -> np.ndarray:
        # engine.hpp:469-483: fake-quant per head_dim group when enabled
        if not self.quant:
            return x_hd
        flat = np.ascontiguousarray(x_hd).reshape(-1)
        c, s, z = self.port.quantize(flat, 8, self.D)
        return self.port.dequantize(c, self.D, s, z).reshape(x_hd.shape)

    def append(self, t: int, k_hd: np.ndarray, v_hd: np.ndarray) -> None:
        self.keys[:, t] = self._store(k_hd)
        self.vals[:, t] = self._store(v_hd)
        self.acc[:, t] = 0.0

    def seed(self, s: int, q_hd: np.ndarray) -> np.ndarray:
        """engine.hpp:508-512: acc_h = last row of causal dense attention."""
        out = np.zeros((self.H, self.D))
        for h in range(self.H):
            attn, aw = self.port.dense_attention(q_hd[h][None, :], self.keys[h, :s], self.vals[h, :s], True)
            self.acc[h, :s] = aw[0]
            out[h] = attn[0]
        return out

    def importance(self, length: int) -> np.ndarray:
        out = np.zeros(length)
        for h in range(self.H):  # attention.hpp:77-85 order
            out += self.acc[h, :length]
        return out

    def step(self, n: int, r: float, q_hd: np.ndarray):
        return self.port.swa_attention(self.keys, self.vals, self.acc, q_hd, r, n)

    def step_variant(self, n: int, r: float, q_hd: np.ndarray, variant: str, stride: int = 0):
        """Engine::variant_selection (engine.hpp:531-569) + attend_over_indices."""
        if variant in ("swa", "dense"):
            return self.step(n, 1.0 if variant == "dense" else r, q_hd)
        idx, _ = self.port.variant_selection(variant, n, r, stride)
        attn, aw = self.port.attend_over_indices(self.keys, self.vals, self.acc, n - 1, q_hd, idx, n)
        return attn, aw, idx


def selection_flip_is_tie(gpu_idx, ora_idx, imp_pre: np.ndarray, n: int, k: int) -> bool:
    """True when the two selections differ only among global candidates whose
    pre-step importance sits within TIE_REL of the k-th largest value."""
    g, o = set(int(x) for x in gpu_idx), set(int(x) for x in ora_idx)
    diff = g ^ o
    if not diff or any(t >= n - k for t in diff):
        return not diff
    cand = imp_pre[: n - k]
    kth = np.sort(cand)[::-1][k - 1]
    return all(abs(cand[t] - kth) <= TIE_REL * abs(kth) for t in diff)
