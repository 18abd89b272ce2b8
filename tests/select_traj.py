"""Helper for test_gpu_parity.test_incremental_select_matches_full (run as a
subprocess: SKV_SELECT_FULL is read once per process). Decodes tie-heavy and
random trajectories through the per-layer call (the attend tail's select) and
the whole-step call (the batched select) and saves every step's selection.

    python tests/select_traj.py OUT.npz
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api  # noqa: E402


def run(kind, r, steps, seed, s=60):
    B, H, D, L = 3, 8, 128, 2
    g = torch.Generator(device="cuda").manual_seed(seed)
    ncap = s + steps + 2  # the last step still selects for n + 1
    kv = torch.randn(B, ncap, 2, H, D, device="cuda", generator=g).half()
    qs = torch.randn(steps + 1, L, B, H, D, device="cuda", generator=g).half()
    if kind == "ties":  # zero queries: equal logits, equal weights, importance ties everywhere
        qs.zero_()
    elif kind == "coarse":  # few distinct logit levels: many exact ties among the weights
        qs = (qs * 4).round() / 4
        kv[..., 0, :, :] = (kv[..., 0, :, :] * 2).round() / 2
    c = api.SwaCache(L, B, H, D, ncap, kv_dtype="f16")
    for layer in range(L):
        c.append_tokens(layer, 0, 0, kv[:, :s, 0].contiguous(), kv[:, :s, 1].contiguous())
        c.prefill_seed(layer, s, qs[0, layer].contiguous())
    sel = []
    for j in range(steps):
        n = s + j + 1
        q, kn, vn = qs[j + 1], kv[:, n - 1, 0], kv[:, n - 1, 1]
        if j % 2 == 0:  # whole step: batched select after the attends
            c.swa_decode_step(n, r, q.contiguous(), kn.unsqueeze(0).expand(L, -1, -1, -1).contiguous(),
                              vn.unsqueeze(0).expand(L, -1, -1, -1).contiguous())
        else:  # per-layer calls: the select in the attend tail
            for layer in range(L):
                c.swa_decode_layer(layer, n, r, q[layer].contiguous(), kn.contiguous(), vn.contiguous())
        for layer in range(L):
            sel.append(c.pending_selection(layer, n + 1, r).cpu().numpy().ravel())
    return np.concatenate(sel)


if __name__ == "__main__":
    out = {}
    for kind in ("ties", "coarse", "random"):
        for r in (0.2, 0.5, 0.05):
            out[f"{kind}_{r}"] = run(kind, r, 40, 7)
    # m = 2k > 4 x 128: the fold's long path (k0 < 512 still selects incrementally)
    for kind in ("ties", "random"):
        out[f"long_{kind}"] = run(kind, 0.2, 30, 9, s=2600)
    np.savez(sys.argv[1], **out)
