"""Generate the golden fixtures from the UNMODIFIED reference.

Runs the reference library itself (oracle/_ref/libskvref.so, compiled from
/root/reference/proj/include by oracle/Makefile) on seeded inputs and stores
inputs + outputs in tests/golden/golden.npz. The fixtures pin the oracle
restatement (tests/test_oracle.py) on machines where /root/reference is
absent, and are the known answers the GPU parity tests reuse.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main() -> None:
    ref = Oracle("reference")
    g: dict[str, np.ndarray] = {}

    # common.hpp:43-54 (test_matrix.cpp:234-244 plus more)
    xs = np.array([0.5, 1.5, 2.5, -0.5, -1.5, 2.3, 2.7, -2.3, 3.0, 51.5, 52.5, 102.5, -7.5, 1e6 + 0.5])
    g["rne_x"] = xs
    g["rne_y"] = np.array([ref.round_half_even(float(x)) for x in xs], np.int64)

    # matrix.hpp:57-105 SeededRng
    g["rng_normal_seed"] = np.array([2403_17312 + 2], np.uint64)
    g["rng_normal"] = ref.fill_normal(2403_17312 + 2, 64)

    # attention.hpp:122-138 k table
    ns = np.array([1, 2, 3, 4, 5, 9, 10, 11, 100, 512, 513, 515, 525, 768, 1024, 2048, 4096], np.int64)
    rs = np.array([0.05, 0.2, 0.5, 0.8, 1.0])
    g["k_n"], g["k_r"] = ns, rs
    g["k_table"] = np.array([[ref.swa_window_k(int(n), float(r)) for r in rs] for n in ns], np.int64)

    # matrix.hpp:162-176 top-k with ties (coarse grids as in test_matrix.cpp:126-137)
    rng = np.random.default_rng(2024)
    tk_v, tk_k, tk_out = [], [], []
    for rep in range(40):
        ln = int(rng.integers(1, 300))
        v = np.round(rng.random(ln) * (4 if rep % 2 else 4096)) / 8.0
        k = int(rng.integers(0, ln + 1))
        tk_v.append(v)
        tk_k.append(k)
        tk_out.append(ref.top_k_indices(v, k))
    g["topk_lens"] = np.array([v.size for v in tk_v], np.int64)
    g["topk_v"] = np.concatenate(tk_v)
    g["topk_k"] = np.array(tk_k, np.int64)
    g["topk_out"] = np.concatenate(tk_out).astype(np.int64)

    # attention.hpp:142-171 swa_select incl. degenerate branches and RNE ties
    sel_n, sel_r, sel_imp, sel_all = [], [], [], []
    for n in [1, 2, 3, 4, 5, 10, 11, 64, 512, 513, 515, 525, 1024]:
        for r in (0.2, 0.8, 1.0):
            imp = np.round(rng.random(max(n - 1, 0)) * 64) / 64.0  # many exact ties
            alls, _, _, _ = ref.swa_select(imp, n, r)
            sel_n.append(n)
            sel_r.append(r)
            sel_imp.append(imp)
            sel_all.append(alls)
    g["sel_n"] = np.array(sel_n, np.int64)
    g["sel_r"] = np.array(sel_r)
    g["sel_imp"] = np.concatenate(sel_imp)
    g["sel_m"] = np.array([a.size for a in sel_all], np.int64)
    g["sel_all"] = np.concatenate(sel_all).astype(np.int64)

    # quant.hpp:43-95
    qx = [np.array([0.0, 255.0]), np.array([5.0, 5.0, 5.0]), np.array([1.0, 2.0]),
          np.zeros(4), rng.uniform(-1, 1, 256), rng.standard_normal(512) * 3]
    q_bits = [8, 8, 8, 8, 8, 4]
    q_cs = [0, 0, 0, 0, 128, 128]
    qc, qs, qz = [], [], []
    for x, b, cs in zip(qx, q_bits, q_cs):
        c, s, z = ref.quantize(x, b, cs)
        qc.append(c)
        qs.append(s)
        qz.append(z)
    g["q_lens"] = np.array([x.size for x in qx], np.int64)
    g["q_x"] = np.concatenate(qx)
    g["q_bits"] = np.array(q_bits, np.int64)
    g["q_cs"] = np.array(q_cs, np.int64)
    g["q_codes"] = np.concatenate(qc).astype(np.int64)
    g["q_scales"] = np.concatenate(qs)
    g["q_zps"] = np.concatenate(qz)

    # attention.hpp:235-244 multi-step trajectory in the engine's order
    # (append then swa_attention), H=4, D=128, s=48 prompt, 8 steps, r=0.2;
    # inputs are fp16-representable so device runs see identical values.
    H, D, s, steps, r = 4, 128, 48, 8, 0.2
    ncap = s + steps
    kv = ref.fill_normal(2403_17312 + 1, 2 * H * ncap * D).reshape(2, H, ncap, D)
    kv = kv.astype(np.float16).astype(np.float64)
    qs_ = ref.fill_normal(2403_17312 + 11, (steps + 1) * H * D).reshape(steps + 1, H, D)
    qs_ = qs_.astype(np.float16).astype(np.float64)
    keys = np.ascontiguousarray(kv[0])
    vals = np.ascontiguousarray(kv[1])
    acc = np.zeros((H, ncap))
    for h in range(H):  # prefill seed: last row of causal dense attention (engine.hpp:508-512)
        _, aw = ref.dense_attention(qs_[0, h][None, :], keys[h, :s], vals[h, :s], True)
        acc[h, :s] = aw[0]
    g["traj_kv"], g["traj_q"], g["traj_acc0"] = kv, qs_, acc.copy()
    t_attn, t_aw, t_idx = [], [], []
    for j in range(steps):
        n = s + j + 1
        attn, aw, idx = ref.swa_attention(keys, vals, acc, qs_[j + 1], r, n)
        t_attn.append(attn)
        t_aw.append(aw)
        t_idx.append(idx)
    g["traj_attn"] = np.stack(t_attn)
    g["traj_aw"] = np.concatenate(t_aw)
    g["traj_idx"] = np.concatenate(t_idx).astype(np.int64)
    g["traj_m"] = np.array([i.size for i in t_idx], np.int64)
    g["traj_acc_final"] = acc
    g["traj_shape"] = np.array([H, D, s, steps], np.int64)
    g["traj_r"] = np.array([r])

    # scheduler.hpp:320-381 step_actions on random ledgers
    sa_rows = []
    for rep in range(30):
        s_len, out_len = int(rng.integers(4, 40)), int(rng.integers(2, 20))
        j = int(rng.integers(0, out_len))
        n_tot = s_len + j + 1
        tiers = rng.choice([0, 0, 0, 1, 2], size=s_len + j).astype(np.int8)
        plan = {"alpha": float(rng.choice([0.1, 0.3, 0.55, 0.9])), "beta": float(rng.choice([0.05, 0.25, 0.5])),
                "p1": int(rng.integers(0, out_len)), "p2": 0, "recompute_enabled": bool(rep % 3)}
        plan["p2"] = int(rng.integers(plan["p1"], out_len + 1))
        alls, k, _, _ = ref.swa_select(rng.random(n_tot - 1), n_tot, 0.4)
        a = ref.step_actions(plan, j, alls, k, tiers, 2, 1, s_len, out_len)
        sa_rows.append((s_len, out_len, j, plan, tiers, alls, k, a))
    g["sa_meta"] = np.array([[r_[0], r_[1], r_[2], r_[3]["p1"], r_[3]["p2"], int(r_[3]["recompute_enabled"]),
                              r_[6], r_[7]["phase"], r_[4].size, r_[5].size] + [r_[7][nm].size for nm in
                                                                                  ("offload", "delete", "reload",
                                                                                   "recompute")]
                             for r_ in sa_rows], np.int64)
    g["sa_ab"] = np.array([[r_[3]["alpha"], r_[3]["beta"]] for r_ in sa_rows])
    g["sa_tiers"] = np.concatenate([r_[4] for r_ in sa_rows])
    g["sa_sel"] = np.concatenate([r_[5] for r_ in sa_rows]).astype(np.int64)
    g["sa_out"] = np.concatenate([np.concatenate([r_[7][nm] for nm in ("offload", "delete", "reload", "recompute")])
                                  for r_ in sa_rows]).astype(np.int64)

    # attention.hpp:247-269 masks and 275-310 sparsity
    mask_rows = []
    for n in (1, 2, 5, 17, 100, 513):
        for w in (1, 3, 50, 600):
            mask_rows.append((0, n, w, ref.local_attention_mask(n, w)))
        for st in (1, 2, 7, 50):
            mask_rows.append((1, n, st, ref.strided_attention_mask(n, st)))
    g["mask_meta"] = np.array([[a, b, c, len(m)] for a, b, c, m in mask_rows], np.int64)
    g["mask_out"] = np.concatenate([m for *_, m in mask_rows]).astype(np.int64)
    sp_in, sp_out = [], []
    for rep in range(12):
        a = rng.random((3, 40))
        a[a < 0.6] = 0.0
        if rep == 0:
            a[:] = 0.0
        sp_in.append(a)
        sp_out.append([ref.attention_sparsity(a, 0.01, False), ref.attention_sparsity(a, 0.01, True)])
    g["sp_in"] = np.stack(sp_in)
    g["sp_out"] = np.array(sp_out)

    # scheduler.hpp:207-303 solve_plan on small workloads (capacity-constrained
    # and not), via the reference itself
    import ctypes as C
    lib = ref.lib
    plans = []
    for rep in range(24):
        hidden, layers, batch = int(rng.choice([16, 64])), int(rng.integers(1, 4)), int(rng.integers(1, 5))
        s_len, out_len = int(rng.integers(4, 40)), int(rng.integers(2, 30))
        bpe = int(rng.choice([1, 2]))
        tb = 2 * bpe * batch * layers * hidden
        cap = int(tb * (s_len + rng.integers(0, out_len + 4)))
        if rep % 6 == 5:
            cap = tb * s_len - 1  # prompt alone exceeds capacity -> InfeasiblePlan
        ratio = float(rng.choice([0.2, 0.5, 1.0]))
        bw, mac = float(rng.choice([1e3, 1e6, 1e9])), float(rng.choice([1e6, 1e9]))
        ovh = float(rng.choice([1.0, 1.5]))
        po, pr = (C.c_double * 4)(), (C.c_double * 14)()
        rc = lib.ref_solve_plan(C.c_size_t(hidden), C.c_size_t(layers), C.c_size_t(batch), C.c_size_t(s_len),
                                C.c_size_t(out_len), C.c_double(ratio), C.c_double(bw), C.c_size_t(bpe),
                                C.c_uint64(cap), C.c_double(mac), C.c_double(ovh), po, pr)
        plans.append([hidden, layers, batch, s_len, out_len, ratio, bw, bpe, cap, mac, ovh, rc] + list(po) + list(pr))
    g["plan_rows"] = np.array(plans, np.float64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
