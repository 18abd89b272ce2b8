"""GPU parity of the tensor-core prefill against the oracle.

Engine::prefill (engine.hpp:485-529): causal dense_attention per head
(attention.hpp:91-117), each head's accumulator seeded with its last attention
row (engine.hpp:508-512), prefill sparsity = mean over heads of
attention_sparsity(aw, 0.01, causal) (engine.hpp:513-518).

Tolerances: outputs 1e-3 (fp16/bf16 inputs; north_star; bf16 caches with
fp32 outputs), importance 1e-4
relative (fp32 weights on device, like the decode path), sparsity within
2e-3 absolute (cells within fp32 rounding of the 0.01 x max threshold may
count differently).
"""
import numpy as np
import pytest
import torch

from skv_testlib import TOL, OracleSeq, assert_close, round_to, selection_flip_is_tie

pytestmark = pytest.mark.gpu

TD = {"f16": torch.float16, "bf16": torch.bfloat16}


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2403_17312_b200 import api as a

    a.lib()
    return a


def cuda(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


def _case(api, port, dt, B, H, s, ncap, seed, out_f32=False):
    D = 128
    rng = np.random.default_rng(seed)
    k = round_to(rng.standard_normal((B, s, H, D)), dt)
    v = round_to(rng.standard_normal((B, s, H, D)), dt)
    q = round_to(rng.standard_normal((B, s, H, D)) * 0.5, dt)
    cache = api.SwaCache(2, B, H, D, ncap, kv_dtype=dt, out_f32=out_f32)
    layer = 1
    cache.append_tokens(layer, 0, 0, cuda(k, TD[dt]), cuda(v, TD[dt]))
    out = cache.prefill_layer(layer, cuda(q, TD[dt])).float().cpu().numpy()
    imp = cache.importance(layer, s).cpu().numpy()
    sp = cache.prefill_sparsity(layer).cpu().numpy()
    for b in range(B):
        seed_row = np.zeros(s)
        sp_ref = 0.0
        for h in range(H):
            attn, aw = port.dense_attention(q[b, :, h], k[b, :, h], v[b, :, h], True)
            assert_close(out[b, :, h], attn, TOL[dt], f"prefill {dt} b{b} h{h}")
            seed_row += aw[s - 1]
            sp_ref += port.attention_sparsity(aw, 0.01, True)
        np.testing.assert_allclose(imp[b], seed_row, rtol=1e-4, atol=1e-7)
        assert abs(sp[b] - sp_ref / H) <= 2e-3, (b, sp[b], sp_ref / H)
    return cache, (q, k, v)


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("s", [1, 77, 128, 200, 300])
def test_prefill_matches_dense_attention(api, port, dt, s):
    # a bf16 output alone rounds at 2^-9 relative: bf16 caches report fp32
    # outputs (out_f32), as in the decode parity tests
    _case(api, port, dt, B=2, H=4, s=s, ncap=s + 19, seed=s, out_f32=(dt == "bf16"))


def test_prefill_fp32_output(api, port):
    _case(api, port, "f16", B=1, H=2, s=257, ncap=300, seed=3, out_f32=True)


def test_prefill_batch_ragged(api, port):
    # several sequences, one query row past a tile boundary, keys past s in
    # the cache (capacity > s) that TMA must not read
    _case(api, port, "bf16", B=3, H=2, s=129, ncap=140, seed=4, out_f32=True)


def test_prefill_long_prompt(api, port):
    # several query and key tiles, causal tile skipping, the K-range clip of PV
    _case(api, port, "f16", B=1, H=2, s=1100, ncap=1100, seed=11)


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_prefill_long_prompt_cta_pairs(api, port, dt):
    # prompts from s = 1536 take the CTA-pair (cta_group::2) kernel by default;
    # s = 1700 leaves the last 256-query super-tile ragged (rows past s in
    # both CTAs of the pair)
    _case(api, port, dt, B=1, H=2, s=1700, ncap=1710, seed=17, out_f32=(dt == "bf16"))


def test_prefill_then_decode(api, port):
    """Prefill on tensor cores, then SWA decode steps: selections and outputs
    follow the oracle engine order (engine.hpp:592-629)."""
    dt, B, H, D, s, steps, r = "f16", 2, 4, 128, 150, 6, 0.25
    ncap = s + steps
    rng = np.random.default_rng(21)
    kv = round_to(rng.standard_normal((B, ncap, 2, H, D)), dt)
    q0 = round_to(rng.standard_normal((B, s, H, D)) * 0.5, dt)
    qs = round_to(rng.standard_normal((steps, B, H, D)) * 2.0, dt)
    cache = api.SwaCache(1, B, H, D, ncap, kv_dtype=dt, out_f32=True)
    cache.append_tokens(0, 0, 0, cuda(kv[:, :s, 0], TD[dt]), cuda(kv[:, :s, 1], TD[dt]))
    cache.prefill_layer(0, cuda(q0, TD[dt]))
    seqs = [OracleSeq(port, H, D, ncap) for _ in range(B)]
    for b in range(B):
        for t in range(s):
            seqs[b].append(t, kv[b, t, 0], kv[b, t, 1])
        for h in range(H):
            _, aw = port.dense_attention(q0[b, :, h], seqs[b].keys[h, :s], seqs[b].vals[h, :s], True)
            seqs[b].acc[h, :s] = aw[s - 1]
    for j in range(steps):
        n = s + j + 1
        imp_pre = [sq.importance(n - 1) for sq in seqs]
        out, idx, _ = cache.swa_decode_layer(0, n, r, cuda(qs[j], TD[dt]), cuda(kv[:, n - 1, 0], TD[dt]),
                                             cuda(kv[:, n - 1, 1], TD[dt]), return_indices=True)
        out, idx = out.cpu().numpy(), idx.cpu().numpy()
        for b in range(B):
            seqs[b].append(n - 1, kv[b, n - 1, 0], kv[b, n - 1, 1])
            attn, aw, oidx = seqs[b].step(n, r, qs[j][b])
            if not np.array_equal(idx[b], oidx):
                assert selection_flip_is_tie(idx[b], oidx, imp_pre[b], n, api.swa_window_k(n, r)), (j, b)
                return
            assert_close(out[b], attn, TOL[dt], f"decode after prefill step {j}")


def test_prefill_rejects_unsupported_and_bad_shapes(api):
    with pytest.raises(api.Unsupported):  # INT8 storage groups heads by 8
        api.SwaCache(1, 1, 2, 128, 64, kv_dtype="u8", q_dtype="f16")
    c = api.SwaCache(1, 1, 8, 128, 64, kv_dtype="u8", q_dtype="f32")  # INT8 needs fp16 queries
    with pytest.raises(api.Unsupported):
        c.prefill_layer(0, torch.zeros((1, 8, 8, 128), dtype=torch.float32, device="cuda"))
    c = api.SwaCache(1, 1, 2, 128, 64, kv_dtype="f16")
    with pytest.raises(api.ContractViolation):
        c.prefill_layer(0, torch.zeros((1, 65, 2, 128), dtype=torch.float16, device="cuda"))
    with pytest.raises(api.ContractViolation):
        c.prefill_sparsity(0)


@pytest.mark.parametrize("s", [300, 1600])
def test_prefill_int8(api, port, s):
    """INT8 KV (fp16 queries): the layer is dequantised to fp16 for the tensor
    cores; the seed row and the last query's output are redone on the exact
    dequantisation. Reference: dense_attention on the fake-quantised K/V
    (engine.hpp:469-483 groups of D per (token, head))."""
    # s = 1600: the dequantised layer goes through the CTA-pair kernel (config 4's prompt path)
    B, H, D = (2, 8, 128) if s < 1000 else (1, 8, 128)
    rng = np.random.default_rng(88 + s)
    k = round_to(rng.standard_normal((B, s, H, D)), "f16")
    v = round_to(rng.standard_normal((B, s, H, D)), "f16")
    q = round_to(rng.standard_normal((B, s, H, D)) * 0.5, "f16")

    def fake_quant(x):
        flat = np.ascontiguousarray(x).reshape(-1)
        c, sc, z = port.quantize(flat, 8, D)
        return port.dequantize(c, D, sc, z).reshape(x.shape)

    kq, vq = fake_quant(k), fake_quant(v)
    cache = api.SwaCache(1, B, H, D, s + 4, kv_dtype="u8", q_dtype="f16")
    cache.append_tokens(0, 0, 0, cuda(k, torch.float16), cuda(v, torch.float16))
    out = cache.prefill_layer(0, cuda(q, torch.float16)).float().cpu().numpy()
    imp = cache.importance(0, s).cpu().numpy()
    sp = cache.prefill_sparsity(0).cpu().numpy()
    for b in range(B):
        seed_row, sp_ref = np.zeros(s), 0.0
        for h in range(H):
            attn, aw = port.dense_attention(q[b, :, h], kq[b, :, h], vq[b, :, h], True)
            assert_close(out[b, :, h], attn, TOL["u8"], f"int8 prefill b{b} h{h}")
            seed_row += aw[s - 1]
            sp_ref += port.attention_sparsity(aw, 0.01, True)
        np.testing.assert_allclose(imp[b], seed_row, rtol=1e-4, atol=1e-7)
        assert abs(sp[b] - sp_ref / H) <= 2e-3, (b, sp[b], sp_ref / H)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["SKV_PREFILL_2CTA", "SKV_PREFILL_1CTA"])
def test_prefill_both_kernels(kernel):
    """The 1-CTA and the CTA-pair (cta_group::2) prefill kernels are chosen by
    prompt length (skv_prefill.cu); each one, forced for every shape of this
    file, matches the oracle. The switch is read once per process, hence the
    subprocess."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, **{kernel: "1"})
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_prefill.py"), "-k", "not both_kernels"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
