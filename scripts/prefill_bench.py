"""Tensor-core prefill timing: one layer of Engine::prefill's
attention (engine.hpp:485-529) at the BASELINE config shapes, CUDA events on
the launching stream, L2 flushed between iterations. Causal attention FLOPs =
2 GEMMs x 2 x (s(s+1)/2) x D per (sequence, head). flash_attn (a library,
for context only) runs the same causal attention without the seed row /
sparsity outputs.

    python scripts/prefill_bench.py [--iters 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api  # noqa: E402

SHAPES = [  # (name, B, H, s, dtype)
    ("config2 OPT-6.7B f16", 64, 32, 512, "f16"),
    ("config3 OPT-13B bf16", 128, 40, 1024, "bf16"),
    ("config5 b256 s2048 f16", 32, 32, 2048, "f16"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--no-flash", action="store_true", help="skip the flash_attn comparison")
    args = ap.parse_args()
    td = {"f16": torch.float16, "bf16": torch.bfloat16}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    for name, B, H, s, dt in SHAPES:
        D = 128
        g = torch.Generator(device="cuda").manual_seed(0)
        k = torch.randn(B, s, H, D, device="cuda", generator=g).to(td[dt])
        v = torch.randn(B, s, H, D, device="cuda", generator=g).to(td[dt])
        q = (torch.randn(B, s, H, D, device="cuda", generator=g) * 0.5).to(td[dt])
        cache = api.SwaCache(1, B, H, D, s, kv_dtype=dt)
        cache.append_tokens(0, 0, 0, k, v)
        for _ in range(2):
            cache.prefill_layer(0, q)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cache.prefill_layer(0, q)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        flops = 4.0 * B * H * (s * (s + 1) / 2) * D
        line = {"shape": name, "B": B, "H": H, "s": s, "ms": round(ms, 3),
                "tflops": round(flops / ms / 1e9, 1), "tokens_per_s": round(B * s / ms * 1e3),
                "peak_tflops": peaks.get("bf16_tflops")}
        try:
            if args.no_flash:
                raise RuntimeError("skipped (--no-flash)")
            from flash_attn import flash_attn_func

            for _ in range(2):
                flash_attn_func(q, k, v, causal=True)
            torch.cuda.synchronize()
            fts = []
            for _ in range(args.iters):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                flash_attn_func(q, k, v, causal=True)
                e1.record()
                torch.cuda.synchronize()
                fts.append(e0.elapsed_time(e1))
            fms = sorted(fts)[len(fts) // 2]
            line["flash_attn_ms"] = round(fms, 3)
            line["flash_attn_tflops"] = round(flops / fms / 1e9, 1)
        except Exception as ex:  # library absent or unsupported arch
            line["flash_attn"] = f"unavailable: {type(ex).__name__}: {ex}"[:160]
        try:
            # cuDNN's fused attention through torch SDPA (a Blackwell-native library kernel), [B, H, s, D] views
            from torch.nn.attention import SDPBackend, sdpa_kernel

            qt, kt, vt = (x.transpose(1, 2) for x in (q, k, v))
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                for _ in range(2):
                    torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
                torch.cuda.synchronize()
                cts = []
                for _ in range(args.iters):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
                    e1.record()
                    torch.cuda.synchronize()
                    cts.append(e0.elapsed_time(e1))
            cms = sorted(cts)[len(cts) // 2]
            line["cudnn_sdpa_ms"] = round(cms, 3)
            line["cudnn_sdpa_tflops"] = round(flops / cms / 1e9, 1)
        except Exception as ex:
            line["cudnn_sdpa"] = f"unavailable: {type(ex).__name__}: {ex}"[:160]
        print(json.dumps(line), flush=True)
        cache.close()
        del k, v, q
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
