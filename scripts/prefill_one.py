"""One prefill layer for ncu captures: config-2 shape (B=64, H=32, s=512, fp16, the 1-CTA kernel) or, with
--c5, config 5's prompt (B=32, H=32, s=2048, fp16, the CTA-pair kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api  # noqa: E402

B, H, s, D = (32, 32, 2048, 128) if "--c5" in sys.argv else (64, 32, 512, 128)
dt = torch.bfloat16 if "--bf16" in sys.argv else torch.float16
k = torch.randn(B, s, H, D, device="cuda").to(dt)
v = torch.randn_like(k)
q = torch.randn_like(k) * 0.5
c = api.SwaCache(1, B, H, D, s, kv_dtype="bf16" if dt == torch.bfloat16 else "f16")
c.append_tokens(0, 0, 0, k, v)
for _ in range(3):
    c.prefill_layer(0, q)
torch.cuda.synchronize()
