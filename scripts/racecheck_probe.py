"""racecheck helper: the multilayer-step shape (B=4, H=8, s=100, fp16) as
single per-layer launches (no PDL) or one PDL-chained whole step."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api

L, B, H, D, s = 3, 4, 8, 128, 100
g = torch.Generator(device="cuda").manual_seed(0)
c = api.SwaCache(L, B, H, D, s + 2, kv_dtype="f16")
for l in range(L):
    k = torch.randn(B, s, H, D, device="cuda", generator=g).half()
    c.append_tokens(l, 0, 0, k, k)
    c.prefill_seed(l, s, torch.randn(B, H, D, device="cuda", generator=g).half())
q = torch.randn(L, B, H, D, device="cuda", generator=g).half()
if sys.argv[1] == "layers":
    for l in range(L):
        c.swa_decode_layer(l, s + 1, 0.2, q[l].contiguous(), q[l].contiguous(), q[l].contiguous())
else:
    c.swa_decode_step(s + 1, 0.2, q, q, q)
torch.cuda.synchronize()
print("ok", c.attend_config())
