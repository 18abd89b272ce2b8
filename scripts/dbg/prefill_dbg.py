import ctypes as C, sys
import numpy as np, torch
from paper_2403_17312_b200 import api
from paper_2403_17312_b200._lib import lib, check

def run(dt, B=1, H=2, s=77, ncap=96):
    D = 128
    td = {"f16": torch.float16, "bf16": torch.bfloat16}[dt]
    g = torch.Generator().manual_seed(0)
    k = torch.randn(B, s, H, D, generator=g).to(td).cuda()
    v = torch.randn(B, s, H, D, generator=g).to(td).cuda()
    q = (torch.randn(B, s, H, D, generator=g) * 0.5).to(td).cuda()
    c = api.SwaCache(1, B, H, D, ncap, kv_dtype=dt, out_f32=True)
    c.append_tokens(0, 0, 0, k, v)
    out = c.prefill_layer(0, q)
    torch.cuda.synchronize()
    base, nbytes = C.c_void_p(), C.c_size_t()
    check(lib().skv_prefill_scratch(c._h, C.byref(base), C.byref(nbytes)))
    buf = torch.empty(nbytes.value, dtype=torch.uint8, device="cuda")
    check(lib().skv_copy(C.c_void_p(buf.data_ptr()), base, nbytes.value, None))
    torch.cuda.synchronize()
    Z = B * H; ld = (s + 255) // 256 * 256
    al = lambda x: (x + 255) // 256 * 256
    o = 0
    S = buf[o:o + Z * s * ld * 4].view(torch.float32).view(Z, s, ld); o += al(Z * s * ld * 4)
    hv = 2 if dt == "bf16" else 1
    P = buf[o:o + Z * s * ld * 2 * hv].view(td).view(Z, s, ld * hv); o += al(Z * s * ld * 2 * hv)
    P = P[:, :, :ld].float() + (P[:, :, ld:].float() if hv == 2 else 0)
    Vt = buf[o:o + Z * D * ld * 2].view(td).view(Z, D, ld)
    qf, kf, vf = (t.float().permute(0, 2, 1, 3).reshape(Z, s, D) for t in (q, k, v))
    Sref = qf @ kf.transpose(1, 2)
    mask = torch.tril(torch.ones(s, s, dtype=torch.bool, device="cuda"))
    dS = ((S[:, :, :s] - Sref).abs() * mask).max().item()
    print(dt, "S err", dS, "S scale", Sref.abs().max().item())
    Pref = torch.softmax((Sref / D ** 0.5).masked_fill(~mask, float("-inf")), -1)
    print(dt, "P err", (P[:, :, :s].float() - Pref).abs().max().item(), "P beyond", P[:, :, s:ld].float().abs().max().item())
    print(dt, "Vt err", (Vt[:, :, :s].float() - vf.transpose(1, 2)).abs().max().item(), "Vt pad", Vt[:, :, s:].float().abs().max().item())
    Oref = Pref @ vf
    Ogemm = P[:, :, :s].float() @ vf
    of = out.float().permute(0, 2, 1, 3).reshape(Z, s, D)
    print(dt, "out vs ref", (of - Oref).abs().max().item(), "out vs P@V", (of - Ogemm).abs().max().item())
    torch.set_printoptions(precision=5, sci_mode=False)
    print("S", S[0, :3, :4].cpu(), Sref[0, :3, :4].cpu())
    print("P", P[0, :3, :4].float().cpu(), Pref[0, :3, :4].cpu())
    bad = ((P[:, :, :s].float() - Pref).abs() > 1e-2).nonzero()
    print("bad cells", bad.shape[0], bad[:10].tolist())
    print("row0", of[0, 0, :4].tolist(), Oref[0, 0, :4].tolist())

for dt in ("f16", "bf16"):
    run(dt)
