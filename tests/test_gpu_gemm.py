"""The tcgen05 GEMM behind recompute_kv (csrc/skv_gemm.cu) against a plain
PyTorch fp32 reference of the same op: C = A . Bt^T, fp16/bf16 in, fp32 out."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def run(lib, A, Bt, bf16):
    M, K = A.shape
    N = Bt.shape[0]
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    st = lib.skv_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(Bt.data_ptr()), C.c_void_p(out.data_ptr()),
                         M, N, K, int(bf16), s)
    assert st == 0, lib.skv_last_error()
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (384, 8192, 4096)])
def test_gemm_tn_matches_torch(dtype, M, N, K):
    from paper_2403_17312_b200._lib import lib

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn((M, K), generator=g, device="cuda").to(dtype)
    Bt = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(dtype)
    got = run(lib(), A, Bt, dtype == torch.bfloat16)
    ref = A.float() @ Bt.float().T
    err = (got - ref).abs().max().item()
    assert err <= 2e-3 * ref.abs().max().item(), err
