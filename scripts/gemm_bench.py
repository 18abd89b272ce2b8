"""Time the recompute tcgen05 GEMM (skv_gemm_tn) at a few shapes; prints TFLOP/s."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_17312_b200._lib import lib  # noqa: E402

L = lib()
res = []
for (M, N, K) in [(1024, 8192, 4096), (4096, 8192, 4096), (8192, 8192, 4096)]:
    A = torch.randn((M, K), device="cuda").half()
    Bt = (torch.randn((N, K), device="cuda") / K ** 0.5).half()
    Cm = torch.empty((M, N), device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = lambda: L.skv_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(Bt.data_ptr()), C.c_void_p(Cm.data_ptr()),
                              M, N, K, 0, s)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tf = 2 * M * N * K / ms / 1e9
    ref = torch.matmul(A, Bt.T)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        torch.matmul(A, Bt.T)
    e1.record()
    torch.cuda.synchronize()
    res.append({"M": M, "N": N, "K": K, "ms": ms, "tflops": tf, "cublas_fp16_tflops": 2 * M * N * K / (e0.elapsed_time(e1) / 10) / 1e9})
print(json.dumps(res))
