"""Diagnostic (not collected): cuBLAS (torch.matmul) bf16 on the C5 shapes with
random and zero operands: the library reference point for gemm_tc."""
import torch

torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
for M, N, K in ((8192, 4096, 4096), (8192, 4096, 2048), (8192, 8192, 8192)):
    for kind in ("random", "zeros"):
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
        if kind == "zeros":
            a.zero_()
            b.zero_()
        for _ in range(5):
            c = a @ b
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(20):
            c = a @ b
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / 20 * 1e-3
        print("cublas %5d x %5d x %5d %-6s %7.1f us %6.0f TF/s" % (M, N, K, kind, t * 1e6, 2 * M * N * K / t / 1e12))
