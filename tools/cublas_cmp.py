"""Compare our GEMM (bias-only epilogue) with cuBLAS (torch.matmul, fp16) on the block's GEMM shapes."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import _lib as L, ops
T, D = 81000, 1024


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for name, k, n in [("qkv", D, 3 * D), ("w1", D, 4 * D), ("w2", 4 * D, D), ("o", D, D)]:
    a = torch.randn(T, k, device="cuda").half()
    w = (torch.randn(n, k, device="cuda") / 32).half()
    bias = torch.zeros(n, device="cuda")
    out = torch.empty(T, n, device="cuda", dtype=torch.half)
    fl = 2.0 * T * k * n
    ours = t(lambda: ops.linear(a, w, L.WM3_EPI_BIAS_BF16, bias=bias, out=out))
    wt = w.t()
    cub = t(lambda: torch.matmul(a, wt, out=out))
    print(f"{name}: ours {ours:.4f} ms {fl / ours / 1e9:.0f} TF/s | cuBLAS {cub:.4f} ms {fl / cub / 1e9:.0f} TF/s")
