"""Time the block GEMMs with different epilogues (CUDA events), to separate mainloop and epilogue cost."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import _lib, ops
from paper_2503_22235_b200.blocks import RopeTables
L = _lib
T, D = 81000, 1024
E = L.ELEM


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


hn = torch.randn(T, D, device="cuda").to(E)
mid = torch.randn(T, 4 * D, device="cuda").to(E)
wqkv = (torch.randn(3 * D, D, device="cuda") / 32).to(E)
w1 = (torch.randn(4 * D, D, device="cuda") / 32).to(E)
w2 = (torch.randn(D, 4 * D, device="cuda") / 64).to(E)
wo = (torch.randn(D, D, device="cuda") / 32).to(E)
b3, b4, b1 = torch.zeros(3 * D, device="cuda"), torch.zeros(4 * D, device="cuda"), torch.zeros(D, device="cuda")
x = torch.randn(T, D, device="cuda")
out3 = torch.empty(T, 3 * D, device="cuda", dtype=E)
out4 = torch.empty(T, 4 * D, device="cuda", dtype=E)
rope = RopeTables((5, 90, 180), 128)
rs = rope.struct((5, 90, 180), 0, 8, 128)
res = {
    "qkv bias": t(lambda: ops.linear(hn, wqkv, L.WM3_EPI_BIAS_BF16, bias=b3, out=out3)),
    "qkv rope": t(lambda: ops.linear(hn, wqkv, L.WM3_EPI_QKV_ROPE, bias=b3, out=out3, rope=rs)),
    "w1 bias": t(lambda: ops.linear(hn, w1, L.WM3_EPI_BIAS_BF16, bias=b4, out=out4)),
    "w1 gelu": t(lambda: ops.linear(hn, w1, L.WM3_EPI_BIAS_GELU_BF16, bias=b4, out=out4)),
    "o resid": t(lambda: ops.linear(hn, wo, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x)),
    "w2 resid": t(lambda: ops.linear(mid, w2, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x)),
}
fl = {"qkv": 6 * T * D * D, "w1": 8 * T * D * D, "o": 2 * T * D * D, "w2": 8 * T * D * D}
for k, v in res.items():
    print(f"{k:10s} {v:.4f} ms  {fl[k.split()[0]] / v / 1e9:.0f} TFLOP/s")
