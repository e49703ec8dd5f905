"""Isolated timing of the folded-LayerNorm GEMM epilogues vs the plain ones (CUDA events)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import _lib as L, ops
from paper_2503_22235_b200.blocks import RopeTables
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
xh = torch.zeros(T, D, device="cuda", dtype=E)
stats = torch.zeros(T, 2 * L.LN_SLOTS, device="cuda")
rows = torch.zeros(T, 2, device="cuda")
ops.ln_fold_prep(x, D, xh, rows)
rs = RopeTables((5, 90, 180), 128).struct((5, 90, 180), 0, 8, 128)
c3, c4 = torch.ones(3 * D, device="cuda"), torch.ones(4 * D, device="cuda")
cons3 = ops.ln_fold_consumer(rows, c3)
cons4 = ops.ln_fold_consumer(rows, c4)
prod = ops.ln_fold_producer(xh, stats)
res = {
    "qkv rope": t(lambda: ops.linear(hn, wqkv, L.WM3_EPI_QKV_ROPE, bias=b3, out=out3, rope=rs)),
    "qkv rope fold": t(lambda: ops.linear(hn, wqkv, L.WM3_EPI_QKV_ROPE, bias=b3, out=out3, rope=rs, fold=cons3)),
    "w1 gelu": t(lambda: ops.linear(hn, w1, L.WM3_EPI_BIAS_GELU_BF16, bias=b4, out=out4)),
    "w1 gelu fold": t(lambda: ops.linear(hn, w1, L.WM3_EPI_BIAS_GELU_BF16, bias=b4, out=out4, fold=cons4)),
    "o resid": t(lambda: ops.linear(hn, wo, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x)),
    "o resid prod": t(lambda: ops.linear(hn, wo, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x, fold=prod)),
    "w2 resid": t(lambda: ops.linear(mid, w2, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x)),
    "w2 resid prod": t(lambda: ops.linear(mid, w2, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x, fold=prod)),
    "ln": t(lambda: ops.layernorm_bf16(x, b1 + 1, b1, out=xh)),
    "ln prep": t(lambda: ops.ln_fold_prep(x, D, xh, rows)),
    "ln finalize": t(lambda: ops.ln_fold_finalize(stats, 8, D, rows)),
}
for k, v in res.items():
    print(f"{k:16s} {v:.4f} ms")
