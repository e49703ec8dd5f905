"""Stress the TMA-residual GEMM epilogue: 1500 residual GEMMs, bitwise re-checks every 100."""
import os, sys, torch, time
sys.path.insert(0, "/root/repo")
from paper_2503_22235_b200 import _lib as L, ops
T, D = 81000, 1024
E = L.ELEM
hn = torch.randn(T, D, device="cuda").to(E); mid = torch.randn(T, 4 * D, device="cuda").to(E)
w2 = (torch.randn(D, 4 * D, device="cuda") / 64).to(E); wo = (torch.randn(D, D, device="cuda") / 32).to(E)
b1 = torch.zeros(D, device="cuda"); x0 = torch.randn(T, D, device="cuda"); x = x0.clone()
ref = x0.clone(); ops.linear(hn, wo, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=ref); torch.cuda.synchronize()
t0 = time.time()
for i in range(1500):
    if i % 100 == 0:
        y = x0.clone()
        ops.linear(hn, wo, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=y); torch.cuda.synchronize()
        assert torch.equal(y, ref), i
    else:
        ops.linear(mid if i % 2 else hn, w2 if i % 2 else wo, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=x)
torch.cuda.synchronize()
print(os.environ.get("WM3_LIB", "default"), "ok", round(time.time() - t0, 1), "s")
