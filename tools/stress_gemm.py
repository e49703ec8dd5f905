"""Bitwise-repeatability stress of the block GEMMs: each GEMM is run N times on identical inputs and compared
with its first result (a mismatch means a race in the kernel)."""
import os, sys, torch, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import _lib as L, ops
from paper_2503_22235_b200.blocks import RopeTables
T, D = 81000, 1024
E = L.ELEM
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = torch.Generator(device="cuda").manual_seed(0)
hn = torch.randn(T, D, device="cuda", generator=g).to(E)
mid = torch.randn(T, 4 * D, device="cuda", generator=g).to(E)
w2 = (torch.randn(D, 4 * D, device="cuda", generator=g) / 64).to(E)
wo = (torch.randn(D, D, device="cuda", generator=g) / 32).to(E)
w1 = (torch.randn(4 * D, D, device="cuda", generator=g) / 32).to(E)
wq = (torch.randn(3 * D, D, device="cuda", generator=g) / 32).to(E)
b1, b3, b4 = (torch.randn(n, device="cuda", generator=g) for n in (D, 3 * D, 4 * D))
x0 = torch.randn(T, D, device="cuda", generator=g)
rs = RopeTables((5, 90, 180), 128).struct((5, 90, 180), 0, 8, 128)


def resid(a, w):
    def f():
        y = x0.clone()
        ops.linear(a, w, L.WM3_EPI_BIAS_RESID_F32, bias=b1, out=y)
        return y
    return f


cases = {
    "oproj": resid(hn, wo), "w2": resid(mid, w2),
    "w1": lambda: ops.linear(hn, w1, L.WM3_EPI_BIAS_GELU_BF16, bias=b4),
    "qkv": lambda: ops.linear(hn, wq, L.WM3_EPI_QKV_ROPE, bias=b3, rope=rs),
}
bad = {}
t0 = time.time()
for name, f in cases.items():
    ref = f().clone()
    torch.cuda.synchronize()
    n_bad = 0
    for i in range(N):
        if not torch.equal(f(), ref):
            n_bad += 1
    torch.cuda.synchronize()
    bad[name] = n_bad
print(os.environ.get("WM3_LIB", "default"), "mismatches per case", bad, f"({N} runs each, {time.time() - t0:.1f} s)")
