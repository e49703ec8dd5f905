import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import ops, _lib
D, H, W, pad = (int(v) for v in sys.argv[1:5])
t = D * H * W
n, k = 256, 128
a = torch.randn(t, k, device="cuda").to(torch.bfloat16)
w = torch.randn(n, k, device="cuda").to(torch.bfloat16)
b = torch.zeros(n, device="cuda")
class G: pass
g = ops.KVGrid((D, H, W), (1, 1, 2 * pad + 1))
out = torch.zeros(g.tokens, n, device="cuda", dtype=torch.bfloat16)
ops.linear_grid(a, w, _lib.WM3_EPI_BIAS_BF16, b, out, g)
torch.cuda.synchronize()
ref = (a.float() @ w.float().T)
got = g.interior(out).float()
print("ok", D, H, W, pad, float((got - ref).abs().max()))
