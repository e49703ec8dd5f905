"""Run-to-run bitwise check of the full block (same inputs, repeated launches): the determinism the checkpoint / offload parity relies on."""
import numpy as np, torch, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2503_22235_b200 import _lib, ops
from paper_2503_22235_b200.blocks import RopeTables, Workspace, block_forward, prepare_block
from paper_2503_22235_b200.params import init_block_params
ext, win, dim, heads = (5, 90, 180), (5, 7, 7), 1024, 8
params = init_block_params(np.random.default_rng(0), dim, heads, "blk", zero_residual=False)
bw = prepare_block(params, "blk", heads)
rope = RopeTables(ext, dim // heads)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(81000, dim, device="cuda", generator=g)
outs = []
for i in range(4):
    y = x.clone()
    block_forward(y, bw, Workspace(ops.KVGrid(ext, win), bw), rope, ext, win)
    torch.cuda.synchronize()
    outs.append(y)
for i in range(1, 4):
    print("run", i, "bitwise equal to run 0:", torch.equal(outs[i], outs[0]), float((outs[i] - outs[0]).abs().max()))
# per-kernel determinism: GEMM with residual
hn = torch.randn(81000, dim, device="cuda", generator=g).to(_lib.ELEM)
r = []
for i in range(3):
    z = x.clone()
    ops.linear(hn, bw.w_o, _lib.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=z, n_valid=dim)
    torch.cuda.synchronize(); r.append(z)
print("oproj resid deterministic:", torch.equal(r[0], r[1]), torch.equal(r[0], r[2]))
