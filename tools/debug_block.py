import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import ops, _lib
from paper_2503_22235_b200.params import init_block_params
from paper_2503_22235_b200.runtime import CACHE
ext, win, dim, heads = eval(sys.argv[1])
t = int(np.prod(ext))
params = init_block_params(np.random.default_rng(0), dim, heads, "blk", zero_residual=False)
bw = CACHE.block(params, "blk", heads)
ws = CACHE.workspace(ext, win, bw)
rope = CACHE.rope(ext, dim // heads)
x = torch.randn(t, dim, device="cuda")
def step(name, fn):
    fn(); torch.cuda.synchronize(); print("ok", name, flush=True)
step("ln", lambda: ops.layernorm_bf16(x, bw.ln1_g, bw.ln1_b, out=ws.hn))
rs = rope.struct(ext, 0, bw.heads, bw.dhp)
step("qkv_plain", lambda: ops.linear(ws.hn, bw.w_qkv, _lib.WM3_EPI_QKV_ROPE, bias=bw.b_qkv, out=torch.empty(t, 3*heads*bw.dhp, device="cuda", dtype=torch.bfloat16), rope=rs))
step("bias_grid", lambda: ops.linear_grid(ws.hn, bw.w_qkv, _lib.WM3_EPI_BIAS_BF16, bw.b_qkv, ws.qkv, ws.grid))
step("qkv_grid", lambda: ops.linear_grid(ws.hn, bw.w_qkv, _lib.WM3_EPI_QKV_ROPE, bw.b_qkv, ws.qkv, ws.grid, rope=rs))

step("na", lambda: ops.natten(ws.qkv, ws.grid, bw.heads, bw.dhp, bw.dh, win, out=ws.ctx))
