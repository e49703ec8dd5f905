"""Run the full-shape block a few times (target for ncu)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200.blocks import block_forward
from paper_2503_22235_b200.params import init_block_params
from paper_2503_22235_b200.runtime import CACHE

EXT, WIN, DIM, HEADS = (5, 90, 180), (5, 7, 7), 1024, 8
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t = int(np.prod(EXT))
params = init_block_params(np.random.default_rng(0), DIM, HEADS, "blk", zero_residual=False)
bw = CACHE.block(params, "blk", HEADS)
ws = CACHE.workspace(EXT, WIN, bw)
rope = CACHE.rope(EXT, DIM // HEADS)
x = torch.randn(t, DIM, device="cuda")
for _ in range(n):
    block_forward(x, bw, ws, rope, EXT, WIN)
torch.cuda.synchronize()
print("ok", float(x.abs().mean()))
