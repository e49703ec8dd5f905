"""Debug: one block on a batch of latents vs each latent alone; report the first differing stage."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m
from paper_2503_22235_b200.blocks import Workspace, block_forward
from paper_2503_22235_b200.runtime import CACHE
from paper_2503_22235_b200 import ops, _lib

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
cfg = {"tiny": m.tiny_config, "desk": m.desk_config, "mid": m.mid_config}[name]()
params = m.init_model_params(cfg, seed=7, zero_residual=False)
ext, win = cfg.latent_extents, cfg.window
t = cfg.tokens
B = 3
x = torch.randn(B * t, cfg.hidden, device="cuda")
bw = CACHE.block(params, "proc6.blk0", cfg.heads)
rope = CACHE.rope(ext, cfg.head_dim)
wsb = Workspace(ops.KVGrid(ext, win, batch=B), bw)
ws1 = Workspace(ops.KVGrid(ext, win), bw)
xb = x.clone()
block_forward(xb, bw, wsb, rope, ext, win)
for b in range(B):
    x1 = x[b * t:(b + 1) * t].clone()
    block_forward(x1, bw, ws1, rope, ext, win)
    torch.cuda.synchronize()
    for nm in ["hn", "ctx", "mid"]:
        A = getattr(wsb, nm)[b * t:(b + 1) * t]
        Bq = getattr(ws1, nm)
        print(b, nm, torch.equal(A, Bq), (A.float() - Bq.float()).abs().max().item())
    qa = wsb.grid.interior(wsb.qkv)[b * t:(b + 1) * t]
    q1 = ws1.grid.interior(ws1.qkv)
    print(b, "qkv", torch.equal(qa, q1), (qa.float() - q1.float()).abs().max().item())
    print(b, "x", torch.equal(xb[b * t:(b + 1) * t], x1), (xb[b * t:(b + 1) * t] - x1).abs().max().item())
print("heads", bw.heads, "dhp", bw.dhp, "dh", bw.dh, "ext", ext, "win", win)
