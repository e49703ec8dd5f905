"""Time the full-scale NA kernel alone (CUDA events), for quick A/B experiments."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import ops, _lib
ext, win, heads, dhp = (5, 90, 180), (5, 7, 7), 8, 128
t = 81000
qkv = (torch.randn(t, 3 * heads * dhp, device="cuda") * 1.5).to(_lib.ELEM)
grid = ops.KVGrid(ext, win)
out = torch.empty(t, heads * dhp, device="cuda", dtype=_lib.ELEM)
for _ in range(3):
    ops.natten(qkv, grid, heads, dhp, dhp, win, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.natten(qkv, grid, heads, dhp, dhp, win, out=out)
e1.record()
torch.cuda.synchronize()
print(f"NA {os.environ.get('WM3_LIB') or 'default'}: {e0.elapsed_time(e1) / 20:.4f} ms")
