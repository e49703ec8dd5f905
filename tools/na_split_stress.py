"""Repeat the band attention row-split comparison (tests/test_bands_gpu.py::test_natten_row_split_bitwise) and
report every mismatch: which launch pattern, how many elements, NaN (unwritten) or numeric, which query rows."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import _lib, ops
from paper_2503_22235_b200.bands import interior_rows, plan_bands

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
ext, win, heads, dhp = (5, 90, 180), (5, 7, 7), 8, 128
d, h, w = ext
C = 3 * heads * dhp
g = torch.Generator(device="cuda").manual_seed(5)
qkv = (torch.randn(d * h * w, C, device="cuda", generator=g) * 1.5).to(_lib.ELEM)
g3 = qkv.view(d, h, w, C)
bands = plan_bands(h, win[1], 8)[:3]
bad = 0
for it in range(N):
    for b in bands:
        grid = ops.KVGrid((d, b.rows, w), win, b.halo_lo, b.halo_hi)
        buf = g3[:, b.row0 - b.halo_lo:b.row0 + b.rows + b.halo_hi].reshape(-1, C).contiguous()
        one = ops.natten(buf, grid, heads, dhp, dhp, win, rows_global=h, row0=b.row0)
        one2 = ops.natten(buf, grid, heads, dhp, dhp, win, rows_global=h, row0=b.row0)
        a, z = interior_rows(b, h, win[1])
        split = torch.full_like(one, float("nan"))
        for lo, hi in ((a, z), (b.row0, a), (z, b.row0 + b.rows)):
            if hi > lo:
                ops.natten(buf, grid, heads, dhp, dhp, win, out=split, rows_global=h, row0=b.row0, q_rows=(lo, hi))
        torch.cuda.synchronize()
        for name, x in (("repeat", one2), ("split", split)):
            if not torch.equal(x, one):
                bad += 1
                diff = (x.float() - one.float())
                nan = torch.isnan(x).any(dim=1)
                rows = torch.nonzero((diff.abs() > 0).any(dim=1) | nan).flatten()
                tok = rows.cpu()
                r_of = ((tok // w) % b.rows + b.row0).unique().tolist()
                heads_bad = torch.nonzero((diff.abs() > 0).view(-1, heads, dhp).any(dim=2).any(dim=0)).flatten().tolist()
                print(f"iter {it} band {b.rank} {name}: {int(rows.numel())} tokens differ, NaN tokens {int(nan.sum())}, "
                      f"max |diff| {float(diff[~torch.isnan(diff)].abs().max()) if (~torch.isnan(diff)).any() else 0:.3e}, "
                      f"global rows {r_of[:12]}, heads {heads_bad}")
print(f"done: {bad} mismatches in {N} iterations x {len(bands)} bands")
