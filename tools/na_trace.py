"""Timeline of the NA hand-off chain in CTA 0 (needs a library built with -DWM3_NA_TRACE, loaded via WM3_LIB).
Prints median cycle counts of every wait and of the softmax work per key half."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import ops, _lib
ext, win, heads, dhp = (5, 90, 180), (5, 7, 7), 8, 128
t = 81000
qkv = (torch.randn(t, 3 * heads * dhp, device="cuda") * 1.5).to(_lib.ELEM)
grid = ops.KVGrid(ext, win)
out = torch.empty(t, heads * dhp, device="cuda", dtype=_lib.ELEM)
lib = _lib.lib()
fn = lib.wm3_na_trace
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1 << 16, 3), dtype=np.int64)
for _ in range(3):
    ops.natten(qkv, grid, heads, dhp, dhp, win, out=out)
torch.cuda.synchronize()
fn(buf.ctypes.data, 1 << 16)  # reset
ops.natten(qkv, grid, heads, dhp, dhp, win, out=out)
torch.cuda.synchronize()
n = fn(buf.ctypes.data, 1 << 16)
ev = buf[:n]
ev = ev[np.argsort(ev[:, 2], kind="stable")]
t0 = ev[0, 2]
span = ev[-1, 2] - t0
print(f"{n} events, CTA 0 span {span} cycles")


def pair(b, e):
    """durations end-begin for matching counters"""
    B = {c: tt for k, c, tt in ev if k == b}
    E = {c: tt for k, c, tt in ev if k == e}
    d = np.array([E[c] - B[c] for c in B if c in E])
    return d


names = {(0, 1): "softmax waits sfull", (3, 4): "MMA waits pfull", (7, 8): "MMA waits kfull",
         (10, 11): "TMA waits empty", (12, 13): "softmax waits ofull"}
for (b, e), nm in names.items():
    d = pair(b, e)
    if d.size:
        print(f"{nm:22s} n={d.size:5d} median {np.median(d):8.0f} mean {d.mean():8.0f} total {d.sum():10.0f} "
              f"({d.sum() / span * 100:5.1f} % of span)")
# softmax work per half: from sfull wake (1) to P arrive (2)
d = pair(1, 2)
print(f"{'softmax half work':22s} n={d.size:5d} median {np.median(d):8.0f} mean {d.mean():8.0f} total {d.sum():10.0f} "
      f"({d.sum() / span * 100:5.1f} % of span)")
# MMA: from pfull wake (4) of half h to the sfull wake of the softmax on the next S of that half
W = {c: tt for k, c, tt in ev if k == 1}
A = {c: tt for k, c, tt in ev if k == 2}
lat = np.array([W[c + 2] - A[c] for c in A if c + 2 in W])
print(f"{'P arrive -> next S_h ready':22s} n={lat.size:5d} median {np.median(lat):8.0f}")
V = pair(4, 6)
print(f"{'MMA pfull0 -> vfull':22s} n={V.size:5d} median {np.median(V):8.0f}")
