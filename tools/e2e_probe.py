"""The serving operator's PCIe bound: attention.NattenBlockStream with page-locked host batches (the bench e2e leg)
against the same pipeline with the block launch removed (uploads / downloads only, same streams and events)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_22235_b200.attention import NattenBlockStream
from paper_2503_22235_b200.params import init_block_params
EXT, WIN, DIM, HEADS = (5, 90, 180), (5, 7, 7), 1024, 8
t = int(np.prod(EXT))
params = init_block_params(np.random.default_rng(0), DIM, HEADS, "blk", zero_residual=False)
r = NattenBlockStream(params, "blk", EXT, WIN, HEADS, DIM)
hin = [torch.randn(t, DIM).pin_memory() for _ in range(2)]
hout = [torch.empty(t, DIM).pin_memory() for _ in range(2)]
def run(n, compute=True):
    for i in range(2): r.submit(hin[i], hout[i])
    r.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(r.s_in)
    for i in range(n): r.submit(hin[i & 1], hout[i & 1])
    e1.record(r.s_out); r.synchronize()
    return e0.elapsed_time(e1) / n
print("e2e", run(20))
# copies only on the same streams, same pattern (no compute)
import paper_2503_22235_b200.attention as A
orig = A.NattenBlockStream.submit
def submit_nocompute(self, host_in, host_out):
    b = self.i % self.NBUF; self.i += 1; dev = self.buf[b]
    with torch.cuda.stream(self.s_in):
        if self.downloaded[b] is not None: self.s_in.wait_event(self.downloaded[b])
        dev.copy_(host_in, non_blocking=True); self.uploaded[b].record(self.s_in)
    with torch.cuda.stream(self.s_out):
        self.s_out.wait_event(self.uploaded[b]); host_out.copy_(dev, non_blocking=True)
        ev = torch.cuda.Event(); ev.record(self.s_out); self.downloaded[b] = ev
A.NattenBlockStream.submit = submit_nocompute
print("copies only, same pipeline", run(20))
A.NattenBlockStream.submit = orig
print("e2e again", run(20))
