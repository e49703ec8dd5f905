"""Probe of the tcgen05 MMA issue latency / throughput (tools/csrc/mma_probe.cu built as a separate library; not part of the product ABI)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
from paper_2503_22235_b200 import _lib
# profiling aid, not part of the public ABI: `make probe` builds tools/libmma_probe.so
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmma_probe.so"))
lib.mma_probe.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 2
for ctas in (148,):
    for mode, n in [(16, 128), (17, 128), (18, 128), (16, 256), (17, 256), (0, 128), (1, 128)]:
        out = torch.zeros(ctas, dtype=torch.int64, device="cuda")
        reps = 200
        _lib.check(lib.mma_probe(mode, n, reps, ctas, out.data_ptr(), _lib.stream_ptr()), "probe")
        torch.cuda.synchronize()
        cyc = out.float().mean().item() / (reps * 8)
        print(f"ctas={ctas} mode={mode} N={n}: {cyc:.1f} cycles per 128x{n}x16 MMA (floor {128 * n / 256:.0f})")
