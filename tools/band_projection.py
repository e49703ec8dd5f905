"""Compute side of the latitude-band split, measured on ONE B200: for N = 1, 2, 4, 8 bands, each band's processor
block (LN1 + QKV into its halo'd K/V grid, attention of its rows, O-proj + MLP) is timed alone with CUDA events —
the work one rank does per block at N GPUs.  The halo rows are not exchanged here (the kernels run on whatever the
halo slots hold: same work, no bytes moved); at N GPUs the exchange (K / V columns of <= 3 rows per neighbour,
~11 MB over NVLink) overlaps the interior-row attention.  Projected N-GPU block time = the slowest band's time.
Not a multi-GPU measurement: ranks are never emulated by kernels waiting on one another."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as M
from paper_2503_22235_b200.bands import BandedProcessor, plan_bands

cfg = M.full_scale_config()
params = M.init_model_params(cfg, seed=0, zero_residual=False)
d, h, w = cfg.latent_extents
flops = 2.1197e12
prefix = "proc6.blk0"


class NoExchange:
    """Stands in for the NCCL exchanger: the halo slots keep their content (timing only)."""

    def start(self, qkv, grid):
        return None

    def wait(self, handle):
        return None


out = {}
for n in (1, 2, 4, 8):
    bands = plan_bands(h, cfg.window[1], n)
    times = []
    for i, b in enumerate(bands):
        proc = BandedProcessor(params, cfg, bands, [i], exchanger=NoExchange())
        x = torch.randn(d * b.rows * w, cfg.hidden, device="cuda")
        for _ in range(3):
            proc.run([x], [prefix])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            proc.run([x], [prefix])
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / reps)
    worst = max(times)
    out[n] = {"band_rows": [b.rows for b in bands], "band_ms": [round(t, 4) for t in times],
              "projected_block_ms": round(worst, 4), "projected_tflops": round(flops / (worst / 1e3) / 1e12, 1)}
    print(f"[WM3_NA_SPLIT={os.environ.get('WM3_NA_SPLIT', 'auto')}] N={n}: rows {out[n]['band_rows']} band ms {out[n]['band_ms']} -> block {worst:.4f} ms = "
          f"{out[n]['projected_tflops']} TFLOP/s, efficiency vs N=1 {out[1]['projected_block_ms'] / (n * worst):.3f}")
print(json.dumps(out))

# per-kernel split of one band at N = 8 against the whole grid (device times from the profiler, one block)
if os.environ.get("BAND_KERNELS", "1") == "1":
    for n, i in ((1, 0), (8, 2)):
        bands = plan_bands(h, cfg.window[1], n)
        proc = BandedProcessor(params, cfg, bands, [i], exchanger=NoExchange())
        x = torch.randn(d * bands[i].rows * w, cfg.hidden, device="cuda")
        proc.run([x], [prefix])
        torch.cuda.synchronize()
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            proc.run([x], [prefix])
            torch.cuda.synchronize()
        rows = [(e.name.split("(")[0][:48], e.device_time / 1e3) for e in prof.events() if e.device_type.name == "CUDA"]
        print(f"N={n} band {i} ({bands[i].rows} rows): " +
              ", ".join(f"{k} {v:.4f}" for k, v in rows) + f" | sum {sum(v for _, v in rows):.4f} ms")
