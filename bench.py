#!/usr/bin/env python
"""Benchmark of the WM-3 forecast hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the metric's "3D NATTEN block TFLOP/s"): one pre-norm neighborhood-
attention processor block forward at the full latent shape (5, 90, 180) = 81000 tokens, D = 1024, 8 heads
(dh 128), window (5, 7, 7), random-init weights (init_block_params seed 0, zero_residual False) and a
synthetic N(0,1) latent.  A step = one block forward (7 kernel launches: LN1, QKV+rotary GEMM, fused NA,
O-proj+residual GEMM, LN2, W1+GELU GEMM, W2+residual GEMM) applied in place to the fp32 latent, as the
processor does (attention.py:146-184, model.py:402-404).  The latent is 332 MB fp32 (> 126 MB L2), so
every step streams from HBM without an explicit flush.

value      = algorithmic block FLOPs (24 T D^2 + 4 T K D = 2.1197e12) x steps x ranks / max-over-ranks time
e2e        = same metric through the public API natten_block() with a pinned host fp32 latent: H2D copy,
             block, D2H copy of the result, all inside the timed region
roofline   = dominant kernel (by device time) against the measured bf16 peak (MEASURED_PEAKS.json)
cpu_baseline / --impl reference = the float64 oracle (oracle/model.py, a numpy restatement of the
             reference's natten_block) on a bounded sample (5, 18, 36) of the same width/heads/window.

N > 1 (torchrun): each rank runs its own replica of the block (weak scaling); max-over-ranks timing.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EXT = (5, 90, 180)
WIN = (5, 7, 7)
DIM, HEADS = 1024, 8
SAMPLE_EXT = (5, 18, 36)
METRIC = "3D NATTEN block TFLOP/s"


def block_flops(tokens: int, dim: int = DIM, keys: int = int(np.prod(WIN))) -> float:
    return 24.0 * tokens * dim * dim + 4.0 * tokens * keys * dim


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"bf16": d.get("bf16_tflops", 1590.0), "bf16_sustained": d.get("bf16_tflops_sustained", 1400.0),
                "hbm": d.get("hbm_gbs", 6650.0), "source": "measured"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        try:
            rows = [ln.split(",") for ln in open(self.path).read().strip().splitlines() if ln.strip()]
        except Exception:
            rows = []
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# CPU legs (oracle = float64 numpy restatement of the reference path)
# ------------------------------------------------------------------------------------------------
def cpu_sample(repeats: int = 1) -> dict:
    from oracle import model as om
    from paper_2503_22235_b200.params import init_block_params
    t = int(np.prod(SAMPLE_EXT))
    params = {k: v.values for k, v in init_block_params(np.random.default_rng(0), DIM, HEADS, "blk",
                                                          zero_residual=False).items()}
    x = np.random.default_rng(2).standard_normal((t, DIM))
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        om.natten_block(x, params, "blk", SAMPLE_EXT, WIN, HEADS, chunk=128)
        times.append(time.perf_counter() - t0)
    sec = min(times)
    return {"value": block_flops(t) / sec / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(),
            "kind": "port", "seconds": sec,
            "sample": f"oracle natten_block float64 on {SAMPLE_EXT} (T={t}), D={DIM}, {HEADS} heads, window {WIN}"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    samples = []
    for _ in range(max(1, args.steps)):
        samples.append(cpu_sample(1))
    secs = [s["seconds"] for s in samples]
    sec = max(secs)
    t = int(np.prod(SAMPLE_EXT))
    value = block_flops(t) / sec / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"natten_block {SAMPLE_EXT} (bounded CPU sample of {EXT}) D={DIM} heads={HEADS} "
                               f"window {WIN}", "tokens": t},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": samples[0]["sample"]},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU leg
# ------------------------------------------------------------------------------------------------
def run_gpu(args, world, rank, local):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2503_22235_b200 import attention as A
    from paper_2503_22235_b200.blocks import block_forward
    from paper_2503_22235_b200.params import init_block_params
    from paper_2503_22235_b200.runtime import CACHE

    t = int(np.prod(EXT))
    params = init_block_params(np.random.default_rng(0), DIM, HEADS, "blk", zero_residual=False)
    bw = CACHE.block(params, "blk", HEADS)
    ws = CACHE.workspace(EXT, WIN, bw)
    rope = CACHE.rope(EXT, DIM // HEADS)
    g = torch.Generator(device="cuda").manual_seed(2 + rank)
    x = torch.randn(t, DIM, device="cuda", generator=g)
    stream = torch.cuda.current_stream()

    def step():
        block_forward(x, bw, ws, rope, EXT, WIN)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, CUDA events, barrier + sync on both sides ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    flops = block_flops(t)
    value = flops * args.steps * world / (ms_max / 1e3) / 1e12

    # ---- per-kernel breakdown (events around each launch, same stream) ----
    from paper_2503_22235_b200 import _lib, ops
    names = ["layernorm1", "qkv_rope_gemm", "natten", "oproj_resid_gemm", "layernorm2",
             "w1_gelu_gemm", "w2_resid_gemm"]
    L = _lib

    def launches():
        rs = rope.struct(EXT, 0, bw.heads, bw.dhp)
        return [
            lambda: ops.layernorm_bf16(x, bw.ln1_g, bw.ln1_b, out=ws.hn),
            lambda: ops.linear_grid(ws.hn, bw.w_qkv, L.WM3_EPI_QKV_ROPE, bw.b_qkv, ws.qkv, ws.grid, rope=rs),
            lambda: ops.natten(ws.qkv, ws.grid, bw.heads, bw.dhp, bw.dh, WIN, out=ws.ctx),
            lambda: ops.linear(ws.ctx, bw.w_o, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=x, n_valid=bw.hidden),
            lambda: ops.layernorm_bf16(x, bw.ln2_g, bw.ln2_b, out=ws.hn),
            lambda: ops.linear(ws.hn, bw.w_1, L.WM3_EPI_BIAS_GELU_BF16, bias=bw.b_1, out=ws.mid),
            lambda: ops.linear(ws.mid, bw.w_2, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_2, out=x, n_valid=bw.hidden),
        ]

    fns = launches()
    reps = max(3, min(args.steps, 10))
    acc = [0.0] * len(fns)
    for _ in range(reps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)]
        evs[0].record(stream)
        for i, fn in enumerate(fns):
            fn()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        for i in range(len(fns)):
            acc[i] += evs[i].elapsed_time(evs[i + 1])
    per_kernel_ms = {n: a / reps for n, a in zip(names, acc)}
    T, D, K = t, DIM, int(np.prod(WIN))
    kflops = {"qkv_rope_gemm": 6.0 * T * D * D, "oproj_resid_gemm": 2.0 * T * D * D,
              "w1_gelu_gemm": 8.0 * T * D * D, "w2_resid_gemm": 8.0 * T * D * D, "natten": 4.0 * T * K * D}
    kbytes = {"layernorm1": T * D * (4 + 2), "layernorm2": T * D * (4 + 2),
              "natten": T * D * 2 * 4}  # q, k, v in + ctx out, bf16
    top = max(per_kernel_ms, key=per_kernel_ms.get)
    peaks = load_peaks()
    if top in kflops:
        ach = kflops[top] / (per_kernel_ms[top] / 1e3) / 1e12
        roof = {"kernel": top, "bound": "tensor", "achieved": ach, "peak": peaks["bf16_sustained"],
                "unit": "TFLOP/s", "frac": ach / peaks["bf16_sustained"], "traffic": None,
                "peak_kind": f"{peaks['source']} bf16 sustained"}
    else:
        ach = kbytes[top] / (per_kernel_ms[top] / 1e3) / 1e9
        roof = {"kernel": top, "bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                "frac": ach / peaks["hbm"], "traffic": None, "peak_kind": f"{peaks['source']} hbm"}
    kernel_table = {}
    for n in names:
        row = {"ms": per_kernel_ms[n]}
        if n in kflops:
            row["tflops"] = kflops[n] / (per_kernel_ms[n] / 1e3) / 1e12
        if n in kbytes:
            row["gbs"] = kbytes[n] / (per_kernel_ms[n] / 1e3) / 1e9
        kernel_table[n] = row

    # ---- e2e through the public API with pinned host buffers ----
    x_host = torch.randn(t, DIM, generator=torch.Generator().manual_seed(7)).pin_memory()
    y_host = torch.empty_like(x_host).pin_memory()

    def e2e_step():
        out = A.natten_block(x_host, params, "blk", EXT, WIN, HEADS)
        y_host.copy_(out.device, non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_steps = max(1, min(args.steps, 10))
    t0 = time.perf_counter()
    c0 = torch.cuda.Event(enable_timing=True)
    c1 = torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(e_steps):
        e2e_step()
    c1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e2e_s = max(wall, c0.elapsed_time(c1) / 1e3)
    e_t = torch.tensor([e2e_s], device="cuda")
    if world > 1:
        dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
    e2e_value = flops * e_steps * world / float(e_t.item()) / 1e12

    if rank == 0:
        cpu = cpu_sample(1) if (world == 1 and not args.no_cpu) else None
        if cpu is not None:
            cpu.pop("seconds", None)
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"natten_block {EXT} D={DIM} heads={HEADS} window {WIN} (processor block)",
                       "tokens": t, "block_tflop": flops / 1e12, "residual": "fp32",
                       "l2": "inputs larger than L2 (332 MB fp32 latent)", "parallelism": f"replicas x{world}"},
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": t * DIM * 4,
                    "d2h_bytes_per_step": t * DIM * 4},
            "gpu_launches": 7 * args.steps,
            "roofline": roof,
            "kernels": kernel_table,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_gpu(args, world, rank, local)


if __name__ == "__main__":
    main()
