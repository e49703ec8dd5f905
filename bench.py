#!/usr/bin/env python
"""Benchmark of the WM-3 forecast hot path on B200 (contract: one JSON line on rank 0).

Metric (BASELINE.json): "14-day 0.25 deg forecast seconds; 3D NATTEN block TFLOP/s at 1/2/4/8 B200".
  value     = 3D NATTEN block TFLOP/s (configs[1]): one pre-norm neighborhood-attention processor block forward
              at the full latent shape (5, 90, 180) = 81000 tokens, D = 1024, 8 heads (dh 128), window (5, 7, 7),
              random-init weights (init_block_params seed 0, zero_residual False), synthetic N(0,1) latent.
              A step = one block applied in place to the fp32 latent as the processor does (attention.py:146-184,
              model.py:402-404): LN1, QKV+rotary GEMM, fused NA, O-proj+residual GEMM, LN2, W1+GELU GEMM,
              W2+residual GEMM (7 launches).  Algorithmic FLOPs 24 T D^2 + 4 T K D = 2.1197e12 per block.
              The 332 MB fp32 latent exceeds the 126 MB L2, so every step streams from HBM (no flush needed).
              N > 1 (torchrun): the latent is split into latitude bands (bands.py), one per rank, with the per-block
              K/V halo exchanged over NCCL: the ranks together process one block per step (strong scaling);
              time = max over ranks.
  e2e       = the same metric through the public API with HOST buffers: pinned host latent (band) -> H2D ->
              block -> D2H, all inside the timed region.
  forecast  = (N = 1) the 14-day forecast of BASELINE configs[4]: forecast(state, 336, params, full_scale_config)
              through the public API from host numpy fields to host fields (encode at 0.25 deg, 56 six-hour
              processor steps replayed as CUDA graphs, decode), random-init full-scale weights, synthetic state.
  roofline  = the dominant kernel of the block (device time), against MEASURED_PEAKS.json.
  cpu_baseline / --impl reference = the float64 oracle (oracle/model.py, the numpy restatement of the
              reference's natten_block) timed on this host on a bounded sample (5, 18, 36) at the same width,
              heads and window.
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
# N > 1: WM3_FUSED_HALO=1 moves the K/V halo rows in the QKV GEMM epilogue over peer memory (bands.PeerHalo)
# for the banded forecast; default is the NCCL point-to-point exchange (bands.HaloExchanger)
FUSED_HALO = os.environ.get("WM3_FUSED_HALO", "0") == "1"
KERNELS = ["layernorm1", "qkv_rope_gemm", "natten", "oproj_resid_gemm", "layernorm2", "w1_gelu_gemm",
           "w2_resid_gemm"]


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


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms while the GPU is under the benchmark load.

    __enter__ returns only once the first sample has been written, so the timed region that follows is
    covered; the sampler spans the timed block steps, the per-kernel breakdown and the e2e steps."""

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
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 5.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
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
def cpu_sample() -> dict:
    from oracle import model as om
    from paper_2503_22235_b200.params import init_block_params
    t = int(np.prod(SAMPLE_EXT))
    params = {k: v.values for k, v in init_block_params(np.random.default_rng(0), DIM, HEADS, "blk",
                                                          zero_residual=False).items()}
    x = np.random.default_rng(2).standard_normal((t, DIM))
    t0 = time.perf_counter()
    om.natten_block(x, params, "blk", SAMPLE_EXT, WIN, HEADS, chunk=128)
    sec = time.perf_counter() - t0
    return {"value": block_flops(t) / sec / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
            "seconds": sec,
            "sample": f"oracle natten_block float64 on {SAMPLE_EXT} (T={t}), D={DIM}, {HEADS} heads, window {WIN}, "
                      f"numpy/OpenBLAS with all {os.cpu_count()} host threads"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    cpu_sample()  # warm-up (imports, BLAS threads, caches)
    secs = [cpu_sample()["seconds"] for _ in range(max(1, args.steps))]
    sec = statistics.mean(secs)
    t = int(np.prod(SAMPLE_EXT))
    value = block_flops(t) / sec / 1e12
    s = cpu_sample()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"natten_block {SAMPLE_EXT} (bounded CPU sample of {EXT}) D={DIM} heads={HEADS} "
                               f"window {WIN}", "tokens": t},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": s["sample"]},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU legs
# ------------------------------------------------------------------------------------------------
def block_setup(world, rank):
    import torch
    from paper_2503_22235_b200 import ops
    from paper_2503_22235_b200.bands import HaloExchanger, plan_bands
    from paper_2503_22235_b200.blocks import RopeTables, Workspace
    from paper_2503_22235_b200.params import init_block_params
    from paper_2503_22235_b200.runtime import CACHE

    params = init_block_params(np.random.default_rng(0), DIM, HEADS, "blk", zero_residual=False)
    bw = CACHE.block(params, "blk", HEADS)
    bands = plan_bands(EXT[1], WIN[1], world)
    me = bands[rank]
    local = (EXT[0], me.rows, EXT[2])
    ws = Workspace(ops.KVGrid(local, WIN, me.halo_lo, me.halo_hi), bw)
    rope = RopeTables(EXT, DIM // HEADS)
    exch = HaloExchanger(bands, rank) if world > 1 else None
    g = torch.Generator(device="cuda").manual_seed(2)
    x_full = torch.randn(int(np.prod(EXT)), DIM, device="cuda", generator=g)
    from paper_2503_22235_b200.bands import local_band_tokens
    x = local_band_tokens(x_full, EXT, me).clone()
    del x_full
    return params, bw, me, local, ws, rope, exch, x


def timed(fn, steps, stream, world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def load_traffic() -> dict:
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the committed ncu capture."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic_r2.json")))["bytes_per_launch"]
    except Exception:
        return {}


def roofline(per_ms: dict, tokens: int, traffic: bool = True) -> tuple[dict, dict]:
    """traffic=False (N > 1: band-sized kernels): no ncu DRAM bytes — the committed capture is of the
    full-domain kernels and does not describe a band's launch."""
    T, D, K = tokens, DIM, int(np.prod(WIN))
    kflops = {"qkv_rope_gemm": 6.0 * T * D * D, "oproj_resid_gemm": 2.0 * T * D * D, "w1_gelu_gemm": 8.0 * T * D * D,
              "w2_resid_gemm": 8.0 * T * D * D, "natten": 4.0 * T * K * D,
              "qkv": 6.0 * T * D * D, "out": 18.0 * T * D * D}
    # algorithmic bytes: LN reads fp32 x and writes the 2-byte operand; NA reads q, k, v and writes ctx
    kbytes = {"layernorm1": T * D * 6.0, "layernorm2": T * D * 6.0, "natten": T * D * 2 * 4.0}
    peaks = load_peaks()
    traffic = load_traffic() if traffic else {}
    top = max((n for n in per_ms if n in kflops or n in kbytes), key=per_ms.get)
    if top in kflops:
        ach = kflops[top] / (per_ms[top] / 1e3) / 1e12
        roof = {"kernel": top, "bound": "tensor", "achieved": ach, "peak": peaks["bf16_sustained"],
                "unit": "TFLOP/s", "frac": ach / peaks["bf16_sustained"], "traffic": traffic.get(top),
                "peak_kind": f"{peaks['source']} bf16 dense, sustained (fp16 operands run at the same rate)"}
    else:
        ach = kbytes[top] / (per_ms[top] / 1e3) / 1e9
        roof = {"kernel": top, "bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                "frac": ach / peaks["hbm"], "traffic": traffic.get(top), "peak_kind": f"{peaks['source']} hbm copy"}
    table = {}
    for n, ms in per_ms.items():
        row = {"ms": round(ms, 5), "dram_bytes_ncu": traffic.get(n)}
        if n in kflops:
            row["tflops"] = round(kflops[n] / (ms / 1e3) / 1e12, 2)
            row["frac_tc"] = round(row["tflops"] / peaks["bf16_sustained"], 4)
        if n in kbytes:
            row["gbs"] = round(kbytes[n] / (ms / 1e3) / 1e9, 1)
            row["frac_hbm"] = round(row["gbs"] / peaks["hbm"], 4)
        if n == "natten":
            hbm_bound_tflops = kflops[n] / (kbytes[n] / (peaks["hbm"] * 1e9)) / 1e12
            row["frac_of_hbm_bound"] = round(row["tflops"] / hbm_bound_tflops, 4)
        table[n] = row
    return roof, table


def measure_backward(reps: int = 3) -> dict:
    """§8f4: the full-shape block's reverse mode on the device (backward.block_vjp_device: forward recompute from
    the block input + backward, fp32 parameter-gradient accumulation), CUDA events; not the headline metric."""
    import torch
    from paper_2503_22235_b200.backward import BlockGrads, block_vjp_device
    from paper_2503_22235_b200.params import init_block_params
    from paper_2503_22235_b200.runtime import CACHE
    t = int(np.prod(EXT))
    params = init_block_params(np.random.default_rng(0), DIM, HEADS, "bwd", zero_residual=False)
    bw = CACHE.block(params, "bwd", HEADS)
    x = torch.randn(t, DIM, device="cuda")
    gy = torch.randn(t, DIM, device="cuda")
    dh = DIM // HEADS
    block_vjp_device(x, bw, EXT, WIN, HEADS, dh, gy, BlockGrads())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        block_vjp_device(x, bw, EXT, WIN, HEADS, dh, gy, BlockGrads())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 3.0 * block_flops(t) / 1e12  # forward recompute + 2x for the backward, algorithmic
    return {"block_vjp_ms": round(ms, 3), "algorithmic_tflop": round(tf, 3), "tflops": round(tf / (ms / 1e3), 1),
            "note": "one full-shape block: forward recompute + backward (dX and all parameter gradients); the "
                    "attention backward on tcgen05 (wm3_natten_bwd: dQ per query tile, dK / dV as per-chunk partials "
                    "reduced per key in a fixed order)"}


def measure_config3(state, params, cfg, reps: int = 3) -> dict:
    """BASELINE configs[2]: full 0.25 deg encode -> one 6 h processor application -> decode through the public API
    (host page-locked fields in, host fields out), each part timed with CUDA events on the launching stream
    (min over `reps`), plus every encoder / decoder conv launch timed individually (pyramid.CONV_HOOK events) with
    its algorithmic FLOPs and fraction of the sustained tensor peak."""
    import torch
    from paper_2503_22235_b200 import model as M
    from paper_2503_22235_b200 import pyramid as P
    from paper_2503_22235_b200.config import conv_flops
    peaks = load_peaks()
    stream = torch.cuda.current_stream()
    lat = M.encode(state, params, cfg)
    lat6 = M.process(lat, params, cfg, 6)
    dec = M.decode(lat6, params, cfg)
    host = dec.to_host()
    torch.cuda.synchronize()

    def ev_time(fn):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best, out

    t_enc, lat = ev_time(lambda: M.encode(state, params, cfg))
    t_proc, lat6 = ev_time(lambda: M.process(lat, params, cfg, 6))
    # decode streams each plane's fields to the page-locked host buffers while the next plane is convolved
    t_dec, _ = ev_time(lambda: M.decode(lat6, params, cfg, host_out=host).to_host(host))
    cf = conv_flops(cfg)
    bf = block_flops(cfg.tokens)
    fl = {"encode": cf["encode_conv"] + cfg.enc_blocks * bf, "process6": cfg.proc_blocks * bf,
          "decode": cf["decode_conv"] + cfg.dec_blocks * bf}
    parts = {}
    for name, ms in (("encode", t_enc), ("process6", t_proc), ("decode", t_dec)):
        tf = fl[name] / (ms / 1e3) / 1e12
        parts[name] = {"ms": round(ms, 3), "tflop": round(fl[name] / 1e12, 3), "tflops": round(tf, 1),
                       "frac_tc": round(tf / peaks["bf16_sustained"], 3)}
    total_ms = t_enc + t_proc + t_dec
    total_tf = sum(fl.values())

    # per-conv launch times (one extra encode + decode with events around every conv launch)
    layers, pending = [], []

    def hook(cw, imgs, h, w, phase):
        if phase == "begin":
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            pending.append((cw, imgs, h, w, ev))
        else:
            cw_, imgs_, h_, w_, e0 = pending.pop()
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            layers.append((cw_, imgs_, h_, w_, e0, e1))

    P.CONV_HOOK = hook
    try:
        lat = M.encode(state, params, cfg)
        n_enc = len(layers)
        M.decode(lat, params, cfg)
        torch.cuda.synchronize()
    finally:
        P.CONV_HOOK = None
    rows = []
    mode_name = {0: "3x3s1", 1: "3x3s2", 2: "4x4s2T"}
    for i, (cw, imgs, h, w, e0, e1) in enumerate(layers):
        ms = e0.elapsed_time(e1)
        f = P.conv_layer_flops(cw, imgs, h, w)
        ho, wo = (h, w) if cw.mode == 0 else ((h // 2, w // 2) if cw.mode == 1 else (2 * h, 2 * w))
        tf = f / (ms / 1e3) / 1e12
        rows.append({"part": "encode" if i < n_enc else "decode", "conv": mode_name[cw.mode], "imgs": imgs,
                     "out_hw": [ho, wo], "cin": cw.cin, "cout": cw.cout, "ms": round(ms, 4),
                     "gflop": round(f / 1e9, 1), "tflops": round(tf, 1),
                     "frac_tc": round(tf / peaks["bf16_sustained"], 3)})
    conv_ms = {p_: sum(r["ms"] for r in rows if r["part"] == p_) for p_ in ("encode", "decode")}
    return {"workload": "full_scale_config encode -> process(6) -> decode, 720x1440, host fields in / out",
            "parts": parts, "total_ms": round(total_ms, 3), "total_tflop": round(total_tf / 1e12, 2),
            "total_tflops": round(total_tf / (total_ms / 1e3) / 1e12, 1),
            "ideal_ms_sustained": round(total_tf / (peaks["bf16_sustained"] * 1e12) * 1e3, 2),
            "conv_tflops": {p_: round(cf[f"{p_}_conv"] / (conv_ms[p_] / 1e3) / 1e12, 1) for p_ in conv_ms},
            "conv_ms": {p_: round(v, 3) for p_, v in conv_ms.items()},
            "conv_layers": rows}


def run_forecast(args, world: int = 1) -> dict:
    """14-day 0.25 deg forecast through the public API, host fields in -> host fields out.  With N > 1 ranks
    the whole forecast is split (bands.forecast_banded): encoder / decoder pyramids by depth plane with
    all-gathers of the token planes and fields, every latent block on latitude bands with the NCCL halo
    exchange per block; time = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2503_22235_b200 import model as M
    from paper_2503_22235_b200 import rollout as R
    from paper_2503_22235_b200.bands import forecast_banded

    def forecast(state, dt, params, cfg, host_out=None):
        if world == 1:
            return R.forecast(state, dt, params, cfg, host_out=host_out)
        return forecast_banded(state, dt, params, cfg, fused=FUSED_HALO)

    def sync_max(sec: float) -> float:
        if world == 1:
            return sec
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = M.full_scale_config()
    t0 = time.perf_counter()
    params = M.init_model_params(cfg, seed=0, zero_residual=False)
    t_init = time.perf_counter() - t0
    g = cfg.grid
    rng = np.random.default_rng(1)
    # host float32 fields in page-locked memory (what a serving process would hold)
    state = M.WeatherState(
        0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).pin_memory(),
        torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32))
        .pin_memory())
    dt = args.forecast_hours
    t0 = time.perf_counter()
    out = forecast(state, dt, params, cfg)   # first call: weight conversion, buffers, graph capture
    host_bufs = out.to_host()                 # pinned output buffers, reused by the timed calls
    torch.cuda.synchronize()
    t_first = time.perf_counter() - t0
    secs = []
    for _ in range(max(1, args.forecast_reps)):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = forecast(state, dt, params, cfg, host_out=host_bufs)  # fields stream out during the decoder
        s_host, a_host = out.to_host(host_bufs)
        torch.cuda.synchronize()
        secs.append(sync_max(time.perf_counter() - t0))
    plan = R.greedy_plan(dt)
    tf_blocks = (len(plan) * cfg.proc_blocks + cfg.enc_blocks + cfg.dec_blocks) * block_flops(cfg.tokens) / 1e12
    finite = bool(np.isfinite(s_host.numpy()).all() and np.isfinite(a_host.numpy()).all())
    res = {"lead_hours": dt, "seconds": min(secs), "seconds_all": [round(s, 4) for s in secs],
           "first_call_seconds": round(t_first, 3), "param_init_host_seconds": round(t_init, 2),
           "block_tflop": round(tf_blocks, 1), "processor_steps": len(plan), "outputs_finite": finite,
           "paper_rtx4090_seconds": 12.0, "gpus": world,
           "latent": "single GPU, CUDA-graph replays" if world == 1 else
                     f"{world} ranks: pyramids by depth plane, blocks on latitude bands with NCCL halo "
                     "exchange per block (bands.forecast_banded)",
           "note": "page-locked host float32 fields in, page-locked host float32 fields out "
                   "(DecodedFields.to_host); H2D/D2H inside the timed region"}
    if world == 1:
        try:
            res["config3"] = measure_config3(state, params, cfg)
        except Exception as exc:
            res["config3"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if args.ensemble > 1:
        # config 5's ensemble: perturbed members, per-member encode / decode, one batched latent rollout; with
        # N ranks the members are sharded round-robin (independent replicas, no communication), time = max
        del out, s_host, a_host
        rank = dist.get_rank() if world > 1 else 0
        mine = [m for m in range(args.ensemble) if m % world == rank]
        all_states = R.perturbed_members(state, args.ensemble, scale=0.01)
        states = [M.WeatherState(all_states[m].valid_time, torch.from_numpy(all_states[m].surface).pin_memory(),
                                 torch.from_numpy(all_states[m].atmos).pin_memory()) for m in mine]
        del all_states
        outs = R.forecast_ensemble(states, dt, params, cfg)   # first call: buffers, graph capture
        bufs = [o.to_host() for o in outs]                      # pinned output buffers, reused below
        del outs
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs = R.forecast_ensemble(states, dt, params, cfg, host_outs=bufs)  # fields stream out per member
        hosts = [o.to_host(b) for o, b in zip(outs, bufs)]
        torch.cuda.synchronize()
        ens_s = sync_max(time.perf_counter() - t0)
        spread = float(np.std([h[0][0].numpy().mean() for h in hosts]))
        # device verification of the ensemble (evaluation.ensemble_curve on the decoded fields in HBM):
        # leading-k ensemble-mean RMSE / blur of surface variable 0 against the unperturbed forecast
        from paper_2503_22235_b200 import evaluation as EV
        ctrl = forecast(state, dt, params, cfg)
        members_dev = torch.stack([o.surface.device[0] for o in outs])[:, None]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        curve = EV.ensemble_curve(members_dev, ctrl.surface.device[0][None], cfg.grid, wavelength_km=2000.0)
        torch.cuda.synchronize()
        t_curve = time.perf_counter() - t0
        res["ensemble"] = {"members": args.ensemble, "gpus": world, "members_per_gpu": len(mine),
                           "seconds": round(ens_s, 4),
                           "seconds_per_member": round(ens_s / args.ensemble, 4),
                           "block_tflop": round(tf_blocks * args.ensemble, 1),
                           "outputs_finite": bool(all(np.isfinite(a.numpy()).all() and np.isfinite(b.numpy()).all()
                                                      for a, b in hosts)),
                           "member_spread_sfc0_mean": spread,
                           "curve_vs_control_sfc0": [{k: (round(v, 6) if isinstance(v, float) else v)
                                                      for k, v in r.items()} for r in curve],
                           "curve_seconds": round(t_curve, 4),
                           "note": "perturbed_members(scale=0.01); batched rollout_ensemble; host fields in/out; "
                                   "curve over this rank's members"}
    return res


def run_gpu(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist

    # WM3_DIST_BACKEND=gloo: host-staged exchanges, for multi-process smoke runs of the N > 1 path on fewer GPUs
    # than ranks (ranks then share devices round-robin; no kernel ever waits on another rank's kernel)
    backend = os.environ.get("WM3_DIST_BACKEND", "nccl")
    device = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    if world > 1:
        if backend == "nccl":
            # communicator lines in the log (ranks, NVLS / NVLink transport) for the scaling run
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    from paper_2503_22235_b200.blocks import block_forward

    params, bw, me, local, ws, rope, exch, x = block_setup(world, rank)
    stream = torch.cuda.current_stream()
    if world > 1:
        # the banded block as the forecast runs it: BandedProcessor (on bands of >= 40 rows the attention is split
        # by query rows, the interior rows overlapping the NCCL halo exchange), with CUDA events between its phases
        from paper_2503_22235_b200.bands import BandedProcessor, plan_bands
        from paper_2503_22235_b200.model import full_scale_config
        cfg = full_scale_config()
        assert cfg.latent_extents == EXT and cfg.window == WIN and cfg.hidden == DIM and cfg.heads == HEADS
        bands = plan_bands(EXT[1], WIN[1], world)
        proc = BandedProcessor(params, cfg, bands, [rank], exch)
        xs = [x]
        phases = ["qkv", "exchange_start", "na_interior", "exchange_wait", "na_boundary", "out", "end"]
        pmarks = []

        def pmark(name):
            if pmarks and name in pmarks[-1]:
                pmarks[-1][name].record(stream)

        proc.timing = pmark

    # per-launch CUDA events recorded on the launching stream inside the timed steps (kernel durations for
    # the roofline are these, averaged over the timed region)
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    cursor = [None]

    def mark(i):
        if cursor[0] is not None:
            cursor[0][i].record(stream)

    # Folded LayerNorm: a step's W2 epilogue leaves x's fp16 copy and row statistics for the next step's QKV
    # GEMM (as between the blocks of a rollout), so after the first warm-up step no separate prep launch runs;
    # that work is inside every timed step's W2 epilogue.
    prepped = [False]

    def step():
        if world > 1:
            proc.run(xs, ["blk"])
            return
        block_forward(x, bw, ws, rope, local, WIN, row0=me.row0, rows_global=EXT[1], halo_exchange=exch, mark=mark,
                      prepped=prepped[0])
        prepped[0] = bw.folded

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(device).__enter__()
    it = iter(marks)

    def timed_step():
        cursor[0] = next(it)
        if world > 1:
            pmarks.append({n: torch.cuda.Event(enable_timing=True) for n in phases})
        step()

    ms = timed(timed_step, args.steps, stream, world)
    cursor[0] = None
    flops = block_flops(int(np.prod(EXT)))
    value = flops * args.steps / (ms / 1e3) / 1e12

    if world > 1:
        # per-phase device time of the banded block (mean over the timed steps); "exchange_wait" is the part of
        # the halo exchange not hidden behind the interior-row attention
        per_ms = {n: sum(pm[n].elapsed_time(pm[phases[i + 1]]) for pm in pmarks) / len(pmarks)
                  for i, n in enumerate(phases[:-1])}
        per_ms["natten"] = per_ms.pop("na_interior") + per_ms.pop("na_boundary")
    else:
        per_ms = {n: sum(ev[i].elapsed_time(ev[i + 1]) for ev in marks) / len(marks) for i, n in enumerate(KERNELS)}
    if bw.folded and world == 1:  # LN1 / LN2 folded into the GEMM epilogues: slot 0 is empty once chained, slot 4 the statistics
        per_ms.pop("layernorm1")
        per_ms["ln_fold_finalize"] = per_ms.pop("layernorm2")
    roof, table = roofline(per_ms, int(np.prod(local)), traffic=(world == 1))

    if world > 1:
        proc.timing = None
    # ---- e2e: pinned host band -> H2D -> block -> D2H ----
    x_host = torch.empty(x.shape, dtype=torch.float32).pin_memory()
    x_host.copy_(x.cpu())
    y_host = torch.empty_like(x_host).pin_memory()
    xd = torch.empty_like(x)
    e_steps = max(3, min(args.steps, 20))
    if world == 1:
        # the public serving operator (attention.NattenBlockStream): page-locked host batches in and out, the
        # uploads / downloads of neighbouring batches overlapped with the block on separate CUDA streams
        from paper_2503_22235_b200.attention import NattenBlockStream
        runner = NattenBlockStream(params, "blk", EXT, WIN, HEADS, DIM)
        hin = [x_host, torch.empty_like(x_host).pin_memory()]
        hin[1].copy_(x_host)
        hout = [y_host, torch.empty_like(y_host).pin_memory()]
        for i in range(2):
            runner.submit(hin[i], hout[i])
        runner.synchronize()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(runner.s_in)
        for i in range(e_steps):
            runner.submit(hin[i & 1], hout[i & 1])
        e1.record(runner.s_out)
        runner.synchronize()
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        e2e_api = ("attention.NattenBlockStream: page-locked host batches, H2D / block / D2H on three CUDA "
                   "streams, neighbouring batches' transfers overlapped")
        # the bound of this leg: the same bytes moved both ways at once with no compute (PCIe, not HBM / SMs)
        for k in range(4):  # each round: both copies start together, the next round starts when both are done
            if k == 1:
                e0.record(runner.s_in)
            runner.s_out.wait_stream(runner.s_in)
            with torch.cuda.stream(runner.s_in):
                runner.buf[0].copy_(hin[0], non_blocking=True)
            with torch.cuda.stream(runner.s_out):
                hout[0].copy_(runner.buf[1], non_blocking=True)
            runner.s_in.wait_stream(runner.s_out)
        e1.record(runner.s_in)
        runner.synchronize()
        link_ms = e0.elapsed_time(e1) / 3
    else:
        def e2e_step():
            xd.copy_(x_host, non_blocking=True)
            proc.run([xd], ["blk"])
            y_host.copy_(xd, non_blocking=True)

        e2e_step()
        e_ms = timed(e2e_step, e_steps, stream, world)
        e2e_api = "BandedProcessor block (overlapped halo exchange) with pinned host copies of the band"
        link_ms = None
    e2e_value = flops * e_steps / (e_ms / 1e3) / 1e12
    clk.__exit__(None, None, None)

    fc = None
    if not args.no_forecast:
        try:
            fc = run_forecast(args, world)
        except Exception as exc:  # keep the block measurement if the (secondary) forecast leg fails
            import traceback
            traceback.print_exc(file=sys.stderr)
            fc = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    bwd = None
    if world == 1 and not args.no_backward:
        try:
            bwd = measure_backward()
        except Exception as exc:
            bwd = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    n_launch = 7
    if world > 1:  # LN1, QKV, O-proj, LN2, W1, W2 + the attention launches of the row split
        a_, z_ = proc.interior[0]  # (row0, row0) when the band's attention runs as one launch
        n_launch = 6 + ((z_ > a_) + (a_ > me.row0) + (z_ < me.row0 + me.rows) if z_ > a_ else 1)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_sample()
            cpu.pop("seconds", None)
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic (random-init weights, N(0,1) latent)",
            "config": {"workload": f"natten_block {EXT} D={DIM} heads={HEADS} window {WIN} (processor block)",
                       "tokens": int(np.prod(EXT)), "block_tflop": round(flops / 1e12, 4), "residual": "fp32",
                       "operands": "fp16 tensor-core operands, fp32 accumulate / residual / softmax",
                       "l2": "inputs larger than L2 (332 MB fp32 latent), no flush",
                       "parallelism": (f"latitude bands x{world} ("
                                       + ("fused QKV-epilogue peer-memory halo" if FUSED_HALO else
                                          f"{os.environ.get('WM3_DIST_BACKEND', 'nccl').upper()} halo")
                                       + ")") if world > 1 else "single GPU",
                       "band_rows_rank0": me.rows,
                       "layernorm": ("folded into the GEMM epilogues: O-proj / W2 write x's fp16 copy and row "
                                     "statistics, QKV / W1 apply the normalisation; steps chained like rollout "
                                     "blocks") if bw.folded else "separate LayerNorm launches"},
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": int(x.numel() * 4),
                    "d2h_bytes_per_step": int(x.numel() * 4), "ms_per_step": e_ms / e_steps,
                    "api": e2e_api,
                    "link_ms_per_step": link_ms,
                    "link_note": ("the step's H2D and D2H bytes copied both ways at once with no compute, same "
                                  "streams and buffers: the PCIe bound of this leg (the block itself takes "
                                  "ms_per_step of the device-timed value)") if link_ms else None},
            "gpu_launches": n_launch * args.steps,
            "roofline": roof,
            "kernels": table,
            "forecast_14d": fc,
            "backward": bwd,
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
    ap.add_argument("--no-forecast", action="store_true", help="skip the 14-day forecast measurement")
    ap.add_argument("--forecast-hours", type=int, default=336)
    ap.add_argument("--forecast-reps", type=int, default=2)
    ap.add_argument("--ensemble", type=int, default=8, help="members of the 14-day ensemble forecast (0/1: skip)")
    ap.add_argument("--no-backward", action="store_true", help="skip the block reverse-mode measurement")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_gpu(args, world, rank, local)


if __name__ == "__main__":
    main()
