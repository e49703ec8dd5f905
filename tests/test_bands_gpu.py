"""Latitude-band path on one B200: every band of a full-width block is computed with the band kernels (QKV GEMM
into a halo'd K/V grid with global-row rotary phases, NA with row0/halos) and must reproduce the single-band
result.  The halo exchange is emulated by device copies between the bands' buffers (the multi-process
NCCL/gloo exchange itself is covered by tests/test_bands_cpu.py); no kernel ever waits on another."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _na_gather_rel(qkv, out, ext, heads, dhp, win, tok_chunk=2048):
    """Per-token squared error and reference norm of the fused attention `out` (T, heads * dhp) against an fp32
    gather over the reference's global neighbor table (oracle.grid.neighborhood = grid.py:107-130), evaluated in
    token chunks so the full (5, 90, 180) shape fits."""
    from oracle.grid import neighborhood
    t = qkv.shape[0]
    tab = torch.from_numpy(neighborhood(ext, win)).cuda()
    sec = heads * dhp
    q = qkv[:, :sec].float().view(t, heads, dhp)
    k = qkv[:, sec:2 * sec].float().view(t, heads, dhp)
    v = qkv[:, 2 * sec:3 * sec].float().view(t, heads, dhp)
    err = torch.empty(t, device="cuda", dtype=torch.float64)
    ref2 = torch.empty(t, device="cuda", dtype=torch.float64)
    for a in range(0, t, tok_chunk):
        b = min(a + tok_chunk, t)
        kn, vn = k[tab[a:b]], v[tab[a:b]]
        s = torch.einsum("thd,tkhd->thk", q[a:b], kn) / math.sqrt(dhp)
        ref = torch.einsum("thk,tkhd->thd", torch.softmax(s, dim=-1), vn).reshape(b - a, sec)
        err[a:b] = ((out[a:b].float() - ref) ** 2).sum(1).double()
        ref2[a:b] = (ref ** 2).sum(1).double()
    return err, ref2


@pytest.mark.parametrize("ext,heads", [((5, 90, 180), 8), ((5, 18, 72), 2)])
def test_band_natten_bitwise_and_vs_gather(ext, heads):
    """Band attention (row0 / halo rows, global rotary rows and bumps) for every band of the 2-, 4- and 8-band
    plans: bitwise equal to the rows of the single-band kernel (query tiles are aligned to global rows, so a
    query sees the same key chunks in the same order), and the single-band result within 2e-3 relative L2 of
    an fp32 gather over the reference's global neighbor table — per band as well as overall."""
    from paper_2503_22235_b200 import _lib, ops
    from paper_2503_22235_b200.bands import plan_bands
    win, dhp = (5, 7, 7), 128
    d, h, w = ext
    t = d * h * w
    C = 3 * heads * dhp
    g = torch.Generator(device="cuda").manual_seed(11)
    qkv = (torch.randn(t, C, device="cuda", generator=g) * 1.5).to(_lib.ELEM)
    full = ops.natten(qkv, ops.KVGrid(ext, win), heads, dhp, dhp, win)
    err, ref2 = _na_gather_rel(qkv, full, ext, heads, dhp, win)
    rel = float((err.sum() / ref2.sum()).sqrt())
    print(f"NA vs fp32 gather {ext}: rel L2 {rel:.2e}")
    assert rel < 2e-3, rel
    err = err.view(d, h, w)
    ref2 = ref2.view(d, h, w)
    g3 = qkv.view(d, h, w, C)
    f3 = full.view(d, h, w, -1)
    for world in (2, 4, 8):
        if h < 7 * world:
            continue
        for b in plan_bands(h, win[1], world):
            grid = ops.KVGrid((d, b.rows, w), win, b.halo_lo, b.halo_hi)
            buf = g3[:, b.row0 - b.halo_lo:b.row0 + b.rows + b.halo_hi].reshape(-1, C).contiguous()
            out = ops.natten(buf, grid, heads, dhp, dhp, win, rows_global=h, row0=b.row0)
            want = f3[:, b.row0:b.row0 + b.rows].reshape(-1, f3.shape[-1])
            assert torch.equal(out, want), (world, b)
            rb = float((err[:, b.row0:b.row0 + b.rows].sum() / ref2[:, b.row0:b.row0 + b.rows].sum()).sqrt())
            assert rb < 2e-3, (world, b, rb)


@pytest.mark.parametrize("world,ext,dim,heads", [(2, (5, 18, 36), 256, 2), (4, (7, 30, 18), 256, 2),
                                                  (8, (5, 90, 180), 1024, 8)])
def test_band_block_matches_full(world, ext, dim, heads, monkeypatch):
    """Band kernels launched one by one with separate LayerNorm launches (the folded-LayerNorm band path is
    covered through BandedProcessor by the rollout / forecast tests below): bitwise the full-domain block."""
    from paper_2503_22235_b200 import _lib, ops
    from paper_2503_22235_b200.bands import gather_bands, local_band_tokens, plan_bands
    from paper_2503_22235_b200.blocks import RopeTables, Workspace, block_forward, prepare_block
    from paper_2503_22235_b200.params import init_block_params

    win = (5, 7, 7)
    d, h, w = ext
    params = init_block_params(np.random.default_rng(0), dim, heads, "blk", zero_residual=False)
    monkeypatch.setenv("WM3_LN_FOLD", "0")
    bw = prepare_block(params, "blk", heads)
    assert not bw.folded
    rope = RopeTables(ext, dim // heads)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(d * h * w, dim, device="cuda", generator=g)

    full = x.clone()
    block_forward(full, bw, Workspace(ops.KVGrid(ext, win), bw), rope, ext, win)

    bands = plan_bands(h, win[1], world)
    xs = [local_band_tokens(x, ext, b).clone() for b in bands]
    wss = [Workspace(ops.KVGrid((d, b.rows, w), win, b.halo_lo, b.halo_hi), bw) for b in bands]
    # phase 1: LN1 + QKV GEMM of every band into its own K/V grid
    for b, xb, ws in zip(bands, xs, wss):
        ops.layernorm_bf16(xb, bw.ln1_g, bw.ln1_b, out=ws.hn)
        ops.linear_grid(ws.hn, bw.w_qkv, _lib.WM3_EPI_QKV_ROPE, bw.b_qkv, ws.qkv, ws.grid,
                        rope=rope.struct((d, b.rows, w), b.row0, bw.heads, bw.dhp))
    # phase 2: halo exchange by copies between neighbouring bands
    for r, (b, ws) in enumerate(zip(bands, wss)):
        gme = ws.qkv.view(d, ws.grid.rows_ext, w, -1)
        if b.halo_lo:
            up, gup = bands[r - 1], wss[r - 1].qkv.view(d, wss[r - 1].grid.rows_ext, w, -1)
            s0 = up.halo_lo + up.rows - b.halo_lo
            gme[:, :b.halo_lo] = gup[:, s0:s0 + b.halo_lo]
        if b.halo_hi:
            dn, gdn = bands[r + 1], wss[r + 1].qkv.view(d, wss[r + 1].grid.rows_ext, w, -1)
            gme[:, b.halo_lo + b.rows:] = gdn[:, dn.halo_lo:dn.halo_lo + b.halo_hi]
    # phase 3: the rest of the block, per band
    for b, xb, ws in zip(bands, xs, wss):
        ops.natten(ws.qkv, ws.grid, bw.heads, bw.dhp, bw.dh, win, out=ws.ctx, rows_global=h, row0=b.row0)
        ops.linear(ws.ctx, bw.w_o, _lib.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=xb, n_valid=bw.hidden)
        ops.layernorm_bf16(xb, bw.ln2_g, bw.ln2_b, out=ws.hn)
        ops.linear(ws.hn, bw.w_1, _lib.WM3_EPI_BIAS_GELU_BF16, bias=bw.b_1, out=ws.mid)
        ops.linear(ws.mid, bw.w_2, _lib.WM3_EPI_BIAS_RESID_F32, bias=bw.b_2, out=xb, n_valid=bw.hidden)
    banded = gather_bands(xs, ext, bands)
    torch.cuda.synchronize()
    assert torch.equal(banded, full)


def test_band_block_forward_with_callback_single_band():
    """block_forward's halo hook path with a no-op exchanger on a band that needs no halos (world = 1)."""
    from paper_2503_22235_b200 import ops
    from paper_2503_22235_b200.blocks import RopeTables, Workspace, block_forward
    from paper_2503_22235_b200.params import init_block_params
    from paper_2503_22235_b200.runtime import CACHE
    ext, win, dim, heads = (5, 18, 36), (5, 7, 7), 256, 2
    params = init_block_params(np.random.default_rng(1), dim, heads, "blk", zero_residual=False)
    bw = CACHE.block(params, "blk", heads)
    rope = RopeTables(ext, dim // heads)
    x = torch.randn(int(np.prod(ext)), dim, device="cuda")
    a, b = x.clone(), x.clone()
    calls = []
    block_forward(a, bw, Workspace(ops.KVGrid(ext, win), bw), rope, ext, win)
    block_forward(b, bw, Workspace(ops.KVGrid(ext, win), bw), rope, ext, win, row0=0, rows_global=ext[1],
                  halo_exchange=lambda buf, grid: calls.append(grid.rows_ext))
    assert calls == [ext[1]]
    assert torch.equal(a, b)


@pytest.mark.parametrize("name,world", [("desk", 2), ("mid", 2), ("mid", 1)])
def test_banded_rollout_matches_single_gpu(name, world):
    """rollout_banded: the latent split into `world` latitude bands (emulated on this GPU: same kernels and
    halo rows as the NCCL path) reproduces the single-GPU mixed-horizon rollout bitwise."""
    import paper_2503_22235_b200.model as m
    import paper_2503_22235_b200.rollout as r
    from paper_2503_22235_b200.bands import rollout_banded
    cfg = {"desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=7, zero_residual=False)
    rng = np.random.default_rng(4)
    g = cfg.grid
    st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    lat = m.encode(st, params, cfg)
    one = r.rollout(lat, (6, 1), params, cfg)
    banded = rollout_banded(lat, (6, 1), params, cfg, world=world)
    assert banded.valid_time == 7 and tuple(banded.extents) == tuple(lat.extents)
    assert torch.equal(banded.tokens.device, one.tokens.device)
    assert rollout_banded(lat, (), params, cfg, world=world) is lat


@pytest.mark.parametrize("name,world", [("desk", 2), ("mid", 2)])
def test_fused_halo_epilogue_matches_exchange(name, world):
    """Halo rows written by the QKV GEMM epilogue straight into the neighbouring bands' K/V grids (the fused
    compute + exchange path; here the "peer" grids are the other bands' buffers on this GPU) give bitwise the
    same rollout as the separate halo copy."""
    import paper_2503_22235_b200.model as m
    from paper_2503_22235_b200.bands import rollout_banded
    cfg = {"desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=9, zero_residual=False)
    rng = np.random.default_rng(5)
    g = cfg.grid
    st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    lat = m.encode(st, params, cfg)
    copied = rollout_banded(lat, (6, 1), params, cfg, world=world)
    fused = rollout_banded(lat, (6, 1), params, cfg, world=world, fused=True)
    assert fused.tokens.values.tobytes() == copied.tokens.values.tobytes()


def test_halo_flag_kernels_self_signal():
    """wm3_halo_signal / wm3_halo_wait on this GPU's own flag words (a rank signalling itself: no cross-kernel
    waiting): release stores land, acquire waits pass once the epoch is reached."""
    from paper_2503_22235_b200 import _lib
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    s = _lib.stream_ptr()
    _lib.check(_lib.lib().wm3_halo_signal(flags.data_ptr() + 4, flags.data_ptr() + 8, 3, s), "signal")
    _lib.check(_lib.lib().wm3_halo_wait(flags.data_ptr() + 4, 2, 3, s), "wait")
    torch.cuda.synchronize()
    assert flags.tolist() == [0, 3, 3, 0]


def test_banded_forecast_full_scale_bands_8():
    """The bench's N = 8 forecast path (bands.forecast_banded: encoder / decoder pyramids split by depth plane,
    every latent block on latitude bands) at full scale, with the eight ranks emulated on this GPU: decoded
    fields bitwise equal to the single-GPU forecast (attention query tiles are aligned to global rows, every
    other kernel is per token or per depth plane)."""
    import paper_2503_22235_b200.model as m
    import paper_2503_22235_b200.rollout as r
    from paper_2503_22235_b200.bands import forecast_banded
    cfg = m.full_scale_config()
    params = m.init_model_params(cfg, seed=0, zero_residual=False)
    g = cfg.grid
    rng = np.random.default_rng(1)
    st = m.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).cuda(),
                        torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols))
                                         .astype(np.float32)).cuda())
    one = r.forecast(st, 7, params, cfg)
    banded = forecast_banded(st, 7, params, cfg, world=8)
    assert banded.valid_time == one.valid_time == 7
    assert torch.equal(one.surface.device, banded.surface.device)
    assert torch.equal(one.atmos.device, banded.atmos.device)


@pytest.mark.parametrize("name", ["desk", "mid"])
def test_pyramid_plane_ranges_bitwise(name):
    """encode_planes / decode_planes over plane ranges (the per-rank split of forecast_banded) write exactly
    the bytes the all-plane launches write: the pyramid never mixes depth planes."""
    import paper_2503_22235_b200.model as m
    from paper_2503_22235_b200.bands import plane_ranges
    from paper_2503_22235_b200.pyramid import decode_planes, encode_planes
    cfg = {"desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=3, zero_residual=False)
    rng = np.random.default_rng(8)
    g = cfg.grid
    st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    dm, prefix = m.stage_inputs(st, params, cfg)
    bufs, enc = dm.buffers(), dm.encoder(prefix)
    full = torch.empty((cfg.tokens, cfg.hidden), device="cuda")
    encode_planes(enc, bufs, cfg, full)
    d = cfg.depth_planes
    sfc_full = torch.empty((cfg.surface_out, g.rows, g.cols), device="cuda")
    atm_full = torch.empty((cfg.atmos_vars, cfg.levels, g.rows, g.cols), device="cuda")
    decode_planes(dm.decoder(), bufs, cfg, full, sfc_full, atm_full)
    for world in (2, 3, d):
        split = torch.full_like(full, float("nan"))
        sfc = torch.full_like(sfc_full, float("nan"))
        atm = torch.full_like(atm_full, float("nan"))
        for lo, hi in plane_ranges(d, world):
            encode_planes(enc, bufs, cfg, split, (lo, hi))
        for lo, hi in reversed(plane_ranges(d, world)):
            decode_planes(dm.decoder(), bufs, cfg, full, sfc, atm, (lo, hi))
        torch.cuda.synchronize()
        assert torch.equal(split, full), world
        assert torch.equal(sfc, sfc_full) and torch.equal(atm, atm_full), world
    with pytest.raises(m.ConfigError):
        encode_planes(enc, bufs, cfg, full, (2, 2))


@pytest.mark.parametrize("name,world", [("desk", 3), ("mid", 2)])
def test_forecast_banded_matches_forecast(name, world):
    """forecast_banded (plane-split pyramids + banded encoder / processor / decoder blocks, ranks emulated on
    this GPU) reproduces forecast() bitwise; validation matches forecast()."""
    import paper_2503_22235_b200.model as m
    import paper_2503_22235_b200.rollout as r
    from paper_2503_22235_b200.bands import forecast_banded
    cfg = {"desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=7, zero_residual=False)
    rng = np.random.default_rng(4)
    g = cfg.grid
    st = m.WeatherState(2, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    for dt in (0, 13):
        one = r.forecast(st, dt, params, cfg)
        banded = forecast_banded(st, dt, params, cfg, world=world)
        assert banded.valid_time == one.valid_time == 2 + dt
        assert torch.equal(one.surface.device, banded.surface.device), dt
        assert torch.equal(one.atmos.device, banded.atmos.device), dt
    with pytest.raises(m.ConfigError):
        forecast_banded(st, cfg.max_dt + 1, params, cfg, world=world)


def test_natten_row_split_bitwise():
    """wm3_natten_fwd_rows: the band's query rows computed in several launches (interior rows first, as while
    the halo exchange is in flight, then the boundary rows) write bitwise the bytes of one launch."""
    from paper_2503_22235_b200 import _lib, ops
    from paper_2503_22235_b200.bands import interior_rows, plan_bands
    ext, win, heads, dhp = (5, 90, 180), (5, 7, 7), 8, 128
    d, h, w = ext
    C = 3 * heads * dhp
    g = torch.Generator(device="cuda").manual_seed(5)
    qkv = (torch.randn(d * h * w, C, device="cuda", generator=g) * 1.5).to(_lib.ELEM)
    g3 = qkv.view(d, h, w, C)
    for b in plan_bands(h, win[1], 8)[:3] + [plan_bands(h, win[1], 1)[0]]:
        grid = ops.KVGrid((d, b.rows, w), win, b.halo_lo, b.halo_hi)
        buf = g3[:, b.row0 - b.halo_lo:b.row0 + b.rows + b.halo_hi].reshape(-1, C).contiguous()
        one = ops.natten(buf, grid, heads, dhp, dhp, win, rows_global=h, row0=b.row0)
        a, z = interior_rows(b, h, win[1])
        split = torch.full_like(one, float("nan"))
        for lo, hi in ((a, z), (b.row0, a), (z, b.row0 + b.rows)):
            if hi > lo:
                ops.natten(buf, grid, heads, dhp, dhp, win, out=split, rows_global=h, row0=b.row0, q_rows=(lo, hi))
        if not torch.equal(split, one):
            diff = split.float() - one.float()
            bad = torch.nonzero(torch.isnan(split).any(1) | torch.isnan(one).any(1) | (diff.abs() > 0).any(1)).flatten()
            rows = ((bad.cpu() // w) % b.rows + b.row0).unique().tolist()
            again = ops.natten(buf, grid, heads, dhp, dhp, win, rows_global=h, row0=b.row0)
            raise AssertionError(f"{b}: {bad.numel()} tokens differ (NaN in split {int(torch.isnan(split).any(1).sum())}, "
                                 f"in one {int(torch.isnan(one).any(1).sum())}), global rows {rows[:16]}, "
                                 f"split launches {(a, z)}, a repeat of the one-launch result equal: "
                                 f"{bool(torch.equal(again, one))}")


@pytest.mark.parametrize("name,world", [("mid", 2), ("desk", 2)])
def test_banded_rollout_graphs_bitwise(name, world):
    """rollout_banded with every horizon's step captured as a CUDA graph (processor-owned band buffers, the
    overlapped interior / boundary attention and the halo copies inside the graph) is bitwise the eager banded
    rollout and the single-GPU rollout; a second call replays the cached graphs."""
    import paper_2503_22235_b200.model as m
    import paper_2503_22235_b200.rollout as r
    from paper_2503_22235_b200.bands import rollout_banded
    cfg = {"desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=11, zero_residual=False)
    rng = np.random.default_rng(6)
    g = cfg.grid
    st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    lat = m.encode(st, params, cfg)
    plan = (6, 6, 1)
    one = r.rollout(lat, plan, params, cfg).tokens.device
    eager = rollout_banded(lat, plan, params, cfg, world=world, graphs=False).tokens.device
    graphed = rollout_banded(lat, plan, params, cfg, world=world, graphs=True).tokens.device
    again = rollout_banded(lat, plan, params, cfg, world=world, graphs=True).tokens.device
    assert torch.equal(eager, one) and torch.equal(graphed, one) and torch.equal(again, one)
