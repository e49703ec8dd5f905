"""CPU: latitude-band sharding host logic with a real 2- and 4-rank gloo process group.

Each rank holds only its band's K/V rows, the HaloExchanger fills the halos from its neighbours, and the
band-local neighborhood attention (computed here with the float64 oracle on the band + halo rows) must equal
the global oracle attention rows of that band exactly.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.grid import neighborhood
from paper_2503_22235_b200.bands import HaloExchanger, band_rows, plan_bands
from paper_2503_22235_b200.ops import KVGrid


def test_band_rows_balanced():
    assert [n for _, n in band_rows(90, 8)] == [12, 11, 11, 11, 11, 11, 11, 12]
    assert [n for _, n in band_rows(90, 4)] == [23, 22, 22, 23]
    assert [n for _, n in band_rows(90, 2)] == [45, 45]
    assert sum(n for _, n in band_rows(17, 3)) == 17


def test_plan_bands_halos():
    bands = plan_bands(90, 7, 8)
    assert bands[0].halo_lo == 0 and bands[-1].halo_hi == 0
    assert all(b.halo_lo == 3 for b in bands[1:]) and all(b.halo_hi == 3 for b in bands[:-1])
    # a pole band's bumped windows stay inside a band of >= 7 rows
    assert plan_bands(90, 7, 1)[0].halo_lo == 0 and plan_bands(90, 7, 1)[0].halo_hi == 0
    with pytest.raises(ValueError):
        plan_bands(9, 7, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _band_attention(q, k, v, ext, win, band, heads):
    """Oracle NA for the band's queries using only band + halo K/V rows (local buffer indexing)."""
    d, h, w = ext
    full_tab = neighborhood(ext, win)  # global indices
    t = np.arange(d * h * w).reshape(d, h, w)[:, band.row0:band.row0 + band.rows].reshape(-1)
    gd, gr, gc = np.unravel_index(full_tab[t], (d, h, w))
    rows_ext = band.rows + band.halo_lo + band.halo_hi
    lr = gr - (band.row0 - band.halo_lo)
    assert lr.min() >= 0 and lr.max() < rows_ext, "halo too small for the window reach"
    local = (gd * rows_ext + lr) * w + gc
    dh = q.shape[-1] // heads
    qq = q.reshape(len(t), heads, dh)
    kk = k.reshape(-1, heads, dh)[local]
    vv = v.reshape(-1, heads, dh)[local]
    s = np.einsum("thd,tkhd->thk", qq, kk) / math.sqrt(dh)
    p = np.exp(s - s.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    return np.einsum("thk,tkhd->thd", p, vv).reshape(len(t), -1)


def _worker(rank, world, port, ext, win, heads, out_q):
    """Overlapped exchange as BandedProcessor runs it: start() -> attention of the band's interior rows (whose
    windows need no halo: the halo rows are still NaN here, so any use would poison the result) -> wait() ->
    attention of the boundary rows.  Only the K and V sections travel (the Q columns of halo rows stay NaN)."""
    from paper_2503_22235_b200.bands import interior_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, h, w = ext
        rng = np.random.default_rng(0)
        c = 8 * heads
        q = rng.standard_normal((d * h * w, c))
        k = rng.standard_normal((d * h * w, c))
        v = rng.standard_normal((d * h * w, c))
        bands = plan_bands(h, win[1], world)
        me = bands[rank]
        grid = KVGrid((d, me.rows, w), win, me.halo_lo, me.halo_hi)
        # this rank's q/k/v grid: only its own rows are filled, halos start as NaN
        qkv = np.concatenate([q, k, v], axis=1).reshape(d, h, w, -1)
        buf = torch.full((grid.tokens, 3 * c), float("nan"), dtype=torch.float64)
        g = buf.view(d, grid.rows_ext, w, -1)
        g[:, me.halo_lo:me.halo_lo + me.rows] = torch.from_numpy(qkv[:, me.row0:me.row0 + me.rows])
        exch = HaloExchanger(bands, rank, sec=c)
        handle = exch.start(buf, grid)
        a, z = interior_rows(me, h, win[1])

        def attend(rows_lo, rows_hi):
            kb = g.numpy().reshape(-1, 3 * c)
            out = _band_attention(np.zeros((d * me.rows * w, c)) + q.reshape(d, h, w, c)[
                :, me.row0:me.row0 + me.rows].reshape(-1, c), kb[:, c:2 * c], kb[:, 2 * c:], ext, win, me, heads)
            out = out.reshape(d, me.rows, w, c)
            return out[:, rows_lo - me.row0:rows_hi - me.row0]

        interior = attend(a, z)  # before wait(): halo rows are NaN
        exch.wait(handle)
        full = attend(me.row0, me.row0 + me.rows)
        got = full.copy()
        got[:, a - me.row0:z - me.row0] = interior
        lo, hi = me.row0 - me.halo_lo, me.row0 + me.rows + me.halo_hi
        gn = g.numpy()
        own = slice(me.halo_lo, me.halo_lo + me.rows)
        ok_halo = (np.array_equal(gn[..., c:], qkv[:, lo:hi, :, c:])              # K / V halo rows filled
                   and np.array_equal(gn[:, own], qkv[:, me.row0:me.row0 + me.rows])
                   and np.isnan(np.delete(gn[..., :c], np.arange(own.start, own.stop), axis=1)).all())  # Q not sent
        out_q.put((rank, ok_halo and np.isfinite(interior).all(), got.reshape(-1, c)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ext", [(2, (3, 16, 12)), (4, (2, 30, 10))])
def test_halo_exchange_gloo_band_attention(world, ext):
    win, heads = (3, 7, 5), 2
    win = (min(win[0], ext[0]), win[1], win[2])
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ext, win, heads, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict((r, (ok, got)) for r, ok, got in (q_out.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # global oracle attention
    d, h, w = ext
    rng = np.random.default_rng(0)
    c = 8 * heads
    q, k, v = (rng.standard_normal((d * h * w, c)) for _ in range(3))
    tab = neighborhood(ext, win)
    dh = c // heads
    s = np.einsum("thd,tkhd->thk", q.reshape(-1, heads, dh), k.reshape(-1, heads, dh)[tab]) / math.sqrt(dh)
    p = np.exp(s - s.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    full = np.einsum("thk,tkhd->thd", p, v.reshape(-1, heads, dh)[tab]).reshape(d, h, w, c)
    for rank, b in enumerate(plan_bands(h, win[1], world)):
        ok, got = results[rank]
        assert ok, f"rank {rank} halo rows differ from the neighbours' rows"
        np.testing.assert_allclose(got.reshape(d, b.rows, w, c), full[:, b.row0:b.row0 + b.rows], atol=1e-12)


class _FakeProcessor:
    """Stands in for BandedProcessor (whose kernels need a GPU): adds (global row + 1) * horizon to every token
    of each held band, so the test checks the sharding, the band bookkeeping and the all-gather."""

    def __init__(self, params, cfg, bands, held, exchanger=None, fused=False):
        self.held = [bands[i] for i in held]
        self.ext = cfg.latent_extents

    def graphs_supported(self):
        return False

    def process(self, xs, horizon):
        d, h, w = self.ext
        for b, x in zip(self.held, xs):
            rows = torch.arange(b.row0, b.row0 + b.rows, dtype=x.dtype).view(1, -1, 1, 1)
            x.view(d, b.rows, w, -1).add_((rows + 1.0) * horizon)


def _rollout_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_22235_b200.bands as B
        import paper_2503_22235_b200.model as M
        from paper_2503_22235_b200.tensor import Tensor
        cfg = M.mid_config()
        B.BandedProcessor = _FakeProcessor
        M.latent_tokens = lambda lat, cfg: lat.tokens.device  # CPU tensor stands in for the device latent
        M.device_model = lambda params, cfg: None
        params = {f"proc{h}.blk0.ln1.gain": None for h in cfg.horizons}
        x = torch.from_numpy(np.random.default_rng(3).standard_normal((cfg.tokens, 4)))
        lat = M.LatentState(Tensor(device=x.clone()), 5, cfg.latent_extents)
        out = B.rollout_banded(lat, (6, 1, 1), params, cfg)
        out_q.put((rank, out.valid_time, out.tokens.device.numpy()))
    finally:
        dist.destroy_process_group()


def test_rollout_banded_gloo_sharding_and_gather():
    import paper_2503_22235_b200.model as M
    cfg = M.mid_config()
    world = 2
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rollout_worker, args=(r, world, port, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_out.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d, h, w = cfg.latent_extents
    x = np.random.default_rng(3).standard_normal((cfg.tokens, 4))
    want = x.reshape(d, h, w, 4) + (np.arange(h) + 1.0).reshape(1, h, 1, 1) * 8
    for rank, vt, got in res:
        assert vt == 5 + 8
        np.testing.assert_allclose(got.reshape(d, h, w, 4), want, rtol=0, atol=1e-12)


def _planes_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_22235_b200.bands as B
        d, pt, hidden, p, a_vars, rows, cols = 5, 6, 3, 2, 3, 4, 5
        rng = np.random.default_rng(11)
        tok_full = torch.from_numpy(rng.standard_normal((d * pt, hidden)))
        sfc_full = torch.from_numpy(rng.standard_normal((2, rows, cols)))
        atm_full = torch.from_numpy(rng.standard_normal((a_vars, (d - 1) * p, rows, cols)))
        ranges = B.plane_ranges(d, world)
        lo, hi = ranges[rank]
        # each rank holds only its own planes; everything else is garbage before the gathers
        tokens = torch.full_like(tok_full, float("nan"))
        tokens[lo * pt:hi * pt] = tok_full[lo * pt:hi * pt]
        sfc = torch.full_like(sfc_full, float("nan"))
        atm = torch.full_like(atm_full, float("nan"))
        if lo == 0 and hi > 0:
            sfc.copy_(sfc_full)
        l0, l1 = B._plane_levels(lo, hi, p)
        atm[:, l0:l1] = atm_full[:, l0:l1]
        B.gather_plane_tokens(tokens, ranges, rank, pt)
        B.gather_plane_fields(sfc, atm, ranges, rank, p)
        ok = (torch.equal(tokens, tok_full) and torch.equal(sfc, sfc_full) and torch.equal(atm, atm_full))
        out_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 7])
def test_plane_gathers_gloo(world):
    """forecast_banded's encoder-token and decoded-field all-gathers by depth plane (surface + level groups),
    including ranks that hold no plane (world > depth)."""
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_planes_worker, args=(r, world, port, q_out)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q_out.get(timeout=120) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert all(ok for _, ok in res), res


def test_plane_ranges():
    from paper_2503_22235_b200.bands import plane_ranges
    assert plane_ranges(5, 1) == [(0, 5)]
    assert plane_ranges(5, 2) == [(0, 3), (3, 5)]
    assert plane_ranges(5, 8)[4:] == [(4, 5), (5, 5), (5, 5), (5, 5)]
    for world in range(1, 10):
        r = plane_ranges(5, world)
        assert r[0][0] == 0 and r[-1][1] == 5 and all(a[1] == b[0] for a, b in zip(r, r[1:]))


class _FakeBlocks(_FakeProcessor):
    def run(self, xs, prefixes):
        d, h, w = self.ext
        for b, x in zip(self.held, xs):
            rows = torch.arange(b.row0, b.row0 + b.rows, dtype=x.dtype).view(1, -1, 1, 1)
            x.view(d, b.rows, w, -1).add_((rows + 1.0) * 0.5 * len(prefixes))


def _fake_pyramid(cfg):
    """CPU stand-ins for the pyramid launches: encode writes fixed per-plane token values, decode writes
    per-plane sums of the (gathered) latent into the plane's surface / atmosphere levels."""
    d, h, w = cfg.latent_extents
    pt = h * w
    base = torch.from_numpy(np.random.default_rng(5).standard_normal((d, pt, cfg.hidden)))

    def encode_planes(enc, bufs, cfg_, tokens, planes):
        lo, hi = planes
        tokens.view(d, pt, -1)[lo:hi] = base[lo:hi].to(tokens.dtype)

    def decode_planes(dec, bufs, cfg_, full, surface, atmos, planes):
        lo, hi = planes
        x = full.view(d, pt, -1)
        p = cfg.level_patch
        if lo == 0:
            surface.copy_(x[0].sum() + torch.arange(surface.numel(), dtype=surface.dtype).view(surface.shape))
        for plane in range(max(lo, 1), hi):
            for lev in range((plane - 1) * p, plane * p):
                atmos[:, lev] = x[plane].sum() + lev + 100 * torch.arange(atmos.shape[0], dtype=atmos.dtype
                                                                          ).view(-1, 1, 1)
    return base, encode_planes, decode_planes


def _forecast_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_22235_b200.bands as B
        import paper_2503_22235_b200.model as M
        import paper_2503_22235_b200.pyramid as P
        cfg = M.mid_config()
        g = cfg.grid
        _, P.encode_planes, P.decode_planes = _fake_pyramid(cfg)
        B.BandedProcessor = _FakeBlocks
        M.device_model = lambda params, cfg: None

        class _DM:
            def buffers(self):
                class _B:
                    sfc_in = torch.zeros(1, dtype=torch.float32)
                    overflow = torch.zeros(1, dtype=torch.int32)  # fields_to_nhwc range flag, never set here
                return _B()

            def encoder(self, prefix):
                return None

            def decoder(self):
                return None

        M.stage_inputs = lambda state, params, cfg, source="primary": (_DM(), "enc")
        params = {f"proc{h}.blk0.ln1.gain": None for h in cfg.horizons}
        st = M.WeatherState(3, np.zeros((cfg.surface_in, g.rows, g.cols)),
                            np.zeros((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
        out = B.forecast_banded(st, 13, params, cfg)
        out_q.put((rank, out.valid_time, out.surface.device.numpy(), out.atmos.device.numpy()))
    finally:
        dist.destroy_process_group()


def test_forecast_banded_gloo_plumbing():
    """forecast_banded's distributed branch (the bench's N > 1 forecast) under a real gloo group, with CPU
    stand-ins for the kernels: plane-split encode -> token all-gather -> banded encoder / processor / decoder
    blocks -> band all-gather -> plane-split decode -> field all-gather; every rank returns the full fields."""
    import paper_2503_22235_b200.model as M
    cfg = M.mid_config()
    world = 2  # mid: 9 latent rows, 7 depth planes -> planes (0, 4), (4, 7)
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_forecast_worker, args=(r, world, port, q_out)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q_out.get(timeout=180) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    # expected: tokens = base + (row + 1) * (0.5 * enc_blocks + 13 + 0.5 * dec_blocks), decoded by the fake
    d, h, w = cfg.latent_extents
    base, _, dec = _fake_pyramid(cfg)
    x = base.view(d, h, w, -1).double() + (torch.arange(h, dtype=torch.float64).view(1, -1, 1, 1) + 1.0) * \
        (0.5 * cfg.enc_blocks + 13 + 0.5 * cfg.dec_blocks)
    g = cfg.grid
    sfc = torch.zeros((cfg.surface_out, g.rows, g.cols), dtype=torch.float32)
    atm = torch.zeros((cfg.atmos_vars, cfg.levels, g.rows, g.cols), dtype=torch.float32)
    dec(None, None, cfg, x.float().reshape(d * h * w, -1), sfc, atm, (0, d))
    for rank, vt, s, a in res:
        assert vt == 3 + 13
        np.testing.assert_allclose(s, sfc.numpy(), rtol=1e-5)
        np.testing.assert_allclose(a, atm.numpy(), rtol=1e-5)
