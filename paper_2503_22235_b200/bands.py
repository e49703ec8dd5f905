"""Latitude-band sharding of the latent processor across GPUs.

The (depth, rows, cols) latent is split into contiguous bands of rows, one per rank; every rank keeps the
full longitude circle (so column wrap stays local) and every depth plane.  Per-token work (LayerNorm, every
GEMM, GELU, residuals) needs nothing from other ranks; the neighborhood attention needs, per block, the K/V
rows of the neighbouring bands that its bumped windows reach: `halo` rows above and below (3 for the paper's
7-row window, fewer where the pole bump keeps windows inside the band).  Rotary phases and window bumps use
global row indices, so a band computes exactly the rows of the global block.

Halo exchange after the QKV GEMM: rank r sends its first `halo_hi[r-1]` band rows to r-1 and its last
`halo_lo[r+1]` rows to r+1 (those rows of every depth plane packed into one message per neighbour) via
torch.distributed point-to-point (NCCL over NVLink on B200, gloo in the CPU tests).  Only the exchanged rows
cross the link: 3 x 180 tokens x 6 KB x 5 planes ~= 16.6 MB per neighbour per block at full scale.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .config import as_config
from .grid import bump_starts


@dataclass(frozen=True)
class Band:
    rank: int
    row0: int
    rows: int
    halo_lo: int
    halo_hi: int


def band_rows(rows_global: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous split; the remainder goes to the outermost bands (pole rows are cheapest to
    exchange), e.g. 90 rows / 8 ranks -> 12, 11, 11, 11, 11, 11, 11, 12."""
    if world < 1 or world > rows_global:
        raise ValueError(f"cannot split {rows_global} latent rows over {world} ranks")
    base, extra = divmod(rows_global, world)
    sizes = [base] * world
    order = []
    lo, hi = 0, world - 1
    while lo <= hi:
        order.append(lo)
        if hi != lo:
            order.append(hi)
        lo, hi = lo + 1, hi - 1
    for r in order[:extra]:
        sizes[r] += 1
    out, r0 = [], 0
    for s in sizes:
        out.append((r0, s))
        r0 += s
    return out


def plan_bands(rows_global: int, window_rows: int, world: int) -> list[Band]:
    """Bands with the halo each needs: rows reached by its bumped windows outside [row0, row0 + rows)."""
    starts = bump_starts(rows_global, window_rows)
    bands = []
    for rank, (r0, n) in enumerate(band_rows(rows_global, world)):
        lo = r0 - int(starts[r0])
        hi = int(starts[r0 + n - 1]) + window_rows - (r0 + n)
        bands.append(Band(rank, r0, n, max(lo, 0), max(hi, 0)))
    for b in bands:  # every halo must come from the single adjacent band
        if b.rank > 0 and b.halo_lo > bands[b.rank - 1].rows:
            raise ValueError("band thinner than the window reach; use fewer ranks")
        if b.rank + 1 < len(bands) and b.halo_hi > bands[b.rank + 1].rows:
            raise ValueError("band thinner than the window reach; use fewer ranks")
    return bands


def interior_rows(band: Band, rows_global: int, window_rows: int) -> tuple[int, int]:
    """Global query rows [a, b) of `band` whose bumped windows (grid.py:96-101) stay inside the band's own rows:
    their attention needs no halo row, so it can run while the halo exchange is in flight (empty: a == b)."""
    starts = bump_starts(rows_global, window_rows)
    rows = [r for r in range(band.row0, band.row0 + band.rows)
            if starts[r] >= band.row0 and starts[r] + window_rows <= band.row0 + band.rows]
    return (rows[0], rows[-1] + 1) if rows else (band.row0, band.row0)


class HaloExchanger:
    """Fills the halo rows of a band's K/V grid buffer ([planes][halo_lo + rows + halo_hi][cols][3 * sec]) from the
    neighbouring ranks.  Only the K and V sections (columns [sec, 3 * sec)) travel: a neighbour's attention reads
    keys and values of halo rows, never their queries.  Works on CUDA (NCCL) and CPU (gloo) tensors alike.

    start() posts the sends / receives and returns at once (NCCL: the transfers run on NCCL's stream, ordered after
    the work already queued on the current stream, i.e. the QKV GEMM); wait(handle) makes the current stream wait
    for them (NCCL: a stream dependency, no host block) and copies the received rows into the halo.  Work queued
    between the two — the attention of the band's interior rows — overlaps the exchange.  __call__ = both."""

    def __init__(self, bands: list[Band], rank: int, group=None, sec: int | None = None):
        self.bands, self.rank, self.group = bands, rank, group
        self.me = bands[rank]
        self.sec = sec  # first K column (heads * dhp); None: deduced as a third of the row width

    def start(self, buf: torch.Tensor, grid):
        import torch.distributed as dist
        me = self.me
        planes = getattr(grid, "planes", grid.depth)  # batch * depth for an ensemble batch
        g = buf.view(planes, grid.rows_ext, grid.cols, -1)
        c0 = self.sec if self.sec is not None else g.shape[-1] // 3
        g = g[..., c0:]  # K and V sections
        # One message per neighbour and direction: the halo rows of every depth plane are packed into one
        # contiguous buffer (a strided copy) instead of one send per plane, so a block costs at most two sends
        # and two receives.  gloo moves host memory only: CUDA rows are staged through the host (multi-process
        # smoke runs of the N > 1 bench path on one device); NCCL sends / receives device buffers.
        stage = buf.is_cuda and dist.get_backend(self.group) == "gloo"
        ops, post = [], []

        def send(rows, peer):
            ops.append(dist.P2POp(dist.isend, rows.cpu() if stage else rows.contiguous(), peer, self.group))

        def recv(rows, peer):
            tmp = torch.empty(rows.shape, dtype=rows.dtype, device="cpu" if stage else rows.device)
            post.append((rows, tmp))
            ops.append(dist.P2POp(dist.irecv, tmp, peer, self.group))

        lo0 = me.halo_lo  # buffer row of band row 0
        if me.rank > 0:
            up = self.bands[me.rank - 1]
            if up.halo_hi:  # my first rows -> upper neighbour's bottom halo
                send(g[:, lo0:lo0 + up.halo_hi], me.rank - 1)
            if me.halo_lo:
                recv(g[:, 0:me.halo_lo], me.rank - 1)
        if me.rank + 1 < len(self.bands):
            dn = self.bands[me.rank + 1]
            if dn.halo_lo:  # my last rows -> lower neighbour's top halo
                send(g[:, lo0 + me.rows - dn.halo_lo:lo0 + me.rows], me.rank + 1)
            if me.halo_hi:
                recv(g[:, lo0 + me.rows:lo0 + me.rows + me.halo_hi], me.rank + 1)
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, post, stage

    def wait(self, handle) -> None:
        reqs, post, stage = handle
        for req in reqs:
            req.wait()
        for rows, tmp in post:
            rows.copy_(tmp, non_blocking=not stage)

    def __call__(self, buf: torch.Tensor, grid) -> None:
        self.wait(self.start(buf, grid))


class CopyExchanger:
    """HaloExchanger's interface over the bands one process holds (the N-rank emulation on one GPU): start()
    copies the neighbouring bands' boundary rows (copy_halos, device copies on the current stream)."""

    def __init__(self, bands: list[Band], workspaces: list):
        self.bands, self.workspaces = bands, workspaces

    def start(self, buf=None, grid=None):
        copy_halos(self.bands, self.workspaces)
        return None

    def wait(self, handle) -> None:
        return None


def local_band_tokens(x_global: torch.Tensor, extents, band: Band) -> torch.Tensor:
    """(D*rows*cols, C) global tokens -> the band's (D*band.rows*cols, C) tokens (band order)."""
    d, h, w = extents
    return x_global.view(d, h, w, -1)[:, band.row0:band.row0 + band.rows].reshape(d * band.rows * w, -1)


def gather_bands(parts: list[torch.Tensor], extents, bands: list[Band]) -> torch.Tensor:
    d, h, w = extents
    return torch.cat([p.view(d, b.rows, w, -1) for p, b in zip(parts, bands)], dim=1).reshape(d * h * w, -1)


# ------------------------------------------------------------------------------------------------
# banded latent processor / rollout
# ------------------------------------------------------------------------------------------------
def copy_halos(bands: list[Band], workspaces: list) -> None:
    """In-process halo fill between the K/V grids of several bands held by one process (device copies);
    the same rows HaloExchanger moves between ranks."""
    for r, (b, ws) in enumerate(zip(bands, workspaces)):
        g = ws.grid
        me = ws.qkv.view(g.planes, g.rows_ext, g.cols, -1)
        if b.halo_lo:
            up, gu = bands[r - 1], workspaces[r - 1].grid
            src = workspaces[r - 1].qkv.view(gu.planes, gu.rows_ext, gu.cols, -1)
            s0 = up.halo_lo + up.rows - b.halo_lo
            me[:, :b.halo_lo] = src[:, s0:s0 + b.halo_lo]
        if b.halo_hi:
            dn, gd = bands[r + 1], workspaces[r + 1].grid
            src = workspaces[r + 1].qkv.view(gd.planes, gd.rows_ext, gd.cols, -1)
            me[:, b.halo_lo + b.rows:] = src[:, dn.halo_lo:dn.halo_lo + b.halo_hi]


@dataclass(frozen=True)
class GridGeo:
    """What a neighbour needs to know about a band's K/V grid to store halo rows into it."""
    rows_ext: int
    qkv_ld: int


def halo_descriptor(me: int, bands: list[Band], grids: list, qkv_ptrs: list, cols: int, sec: int):
    """wm3_halo_t for band `me`: its first halo_hi[up] rows go to the bottom halo of the band above, its last
    halo_lo[down] rows to the top halo of the band below (same rows HaloExchanger / copy_halos move).
    grids[i] / qkv_ptrs[i]: K/V grid geometry and device (or peer-mapped) address of band i; sec = first
    column of the K section (q is not needed by neighbours)."""
    from . import _lib
    h = _lib.HaloT()
    h.ld = grids[me].qkv_ld
    h.col_lo = sec
    if me > 0 and bands[me - 1].halo_hi:
        up, gu = bands[me - 1], grids[me - 1]
        h.up = qkv_ptrs[me - 1]
        h.n_up = up.halo_hi * cols
        h.up_plane_stride = gu.rows_ext * cols
        h.up_row_off = (up.halo_lo + up.rows) * cols
    if me + 1 < len(bands) and bands[me + 1].halo_lo:
        dn, gd = bands[me + 1], grids[me + 1]
        h.dn = qkv_ptrs[me + 1]
        h.n_dn = dn.halo_lo * cols
        h.dn_plane_stride = gd.rows_ext * cols
        h.dn_row_off = 0
    return h


class PeerHalo:
    """Fused halo exchange across ranks: every rank's K/V grid and a 4-word epoch-flag block are shared with its
    neighbours through CUDA IPC (torch's CUDA tensor reductions, handles exchanged over the process group), the
    QKV epilogue writes boundary rows straight into the neighbours' grids over NVLink, and per block:
        wait  consumed(e-1) from both neighbours   (their attention no longer reads the halo rows we overwrite)
        QKV GEMM with peer stores  -> signal ready(e) to both neighbours -> wait ready(e) from both
        attention -> signal consumed(e) to both neighbours
    Flags (int32, monotonic epochs) in each rank's block: [ready_from_up, ready_from_dn, consumed_from_up,
    consumed_from_dn]; a missing neighbour's flags start at INT32_MAX so its waits pass."""

    def __init__(self, bands: list[Band], rank: int, qkv: torch.Tensor, grid, group=None):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        self.bands, self.rank = bands, rank
        n = len(bands)
        big = 2 ** 31 - 1
        self.flags = torch.zeros(4, dtype=torch.int32, device=qkv.device)
        if rank == 0:
            self.flags[0] = big
            self.flags[2] = big
        if rank == n - 1:
            self.flags[1] = big
            self.flags[3] = big
        torch.cuda.synchronize()
        mine = (reduce_tensor(qkv), reduce_tensor(self.flags),
                {"rows_ext": grid.rows_ext, "qkv_ld": qkv.stride(0)})
        allv = [None] * n
        dist.all_gather_object(allv, mine, group=group)
        self.peer_qkv, self.peer_flags, self.geo = {}, {}, {}
        for r in (rank - 1, rank + 1):
            if 0 <= r < n:
                fq, aq = allv[r][0]
                ff, af = allv[r][1]
                self.peer_qkv[r] = fq(*aq)      # peer-mapped views (keep the objects alive)
                self.peer_flags[r] = ff(*af)
                self.geo[r] = allv[r][2]
        self.epoch = 0
        self.qkv_ld = qkv.stride(0)

    def descriptor(self, grid, cols: int, sec: int):
        """wm3_halo_t pointing at the neighbours' peer-mapped K/V grids."""
        grids = [None] * len(self.bands)
        ptrs = [None] * len(self.bands)
        for r, t in self.peer_qkv.items():
            grids[r] = GridGeo(self.geo[r]["rows_ext"], self.geo[r]["qkv_ld"])
            ptrs[r] = t.data_ptr()
        grids[self.rank] = GridGeo(grid.rows_ext, self.qkv_ld)
        return halo_descriptor(self.rank, self.bands, grids, ptrs, cols, sec)

    def _signal(self, idx_in_up: int, idx_in_dn: int, epoch: int) -> None:
        from . import _lib
        up = self.peer_flags.get(self.rank - 1)
        dn = self.peer_flags.get(self.rank + 1)
        a = None if up is None else up.data_ptr() + 4 * idx_in_up
        b = None if dn is None else dn.data_ptr() + 4 * idx_in_dn
        _lib.check(_lib.lib().wm3_halo_signal(a, b, int(epoch), _lib.stream_ptr()), "wm3_halo_signal")

    def _wait(self, first: int, epoch: int) -> None:
        from . import _lib
        _lib.check(_lib.lib().wm3_halo_wait(self.flags.data_ptr() + 4 * first, 2, int(epoch), _lib.stream_ptr()),
                   "wm3_halo_wait")

    def before_qkv(self) -> None:
        self.epoch += 1
        self._wait(2, self.epoch - 1)          # consumed flags of the previous block

    def after_qkv(self) -> None:
        # my rows are in the band above's "ready_from_dn" slot and the band below's "ready_from_up" slot
        self._signal(1, 0, self.epoch)
        self._wait(0, self.epoch)

    def after_attention(self) -> None:
        self._signal(3, 2, self.epoch)


class BandedProcessor:
    """Processor blocks over latitude bands: for each block, LN1 + QKV (into each band's halo'd K/V grid)
    for every held band, the halo exchange, then attention and the rest of the block per band.

    `held` are the bands this process computes: its own band under torch.distributed (exchange =
    HaloExchanger over NCCL / gloo), or every band when one process emulates the split on one GPU
    (exchange = copy_halos).  Kernels never wait on one another either way.

    With a separate exchange (not fused) the attention is split by query rows (wm3_block_na_rows): the rows
    whose windows stay inside the band run between starting the exchange and waiting for it, the boundary rows
    after; attention query tiles are aligned to global rows, so the split changes no bit of the result.

    graphs(): the blocks of each processor horizon captured once as a CUDA graph over processor-owned band
    buffers (`buffers()`), replayed per step — on by default for the one-GPU emulation; for the NCCL exchange
    opt-in (WM3_BAND_GRAPHS=1: NCCL point-to-point inside stream capture, not exercised on more than one GPU
    here); never for PeerHalo, whose epoch flags are host-side counters."""

    def __init__(self, params: dict, cfg, bands: list[Band], held: list[int], exchanger=None, fused: bool = False):
        """fused: halo rows travel in the QKV GEMM epilogue (peer stores) instead of a separate exchange —
        between the held bands' own grids when emulating, through PeerHalo (`exchanger`) across ranks."""
        from .runtime import CACHE
        self.params, self.cfg, self.bands = params, cfg, bands
        self.held = [bands[i] for i in held]
        self.held_idx = list(held)
        self.exchanger = exchanger
        self.fused = fused
        d, h, w = cfg.latent_extents
        self.rope = CACHE.rope(cfg.latent_extents, cfg.head_dim)
        self.local = [(d, b.rows, w) for b in self.held]
        self.interior = [interior_rows(b, h, cfg.window[1]) if self._split_na(b) else (b.row0, b.row0)
                         for b in self.held]
        self._bufs = None
        self._graphs: dict = {}
        self.timing = None  # optional callback(name) between phases (bench: CUDA events per phase)

    @staticmethod
    def _split_na(band: Band) -> bool:
        """Split this band's attention into interior rows (run while the halo exchange is in flight) and
        boundary rows (after it)?  WM3_NA_SPLIT=1 / 0 forces it; by default only bands of >= 40 rows split:
        each extra launch covers whole 5-row query tiles for a few rows, which on a narrow band costs more than
        the exchange it hides (tools/band_projection.py)."""
        import os
        env = os.environ.get("WM3_NA_SPLIT")
        if env in ("0", "1"):
            return env == "1"
        return band.rows >= 40

    def _ws(self, bw):
        from .runtime import CACHE
        # one workspace per band (tagged by rank): bands of equal shape must not share K/V grids
        return [CACHE.workspace(ext, self.cfg.window, bw, halo=(b.halo_lo, b.halo_hi), tag=f"band{b.rank}")
                for ext, b in zip(self.local, self.held)]

    def process(self, xs: list[torch.Tensor], horizon: int) -> None:
        """In place on the held bands' token buffers xs[i] ((d * rows_i * w, hidden) fp32, band order)."""
        self.run(xs, [f"proc{horizon}.blk{i}" for i in range(self.cfg.proc_blocks)])

    # ---------------- CUDA graphs over processor-owned buffers ----------------
    def graphs_supported(self) -> bool:
        import os
        if isinstance(self.exchanger, PeerHalo):
            return False
        if isinstance(self.exchanger, HaloExchanger):
            return os.environ.get("WM3_BAND_GRAPHS", "0") == "1"
        return True

    def buffers(self) -> list[torch.Tensor]:
        """The held bands' token buffers the captured graphs run on (allocated once)."""
        if self._bufs is None:
            d, _, w = self.cfg.latent_extents
            self._bufs = [torch.zeros((d * b.rows * w, self.cfg.hidden), dtype=torch.float32, device="cuda")
                          for b in self.held]
        return self._bufs

    def graph(self, horizon: int):
        """The captured processor step of `horizon` over buffers() (warm-up and capture on the buffers'
        current content: call before loading the latent)."""
        g = self._graphs.get(horizon)
        if g is None:
            from .runtime import CACHE
            bufs = self.buffers()
            self.process(bufs, horizon)  # warm-up outside capture: weights, workspaces, kernel attributes
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.process(bufs, horizon)
            # the graph holds raw device pointers: keep the captured weights alive with it
            self._keep = getattr(self, "_keep", []) + [CACHE.block(self.params, f"proc{horizon}.blk{i}",
                                                                   self.cfg.heads)
                                                       for i in range(self.cfg.proc_blocks)]
            self._graphs[horizon] = g
        return g

    # ---------------- the blocks ----------------
    def run(self, xs: list[torch.Tensor], prefixes) -> None:
        """The blocks named by `prefixes` (encoder, processor or decoder blocks) in order, in place on xs."""
        import ctypes

        from . import _lib
        from .runtime import CACHE
        cfg = self.cfg
        h = cfg.latent_extents[1]
        cols = cfg.latent_extents[2]
        mark = self.timing if self.timing is not None else (lambda name: None)
        for bi, prefix in enumerate(prefixes):
            bw = CACHE.block(self.params, prefix, cfg.heads)
            wss = self._ws(bw)
            sec = bw.heads * bw.dhp
            peer = self.exchanger if (self.fused and isinstance(self.exchanger, PeerHalo)) else None
            if peer is not None:
                peer.before_qkv()
            # folded LayerNorm: after the first block the previous W2 epilogue left each band's hn / stats
            geoms = [_lib.BlockGeomT(1, ext[0], ext[1], ext[2], h, b.row0, b.halo_lo, b.halo_hi, *cfg.window,
                                     int(bi > 0))
                     for b, ext in zip(self.held, self.local)]
            local_grids = [GridGeo(w_.grid.rows_ext, w_.qkv.stride(0)) for w_ in wss]
            mark("qkv")
            for j, (b, ext, xb, ws) in enumerate(zip(self.held, self.local, xs, wss)):
                halo = None
                if self.fused:
                    if peer is not None:
                        halo = peer.descriptor(ws.grid, cols, sec)
                    else:  # emulation: the neighbours are the other held bands' grids on this GPU
                        halo = halo_descriptor(self.held_idx[j], self.held, local_grids,
                                               [w_.qkv.data_ptr() for w_ in wss], cols, sec)
                # LN1 + QKV (+rotary, + fused halo stores) in one library call
                rs = self.rope.struct(ext, b.row0, bw.heads, bw.dhp)
                _lib.check(_lib.lib().wm3_block_qkv(xb.data_ptr(), ctypes.byref(bw.native()), ctypes.byref(ws.native()),
                                                    ctypes.byref(geoms[j]), ctypes.byref(rs),
                                                    None if halo is None else ctypes.byref(halo), _lib.stream_ptr()),
                           "wm3_block_qkv")

            def na_rows(j, lo, hi):
                if hi > lo:
                    _lib.check(_lib.lib().wm3_block_na_rows(ctypes.byref(bw.native()), ctypes.byref(wss[j].native()),
                                                            ctypes.byref(geoms[j]), int(lo), int(hi - lo),
                                                            _lib.stream_ptr()), "wm3_block_na_rows")

            if self.fused:
                if peer is not None:
                    peer.after_qkv()
                # emulation: stream order already puts every band's halo stores before any attention
                mark("na")
                for j, b in enumerate(self.held):
                    na_rows(j, b.row0, b.row0 + b.rows)
            else:
                exch = self.exchanger if self.exchanger is not None else CopyExchanger(self.held, wss)
                mark("exchange_start")
                handles = [exch.start(ws.qkv, ws.grid) for ws in wss] if self.exchanger is not None \
                    else [exch.start()]
                mark("na_interior")  # attention of rows that need no halo, overlapping the exchange
                for j, (a, z) in enumerate(self.interior):
                    na_rows(j, a, z)
                mark("exchange_wait")
                for hd in handles:
                    exch.wait(hd)
                mark("na_boundary")
                for j, (b, (a, z)) in enumerate(zip(self.held, self.interior)):
                    if z > a:
                        na_rows(j, b.row0, a)
                        na_rows(j, z, b.row0 + b.rows)
                    else:
                        na_rows(j, b.row0, b.row0 + b.rows)
            mark("out")
            for j, (xb, ws) in enumerate(zip(xs, wss)):
                # O-proj -> LN2 -> MLP in one library call
                _lib.check(_lib.lib().wm3_block_out(xb.data_ptr(), ctypes.byref(bw.native()), ctypes.byref(ws.native()),
                                                    ctypes.byref(geoms[j]), _lib.stream_ptr()), "wm3_block_out")
                if peer is not None:
                    peer.after_attention()  # neighbours may overwrite our halo rows for the next block
            mark("end")


def plane_ranges(depth: int, world: int) -> list[tuple[int, int]]:
    """Depth planes [lo, hi) per rank for the encoder / decoder pyramids: contiguous, sizes differing by at
    most one; with more ranks than planes the extra ranks get an empty range (they only run latent bands)."""
    if depth < 1 or world < 1:
        raise ValueError(f"cannot split {depth} planes over {world} ranks")
    base, extra = divmod(depth, world)
    out, lo = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((lo, lo + n))
        lo += n
    return out


_PROCS: dict = {}


def _banded_setup(params: dict, cfg, world, group, fused: bool, first_prefix: str):
    """(processor, bands, rank, world, distributed) for a banded run; see rollout_banded.  Processors (with
    their exchangers, peer mappings and captured graphs) are cached per (params, cfg, split) and rebuilt when
    the parameters' content tags change (as the single-GPU rollout graphs)."""
    import torch.distributed as dist

    from .model import device_model
    fp = getattr(device_model(params, cfg), "_fp", None)
    d, h, w = cfg.latent_extents
    distributed = world is None and dist.is_available() and dist.is_initialized() and \
        dist.get_world_size(group) > 1
    n = dist.get_world_size(group) if distributed else int(world or 1)
    rank = dist.get_rank(group) if distributed else 0
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    key = (id(params), cfg, n, bool(fused), distributed, rank, id(group), dev)
    hit = _PROCS.get(key)
    if hit is not None and hit[0] is params and hit[1] == fp:
        return hit[2], hit[3], rank, n, distributed
    bands = plan_bands(h, cfg.window[1], n)
    if not distributed:
        proc = BandedProcessor(params, cfg, bands, list(range(n)), fused=fused)
    else:
        if fused:
            from .runtime import CACHE
            me = bands[rank]
            bw0 = CACHE.block(params, first_prefix, cfg.heads)
            ws0 = CACHE.workspace((d, me.rows, w), cfg.window, bw0, halo=(me.halo_lo, me.halo_hi), tag=f"band{rank}")
            exch = PeerHalo(bands, rank, ws0.qkv, ws0.grid, group)
        else:
            exch = HaloExchanger(bands, rank, group)
        proc = BandedProcessor(params, cfg, bands, [rank], exch, fused=fused)
    _PROCS[key] = (params, fp, proc, bands)
    return proc, bands, rank, n, distributed


def _gather_latent(xs: list[torch.Tensor], bands: list[Band], extents, distributed: bool, group) -> torch.Tensor:
    """The full latent from the bands (all-gather across ranks, padded to the largest band)."""
    import torch.distributed as dist
    d, _, w = extents
    if distributed:
        hidden = xs[0].shape[1]
        mx = max(b.rows for b in bands) * d * w
        buf = torch.zeros((mx, hidden), dtype=xs[0].dtype, device=xs[0].device)
        buf[:xs[0].shape[0]] = xs[0]
        parts = [torch.empty_like(buf) for _ in bands]
        dist.all_gather(parts, buf, group=group)
        xs = [p[:d * b.rows * w] for p, b in zip(parts, bands)]
    return gather_bands(xs, extents, bands)


def rollout_banded(lat, plan, params: dict, cfg, world: int | None = None, group=None, fused: bool = False,
                   graphs: bool | None = None):
    """rollout() with the latent split into latitude bands.

    Under an initialised torch.distributed group of size N > 1 (and world None): rank r keeps band r, halos
    move over the group (NCCL over NVLink on B200), and the bands are all-gathered at the end so every rank
    returns the full latent.  With `world` given and no group, one process emulates `world` bands on its GPU
    (the same kernels and halo rows; used to verify the split on one device).  fused=True moves the halo rows
    in the QKV GEMM epilogue (peer stores into the neighbours' K/V grids, PeerHalo epoch flags across ranks)
    instead of a separate exchange.  graphs (default: plans of more than one step, where the split supports it,
    BandedProcessor.graphs_supported): each horizon's step replayed as a CUDA graph, bitwise the eager result.
    Validation as rollout()."""
    cfg = as_config(cfg)
    from .model import CALL_COUNTS, LatentState, latent_tokens
    from .rollout import _check_plan, plan_hours
    from .tensor import Tensor

    plan = _check_plan(plan, params, cfg)
    if not plan:
        return lat
    x = latent_tokens(lat, cfg)
    proc, bands, rank, n, distributed = _banded_setup(params, cfg, world, group, fused, f"proc{plan[0]}.blk0")
    held = [bands[rank]] if distributed else bands
    use_graphs = (len(plan) > 1 if graphs is None else bool(graphs)) and proc.graphs_supported()
    if use_graphs:
        steps = {hz: proc.graph(hz) for hz in sorted(set(plan))}  # warm-up / capture before the latent loads
        xs = proc.buffers()
        for xb, b in zip(xs, held):
            xb.copy_(local_band_tokens(x, cfg.latent_extents, b))
        for hz in plan:
            steps[hz].replay()
            CALL_COUNTS[f"process{hz}"] += 1
    else:
        xs = [local_band_tokens(x, cfg.latent_extents, b).clone() for b in held]
        for hz in plan:
            proc.process(xs, hz)
            CALL_COUNTS[f"process{hz}"] += 1
    full = _gather_latent(xs, bands, cfg.latent_extents, distributed, group)
    return LatentState(Tensor(device=full), lat.valid_time + plan_hours(plan), tuple(lat.extents))


def _all_gather_var(local: torch.Tensor, sizes: list[int], group) -> list[torch.Tensor]:
    """all_gather of 1-D/2-D row blocks of per-rank `sizes` rows (padded to the largest)."""
    import torch.distributed as dist
    mx = max(max(sizes), 1)
    buf = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[:local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in sizes]
    dist.all_gather(parts, buf, group=group)
    return [p[:k] for p, k in zip(parts, sizes)]


def gather_plane_tokens(tokens: torch.Tensor, ranges: list[tuple[int, int]], rank: int, plane_tokens: int,
                        group=None) -> None:
    """In place: every rank's encoded planes (rows [lo * plane_tokens, hi * plane_tokens) of `tokens`, ranges[r]
    for rank r) copied into every other rank's `tokens` (one all-gather)."""
    lo, hi = ranges[rank]
    pt = plane_tokens
    parts = _all_gather_var(tokens[lo * pt:hi * pt], [(b - a) * pt for a, b in ranges], group)
    for r, ((a, b), part) in enumerate(zip(ranges, parts)):
        if b > a and r != rank:
            tokens[a * pt:b * pt] = part


def _plane_levels(a: int, b: int, level_patch: int) -> tuple[int, int]:
    """Atmosphere levels [l0, l1) decoded from depth planes [a, b) (plane 0 = surface, p = level group p-1)."""
    return (max(a, 1) - 1) * level_patch, max(b - 1, 0) * level_patch


def gather_plane_fields(surface: torch.Tensor, atmos: torch.Tensor, ranges: list[tuple[int, int]], rank: int,
                        level_patch: int, group=None) -> None:
    """In place: the decoded fields of every rank's planes (surface from the rank holding plane 0, atmosphere
    levels of its level groups, all variables) copied into every rank's (surface, atmos) (one all-gather of
    packed [surface | atmos[:, l0:l1]] chunks)."""
    a_vars, _, rows, cols = atmos.shape

    def count(a, b):
        l0, l1 = _plane_levels(a, b, level_patch)
        return (surface.numel() if a == 0 and b > 0 else 0) + a_vars * max(l1 - l0, 0) * rows * cols

    lo, hi = ranges[rank]
    l0, l1 = _plane_levels(lo, hi, level_patch)
    chunks = ([surface.reshape(-1)] if lo == 0 and hi > 0 else []) + \
        ([atmos[:, l0:l1].reshape(-1)] if l1 > l0 else [])
    local = torch.cat(chunks) if chunks else surface.new_empty(0)
    parts = _all_gather_var(local, [count(a, b) for a, b in ranges], group)
    for r, ((a, b), part) in enumerate(zip(ranges, parts)):
        if b <= a or r == rank:
            continue
        off = 0
        if a == 0:
            surface.view(-1).copy_(part[:surface.numel()])
            off = surface.numel()
        m0, m1 = _plane_levels(a, b, level_patch)
        if m1 > m0:
            atmos[:, m0:m1] = part[off:].view(a_vars, m1 - m0, rows, cols)


def forecast_banded(state, dt: int, params: dict, cfg, world: int | None = None, group=None, fused: bool = False,
                    source: str = "primary"):
    """forecast() (rollout.py:84-91) with every stage split across ranks.

    The encoder and decoder pyramids treat the depth planes independently, so each rank convolves only its
    planes (`plane_ranges`: surface and level groups) and the latent tokens / decoded fields are all-gathered
    by plane; the encoder, processor and decoder blocks run on latitude bands with the per-block halo exchange
    (`BandedProcessor`, as rollout_banded).  Every rank returns the full DecodedFields.  `world` without a
    group emulates the split in one process (plane ranges and bands one after another on one GPU).
    Validation as forecast(), before any launch."""
    cfg = as_config(cfg)
    from .model import CALL_COUNTS, DecodedFields, stage_inputs
    from .pyramid import check_input_range, decode_planes, encode_planes
    from .rollout import _check_plan, greedy_plan, plan_hours
    from .tensor import Tensor

    plan = _check_plan(greedy_plan(dt, cfg.max_dt), params, cfg)
    dm, prefix = stage_inputs(state, params, cfg, source)
    enc_p = [f"{prefix}.blk{i}" for i in range(cfg.enc_blocks)]
    dec_p = [f"dec.blk{i}" for i in range(cfg.dec_blocks)]
    first = (enc_p + [f"proc{hz}.blk0" for hz in plan] + dec_p + [None])[0]
    fused = fused and first is not None
    proc, bands, rank, n, distributed = _banded_setup(params, cfg, world, group, fused, first)
    d, h, w = cfg.latent_extents
    g = cfg.grid
    pt = h * w  # tokens per depth plane
    ranges = plane_ranges(d, n)
    mine = [ranges[rank]] if distributed else ranges
    bufs = dm.buffers()
    dev = bufs.sfc_in.device

    # encoder pyramid by planes -> all-gather the token planes
    tokens = torch.empty((cfg.tokens, cfg.hidden), dtype=torch.float32, device=dev)
    enc = dm.encoder(prefix)
    for lo, hi in mine:
        if hi > lo:
            encode_planes(enc, bufs, cfg, tokens, (lo, hi))
            check_input_range(bufs)
    if distributed:
        gather_plane_tokens(tokens, ranges, rank, pt, group)

    # latent blocks by latitude bands
    held = [bands[rank]] if distributed else bands
    steps = {}
    if len(plan) > 1 and proc.graphs_supported():
        steps = {hz: proc.graph(hz) for hz in sorted(set(plan))}  # capture before the latent loads
        xs = proc.buffers()
        for xb, b in zip(xs, held):
            xb.copy_(local_band_tokens(tokens, cfg.latent_extents, b))
    else:
        xs = [local_band_tokens(tokens, cfg.latent_extents, b).clone() for b in held]
    del tokens
    proc.run(xs, enc_p)
    for hz in plan:
        if steps:
            steps[hz].replay()
        else:
            proc.process(xs, hz)
        CALL_COUNTS[f"process{hz}"] += 1
    proc.run(xs, dec_p)
    CALL_COUNTS["decode"] += 1
    full = _gather_latent(xs, bands, cfg.latent_extents, distributed, group)
    del xs

    # decoder pyramid by planes -> all-gather the fields
    surface = torch.empty((cfg.surface_out, g.rows, g.cols), dtype=torch.float32, device=dev)
    atmos = torch.empty((cfg.atmos_vars, cfg.levels, g.rows, g.cols), dtype=torch.float32, device=dev)
    dec = dm.decoder()
    for lo, hi in mine:
        if hi > lo:
            decode_planes(dec, bufs, cfg, full, surface, atmos, (lo, hi))
    if distributed:
        gather_plane_fields(surface, atmos, ranges, rank, cfg.level_patch, group)
    return DecodedFields(state.valid_time + plan_hours(plan), Tensor(device=surface), Tensor(device=atmos))
