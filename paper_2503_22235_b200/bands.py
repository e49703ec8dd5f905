"""Latitude-band sharding of the latent processor across GPUs.

The (depth, rows, cols) latent is split into contiguous bands of rows, one per rank; every rank keeps the
full longitude circle (so column wrap stays local) and every depth plane.  Per-token work (LayerNorm, every
GEMM, GELU, residuals) needs nothing from other ranks; the neighborhood attention needs, per block, the K/V
rows of the neighbouring bands that its bumped windows reach: `halo` rows above and below (3 for the paper's
7-row window, fewer where the pole bump keeps windows inside the band).  Rotary phases and window bumps use
global row indices, so a band computes exactly the rows of the global block.

Halo exchange after the QKV GEMM: rank r sends its first `halo_hi[r-1]` band rows to r-1 and its last
`halo_lo[r+1]` rows to r+1, per depth plane, via torch.distributed point-to-point (NCCL over NVLink on B200,
gloo in the CPU tests).  Only the exchanged rows cross the link: 3 x 180 tokens x 6 KB x 5 planes ~= 16.6 MB
per neighbour per block at full scale.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

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


class HaloExchanger:
    """Fills the halo rows of a band's K/V grid buffer ([planes][halo_lo + rows + halo_hi][cols][C]) from the
    neighbouring ranks.  Works on CUDA (NCCL) and CPU (gloo) tensors alike."""

    def __init__(self, bands: list[Band], rank: int, group=None):
        self.bands, self.rank, self.group = bands, rank, group
        self.me = bands[rank]

    def __call__(self, buf: torch.Tensor, grid) -> None:
        import torch.distributed as dist
        me = self.me
        planes = getattr(grid, "planes", grid.depth)  # batch * depth for an ensemble batch
        g = buf.view(planes, grid.rows_ext, grid.cols, -1)
        ops = []
        lo0 = me.halo_lo  # buffer row of band row 0
        if me.rank > 0:
            up = self.bands[me.rank - 1]
            for d in range(planes):
                if up.halo_hi:  # my first rows -> upper neighbour's bottom halo
                    ops.append(dist.P2POp(dist.isend, g[d, lo0:lo0 + up.halo_hi].contiguous(), me.rank - 1,
                                          self.group))
                if me.halo_lo:
                    ops.append(dist.P2POp(dist.irecv, g[d, 0:me.halo_lo], me.rank - 1, self.group))
        if me.rank + 1 < len(self.bands):
            dn = self.bands[me.rank + 1]
            for d in range(planes):
                if dn.halo_lo:  # my last rows -> lower neighbour's top halo
                    ops.append(dist.P2POp(dist.isend, g[d, lo0 + me.rows - dn.halo_lo:lo0 + me.rows].contiguous(),
                                          me.rank + 1, self.group))
                if me.halo_hi:
                    ops.append(dist.P2POp(dist.irecv, g[d, lo0 + me.rows:lo0 + me.rows + me.halo_hi],
                                          me.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


def local_band_tokens(x_global: torch.Tensor, extents, band: Band) -> torch.Tensor:
    """(D*rows*cols, C) global tokens -> the band's (D*band.rows*cols, C) tokens (band order)."""
    d, h, w = extents
    return x_global.view(d, h, w, -1)[:, band.row0:band.row0 + band.rows].reshape(d * band.rows * w, -1)


def gather_bands(parts: list[torch.Tensor], extents, bands: list[Band]) -> torch.Tensor:
    d, h, w = extents
    return torch.cat([p.view(d, b.rows, w, -1) for p, b in zip(parts, bands)], dim=1).reshape(d * h * w, -1)
