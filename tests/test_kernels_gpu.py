"""Kernel-level parity on the B200: each libwm3 kernel against the oracle / a torch fp32 reference."""

import math

import numpy as np
import pytest
import torch

from oracle.grid import neighborhood

pytestmark = pytest.mark.gpu


def ops():
    from paper_2503_22235_b200 import ops as o
    return o


def lib():
    from paper_2503_22235_b200 import _lib
    return _lib


# ------------------------------------------------------------------------------------------------
# bit-exact window arithmetic
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("ext,win", [
    ((3, 5, 8), (3, 3, 3)), ((4, 6, 10), (3, 3, 3)), ((1, 5, 6), (1, 3, 1)), ((1, 1, 8), (1, 1, 5)),
    ((7, 9, 18), (5, 7, 7)), ((5, 18, 36), (5, 7, 7)), ((3, 3, 3), (3, 3, 3)), ((2, 7, 10), (1, 4, 4)),
    ((3, 5, 10), (2, 2, 2)), ((6, 8, 10), (5, 5, 5)),
])
def test_neighbor_table_bit_exact(ext, win):
    got = ops().neighbor_table(ext, win).cpu().numpy()
    want = neighborhood(ext, win)
    assert got.dtype == np.int64 and got.shape == want.shape
    assert np.array_equal(got, want)


def test_neighbor_table_all_golden_cases():
    """Every neighbor-table case the reference generated (tests/golden/make_golden.py: the 40-case sweep of the
    reference's tests/test_grid.py:107-120 incl. even windows, plus the named shapes): sha256 of the int64 table
    and token 0's neighbors, from the GPU kernel."""
    import hashlib
    import json
    import os
    meta = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")))
    assert len(meta["neighborhood"]) == 50
    for case in meta["neighborhood"]:
        got = ops().neighbor_table(tuple(case["extents"]), tuple(case["window"])).cpu().numpy()
        assert list(got.shape) == case["shape"], case
        assert hashlib.sha256(got.astype("<i8").tobytes()).hexdigest() == case["sha256"], case
        assert got[0, :len(case["row0"])].tolist() == case["row0"], case


def test_neighbor_table_full_scale_checksum():
    import hashlib
    got = ops().neighbor_table((5, 90, 180), (5, 7, 7)).cpu().numpy()
    h = hashlib.sha256(got.astype("<i8").tobytes()).hexdigest()
    assert h.startswith("600ad28a33324093936c5ca3888cb6f1")
    assert got[0, :10].tolist() == [177, 178, 179, 0, 1, 2, 3, 357, 358, 359]


def test_neighbor_table_band_rows_match_full():
    full = neighborhood((5, 90, 180), (5, 7, 7)).reshape(5, 90, 180, -1)
    for row0, nrows in [(0, 12), (12, 11), (78, 12), (45, 45)]:
        got = ops().neighbor_table((5, 90, 180), (5, 7, 7), row0=row0, nrows=nrows).cpu().numpy()
        assert np.array_equal(got, full[:, row0:row0 + nrows].reshape(-1, full.shape[-1]))


# ------------------------------------------------------------------------------------------------
# GEMM (tcgen05) + epilogues
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (300, 256, 128), (1000, 384, 1024), (4096, 3072, 1024),
                                   (777, 1024, 4096), (81, 128, 192)])
def test_gemm_f32(m, n, k):
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda", generator=g).to(lib().ELEM)
    w = torch.randn(n, k, device="cuda", generator=g).to(lib().ELEM)
    out = ops().linear(a, w, lib().WM3_EPI_F32)
    ref = a.float() @ w.float().T
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    assert err <= 2e-3 * ref.abs().max().item() + 1e-3, err


def test_gemm_epilogues():
    m, n, k = 517, 512, 256
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(m, k, device="cuda", generator=g).to(lib().ELEM)
    w = (torch.randn(n, k, device="cuda", generator=g) / 16).to(lib().ELEM)
    b = torch.randn(n, device="cuda", generator=g)
    ref = a.float() @ w.float().T + b
    L = lib()
    # 16-bit outputs: one rounding of the fp32 result (2^-11 relative for fp16, 2^-8 for bf16) + accumulation
    ulp = 2.0 ** -10 if L.ELEM == torch.float16 else 2.0 ** -7
    o1 = ops().linear(a, w, L.WM3_EPI_BIAS_BF16, bias=b)
    assert ((o1.float() - ref).abs() <= ulp * ref.abs() + 2e-3).all()
    o2 = ops().linear(a, w, L.WM3_EPI_BIAS_GELU_BF16, bias=b)
    gel = 0.5 * ref * (1 + torch.erf(ref / math.sqrt(2)))
    # + the fitted erf form (|err| <= 2.5e-5) and tanh.approx (2^-11 relative)
    d = (o2.float() - gel).abs()
    print(f"GELU epilogue: max abs {d.max().item():.2e}")
    assert (d <= ulp * gel.abs() + 3e-3).all()
    x = torch.randn(m, n, device="cuda", generator=g)
    x0 = x.clone()
    ops().linear(a, w, L.WM3_EPI_BIAS_RESID_F32, bias=b, out=x)
    assert (x - (x0 + ref)).abs().max().item() < 1e-3
    # partial store (n_valid)
    out = torch.zeros(m, n, device="cuda")
    ops().linear(a, w, L.WM3_EPI_F32, out=out, n_valid=n - 44)
    assert out[:, n - 44:].abs().max().item() == 0
    assert (out[:, :n - 44] - (a.float() @ w.float().T)[:, :n - 44]).abs().max().item() < 1e-2


def test_layernorm():
    for m, n, ldo in [(1000, 1024, 1024), (33, 256, 256), (17, 12, 64), (64, 4096, 4096)]:
        x = torch.randn(m, n, device="cuda") * 3 + 1.5
        gain = torch.randn(n, device="cuda")
        bias = torch.randn(n, device="cuda")
        out = ops().layernorm_bf16(x, gain, bias, ldo=ldo)
        ref = torch.nn.functional.layer_norm(x, (n,), gain, bias, eps=1e-6)
        assert (out[:, :n].float() - ref).abs().max().item() < 0.05
        if ldo > n:
            assert out[:, n:].float().abs().max().item() == 0


# ------------------------------------------------------------------------------------------------
# fused neighborhood attention
# ------------------------------------------------------------------------------------------------
def na_reference(qkv, ext, heads, dhp, dh, win):
    d, h, w = ext
    t = d * h * w
    tab = torch.from_numpy(neighborhood(ext, win)).cuda()
    q = qkv[:, :heads * dhp].float().view(t, heads, dhp)
    k = qkv[:, heads * dhp:2 * heads * dhp].float().view(t, heads, dhp)
    v = qkv[:, 2 * heads * dhp:].float().view(t, heads, dhp)
    kn = k[tab]  # (T, K, heads, dhp)
    vn = v[tab]
    s = torch.einsum("thd,tkhd->thk", q, kn) / math.sqrt(dh)
    p = torch.softmax(s, dim=-1)
    return torch.einsum("thk,tkhd->thd", p, vn).reshape(t, heads * dhp), p


@pytest.mark.parametrize("ext,win,heads,dhp", [
    ((7, 9, 18), (5, 7, 7), 2, 128), ((5, 18, 36), (5, 7, 7), 8, 128), ((3, 5, 10), (3, 3, 3), 2, 64),
    ((2, 7, 10), (1, 3, 3), 4, 64), ((3, 3, 3), (3, 3, 3), 2, 64), ((5, 12, 200), (5, 7, 7), 1, 128),
    ((4, 6, 10), (2, 4, 4), 3, 128),
])
def test_natten_matches_gather_reference(ext, win, heads, dhp):
    t = int(np.prod(ext))
    g = torch.Generator(device="cuda").manual_seed(t)
    qkv = (torch.randn(t, 3 * heads * dhp, device="cuda", generator=g) * 1.5).to(lib().ELEM)
    grid = ops().KVGrid(ext, win)
    out = ops().natten(ops().pad_tokens_to_grid(qkv, grid), grid, heads, dhp, dhp, win)
    ref, _ = na_reference(qkv, ext, heads, dhp, dhp, win)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    print(f"NA vs fp32 gather {ext} {win}: rel L2 {rel:.2e} max abs {err:.2e}")
    # expected: fp16 P and output rounding, ~3e-4 relative; one wrong key per query (weight ~1/K) would be >1e-2
    assert rel < 2e-3 and err < 1e-2, (err, rel)


@pytest.mark.parametrize("ext,win,heads,dhp,batch", [
    ((7, 9, 18), (5, 7, 7), 2, 128, 3), ((3, 5, 10), (3, 3, 3), 2, 64, 2), ((4, 6, 10), (2, 4, 4), 3, 128, 4),
])
def test_natten_batched_members_equal_single(ext, win, heads, dhp, batch):
    """Ensemble batching: member b of one batched launch is bitwise the single-member result on its own data."""
    t = int(np.prod(ext))
    g = torch.Generator(device="cuda").manual_seed(7 * t + batch)
    qkv = (torch.randn(batch, t, 3 * heads * dhp, device="cuda", generator=g) * 1.5).to(lib().ELEM)
    gb = ops().KVGrid(ext, win, batch=batch)
    out = ops().natten(qkv.reshape(batch * t, -1).contiguous(), gb, heads, dhp, dhp, win)
    g1 = ops().KVGrid(ext, win)
    for b in range(batch):
        one = ops().natten(qkv[b].contiguous(), g1, heads, dhp, dhp, win)
        assert torch.equal(out[b * t:(b + 1) * t], one), b
    ref, _ = na_reference(qkv[batch - 1].contiguous(), ext, heads, dhp, dhp, win)
    rel = ((out[(batch - 1) * t:].float() - ref).norm() / ref.norm()).item()
    assert rel < 2e-3, rel


def test_natten_windows_bit_exact():
    from oracle.grid import bump_starts
    for ext, win in [((5, 90, 180), (5, 7, 7)), ((7, 9, 18), (5, 7, 7)), ((4, 6, 10), (2, 4, 4))]:
        d, h, w = ext
        got = ops().natten_windows(ext, win).cpu().numpy().reshape(d, h, w, 3)
        sd = bump_starts(d, win[0])
        sh = bump_starts(h, win[1])
        assert np.array_equal(got[..., 0], np.broadcast_to(sd[:, None, None], (d, h, w)))
        assert np.array_equal(got[..., 1], np.broadcast_to(sh[None, :, None], (d, h, w)))
        assert np.array_equal(got[..., 2], np.broadcast_to(((np.arange(w) - (win[2] - 1) // 2) % w)[None, None, :],
                                                          (d, h, w)))


def test_residual_gemm_bitwise_repeatable():
    """The residual epilogue streams fp32 residual chunks through smem slots by TMA (gemm.cu RESID_TMA); a slot
    hand-off race would show up as run-to-run differences.  40 repeats of the O-proj and W2 shapes (CTA pairs)
    and of a single-CTA residual GEMM must all be bitwise identical."""
    E = lib().ELEM
    g = torch.Generator(device="cuda").manual_seed(3)
    T, D = 40000, 1024
    x0 = torch.randn(T, D, device="cuda", generator=g)
    b = torch.randn(D, device="cuda", generator=g)
    for k, n in ((1024, 1024), (4096, 1024), (256, 128)):
        a = torch.randn(T, k, device="cuda", generator=g).to(E)
        w = (torch.randn(n, k, device="cuda", generator=g) / 32).to(E)
        xs = x0[:, :n].contiguous()
        ref = xs.clone()
        ops().linear(a, w, lib().WM3_EPI_BIAS_RESID_F32, bias=b[:n].contiguous(), out=ref)
        for _ in range(40):
            y = xs.clone()
            ops().linear(a, w, lib().WM3_EPI_BIAS_RESID_F32, bias=b[:n].contiguous(), out=y)
            assert torch.equal(y, ref), (k, n)
        want = xs + (a.float() @ w.float().T) + b[:n]
        assert ((ref - want).norm() / want.norm()).item() < 1e-3


@pytest.mark.parametrize("tile", ["5,5,5", "6,4,5", "1,2,40", "3,6,7", "1,1,58"])
def test_natten_both_mask_paths_match_reference(tile, monkeypatch):
    """The attention window mask runs inside the QK^T MMA (one-hot query classes x precomputed key bias) when a
    tile's depth + row + column classes fit in 16, else in the softmax; force tile shapes on both sides of that
    limit (WM3_NA_TILE) and check each against the fp32 gather reference on the same fp16 inputs."""
    monkeypatch.setenv("WM3_NA_TILE", tile)
    ext, win, heads, dhp = (5, 18, 72), (5, 7, 7), 2, 128
    t = int(np.prod(ext))
    g = torch.Generator(device="cuda").manual_seed(17)
    qkv = (torch.randn(t, 3 * heads * dhp, device="cuda", generator=g) * 1.5).to(lib().ELEM)
    grid = ops().KVGrid(ext, win)
    out = ops().natten(ops().pad_tokens_to_grid(qkv, grid), grid, heads, dhp, dhp, win)
    ref, _ = na_reference(qkv, ext, heads, dhp, dhp, win)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    print(f"NA tile {tile}: rel L2 {rel:.2e} max abs {err:.2e}")
    assert rel < 2e-3 and err < 1e-2, (tile, err, rel)


_TILE_PROBE = r"""
import hashlib, sys, torch
sys.path.insert(0, {root!r})
from paper_2503_22235_b200 import _lib, ops
g = torch.Generator(device="cuda").manual_seed(0)
h = hashlib.sha256()
for m, n, k in ((9900, 1024, 1024), (5000, 3072, 1024), (777, 1024, 4096)):
    a = torch.randn(m, k, device="cuda", generator=g).to(_lib.ELEM)
    w = (torch.randn(n, k, device="cuda", generator=g) / 32).to(_lib.ELEM)
    b = torch.randn(n, device="cuda", generator=g)
    x = torch.randn(m, n, device="cuda", generator=g)
    ops.linear(a, w, _lib.WM3_EPI_BIAS_RESID_F32, bias=b, out=x, n_valid=n)
    y = ops.linear(a, w, _lib.WM3_EPI_BIAS_GELU_BF16, bias=b)
    torch.cuda.synchronize()
    h.update(x.cpu().numpy().tobytes()); h.update(y.cpu().view(torch.int16).numpy().tobytes())
print(h.hexdigest())
"""


def test_gemm_results_independent_of_tile_width():
    """The CTA-pair GEMM picks 256 x 128 tiles where 256 x 256 ones would leave most of a wave idle (latitude
    bands at 8 GPUs); per-element MMA and epilogue arithmetic must not depend on that choice (band results are
    bitwise the single-GPU ones): every pair GEMM on 256-wide vs on 128-wide tiles, bitwise."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _TILE_PROBE.format(root=root)
    out = {}
    for v in ("0", "2"):
        env = dict(os.environ, WM3_GEMM_NARROW=v)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[v] = r.stdout.strip().splitlines()[-1]
    assert out["0"] == out["2"], out


def _pad_nhwc(x, cinp):
    """(imgs, c, h, w) fp32 -> padded NHWC (imgs, h + 2, w + 2, cinp) operand: zero rows, wrapped columns."""
    from paper_2503_22235_b200 import _lib
    imgs, c, h, w = x.shape
    p = torch.zeros((imgs, h + 2, w + 2, cinp), dtype=_lib.ELEM, device="cuda")
    xn = x.permute(0, 2, 3, 1).to(_lib.ELEM)
    p[:, 1:h + 1, 1:w + 1, :c] = xn
    p[:, 1:h + 1, 0, :c] = xn[:, :, w - 1]
    p[:, 1:h + 1, w + 1, :c] = xn[:, :, 0]
    return p


def _ref_conv(mode, xq, w, b):
    """fp32 reference of the three conv modes on the (fp16-rounded) input, reference geometry (model.py:296-325):
    rows zero-padded by 1, columns periodic."""
    import torch.nn.functional as F
    from paper_2503_22235_b200 import _lib
    xp = F.pad(F.pad(xq, (1, 1, 0, 0), mode="circular"), (0, 0, 1, 1))
    if mode == _lib.WM3_CONV_S1:
        return F.conv2d(xp, w) + b[None, :, None, None]
    if mode == _lib.WM3_CONV_S2:
        return F.conv2d(xp, w, stride=2) + b[None, :, None, None]
    imgs, cin, h, wd = xq.shape
    cout = w.shape[1]
    out = torch.zeros((imgs, cout, 2 * h, 2 * wd), device=xq.device)
    for a in range(2):
        for bb in range(2):
            acc = torch.zeros((imgs, cout, h, wd), device=xq.device)
            for tr in range(2):
                for tc in range(2):
                    tap = w[:, :, 3 - a - 2 * tr, 3 - bb - 2 * tc]  # (cin, cout)
                    win = xp[:, :, a + tr:a + tr + h, bb + tc:bb + tc + wd]
                    acc += torch.einsum("nchw,co->nohw", win, tap)
            out[:, :, a::2, bb::2] = acc
    return out + b[None, :, None, None]


@pytest.mark.parametrize("mode,h,w,cin,cout,gelu,resid", [
    ("s1", 7, 36, 96, 64, True, False),     # two-row tiles, odd rows: the bottom pad row must stay zero
    ("s1", 5, 250, 64, 192, False, True),   # one-row tiles, CTA pairs, A strips, TMA residual / output
    ("s1", 6, 180, 128, 256, False, True),  # two-row tiles with residual (the 90 x 180 stage shape class)
    ("s2", 6, 72, 64, 128, False, False),   # stride 2
    ("t2", 5, 36, 128, 64, False, False),   # transposed, two-row tiles, strided store box
    ("t2", 4, 250, 64, 192, False, False),  # transposed, one-row tiles, A strips over two column taps
])
def test_conv_kernel_against_torch(mode, h, w, cin, cout, gelu, resid):
    """wm3_conv (epilogue through TMA staging, one- and two-row tiles, strips) against an fp32 torch conv on
    the same fp16 operands, interior within fp16 output rounding; the padded output's halo: pad rows zero, pad
    columns the wrapped copies of the opposite edge."""
    from paper_2503_22235_b200 import _lib
    from paper_2503_22235_b200.pyramid import conv3_weights, convT_weights, cpad, run_conv
    torch.manual_seed(h * w + cin)
    imgs = 2
    x = torch.randn(imgs, cin, h, w, device="cuda")
    xq = x.to(_lib.ELEM).float()
    m = {"s1": _lib.WM3_CONV_S1, "s2": _lib.WM3_CONV_S2, "t2": _lib.WM3_CONV_T2}[mode]
    if m == _lib.WM3_CONV_T2:
        wt = torch.randn(cin, cout, 4, 4, device="cuda") / (2 * cin) ** 0.5
        cw = convT_weights(wt.cpu().numpy(), np.zeros(cout, np.float32))
        ho, wo = 2 * h, 2 * w
    else:
        wt = torch.randn(cout, cin, 3, 3, device="cuda") / (9 * cin) ** 0.5
        cw = conv3_weights(wt.cpu().numpy(), np.zeros(cout, np.float32), 1 if m == _lib.WM3_CONV_S1 else 2)
        ho, wo = (h, w) if m == _lib.WM3_CONV_S1 else ((h - 1) // 2 + 1, w // 2)
    bias = torch.randn(cout, device="cuda") * 0.1
    cw.b[:cout] = bias
    wt_q = wt.to(_lib.ELEM).float()  # the kernel's operand weights are the same rounding
    ref = _ref_conv(m, xq, wt_q, bias)
    rp = None
    if resid:
        r = torch.randn(imgs, cout, ho, wo, device="cuda")
        rp = _pad_nhwc(r, cpad(cout))
        ref = ref + r.to(_lib.ELEM).float()
    if gelu:
        ref = torch.nn.functional.gelu(ref)
    out = torch.zeros((imgs, ho + 2, wo + 2, cpad(cout)), dtype=_lib.ELEM, device="cuda")
    run_conv(cw, _pad_nhwc(x, cw.cinp), imgs, h, w, out, gelu=gelu, resid=rp)
    torch.cuda.synchronize()
    got = out[:, 1:ho + 1, 1:wo + 1, :cout].float().permute(0, 3, 1, 2)
    err = float((got - ref).norm() / ref.norm())
    print(f"conv {mode} {h}x{w} {cin}->{cout}: rel err {err:.2e}")
    assert err < 3e-3, err
    assert not out[:, 0].any() and not out[:, ho + 1].any()  # pad rows untouched
    assert torch.equal(out[:, 1:ho + 1, 0], out[:, 1:ho + 1, wo]) and torch.equal(out[:, 1:ho + 1, wo + 1],
                                                                                    out[:, 1:ho + 1, 1])
