"""§8f4 on the B200: the processor block's reverse mode (backward.block_vjp) and the reference's own training
machinery running on it through the operator seam (integration.install(operator=True)).

Oracle: the reference's float64 tape (gridcast.autodiff backward over attention.natten_block, staged into
baseline/_ref by baseline/stage_ref.sh).  Tolerances: relative L2 <= 1e-2 per gradient (fp16 tensor-core operands,
fp32 accumulation; measured values printed); determinism and the checkpoint / offload parity of verify.py:73-113
bitwise.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
GRAD_TOL = 1e-2


@pytest.fixture(scope="module")
def gc():
    if not os.path.isdir(os.path.join(REF, "gridcast")):
        pytest.skip("reference not staged: run baseline/stage_ref.sh")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gridcast
    import gridcast.attention
    import gridcast.autodiff
    import gridcast.model
    import gridcast.training
    import gridcast.verify
    return gridcast


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("ext,win,dim,heads", [
    ((3, 5, 10), (3, 3, 3), 48, 4),     # desk latent
    ((2, 7, 10), (1, 3, 3), 24, 4),     # dh = 6 (heads padded to 64)
    ((7, 9, 18), (5, 7, 7), 256, 2),    # paper window: depth bump, row bump, column wrap
    ((4, 6, 10), (2, 4, 4), 128, 2),    # even windows
])
def test_block_vjp_matches_reference_tape(gc, ext, win, dim, heads):
    """Input and all 16 parameter gradients of one block vs the reference tape's float64 gradients of
    sum(natten_block(x) * R)."""
    from gridcast import autodiff as ad
    from paper_2503_22235_b200.backward import block_vjp
    t = int(np.prod(ext))
    rng = np.random.default_rng(t)
    params = gc.attention.init_block_params(rng, dim, heads, "blk", zero_residual=False)
    xv = rng.standard_normal((t, dim))
    r = rng.standard_normal((t, dim))
    x = ad.Tensor(xv, requires_grad=True)
    y = gc.attention.natten_block(x, params, "blk", ext, win, heads)
    grads = ad.backward((y * ad.Tensor(r)).sum(), leaves=[x] + list(params.values()))
    gx, pg = block_vjp(xv, params, "blk", ext, win, heads, r)
    errs = {"x": _rel(gx, grads[x])}
    for n, p in params.items():
        assert pg[n].shape == p.values.shape, n
        errs[n] = _rel(pg[n], grads[p])
    worst = max(errs, key=errs.get)
    print(f"block VJP {ext} {win} D={dim}: worst {worst} {errs[worst]:.2e}, x {errs['x']:.2e}")
    assert errs[worst] < GRAD_TOL, (worst, errs[worst])


def test_block_vjp_deterministic(gc):
    from paper_2503_22235_b200.backward import block_vjp
    ext, win, dim, heads = (7, 9, 18), (5, 7, 7), 256, 2
    rng = np.random.default_rng(3)
    params = gc.attention.init_block_params(rng, dim, heads, "blk", zero_residual=False)
    x = rng.standard_normal((int(np.prod(ext)), dim))
    r = rng.standard_normal(x.shape)
    a = block_vjp(x, params, "blk", ext, win, heads, r)
    b = block_vjp(x, params, "blk", ext, win, heads, r)
    assert np.array_equal(a[0], b[0])
    assert all(np.array_equal(a[1][n], b[1][n]) for n in a[1])


def test_reference_offload_parity_check_through_seam(gc):
    """The reference's own verify.check_offload_parity (checkpointed vs OffloadEngine segments of the tiny
    processor, gradients compared as bytes) with every block on the B200, forward and backward; and its
    gradients against the pure-reference run of the same construction."""
    from gridcast import autodiff as ad
    from gridcast.model import LatentState, init_model_params, process, tiny_config
    from paper_2503_22235_b200 import integration

    cfg = tiny_config()
    params = init_model_params(cfg, seed=0, zero_residual=False)
    ext = (cfg.depth_planes, cfg.grid.rows // 8, cfg.grid.cols // 8)
    z0v = np.random.default_rng(2).standard_normal((int(np.prod(ext)), cfg.hidden))

    def run():
        z0 = ad.Tensor(z0v, requires_grad=True)
        z = z0
        for _ in range(3):
            z = ad.checkpoint_segment(lambda tk: process(LatentState(tk, 0, ext), params, cfg, 6).tokens, z)
        loss = (z * z).mean()
        return loss.values, ad.backward(loss, leaves=[z0])[z0]

    ref_loss, ref_g = run()
    integration.install(gc, operator=True, model_level=False)
    try:
        gc.verify.check_offload_parity()  # raises AssertionError on any byte difference
        loss, g = run()
    finally:
        integration.uninstall(gc)
    print(f"tiny 3-segment loss {float(loss):.6f} vs reference {float(ref_loss):.6f}; "
          f"dL/dz0 rel {_rel(g, ref_g):.2e}")
    assert abs(float(loss) - float(ref_loss)) < 1e-2 * abs(float(ref_loss))
    assert _rel(g, ref_g) < GRAD_TOL


def test_reference_train_step_and_driver_through_seam(gc):
    """The reference's shared-prefix train_step (training.py:211-241: encode, 6 h chain, hour tails, decode,
    normalized loss) and its training driver with the B200 blocks: loss and every block parameter gradient vs
    the pure reference; the driver's 20-step loss curve is repeatable and falls (reference test_training.py:204)."""
    from gridcast import autodiff as ad
    from gridcast.model import init_model_params, tiny_config
    from gridcast.synthdata import generate_dataset
    from gridcast.training import train, train_step
    from paper_2503_22235_b200 import integration

    cfg = tiny_config()
    ds = generate_dataset(cfg.grid, cfg.surface_in, cfg.surface_out, cfg.atmos_vars, cfg.levels, hours=26, seed=2)
    sig = ds.plane_sigmas()

    def step():
        params = init_model_params(cfg, seed=0, zero_residual=False)
        loss = train_step(params, cfg, ds, (1, 6, 7), 0, sig, stage="1h")
        grads = ad.backward(loss, leaves=list(params.values()))
        return float(loss.values), {n: grads[p] for n, p in params.items()}

    ref_loss, ref_grads = step()
    integration.install(gc, operator=True, model_level=False)
    try:
        loss, grads = step()
        hist = [train(init_model_params(cfg, seed=0), cfg, ds, "pretrain", steps=20, seed=5, lr_max=3e-3)
                for _ in range(2)]
    finally:
        integration.uninstall(gc)
    blk = [n for n in grads if ".blk" in n]
    errs = {n: _rel(grads[n], ref_grads[n]) for n in blk if np.linalg.norm(ref_grads[n]) > 0}
    worst = max(errs, key=errs.get)
    print(f"train_step loss {loss:.6f} vs reference {ref_loss:.6f}; worst block grad {worst} {errs[worst]:.2e}")
    assert abs(loss - ref_loss) < 1e-2 * abs(ref_loss)
    assert errs[worst] < 2 * GRAD_TOL, (worst, errs[worst])
    # the reference's test_training.py:204-216 on the B200 blocks: deterministic, and the loss falls
    l1, l2 = [r["loss"] for r in hist[0]], [r["loss"] for r in hist[1]]
    assert l1 == l2
    assert np.mean(l1[-5:]) < 0.8 * np.mean(l1[:5]), l1


def _ref_rollout_grads(gc, cfg_ref, params_ref, z0v, plan, R):
    from gridcast import autodiff as ad
    from gridcast.model import LatentState, process
    z0 = ad.Tensor(z0v, requires_grad=True)
    z = z0
    for h in plan:
        z = process(LatentState(z, 0, cfg_ref.latent_extents), params_ref, cfg_ref, h).tokens
    loss = (z * ad.Tensor(R)).sum()
    names = [n for n in params_ref if n.startswith("proc")]
    g = ad.backward(loss, leaves=[z0] + [params_ref[n] for n in names])
    return z.values, g[z0], {n: g[params_ref[n]] for n in names}


def test_rollout_vjp_matches_reference_tape(gc):
    """backward.rollout_vjp (device reverse mode of a (6, 1) greedy rollout, checkpointed per block) vs the
    reference tape through its own process() chain (float64): final latent, dL/dz0 and every processor-block
    parameter gradient (summed over the steps that apply it)."""
    import paper_2503_22235_b200.model as M
    from paper_2503_22235_b200.backward import rollout_vjp
    cfg = M.desk_config()
    params = M.init_model_params(cfg, seed=3, zero_residual=False)
    cfg_ref = gc.model.desk_config()
    params_ref = gc.model.init_model_params(cfg_ref, seed=3, zero_residual=False)
    t = int(np.prod(cfg.latent_extents))
    rng = np.random.default_rng(11)
    z0v = rng.standard_normal((t, cfg.hidden))
    R = rng.standard_normal((t, cfg.hidden))
    plan = (6, 1)
    ref_z, ref_gz, ref_pg = _ref_rollout_grads(gc, cfg_ref, params_ref, z0v, plan, R)
    z, gz, pg, st = rollout_vjp(z0v, plan, params, cfg, R)
    errs = {n: _rel(pg[n], ref_pg[n]) for n in pg if np.linalg.norm(ref_pg[n]) > 0}
    worst = max(errs, key=errs.get)
    zr, gr = _rel(z.double().cpu().numpy(), ref_z), _rel(gz, ref_gz)
    print(f"rollout (6, 1) desk: z {zr:.2e}, dL/dz0 {gr:.2e}, worst param {worst} {errs[worst]:.2e} "
          f"({len(errs)} tensors), store {st}")
    assert set(pg) == {n for n in ref_pg if any(n.startswith(f"proc{h}.") for h in plan)}
    assert zr < 1e-2 and gr < GRAD_TOL, (zr, gr)
    assert errs[worst] < GRAD_TOL, (worst, errs[worst])


@pytest.mark.parametrize("lookahead", [1, 2, 3])
def test_rollout_vjp_host_offload_bitwise(lookahead):
    """Saved block inputs offloaded to page-locked host memory on a side stream and prefetched `lookahead`
    blocks ahead (HostOffloadStore, the OffloadEngine counterpart of offload.py:287-412): gradients bitwise equal
    to keeping them in HBM (verify.py:73-113's offload-parity contract), no demand stalls, and device residency
    of saved inputs bounded by the ring (lookahead + 1 latents) instead of one latent per block."""
    import paper_2503_22235_b200.model as M
    from paper_2503_22235_b200.backward import rollout_vjp
    cfg = M.mid_config()
    params = M.init_model_params(cfg, seed=5, zero_residual=False)
    t = int(np.prod(cfg.latent_extents))
    rng = np.random.default_rng(4)
    z0v = rng.standard_normal((t, cfg.hidden))
    R = rng.standard_normal((t, cfg.hidden))
    plan = (6, 1)
    z_a, g_a, p_a, st_a = rollout_vjp(z0v, plan, params, cfg, R, offload=False)
    z_b, g_b, p_b, st_b = rollout_vjp(z0v, plan, params, cfg, R, offload=True, lookahead=lookahead)
    print(f"lookahead {lookahead}: {st_a} vs {st_b}")
    assert torch_equal(z_a, z_b)
    assert np.array_equal(g_a, g_b)
    assert set(p_a) == set(p_b) and all(np.array_equal(p_a[n], p_b[n]) for n in p_a)
    nbytes = t * cfg.hidden * 4
    assert st_a["high_water_bytes"] == 2 * cfg.proc_blocks * nbytes
    assert st_b["high_water_bytes"] == (lookahead + 1) * nbytes
    assert st_b["demand_stalls"] == 0 and st_b["transfers"] == 2 * 2 * cfg.proc_blocks


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


@pytest.mark.parametrize("ext,win,dim,heads", [
    ((5, 18, 36), (5, 7, 7), 1024, 8),   # full-scale block width on a smaller grid: row bump, column wrap
    ((5, 30, 60), (5, 7, 7), 256, 2),
    ((5, 90, 180), (5, 7, 7), 1024, 8),  # full scale
    ((6, 12, 20), (3, 5, 5), 256, 2),    # depth bump, smaller window
])
def test_tensor_core_attention_backward_matches_cuda_core(ext, win, dim, heads, monkeypatch):
    """The tcgen05 attention backward (wm3_natten_bwd: dQ per query tile, dK / dV as CSR-ordered sums of per-chunk
    partials) against the CUDA-core gather kernels (wm3_bw_natten) inside the same block VJP: input and every
    parameter gradient, and bitwise repeatable."""
    from paper_2503_22235_b200.backward import _TcAttention, block_vjp
    from paper_2503_22235_b200.params import init_block_params
    t = int(np.prod(ext))
    rng = np.random.default_rng(t + dim)
    params = init_block_params(rng, dim, heads, "blk", zero_residual=False)
    x = rng.standard_normal((t, dim))
    gy = rng.standard_normal((t, dim))
    dhp = (dim // heads + 63) // 64 * 64
    if _TcAttention.get(ext, win, heads, dhp) is None:
        assert ext != (5, 90, 180), "the full-scale geometry must run on the tensor-core path"
        pytest.skip("geometry outside the tensor-core backward (window mask does not fit the MMA bias step)")
    gx_tc, pg_tc = block_vjp(x, params, "blk", ext, win, heads, gy)
    gx_tc2, pg_tc2 = block_vjp(x, params, "blk", ext, win, heads, gy)
    monkeypatch.setenv("WM3_BW_NA", "cuda")
    gx_cc, pg_cc = block_vjp(x, params, "blk", ext, win, heads, gy)
    errs = {"x": _rel(gx_tc, gx_cc)}
    errs.update({n: _rel(pg_tc[n], pg_cc[n]) for n in pg_cc if np.linalg.norm(pg_cc[n]) > 0})
    worst = max(errs, key=errs.get)
    print(f"tc vs cuda-core attention backward {ext} D={dim}: x {errs['x']:.2e}, worst {worst} {errs[worst]:.2e}")
    assert errs[worst] < 5e-3, (worst, errs[worst])
    assert np.array_equal(gx_tc, gx_tc2) and all(np.array_equal(pg_tc[n], pg_tc2[n]) for n in pg_tc)


def test_host_offload_store_out_of_order_take():
    """HostOffloadStore: a take() the prefetch order did not anticipate is served on demand (counted as a stall)
    with the exact bytes; the ring slots are reused only after their last use (every saved latent comes back
    intact even with lookahead 1)."""
    import torch
    from paper_2503_22235_b200.backward import HostOffloadStore
    shape = (1000, 64)
    xs = [torch.randn(shape, device="cuda") for _ in range(6)]
    st = HostOffloadStore(shape, lookahead=1)
    for k, x in enumerate(xs):
        st.put(k, x)
    st.begin_backward([5, 4, 3, 2, 1, 0])
    got = {}
    for k in (5, 3, 4, 0, 2, 1):  # 3 and 0 out of order
        got[k] = st.take(k).clone()
        st.release(k)
    torch.cuda.synchronize()
    assert all(torch.equal(got[k], xs[k]) for k in range(6))
    assert st.stats()["demand_stalls"] >= 1


def test_gelu_rebuild_and_fused_stats_kernels():
    """wm3_bw_gelu_fwd rebuilds the forward's GELU activation bitwise from the fp32 pre-activation (the W1 GEMM
    is not re-run in the backward); wm3_bw_colsum_amax gives the same column sums and maxima as the separate
    wm3_bw_colsum / wm3_bw_amax passes, and its fused GELU backward the same values as wm3_bw_gelu."""
    import torch
    from paper_2503_22235_b200 import _lib, ops
    from paper_2503_22235_b200 import backward as bwd
    from paper_2503_22235_b200._lib import check, ptr, stream_ptr
    torch.manual_seed(3)
    T, k, n = 1000, 256, 512
    a = (torch.randn(T, k, device="cuda") * 0.5).to(_lib.ELEM)
    w = (torch.randn(n, k, device="cuda") * 0.1).to(_lib.ELEM)
    b = torch.randn(n, device="cuda") * 0.3
    ref = ops.linear(a, w, _lib.WM3_EPI_BIAS_GELU_BF16, bias=b)
    a0 = bwd._gemm(a, w, T, n, k)
    mid = torch.empty((T, n), dtype=_lib.ELEM, device="cuda")
    check(_lib.lib().wm3_bw_gelu_fwd(ptr(a0), n, ptr(b), T, n, ptr(mid), n, stream_ptr()), "wm3_bw_gelu_fwd")
    assert torch.equal(mid.view(torch.int16), ref[:, :n].contiguous().view(torch.int16))

    g = torch.randn(T, n, device="cuda") * 1e3
    cs, s = bwd._colsum_amax(g, T, n)
    assert torch.equal(cs, bwd._colsum(g, T, n))
    assert torch.equal(s.bits, bwd._amax(g, T, n).bits)
    s_in = bwd._amax(g, T, n)
    cs2, s2, ga = bwd._colsum_amax(g, T, n, gelu_of=a0, bias=b, in_scale=s_in)
    ga_ref = torch.empty_like(g)
    check(_lib.lib().wm3_bw_gelu(ptr(g), n, ptr(a0), n, ptr(b), T, n, s_in.ptr(), ptr(ga_ref), n, stream_ptr()),
          "wm3_bw_gelu")
    torch.testing.assert_close(ga, ga_ref, rtol=1e-6, atol=0)
    torch.testing.assert_close(cs2, bwd._colsum(ga, T, n), rtol=0, atol=0)
    assert torch.equal(s2.bits, bwd._amax(ga, T, n).bits)


def test_gelu_grad_gemm_epilogue():
    """wm3_linear_gelu_grad (the GELU backward in the gradient GEMM's epilogue, in place over the stored
    pre-activation) equals the separate path: fp32 GEMM, then wm3_bw_gelu."""
    import torch
    from paper_2503_22235_b200 import _lib
    from paper_2503_22235_b200 import backward as bwd
    from paper_2503_22235_b200._lib import check, ptr, stream_ptr
    torch.manual_seed(5)
    for T, n, k in ((1000, 512, 256), (333, 256, 64), (4096, 1024, 1024)):
        a = (torch.randn(T, k, device="cuda")).to(_lib.ELEM)
        w = (torch.randn(n, k, device="cuda") * 0.1).to(_lib.ELEM)
        b = torch.randn(n, device="cuda") * 0.3
        pre = torch.randn(T, n, device="cuda") * 2
        s = bwd._Scale(a.device)
        s.bits.view(torch.float32).fill_(3.0e-3)   # scale 2^(14 - ceil(log2 3e-3)) = 2^23
        g = bwd._gemm(a, w, T, n, k)
        ref = torch.empty_like(g)
        check(_lib.lib().wm3_bw_gelu(ptr(g), n, ptr(pre), n, ptr(b), T, n, s.ptr(), ptr(ref), n, stream_ptr()),
              "wm3_bw_gelu")
        out = pre.clone()
        so = bwd._Scale(a.device)
        check(_lib.lib().wm3_linear_gelu_grad(ptr(a), k, ptr(w), k, T, n, k, ptr(out), n, ptr(b), s.ptr(), so.ptr(),
                                              stream_ptr()), "wm3_linear_gelu_grad")
        torch.testing.assert_close(out, ref, rtol=2e-6, atol=1e-30)
        assert torch.equal(so.bits, bwd._amax(out, T, n).bits)  # the epilogue's max |out| = a separate pass
        # the one-pass cast + column sums against the separate cast and column sums
        oh, cs = bwd._cast_colsum(out, T, n, n + 64, so)
        assert torch.equal(oh[:, :n], bwd._cast(out, T, n, n, scale=so)) and not oh[:, n:].any()
        torch.testing.assert_close(cs, bwd._colsum(out, T, n), rtol=0, atol=0)


@pytest.mark.parametrize("m,n,k", [(256, 256, 20000), (1024, 1024, 81000), (3072, 1024, 5000), (128, 192, 700)])
def test_linear_tn_split_k(m, n, k):
    """wm3_linear_tn_split (weight-gradient GEMM C = A^T B over the token axis, K range split over the CTA pairs
    when the output has few tiles): equal to the fp64 product within fp32 accumulation error, and run-to-run
    bitwise (the split partials are summed in a fixed order)."""
    import torch
    from paper_2503_22235_b200 import _lib
    from paper_2503_22235_b200 import backward as bwd
    torch.manual_seed(m + k)
    a = torch.randn(k, m, device="cuda").to(_lib.ELEM)
    b = torch.randn(k, n, device="cuda").to(_lib.ELEM)
    c = bwd._gemm_tn(a, b, m, n, k)
    ref = a.double().T @ b.double()
    err = float((c.double() - ref).norm() / ref.norm())
    print(f"linear_tn_split {m}x{n}x{k}: rel err {err:.2e}")
    assert err < 2e-6 * max(1.0, (k / 1000) ** 0.5), err  # fp32 accumulation over k terms
    assert torch.equal(c, bwd._gemm_tn(a, b, m, n, k))
