"""INTEGRATION.md §2 applied to the UNMODIFIED reference package (gridcast, staged into baseline/_ref by
baseline/stage_ref.sh; it travels to the GPU box with the repo snapshot): the reference's own callers run
through the B200 seam and must reproduce the reference's own results within the stated tolerances.

  * operator seam: only `gridcast.model.natten_block` rebound — the reference's encode / process / decode
    (model.py:363-421, with its own convolutions and `tokens.reshape`, model.py:357-360) call the B200 block;
  * full rebinding (INTEGRATION.md §2 verbatim): gridcast.rollout.forecast / rollout and gridcast.model names;
  * verify.check_roll_equivariance's construction (verify.py:51-70) through gridcast.attention.natten_block;
  * the seam is recorded on the reference's tape and refuses backward (forward-only) instead of cutting
    gradients;
  * in-place parameter updates (training.py:144) reach the device weights and rollout graphs.
"""

import contextlib
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

ONE_STEP_TOL = 1e-2    # one step, per variable relative L2
ROLLOUT_TOL = 2e-2     # full rollout


@pytest.fixture(scope="module")
def gc():
    if not os.path.isdir(os.path.join(REF, "gridcast")):
        pytest.skip("reference not staged: run baseline/stage_ref.sh")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gridcast
    import gridcast.attention
    import gridcast.cli
    import gridcast.model
    import gridcast.rollout
    return gridcast


@contextlib.contextmanager
def rebound(gc, operator_only=False):
    """paper_2503_22235_b200.integration.install (the assignments of INTEGRATION.md §2), undone afterwards."""
    from paper_2503_22235_b200 import integration
    if operator_only:
        integration.install(gc, operator=True, model_level=False)
    else:
        integration.install(gc, operator=True)
    try:
        yield
    finally:
        integration.uninstall(gc)


def _state(gc, cfg, seed=1):
    rng = np.random.default_rng(seed)
    g = cfg.grid
    return gc.model.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                                 rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))


def _per_variable(a_sfc, a_atm, b_sfc, b_atm):
    out = {}
    for i in range(a_sfc.shape[0]):
        out[f"sfc{i}"] = np.linalg.norm(a_sfc[i] - b_sfc[i]) / np.linalg.norm(b_sfc[i])
    for a in range(a_atm.shape[0]):
        for lev in range(a_atm.shape[1]):
            out[f"atm{a}.lev{lev}"] = np.linalg.norm(a_atm[a, lev] - b_atm[a, lev]) / np.linalg.norm(b_atm[a, lev])
    return out


def test_operator_seam_runs_reference_encode_process_decode(gc):
    """Only gridcast.model.natten_block rebound: the reference's encode -> process(6) -> decode, with its own
    convolutions and token relayouts, gets reference Tensors back from every B200 block."""
    cfg = gc.model.desk_config()
    params = gc.model.init_model_params(cfg, seed=3, zero_residual=False)
    st = _state(gc, cfg)
    ref_lat = gc.model.process(gc.model.encode(st, params, cfg), params, cfg, 6)
    ref = gc.model.decode(ref_lat, params, cfg)
    with rebound(gc, operator_only=True):
        lat = gc.model.encode(st, params, cfg)
        assert type(lat.tokens) is type(ref_lat.tokens)  # the reference's Tensor class, not ours
        lat = gc.model.process(lat, params, cfg, 6)
        out = gc.model.decode(lat, params, cfg)
    rel_lat = np.linalg.norm(lat.tokens.values - ref_lat.tokens.values) / np.linalg.norm(ref_lat.tokens.values)
    assert rel_lat < ONE_STEP_TOL, rel_lat
    errs = _per_variable(out.surface.values, out.atmos.values, ref.surface.values, ref.atmos.values)
    worst = max(errs, key=errs.get)
    print(f"operator seam desk: latent {rel_lat:.2e}, worst variable {worst} {errs[worst]:.2e}")
    assert errs[worst] < ONE_STEP_TOL, (worst, errs[worst])
    assert not np.array_equal(out.surface.values, ref.surface.values)  # the B200 blocks really ran


def test_full_rebinding_forecast_and_rollout(gc):
    """INTEGRATION.md §2 verbatim: gridcast.rollout.forecast(state, 7) (plan (6, 1)) and gridcast.rollout.rollout
    through the B200 path vs the plain reference, per variable."""
    cfg = gc.model.desk_config()
    params = gc.model.init_model_params(cfg, seed=5, zero_residual=False)
    st = _state(gc, cfg, seed=2)
    ref = gc.rollout.forecast(st, 7, params, cfg)
    ref_lat = gc.rollout.rollout(gc.model.encode(st, params, cfg), (6, 6), params, cfg)
    with rebound(gc):
        out = gc.rollout.forecast(st, 7, params, cfg)
        lat = gc.rollout.rollout(gc.model.encode(st, params, cfg), (6, 6), params, cfg)
        dec = gc.model.decode(lat, params, cfg)  # rebound too: a B200 latent never reaches reference code
    assert out.valid_time == ref.valid_time == 7 and lat.valid_time == ref_lat.valid_time == 12
    errs = _per_variable(out.surface.values, out.atmos.values, ref.surface.values, ref.atmos.values)
    worst = max(errs, key=errs.get)
    print(f"rebound forecast(7) desk: worst variable {worst} {errs[worst]:.2e}")
    assert errs[worst] < ROLLOUT_TOL, (worst, errs[worst])
    rel = np.linalg.norm(lat.tokens.values - ref_lat.tokens.values) / np.linalg.norm(ref_lat.tokens.values)
    assert rel < ROLLOUT_TOL, rel
    assert dec.surface.values.shape == ref.surface.values.shape


def test_reference_cli_forecast_through_install(gc, tmp_path):
    """The reference's own CLI (`gridcast forecast`, cli.py:160-224: its config / LMTW / WMD3 loaders, blend,
    greedy plan and writer) with the B200 path installed, on the reference-generated CLI fixtures: equal to the
    reference CLI's own output file within the one-step tolerance per variable."""
    import gridcast.cli as gcli
    from paper_2503_22235_b200 import integration
    from paper_2503_22235_b200.serialization import load_params_file
    gold = os.path.join(ROOT, "tests", "golden", "cli")
    out = tmp_path / "fc.lmtw"
    argv = ["forecast", "--config", os.path.join(gold, "tiny.cfg"), "--params", os.path.join(gold, "params.lmtw"),
            "--init", os.path.join(gold, "data.wmd3"), "--init-hour", "4", "--dt", "7", "--source", "primary",
            "--source", "op1", "--out", str(out)]
    integration.install(gc)
    try:
        assert "gridcast.cli.rollout" in integration.installed()
        assert gcli.main(argv) == 0
    finally:
        integration.uninstall(gc)
    got, ref = load_params_file(out), load_params_file(os.path.join(gold, "fc_blend.lmtw"))
    assert float(got["valid_time"]) == float(ref["valid_time"])
    errs = _per_variable(got["surface"], got["atmos"], ref["surface"], ref["atmos"])
    worst = max(errs, key=errs.get)
    assert errs[worst] < ONE_STEP_TOL, (worst, errs[worst])
    assert not np.array_equal(got["surface"], ref["surface"])  # the B200 path really ran


def test_roll_equivariance_through_seam(gc):
    """verify.check_roll_equivariance's construction (verify.py:51-70: extents (3, 4, 8), window (3, 3, 3), dim
    12, 2 heads, a 3-column longitude roll) through the rebound gridcast.attention.natten_block.  The reference
    demands 1e-9 in float64; the B200 block's 16-bit operands bound it at fp16 rounding of the block update."""
    from gridcast import autodiff as ad
    extents, dim, heads = (3, 4, 8), 12, 2
    rng = np.random.default_rng(1)
    params = gc.attention.init_block_params(rng, dim, heads, "blk", zero_residual=False)
    t = extents[0] * extents[1] * extents[2]
    x = rng.standard_normal((t, dim))
    with rebound(gc):
        def run(arr):
            with ad.no_grad():
                return gc.attention.natten_block(ad.Tensor(arr), params, "blk", extents, (3, 3, 3), heads).values
        y = run(x).reshape(*extents, dim)
        xs = np.roll(x.reshape(*extents, dim), 3, axis=2).reshape(t, dim)
        ys = run(xs).reshape(*extents, dim)
    err = np.max(np.abs(np.roll(y, 3, axis=2) - ys))
    print(f"roll equivariance through the seam: max abs {err:.2e}")
    assert err < 5e-3, err


def test_seam_on_the_reference_tape(gc):
    """Grad mode on, input requiring grad: the B200 block is recorded on the reference's tape like the reference
    block (its output requires grad) with the B200 block VJP as its rule (backward.py), so a backward sweep that
    reaches it returns the reference tape's input gradient within the gradient tolerance; under no_grad
    nothing is recorded and the forward values are the same."""
    from gridcast import autodiff as ad
    extents, dim, heads = (3, 4, 8), 12, 2
    rng = np.random.default_rng(4)
    params = gc.attention.init_block_params(rng, dim, heads, "blk", zero_residual=False)
    xv = rng.standard_normal((96, dim))
    x_ref = ad.Tensor(xv, requires_grad=True)
    y_ref = gc.attention.natten_block(x_ref, params, "blk", extents, (3, 3, 3), heads)
    g_ref = ad.backward((y_ref * y_ref).mean(), leaves=[x_ref])[x_ref]
    x = ad.Tensor(xv, requires_grad=True)
    with rebound(gc):
        y = gc.attention.natten_block(x, params, "blk", extents, (3, 3, 3), heads)
        assert isinstance(y, ad.Tensor) and y.requires_grad and y.node is not None
        g = ad.backward((y * y).mean(), leaves=[x])[x]
        with ad.no_grad():
            z = gc.attention.natten_block(x, params, "blk", extents, (3, 3, 3), heads)
    g_ref, g = np.asarray(getattr(g_ref, "values", g_ref)), np.asarray(getattr(g, "values", g))
    rel = np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref)
    print(f"input gradient through the seam vs the reference tape: rel L2 {rel:.2e}")
    assert rel < 1e-2, rel
    assert not z.requires_grad and z.node is None
    np.testing.assert_array_equal(y.values, z.values)


def test_in_place_parameter_update_reaches_the_device():
    """The reference's optimizer updates parameters in place (training.py:144, `p.values -= lr * ...`): the
    next process / graph-captured rollout must use the new values, equal to a fresh parameter dict's."""
    import paper_2503_22235_b200.model as M
    import paper_2503_22235_b200.rollout as R
    from paper_2503_22235_b200.tensor import Tensor
    cfg = M.desk_config()
    params = M.init_model_params(cfg, seed=7, zero_residual=False)
    rng = np.random.default_rng(3)
    lat = M.LatentState(Tensor(rng.standard_normal((cfg.tokens, cfg.hidden))), 0, cfg.latent_extents)
    before_p = M.process(lat, params, cfg, 6).tokens.values
    before_r = R.rollout(lat, (6, 6), params, cfg).tokens.values  # captures the rollout graph
    for name in ("proc6.blk0.attn.wo", "proc6.blk3.mlp.w2", "proc6.blk1.ln1.gain"):
        params[name].values -= 0.05 * rng.standard_normal(params[name].values.shape)
    after_p = M.process(lat, params, cfg, 6).tokens.values
    after_r = R.rollout(lat, (6, 6), params, cfg).tokens.values
    fresh = {k: Tensor(v.values.copy()) for k, v in params.items()}
    want_p = M.process(lat, fresh, cfg, 6).tokens.values
    want_r = R.rollout(lat, (6, 6), fresh, cfg).tokens.values
    assert not np.array_equal(after_p, before_p) and not np.array_equal(after_r, before_r)
    assert np.array_equal(after_p, want_p)
    assert np.array_equal(after_r, want_r)


def test_in_place_pyramid_update_reaches_the_device():
    """Encoder / decoder pyramid weights updated in place (the same optimizer step) are picked up by the next
    encode / decode: the device model checks the content of the pyramid arrays it uses on every call."""
    import paper_2503_22235_b200.model as M
    from paper_2503_22235_b200.tensor import Tensor
    cfg = M.desk_config()
    params = M.init_model_params(cfg, seed=11, zero_residual=False)
    rng = np.random.default_rng(5)
    g = cfg.grid
    st = M.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32))
    lat0 = M.encode(st, params, cfg)
    dec0 = M.decode(lat0, params, cfg).surface.device.cpu().numpy()
    before = lat0.tokens.device.cpu().numpy()
    for name in ("enc.stem_atm.w", "enc.stage1.res0.conv2.w", "dec.stage0.res1.conv1.w"):
        if name in params:
            params[name].values -= 0.05 * rng.standard_normal(params[name].values.shape)
    fresh = {k: Tensor(v.values.copy()) for k, v in params.items()}
    lat1 = M.encode(st, params, cfg)
    after = lat1.tokens.device.cpu().numpy()
    want = M.encode(st, fresh, cfg).tokens.device.cpu().numpy()
    assert not np.array_equal(after, before) and np.array_equal(after, want)
    dec1 = M.decode(lat0, params, cfg).surface.device.cpu().numpy()
    dec_want = M.decode(lat0, fresh, cfg).surface.device.cpu().numpy()
    assert not np.array_equal(dec1, dec0) and np.array_equal(dec1, dec_want)
