"""Model-level parity on the B200: encode / process / rollout / decode / forecast vs the float64 oracle.

Stated tolerances: one step per-variable relative L2 <= 1e-2; latent after a
multi-step rollout <= 2e-2.  Composition identities of the reference (test_rollout.py) hold bitwise.
"""

import numpy as np
import pytest

from oracle import model as om

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2503_22235_b200.model as m
    import paper_2503_22235_b200.rollout as r
    return m, r


def _state(cfg, seed=1, t=0):
    m, _ = _pkg()
    rng = np.random.default_rng(seed)
    g = cfg.grid
    return m.WeatherState(t, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                          rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def per_variable_rel(surface, atmos, ref_surface, ref_atmos):
    """Relative L2 keyed like the reference CLI's evaluation report (cli.py:248-268)."""
    out = {f"sfc{i}": _rel(surface[i], ref_surface[i]) for i in range(surface.shape[0])}
    for a in range(atmos.shape[0]):
        for lev in range(atmos.shape[1]):
            out[f"atm{a}.lev{lev}"] = _rel(atmos[a, lev], ref_atmos[a, lev])
    return out


@pytest.fixture(scope="module", params=["tiny", "desk", "mid"])
def setup(request):
    m, _ = _pkg()
    cfg = {"tiny": m.tiny_config, "desk": m.desk_config, "mid": m.mid_config}[request.param]()
    params = m.init_model_params(cfg, seed=7, zero_residual=False)
    host = {k: v.values for k, v in params.items()}
    return request.param, cfg, params, host


def test_encode_matches_oracle(setup):
    name, cfg, params, host = setup
    m, _ = _pkg()
    st = _state(cfg)
    lat = m.encode(st, params, cfg)
    ref = om.encode(st.surface, st.atmos, host, cfg)
    assert lat.tokens.shape == (cfg.tokens, cfg.hidden)
    assert lat.valid_time == 0 and tuple(lat.extents) == cfg.latent_extents
    assert _rel(lat.tokens.values, ref) < 1e-2


def test_one_step_forecast_per_variable(setup):
    name, cfg, params, host = setup
    m, r = _pkg()
    st = _state(cfg, seed=3)
    out = r.forecast(st, 6, params, cfg)
    ref_s, ref_a = om.forecast(st.surface, st.atmos, 6, host, cfg)
    assert out.valid_time == 6
    g = cfg.grid
    assert out.surface.shape == (cfg.surface_out, g.rows, g.cols)
    assert out.atmos.shape == (cfg.atmos_vars, cfg.levels, g.rows, g.cols)
    rel = per_variable_rel(out.surface.values, out.atmos.values, ref_s, ref_a)
    worst = max(rel, key=rel.get)
    vals = np.array(sorted(rel.values()))
    print(f"[{name}] per-variable rel L2: median {np.median(vals):.2e} p90 {vals[int(0.9 * len(vals))]:.2e} "
          f"max {vals[-1]:.2e} ({worst})")
    assert rel[worst] < 1e-2, (worst, rel[worst])


def test_mixed_rollout_latent_parity(setup):
    """(6, 1): both processors, latent-space parity (config 4 of BASELINE.json at test scale)."""
    name, cfg, params, host = setup
    m, r = _pkg()
    st = _state(cfg, seed=4)
    lat = m.encode(st, params, cfg)
    out = r.rollout(lat, r.greedy_plan(7), params, cfg)
    ref = om.rollout(om.encode(st.surface, st.atmos, host, cfg), (6, 1), host, cfg)
    assert out.valid_time == 7
    assert _rel(out.tokens.values, ref) < 2e-2


def test_rollout_composition_bitwise(setup):
    name, cfg, params, host = setup
    m, r = _pkg()
    lat = m.encode(_state(cfg, seed=5), params, cfg)
    direct = m.process(m.process(lat, params, cfg, 6), params, cfg, 6)
    rolled = r.rollout(lat, (6, 6), params, cfg)                 # CUDA-graph replay
    plain = r.rollout(lat, (6, 6), params, cfg, graphs=False)    # eager launches
    assert rolled.tokens.values.tobytes() == direct.tokens.values.tobytes()
    assert plain.tokens.values.tobytes() == direct.tokens.values.tobytes()
    assert rolled.valid_time == 12


def test_forecast_matches_manual_composition_bitwise(setup):
    name, cfg, params, host = setup
    m, r = _pkg()
    st = _state(cfg, seed=6)
    out = r.forecast(st, 12, params, cfg)
    manual = m.decode(m.process(m.process(m.encode(st, params, cfg), params, cfg, 6), params, cfg, 6), params, cfg)
    assert out.surface.values.tobytes() == manual.surface.values.tobytes()
    assert out.atmos.values.tobytes() == manual.atmos.values.tobytes()
    zero = r.forecast(st, 0, params, cfg)
    enc_dec = m.decode(m.encode(st, params, cfg), params, cfg)
    assert zero.surface.values.tobytes() == enc_dec.surface.values.tobytes()


def test_ensemble_rollout_members_bitwise(setup):
    """Config 5's ensemble batch: every member of one batched rollout equals its own single rollout."""
    name, cfg, params, host = setup
    m, r = _pkg()
    members = r.perturbed_members(_state(cfg, seed=8), 3, scale=0.05)
    lats = [m.encode(s, params, cfg) for s in members]
    ens = r.rollout_ensemble(lats, (6, 1), params, cfg)
    eager = r.rollout_ensemble(lats, (6, 1), params, cfg, graphs=False)
    for k, lt in enumerate(lats):
        one = r.rollout(lt, (6, 1), params, cfg)
        assert ens[k].valid_time == 7
        assert ens[k].tokens.values.tobytes() == one.tokens.values.tobytes(), k
        assert eager[k].tokens.values.tobytes() == one.tokens.values.tobytes(), k
    assert not np.array_equal(ens[0].tokens.values, ens[1].tokens.values)
    assert r.rollout_ensemble(lats, (), params, cfg)[0] is lats[0]
    fc = r.forecast_ensemble(members[:2], 6, params, cfg)
    single = r.forecast(members[1], 6, params, cfg)
    assert fc[1].surface.values.tobytes() == single.surface.values.tobytes()


def test_call_counts_and_plan_rejection(setup):
    name, cfg, params, host = setup
    m, r = _pkg()
    from paper_2503_22235_b200.errors import ConfigError
    lat = m.encode(_state(cfg), params, cfg)
    m.reset_call_counts()
    r.rollout(lat, r.greedy_plan(14), params, cfg)
    assert m.CALL_COUNTS == {"encode": 0, "process1": 2, "process6": 2, "decode": 0}
    assert r.rollout(lat, (), params, cfg) is lat
    pruned = {k: v for k, v in params.items() if not k.startswith("proc1.")}
    m.reset_call_counts()
    with pytest.raises(ConfigError):
        r.rollout(lat, (6, 1), pruned, cfg)
    assert m.CALL_COUNTS["process6"] == 0


def test_zero_residual_decodes_to_zero():
    m, r = _pkg()
    cfg = m.tiny_config()
    params = m.init_model_params(cfg, seed=3, zero_residual=True)
    out = m.decode(m.encode(_state(cfg), params, cfg), params, cfg)
    assert np.abs(out.surface.values).max() == 0.0
    assert np.abs(out.atmos.values).max() == 0.0


def test_encode_rejects_bad_shapes():
    m, _ = _pkg()
    from paper_2503_22235_b200.errors import ConfigError
    cfg = m.tiny_config()
    params = m.init_model_params(cfg, seed=7, zero_residual=False)
    st = _state(cfg)
    st.surface = st.surface[:1]
    with pytest.raises(ConfigError):
        m.encode(st, params, cfg)
    with pytest.raises(ConfigError):
        m.encode(_state(cfg), params, cfg, source="ghost")


def test_folded_layernorm_chain(monkeypatch):
    """WM3_LN_FOLD=1 (LayerNorm folded into the GEMM epilogues): blocks after the first of each chain take x's fp16
    copy and row statistics from the previous block's W2 epilogue (graph-captured rollout, banded processor).
    Forecast parity with the oracle and agreement with the separate-LayerNorm path."""
    m, r = _pkg()
    from paper_2503_22235_b200.bands import forecast_banded
    cfg = m.mid_config()
    st = _state(cfg, seed=6)
    plain = m.init_model_params(cfg, seed=7, zero_residual=False)
    ref_s, ref_a = om.forecast(st.surface, st.atmos, 7, {k: v.values for k, v in plain.items()}, cfg)
    base = r.forecast(st, 7, plain, cfg)
    monkeypatch.setenv("WM3_LN_FOLD", "1")
    folded = m.init_model_params(cfg, seed=7, zero_residual=False)  # fresh dict: blocks prepared folded
    out = r.forecast(st, 7, folded, cfg)
    from paper_2503_22235_b200.runtime import CACHE
    assert CACHE.block(folded, "proc6.blk3", cfg.heads).folded
    rel = per_variable_rel(out.surface.values, out.atmos.values, ref_s, ref_a)
    assert max(rel.values()) < 1e-2, max(rel.values())
    assert _rel(out.surface.values, base.surface.values) < 5e-3
    banded = forecast_banded(st, 7, folded, cfg, world=2)
    assert _rel(banded.surface.values, out.surface.values) < 5e-3


@pytest.mark.parametrize("scale", [1e3, 1e5, float("nan")])
def test_input_range_guard(scale):
    """fp16 operands hold |x| <= 65504: inputs scaled by 1e3 (max ~5e3) still forecast within the one-step
    tolerance of the float64 oracle on the same scaled input; 1e5 (beyond the fp16 range) and non-finite
    inputs raise ConfigError from encode instead of convolving infinities (the reference accepts any float64
    magnitude, fields_to_nhwc sets a device flag that encode checks)."""
    m, r = _pkg()
    from paper_2503_22235_b200.errors import ConfigError
    cfg = m.desk_config()
    params = m.init_model_params(cfg, seed=7, zero_residual=False)
    st = _state(cfg, seed=9)
    if np.isnan(scale):
        st.atmos = st.atmos.copy()
        st.atmos[1, 2, 3, 4] = np.nan
    else:
        st = m.WeatherState(0, st.surface * scale, st.atmos * scale)
    if np.isnan(scale) or scale > 65504 / 8:
        with pytest.raises(ConfigError):
            m.encode(st, params, cfg)
        with pytest.raises(ConfigError):
            r.forecast(st, 6, params, cfg)
        return
    out = r.forecast(st, 6, params, cfg)
    host = {k: v.values for k, v in params.items()}
    ref_s, ref_a = om.forecast(st.surface, st.atmos, 6, host, cfg)
    rel = per_variable_rel(out.surface.values, out.atmos.values, ref_s, ref_a)
    worst = max(rel, key=rel.get)
    print(f"inputs x{scale:g}: worst per-variable rel L2 {rel[worst]:.2e} ({worst})")
    assert np.isfinite(out.surface.values).all() and np.isfinite(out.atmos.values).all()
    assert rel[worst] < 1e-2, (worst, rel[worst])


def test_decode_streamed_to_host_equals_batched():
    """decode(..., host_out=bufs): the full-resolution stage runs plane by plane with each plane's fields copied out
    on a side stream; the host fields are bitwise the batched decode's, and to_host(bufs) returns them as is."""
    import torch
    import paper_2503_22235_b200.model as M
    from paper_2503_22235_b200.tensor import Tensor
    for cfg in (M.desk_config(), M.mid_config()):
        params = M.init_model_params(cfg, seed=4, zero_residual=False)
        rng = np.random.default_rng(9)
        lat = M.LatentState(Tensor(rng.standard_normal((cfg.tokens, cfg.hidden))), 6, cfg.latent_extents)
        ref = M.decode(lat, params, cfg)
        s_ref, a_ref = ref.to_host()
        bufs = (torch.full_like(s_ref, float("nan")), torch.full_like(a_ref, float("nan")))
        bufs = tuple(b.pin_memory() for b in bufs)
        out = M.decode(lat, params, cfg, host_out=bufs)
        s, a = out.to_host(bufs)
        assert s is bufs[0] and a is bufs[1]
        assert torch.equal(s, s_ref) and torch.equal(a, a_ref)
        assert torch.equal(out.surface.device.cpu(), s_ref)


def test_encode_streamed_from_pinned_equals_numpy():
    """encode() of page-locked float32 host fields streams the planes in on a copy stream with per-plane stem
    convolutions; the latent is bitwise the one encoded from the same values as numpy arrays."""
    import torch
    import paper_2503_22235_b200.model as M
    for cfg in (M.desk_config(), M.mid_config()):
        params = M.init_model_params(cfg, seed=6, zero_residual=False)
        g = cfg.grid
        rng = np.random.default_rng(2)
        s = rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)
        a = rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32)
        ref = M.encode(M.WeatherState(0, s, a), params, cfg).tokens.device.clone()
        st = M.WeatherState(0, torch.from_numpy(s).pin_memory(), torch.from_numpy(a).pin_memory())
        got = M.encode(st, params, cfg).tokens.device
        assert torch.equal(got, ref)
