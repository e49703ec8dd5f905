"""CPU: host-side logic of the B200 path (config, plan, weight layout, rotary tables, C ABI surface)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from oracle import model as om
from paper_2503_22235_b200 import config as C
from paper_2503_22235_b200.errors import ConfigError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------------------------------------
# configuration (model.py:61-124, 456-607)
# ------------------------------------------------------------------------------------------------
def test_named_configs():
    assert C.desk_config().latent_extents == (3, 5, 10) and C.desk_config().tokens == 150
    full = C.full_scale_config()
    assert full.latent_extents == (5, 90, 180) and full.window == (5, 7, 7) and full.hidden == 1024
    assert C.tiny_config().latent_extents == (3, 3, 3)
    assert C.mid_config().latent_extents == (7, 9, 18) and C.mid_config().head_dim == 128


@pytest.mark.parametrize("kw", [dict(levels=7, level_patch=4), dict(window=(5, 3, 3)),
                                dict(hidden=50, stage_channels=(24, 32, 50)), dict(horizons=(1, 1))])
def test_config_validation(kw):
    with pytest.raises(ConfigError):
        C.ModelConfig(grid=C.desk_grid(), **kw)


def test_grid_validation():
    with pytest.raises(ConfigError):
        C.ModelConfig(grid=C.GridSpec(rows=36, cols=80, lat_step=4.5, lon_step=4.5))
    with pytest.raises(ConfigError):
        C.GridSpec(rows=10, cols=7, lon_step=4.5)
    with pytest.raises(ConfigError):
        C.GridSpec(rows=721, cols=1440)  # reaches the south pole, declared omitted


def test_config_file_round_trip(tmp_path):
    cfg = C.desk_config()
    path = tmp_path / "model.cfg"
    C.save_config(path, cfg)
    assert C.load_config(path) == cfg
    text = path.read_text()
    assert "rows = 40" in text and "window = 3,3,3" in text
    path.write_text(text + "banana = 1\n")
    with pytest.raises(ConfigError):
        C.load_config(path)
    (tmp_path / "short.cfg").write_text("rows = 40\n")
    with pytest.raises(ConfigError):
        C.load_config(tmp_path / "short.cfg")
    assert C.config_from_dict(C.config_to_dict(C.tiny_config())) == C.tiny_config()


def test_shape_plan():
    from paper_2503_22235_b200.params import init_model_params
    plan = C.shape_plan(C.full_scale_config())
    assert plan["latent_extents"] == (5, 90, 180) and plan["attention_keys"] == 245
    assert plan["surface_output"] == (17, 720, 1440) and plan["atmos_output"] == (5, 28, 720, 1440)
    assert plan["param_elements"] == 382_781_428
    for cfg in (C.tiny_config(), C.desk_config()):
        p = init_model_params(cfg, seed=0)
        assert C.shape_plan(cfg)["param_elements"] == sum(v.size for v in p.values())


# ------------------------------------------------------------------------------------------------
# rollout plan (rollout.py:33-53)
# ------------------------------------------------------------------------------------------------
def test_greedy_plan():
    from paper_2503_22235_b200.rollout import greedy_plan, plan_hours
    for dt in range(0, 337):
        plan = greedy_plan(dt)
        assert plan == (6,) * (dt // 6) + (1,) * (dt % 6) and plan_hours(plan) == dt
    assert greedy_plan(7) == (6, 1) and greedy_plan(23) == (6, 6, 6, 1, 1, 1, 1, 1)
    assert greedy_plan(400, max_dt=500) == (6,) * 66 + (1,) * 4
    for bad in (-1, 337, 2.5, True):
        with pytest.raises(ConfigError):
            greedy_plan(bad)


# ------------------------------------------------------------------------------------------------
# weight layout / rotary tables used by the kernels
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dh", [6, 12, 64, 128])
def test_qk_permutation_preserves_rotated_dot_products(dh):
    """Interleaving rotary pairs (j, j+dh/2) -> (2j, 2j+1) on q and k leaves q.k of rotated vectors unchanged."""
    from paper_2503_22235_b200.blocks import _qk_perm, head_pad
    heads, dhp = 2, head_pad(dh)
    perm = _qk_perm(heads, dh, dhp)
    rng = np.random.default_rng(0)
    q, k = rng.standard_normal((heads * dh,)), rng.standard_normal((heads * dh,))
    ang = rng.uniform(0, 6.3, dh // 2)
    c, s = np.cos(ang), np.sin(ang)

    def rot_ref(v):
        v = v.reshape(heads, dh)
        a, b = v[:, :dh // 2], v[:, dh // 2:]
        return np.concatenate([a * c - b * s, a * s + b * c], axis=1).reshape(-1)

    def rot_perm(v):  # what the QKV epilogue does on interleaved pairs
        w = np.zeros(heads * dhp)
        w[perm >= 0] = v[perm[perm >= 0]]
        w = w.reshape(heads, dhp)
        x1, x2 = w[:, 0:dh:2].copy(), w[:, 1:dh:2].copy()
        w[:, 0:dh:2], w[:, 1:dh:2] = x1 * c - x2 * s, x1 * s + x2 * c
        return w.reshape(-1)

    for hh in range(heads):
        ref = rot_ref(q)[hh * dh:(hh + 1) * dh] @ rot_ref(k)[hh * dh:(hh + 1) * dh]
        got = rot_perm(q)[hh * dhp:(hh + 1) * dhp] @ rot_perm(k)[hh * dhp:(hh + 1) * dhp]
        assert abs(ref - got) < 1e-12


@pytest.mark.parametrize("ext,dh", [((5, 90, 180), 128), ((7, 9, 18), 128), ((3, 5, 10), 12), ((2, 7, 10), 6)])
def test_rope_axis_tables_match_reference_angles(ext, dh):
    from paper_2503_22235_b200.blocks import rope_axis_tables
    cos, sin, pd, pr, emax = rope_axis_tables(ext, dh)
    ang = om.rotary_angles(ext, dh)
    d, h, w = ext
    di, hi, wi = np.unravel_index(np.arange(d * h * w), (d, h, w))
    n = dh // 2
    idx = np.arange(n)
    axis = np.where(idx < pd, 0, np.where(idx < pd + pr, 1, 2))
    coord = np.stack([di, hi, wi])[axis]  # (n, T)
    got_c = cos[axis[:, None], coord, idx[:, None]].T
    got_s = sin[axis[:, None], coord, idx[:, None]].T
    np.testing.assert_allclose(got_c, np.cos(ang), atol=2e-7)
    np.testing.assert_allclose(got_s, np.sin(ang), atol=2e-7)


def test_static_fields_match_oracle():
    from paper_2503_22235_b200.grid import static_fields
    for g in (C.desk_grid(), C.GridSpec(72, 144, lat_step=2.5, lon_step=2.5), C.tiny_config().grid):
        want = om.static_fields(g.rows, g.cols, g.north_lat, g.lat_step, g.lon_step) if hasattr(
            om, "static_fields") else None
        from oracle.grid import static_fields as osf
        want = osf(g.rows, g.cols, g.north_lat, g.lat_step, g.lon_step)
        np.testing.assert_array_equal(static_fields(g), want)


def test_conv_weight_layouts_reproduce_reference_convs():
    """The implicit-GEMM weight/tap arrangement, applied with numpy, equals the oracle convolutions."""
    from paper_2503_22235_b200 import pyramid as P
    rng = np.random.default_rng(3)
    cin, cout, h, w = 5, 7, 6, 8
    x = rng.standard_normal((cin, h, w))
    xp = np.zeros((cin, h + 2, w + 2))
    xp[:, 1:-1, 1:-1] = x
    xp[:, 1:-1, 0], xp[:, 1:-1, -1] = x[:, :, -1], x[:, :, 0]
    w3 = rng.standard_normal((cout, cin, 3, 3))
    b3 = rng.standard_normal(cout)
    for stride in (1, 2):
        ho, wo = (h - 1) // stride + 1, w // stride
        y = np.zeros((cout, ho, wo)) + b3[:, None, None]
        for kh in range(3):
            for kw in range(3):
                tap = xp[:, kh:kh + stride * (ho - 1) + 1:stride, kw:kw + stride * (wo - 1) + 1:stride]
                y += np.einsum("oc,chw->ohw", w3[:, :, kh, kw], tap)
        np.testing.assert_allclose(y, om.conv3x3(x, w3, b3, stride), atol=1e-12)
    # transposed conv as four parity classes of 2x2 taps (csrc/conv.cu)
    wt = rng.standard_normal((cin, cout, 4, 4))
    bt = rng.standard_normal(cout)
    y = np.zeros((cout, 2 * h, 2 * w))
    for a in range(2):
        for bb in range(2):
            acc = np.zeros((cout, h, w)) + bt[:, None, None]
            for tr in range(2):
                for tc in range(2):
                    tap = xp[:, a + tr:a + tr + h, bb + tc:bb + tc + w]
                    acc += np.einsum("co,chw->ohw", wt[:, :, 3 - a - 2 * tr, 3 - bb - 2 * tc], tap)
            y[:, a::2, bb::2] = acc
    np.testing.assert_allclose(y, om.conv_transpose4x4s2(x, wt, bt, (2 * h, 2 * w)), atol=1e-12)
    assert P.conv_bn(17) == 64 and P.conv_bn(100) == 128 and P.conv_bn(192) == 192 and P.conv_bn(1024) == 256


# ------------------------------------------------------------------------------------------------
# C ABI: the library loads (no GPU needed) and exports every symbol include/wm3.h declares
# ------------------------------------------------------------------------------------------------
def test_library_exports_declared_symbols():
    from paper_2503_22235_b200 import _lib
    header = open(os.path.join(ROOT, "include", "wm3.h")).read()
    declared = set(re.findall(r"\b(wm3_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.exported_symbols())
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    lib.wm3_version.restype = ctypes.c_int
    assert lib.wm3_version() >= 1


def test_library_reports_errors_without_launching():
    from paper_2503_22235_b200 import _lib
    lib = _lib.load_library()
    assert lib.wm3_neighbor_table(2, 5, 8, 3, 3, 3, 0, 5, None, None) != 0
    assert b"exceeds" in lib.wm3_last_error()
    assert lib.wm3_natten_fwd(None, 768, None, 256, 1, 3, 5, 8, 5, 0, 0, 0, 2, 96, 3, 3, 3, 0.1, None) != 0
    assert b"dhp" in lib.wm3_last_error()


def test_product_path_refuses_to_run_without_gpu():
    """No CPU fallback: with no CUDA device the device entry points raise instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_22235_b200 import _lib
    with pytest.raises(RuntimeError):
        _lib.lib()


def test_block_flops_formula():
    assert math.isclose(om.block_flops(81000, 1024, 245), 2.119716864e12)


def test_operand_dtype_export_matches_host_layer():
    """The header's operand-type query: the host layer's ELEM must be the library's build type."""
    import torch
    from paper_2503_22235_b200 import _lib
    lib = _lib.load_library()  # refuses a mismatched build
    assert lib.wm3_operand_dtype() == {torch.float16: 1, torch.bfloat16: 2}[_lib.ELEM]


# ------------------------------------------------------------------------------------------------
# latent validation before any launch (a mismatched latent must not reach the kernels)
# ------------------------------------------------------------------------------------------------
def _lat(tokens, extents, vt=0):
    from paper_2503_22235_b200.model import LatentState
    from paper_2503_22235_b200.tensor import Tensor
    return LatentState(Tensor(tokens), vt, extents)


@pytest.mark.parametrize("shape,extents", [((150, 64), (3, 5, 10)), ((149, 48), (3, 5, 10)),
                                           ((150, 48), (3, 10, 5)), ((300, 48), (3, 10, 10))])
def test_mismatched_latent_rejected_before_launch(shape, extents):
    """process / rollout / decode / rollout_ensemble / rollout_banded raise ConfigError (attention.py:150-151
    style) for a latent whose token count, width or extents differ from the config's, before touching the
    device (this runs with no GPU: reaching a launch would raise RuntimeError instead)."""
    import paper_2503_22235_b200.model as M
    import paper_2503_22235_b200.rollout as R
    from paper_2503_22235_b200.bands import rollout_banded
    cfg = M.desk_config()
    assert cfg.latent_extents == (3, 5, 10) and cfg.hidden == 48
    params = {f"proc{h}.blk0.ln1.gain": None for h in cfg.horizons}
    lat = _lat(np.zeros(shape), extents)
    with pytest.raises(ConfigError):
        M.process(lat, params, cfg, 6)
    with pytest.raises(ConfigError):
        R.rollout(lat, (6, 1), params, cfg)
    with pytest.raises(ConfigError):
        M.decode(lat, params, cfg)
    with pytest.raises(ConfigError):
        R.rollout_ensemble([lat], (6,), params, cfg)
    with pytest.raises(ConfigError):
        rollout_banded(lat, (6,), params, cfg, world=1)
    assert R.rollout(lat, (), params, cfg) is lat  # empty plan: the same object, no validation (rollout.py:66-67)


def test_process_inplace_rejects_bad_buffer():
    import torch
    import paper_2503_22235_b200.model as M
    cfg = M.desk_config()
    for x in (torch.zeros(cfg.tokens, cfg.hidden), torch.zeros(cfg.tokens, cfg.hidden, dtype=torch.float64),
              np.zeros((cfg.tokens, cfg.hidden))):
        with pytest.raises(ConfigError):
            M.process_inplace(x, {}, cfg, 6)


def test_content_tag_sees_in_place_updates():
    """The device weight caches key on tensor.content_tag: the reference's in-place optimizer step
    (training.py:144) and np.copyto reloads change it; reads do not."""
    import torch
    from paper_2503_22235_b200.tensor import Tensor, content_tag
    rng = np.random.default_rng(0)
    for shape in ((7,), (1024, 4096), (3, 1000, 7)):
        p = Tensor(rng.standard_normal(shape))
        t0 = content_tag(p)
        assert content_tag(p) == t0
        p.values -= 1e-3 * rng.standard_normal(shape)  # in place: same array object
        t1 = content_tag(p)
        assert t1 != t0 and t1[0] == t0[0]
        np.copyto(p.values, rng.standard_normal(shape))
        assert content_tag(p) != t1
    t = torch.zeros(10)
    a = content_tag(t)
    t.add_(1.0)
    assert content_tag(t) != a
