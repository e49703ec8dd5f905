"""On-disk formats: LMTW parameter container and WMD3 dataset container.

Mirrors the reference's test_serialization.py:18-64 and test_synthdata.py:98-144, and pins both readers to
files the reference itself wrote (tests/golden/cli/, made by tests/golden/make_cli_golden.py)."""

import os
import struct

import numpy as np
import pytest

from paper_2503_22235_b200.dataset import WeatherDataset, dump_dataset, load_dataset, load_dataset_file
from paper_2503_22235_b200.errors import DataError
from paper_2503_22235_b200.serialization import (ContainerError, dump_params, index_params, load_params,
                                                 load_params_file, save_params_file)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


# ---------------------------------------------------------------- LMTW
def test_lmtw_header_layout():
    buf = dump_params({})
    assert buf[:4] == b"LMTW" and struct.unpack_from("<II", buf, 4) == (1, 0) and len(buf) == 12


def test_lmtw_single_param_layout():
    arr = np.arange(6, dtype=np.float64).reshape(2, 3)
    buf = dump_params({"w": arr})
    assert struct.unpack_from("<I", buf, 12) == (1,) and buf[16:17] == b"w"
    assert struct.unpack_from("<I", buf, 17) == (2,) and struct.unpack_from("<2Q", buf, 21) == (2, 3)
    np.testing.assert_array_equal(np.frombuffer(buf, "<f8", 6, 37).reshape(2, 3), arr)


def test_lmtw_sorted_names_and_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    params = {"zz": rng.standard_normal((3, 4, 5)), "scalar": np.float64(2.5), "aa": rng.standard_normal(7),
              "empty": np.zeros((0, 2))}
    buf = dump_params(params)
    assert buf.index(b"aa") < buf.index(b"zz")
    p = tmp_path / "p.lmtw"
    save_params_file(p, params)
    back = load_params_file(p)
    for k, v in params.items():
        want = np.asarray(v, dtype=np.float64)
        assert back[k].shape == want.shape and back[k].tobytes() == want.tobytes()
        assert back[k].flags.writeable
    assert dump_params(back) == p.read_bytes()


@pytest.mark.parametrize("mutate", ["magic", "version", "truncate", "trailing", "short"])
def test_lmtw_rejects_malformed(mutate):
    buf = dump_params({"w": np.ones((2, 2))})
    bad = {"magic": b"XXXX" + buf[4:], "version": buf[:4] + struct.pack("<I", 2) + buf[8:],
           "truncate": buf[:-1], "trailing": buf + b"\0", "short": buf[:7]}[mutate]
    with pytest.raises(ContainerError):
        load_params(bad)


def test_lmtw_reference_written_file_round_trips_bitwise():
    raw = open(os.path.join(GOLD, "params.lmtw"), "rb").read()
    params = load_params(raw)
    assert "enc.stem_sfc.w" in params and "enc_op.op1.stem_sfc.w" in params
    np.testing.assert_array_equal(params["blend.logits"], [0.4, -0.3])
    assert dump_params(params) == raw
    assert [e[0] for e in index_params(raw)] == sorted(params)
    fc = load_params(open(os.path.join(GOLD, "fc_primary.lmtw"), "rb").read())
    assert fc["surface"].shape == (3, 24, 24) and fc["atmos"].shape == (2, 4, 24, 24)
    assert int(fc["valid_time"]) == 13 and fc["valid_time"].shape == ()


# ---------------------------------------------------------------- WMD3
def test_wmd3_reference_written_file():
    raw = open(os.path.join(GOLD, "data.wmd3"), "rb").read()
    ds = load_dataset(raw)
    assert (ds.grid.rows, ds.grid.cols, ds.grid.south_pole_omitted) == (24, 24, True)
    assert (ds.surface_in, ds.surface_out, ds.atmos_vars, ds.levels, ds.n_sources) == (2, 3, 2, 4, 2)
    assert ds.n_times == 19 and ds.times.dtype == np.int64 and list(ds.times[:3]) == [0, 1, 2]
    assert ds.truth.shape == (19, 11, 24, 24) and ds.sources[1].shape == (19, 10, 24, 24)
    assert dump_dataset(ds) == raw  # bitwise round trip of a reference-written container
    st = ds.input_state(ds.index_at(4), 1)
    assert st.valid_time == 4 and st.surface.shape == (2, 24, 24) and st.atmos.shape == (2, 4, 24, 24)
    assert st.surface.dtype == np.float64
    # time-major payload: the first source plane of time 4 sits right after the truth planes of time 4
    hw, row = 24 * 24, 11 + 2 * 10
    off = struct.calcsize("<4sI6dB6I") + 8 * 19 + 4 * (4 * row + 11) * hw
    np.testing.assert_array_equal(np.frombuffer(raw, "<f4", hw, off).reshape(24, 24), ds.sources[0][4, 0])
    sfc, atm = ds.truth_fields(0)
    assert sfc.shape == (3, 24, 24) and atm.shape == (2, 4, 24, 24)
    assert ds.plane_sigmas().shape == (11,) and (ds.plane_sigmas() > 0).all()
    with pytest.raises(DataError):
        ds.index_at(99)


@pytest.mark.parametrize("mutate", ["magic", "version", "truncate", "trailing", "header"])
def test_wmd3_rejects_malformed(mutate):
    raw = open(os.path.join(GOLD, "data.wmd3"), "rb").read()
    bad = {"magic": b"XXXX" + raw[4:], "version": raw[:4] + struct.pack("<I", 2) + raw[8:],
           "truncate": raw[:-5], "trailing": raw + b"\0\0", "header": raw[:40]}[mutate]
    with pytest.raises(DataError):
        load_dataset(bad)


def test_wmd3_validation_and_file_round_trip(tmp_path):
    ds = load_dataset_file(os.path.join(GOLD, "data.wmd3"))
    with pytest.raises(DataError):
        WeatherDataset(ds.grid, ds.surface_in, ds.surface_out, ds.atmos_vars, ds.levels, ds.times.astype(np.int32),
                       ds.truth, ds.sources)
    with pytest.raises(DataError):
        WeatherDataset(ds.grid, ds.surface_in, ds.surface_out, ds.atmos_vars, ds.levels, ds.times, ds.truth, ())
    from paper_2503_22235_b200.dataset import save_dataset_file
    p = tmp_path / "d.wmd3"
    save_dataset_file(ds, p)
    assert p.read_bytes() == open(os.path.join(GOLD, "data.wmd3"), "rb").read()
