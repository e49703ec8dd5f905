"""`forecast` CLI on the B200 path vs the reference CLI's own outputs (tests/golden/cli, reference-generated).

Tolerance as the model tests: per-variable relative L2 <= 1e-2 after a 13 h (6, 6, 1) forecast
and a 2-source blended 7 h forecast; --offload bitwise equal to the plain run (reference test_cli.py:128-139).
"""

import json
import os

import numpy as np
import pytest

from paper_2503_22235_b200.cli import main
from paper_2503_22235_b200.serialization import load_params_file

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
BASE = ["forecast", "--config", os.path.join(GOLD, "tiny.cfg"), "--params", os.path.join(GOLD, "params.lmtw"),
        "--init", os.path.join(GOLD, "data.wmd3")]


def _per_var_rel(got, ref):
    out = {}
    for i in range(ref["surface"].shape[0]):
        out[f"sfc{i}"] = np.linalg.norm(got["surface"][i] - ref["surface"][i]) / np.linalg.norm(ref["surface"][i])
    for a in range(ref["atmos"].shape[0]):
        for lev in range(ref["atmos"].shape[1]):
            r = ref["atmos"][a, lev]
            out[f"atm{a}.lev{lev}"] = np.linalg.norm(got["atmos"][a, lev] - r) / np.linalg.norm(r)
    return out


@pytest.mark.parametrize("extra,ref_name", [
    (["--init-hour", "0", "--dt", "13"], "fc_primary.lmtw"),
    (["--init-hour", "4", "--dt", "7", "--source", "primary", "--source", "op1"], "fc_blend.lmtw"),
])
def test_forecast_matches_reference_cli(tmp_path, extra, ref_name):
    out = tmp_path / "fc.lmtw"
    assert main(BASE + extra + ["--out", str(out)]) == 0
    got, ref = load_params_file(out), load_params_file(os.path.join(GOLD, ref_name))
    assert set(got) == {"surface", "atmos", "valid_time"}
    assert got["surface"].shape == ref["surface"].shape and got["atmos"].shape == ref["atmos"].shape
    assert float(got["valid_time"]) == float(ref["valid_time"])
    rel = _per_var_rel(got, ref)
    worst = max(rel, key=rel.get)
    assert rel[worst] < 1e-2, (worst, rel[worst])
    man = json.loads(open(str(out) + ".manifest.json").read())
    assert man["outputs"] == [str(out)] and man["config"]["rows"] == 24 and man["seed"] is None


def test_offload_flag_matches_plain_bitwise(tmp_path):
    a, b = tmp_path / "a.lmtw", tmp_path / "b.lmtw"
    args = BASE + ["--init-hour", "0", "--dt", "13"]
    assert main(args + ["--out", str(a)]) == 0
    assert main(args + ["--out", str(b), "--offload"]) == 0
    assert a.read_bytes() == b.read_bytes()


def test_out_dir_env(tmp_path, monkeypatch):
    monkeypatch.setenv("GRIDCAST_OUT_DIR", str(tmp_path))
    assert main(BASE + ["--dt", "1", "--out", "rel/fc.lmtw"]) == 0
    assert (tmp_path / "rel" / "fc.lmtw").exists()


def test_evaluate_and_scorecard_match_reference(tmp_path):
    ev = tmp_path / "eval.json"
    assert main(["evaluate", "--forecast", os.path.join(GOLD, "fc_primary.lmtw"), "--truth",
                 os.path.join(GOLD, "data.wmd3"), "--wavelength-km", "12000", "--out", str(ev)]) == 0
    got = json.loads(ev.read_text())
    ref = json.loads(open(os.path.join(GOLD, "eval_primary.json")).read())
    assert got["valid_time"] == ref["valid_time"] == 13 and len(got["rmse"]) == 3 + 8
    for k in ref["rmse"]:
        assert abs(got["rmse"][k] - ref["rmse"][k]) <= 1e-10 * ref["rmse"][k], k
        if ref["blur"][k] is None:
            assert got["blur"][k] is None
        else:
            assert abs(got["blur"][k] - ref["blur"][k]) <= 1e-8 * ref["blur"][k], k
    sc = tmp_path / "sc.json"
    assert main(["scorecard", "--a", str(ev), "--b", os.path.join(GOLD, "eval_primary.json"), "--out", str(sc)]) == 0
    pct = json.loads(sc.read_text())["percent_vs_baseline"]
    assert all(abs(v) < 1e-6 for v in pct.values())
