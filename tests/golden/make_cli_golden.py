"""Generate the CLI / container fixtures with the reference itself (run in the build container, where
/root/reference exists; the outputs are committed and travel to the GPU box, the reference does not).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Writes tests/golden/cli/:
    tiny.cfg            reference save_config(tiny_config())
    params.lmtw         reference init_model_params(tiny, seed=5, zero_residual=False) + an "op1" encoder
                        (training.add_source_encoders) and blend.logits = [0.4, -0.3]
    data.wmd3           reference CLI `gen-data --hours 18 --seed 3 --sources 2`
    fc_primary.lmtw     reference CLI `forecast --init-hour 0 --dt 13`
    fc_blend.lmtw       reference CLI `forecast --init-hour 4 --dt 7 --source primary --source op1`
    eval_primary.json   reference CLI `evaluate --forecast fc_primary.lmtw --truth data.wmd3 --wavelength-km 12000`
"""
import os
import sys

import numpy as np

from gridcast.cli import main
from gridcast.model import init_model_params, save_config, tiny_config
from gridcast.serialization import save_params_file
from gridcast.training import add_source_encoders

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")


def run():
    os.makedirs(HERE, exist_ok=True)
    cfg = tiny_config()
    spec = os.path.join(HERE, "tiny.cfg")
    save_config(spec, cfg)
    params = init_model_params(cfg, seed=5, zero_residual=False)
    add_source_encoders(params, cfg, ["op1"], seed=6)
    params["blend.logits"].values[:] = [0.4, -0.3]
    save_params_file(os.path.join(HERE, "params.lmtw"), {k: v.values for k, v in params.items()})
    data = os.path.join(HERE, "data.wmd3")
    assert main(["gen-data", "--spec", spec, "--hours", "18", "--seed", "3", "--sources", "2", "--out", data]) == 0
    base = ["forecast", "--config", spec, "--params", os.path.join(HERE, "params.lmtw"), "--init", data]
    assert main(base + ["--init-hour", "0", "--dt", "13", "--out", os.path.join(HERE, "fc_primary.lmtw")]) == 0
    assert main(base + ["--init-hour", "4", "--dt", "7", "--source", "primary", "--source", "op1",
                        "--out", os.path.join(HERE, "fc_blend.lmtw")]) == 0
    assert main(["evaluate", "--forecast", os.path.join(HERE, "fc_primary.lmtw"), "--truth", data,
                 "--wavelength-km", "12000", "--out", os.path.join(HERE, "eval_primary.json")]) == 0
    for f in os.listdir(HERE):  # manifests carry host paths and timings: not fixtures
        if f.endswith(".manifest.json"):
            os.remove(os.path.join(HERE, f))


if __name__ == "__main__":
    sys.exit(run())
