"""Command line front end for the B200 forecast path (gridcast/cli.py), subcommand `forecast` (cli.py:162-224).

    python -m paper_2503_22235_b200.cli forecast --config C --params P.lmtw --init D.wmd3 --dt H --out F.lmtw
        [--init-hour N] [--source NAME ...] [--offload] [--budget-bytes B] [--lookahead K]

Same contract as the reference: LMTW parameters and output, WMD3 input dataset, multi-source forecasts blended
with softmax(blend.logits) over the chosen sources (model.py:424-449), a manifest JSON next to the artifact,
GRIDCAST_OUT_DIR prepended to relative output paths, exit code 0 / 1 (one line "error: <category>: message" on
stderr, category io | config | data | compute) / 2 (usage).  `--offload` selects the reference's activation
offload engine for the latent chain; the inference forward keeps no activations, so it is accepted and the
output is bitwise identical (the reference's own test_cli.py:128-139 property).  Validation (sources, dt cap)
runs before any device work.  `evaluate` (cli.py:235-276) scores a forecast file against the truth planes of a
WMD3 dataset with the device metrics (evaluation.py: every plane's RMSE and blur in one launch each) and
`scorecard` (cli.py:279-300) compares two evaluation reports.  The other reference subcommands (gen-data,
train, bench-offload, verify) are not part of the forecast path and are not provided.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

from . import __version__
from .config import load_config
from .dataset import load_dataset_file
from .errors import ConfigError, DataError
from .serialization import ContainerError, load_params_file, save_params_file

OUT_DIR_ENV = "GRIDCAST_OUT_DIR"


def _resolve_out(path: str) -> str:
    base = os.environ.get(OUT_DIR_ENV)
    return os.path.join(base, path) if base and not os.path.isabs(path) else path


def _versions() -> dict:
    import torch
    out = {"paper_2503_22235_b200": __version__, "numpy": np.__version__, "python": platform.python_version(),
           "torch": torch.__version__}
    if torch.cuda.is_available():
        out["device"] = torch.cuda.get_device_name(0)
    return out


def _manifest_config(cfg) -> dict:
    g = cfg.grid
    return {"rows": g.rows, "cols": g.cols, "north_lat": g.north_lat, "lat_step": g.lat_step,
            "lon_step": g.lon_step, "surface_in": cfg.surface_in, "surface_out": cfg.surface_out,
            "atmos_vars": cfg.atmos_vars, "levels": cfg.levels, "level_patch": cfg.level_patch,
            "stem_channels": cfg.stem_channels, "stage_channels": list(cfg.stage_channels), "hidden": cfg.hidden,
            "heads": cfg.heads, "window": list(cfg.window), "enc_blocks": cfg.enc_blocks,
            "dec_blocks": cfg.dec_blocks, "proc_blocks": cfg.proc_blocks, "horizons": list(cfg.horizons),
            "max_dt": cfg.max_dt}


def write_manifest(target, command, config: dict, seed, outputs, wall_time_s) -> str:
    """Run record next to an artifact (cli.py:72-86): `<target>.manifest.json` or `<dir>/manifest.json`."""
    path = os.path.join(target, "manifest.json") if os.path.isdir(target) else str(target) + ".manifest.json"
    doc = {"command": list(command), "config": config, "seed": seed, "versions": _versions(),
           "outputs": [str(p) for p in outputs], "wall_time_s": round(float(wall_time_s), 6)}
    with open(path, "w") as f:
        json.dump(doc, f, indent=2, sort_keys=True)
        f.write("\n")
    return path


def _stream_index(name: str, n_streams: int) -> int:
    """Dataset stream 0 feeds the primary encoder, stream j the encoder "op<j>" (cli.py:177-185)."""
    if name == "primary":
        return 0
    j = int(name[2:]) if name.startswith("op") and name[2:].isdigit() else -1
    if not 1 <= j < n_streams:
        raise ConfigError(f"source {name!r} has no dataset stream (dataset carries {n_streams})")
    return j


def _cmd_forecast(args, argv) -> int:
    from .model import available_sources, blend_latents, decode, encode
    from .rollout import greedy_plan, rollout

    t0 = time.time()
    cfg = load_config(args.config)
    params = load_params_file(args.params)
    ds = load_dataset_file(args.init)
    init_hour = args.init_hour if args.init_hour is not None else int(ds.times[-1])
    idx = ds.index_at(init_hour)
    sources = args.source or ["primary"]
    known = available_sources(params)
    for s in sources:
        if s not in known:
            raise ConfigError(f"no encoder for source {s!r}; have {known}")
    streams = [_stream_index(s, ds.n_sources) for s in sources]
    weights = None
    if len(sources) > 1:
        if "blend.logits" not in params:
            raise ConfigError("multi-source forecast needs blend.logits in params")
        logits = np.asarray(params["blend.logits"], dtype=np.float64)
        if logits.shape != (len(known),):
            raise ConfigError(f"blend.logits covers {logits.shape[0]} sources, model has {len(known)}")
        w = np.exp(logits[[known.index(s) for s in sources]])
        weights = w / w.sum()
    plan = greedy_plan(args.dt, cfg.max_dt)  # dt validated before any device work

    lats = [encode(ds.input_state_device(idx, j), params, cfg, source=s) for s, j in zip(sources, streams)]
    lat = lats[0] if weights is None else blend_latents(lats, weights)
    lat = rollout(lat, plan, params, cfg)  # --offload: no activations to offload in the forward; same result
    dec = decode(lat, params, cfg)

    out = _resolve_out(args.out)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    save_params_file(out, {"surface": dec.surface.values, "atmos": dec.atmos.values,
                           "valid_time": np.float64(dec.valid_time)})
    write_manifest(out, argv, _manifest_config(cfg), None, [out], time.time() - t0)
    print(f"forecast +{args.dt} h from hour {init_hour} ({len(plan)} latent steps) -> {out}")
    return 0


def _load_forecast_fields(path):
    blobs = load_params_file(path)
    for key in ("surface", "atmos", "valid_time"):
        if key not in blobs:
            raise DataError(f"forecast file lacks {key!r}")
    return blobs["surface"], blobs["atmos"], int(blobs["valid_time"])


def _cmd_evaluate(args, argv) -> int:
    from .evaluation import plane_scores

    t0 = time.time()
    sfc, atm, valid_time = _load_forecast_fields(args.forecast)
    ds = load_dataset_file(args.truth)
    true_sfc, true_atm = ds.truth_fields(ds.index_at(valid_time))
    if sfc.shape != true_sfc.shape or atm.shape != true_atm.shape:
        raise DataError(f"forecast shapes {sfc.shape}/{atm.shape} do not match truth "
                        f"{true_sfc.shape}/{true_atm.shape}")
    names = [f"sfc{i}" for i in range(sfc.shape[0])]
    names += [f"atm{a}.lev{lev}" for a in range(atm.shape[0]) for lev in range(atm.shape[1])]
    h, w = ds.grid.rows, ds.grid.cols
    pred = np.concatenate([sfc, atm.reshape(-1, h, w)])
    true = np.concatenate([true_sfc, true_atm.reshape(-1, h, w)])
    rmse_v, blur_v = plane_scores(pred, true, ds.grid, args.wavelength_km)
    doc = {"valid_time": valid_time, "wavelength_km": args.wavelength_km, "rmse": dict(zip(names, rmse_v)),
           "blur": dict(zip(names, blur_v))}
    out = _resolve_out(args.out)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with open(out, "w") as f:
        json.dump(doc, f, indent=2, sort_keys=True)
        f.write("\n")
    write_manifest(out, argv, {"wavelength_km": args.wavelength_km}, None, [out], time.time() - t0)
    print(f"evaluated {len(names)} planes at hour {valid_time}; mean rmse {float(np.mean(rmse_v)):.6f} -> {out}")
    return 0


def _cmd_scorecard(args, argv) -> int:
    from .evaluation import scorecard

    t0 = time.time()
    docs = []
    for name, path in (("a", args.a), ("b", args.b)):
        with open(path) as f:
            doc = json.load(f)
        if "rmse" not in doc:
            raise DataError(f"file {name} is not an evaluation report")
        docs.append(doc)
    pct = scorecard(docs[0]["rmse"], docs[1]["rmse"])
    width = max(len(k) for k in pct)
    for k in sorted(pct):
        print(f"{k:<{width}}  {docs[0]['rmse'][k]:12.6f}  {docs[1]['rmse'][k]:12.6f}  {pct[k]:+8.3f}%")
    if args.out:
        out = _resolve_out(args.out)
        os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
        with open(out, "w") as f:
            json.dump({"percent_vs_baseline": pct}, f, indent=2, sort_keys=True)
            f.write("\n")
        write_manifest(out, argv, {}, None, [out], time.time() - t0)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2503_22235_b200", description=__doc__.split("\n\n")[0])
    p.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = p.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("forecast", help="roll a forecast from a dataset state")
    f.add_argument("--config", required=True)
    f.add_argument("--params", required=True)
    f.add_argument("--init", required=True, help="WMD3 dataset file")
    f.add_argument("--init-hour", type=int, default=None)
    f.add_argument("--dt", type=int, required=True)
    f.add_argument("--out", required=True)
    f.add_argument("--source", action="append", help="input source name; repeat to blend several")
    f.add_argument("--offload", action="store_true", help="accepted for compatibility; identical output")
    f.add_argument("--budget-bytes", type=int, default=1 << 28)
    f.add_argument("--lookahead", type=int, default=2)
    e = sub.add_parser("evaluate", help="score a forecast file against truth")
    e.add_argument("--forecast", required=True)
    e.add_argument("--truth", required=True, help="WMD3 dataset file")
    e.add_argument("--wavelength-km", type=float, default=2000.0)
    e.add_argument("--out", required=True)
    sc = sub.add_parser("scorecard", help="percent RMSE change of a versus b")
    sc.add_argument("--a", required=True, help="evaluation JSON")
    sc.add_argument("--b", required=True, help="baseline evaluation JSON")
    sc.add_argument("--out")
    return p


_HANDLERS = {"forecast": _cmd_forecast, "evaluate": _cmd_evaluate, "scorecard": _cmd_scorecard}


def _categorize(exc: BaseException) -> str:
    """Exception class -> error category (cli.py:456-463)."""
    if isinstance(exc, OSError):
        return "io"
    if isinstance(exc, ConfigError):
        return "config"
    if isinstance(exc, (DataError, ContainerError, json.JSONDecodeError)):
        return "data"
    return "compute"


def main(argv=None) -> int:
    argv = list(sys.argv[1:]) if argv is None else list(argv)
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:  # argparse: usage error (2) or --help / --version (0)
        return int(e.code or 0)
    try:
        return _HANDLERS[args.cmd](args, argv)
    except Exception as exc:  # one machine-parseable line, exit 1
        msg = str(exc).replace("\n", " ")
        print(f"error: {_categorize(exc)}: {msg}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
