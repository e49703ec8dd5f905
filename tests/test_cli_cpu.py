"""CLI contract checks that fail before any device work (reference test_cli.py)."""

import os

import pytest

from paper_2503_22235_b200.cli import main

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
BASE = ["forecast", "--config", os.path.join(GOLD, "tiny.cfg"), "--params", os.path.join(GOLD, "params.lmtw"),
        "--init", os.path.join(GOLD, "data.wmd3")]


def test_usage_error_is_exit_2(capsys):
    assert main(["forecast", "--bogus"]) == 2
    assert main([]) == 2


def test_version_flag(capsys):
    assert main(["--version"]) == 0
    assert "paper_2503_22235_b200" in capsys.readouterr().out


def test_dt_beyond_cap_is_config_error(tmp_path, capsys):
    assert main(BASE + ["--dt", "999", "--out", str(tmp_path / "x.lmtw")]) == 1
    assert capsys.readouterr().err.startswith("error: config: ")
    assert not (tmp_path / "x.lmtw").exists()


def test_unknown_source_is_config_error(tmp_path, capsys):
    assert main(BASE + ["--dt", "6", "--source", "op9", "--out", str(tmp_path / "x.lmtw")]) == 1
    assert capsys.readouterr().err.startswith("error: config: ")


def test_source_without_stream_is_config_error(tmp_path, capsys):
    # op1 has an encoder but a single-stream dataset would not carry it: here the dataset has 2 streams, so
    # ask for an init hour that does not exist instead -> data error
    assert main(BASE + ["--dt", "6", "--init-hour", "99", "--out", str(tmp_path / "x.lmtw")]) == 1
    assert capsys.readouterr().err.startswith("error: data: ")


def test_missing_file_is_io_error(tmp_path, capsys):
    args = ["forecast", "--config", str(tmp_path / "nope.cfg"), "--params", "p", "--init", "d", "--dt", "6",
            "--out", str(tmp_path / "x")]
    assert main(args) == 1
    assert capsys.readouterr().err.startswith("error: io: ")


def test_corrupt_params_is_data_error(tmp_path, capsys):
    bad = tmp_path / "bad.lmtw"
    bad.write_bytes(open(os.path.join(GOLD, "params.lmtw"), "rb").read()[:-8])
    args = list(BASE)
    args[args.index("--params") + 1] = str(bad)
    assert main(args + ["--dt", "6", "--out", str(tmp_path / "x.lmtw")]) == 1
    assert capsys.readouterr().err.startswith("error: data: ")
