"""ADSK1 files and the command line (adasketch/problem.py:337-365, cli.py).
CPU tests cover the file format and flag handling; the GPU tests stream a
file into HBM and run the solve / compare commands end to end."""
import csv
import json
import struct

import numpy as np
import pytest

from paper_2104_14101_b200 import cli
from paper_2104_14101_b200.errors import IoFormatError
from paper_2104_14101_b200.io import load_matrix, read_header, save_matrix


def test_adsk1_layout_and_round_trip(tmp_path):
    M = np.arange(12.0).reshape(3, 4) - 5.5
    f = tmp_path / "M.adsk"
    save_matrix(f, M)
    raw = f.read_bytes()
    assert raw[:5] == b"ADSK1"
    assert struct.unpack("<QQ", raw[5:21]) == (3, 4)
    assert np.array_equal(np.frombuffer(raw[21:], dtype="<f8").reshape(3, 4), M)
    assert read_header(f) == (3, 4)
    assert np.array_equal(load_matrix(f), M)


def test_adsk1_errors(tmp_path):
    f = tmp_path / "bad.adsk"
    f.write_bytes(b"ADSK2" + struct.pack("<QQ", 1, 1) + b"\0" * 8)
    with pytest.raises(IoFormatError):
        load_matrix(f)
    g = tmp_path / "short.adsk"
    g.write_bytes(b"ADSK1" + struct.pack("<QQ", 2, 2) + b"\0" * 8)
    with pytest.raises(IoFormatError):
        load_matrix(g)


def test_cli_flag_errors_exit_2(tmp_path):
    assert cli.main(["solve", "--data", str(tmp_path), "--solver", "nope", "--out", "x.csv"]) == 2
    with pytest.raises(Exception):
        cli.resolve_options("cg", {"m": 5, "m_init": None, "rho": None, "sketch": None, "s": None})
    with pytest.raises(Exception):
        cli.resolve_options("pcg", {"m": None, "m_init": None, "rho": None, "sketch": None, "s": None})
    assert cli.resolve_options("ada-pcg", {"m": None, "m_init": None, "rho": None, "sketch": None, "s": None}) == \
        {"m": None, "m_init": 1, "rho": 0.125, "sketch": "gaussian", "s": 1}
    assert cli.parse_sketch_size("3d", 10) == 30
    assert cli.parse_run("ada-pcg:srht:m_init=16", 10) == \
        ("ada-pcg", {"m": None, "m_init": 16, "rho": 0.125, "sketch": "srht", "s": 1})
    assert cli.main(["solve", "--data", str(tmp_path), "--solver", "cg", "--nu", "-1", "--out", "x.csv"]) == 2


def test_cli_missing_data_exit_3(tmp_path):
    assert cli.main(["solve", "--data", str(tmp_path / "none"), "--solver", "cg", "--out",
                     str(tmp_path / "t.csv")]) == 3


@pytest.mark.gpu
def test_stream_to_device_and_narrow(tmp_path):
    import torch

    from paper_2104_14101_b200.io import load_matrix_device

    rng = np.random.default_rng(0)
    M = rng.standard_normal((1000, 37))
    f = tmp_path / "M.adsk"
    save_matrix(f, M)
    d64 = load_matrix_device(f, torch.float64, chunk_bytes=37 * 8 * 128)
    d32 = load_matrix_device(f, torch.float32, chunk_bytes=37 * 8 * 100)
    assert np.array_equal(d64.cpu().numpy(), M)
    assert np.array_equal(d32.cpu().numpy(), M.astype(np.float32))


@pytest.mark.gpu
def test_cli_gen_solve_compare(tmp_path):
    data = tmp_path / "cfg0"
    assert cli.main(["gen-config", "--config", "0", "--out", str(data)]) == 0
    out = tmp_path / "trace.csv"
    assert cli.main(["solve", "--data", str(data), "--solver", "ada-ihs", "--sketch", "gaussian",
                     "--m-init", "16", "--T", "10", "--seed", "1", "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == cli.TRACE_COLUMNS
    rel = float(rows[-1][5])
    assert rel <= 1e-9
    man = json.loads((tmp_path / "trace.csv.manifest.json").read_text())
    assert man["command"] == "solve" and "A.adsk" in man["input_digests"]
    out2 = tmp_path / "cmp.csv"
    assert cli.main(["compare", "--data", str(data), "--run", "ada-pcg:srht:m_init=16", "--run", "cg",
                     "--run", "direct", "--T", "8", "--out", str(out2)]) == 0
    rows = list(csv.reader(open(out2)))
    assert rows[0][0] == "solver" and {r[0] for r in rows[1:]} == {"ada-pcg:srht:m_init=16", "cg", "direct"}
    # numerical failures exit 4: a negative nu override is a flag error (2)
    assert cli.main(["solve", "--data", str(data), "--solver", "cg", "--nu", "-1", "--out", str(out)]) == 2
