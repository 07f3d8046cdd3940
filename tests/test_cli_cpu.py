"""CLI host-side pieces (no GPU): literal / scan / config parsing, the vector
file format, and the transcripts of the reference's CLI that end before any
device work (argument and configuration errors, exit code 2)."""

import math
import os

import numpy as np
import pytest

import cli_util as C
from paper_2105_00115_b200 import cli


def test_parse_epsilon_and_scan():
    assert cli.parse_epsilon("2^-34") == 2.0 ** -34 and cli.parse_epsilon(" 1e-8 ") == 1e-8
    grid = cli.parse_epsilon_scan("1e-12:1e-4:x100")
    assert len(grid) == 5 and grid[0] == 1e-12 and grid[1] == 1e-12 * 100.0
    assert cli.parse_epsilon_scan("2^-40:2^-10:x1024") == [2.0 ** -40, 2.0 ** -30, 2.0 ** -20, 2.0 ** -10]
    for bad in ("1:0.1:x10", "1e-3:1e-1", "1e-3:1e-1:10", "0:1:x10", "1e-3:1:x1"):
        with pytest.raises(ValueError):
            cli.parse_epsilon_scan(bad)


def test_parse_config():
    cfg = cli.parse_config("# c\nepsilon = 1e-5\nsplit=per-bin   # t\n\nstrategy=ranged:2\n")
    assert cfg == {"epsilon": "1e-5", "split": "per-bin", "strategy": "ranged:2"}
    assert cli.serialize_config(cfg) == "epsilon=1e-5\nsplit=per-bin\nstrategy=ranged:2\n"
    with pytest.raises(ValueError):
        cli.parse_config("epsilon 1e-5\n")


def test_vector_roundtrip(tmp_path):
    v = np.array([1.5, -0.0, 5e-324, math.pi, 1e308])
    p = str(tmp_path / "v.bin")
    cli.write_vector_binary(p, v)
    assert os.path.getsize(p) == 8 + 8 * v.size
    assert cli.read_vector(p).tobytes() == v.tobytes()
    t = tmp_path / "v.txt"
    t.write_text("1.5\n-2 3e-3   4\n")
    assert cli.read_vector(str(t)).tolist() == [1.5, -2.0, 3e-3, 4.0]


def test_golden_vector_files_parse():
    a = cli.read_vector(os.path.join(C.CLI_DIR, "a.bin"))
    assert a.shape == (3000,) and a.dtype == np.float64


HOST_ONLY = [r for r in C.runs() if r["code"] == 2 and any(
    k in r["stderr"] for k in ("length mismatch", "config", "bad scan spec"))]


@pytest.mark.parametrize("run", HOST_ONLY, ids=lambda r: " ".join(r["argv"]))
def test_reference_error_transcripts(run):
    code, out, err = C.run(run["argv"])
    assert (code, out, err) == (run["code"], run["stdout"], run["stderr"])
