"""Golden CLI transcripts BY RUNNING THE REFERENCE's cli.main.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Writes small vector files under tests/golden/cli/ and, per command line, the
reference's stdout, stderr and exit code to cli_golden.json.  Paths in argv
are relative to tests/golden/cli/ (the test chdirs there)."""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
CLI = os.path.join(HERE, "cli")

from qdot import cli  # noqa: E402

COMMANDS = [
    ["dot", "--x", "a.bin", "--y", "b.bin"],
    ["dot", "--x", "a.bin", "--y", "b.bin", "--epsilon", "1e-6", "--split", "per-bin", "--strategy", "ranged:3",
     "--with-reference"],
    ["dot", "--x", "a.bin", "--y", "b.bin", "--strategy", "split:4", "--epsilon", "1e-3", "--with-reference"],
    ["dot", "--x", "t1.txt", "--y", "t2.txt", "--with-reference"],
    ["dot", "--x", "a.bin", "--y", "a.bin", "--epsilon", "1e-10", "--with-reference"],
    ["dot", "--x", "a.bin", "--y", "short.bin"],
    ["dot", "--x", "a.bin", "--y", "b.bin", "--config", "dot.cfg"],
    ["dot", "--x", "a.bin", "--y", "b.bin", "--config", "dot.cfg", "--epsilon", "2^-20"],
    ["dot", "--x", "a.bin", "--y", "b.bin", "--config", "bad.cfg"],
    ["dot", "--x", "a.bin", "--y", "b.bin", "--config", "missing.cfg"],
    ["dot", "--x", "inf.txt", "--y", "t2.txt"],
    ["dot", "--x", "toy_x.txt", "--y", "toy_y.txt", "--with-reference"],
    ["dot", "--x", "wide_x.bin", "--y", "wide_y.bin", "--epsilon", "1e-12", "--with-reference"],
    ["verify", "--family", "B", "--t", "13", "--n", "1e3", "--trials", "4"],
    ["verify", "--family", "A", "--t", "20,40", "--n", "500", "--trials", "3", "--norm-mode", "false",
     "--epsilon", "1e-4"],
    ["verify", "--family", "B", "--t", "5", "--n", "300", "--trials", "2", "--split", "none", "--strategy",
     "split:2"],
    ["bench", "--family", "B", "--t", "5,9", "--n", "2000", "--trials", "2", "--epsilons", "1e-12:1e-4:x100"],
    ["bench", "--family", "A", "--t", "30", "--n", "700,1500", "--trials", "1", "--epsilons", "2^-40:2^-10:x1024",
     "--threads", "3"],
    ["bench", "--epsilons", "1:0.1:x10"],
    ["cg", "--nx", "10", "--ny", "10", "--nz", "1", "--epsilon", "1e-6"],
    ["cg", "--nx", "8", "--ny", "8", "--nz", "2", "--epsilon-scan", "1e-10:1e-2:x1000"],
    ["power", "--n", "200", "--edge-prob", "0.05"],
    ["power", "--n", "300", "--edge-prob", "0.03", "--epsilon", "1e-4", "--split", "none", "--seed", "4"],
]


def write_inputs():
    os.makedirs(CLI, exist_ok=True)
    rng = np.random.default_rng(11)
    cli.write_vector_binary(os.path.join(CLI, "a.bin"), rng.standard_normal(3000))
    cli.write_vector_binary(os.path.join(CLI, "b.bin"), rng.standard_normal(3000))
    cli.write_vector_binary(os.path.join(CLI, "short.bin"), rng.standard_normal(10))
    cli.write_vector_binary(os.path.join(CLI, "wide_x.bin"), np.ldexp(rng.normal(size=5000), rng.integers(-300, 300, 5000)))
    cli.write_vector_binary(os.path.join(CLI, "wide_y.bin"), np.ldexp(rng.normal(size=5000), rng.integers(-300, 300, 5000)))
    with open(os.path.join(CLI, "t1.txt"), "w") as f:
        f.write(" ".join(repr(float(v)) for v in rng.standard_normal(57)) + "\n")
    with open(os.path.join(CLI, "t2.txt"), "w") as f:
        f.write("\n".join(repr(float(v)) for v in rng.standard_normal(57)) + "\n")
    with open(os.path.join(CLI, "inf.txt"), "w") as f:
        f.write(" ".join(["1.0"] * 56 + ["inf"]) + "\n")
    with open(os.path.join(CLI, "toy_x.txt"), "w") as f:
        f.write(" ".join(repr(v) for v in [2.0**27, 2.0**8, 2.0**-3, 2.0**20]) + "\n")
    with open(os.path.join(CLI, "toy_y.txt"), "w") as f:
        f.write(" ".join(repr(v) for v in [2.0**23, 2.0**-14, 2.0**7, 2.0**-3]) + "\n")
    with open(os.path.join(CLI, "dot.cfg"), "w") as f:
        f.write("# dot settings\nepsilon = 1e-5\nsplit=per-bin   # trailing comment\n\nstrategy=ranged:2\n")
    with open(os.path.join(CLI, "bad.cfg"), "w") as f:
        f.write("epsilon 1e-5\n")


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return {"argv": argv, "code": code, "stdout": out.getvalue(), "stderr": err.getvalue()}


def main():
    write_inputs()
    cwd = os.getcwd()
    os.chdir(CLI)
    try:
        runs = [run(a) for a in COMMANDS]
    finally:
        os.chdir(cwd)
    for r in runs:
        print(r["code"], " ".join(r["argv"]), len(r["stdout"]))
    with open(os.path.join(HERE, "cli_golden.json"), "w") as f:
        json.dump({"reference": "qdot 0.1.0 cli.main", "runs": runs}, f, indent=0)


if __name__ == "__main__":
    main()
