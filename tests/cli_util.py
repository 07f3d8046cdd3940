"""Run the package CLI in-process like the golden transcripts were recorded."""

import contextlib
import functools
import io
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CLI_DIR = os.path.join(GOLDEN, "cli")


@functools.lru_cache(maxsize=1)
def runs():
    with open(os.path.join(GOLDEN, "cli_golden.json")) as f:
        return json.load(f)["runs"]


def run(argv):
    from paper_2105_00115_b200 import cli
    out, err = io.StringIO(), io.StringIO()
    cwd = os.getcwd()
    os.chdir(CLI_DIR)
    try:
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            code = cli.main(argv)
    finally:
        os.chdir(cwd)
    return code, out.getvalue(), err.getvalue()
