"""The reference's own test suite (pkg/tests: 234 tests, acceptance criteria
1-12 at their stated trial counts) run UNMODIFIED on top of the B200 hot path:
tests/ref_suite/qdot_b200_adapter.py swaps the reference's kernel.qdot /
select_parameters / reference_dot for the B200 ones in every reference module
(its harness, solvers and CLI then call the device pipeline too).

The suite and the reference package are staged, unmodified and git-ignored,
into baseline/_ref_tests and baseline/_ref by tests/ref_suite/fetch_suite.py
(run by __graft_entry__.build() where /root/reference exists); they travel
to the GPU box with the working tree.  Without them this test skips.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref_tests")
REF = os.path.join(ROOT, "baseline", "_ref", "qdot")


@pytest.mark.skipif(not (os.path.isdir(SUITE) and os.path.isdir(REF)),
                    reason="reference suite not staged (tests/ref_suite/fetch_suite.py)")
def test_reference_suite_on_the_b200_path():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.path.join(ROOT, "tests", "ref_suite") + os.pathsep + env.get("PYTHONPATH", "")
    env.setdefault("QDOT_ACCEPT_TRIALS", "10000")
    env.setdefault("QDOT_ACCEPT_CELL_TRIALS", "1000")
    p = subprocess.run([sys.executable, "-m", "pytest", "-p", "qdot_b200_adapter", SUITE, "-q", "-rA",
                        "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=3000)
    out = p.stdout + p.stderr
    lines = [ln for ln in out.splitlines() if ln.startswith("ACCEPTANCE") or "qdot_b200_adapter" in ln
             or re.search(r"\d+ (passed|failed)", ln)]
    log = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log):
        with open(os.path.join(log, "ref_suite_b200.log"), "w") as f:
            f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    assert p.returncode == 0, out[-4000:]
    assert sum(ln.startswith("ACCEPTANCE") and ": PASS" in ln for ln in lines) == 12
    calls = re.search(r"entry-point calls \{'qdot': (\d+), 'select_parameters': (\d+), 'reference_dot': (\d+)\}", out)
    assert calls and min(int(c) for c in calls.groups()) > 0          # the B200 path really ran
