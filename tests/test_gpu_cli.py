"""The package CLI reproduces the reference CLI's transcripts byte for byte
(stdout, stderr, exit code): dot / verify / bench / cg / power, recorded by
running the reference (tests/golden/make_cli_golden.py)."""

import pytest

import cli_util as C

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.mark.parametrize("run", C.runs(), ids=lambda r: " ".join(r["argv"]))
def test_cli_transcript(run):
    code, out, err = C.run(run["argv"])
    assert out == run["stdout"]
    assert err == run["stderr"]
    assert code == run["code"]
