"""Stage the reference's own tests for the adapter run (build container only).

    python tests/ref_suite/fetch_suite.py

Copies /root/reference/pkg/tests into baseline/_ref_tests (git-ignored like
baseline/_ref, but shipped to the GPU box with the working tree) and installs
the unmodified reference package into baseline/_ref if it is missing.  The
copied files are the reference's, unmodified; nothing of them is committed.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SRC = "/root/reference/pkg"
DST_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")
DST_PKG = os.path.join(ROOT, "baseline", "_ref")


def main() -> int:
    if not os.path.isdir(SRC):
        print("no /root/reference here; nothing to stage")
        return 0
    if not os.path.isdir(os.path.join(DST_PKG, "qdot")):
        with tempfile.TemporaryDirectory() as tmp:
            pkg = os.path.join(tmp, "pkg")
            shutil.copytree(SRC, pkg, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
            subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                            "--find-links", "/opt/wheelhouse", "--target", DST_PKG, pkg], check=True)
    if os.path.isdir(DST_TESTS):
        shutil.rmtree(DST_TESTS)
    shutil.copytree(os.path.join(SRC, "tests"), DST_TESTS, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    print(f"staged {DST_TESTS} and {DST_PKG}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
