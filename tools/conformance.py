"""Conformance harness: run the reference's OWN test suite with its hot
path replaced by the B200 drop-in.

    tools/stage_reference.sh                    # once, in the build container
    python tools/conformance.py [PKG_DIR] [-- extra pytest args]

PKG_DIR (default baseline/_ref/pkg, a git-ignored copy that travels to the GPU box) holds the
reference's src/apxmm and tests/. ``apxmm_shim.install`` registers a package named ``apxmm``
whose core / svd / circulant / fsparse / report modules are this repo's (every product runs
through the C-ABI on the GPU) and whose errest / genmat / baseline / cli are the reference's,
loaded before pytest imports the test modules. The reference's acceptance tests print their
CRITERION lines (run with -s); the 4 deliberate acceptance failures are expected to fail with
the same numbers as the reference's own pkg/test_output.txt.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


class ShimPlugin:
    """pytest plugin: install the shim before collection imports the reference tests."""

    def __init__(self, src):
        self.src = src

    def pytest_configure(self, config):
        from paper_2504_19308_b200 import _native
        from paper_2504_19308_b200.apxmm_shim import install

        _native.lib()  # fail loudly without the CUDA extension
        apx = install(self.src)
        print(f"[conformance] apxmm -> {apx.svd.__name__}, {apx.circulant.__name__}, {apx.fsparse.__name__}, "
              f"{apx.core.__name__} (GPU); cli/genmat/errest/baseline from {self.src}")


def main(argv):
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    pkg = argv[0] if argv else os.path.join(ROOT, "baseline", "_ref", "pkg")
    src, tests = os.path.join(pkg, "src"), os.path.join(pkg, "tests")
    if not os.path.isdir(os.path.join(src, "apxmm")) or not os.path.isdir(tests):
        raise SystemExit(f"no reference package under {pkg!r} (run tools/stage_reference.sh)")
    import pytest

    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    args = [tests, "-q", "-s", "-rfE", "-p", "no:cacheprovider", "--rootdir", pkg, *extra]
    return pytest.main(args, plugins=[ShimPlugin(src)])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
