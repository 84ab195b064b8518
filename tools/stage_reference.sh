#!/bin/bash
# Stage a copy of the reference package (sources + its own test suite) into the git-ignored
# baseline/_ref/pkg, so the conformance run (tools/conformance.py) can use it on the GPU box,
# where /root/reference does not exist. Nothing from it is committed or imported by the product.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf "$ROOT/baseline/_ref/pkg"
mkdir -p "$ROOT/baseline/_ref"
cp -r /root/reference/pkg "$ROOT/baseline/_ref/pkg"
find "$ROOT/baseline/_ref/pkg" -name __pycache__ -prune -exec rm -rf {} +
echo "staged $(find "$ROOT/baseline/_ref/pkg" -name '*.py' | wc -l) python files into baseline/_ref/pkg"
