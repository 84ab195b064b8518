#!/bin/bash
# The checked build (APX_DCHECK device bounds checks; compute-sanitizer is closed on this pool)
# over every path at small n and the GPU parity suite minus the full-size configs.
cd "$(dirname "$0")/.."
export APX_LIB=$PWD/paper_2504_19308_b200/_apx_checked.so
test -f "$APX_LIB" || { echo "build it: APX_CHECKED=1 python -m paper_2504_19308_b200.build"; exit 1; }
python tools/sanitize_cases.py 2>&1
python -m pytest tests -m gpu -q -k "not c5 and not c4_full and not robust and not bigfft" 2>&1 | tail -5
