"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's approximate-product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import this package, and only as the checker / the timed CPU
reference. The product package ``paper_2504_19308_b200`` never imports it: its path is CUDA-only
and fails loudly when the extension is missing.

Parity pinning: every function is checked against golden vectors produced by importing the
reference package itself (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``). The cycle
and mixed products have no reference function; their golden vectors are composed from the
reference's own primitives (``cycle_reorder``, ``apply_cycle_power``, ``top_indices``,
``randomized_partial_svd``) by the same script, so those two are pinned at the primitive level
only ("parity pinned via primitives").
"""

from .apx_oracle import *  # noqa: F401,F403
from .apx_oracle import __all__  # noqa: F401
