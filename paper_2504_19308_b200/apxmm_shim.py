"""Put the GPU path behind the reference's own CLI and tests: build a package named ``apxmm``
whose hot-path modules are this package's, and whose remaining modules (errest, genmat,
baseline, cli) are loaded from an existing reference tree at call time -- never copied here
(SURVEY.md §8(b) "Conformance wiring").

    from paper_2504_19308_b200.apxmm_shim import install
    apxmm = install("/path/to/reference/pkg/src")   # directory that contains apxmm/
    apxmm.cli.main(["multiply", "--method", "svd", ...])   # svd / cd / sfft now run on the B200

The reference binds product names at import time with relative imports (cli.py:26-47), so the
GPU modules must be in place before its modules execute; monkey-patching after import would
not reach them.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

from . import circulant, core, errest, fsparse, report, svd

# reference module -> ours (the hot path); everything else is loaded from the reference tree
GPU_MODULES = {"core": core, "svd": svd, "circulant": circulant, "fsparse": fsparse, "report": report}
REFERENCE_MODULES = ("errest", "genmat", "baseline", "cli")
# device implementations that replace single functions of a reference-loaded module (bound before
# the modules after it execute their imports)
GPU_FUNCTIONS = {"errest": {"sketch_norm_estimate": errest.sketch_norm_estimate}}


def install(reference_src: str, name: str = "apxmm") -> types.ModuleType:
    """Register ``name`` (default ``apxmm``) in sys.modules and return it."""
    src = os.path.join(reference_src, "apxmm")
    if not os.path.isfile(os.path.join(src, "cli.py")):
        raise FileNotFoundError(f"no reference apxmm package under {reference_src!r}")
    for key in [m for m in sys.modules if m == name or m.startswith(name + ".")]:
        del sys.modules[key]
    pkg = types.ModuleType(name, "apxmm with the B200 hot path (paper_2504_19308_b200)")
    pkg.__path__ = []  # submodules come only from the table below
    pkg.__package__ = name
    sys.modules[name] = pkg
    for sub, mod in GPU_MODULES.items():
        sys.modules[f"{name}.{sub}"] = mod
        setattr(pkg, sub, mod)
    for sub in REFERENCE_MODULES:
        spec = importlib.util.spec_from_file_location(f"{name}.{sub}", os.path.join(src, sub + ".py"))
        mod = importlib.util.module_from_spec(spec)
        mod.__package__ = name
        sys.modules[f"{name}.{sub}"] = mod
        spec.loader.exec_module(mod)
        for fname, fn in GPU_FUNCTIONS.get(sub, {}).items():
            setattr(mod, fname, fn)
        setattr(pkg, sub, mod)
    # the package-level names of the reference __init__ (its re-exports), resolved to the above
    init = os.path.join(src, "__init__.py")
    spec = importlib.util.spec_from_file_location(name, init, submodule_search_locations=[])
    code = compile(open(init).read(), init, "exec")
    exec(code, pkg.__dict__)
    return pkg
