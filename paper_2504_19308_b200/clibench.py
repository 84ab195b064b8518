"""The reference's own CLI (cli.py: multiply / sweep / bench) on the GPU path,
and its bench CSV extended with throughput and roofline columns.

``run(argv, reference_src)`` installs the ``apxmm`` shim (apxmm_shim.install: the hot-path modules
are this package's, cli / genmat / errest / baseline are loaded from the reference tree) and calls
``apxmm.cli.main(argv)`` unchanged, so ``run_method``'s svd / cd / sfft products run through the
C-ABI on the device. ``extend_bench_csv`` appends, per row of the reference's fixed-schema bench
CSV (cli.py:51, BENCH_HEADER):

    products_per_s      1 / wall_time_s (the row's own measured wall time)
    flops_model         the reference's operation_count(method, n, k) (cli.py:69-92)
    achieved_tflops     flops_model / wall_time_s / 1e12
    roofline_peak_tflops the measured FP64 FMA peak of this pool (the methods are fp64)
    roofline_frac       achieved_tflops / roofline_peak_tflops

    python -m paper_2504_19308_b200.clibench REF_SRC bench --config conf.txt --out out.csv [--gpu-columns]
"""

from __future__ import annotations

import csv
import sys

EXTRA = ["products_per_s", "flops_model", "achieved_tflops", "roofline_peak_tflops", "roofline_frac"]


def run(argv, reference_src: str, name: str = "apxmm") -> int:
    """apxmm.cli.main(argv) with the GPU hot path bound in (exit code of the reference CLI)."""
    from . import _native
    from .apxmm_shim import install

    _native.lib()  # fail loudly without the CUDA extension
    apx = install(reference_src, name=name)
    return apx.cli.main(list(argv))


def extend_bench_csv(path_in: str, path_out: str, peak_tflops: float, operation_count) -> int:
    """Copy the bench CSV adding EXTRA columns; returns the number of rows written."""
    with open(path_in, newline="", encoding="ascii") as fh:
        rows = list(csv.reader(fh))
    if not rows:
        raise ValueError(f"{path_in}: empty bench CSV")
    head = rows[0]
    col = {c: i for i, c in enumerate(head)}
    out = [head + EXTRA]
    for r in rows[1:]:
        wall = float(r[col["wall_time_s"]])
        method, n = r[col["method"]], int(r[col["n"]])
        kcell = r[col["k"]]
        k = int(kcell) if kcell not in ("-", "") else 0
        flops = operation_count(method, n, k=k, c=k)
        ach = flops / wall / 1e12 if wall > 0 else float("nan")
        out.append(r + [f"{1.0 / wall:.10g}" if wall > 0 else "inf", f"{flops:.10g}", f"{ach:.10g}",
                        f"{peak_tflops:.6g}", f"{ach / peak_tflops:.10g}"])
    with open(path_out, "w", newline="", encoding="ascii") as fh:
        csv.writer(fh).writerows(out)
    return len(out) - 1


def fp64_peak_tflops(default: float = 35.8) -> float:
    """Measured FP64 FMA peak (profiles/r*_pipe_peaks.jsonl), else `default` (the round-1 measurement)."""
    import glob
    import json
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    files = sorted(glob.glob(os.path.join(root, "profiles", "r[0-9][0-9]_pipe_peaks.jsonl")))
    best = 0.0
    for f in files[-1:]:
        for line in open(f):
            try:
                best = max(best, float(json.loads(line).get("fp64_dfma_tflops", 0.0)))
            except ValueError:
                pass
    return best or default


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv:
        raise SystemExit(__doc__)
    ref, rest = argv[0], argv[1:]
    extend = "--gpu-columns" in rest
    rest = [a for a in rest if a != "--gpu-columns"]
    rc = run(rest, ref)
    if rc == 0 and extend and rest and rest[0] == "bench":
        out = rest[rest.index("--out") + 1]
        apx = sys.modules["apxmm"]
        stem = out[:-4] if out.endswith(".csv") else out
        extend_bench_csv(out, stem + ".gpu.csv", fp64_peak_tflops(), apx.cli.operation_count)
    return rc


if __name__ == "__main__":
    sys.exit(main())
