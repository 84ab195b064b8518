"""run_method mirror (cli.py:138-158) and the apxmm conformance wiring."""
import os

import numpy as np
import pytest

import oracle as O

REF_SRC = "/root/reference/pkg/src"


def test_dispatch_errors_without_gpu():
    from paper_2504_19308_b200.dispatch import run_method
    A = np.eye(4)
    with pytest.raises(ValueError):
        run_method("bogus", 1, A, A)
    with pytest.raises(NotImplementedError):
        run_method("lowrank", 0, A, A, c=2)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present (GPU box)")
def test_apxmm_shim_binds_the_gpu_path():
    """The reference's cli module, loaded into the shim namespace, calls our product functions
    (bound at import through its relative imports)."""
    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200.apxmm_shim import install
    apxmm = install(REF_SRC, name="apxmm_gpu_test")
    try:
        assert apxmm.cli.svd_first_order_multiply is P.svd_first_order_multiply
        assert apxmm.cli.circulant_first_order_multiply is P.circulant_first_order_multiply
        assert apxmm.cli.fft_sparse_first_order_multiply is P.fft_sparse_first_order_multiply
        assert apxmm.cli.matmul_naive is P.matmul_naive
        assert apxmm.ApproxReport is P.ApproxReport
        assert apxmm.svd_first_order_multiply is P.svd_first_order_multiply
        assert apxmm.sketch_norm_estimate is P.sketch_norm_estimate
        # out-of-scope modules stay the reference's (CPU): the lowrank baseline still runs
        rng = np.random.default_rng(0)
        A, B = rng.standard_normal((8, 8)), rng.standard_normal((8, 8))
        M, rep = apxmm.cli.run_method("lowrank", 0, A, B, c=4, seed=1)
        assert M.shape == (8, 8) and rep.method == "lowrank"
    finally:
        import sys
        for k in [m for m in sys.modules if m.startswith("apxmm_gpu_test")]:
            del sys.modules[k]


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["naive", "svd", "cd", "sfft", "cycle", "mixed"])
def test_dispatch_matches_oracle(method):
    from conftest import rel
    from paper_2504_19308_b200.dispatch import run_method
    n = 64
    if method in ("cycle", "mixed"):
        A = O.gen_cycle_operand(n, 9, 3)
        B = O.gen_cycle_operand(n, 9, 4)
    else:
        rng = np.random.default_rng(5)
        A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    M, rep = run_method(method, 1, A, B, s=2, k=8, seed=3)
    if method == "naive":
        Mo = A @ B
    elif method == "svd":
        Mo, _ = O.svd_first_order_multiply(A, B, 2, 1, 3)
    elif method == "cd":
        Mo, ro = O.circulant_first_order_multiply(A, B, 8, 1, force_sel_a=rep.selected_a,
                                                  force_sel_b=rep.selected_b)
    elif method == "sfft":
        Mo, ro = O.fft_sparse_first_order_multiply(A, B, 8, 1, force_a=rep.selected_a, force_b=rep.selected_b)
    elif method == "cycle":
        Mo, _ = O.cycle_first_order_multiply(A, B, 8, 1)
    else:
        Mo, _ = O.mixed_first_order_multiply(A, B, 8, 8, 1, 3)
    assert rel(np.asarray(M), Mo) < 1e-10
    assert rep.method == {"naive": "naive", "svd": "svd", "cd": "cd", "sfft": "sfft", "cycle": "cycle",
                          "mixed": "mixed"}[method]


def test_sketch_validation_before_device():
    """errest.py:147-150: shape and k errors are raised before any device work."""
    from paper_2504_19308_b200 import sketch_norm_estimate
    with pytest.raises(ValueError):
        sketch_norm_estimate(np.eye(3), np.eye(4), 2, 0)
    with pytest.raises(ValueError):
        sketch_norm_estimate(np.eye(3), np.eye(3), 0, 0)


def test_extend_bench_csv(tmp_path):
    """clibench.extend_bench_csv: the reference's bench schema plus products/s and roofline columns."""
    from paper_2504_19308_b200.clibench import EXTRA, extend_bench_csv
    src = tmp_path / "b.csv"
    src.write_text("method,order,n,kind_a,kind_b,s,k,rel_err,apriori_est,posterior_est,wall_time_s,seed\n"
                   "svd,first,512,kappa,kappa,1,10,0.01,0.02,0.03,0.002,0\n"
                   "naive,-,512,kappa,kappa,-,-,0,-,-,0.5,0\n")
    dst = tmp_path / "b.gpu.csv"
    assert extend_bench_csv(str(src), str(dst), 35.8, lambda m, n, k=0, c=0: 6.0 * k * n * n if m == "svd" else 2.0 * n ** 3) == 2
    rows = [line.split(",") for line in dst.read_text().splitlines()]
    assert rows[0][12:] == EXTRA
    assert float(rows[1][12]) == pytest.approx(500.0)
    assert float(rows[1][13]) == pytest.approx(6.0 * 10 * 512 * 512)
    assert float(rows[1][16]) == pytest.approx(6.0 * 10 * 512 * 512 / 0.002 / 1e12 / 35.8, rel=1e-5)
