"""The reference's own CLI (cli.py bench / multiply / sweep) on the GPU path via
the apxmm shim, from the staged reference copy baseline/_ref/pkg (tools/stage_reference.sh; the
reference tree itself is never read at test time). Skips when the copy is absent."""
import csv
import json
import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = os.path.join(ROOT, "baseline", "_ref", "pkg", "src")
need_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "apxmm")),
                              reason="staged reference copy baseline/_ref/pkg absent")


@need_ref
def test_cli_bench_gpu_columns(tmp_path, capsys):
    from paper_2504_19308_b200 import clibench
    conf = tmp_path / "bench.conf"
    conf.write_text("methods = svd:first, cd:first, sfft:zeroth, naive\n"
                    "kinds = kappa:kappa, circulant:general\n"
                    "sizes = 64, 128\ns = 1, 2\ntrials = 2\nseed_base = 3\n")
    out = tmp_path / "bench.csv"
    rc = clibench.main([REF_SRC, "bench", "--config", str(conf), "--out", str(out), "--gpu-columns"])
    assert rc == 0
    rows = list(csv.reader(open(tmp_path / "bench.gpu.csv")))
    head = rows[0]
    assert head[:12] == "method,order,n,kind_a,kind_b,s,k,rel_err,apriori_est,posterior_est,wall_time_s,seed".split(",")
    assert head[12:] == clibench.EXTRA
    assert len(rows) - 1 == (3 * 2 * 2 * 2 + 1 * 2 * 2) * 2
    for r in rows[1:]:
        if r[0] != "naive":
            assert float(r[7]) < 1.0 and float(r[12]) > 0 and 0 < float(r[16]) < 1.0


@need_ref
def test_cli_multiply_and_sweep(tmp_path, capsys):
    from paper_2504_19308_b200 import clibench
    rc = clibench.run(["multiply", "--method", "cd", "--order", "first", "--kind-a", "circulant", "--kind-b",
                       "general", "--n", "96", "--k", "5", "--check"], REF_SRC)
    assert rc == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["method"] == "cd" and line["rel_err"] < 1.0
    rc = clibench.run(["sweep", "--method", "svd", "--order", "first", "--tol", "0.05", "--kind-a", "kappa",
                       "--kind-b", "kappa", "--n", "64", "--trials", "2", "--s-max", "6"], REF_SRC)
    assert rc == 0
