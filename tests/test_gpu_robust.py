"""Robustness of the multi-stream C4 plan: the Q.W epilogue's bounded wait on the gather's
ready flags. With APX_QW_STALL_NS=0 every tile defers itself (the path a tile takes when the
gather's CTAs are not co-resident, e.g. under MPS SM limits, and its rows make no progress for
20 ms), and qw_fixup_sum_kernel completes it after the gather: M must still match the normal plan and
the oracle. Also: per-device side streams survive a device re-selection."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2504_19308_b200 as P
from paper_2504_19308_b200 import _native as N
n, k = 2048, 64
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn(n, n, device="cuda", generator=g) / n ** 0.5
B = 1e-3 * torch.randn(n, n, device="cuda", generator=g)
idx = torch.arange(n, device="cuda")
for j in range(0, n, n // 64):
    B[idx, (idx - j) %% n] += torch.randn(n, device="cuda", generator=g)
M, rep = P.mixed_first_order_multiply(A, B, k, k, 1, seed=5)
M2, rep2 = P.mixed_first_order_multiply(A, B, k, k, 1, seed=5)
torch.cuda.synchronize()
np.save(sys.argv[1], M.cpu().numpy())
print(json.dumps({"sel": rep.selected_b, "nm": rep.posterior_estimate, "rep_equal": bool(torch.equal(M, M2))}))
"""


def _run(tmp_path, env_extra, tag):
    out = tmp_path / f"{tag}.npy"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT, str(out)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out), json.loads(r.stdout.strip().splitlines()[-1])


def test_deferred_qw_tiles_match_normal_plan(tmp_path):
    M0, j0 = _run(tmp_path, {}, "normal")
    M1, j1 = _run(tmp_path, {"APX_QW_STALL_NS": "0"}, "deferred")
    assert j0["sel"] == j1["sel"]
    assert j0["rep_equal"]  # the normal plan is bitwise reproducible
    d = np.linalg.norm(M1.astype(np.float64) - M0) / np.linalg.norm(M0)
    assert d < 1e-5, d
    # deferral did happen: the fp32-FMA fixup tiles differ from tcgen05 tiles in the last bits
    assert not np.array_equal(M0, M1)
    assert j1["nm"] == pytest.approx(j0["nm"], rel=1e-5)


def test_side_streams_per_device():
    """Re-selecting the device between calls keeps each product on that device's side streams."""
    import torch
    import oracle as O
    import paper_2504_19308_b200 as P
    n = 512
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 3).astype(np.float32)
    B = O.gen_cycle_operand(n, 16, 4).astype(np.float32)
    outs = []
    for dev in range(torch.cuda.device_count()):
        torch.cuda.set_device(dev)
        M, _ = P.mixed_first_order_multiply(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 16, 16, 1, 5)
        outs.append(M.cpu().numpy())
    torch.cuda.set_device(0)
    M, _ = P.mixed_first_order_multiply(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 16, 16, 1, 5)
    assert all(np.array_equal(o, M.cpu().numpy()) for o in outs)
