import sys, torch
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from devgen import c5_operand
for (n, nc, r) in ((32768, 16, 2), (32768, 128, 0), (32768, 128, 32)):
    try:
        A, J = c5_operand(n, nc, r, seed=5, operand=0)
        torch.cuda.synchronize()
        print(n, nc, r, 'ok', float(A.abs().max()), flush=True)
        del A
    except Exception as e:
        print(n, nc, r, 'FAIL', str(e)[:200], flush=True)
        raise
