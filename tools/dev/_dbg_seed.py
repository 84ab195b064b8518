"""debug: single-device cycle product on C5-style operands (n, k, seed from argv)"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2504_19308_b200 as P
from devgen import c5_operand
n, k, seed = (int(v) for v in sys.argv[1:4])
A, JA = c5_operand(n, k, 8, seed=seed, operand=0)
B, JB = c5_operand(n, k, 8, seed=seed, operand=1)
try:
    r = P.cycle_product_device(A, B, k, k, 1); torch.cuda.synchronize(); print(n, k, seed, "ok", flush=True)
except Exception as e:
    print(n, k, seed, "FAIL", str(e)[-120:], flush=True)
