"""debug: sharded cycle product at a C5-like shape (n from argv), 2 shards, vs single device"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2504_19308_b200 as P
from paper_2504_19308_b200 import sharded as SH
from devgen import c5_operand
n = int(sys.argv[1]); k = int(sys.argv[2]); world = int(sys.argv[3])
A, JA = c5_operand(n, k, 8, seed=13, operand=0)
B, JB = c5_operand(n, k, 8, seed=13, operand=1)
torch.cuda.synchronize(); print("gen ok", flush=True)
full = P.cycle_product_device(A, B, k, k, 1); torch.cuda.synchronize(); print("full ok", flush=True)
blocks = [SH.cycle_row_range(n, world, r, 128) for r in range(world)]
gens = [SH.cycle_rows_steps(A[r0:r1], r0, B, k, k, 1) for r0, r1 in blocks]
res = SH.lockstep(gens); torch.cuda.synchronize(); print("sharded ok", flush=True)
M = torch.cat([r["M"] for r in res])
print("rel", float(torch.linalg.norm((M - full["M"]).double()) / torch.linalg.norm(full["M"].double())))
