import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, oracle as O, paper_2504_19308_b200 as P
dev = torch.device("cuda")
n = 2048
A = torch.from_numpy(O.gen_cycle_operand(n, 32, 3)).to(dev)
B = torch.from_numpy(O.gen_cycle_operand(n, 32, 4)).to(dev)
for _ in range(3): P.cycle_product_device(A, B, 32, 32, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): P.cycle_product_device(A, B, 32, 32, 1)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("APX_GATHER_R"), e0.elapsed_time(e1) / 20)
