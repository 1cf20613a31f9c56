"""Run one plan build at the C3 shape (32 q / 8 kv heads, d=128, bf16, S=2048) -- for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_22575_b200 as s2o
L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
torch.manual_seed(0)
q = torch.randn(1, 32, L, 128, device='cuda').to(torch.bfloat16)
k = torch.randn(1, 8, L, 128, device='cuda').to(torch.bfloat16)
s2o.build_plan(q, k, 2048)
torch.cuda.synchronize()
