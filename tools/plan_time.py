import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_25401_b200 as fo
from bench import random_masks
from paper_2509_25401_b200.plan import Plan
cb, sb = random_masks(np.random.default_rng(0), 24, 258, 0.25, 0.5)
sym = fo.encode_symbols(cb, sb, 1)
ws = torch.empty(fo._lib.load().fo_plan_workspace_bytes(24, 258), dtype=torch.uint8, device='cuda')
for _ in range(3): Plan.build(sym, ws=ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): Plan.build(sym, ws=ws, check=False)
e1.record(); torch.cuda.synchronize()
print("plan us", e0.elapsed_time(e1) / 20 * 1000)
