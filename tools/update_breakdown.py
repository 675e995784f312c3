import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2509_25401_b200 as fo
from paper_2509_25401_b200 import _lib
from paper_2509_25401_b200.engine import Engine, EngineConfig
cfg = EngineConfig(n_text=256, n_vision=32768, d_model=3072, heads=24, tau_q=0.3, tau_kv=0.5,
                   interval_n=6, order_d=1, steps=13, layers=1)
eng = Engine(cfg)
for t in range(7): eng.step(t)
torch.cuda.synchronize()
L = eng.layers[0]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(10)]
x = eng.x_buf
p = L.params
from paper_2509_25401_b200.gemm import project_q, project_out_update
from paper_2509_25401_b200.pipeline import project_kv
from paper_2509_25401_b200.policy import generate_masks_heads
from paper_2509_25401_b200.symbols import encode_symbols
from paper_2509_25401_b200.attention import dense_attention_update
from paper_2509_25401_b200.plan import Plan
for rep in range(2):
    ev[0].record()
    project_q(x, p.w_q, p.q_norm, None, "update", out=L.q, fill=None, check=False)
    ev[1].record()
    project_kv(x, p, k_out=L.k, v_out=L.v, check=False)
    ev[2].record()
    generate_masks_heads(L.q, L.k, pool_n=1, n_text=256, tau_q=0.3, tau_kv=0.5, cache_out=L.cb, skip_out=L.sb, check=False)
    ev[3].record()
    encode_symbols(L.cb, L.sb, 1, check=False, out=L.sym)
    ev[4].record()
    dense_attention_update(L.q, L.k, L.v, L.cache, out=L.o, check=False)
    ev[5].record()
    Plan.build(L.sym, valid=L.cache.valid, order_d=1, check=False, ws=L.plan_c.ws)
    ev[6].record()
    project_out_update(L.o, p.w_out, L.sym, L.cache, 1, out=L.out, bias=L.bias, plan=L.plan_c, check=False)
    ev[7].record()
    torch.cuda.synchronize()
names = ["gemm_q", "kv", "policy", "encode", "dense_attn+push", "plan", "gemm_o_update"]
print({n: round(ev[i].elapsed_time(ev[i+1]), 3) for i, n in enumerate(names)})
