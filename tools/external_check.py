"""External dense baselines on the same B200: cuDNN SDPA and
cuBLAS GEMM next to this engine's dense attention / dense GEMM-Q at C4.

    python tools/external_check.py
"""

import json
import pathlib
import sys
import time

import torch
import torch.nn.functional as F

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2509_25401_b200 as fo  # noqa: E402
from tools.sweep import timeit  # noqa: E402


def main():
    S, H, D, dm = 33024, 24, 128, 3072
    torch.manual_seed(0)
    q, k, v = (torch.randn(S, H, D, device="cuda").bfloat16() for _ in range(3))
    res = {"config": dict(seq=S, heads=H, head_dim=D, d_model=dm)}
    attn_flops = 4.0 * H * S * S * D
    ours = timeit(lambda: fo.dense_attention_update(q, k, v, None, check=False), 2, 5)
    res["engine_dense_attention"] = dict(ms=ours, tflops=attn_flops / ours / 1e9)
    qb, kb, vb = (a.permute(1, 0, 2).unsqueeze(0) for a in (q, k, v))  # [1, H, S, D] views
    from torch.nn.attention import SDPBackend, sdpa_kernel

    for name, be in (("cudnn_sdpa", SDPBackend.CUDNN_ATTENTION),
                     ("flash_sdpa", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                time.sleep(1)
                ms = timeit(lambda: F.scaled_dot_product_attention(qb, kb, vb), 2, 5)
            res[name] = dict(ms=ms, tflops=attn_flops / ms / 1e9)
        except Exception as exc:  # noqa: BLE001
            res[name] = f"unavailable: {type(exc).__name__}: {str(exc)[:120]}"
    x = torch.randn(S, dm, device="cuda").bfloat16()
    w = torch.randn(H * D, dm, device="cuda").bfloat16() * dm ** -0.5
    gflop = 2.0 * S * dm * H * D
    time.sleep(1)
    ms = timeit(lambda: x @ w.t(), 3, 10)
    res["cublas_gemm_q_dense"] = dict(ms=ms, tflops=gflop / ms / 1e9)
    wq = fo.pack_w_q(w.float().view(H, D, dm).permute(0, 2, 1))
    time.sleep(1)
    qo = torch.empty(S, H, D, dtype=torch.bfloat16, device="cuda")
    ms = timeit(lambda: fo.project_q(x, wq, None, None, "update", rope=False, fill=None, out=qo,
                                     check=False), 3, 10)
    res["engine_gemm_q_dense_plain"] = dict(ms=ms, tflops=gflop / ms / 1e9)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
