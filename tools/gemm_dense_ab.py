"""Dense GEMM-Q (K/V projection shape) timing, for FO_GEMM_2SM A/B runs:
    FO_GEMM_2SM=0 python tools/gemm_dense_ab.py ; python tools/gemm_dense_ab.py"""
import os
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo  # noqa: E402
from tools.sweep import timeit  # noqa: E402

S, H, D, dm = 33024, 24, 128, 3072
x = torch.randn(S, dm, device="cuda").bfloat16()
w = fo.pack_w_q(torch.randn(H, dm, D, device="cuda") * dm ** -0.5)
nw = torch.ones(H, D, device="cuda")
out = torch.empty(S, H, D, dtype=torch.bfloat16, device="cuda")
gf = 2.0 * S * dm * H * D
plain = timeit(lambda: fo.project_q(x, w, None, None, "update", rope=False, out=out, fill=None,
                                    check=False), 3, 20)
normrope = timeit(lambda: fo.project_q(x, w, nw, None, "update", out=out, fill=None, check=False),
                  3, 20)
print(f"FO_GEMM_2SM={os.environ.get('FO_GEMM_2SM', '1')} plain {plain:.4f} ms "
      f"({gf / plain / 1e9:.0f} TF/s)  norm+rope {normrope:.4f} ms ({gf / normrope / 1e9:.0f} TF/s)")
