"""Per-CTA timeline of one attention launch (bench C4 workload), from a
library built with -DFO_CS_TIMING (tools/build_variant.sh). Prints the spread
of CTA end times and per-SM tile rates."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_25401_b200 as fo  # noqa: E402
from paper_2509_25401_b200 import _lib  # noqa: E402
from bench import random_masks  # noqa: E402

T, S, H = 128, 33024, 24
t = S // T
cached, skip = (float(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (0.25, 0.5)))
dev = torch.device("cuda", 0)
cb, sb = random_masks(np.random.default_rng(0), H, t, cached, skip)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn(S, H, T, device=dev, generator=g).bfloat16() for _ in range(3))
sym = fo.encode_symbols(cb, sb, 1)
cache = fo.FeatureCache(H, t, 1, seq=S)
for _ in range(2):
    cache.push(torch.randn(S, H, T, device=dev, generator=g).bfloat16())
o = torch.empty_like(q)
for _ in range(5):
    fo.sparse_attention(q, k, v, sym, cache, None, 2, 6, 1, mode="bias", out=o, check=False)
torch.cuda.synchronize()
lib = _lib.load()
n = 148
buf = (ctypes.c_ulonglong * (4 * 1024))()
assert lib.fo_debug_cs_timing(buf, 1024) == 0
a = np.array(buf[:4 * n], dtype=np.int64).reshape(n, 4)
t0 = a[:, 0].min()
start, end, sm, tiles = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2], a[:, 3]
busy = end - start
rate = busy * 1e3 / np.maximum(tiles, 1)  # ns per tile
print(f"kernel span {end.max():.1f} us; CTA start spread {start.max() - start.min():.1f} us")
print(f"end: min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f} us; "
      f"mean idle at tail {(end.max() - end).mean():.1f} us ({(end.max() - end).mean() / end.max() * 100:.2f}%)")
print(f"tiles per CTA: min {tiles.min()} max {tiles.max()} mean {tiles.mean():.1f}")
print(f"ns per tile: min {rate.min():.0f} median {np.median(rate):.0f} max {rate.max():.0f}")
order = np.argsort(sm)
print("by SM (sm: ns/tile):", " ".join(f"{s}:{r:.0f}" for s, r in zip(sm[order][:148:8], rate[order][:148:8])))
