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

T, H = 128, 24
S = int(sys.argv[3]) if len(sys.argv) > 3 else 33024
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
buf = (ctypes.c_ulonglong * (16 * 1024))()
assert lib.fo_debug_cs_timing(buf, 1024) == 0
raw = [int(v) for v in buf[:16 * n]]
raw0 = [v - (1 << 64) if v >= (1 << 63) else v for v in raw]
qk_to_s = np.array([float('nan')] * n)
for b in range(n):
    raw[16 * b + 10] = 0
a = np.array(raw, dtype=np.int64).reshape(n, 16)
t0 = a[:, 0].min()
start, end, sm, tiles = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2], a[:, 3]
ga, gb, gc, nit = a[:, 4] / 1e3, a[:, 5] / 1e3, a[:, 6] / 1e3, np.maximum(a[:, 7], 1)
busy = end - start
rate = busy * 1e3 / np.maximum(tiles, 1)  # ns per tile
print(f"kernel span {end.max():.1f} us; CTA start spread {start.max() - start.min():.1f} us")
print(f"end: min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f} us; "
      f"mean idle at tail {(end.max() - end).mean():.1f} us ({(end.max() - end).mean() / end.max() * 100:.2f}%)")
print(f"tiles per CTA: min {tiles.min()} max {tiles.max()} mean {tiles.mean():.1f}")
print(f"ns per tile: min {rate.min():.0f} median {np.median(rate):.0f} max {rate.max():.0f}")
print(f"per item (us): last P -> last PV done {np.mean(ga / nit):.2f}, epilogue {np.mean(gb / nit):.2f}, "
      f"epilogue end -> next first S {np.mean(gc / np.maximum(nit - 1, 1)):.2f}; items/CTA {nit.mean():.1f}; "
      f"boundary share of the span {np.mean(ga + gb + gc) / end.max():.2%}")
print(f"per item (us): producer waits q_empty {np.mean(a[:, 8] / 1e3 / nit):.2f}; "
      f"MMA last PV issued -> next Q landed {np.mean(a[:, 9] / 1e3 / nit):.2f}")
print(f"per item (us): softmax epilogue end -> reaches the first S wait {np.mean(np.array([raw0[16 * b + 10] for b in range(n)], dtype=np.float64) / 1e3 / np.maximum(nit - 1, 1)):.2f}")
print(f"per item (us): first QK issued -> its s_full completes (MMA warp polling) {np.mean(np.array([raw0[16 * b + 11] for b in range(n)], dtype=np.float64) / 1e3 / np.maximum(nit - 1, 1)):.2f}")
order = np.argsort(sm)
print("by SM (sm: ns/tile):", " ".join(f"{s}:{r:.0f}" for s, r in zip(sm[order][:148:8], rate[order][:148:8])))
st = np.maximum(a[:, 14], 1)
print(f"steady-state tile (cycles, softmax thread 128): waiting for S {np.mean(a[:, 12] / st):.0f}, "
      f"S landed -> P stored {np.mean(a[:, 13] / st):.0f}, tiles/CTA {np.mean(a[:, 14]):.0f}")
ph = (ctypes.c_longlong * (5 * 1024))()
if hasattr(lib, "fo_debug_cs_phases") and lib.fo_debug_cs_phases(ph, 1024) == 0:
    P = np.array(ph[:5 * n], dtype=np.int64).reshape(n, 5) / st[:, None]
    names = ["S tmem->reg", "max+exchange", "exp+pack", "P reg->tmem", "check+arrive"]
    print("softmax phases (cycles/tile): " + ", ".join(f"{k} {v:.0f}" for k, v in zip(names, P.mean(0))))

ep = (ctypes.c_longlong * (6 * 1024))()
if hasattr(lib, "fo_debug_cs_epilogue") and lib.fo_debug_cs_epilogue(ep, 1024) == 0:
    E = np.array(ep[:6 * n], dtype=np.int64).reshape(n, 6) / nit[:, None]
    names = ["l from TMEM", "next record+counters", "O chunk0 TMEM ld", "chunk1 scale/stage/TMA store",
             "chunk0 scale/stage/TMA store + chunk1 TMEM ld", "fence+arrive o_free"]
    print("epilogue (cycles/item): " + ", ".join(f"{k} {v:.0f}" for k, v in zip(names, E.mean(0))))
