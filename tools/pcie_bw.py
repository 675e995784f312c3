import torch, time
n = 33024 * 3072
h1 = torch.empty(n, dtype=torch.bfloat16, pin_memory=True); h2 = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
d1 = torch.empty(n, dtype=torch.bfloat16, device='cuda'); d2 = torch.empty(n, dtype=torch.bfloat16, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2): d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def bench(fn, k=10):
    torch.cuda.synchronize(); t = time.time()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.time() - t) / k * 1e3
b = n * 2
h2d = bench(lambda: d1.copy_(h1, non_blocking=True)); print(f"H2D {h2d:.2f} ms {b/h2d/1e6:.1f} GB/s")
d2h = bench(lambda: h2.copy_(d2, non_blocking=True)); print(f"D2H {d2h:.2f} ms {b/d2h/1e6:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bo = bench(both); print(f"both {bo:.2f} ms per pair")
