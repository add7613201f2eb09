import torch, time
dev = torch.device("cuda")
for mb in (64, 168):
    n = mb * (1 << 20) // 8
    h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
    d1 = torch.empty(n, dtype=torch.float64, device=dev); d2 = torch.empty(n, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    def t(fn, k=5):
        torch.cuda.synchronize(); a = time.perf_counter()
        for _ in range(k): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - a) / k
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    tb = t(both)
    B = n * 8 / 1e9
    print(f"{mb} MB: H2D {B/th:.1f} GB/s, D2H {B/td:.1f} GB/s, both {2*B/tb:.1f} GB/s total")
