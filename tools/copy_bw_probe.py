import torch, time
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
hin = torch.empty(n, dtype=torch.uint8).pin_memory()
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for j, s in enumerate(ss):
            with torch.cuda.stream(s):
                a, b = j * n // k, (j + 1) * n // k
                h[a:b].copy_(d[a:b], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"D2H 1 GiB on {k} streams: {n / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d.copy_(hin, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"D2H + H2D 1 GiB each concurrently: {2 * n / dt / 1e9:.1f} GB/s total")
