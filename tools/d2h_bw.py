import torch, time
n = 1 << 27  # 1 GiB of doubles
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = n // streams
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                h[i*chunk:(i+1)*chunk].copy_(d[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print("D2H streams", streams, round(8 * n / dt / 1e9, 1), "GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print("H2D", round(8 * n / dt / 1e9, 1), "GB/s")
