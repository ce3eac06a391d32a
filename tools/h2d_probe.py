"""Pinned host <-> device copy bandwidth of the box (the e2e arm's ceiling): 4 GiB H2D in
1 / 4 / 16 chunks over 4 streams, then D2H."""
import torch, time
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunks in (1, 4, 16):
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(3):
        step = n // chunks
        for c in range(chunks):
            with torch.cuda.stream(streams[c % 4]):
                d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"H2D {chunks} chunks over 4 streams: {n / dt / 1e9:.1f} GB/s", flush=True)
t0 = time.perf_counter()
for r in range(3):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H: {n * 3 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
