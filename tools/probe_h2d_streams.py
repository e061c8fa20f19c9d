"""Pinned host-to-device bandwidth over 1 / 2 / 4 / 8 concurrent copy streams
and over interleaved 16-256 MiB chunks on two streams (2 GiB, torch copies):
is the e2e link limit a single-stream artefact?  (It is not: 55.1-55.5 GB/s.)"""
import torch, time, json
n = 1 << 29  # 2 GiB of float32
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
res = {}
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        res.setdefault(k, []).append(round(4 * n / dt / 1e9, 2))
print(json.dumps(res))
# interleaved small chunks on 2 streams
for csz in (16 << 20, 64 << 20, 256 << 20):
    s2 = [torch.cuda.Stream(), torch.cuda.Stream()]
    m = csz // 4
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for j, off in enumerate(range(0, n, m)):
        with torch.cuda.stream(s2[j & 1]):
            d[off:off+m].copy_(h[off:off+m], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("chunk", csz >> 20, "MiB x2 streams", round(4 * n / dt / 1e9, 2))
