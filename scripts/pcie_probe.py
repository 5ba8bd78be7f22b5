"""PCIe copy bandwidth probe (not product code): pinned H2D / D2H alone, on
one or two streams, and H2D + D2H concurrently -- the bound on config B's
end-to-end number."""
import time

import torch

MB = 1 << 20
n = 512 * MB // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n // 2, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n // 2, dtype=torch.float32, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d(streams, chunks=16):
    k = n // chunks
    for i in range(chunks):
        with torch.cuda.stream(streams[i % len(streams)]):
            d[i * k:(i + 1) * k].copy_(h[i * k:(i + 1) * k], non_blocking=True)


def d2h(streams, chunks=16):
    k = (n // 2) // chunks
    for i in range(chunks):
        with torch.cuda.stream(streams[i % len(streams)]):
            h2[i * k:(i + 1) * k].copy_(d2[i * k:(i + 1) * k], non_blocking=True)


for name, fn, nbytes in [
    ("H2D 1 stream", lambda: h2d(s[:1]), n * 4),
    ("H2D 2 streams", lambda: h2d(s[:2]), n * 4),
    ("D2H 1 stream", lambda: d2h(s[2:3]), n * 2),
    ("D2H 2 streams", lambda: d2h(s[2:4]), n * 2),
    ("H2D+D2H concurrent", lambda: (h2d(s[:1]), d2h(s[2:3])), n * 6),
    ("H2D(2)+D2H(2) concurrent", lambda: (h2d(s[:2]), d2h(s[2:4])), n * 6),
]:
    t = timed(fn)
    print(f"{name:28s} {nbytes / t / 1e9:7.1f} GB/s  ({t * 1e3:.2f} ms for {nbytes / 1e6:.0f} MB)")
