"""PCIe copy probe (host <-> B200): single vs split copies, one vs several streams."""
import time

import torch

n = 19092072 // 8
big = torch.empty(n, dtype=torch.float64).pin_memory()
parts = [big[i * (n // 3):(i + 1) * (n // 3)] for i in range(3)]
sep = [torch.empty(n // 3, dtype=torch.float64).pin_memory() for _ in range(3)]
d = torch.empty(n, dtype=torch.float64, device="cuda")
dparts = [d[i * (n // 3):(i + 1) * (n // 3)] for i in range(3)]
streams = [torch.cuda.Stream() for _ in range(3)]


def multi(src, dst, h2d):
    ev = torch.cuda.current_stream().record_event()
    for s, a, b in zip(streams, dst, src):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            (a if h2d else b).copy_(b if h2d else a, non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)


cases = [
    ("h2d 1x19MB", lambda: d.copy_(big, non_blocking=True)),
    ("h2d 1x6MB", lambda: dparts[0].copy_(parts[0], non_blocking=True)),
    ("h2d 3x6MB slices, 1 stream", lambda: [a.copy_(b, non_blocking=True) for a, b in zip(dparts, parts)]),
    ("h2d 3x6MB separate, 1 stream", lambda: [a.copy_(b, non_blocking=True) for a, b in zip(dparts, sep)]),
    ("h2d 3x6MB separate, 3 streams", lambda: multi(sep, dparts, True)),
    ("d2h 3x6MB separate, 1 stream", lambda: [b.copy_(a, non_blocking=True) for a, b in zip(dparts, sep)]),
    ("d2h 3x6MB separate, 3 streams", lambda: multi(dparts, sep, False)),
]
for name, fn in cases:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    mb = 6.36 if "1x6" in name else 19.09
    print(f"{name:32s} {dt * 1e3:.3f} ms  {mb / dt / 1e3:.1f} GB/s")
