import time, torch
n = 19092072 // 8
a = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
f = torch.zeros(64, dtype=torch.int64).pin_memory()
fd = torch.zeros(64, dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()
def run(ns, flags):
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(a, non_blocking=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            ch = (n + ns - 1) // ns
            for k in range(ns):
                d[k*ch:(k+1)*ch].copy_(a[k*ch:(k+1)*ch], non_blocking=True)
                if flags:
                    fd[k:k+1].copy_(f[k:k+1], non_blocking=True)
            s.synchronize()
            ts.append(time.perf_counter() - t0)
    ts.sort()
    print(ns, flags, f"{ts[5]*1e3:.3f} ms", flush=True)
for ns in (1, 8, 24, 64):
    for fl in (False, True):
        run(ns, fl)
# 3 copies per slab like x, v, e
