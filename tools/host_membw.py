import os, time, threading
import numpy as np
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
n = 1 << 28  # 1 GiB of float32
src = np.ones(n // 4, np.float32); dst = np.empty_like(src)
dst[:] = 0
for _ in range(2):
    t = time.perf_counter(); np.copyto(dst, src); dt = time.perf_counter() - t
    print(f"numpy copy 1 GiB: {1/dt:.1f} GiB/s")
import torch
pin = torch.empty(n // 4, dtype=torch.float32, pin_memory=True).numpy()
for _ in range(2):
    t = time.perf_counter(); np.copyto(pin, src); dt = time.perf_counter() - t
    print(f"numpy copy into pinned 1 GiB: {1/dt:.1f} GiB/s")
def part(i, k):
    s = slice(i * (len(src) // k), (i + 1) * (len(src) // k))
    np.copyto(pin[s], src[s])
for k in (4, 8, 16):
    t = time.perf_counter()
    th = [threading.Thread(target=part, args=(i, k)) for i in range(k)]
    [x.start() for x in th]; [x.join() for x in th]
    dt = time.perf_counter() - t
    print(f"{k} threads into pinned: {1/dt:.1f} GiB/s")
