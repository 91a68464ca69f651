"""Host<->device copy bandwidth on the box (pinned memory), for the e2e roofline."""
import torch, time
n = 12 * 1024**3 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name}: {n*4/ms/1e6:.1f} GB/s ({ms:.1f} ms for {n*4/1e9:.1f} GB)")
# concurrent h2d + d2h on two streams (full duplex?)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2):
    h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"duplex: {n*4/dt/1e9:.1f} GB/s total ({dt*1e3:.1f} ms)")
