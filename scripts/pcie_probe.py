"""Host<->device copy bandwidth of this box: H2D alone, D2H alone, both at once (sets the ceiling of bench.py's e2e)."""
import torch
n = 1 << 29   # 4 GiB of f64
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best
gb = n * 8 / 1e9
t = timed(lambda: d1.copy_(h1, non_blocking=True)); print(f"H2D alone  {gb / t * 1e3:.1f} GB/s ({t:.1f} ms)")
t = timed(lambda: h2.copy_(d2, non_blocking=True)); print(f"D2H alone  {gb / t * 1e3:.1f} GB/s ({t:.1f} ms)")
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
t = timed(both); print(f"H2D + D2H concurrently: {2 * gb / t * 1e3:.1f} GB/s aggregate ({t:.1f} ms for {gb:.1f} GB each way)")
