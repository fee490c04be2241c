"""Host<->device copy bandwidth of this box: H2D alone, D2H alone, both at once (the ceiling of bench.py's e2e),
with the pinned buffers first-touched (a) under the process's default CPU affinity and (b) on the CPUs of the
GPU's own NUMA node.  Prints the NUMA facts it finds; everything is best effort inside a container."""
import glob
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import gpu_numa_cpus  # noqa: E402

n = 1 << 28   # 2 GiB of f64


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def measure(tag):
    h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h1.zero_()
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2.zero_()
    d1 = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    gb = n * 8 / 1e9
    t1 = timed(lambda: d1.copy_(h1, non_blocking=True))
    t2 = timed(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)
    t3 = timed(both)
    print(f"[{tag}] H2D {gb / t1 * 1e3:.1f} GB/s, D2H {gb / t2 * 1e3:.1f} GB/s, both at once {2 * gb / t3 * 1e3:.1f} GB/s aggregate "
          f"({t3:.1f} ms for {gb:.1f} GB each way)", flush=True)


print("nodes:", [os.path.basename(p) for p in glob.glob("/sys/devices/system/node/node[0-9]*")])
print("affinity now:", len(os.sched_getaffinity(0)), "cpus")
cpus, node = gpu_numa_cpus(0)
print("GPU 0 NUMA node:", node, "cpus:", None if cpus is None else len(cpus))
measure("default affinity")
if cpus:
    os.sched_setaffinity(0, cpus)
    measure(f"bound to NUMA node {node}")
