import os, sys, time, subprocess, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_17101_b200 import B200ArrayContext
from paper_2512_17101_b200.operators import NavierStokesOperator
from tests.common import make_dcoll, random_state
gpu = B200ArrayContext()
d = make_dcoll(gpu, 3, 3, 94, "periodic")
op = NavierStokesOperator(d, mu=1e-3)
q = d.from_numpy(random_state(3, d.nelements, d.Np, seed=1))
def timeit(fn, n=30):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n+1)]
    ev[0].record()
    for i in range(n):
        fn(); ev[i+1].record()
    torch.cuda.synchronize()
    ts = [ev[i].elapsed_time(ev[i+1]) for i in range(n)]
    return np.median(ts), min(ts), max(ts)
samples = []
stop = False
def sampler():
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active,temperature.gpu", "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    while not stop:
        l = p.stdout.readline()
        if l: samples.append((time.time(), l.strip()))
    p.kill()
th = threading.Thread(target=sampler); th.start()
time.sleep(1.0)
T = op.flux(q)
t0=time.time(); r = timeit(lambda: op.flux(q), 60); print("pass1 alone", r, flush=True); t1=time.time()
r = timeit(lambda: op.rhs(q), 60); print("both", r, flush=True); t2=time.time()
from paper_2512_17101_b200 import fused
r = timeit(lambda: op._div(q.data if hasattr(q,'data') else q, T, *op._div_args()), 60) if False else None
time.sleep(0.5)
stop = True; th.join()
for (a,b,name) in [(t0,t1,"pass1 alone"),(t1,t2,"both")]:
    s=[x[1] for x in samples if a+0.3<x[0]<b]
    print(name, len(s), "samples; first/last:", s[:2], s[-2:])
    clk=[int(x.split(',')[0]) for x in s]; pw=[float(x.split(',')[1]) for x in s]
    print("   clk min/med/max", min(clk), np.median(clk), max(clk), "power med/max", np.median(pw), max(pw))
