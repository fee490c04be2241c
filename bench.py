#!/usr/bin/env python
"""Headline benchmark: 3D compressible Navier-Stokes DG right-hand side, order 3, ~100M DOFs
per GPU (BASELINE.json configs[2]); metric GDOF/s and fraction of the HBM roofline.

    python bench.py --gpus N --steps K --warmup W            # the B200 path
    python bench.py --impl reference --steps K --warmup W    # the CPU reference path (oracle port)

One "step" = one full RHS evaluation (gradient pass + flux/divergence pass, plus the halo
exchanges when N > 1) on synthetic seeded data.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIM, ORDER = 3, 3
NP = 20
B_ALG_RHS = 360.0      # algorithmic bytes per node-DOF per NS RHS: (3C + 2Cd) * 8, C=5, d=3
B_ALG_GRAD = 160.0     # pass 1: read q (40) + write grad q (120)
B_ALG_DIV = 200.0      # pass 2: read q (40) + read grad q (120) + write rhs (40)
# The flux arrangement (default) stores 16 planes (15 contravariant flux + wave speed) instead of 15; its
# roofline fractions are still quoted against the SURVEY figures above (160 / 200 / 360 B per DOF), i.e.
# the extra plane counts as overhead, not as useful traffic.
PHYS = dict(gamma=1.4, mu=1e-3, prandtl=0.72, rgas=1.0)
CPU_REPS = 16          # RHS evaluations per process in one CPU sample (~10-15 s of CPU work)


def workload_name(n, workload="ns", species=3):
    E = 6 * n ** 3
    if workload == "multispecies":
        return (f"3D multi-species reactive Navier-Stokes DG RHS ({species} species, 1 Arrhenius step, C = {5 + species} fields; fused kernels "
                f"dgb_ms_flux + dgb_ms_div), Kuhn tets order {ORDER}, periodic {n}^3 box per GPU: {E} elements, "
                f"{E * NP} DOFs per GPU (BASELINE configs[4])")
    if workload == "euler":
        return (f"3D compressible Euler DG RHS, Kuhn tets order {ORDER}, periodic {n}^3 box per GPU: {E} elements, "
                f"{E * NP} DOFs per GPU (BASELINE configs[1])")
    return (f"3D compressible Navier-Stokes DG RHS (BR1, two derivative passes), Kuhn tets order {ORDER}, periodic "
            f"{n}^3 box per GPU: {E} elements, {E * NP} DOFs per GPU (BASELINE configs[2])")


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def state_for(nodes_shape, seed):
    """SURVEY.md §8d config c2 generator: rho~U[.9,1.1], u~U[-.1,.1]^3, p~U[.9,1.1]/gamma."""
    rng = np.random.default_rng(seed)
    E, Np = nodes_shape
    q = np.empty((DIM + 2, E, Np))
    q[0] = rng.uniform(0.9, 1.1, (E, Np))
    vel = rng.uniform(-0.1, 0.1, (DIM, E, Np))
    p = rng.uniform(0.9, 1.1, (E, Np)) / PHYS["gamma"]
    q[1] = p / (PHYS["gamma"] - 1.0) + 0.5 * q[0] * (vel ** 2).sum(axis=0)
    q[2:] = q[0] * vel
    return q


# {{{ clocks sampling (B200_PROFILING.md)

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=self.file, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.file.flush()
        self.file.seek(0)
        sm, mx, reasons, power = [], [], set(), []
        for line in self.file.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1])); mx.append(float(parts[2])); power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.file.name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        # "under load" = the upper half of the power samples
        order = np.argsort(power)
        load = [sm[i] for i in order[len(order) // 2:]]
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "power_w_max": float(max(power)), "samples": len(sm)}

# }}}


# {{{ CPU reference arm (oracle port = the reference's eager NumPy context, oracle/laze_port.py)

REF_DIR = os.path.join(ROOT, "baseline", "_ref")     # pip install --target of /root/reference/pkg


def reference_context():
    """(array context, kind): the UNMODIFIED reference's own eager context when `laze` is installed under
    baseline/_ref (it travels to the GPU box with the repository), else its restatement oracle/laze_port.py."""
    if os.path.isdir(os.path.join(REF_DIR, "laze")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import laze
            return laze.ArrayContext(mode="eager"), "reference"
        except Exception:
            pass
    from oracle.laze_port import NumpyArrayContext
    return NumpyArrayContext(), "port"


def _cpu_worker(args):
    n, reps, seed = args
    from paper_2512_17101_b200 import DGDiscretization, NavierStokesOperator, box_mesh
    actx, _ = reference_context()
    mesh = box_mesh((n,) * DIM, (-1.0,) * DIM, (1.0,) * DIM, periodic=(True,) * DIM)
    d = DGDiscretization(actx, mesh, ORDER)
    op = NavierStokesOperator(d, **PHYS)
    q = d.from_numpy(state_for((d.nelements, d.Np), seed))
    op.rhs(q)                                   # warm-up
    t0 = time.perf_counter()
    for _ in range(reps):
        op.rhs(q)
    return d.nelements * d.Np * reps, time.perf_counter() - t0


def cpu_throughput(cores: int, n: int, reps: int):
    """Aggregate DOF/s of `cores` independent processes, each evaluating the NS RHS `reps` times
    on its own periodic n^3 Kuhn mesh (halo exchange ignored: favours the CPU)."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    if cores == 1:
        results = [_cpu_worker((n, reps, 1))]
    else:
        with ctx.Pool(cores) as pool:
            results = pool.map(_cpu_worker, [(n, reps, 1 + k) for k in range(cores)])
    wall = time.perf_counter() - t0
    dofs = sum(r[0] for r in results)
    busy = max(r[1] for r in results)
    return dofs / busy / 1e9, dofs, busy, wall


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    n, reps = args.cpu_n, 1
    for _ in range(min(args.warmup, 1)):
        cpu_throughput(cores, n, reps)
    t0 = time.perf_counter()
    dofs = 0
    busy = 0.0
    for _ in range(args.steps):
        _, d, b, _ = cpu_throughput(cores, n, reps)
        dofs += d
        busy += b
    wall = time.perf_counter() - t0
    value = dofs / busy / 1e9
    kind = reference_context()[1]
    ctx_name = ("laze.ArrayContext(mode='eager') from baseline/_ref (the unmodified reference)" if kind == "reference"
                else "NumPy eager context (oracle/laze_port.py, the reference's restatement)")
    sample = (f"{cores} processes x NS p3 RHS on a periodic {n}^3 Kuhn mesh ({6 * n ** 3} elements, "
              f"{6 * n ** 3 * NP} DOFs each), {reps} evaluation(s) per step; {ctx_name}")
    line = {
        "impl": "reference", "metric": "3D Navier-Stokes DG RHS throughput", "value": value, "unit": "GDOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * busy / max(args.steps, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.n), "sample": sample},
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line))

# }}}


FP64_PEAK_TFLOPS = 37.15   # DMMA.8x8x4, registers only, measured on B200 at 1965 MHz (profiles/r01_fp64_peak.txt)


def fp64_ceiling(args, ndof, ms_step, hbm_frac, multi, euler, grad_form, world):
    """the FP64 ceiling next to the HBM roofline.  Lane-operations per DOF are the ISSUED
    FP64 work of the kernels (cost.py: tensor-core FMAs incl. padding + pointwise), so
    `frac` = the share of the measured FP64 datapath peak the path sustains; `min_frac` = its position under
    min(HBM roofline, FP64 ceiling)."""
    if multi or ORDER != 3 or DIM != 3:
        return None
    ops = 896.0 if euler else (1920.0 if grad_form else 1720.0)
    tflops = 2.0 * ops * ndof / (ms_step * 1e-3) / 1e12
    peak_gdofs = FP64_PEAK_TFLOPS * 1e12 / (2.0 * ops) / 1e9
    return {"fp64_lane_ops_per_dof": ops, "achieved": tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": tflops / FP64_PEAK_TFLOPS, "ceiling_gdofs_per_gpu": peak_gdofs,
            "peak_source": "measured DMMA register-only microbenchmark (profiles/r01_fp64_peak.txt)",
            "min_frac": max(hbm_frac, tflops / FP64_PEAK_TFLOPS),
            "note": "the path is FP64-bound: its distance to min(HBM roofline, FP64 ceiling) is the larger of the two fractions"}


def gpu_numa_cpus(device_index: int):
    """CPUs of the NUMA node the GPU hangs off (sysfs), or (None, node) when that cannot be determined."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(device_index)
        addr = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{addr}/numa_node") as fh:
            node = int(fh.read().strip())
        if node < 0:
            return None, node
        with open(f"/sys/devices/system/node/node{node}/cpulist") as fh:
            spec = fh.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        return (cpus or None), node
    except Exception:
        return None, None


def bind_to_gpu_numa_node(device_index: int):
    """Pinned staging buffers are first-touched by this process: run it on the CPUs next to the GPU so that
    host<->device copies do not cross the socket interconnect (the r01 driver box reached 58 GB/s for
    H2D + D2H together where the builder box reached 82 GB/s).  Returns the node or None."""
    cpus, node = gpu_numa_cpus(device_index)
    if cpus:
        try:
            os.sched_setaffinity(0, cpus)
            return node
        except OSError:
            return None
    return None


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2512_17101_b200 import B200ArrayContext, DGDiscretization, NavierStokesOperator, box_mesh
    from paper_2512_17101_b200.dofarray import DOFArray

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # DGB_BENCH_SHARE_GPU=1: dry run of the N>1 code path on a box with a single GPU (all ranks on cuda:0,
    # gloo with host-staged messages).  Its numbers mean nothing; the driver never sets it.
    share = os.environ.get("DGB_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    numa_node = bind_to_gpu_numa_node(local_rank)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            # NCCL's init lines (communicator, nranks, transports: NVLS / P2P) on stderr, for the record of an N-GPU run
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)

    actx = B200ArrayContext(device=local_rank)
    n = args.n
    t_setup = time.perf_counter()
    # weak scaling: every rank owns one periodic n^3 block of the same size (configs[2] per GPU)
    mesh = box_mesh((n,) * DIM, (-1.0,) * DIM, (1.0,) * DIM, periodic=(True,) * DIM)
    halo = None
    strong = args.scaling == "strong"
    if world > 1 and strong:
        # strong scaling (BASELINE configs[3]): ONE periodic n^3 box, recursive coordinate bisection into
        # `world` parts, interior-first renumbering; every rank builds the global mesh once (host, setup only)
        from paper_2512_17101_b200.dg.partition import interior_first, partition_elements, rank_mesh
        from paper_2512_17101_b200.dg.simplex import simplex_element
        from paper_2512_17101_b200.halo import HaloExchange, TorchCommunicator
        part = partition_elements(mesh, world)
        mesh, plan = interior_first(*rank_mesh(mesh, part, rank))
        halo = HaloExchange(actx, plan, TorchCommunicator(), simplex_element(DIM, ORDER).Np, transport=args.halo)
    elif world > 1:
        from paper_2512_17101_b200.halo import ring_slab_halo
        mesh, halo = ring_slab_halo(actx, mesh, n, rank, world, ORDER, transport=args.halo)
    d = DGDiscretization(actx, mesh, ORDER, ghost_elements=0 if halo is None else halo.nghost)
    euler = args.workload == "euler"
    multi = args.workload == "multispecies"
    if multi:
        from paper_2512_17101_b200 import Mixture, MultispeciesOperator
        mixtures = {2: dict(R=(1.0, 0.8), cv=(2.5, 2.0), h0=(0.5, -0.5), reaction=(0, 1)), 3: {},
                    4: dict(R=(1.0, 0.8, 1.2, 0.9), cv=(2.5, 2.0, 3.0, 2.2), h0=(0.5, -0.5, 0.0, 0.1), reaction=(0, 3))}
        op = MultispeciesOperator(d, Mixture(**mixtures[args.species]))
    elif euler:
        from paper_2512_17101_b200 import EulerOperator
        op = EulerOperator(d, gamma=PHYS["gamma"])
    else:
        op = NavierStokesOperator(d, **PHYS)
    E, Np = d.nelements, d.Np
    ndof = E * Np
    ncomp = op.ncomp if multi else DIM + 2
    q_host = actx.pinned_empty((ncomp, E, Np))
    if multi:       # smooth seeded state: rho, u, T perturbed, the mass fractions
        rng = np.random.default_rng(20251217 + rank)
        Y = rng.uniform(0.2, 0.4, (args.species, E, Np)); Y /= Y.sum(axis=0)
        q_host[...] = op.state_from_primitive(rng.uniform(0.9, 1.1, (E, Np)), rng.uniform(-0.1, 0.1, (DIM, E, Np)),
                                              rng.uniform(0.9, 1.1, (E, Np)), Y)
    else:
        q_host[...] = state_for((E, Np), 20251217 + rank)
    out_host = actx.pinned_empty((ncomp, E, Np))
    q = DOFArray(actx, actx.from_numpy(q_host))
    actx.synchronize()
    t_setup = time.perf_counter() - t_setup

    grad_form = args.form == "grad" and not euler and not multi

    def rhs_step(qarr):
        if halo is None:
            return op.rhs_grad_form(qarr) if grad_form else op.rhs(qarr)
        if euler:
            return halo.euler_rhs(op, qarr)
        if multi:
            return halo.ms_rhs(op, qarr)
        return halo.ns_rhs_grad_form(op, qarr) if grad_form else halo.ns_rhs(op, qarr)

    # ---- device-resident measurement --------------------------------------------------------
    stream = actx.stream
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]

    def one_step(marks=None):
        """One RHS evaluation; `marks` = three events recorded before pass 1, between the passes and
        after pass 2.  Warm-up and timed steps run this same code, so the caching allocator sees the
        same request pattern and never calls cudaMalloc inside the timed region."""
        rec = (lambda i: marks[i].record(stream)) if marks is not None else (lambda i: None)
        if multi and halo is None:
            rec(0)
            T = op.flux(q, None)
            rec(1)
            op.div(q, T)
            rec(2)
        elif halo is None and not euler and grad_form:
            rec(0)
            gq = op.grad(q)
            rec(1)
            op._f(q.data, gq.data, *op._common(), op.phys)
            rec(2)
        elif halo is None and not euler:
            rec(0)
            T = op.flux(q)
            rec(1)
            op._div(q.data, T, *op._div_args())
            rec(2)
        elif halo is None:
            rec(0)
            rec(1)
            op.rhs(q)
            rec(2)
        else:
            rhs_step(q)

    for _ in range(max(args.warmup, 3)):
        one_step()
    actx.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    launches0 = actx.launch_count
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(K):
        one_step(ev[k])
    stop.record(stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    launches = actx.launch_count - launches0
    ms_total = start.elapsed_time(stop)
    ms_step = ms_total / K
    if world > 1:
        t = torch.tensor([ms_step], device="cpu" if share else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    total_dofs = ndof
    if world > 1:
        td = torch.tensor([float(ndof)], device="cpu" if share else "cuda", dtype=torch.float64)
        dist.all_reduce(td, op=dist.ReduceOp.SUM)
        total_dofs = int(td.item())
    value = total_dofs / (ms_step * 1e-3) / 1e9

    peak, peak_src = measured_peaks()
    roofline = None
    if halo is None:
        ms_grad = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
        ms_div = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
        if multi:       # the NS split of the 72 C bytes: pass 1 reads q, writes d C planes; pass 2 reads both, writes rhs
            dom = ((f"k_nsdiv8<C={ncomp}> (dgb_ms_div)", ms_div, 40.0 * ncomp) if ms_div >= ms_grad else
                   (f"k_nsflux3<C={ncomp}> (dgb_ms_flux)", ms_grad, 32.0 * ncomp))
        elif euler:
            dom = ("k_euler4 (fused Euler RHS)", ms_div, 80.0)
        else:
            names = ("k_rhs3<viscous> (flux + divergence pass)", "k_grad3 (BR1 gradient pass)") if grad_form else \
                    ("k_nsdiv8 (divergence + face pass, TMA-staged)", "k_nsflux3 (BR1 gradient + flux pass)")
            dom = (names[0], ms_div, B_ALG_DIV) if ms_div >= ms_grad else (names[1], ms_grad, B_ALG_GRAD)
        achieved = ndof * dom[2] / (dom[1] * 1e-3) / 1e9
        traffic = None
        traffic_source = None
        tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
        if not os.path.exists(tpath):
            tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as fh:
                tj = json.load(fh)
            if tj.get("n") == n and ORDER == 3 and euler and "k_euler4" in tj:
                traffic = tj["k_euler4"]["dram_read_bytes"] + tj["k_euler4"]["dram_write_bytes"]
            if tj.get("n") == n and ORDER == 3 and not euler:      # ncu capture of exactly this workload (bytes per launch)
                if grad_form:
                    key = "k_rhs3_viscous" if ms_div >= ms_grad else "k_grad3"
                else:
                    key = "k_nsdiv8" if ms_div >= ms_grad else "k_nsflux3"
                if key in tj:
                    traffic = tj[key]["dram_read_bytes"] + tj[key]["dram_write_bytes"]
        if traffic is not None:
            traffic_source = (f"static: dram__bytes_read.sum + dram__bytes_write.sum of one `ncu --set full` capture of this "
                              f"kernel on this workload ({os.path.relpath(tpath, ROOT)}); not measured in this run")
        per_step = [e[0].elapsed_time(e[2]) for e in ev]
        roofline = {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_source, "peak_source": peak_src,
                    "algorithmic_bytes_per_dof": dom[2], "ms_per_launch": dom[1],
                    "ms_grad_pass": ms_grad, "ms_div_pass": ms_div,
                    "ms_step_min_median_max": [float(np.min(per_step)), float(np.median(per_step)),
                                               float(np.max(per_step))],
                    "value_at_median_step": ndof / (float(np.median(per_step)) * 1e-3) / 1e9}
    b_alg = 72.0 * ncomp if multi else (80.0 if euler else B_ALG_RHS)      # (3C + 2Cd) * 8 = 72 C for NS-type two-pass schemes
    rhs_gbs = ndof * b_alg / (ms_step * 1e-3) / 1e9
    if roofline is None:
        # partitioned run: the passes interleave with the halo exchange, so the roofline entry is the
        # whole right-hand side of one rank (both kernels + exchange) against one GPU's HBM peak
        roofline = {"bound": "hbm", "kernel": "whole RHS of one rank (both passes + halo exchange)",
                    "achieved": rhs_gbs, "peak": peak, "unit": "GB/s", "frac": rhs_gbs / peak, "traffic": None,
                    "peak_source": peak_src, "algorithmic_bytes_per_dof": b_alg, "ms_per_launch": ms_step}

    # ---- end to end through the public API with host buffers ---------------------------------
    e2e = None
    if not args.no_e2e:
        Ke = max(1, min(K, args.e2e_steps))
        for _ in range(2):
            qd = DOFArray(actx, actx.from_numpy(q_host))
            actx.to_numpy(rhs_step(qd).data, out=out_host)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # Pipelined like a streaming user would: the H2D copy of step k+1 (upload stream), the compute of
        # step k (compute stream) and the D2H of step k-1 (download stream) overlap.  Every step still uploads its full input from pinned
        # host memory and downloads its full result; both are inside the timed region.
        # two device input buffers, ping-ponged (a streaming caller allocates them once)
        dev_in = [actx.empty(q_host.shape), actx.empty(q_host.shape)]

        def pipeline(nsteps):
            """nsteps streamed evaluations; returns the events bracketing them on the compute stream."""
            read_done = [None, None]
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            actx.copy_stream.wait_event(s0)
            nxt = actx.from_numpy_async(q_host, out=dev_in[0])
            d2h_done = None
            for k in range(nsteps):
                cur = actx.wait_for(nxt)
                res = rhs_step(DOFArray(actx, cur)).data
                read_done[k % 2] = torch.cuda.Event()
                read_done[k % 2].record(stream)                       # step k no longer reads dev_in[k % 2]
                if k + 1 < nsteps:                                    # H2D of step k+1 into the other buffer
                    nxt = actx.from_numpy_async(q_host, after=read_done[(k + 1) % 2], out=dev_in[(k + 1) % 2])
                d2h_done = actx.to_numpy_async(res, out_host)         # D2H of step k's result (download stream)
            stream.wait_event(d2h_done)                               # the last result is on the host
            s1.record(stream)
            torch.cuda.synchronize()
            return s0, s1

        # warm-up THROUGH THE SAME PIPELINE: the result blocks are held by the download stream while they are
        # copied out, so the caching allocator needs a third and fourth result block before its request pattern
        # repeats; a cudaMalloc inside the timed region synchronises the device and serialises the copies
        # (r01: 138 ms per step on the driver box where the link does 85 ms)
        pipeline(4)
        s0, s1 = pipeline(Ke)
        ms_e2e = s0.elapsed_time(s1) / Ke
        if world > 1:
            t = torch.tensor([ms_e2e], device="cpu" if share else "cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
        e2e = {"value": total_dofs / (ms_e2e * 1e-3) / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": int(q_host.nbytes), "d2h_bytes_per_step": int(out_host.nbytes),
               "ms_per_step": ms_e2e, "steps": Ke, "checksum": float(out_host[0, 0, 0])}

    # ---- CPU baseline beside it (rank 0, N=1 only, bounded sample) ---------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        v, dofs, busy, wall = cpu_throughput(cores, args.cpu_n, CPU_REPS)
        kind = reference_context()[1]
        cpu = {"value": v, "unit": "GDOF/s", "cores": cores, "kind": kind,
               "sample": f"{cores} processes x {CPU_REPS} NS p3 RHS on a periodic {args.cpu_n}^3 Kuhn mesh "
                         f"({6 * args.cpu_n ** 3 * NP} DOFs each), "
                         + ("laze.ArrayContext(mode='eager') from baseline/_ref (the unmodified reference); " if kind == "reference"
                            else "oracle/laze_port.py NumPy eager context; ") + f"{busy:.1f} s busy"}

    if rank == 0:
        line = {
            "metric": ("3D multispecies reactive Navier-Stokes DG RHS throughput" if multi else
                       "3D Navier-Stokes DG RHS throughput" if not euler else "3D Euler DG RHS throughput"),
            "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": K, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if (strong and world > 1) else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"numa_node_bound": numa_node,
                       "workload": workload_name(n, args.workload, args.species) if not (strong and world > 1) else
                       workload_name(n, args.workload, args.species).replace("per GPU", "in total"),
                       "elements_per_gpu": E, "dofs_per_gpu": ndof, "order": ORDER, "dim": DIM,
                       "l2_policy": "inputs larger than L2 (q 4.0 GB, grad q 12 GB per GPU vs 126 MB L2)"
                       if ndof * 40 > 126e6 * 4 else "inputs comparable to L2: reduced size, not the headline config",
                       "arrangement": ("flux (dg_ms_flux + dg_ms_div), fused" if multi else
                                       "euler single pass" if euler else
                                       "gradient (dg_ns_grad + dg_ns_rhs)" if grad_form else "flux (dg_ns_flux + dg_ns_div)"),
                       "parallelism": (f"mesh partition x{world}, " + ("NCCL face-halo exchange" if args.halo == "nccl" else
                                       "peer-memory face-halo exchange (pack kernel stores over NVLink)"))
                       if world > 1 else "single GPU",
                       "setup_s": t_setup},
            "roofline": roofline,
            "rhs_roofline": {"bound": "hbm", "achieved": rhs_gbs, "peak": peak, "unit": "GB/s",
                             "frac": rhs_gbs / peak, "algorithmic_bytes_per_dof": b_alg,
                             "peak_source": peak_src},
            "fp64_ceiling": fp64_ceiling(args, ndof, ms_step, rhs_gbs / peak, multi, euler, grad_form, world),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
    if world > 1:
        if halo is not None:
            halo.close()
        dist.destroy_process_group()
    if rank == 0:
        sys.stdout.flush()
        print(json.dumps(line), flush=True)          # last line of stdout, after NCCL's own log lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--cells", dest="n", type=int, default=94, help="cells per axis per GPU (94 -> 4,983,504 elements, 99.67M DOFs); under torchrun spell it --cells "
                         "(argparse in torch.distributed.run rejects `--n` as an ambiguous abbreviation of its own options)")
    ap.add_argument("--cpu-n", type=int, default=10, help="cells per axis of each CPU-baseline sample mesh")
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="streamed end-to-end evaluations timed (pipeline fill and drain included); at most --steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--order", type=int, default=3, help="polynomial order (headline: 3)")
    ap.add_argument("--form", default="flux", choices=["flux", "grad"],
                    help="arrangement of the NS scheme: flux (default; dg_ns_flux + dg_ns_div) or grad (dg_ns_grad + dg_ns_rhs)")
    ap.add_argument("--halo", default="nccl", choices=["nccl", "peer"],
                    help="N>1 halo transport: nccl = grouped send/recv on a communication stream (default); peer = the "
                         "pack kernel stores into the neighbour's ghost array through CUDA-IPC peer memory (NVLink)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = one n^3 box per GPU in a ring (default); strong = one n^3 box partitioned over the GPUs")
    ap.add_argument("--species", type=int, default=3, choices=[2, 3, 4], help="--workload multispecies: species count")
    ap.add_argument("--workload", default="ns", choices=["ns", "euler", "multispecies"],
                    help="ns = BASELINE configs[2] (headline); euler = configs[1] (3D Euler, read q + write rhs = 80 B/DOF)")
    args = ap.parse_args()
    global ORDER, NP
    ORDER = args.order
    NP = (ORDER + 1) * (ORDER + 2) * (ORDER + 3) // 6
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
