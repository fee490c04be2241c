"""Build tuning variants of libdgb200.so (compile-time knobs of the flux-arrangement kernels) and,
with --run, bench each one on the GPU (A/B numbers for profiles/).

    python scripts/ab_variants.py --build            # here (CPU box): nvcc each variant
    python scripts/ab_variants.py --run --n 64       # on the GPU box: one JSON line per variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PKG = os.path.join(ROOT, "paper_2512_17101_b200")

VARIANTS = {
    "timing": ["DGB_PHASE_TIMING=1"],                 # scripts/phase_timing_flux.py
    "base": [],
    "tcs": ["DGB_FLUX_T_STCS=1"],
    "tcs_ocs": ["DGB_FLUX_T_STCS=1", "DGB_STREAMING_STORES=1"],
    "nopb": ["DGB_DIV8_PLANEBASE=0"],
    "roll2": ["DGB_DIV8_ROLLED=1"],
    "roll3": ["DGB_DIV8_ROLLED=1", "DGB_DIV8_NB=3"],
    "roll1": ["DGB_DIV8_ROLLED=1", "DGB_DIV8_NB=1"],
    "pwu4": ["DGB_FLUX_PW_UNROLL=4"],
    "epwu1": ["DGB_EULER_PW_UNROLL=1"],
    "mt": ["DGB_FLUX_MT=1"],
    "mtu": ["DGB_FLUX_MT=2"],
    "mtu_w8": ["DGB_FLUX_MT=2", "DGB_FLUX_WARPS=8"],
    "mt_w8": ["DGB_FLUX_MT=1", "DGB_FLUX_WARPS=8"],
    "flux_w14": ["DGB_FLUX_WARPS=16"],
    "stcs": ["DGB_STREAMING_STORES=1"],
    "tk2": ["DGB_TICKET_BLOCKS=2"],
    "euler_w8": ["DGB_EULER_WARPS=8"],
    "div_w12_nb1": ["DGB_DIV_WARPS=12", "DGB_DIV_NB=1"],
    "f_w11": ["DGB_FLUX_WARPS=11"],
    "f_w10": ["DGB_FLUX_WARPS=10"],
    "f_w8": ["DGB_FLUX_WARPS=8"],
    "d12_nb2": ["DGB_DIV8_WARPS=12", "DGB_DIV8_NB=2"],
    "d12_nb2_cg": ["DGB_DIV8_WARPS=12", "DGB_DIV8_NB=2", "DGB_GATHER_LD=1"],
    "d12_nb4_cg": ["DGB_DIV8_WARPS=12", "DGB_DIV8_NB=4", "DGB_GATHER_LD=1"],
    "d10_nb2": ["DGB_DIV8_WARPS=10", "DGB_DIV8_NB=2"],
    "nb2": ["DGB_DIV8_NB=2"],
    "nb3": ["DGB_DIV8_NB=3"],
    "noearly": ["DGB_DIV8_EARLY=0"],
    "nosq": ["DGB_FLUX_SINGLEQ=0"],
    "agg": ["DGB_TICKET_NOAGG=0"],
    "k3": ["DGB_DIV_KERNEL_DEFAULT=3"],
    "w8": ["DGB_DIV8_WARPS=8"],
    "w8_nb1": ["DGB_DIV8_WARPS=8", "DGB_DIV_NB=1"],
    "w8_nb4": ["DGB_DIV8_WARPS=8", "DGB_DIV_NB=4"],
    "w12": ["DGB_DIV8_WARPS=12"],
    "w12_cg": ["DGB_DIV8_WARPS=12", "DGB_GATHER_LD=1"],
    "x_local": ["DGB_EXP_LOCALGATHER=1"],
    "x_nomma": ["DGB_EXP_NOMMA=1"],
    "x_noface": ["DGB_EXP_NOFACE=1"],
    "ss_w8": ["DGB_DIV_SINGLE_SMALL=1"],
    "ss_w9": ["DGB_DIV_SINGLE_SMALL=1", "DGB_DIV_WARPS=9"],
    "ss_w10": ["DGB_DIV_SINGLE_SMALL=1", "DGB_DIV_WARPS=10"],
    "ss_w10_nb1": ["DGB_DIV_SINGLE_SMALL=1", "DGB_DIV_WARPS=10", "DGB_DIV_NB=1"],
    "ss_w12": ["DGB_DIV_SINGLE_SMALL=1", "DGB_DIV_WARPS=12"],
    "ss_w12_nb1": ["DGB_DIV_SINGLE_SMALL=1", "DGB_DIV_WARPS=12", "DGB_DIV_NB=1"],
}


def lib(name):
    return os.path.join(PKG, f"libdgb200_{name}.so")


def main():
    names = [a for a in sys.argv[1:] if a in VARIANTS] or list(VARIANTS)
    kernels = {}
    if "--build" in sys.argv:
        # only dgb_nsflux.cu depends on the knobs: compile the other translation units once
        from paper_2512_17101_b200.csrc.build import FLAGS, HERE
        cflags = [f for f in FLAGS if f != "-shared"] + (["-DDGB_ONLY_3D_P3"] if "--p3only" in sys.argv else [])
        objs = []
        for src in ("dgb200.cu", "dgb_arrayops.cu", "dgb_msflux.cu", "dgb_msflux2.cu", "dgb_msflux3.cu", "dgb_msflux4.cu"):
            obj = os.path.join("/tmp", src.replace(".cu", ".o"))
            if not os.path.exists(obj) or os.path.getmtime(obj) < max(
                    os.path.getmtime(os.path.join(HERE, f)) for f in os.listdir(HERE) if f.endswith((".cu", ".cuh", ".h"))):
                subprocess.run(["nvcc"] + cflags + ["-c", src, "-o", obj], cwd=HERE, check=True)
            objs.append(obj)
        for name in names:
            obj = f"/tmp/dgb_nsflux_{name}.o"
            subprocess.run(["nvcc"] + cflags + [f"-D{d}" for d in VARIANTS[name]] + ["-c", "dgb_nsflux.cu", "-o", obj],
                           cwd=HERE, check=True)
            subprocess.run(["nvcc", "-shared", "-o", lib(name), obj] + objs, cwd=HERE, check=True)
            print("built", lib(name), flush=True)
    if "--run" in sys.argv:
        n = sys.argv[sys.argv.index("--n") + 1] if "--n" in sys.argv else "64"
        for name, kern in [(nm, k) for nm in names for k in kernels.get(nm, [None])]:
            env = dict(os.environ, DGB_LIB=lib(name))
            if kern:
                env["DGB_DIV_KERNEL"] = kern
                name = f"{name}:k_nsdiv{kern}"
            extra = sys.argv[sys.argv.index("--bench-args") + 1].split() if "--bench-args" in sys.argv else []
            res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-e2e", "--no-cpu", "--n", n,
                                  "--steps", "10"] + extra, env=env, capture_output=True, text=True)
            try:
                d = json.loads(res.stdout.strip().splitlines()[-1])
                r = d["roofline"]
                print(f"{name:18s} n={n} {d['value']:.3f} GDOF/s  pass1 {r['ms_grad_pass']:.3f} ms  pass2 {r['ms_div_pass']:.3f} ms"
                      f"  step min/med/max {r['ms_step_min_median_max']}", flush=True)
            except Exception:
                print(name, "FAILED", res.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
