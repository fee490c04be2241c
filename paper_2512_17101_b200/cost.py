"""Cost accounting of the hand-fused path.

The reference reports, per graph, how many materialised arrays an evaluation reads (R), writes (W)
and how many node evaluations it performs (C) -- ``cost_report``
(/root/reference/pkg/src/laze/graph_passes.py:744-815).  The fused kernels have no graph, so the
same three quantities are stated per kernel in physical units: HBM bytes read / written per
evaluation and FP64 lane-operations issued (1 FMA = 1 lane-operation; DMMA counted with its tile
padding).  ``bytes_*`` are *compulsory* traffic of the arrays each kernel is handed -- what
``bench.py`` divides by the measured time, and what ``tests/test_cabi_and_host.py`` checks against
the DRAM bytes ncu measured (profiles/r01_traffic.json) so the algorithmic-bytes claim stays
machine-checkable.
"""
from __future__ import annotations

from dataclasses import dataclass

from .dg.simplex import simplex_element


@dataclass(frozen=True)
class KernelCost:
    kernel: str
    bytes_read: int          # field arrays + geometry/connectivity streamed once
    bytes_written: int
    bytes_field_read: int    # field arrays only (the SURVEY §8d accounting excludes geometry)
    bytes_field_written: int
    fp64_dmma: int           # lane-operations issued on the tensor-core path (incl. tile padding)
    fp64_pointwise: int      # estimate of the pointwise / combination work

    @property
    def bytes_total(self) -> int:
        return self.bytes_read + self.bytes_written

    def as_text(self) -> str:
        return (f"{self.kernel}: R:{self.bytes_read} W:{self.bytes_written} "
                f"C:{self.fp64_dmma + self.fp64_pointwise} (dmma {self.fp64_dmma})")


def _ceil(x, m):
    return (x + m - 1) // m * m


def cost_report(dim: int, order: int, nelements: int, equations: str = "ns", arrangement: str = "flux"):
    """Per-kernel costs of one right-hand-side evaluation on ``nelements`` simplices."""
    el = simplex_element(dim, order)
    C, Np, Nf, Nfp = dim + 2, el.Np, el.Nf, el.Nfp
    E, N = nelements, nelements * el.Np
    KW = 3 if dim == 3 else 4
    rows = _ceil(Np, 8)                       # output-node padding of every W
    cols = _ceil(C * KW, 8) / (C * KW)        # column-tile padding
    npk, nfpk, kf = _ceil(Np, 4), _ceil(Nfp, 4), _ceil(Nf * Nfp, 4)
    geo_grad = E * 8 * (dim * dim + dim * Nf + 2 * Nf + 1)      # drdx, normals, fscale, conn, jac
    geo_div = E * 8 * (2 * Nf + 1)                              # sj, conn, rj
    f = lambda planes: planes * N * 8

    def dmma(k_per_column):                    # lane-ops per RHS for a contraction of length k per column
        return int(round(E * C * rows * k_per_column * cols))

    out = []
    if equations == "euler":
        out.append(KernelCost("k_euler4", f(C) + geo_grad, f(C), f(C), f(C),
                              dmma(dim * npk + kf), N * 230))
    elif arrangement == "flux":
        npl = (dim + 1) * C + 1                 # dim + 1 plane groups (the last is the sum of the others) + wave speed
        gmap = E * 4 * Nf * Nfp                 # 32-bit gather map
        out.append(KernelCost("k_nsflux3", f(C) + geo_grad + gmap, f(npl), f(C), f(npl),
                              dmma(dim * npk + Nf * nfpk), N * (C * (dim * dim + dim) * rows // Np + 245)))
        # pass 2 streams q, the dim*C volume planes and the wave speed (TMA boxes) and reaches the sum planes only
        # through the neighbour gathers: every plane is read from HBM once
        out.append(KernelCost("k_nsdiv8", f(C) + f(npl) + geo_div + gmap, f(C), f(C) + f(npl), f(C),
                              dmma(dim * npk + kf), N * 30))
    else:
        out.append(KernelCost("k_grad3", f(C) + geo_grad, f(dim * C), f(C), f(dim * C),
                              dmma(dim * npk + Nf * nfpk), N * 150))
        out.append(KernelCost("k_rhs3<viscous>", f(C) + f(dim * C) + geo_grad, f(C), f(C) + f(dim * C), f(C),
                              dmma(dim * npk + kf), N * 500))
    return out
