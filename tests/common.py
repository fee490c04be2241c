"""Shared builders for the parity tests: seeded states and discretisations."""
import numpy as np

from paper_2512_17101_b200.dg.mesh import box_mesh
from paper_2512_17101_b200.discretization import BC_FARFIELD, BC_WALL, DGDiscretization


def random_state(dim, E, Np, seed=20251217, gamma=1.4):
    """SURVEY.md §8d config c2 generator: smooth state + seeded perturbation."""
    rng = np.random.default_rng(seed)
    q = np.empty((dim + 2, E, Np))
    q[0] = rng.uniform(0.9, 1.1, (E, Np))
    q[2:] = rng.uniform(-0.1, 0.1, (dim, E, Np))
    p = rng.uniform(0.9, 1.1, (E, Np)) / gamma
    q[1] = p / (gamma - 1.0) + 0.5 * (q[2:] ** 2).sum(axis=0) / q[0]
    q[2:] *= q[0]
    return q


def smooth_state(nodes, gamma=1.4):
    """Acoustic-pulse-like smooth state (config c1) on arbitrary nodes ``(dim, E, Np)``."""
    dim = nodes.shape[0]
    r2 = (nodes ** 2).sum(axis=0)
    rho = 1.0 + 0.1 * np.exp(-r2 / (2 * 0.3 ** 2))
    p = (1.0 / gamma) * (1.0 + 0.1 * np.exp(-r2 / (2 * 0.3 ** 2)))
    vel = [0.1 * np.sin(np.pi * nodes[(i + 1) % dim]) for i in range(dim)]
    q = np.empty((dim + 2,) + r2.shape)
    q[0] = rho
    for i in range(dim):
        q[2 + i] = rho * vel[i]
    q[1] = p / (gamma - 1.0) + 0.5 * rho * sum(v * v for v in vel)
    return q


BC_CASES = {
    "periodic": (True, None),
    "farfield": (False, "far"),
    "mixed": (False, "mixed"),
}


def make_dcoll(actx, dim, order, n, bc="periodic", lo=-1.0, hi=1.0):
    periodic, kind = BC_CASES[bc]
    mesh = box_mesh((n,) * dim, (lo,) * dim, (hi,) * dim, periodic=(periodic,) * dim)
    if kind is None:
        bc_map = None
    elif kind == "far":
        bc_map = {k: BC_FARFIELD for k in range(1, 2 * dim + 1)}
    else:
        bc_map = {k: (BC_WALL if k % 2 else BC_FARFIELD) for k in range(1, 2 * dim + 1)}
    return DGDiscretization(actx, mesh, order, bc_map=bc_map)


FARFIELD = {2: np.array([1.05, 2.6, 0.21, -0.1]), 3: np.array([1.05, 2.6, 0.21, -0.1, 0.05])}
