"""Reference-simplex nodal DG building blocks (setup time only, NumPy, FP64).

Nothing in the reference (`laze`) defines a DG discretisation: the paper
only says the operators are "tensor contractions of reference matrices with nodal data"
(/root/reference/PAPER.md:1738-1739).  The choices made here are therefore this
repository's own and are documented in DESIGN.md:

* biunit reference simplex, vertices ``v0=(-1,..,-1)``, ``v_k = v0 + 2 e_k``;
* face ``f`` is the face opposite vertex ``f`` (barycentric ``lambda_f == 0``);
* nodes: barycentric GLL blend ``lambda_a = g(i_a) / sum_b g(i_b)`` over the multi-indices
  ``|i| = p`` (``g`` = Gauss-Lobatto-Legendre points on [0,1]); symmetric under every
  vertex permutation, GLL on every edge, and the face nodes of the d-simplex are the node
  set of the (d-1)-simplex, which is what makes conforming face matching exact;
* orthonormal Proriol-Koornwinder-Dubiner basis for the Vandermonde matrices.

Matrices produced (``Np`` volume nodes, ``Nfp`` nodes per face, ``Nf = d+1`` faces):

``D[r]``      ``(d, Np, Np)``   strong reference derivative  ``D_r = V_r V^-1``
``Sw[r]``     ``(d, Np, Np)``   weak reference derivative    ``M^-1 D_r^T M``
``lift``      ``(Np, Nf*Nfp)``  ``M^-1 E`` with ``E`` the face mass matrices
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from functools import lru_cache

import numpy as np


# {{{ 1D building blocks

def gll_points(p: int) -> np.ndarray:
    """p+1 Gauss-Lobatto-Legendre points on [-1, 1] (ascending)."""
    if p == 0:
        return np.array([0.0])
    if p == 1:
        return np.array([-1.0, 1.0])
    leg = np.polynomial.legendre.Legendre.basis(p)
    interior = np.sort(leg.deriv().roots().real)
    # polish with Newton on P'_p
    d1, d2 = leg.deriv(), leg.deriv(2)
    for _ in range(3):
        interior = interior - d1(interior) / d2(interior)
    x = np.concatenate([[-1.0], interior, [1.0]])
    return 0.5 * (x - x[::-1])  # enforce exact antisymmetry


def jacobi_p(x: np.ndarray, alpha: float, beta: float, n: int) -> np.ndarray:
    """Orthonormal Jacobi polynomial P_n^{(alpha,beta)}(x) (three-term recurrence)."""
    from math import gamma
    x = np.asarray(x, dtype=np.float64)
    g0 = (2.0 ** (alpha + beta + 1) / (alpha + beta + 1)
          * gamma(alpha + 1) * gamma(beta + 1) / gamma(alpha + beta + 1))
    p0 = np.full_like(x, 1.0 / np.sqrt(g0))
    if n == 0:
        return p0
    g1 = (alpha + 1) * (beta + 1) / (alpha + beta + 3) * g0
    p1 = ((alpha + beta + 2) * x / 2 + (alpha - beta) / 2) / np.sqrt(g1)
    if n == 1:
        return p1
    aold = 2.0 / (2 + alpha + beta) * np.sqrt((alpha + 1) * (beta + 1) / (alpha + beta + 3))
    for i in range(1, n):
        h1 = 2 * i + alpha + beta
        anew = 2.0 / (h1 + 2) * np.sqrt((i + 1) * (i + 1 + alpha + beta) * (i + 1 + alpha)
                                        * (i + 1 + beta) / (h1 + 1) / (h1 + 3))
        bnew = -(alpha ** 2 - beta ** 2) / h1 / (h1 + 2)
        p0, p1 = p1, (-aold * p0 + (x - bnew) * p1) / anew
        aold = anew
    return p1


def grad_jacobi_p(x: np.ndarray, alpha: float, beta: float, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros_like(np.asarray(x, dtype=np.float64))
    return np.sqrt(n * (n + alpha + beta + 1)) * jacobi_p(x, alpha + 1, beta + 1, n - 1)

# }}}


# {{{ orthonormal simplex bases and their gradients

def _basis_1d(rst, idx):
    (i,) = idx
    return jacobi_p(rst[0], 0, 0, i)


def _grad_basis_1d(rst, idx):
    (i,) = idx
    return (grad_jacobi_p(rst[0], 0, 0, i),)


def _rs_to_ab(r, s):
    a = np.where(np.abs(s - 1.0) > 1e-14, 2 * (1 + r) / np.where(np.abs(s - 1.0) > 1e-14, 1 - s, 1.0) - 1, -1.0)
    return a, s


def _basis_2d(rst, idx):
    i, j = idx
    a, b = _rs_to_ab(rst[0], rst[1])
    return np.sqrt(2.0) * jacobi_p(a, 0, 0, i) * jacobi_p(b, 2 * i + 1, 0, j) * (1 - b) ** i


def _grad_basis_2d(rst, idx):
    i, j = idx
    a, b = _rs_to_ab(rst[0], rst[1])
    fa, dfa = jacobi_p(a, 0, 0, i), grad_jacobi_p(a, 0, 0, i)
    gb, dgb = jacobi_p(b, 2 * i + 1, 0, j), grad_jacobi_p(b, 2 * i + 1, 0, j)
    dr = dfa * gb
    if i > 0:
        dr = dr * (0.5 * (1 - b)) ** (i - 1)
    ds = dfa * (gb * (0.5 * (1 + a)))
    if i > 0:
        ds = ds * (0.5 * (1 - b)) ** (i - 1)
    tmp = dgb * (0.5 * (1 - b)) ** i
    if i > 0:
        tmp = tmp - 0.5 * i * gb * (0.5 * (1 - b)) ** (i - 1)
    ds = ds + fa * tmp
    scale = 2.0 ** (i + 0.5)
    return dr * scale, ds * scale


def _rst_to_abc(r, s, t):
    den = -s - t
    ok = np.abs(den) > 1e-14
    a = np.where(ok, 2 * (1 + r) / np.where(ok, den, 1.0) - 1, -1.0)
    ok2 = np.abs(1 - t) > 1e-14
    b = np.where(ok2, 2 * (1 + s) / np.where(ok2, 1 - t, 1.0) - 1, -1.0)
    return a, b, t


def _basis_3d(rst, idx):
    i, j, k = idx
    a, b, c = _rst_to_abc(*rst)
    return (2 * np.sqrt(2.0) * jacobi_p(a, 0, 0, i) * jacobi_p(b, 2 * i + 1, 0, j) * (1 - b) ** i
            * jacobi_p(c, 2 * (i + j) + 2, 0, k) * (1 - c) ** (i + j))


def _grad_basis_3d(rst, idx):
    i, j, k = idx
    a, b, c = _rst_to_abc(*rst)
    fa, dfa = jacobi_p(a, 0, 0, i), grad_jacobi_p(a, 0, 0, i)
    gb, dgb = jacobi_p(b, 2 * i + 1, 0, j), grad_jacobi_p(b, 2 * i + 1, 0, j)
    hc, dhc = jacobi_p(c, 2 * (i + j) + 2, 0, k), grad_jacobi_p(c, 2 * (i + j) + 2, 0, k)
    hb = 0.5 * (1 - b)
    hcc = 0.5 * (1 - c)

    dr = dfa * (gb * hc)
    if i > 0:
        dr = dr * hb ** (i - 1)
    if i + j > 0:
        dr = dr * hcc ** (i + j - 1)

    ds = 0.5 * (1 + a) * dr
    tmp = dgb * hb ** i
    if i > 0:
        tmp = tmp + (-0.5 * i) * (gb * hb ** (i - 1))
    if i + j > 0:
        tmp = tmp * hcc ** (i + j - 1)
    tmp = fa * (tmp * hc)
    ds = ds + tmp

    dt = 0.5 * (1 + a) * dr + 0.5 * (1 + b) * tmp
    tmp = dhc * hcc ** (i + j)
    if i + j > 0:
        tmp = tmp - 0.5 * (i + j) * (hc * hcc ** (i + j - 1))
    tmp = fa * (gb * tmp)
    tmp = tmp * hb ** i
    dt = dt + tmp

    scale = 2.0 ** (2 * i + j + 1.5)
    return dr * scale, ds * scale, dt * scale


_BASIS = {1: _basis_1d, 2: _basis_2d, 3: _basis_3d}
_GRAD_BASIS = {1: _grad_basis_1d, 2: _grad_basis_2d, 3: _grad_basis_3d}


def mode_ids(dim: int, p: int) -> list[tuple[int, ...]]:
    return [idx for idx in itertools.product(range(p + 1), repeat=dim) if sum(idx) <= p]


def vandermonde(dim: int, p: int, rst: np.ndarray) -> np.ndarray:
    """``V[n, m] = psi_m(rst[:, n])`` for the orthonormal PKD basis; ``rst`` is ``(dim, n)``."""
    return np.stack([_BASIS[dim](rst, idx) for idx in mode_ids(dim, p)], axis=1)


def grad_vandermonde(dim: int, p: int, rst: np.ndarray) -> np.ndarray:
    """``(dim, n, Nmodes)`` reference-coordinate derivatives of the basis at ``rst``."""
    cols = [_GRAD_BASIS[dim](rst, idx) for idx in mode_ids(dim, p)]
    return np.stack([np.stack([c[r] for c in cols], axis=1) for r in range(dim)])

# }}}


# {{{ nodes

def node_multi_indices(dim: int, p: int) -> np.ndarray:
    """All ``(i_0..i_dim)`` with ``sum == p``; ``i_a`` counts steps towards vertex ``a``.

    Order: lexicographic in ``(i_dim, ..., i_1)`` ascending, i.e. the first barycentric
    direction varies fastest -- the usual "r fastest" nodal ordering.
    """
    out = []
    for tail in itertools.product(range(p + 1), repeat=dim):
        if sum(tail) <= p:
            # tail = (i_dim, ..., i_1) slowest..fastest
            idx = (p - sum(tail),) + tuple(reversed(tail))
            out.append(idx)
    return np.array(out, dtype=np.int64)


def barycentric_nodes(dim: int, p: int) -> np.ndarray:
    """``(Np, dim+1)`` barycentric coordinates of the GLL-blend nodes."""
    mi = node_multi_indices(dim, p)
    if p == 0:
        return np.full((1, dim + 1), 1.0 / (dim + 1))
    g = 0.5 * (gll_points(p) + 1.0)
    g[0], g[-1] = 0.0, 1.0
    w = g[mi]
    return w / w.sum(axis=1, keepdims=True)


def bary_to_rst(lam: np.ndarray) -> np.ndarray:
    """``(n, dim+1)`` barycentric -> ``(dim, n)`` biunit coordinates (``r_k = 2 lambda_k - 1``)."""
    return (2.0 * lam[:, 1:] - 1.0).T.copy()

# }}}


@dataclass(frozen=True)
class SimplexElement:
    """All reference-element data for one ``(dim, order)`` pair."""
    dim: int
    order: int
    multi_indices: np.ndarray   # (Np, dim+1) int64
    bary: np.ndarray            # (Np, dim+1)
    rst: np.ndarray             # (dim, Np)
    V: np.ndarray               # (Np, Np)
    mass: np.ndarray            # (Np, Np)
    D: np.ndarray               # (dim, Np, Np)
    Sw: np.ndarray              # (dim, Np, Np)
    lift: np.ndarray            # (Np, Nf*Nfp)
    face_nodes: np.ndarray      # (Nf, Nfp) int64 volume-node ids of each face's nodes
    face_vertices: np.ndarray   # (Nf, dim) int64 local vertex ids of each face (ascending)
    face_perms: np.ndarray      # (dim!, Nfp) int64: face-node permutation per vertex permutation
    perm_table: np.ndarray      # (dim!, dim) the vertex permutations themselves

    @property
    def Np(self) -> int:
        return self.rst.shape[1]

    @property
    def Nf(self) -> int:
        return self.dim + 1

    @property
    def Nfp(self) -> int:
        return self.face_nodes.shape[1]


def _face_node_table(dim: int, p: int, mi: np.ndarray):
    """Face ``f`` = nodes with ``i_f == 0``, ordered like the (dim-1)-simplex node set whose
    vertices are the face's vertices in ascending local order."""
    face_vertices = np.array([[v for v in range(dim + 1) if v != f] for f in range(dim + 1)], dtype=np.int64)
    sub = node_multi_indices(dim - 1, p) if dim > 1 else np.array([[p]], dtype=np.int64)
    lookup = {tuple(row): n for n, row in enumerate(mi)}
    face_nodes = np.empty((dim + 1, sub.shape[0]), dtype=np.int64)
    for f in range(dim + 1):
        for m, srow in enumerate(sub):
            full = np.zeros(dim + 1, dtype=np.int64)
            full[face_vertices[f]] = srow
            face_nodes[f, m] = lookup[tuple(full)]
    return face_nodes, face_vertices, sub


def _face_perm_table(dim: int, sub: np.ndarray):
    """``face_perms[s][m]``: position, in a neighbour face whose k-th vertex is OUR
    ``sigma_s(k)``-th face vertex, of the node that coincides with our face node ``m``."""
    perms = list(itertools.permutations(range(dim)))
    lookup = {tuple(row): n for n, row in enumerate(sub)}
    table = np.empty((len(perms), sub.shape[0]), dtype=np.int64)
    for s, sigma in enumerate(perms):
        for m, row in enumerate(sub):
            # neighbour's k-th face vertex is our sigma[k]-th: its multi-index entry k equals ours at sigma[k]
            table[s, m] = lookup[tuple(row[list(sigma)])]
    return table, np.array(perms, dtype=np.int64)


@lru_cache(maxsize=None)
def simplex_element(dim: int, order: int) -> SimplexElement:
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    if order < 1:
        raise ValueError("order must be >= 1")
    mi = node_multi_indices(dim, order)
    lam = barycentric_nodes(dim, order)
    rst = bary_to_rst(lam)
    V = vandermonde(dim, order, rst)
    Vinv = np.linalg.inv(V)
    gV = grad_vandermonde(dim, order, rst)
    D = np.stack([gV[r] @ Vinv for r in range(dim)])
    minv = V @ V.T
    mass = Vinv.T @ Vinv
    Sw = np.stack([minv @ D[r].T @ mass for r in range(dim)])

    face_nodes, face_vertices, sub = _face_node_table(dim, order, mi)
    Nf, Nfp = face_nodes.shape
    # face mass matrix on the standard (dim-1) biunit simplex, from the face nodes' own
    # barycentric coordinates with respect to the face's vertices
    emat = np.zeros((lam.shape[0], Nf * Nfp))
    for f in range(Nf):
        flam = lam[face_nodes[f]][:, face_vertices[f]]
        frst = bary_to_rst(flam)
        Vf = vandermonde(dim - 1, order, frst)
        mf = np.linalg.inv(Vf @ Vf.T)
        emat[face_nodes[f], f * Nfp:(f + 1) * Nfp] = mf
    lift = minv @ emat
    face_perms, perm_table = _face_perm_table(dim, sub)
    for a in (mi, lam, rst, V, mass, D, Sw, lift, face_nodes, face_vertices, face_perms, perm_table):
        a.setflags(write=False)
    return SimplexElement(dim, order, mi, lam, rst, V, mass, D, Sw, lift,
                          face_nodes, face_vertices, face_perms, perm_table)
