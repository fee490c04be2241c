"""Conforming simplicial box meshes and their face connectivity (setup time, NumPy).

The reference has no mesh code ("meshes, connectivity, face index maps: no").
What the reference *does* fix is the form an index map must take to be used through its
array context: an ``int64`` index array applied to a flattened array
(/root/reference/pkg/src/laze/adfg.py:502-560, dtype check at :540-541).  ``vmap_m`` /
``vmap_p`` below are exactly that: flat indices into ``u.reshape(E*Np)``.

Meshes: structured boxes split into triangles (2 per cell) or Kuhn tetrahedra (6 per cell),
optionally periodic per axis.  Cells are visited along a Morton (Z-order) curve so that
face neighbours are close in memory (L2 locality for the face gather).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from .simplex import SimplexElement, simplex_element

BTAG_INTERIOR = 0   # face has a neighbour element


@dataclass
class Mesh:
    dim: int
    vertices: np.ndarray        # (E, dim+1, dim) float64 physical vertex coordinates per element
    vertex_ids: np.ndarray      # (E, dim+1) int64 global (periodically identified) vertex ids
    nbr_elem: np.ndarray        # (E, Nf) int64 neighbour element (self on boundary faces)
    nbr_face: np.ndarray        # (E, Nf) int64 neighbour's local face id (own face on boundary)
    nbr_perm: np.ndarray        # (E, Nf) int64 vertex-permutation id (see SimplexElement.face_perms)
    btag: np.ndarray            # (E, Nf) int64 0 = interior, k>0 = boundary tag (1+2*axis+side for boxes)
    nbr_rank: np.ndarray | None = None   # (E, Nf) int64 owning rank of the neighbour (partitioned meshes)

    @property
    def nelements(self) -> int:
        return self.vertices.shape[0]


def _morton_order(counts: tuple[int, ...]) -> np.ndarray:
    """Cell multi-indices ``(ncells, dim)`` sorted along a Z-order curve."""
    dim = len(counts)
    grids = np.meshgrid(*[np.arange(n, dtype=np.int64) for n in counts], indexing="ij")
    ijk = np.stack([g.ravel() for g in grids], axis=1)
    code = np.zeros(ijk.shape[0], dtype=np.int64)
    nbits = max(int(np.ceil(np.log2(max(counts)))) if max(counts) > 1 else 1, 1)
    for b in range(nbits):
        for a in range(dim):
            code |= ((ijk[:, a] >> b) & 1) << (dim * b + a)
    return ijk[np.argsort(code, kind="stable")]


def _kuhn_simplices(dim: int) -> list[np.ndarray]:
    """Corner offsets (dim+1, dim) of the dim! Kuhn simplices of the unit cube, positively oriented."""
    out = []
    for perm in itertools.permutations(range(dim)):
        pts = [np.zeros(dim, dtype=np.int64)]
        for ax in perm:
            nxt = pts[-1].copy()
            nxt[ax] += 1
            pts.append(nxt)
        pts = np.array(pts)
        edges = (pts[1:] - pts[0]).astype(np.float64)
        if np.linalg.det(edges) < 0:
            pts[[dim - 1, dim]] = pts[[dim, dim - 1]]
        out.append(pts)
    return out


def box_mesh(counts, lo, hi, periodic=None, morton: bool = True) -> Mesh:
    """Kuhn-split box mesh with ``counts[a]`` cells along axis ``a`` between ``lo`` and ``hi``."""
    counts = tuple(int(c) for c in counts)
    dim = len(counts)
    if dim not in (2, 3):
        raise ValueError("box_mesh supports dim 2 and 3")
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    periodic = tuple(bool(x) for x in (periodic if periodic is not None else (False,) * dim))
    for a in range(dim):
        if periodic[a] and counts[a] < 3:
            raise ValueError("periodic axes need at least 3 cells so that face keys stay unique")
    h = (hi - lo) / np.asarray(counts, dtype=np.float64)
    cells = _morton_order(counts) if morton else _morton_order(counts)[np.lexsort(
        _morton_order(counts).T[::-1])]
    simplices = _kuhn_simplices(dim)
    ns = len(simplices)
    ncells = cells.shape[0]
    corner = cells[:, None, None, :] + np.stack(simplices)[None, :, :, :]      # (ncells, ns, dim+1, dim)
    corner = corner.reshape(ncells * ns, dim + 1, dim)
    vertices = lo + corner.astype(np.float64) * h
    nv = tuple(counts[a] if periodic[a] else counts[a] + 1 for a in range(dim))
    wrapped = corner.copy()
    for a in range(dim):
        if periodic[a]:
            wrapped[..., a] %= counts[a]
    vid = np.zeros(corner.shape[:2], dtype=np.int64)
    for a in range(dim):
        vid = vid * nv[a] + wrapped[..., a]
    mesh = _connect(dim, vertices, vid)
    # boundary tags: 1 + 2*axis + side from the face centroid
    E, Nf = mesh.btag.shape
    fv = np.array([[v for v in range(dim + 1) if v != f] for f in range(dim + 1)])
    bnd = np.argwhere(mesh.btag != 0)
    if bnd.size:
        cent = vertices[bnd[:, 0][:, None], fv[bnd[:, 1]]].mean(axis=1)
        tag = np.zeros(bnd.shape[0], dtype=np.int64)
        for a in range(dim):
            tol = 1e-9 * max(1.0, abs(hi[a] - lo[a]))
            tag[np.abs(cent[:, a] - lo[a]) < tol] = 1 + 2 * a
            tag[np.abs(cent[:, a] - hi[a]) < tol] = 2 + 2 * a
        if np.any(tag == 0):
            raise RuntimeError("boundary face not on the box surface")
        mesh.btag[bnd[:, 0], bnd[:, 1]] = tag
    return mesh


_KEY_LIMIT = 2.0 ** 62        # packed face keys stay below this (tests lower it to force the two-level path)


def _connect(dim: int, vertices: np.ndarray, vid: np.ndarray) -> Mesh:
    """Face matching by sorted global vertex ids; integer-exact."""
    E = vid.shape[0]
    Nf = dim + 1
    fv = np.array([[v for v in range(dim + 1) if v != f] for f in range(dim + 1)])   # (Nf, dim)
    fvid = vid[:, fv]                                   # (E, Nf, dim) in local ascending order
    srt = np.sort(fvid, axis=2)
    nvert = int(vid.max()) + 1
    key = np.zeros((E, Nf), dtype=np.int64)
    span = 1.0                                           # upper bound of the keys packed so far
    for a in range(dim):
        if span * nvert >= _KEY_LIMIT:                   # would overflow: rank the partial keys first (equality-preserving)
            if float(E * Nf) * nvert >= 2.0 ** 62:
                raise ValueError("mesh too large for packed face keys")
            key = np.unique(key.ravel(), return_inverse=True)[1].reshape(E, Nf).astype(np.int64)
            span = float(E * Nf)
        key = key * nvert + srt[..., a]
        span *= nvert
    flat = key.ravel()
    order = np.argsort(flat, kind="stable")
    sk = flat[order]
    same_next = np.zeros(sk.shape[0], dtype=bool)
    same_next[:-1] = sk[:-1] == sk[1:]
    same_prev = np.zeros_like(same_next)
    same_prev[1:] = same_next[:-1]
    if np.any(same_next & same_prev):
        raise ValueError("a face is shared by more than two elements (non-manifold or too-coarse periodic mesh)")
    a_idx = order[same_next]
    b_idx = order[np.nonzero(same_next)[0] + 1]
    nbr = np.arange(E * Nf, dtype=np.int64)             # boundary: self
    nbr[a_idx] = b_idx
    nbr[b_idx] = a_idx
    nbr_elem = (nbr // Nf).reshape(E, Nf)
    nbr_face = (nbr % Nf).reshape(E, Nf)
    btag = np.ones((E, Nf), dtype=np.int64)
    btag.ravel()[a_idx] = 0
    btag.ravel()[b_idx] = 0
    # permutation id: neighbour's k-th face vertex is our sigma[k]-th face vertex
    mine = fvid                                          # (E, Nf, dim)
    theirs = fvid[nbr_elem, nbr_face]                    # (E, Nf, dim)
    sigma = np.argmax(theirs[..., :, None] == mine[..., None, :], axis=-1)     # (E, Nf, dim)
    if not np.array_equal(np.take_along_axis(mine, sigma, axis=-1), theirs):
        raise RuntimeError("face vertex matching failed")
    perms = np.array(list(itertools.permutations(range(dim))), dtype=np.int64)
    code = np.zeros(sigma.shape[:2], dtype=np.int64)
    for a in range(dim):
        code = code * dim + sigma[..., a]
    pcode = np.zeros(perms.shape[0], dtype=np.int64)
    for a in range(dim):
        pcode = pcode * dim + perms[:, a]
    lut = np.full(dim ** dim, -1, dtype=np.int64)
    lut[pcode] = np.arange(perms.shape[0])
    nbr_perm = lut[code]
    if np.any(nbr_perm < 0):
        raise RuntimeError("invalid face permutation")
    return Mesh(dim, vertices, vid, nbr_elem, nbr_face, nbr_perm, btag)


# {{{ geometry + index maps

@dataclass
class Geometry:
    """Affine geometric factors.  ``drdx[r, x, e] = d r / d x`` (so that
    ``d/dx_x = sum_r drdx[r, x, e] d/dr``), unit outward normals and face scales."""
    drdx: np.ndarray      # (dim, dim, E)
    jac: np.ndarray       # (E,)
    normals: np.ndarray   # (dim, E, Nf)
    fscale: np.ndarray    # (E, Nf)  surface Jacobian / volume Jacobian
    nodes: np.ndarray     # (dim, E, Np) physical node coordinates


def geometry(mesh: Mesh, el: SimplexElement) -> Geometry:
    dim = mesh.dim
    v = mesh.vertices                                     # (E, dim+1, dim)
    # x = sum_a lambda_a v_a, lambda_k = (1 + r_k)/2 for k>=1  =>  dx/dr_k = (v_k - v_0)/2
    dxdr = 0.5 * (v[:, 1:, :] - v[:, :1, :])              # (E, r, x)
    jac = np.linalg.det(dxdr)
    if np.any(jac <= 0):
        raise ValueError("negatively oriented element")
    drdx_e = np.linalg.inv(dxdr)                          # (E, x, r): inverse of [r,x] -> rows x, cols r
    drdx = np.ascontiguousarray(np.transpose(drdx_e, (2, 1, 0)))   # (r, x, E)
    # grad lambda_k = drdx[k-1]/2 for k>=1, grad lambda_0 = -sum
    glam = np.empty((dim + 1, dim, v.shape[0]))
    glam[1:] = 0.5 * drdx
    glam[0] = -glam[1:].sum(axis=0)
    nrm = -glam                                           # outward normal direction of face f
    mag = np.sqrt((nrm ** 2).sum(axis=1))                 # (Nf, E)
    normals = np.ascontiguousarray(np.transpose(nrm / mag[:, None, :], (1, 2, 0)))   # (dim, E, Nf)
    fscale = np.ascontiguousarray((2.0 * mag).T)          # (E, Nf)
    nodes = np.einsum("na,eax->xen", el.bary, v)
    return Geometry(drdx, jac, normals, fscale, np.ascontiguousarray(nodes))


def face_index_maps(mesh: Mesh, el: SimplexElement) -> tuple[np.ndarray, np.ndarray]:
    """``vmap_m, vmap_p``: ``(E, Nf, Nfp)`` int64 flat indices into ``u.reshape(E*Np)`` of each
    face node's own value and of the coinciding node in the neighbour (== ``vmap_m`` on
    boundary faces)."""
    E = mesh.nelements
    Np = el.Np
    own = el.face_nodes[None, :, :]                                       # (1, Nf, Nfp)
    vmap_m = np.arange(E, dtype=np.int64)[:, None, None] * Np + own
    pos = el.face_perms[mesh.nbr_perm]                                    # (E, Nf, Nfp)
    nfn = el.face_nodes[mesh.nbr_face]                                    # (E, Nf, Nfp) neighbour's face nodes
    vmap_p = mesh.nbr_elem[:, :, None] * Np + np.take_along_axis(nfn, pos, axis=2)
    bnd = mesh.btag != 0
    vmap_p[bnd] = vmap_m[bnd]
    return np.ascontiguousarray(vmap_m), np.ascontiguousarray(vmap_p)

# }}}
