"""``DGDiscretization``: reference matrices, affine geometry and face index maps of one mesh,
uploaded once through an array context.

Everything here is computed on the host in NumPy (integer-exact connectivity, FP64
matrices) and handed to the context with ``actx.from_numpy``
(/root/reference/pkg/src/laze/frontend.py:327-332), so the *same* arrays feed the CPU
reference context and the B200 context.
"""
from __future__ import annotations

import numpy as np

from .dg.mesh import Mesh, face_index_maps, geometry
from .dg.simplex import simplex_element
from .dofarray import DOFArray

# boundary-condition kinds understood by the operator program (operators.py)
BC_NONE = 0        # interior face
BC_FARFIELD = 1    # exterior state prescribed (constant free-stream)
BC_WALL = 2        # Euler: slip wall; Navier-Stokes: adiabatic no-slip wall


class DGDiscretization:
    def __init__(self, actx, mesh: Mesh, order: int, bc_map: dict[int, int] | None = None,
                 ghost_elements: int = 0):
        self.actx = actx
        self.mesh = mesh
        self.order = order
        self.dim = mesh.dim
        el = self.element = simplex_element(mesh.dim, order)
        self.geo = geo = geometry(mesh, el)
        E, Nf, Nfp, Np = mesh.nelements, el.Nf, el.Nfp, el.Np
        self.nelements, self.Np, self.Nf, self.Nfp = E, Np, Nf, Nfp
        self.ghost_elements = int(ghost_elements)
        vmap_m, vmap_p = face_index_maps(mesh, el)
        self.vmap_m_host, self.vmap_p_host = vmap_m, vmap_p
        bc_kind = np.zeros((E, Nf), dtype=np.int64)
        tags = np.unique(mesh.btag[mesh.btag != 0])
        bc_map = dict(bc_map or {})
        for t in tags:
            if int(t) not in bc_map:
                raise ValueError(f"no boundary condition given for boundary tag {int(t)}")
            bc_kind[mesh.btag == t] = bc_map[int(t)]
        self.bc_kind_host = bc_kind

        f = actx.from_numpy
        self.Sw = f(np.ascontiguousarray(el.Sw))                    # (d, Np, Np)
        self.D = f(np.ascontiguousarray(el.D))                      # (d, Np, Np)
        self.lift = f(np.ascontiguousarray(el.lift))                # (Np, Nf*Nfp)
        self.drdx = f(geo.drdx)                                     # (d, d, E)   [r, x, e]
        self.normals = f(geo.normals.reshape(self.dim, E, Nf, 1))   # (d, E, Nf, 1)
        self.fscale = f(geo.fscale.reshape(E, Nf, 1))               # (E, Nf, 1)
        self.jac = f(np.ascontiguousarray(geo.jac))                 # (E,) volume Jacobian
        # fscale * jac * n_x (face f) == sum_r facemat[r, f] * jac * drdx[r, x]: face 0 (opposite vertex 0)
        # is the sum of the reference gradients, face f >= 1 is minus gradient f-1 (dg/mesh.py: geometry)
        fm = np.zeros((self.dim, Nf))
        fm[:, 0] = 1.0
        for r in range(self.dim):
            fm[r, r + 1] = -1.0
        lhs = geo.fscale[None] * geo.normals                        # (x, E, Nf)
        assert np.allclose(lhs, np.einsum("rf,rxe->xef", fm, geo.drdx), rtol=1e-12, atol=1e-12)
        # The flux arrangement stores that sum as a plane group of its own (operators.py: dg_ns_flux), so a face
        # selects exactly ONE of dim + 1 groups: face 0 -> +group dim, face f >= 1 -> -group f-1.
        fm = np.zeros((self.dim + 1, Nf))
        fm[self.dim, 0] = 1.0
        for r in range(self.dim):
            fm[r, r + 1] = -1.0
        self.facemat_host = fm
        self.facemat = f(fm.reshape(self.dim + 1, Nf, 1))           # (d+1, Nf, 1), broadcasts over elements
        self.facemat_p = f(np.ascontiguousarray(fm[:, mesh.nbr_face]).reshape(self.dim + 1, E, Nf, 1))
        self.vmap_m = f(vmap_m.reshape(-1))                         # (E*Nf*Nfp,) int64
        self.vmap_p = f(vmap_p.reshape(-1))
        self.bc_kind = f(bc_kind.reshape(E, Nf, 1))                 # (E, Nf, 1) int64

    def nodes(self) -> np.ndarray:
        """Host node coordinates ``(dim, E, Np)``."""
        return self.geo.nodes

    def from_numpy(self, host) -> DOFArray:
        return DOFArray(self.actx, self.actx.from_numpy(np.ascontiguousarray(host, dtype=np.float64)))

    def to_numpy(self, dof: DOFArray) -> np.ndarray:
        return np.asarray(self.actx.to_numpy(dof.data))

    def interp(self, fn) -> DOFArray:
        """Nodal interpolant of ``fn(x) -> (..., E, Np)``."""
        return self.from_numpy(fn(self.geo.nodes))

    def norm_inf(self, dof: DOFArray) -> float:
        return float(np.max(np.abs(self.to_numpy(dof))))

    def norm_l2(self, host: np.ndarray) -> float:
        """Discrete L2 norm of host nodal data ``(..., E, Np)`` with the exact mass matrix."""
        m = self.element.mass
        h = np.asarray(host).reshape(-1, self.nelements, self.Np)
        val = np.einsum("cei,ij,cej,e->", h, m, h, self.geo.jac)
        return float(np.sqrt(val))
