"""The DG operator program: compressible Euler / Navier-Stokes right-hand sides and RK4,
written ONCE against the array-context API of the reference
(/root/reference/pkg/src/laze/frontend.py:257-302 op namespace, :222-250 subscripts,
:488-519 ``outline``) and nothing else.

The same functions run
* on ``laze.ArrayContext(mode="eager")`` / ``mode="lazy"``   -- the CPU reference,
* on ``oracle.laze_port.NumpyArrayContext``                  -- its travelling restatement,
* on ``paper_2512_17101_b200.B200ArrayContext``              -- where the *outlined*
  functions below (``dg_euler_rhs``, ``dg_ns_grad``, ``dg_ns_rhs``) are dispatched BY NAME to
  the fused sm_100a kernels behind the C ABI (include/dgb200.h), exactly at the call
  boundary the reference creates for an outlined function
  (/root/reference/pkg/src/laze/adfg.py:722-803: arguments and results are materialised).

The physics is not pinned by the reference ("parity unpinned" at the physics
level); the formulation chosen here, following the paper's MIRGE-Com description
(/root/reference/PAPER.md:1738-1739,1778-1791), is:

* conserved state ``q = [rho, rho E, rho u_1..rho u_d]`` stored ``(C, E, Np)``;
* weak-form nodal DG on affine simplices,
  ``rhs = sum_{r,x} Sw_r (drdx[r,x] F_x) - lift(fscale * F*.n)``;
* inviscid numerical flux: local Lax-Friedrichs / Rusanov with
  ``lambda = max(|u-| + c-, |u+| + c+)``;
* viscous terms: BR1 -- ``grad q`` by a weak-form gradient with the central flux (first
  derivative pass), viscous flux from ``(q, grad q)`` with the central flux (second pass);
* ideal gas ``p = (gamma-1)(rho E - rho |u|^2/2)``, ``T = p/(rho R)``, constant ``mu, kappa``;
* boundary conditions by exterior ("plus") states: prescribed far-field state, or wall
  (Euler: slip, momentum reflected about the normal; Navier-Stokes: adiabatic no-slip,
  momentum negated); on boundary faces the viscous flux is the interior one,
  ``Fv(q-, grad q-)``, and the inviscid flux uses the exterior state.

The Navier-Stokes right-hand side exists in two algebraically identical arrangements of the same
scheme.  ``rhs_grad_form`` = ``dg_ns_grad`` (pass 1 writes ``grad q``) + ``dg_ns_rhs`` (pass 2
evaluates every flux).  ``rhs`` (default) = ``dg_ns_flux`` + ``dg_ns_div``: pass 1 finishes the BR1
gradient in registers, evaluates the total flux ``F = F_inv - F_visc`` once per node and stores its
contravariant, Jacobian-scaled components ``T[r] = sum_x (J dr/dx)[r,x] F[x]``, their sum over ``r`` and the
local wave speed; pass 2 is then a pure contraction: the volume term contracts ``T`` directly, and the
scaled normal flux of either side of a face is a signed sum of ``T`` rows (``facemat``), so the
neighbour's flux is *gathered*, not recomputed.  Each face flux is evaluated once per node
instead of three times (own volume, own face, neighbour's face), which is what makes the B200
path FP64-cheaper.
"""
from __future__ import annotations

import numpy as np

from .discretization import BC_FARFIELD, BC_NONE, BC_WALL, DGDiscretization
from .dofarray import DOFArray

# {{{ pointwise physics (array-context generic)


def _split(q, dim):
    rho, ener = q[0], q[1]
    mom = [q[2 + i] for i in range(dim)]
    return rho, ener, mom


def _pressure(actx, gamma, rho, ener, mom, vel):
    ke = mom[0] * vel[0]
    for i in range(1, len(mom)):
        ke = ke + mom[i] * vel[i]
    return (gamma - 1.0) * (ener - 0.5 * ke)


def inviscid_flux(actx, q, gamma, dim):
    """``F[x][c]`` as nested lists of arrays shaped like ``q[0]``."""
    rho, ener, mom = _split(q, dim)
    vel = [m / rho for m in mom]
    p = _pressure(actx, gamma, rho, ener, mom, vel)
    flux = []
    for x in range(dim):
        fx = [mom[x], vel[x] * (ener + p)]
        for i in range(dim):
            mi = mom[i] * vel[x]
            fx.append(mi + p if i == x else mi)
        flux.append(fx)
    return flux, vel, p


def viscous_flux(actx, q, gq, vel, phys, dim):
    """``Fv[x][c]`` from the state ``q`` and ``gq[x][c] = d q_c / d x_x``."""
    gamma, mu, kappa, rgas = phys
    rho, ener, mom = _split(q, dim)
    inv_rho = 1.0 / rho
    # velocity gradient  du[i][x] = d u_i / d x_x
    du = [[(gq[x][2 + i] - vel[i] * gq[x][0]) * inv_rho for x in range(dim)] for i in range(dim)]
    div = du[0][0]
    for i in range(1, dim):
        div = div + du[i][i]
    etot = ener * inv_rho
    # temperature gradient: T = (gamma-1)/R * (E/rho - |u|^2/2)
    dT = []
    for x in range(dim):
        de = (gq[x][1] - etot * gq[x][0]) * inv_rho
        for i in range(dim):
            de = de - vel[i] * du[i][x]
        dT.append(((gamma - 1.0) / rgas) * de)
    tau = [[None] * dim for _ in range(dim)]
    for i in range(dim):
        for x in range(dim):
            t = mu * (du[i][x] + du[x][i])
            if i == x:
                t = t - (2.0 / 3.0) * mu * div
            tau[i][x] = t
    flux = []
    for x in range(dim):
        work = vel[0] * tau[0][x]
        for i in range(1, dim):
            work = work + vel[i] * tau[i][x]
        fx = [None, work + kappa * dT[x]]
        for i in range(dim):
            fx.append(tau[i][x])
        flux.append(fx)
    return flux


def _normal_dot(flux, nrm, dim, comps):
    out = []
    for c in comps:
        acc = None
        for x in range(dim):
            if flux[x][c] is None:
                continue
            term = flux[x][c] * nrm[x]
            acc = term if acc is None else acc + term
        out.append(acc)
    return out


def _wavespeed(actx, gamma, q, vel, p, dim):
    v2 = vel[0] * vel[0]
    for i in range(1, dim):
        v2 = v2 + vel[i] * vel[i]
    return actx.np.sqrt(v2) + actx.np.sqrt(gamma * p / q[0])

# }}}


# {{{ traces and boundary states

def _traces(actx, q, ghost, vmap_m, vmap_p, lead, E, Np, Nf, Nfp):
    """Minus/plus face traces ``(lead, E, Nf, Nfp)`` through the flat int64 index maps
    (/root/reference/pkg/src/laze/adfg.py:502-560: one index array per subscript)."""
    flat = actx.np.reshape(q, (lead, E * Np))
    tm = actx.np.reshape(flat[:, vmap_m], (lead, E, Nf, Nfp))
    if ghost is not None:
        G = ghost.shape[-2]
        flat = actx.np.concatenate([flat, actx.np.reshape(ghost, (lead, G * Np))], axis=1)
    tp = actx.np.reshape(flat[:, vmap_p], (lead, E, Nf, Nfp))
    return tm, tp


def _bc_state(actx, qm, qp, nrm, bc_kind, qfar, dim, wall):
    """Exterior state per field: interior faces keep ``qp``."""
    C = dim + 2
    is_far = actx.np.equal(bc_kind, BC_FARFIELD)
    is_wall = actx.np.equal(bc_kind, BC_WALL)
    mom_m = [qm[2 + i] for i in range(dim)]
    if wall == "slip":
        mn = mom_m[0] * nrm[0]
        for i in range(1, dim):
            mn = mn + mom_m[i] * nrm[i]
        mom_w = [mom_m[i] - 2.0 * mn * nrm[i] for i in range(dim)]
    else:  # no-slip
        mom_w = [-mom_m[i] for i in range(dim)]
    wall_state = [qm[0], qm[1]] + mom_w
    out = []
    for c in range(C):
        v = actx.np.where(is_wall, wall_state[c], qp[c])
        v = actx.np.where(is_far, qfar[c], v)
        out.append(v)
    return out

# }}}


# {{{ the three outlined DG functions -- the plugin boundary

def _make_euler_rhs(dim, with_ghost):
    def body(actx, q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
        C, E, Np = q.shape
        Nf = dim + 1
        Nfp = lift.shape[1] // Nf
        gamma = phys[0]
        qc = [q[c] for c in range(C)]
        flux, _, _ = inviscid_flux(actx, qc, gamma, dim)
        fstack = actx.np.stack([actx.np.stack(fx) for fx in flux])            # (d, C, E, Np)
        vol = actx.np.einsum("rij,rxe,xcej->cei", Sw, drdx, fstack)
        tm, tp = _traces(actx, q, ghost, vmap_m, vmap_p, C, E, Np, Nf, Nfp)
        nrm = [normals[x] for x in range(dim)]
        qm = [tm[c] for c in range(C)]
        qp = _bc_state(actx, qm, [tp[c] for c in range(C)], nrm, bc_kind,
                       [qfar[c] for c in range(C)], dim, "slip")
        fm, vm, pm = inviscid_flux(actx, qm, gamma, dim)
        fp, vp, pp = inviscid_flux(actx, qp, gamma, dim)
        lam = actx.np.maximum(_wavespeed(actx, gamma, qm, vm, pm, dim),
                              _wavespeed(actx, gamma, qp, vp, pp, dim))
        fnm = _normal_dot(fm, nrm, dim, range(C))
        fnp = _normal_dot(fp, nrm, dim, range(C))
        fstar = [fscale * (0.5 * (fnm[c] + fnp[c]) + 0.5 * lam * (qm[c] - qp[c])) for c in range(C)]
        fs = actx.np.reshape(actx.np.stack(fstar), (C, E, Nf * Nfp))
        return vol - actx.np.einsum("if,cef->cei", lift, fs)

    if with_ghost:
        def dg_euler_rhs(q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
            return body(dg_euler_rhs.actx, q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p,
                        bc_kind, qfar, phys)
    else:
        def dg_euler_rhs(q, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
            return body(dg_euler_rhs.actx, q, None, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p,
                        bc_kind, qfar, phys)
    return dg_euler_rhs


def _make_ns_grad(dim, with_ghost):
    def body(actx, q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar):
        C, E, Np = q.shape
        Nf = dim + 1
        Nfp = lift.shape[1] // Nf
        vol = actx.np.einsum("rij,rxe,cej->xcei", Sw, drdx, q)
        tm, tp = _traces(actx, q, ghost, vmap_m, vmap_p, C, E, Np, Nf, Nfp)
        nrm = [normals[x] for x in range(dim)]
        qm = [tm[c] for c in range(C)]
        qp = _bc_state(actx, qm, [tp[c] for c in range(C)], nrm, bc_kind,
                       [qfar[c] for c in range(C)], dim, "noslip")
        qstar = [fscale * (0.5 * (qm[c] + qp[c])) for c in range(C)]
        fs = actx.np.stack([actx.np.stack([nrm[x] * qstar[c] for c in range(C)]) for x in range(dim)])
        fs = actx.np.reshape(fs, (dim, C, E, Nf * Nfp))
        return actx.np.einsum("if,xcef->xcei", lift, fs) - vol

    if with_ghost:
        def dg_ns_grad(q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar):
            return body(dg_ns_grad.actx, q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p,
                        bc_kind, qfar)
    else:
        def dg_ns_grad(q, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar):
            return body(dg_ns_grad.actx, q, None, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p,
                        bc_kind, qfar)
    return dg_ns_grad


def _make_ns_rhs(dim, with_ghost):
    def body(actx, q, gq, ghost, gghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind,
             qfar, phys):
        C, E, Np = q.shape
        Nf = dim + 1
        Nfp = lift.shape[1] // Nf
        ph = [phys[k] for k in range(4)]
        gamma = ph[0]
        qc = [q[c] for c in range(C)]
        gc = [[gq[x][c] for c in range(C)] for x in range(dim)]
        finv, vel, _ = inviscid_flux(actx, qc, gamma, dim)
        fvis = viscous_flux(actx, qc, gc, vel, ph, dim)
        ftot = [[finv[x][c] if fvis[x][c] is None else finv[x][c] - fvis[x][c] for c in range(C)]
                for x in range(dim)]
        fstack = actx.np.stack([actx.np.stack(fx) for fx in ftot])            # (d, C, E, Np)
        vol = actx.np.einsum("rij,rxe,xcej->cei", Sw, drdx, fstack)

        tm, tp = _traces(actx, q, ghost, vmap_m, vmap_p, C, E, Np, Nf, Nfp)
        gflat = actx.np.reshape(gq, (dim * C, E, Np))
        gg = None if gghost is None else actx.np.reshape(gghost, (dim * C, gghost.shape[-2], Np))
        gtm, gtp = _traces(actx, gflat, gg, vmap_m, vmap_p, dim * C, E, Np, Nf, Nfp)
        nrm = [normals[x] for x in range(dim)]
        qm = [tm[c] for c in range(C)]
        qp = _bc_state(actx, qm, [tp[c] for c in range(C)], nrm, bc_kind,
                       [qfar[c] for c in range(C)], dim, "noslip")
        gm = [[gtm[x * C + c] for c in range(C)] for x in range(dim)]
        gp = [[gtp[x * C + c] for c in range(C)] for x in range(dim)]
        fm, vm, pm = inviscid_flux(actx, qm, gamma, dim)
        fp, vp, pp = inviscid_flux(actx, qp, gamma, dim)
        lam = actx.np.maximum(_wavespeed(actx, gamma, qm, vm, pm, dim),
                              _wavespeed(actx, gamma, qp, vp, pp, dim))
        fnm = _normal_dot(fm, nrm, dim, range(C))
        fnp = _normal_dot(fp, nrm, dim, range(C))
        vnm = _normal_dot(viscous_flux(actx, qm, gm, vm, ph, dim), nrm, dim, range(C))
        vnp = _normal_dot(viscous_flux(actx, qp, gp, vp, ph, dim), nrm, dim, range(C))
        is_bnd = actx.np.not_equal(bc_kind, BC_NONE)
        fstar = []
        for c in range(C):
            f = 0.5 * (fnm[c] + fnp[c]) + 0.5 * lam * (qm[c] - qp[c])
            if vnm[c] is not None:
                # boundary faces take the viscous flux of the interior state, Fv(q-, grad q-)
                f = f - 0.5 * (vnm[c] + actx.np.where(is_bnd, vnm[c], vnp[c]))
            fstar.append(fscale * f)
        fs = actx.np.reshape(actx.np.stack(fstar), (C, E, Nf * Nfp))
        return vol - actx.np.einsum("if,cef->cei", lift, fs)

    if with_ghost:
        def dg_ns_rhs(q, gq, ghost, gghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind,
                      qfar, phys):
            return body(dg_ns_rhs.actx, q, gq, ghost, gghost, Sw, drdx, lift, normals, fscale, vmap_m,
                        vmap_p, bc_kind, qfar, phys)
    else:
        def dg_ns_rhs(q, gq, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
            return body(dg_ns_rhs.actx, q, gq, None, None, Sw, drdx, lift, normals, fscale, vmap_m,
                        vmap_p, bc_kind, qfar, phys)
    return dg_ns_rhs


def _make_ns_flux(dim, with_ghost):
    """Pass 1 of the flux arrangement: BR1 gradient -> total flux -> contravariant components.
    Returns ``((dim+1)*C + 1, E, Np)``: planes ``r*C + c`` (``r < dim``) hold ``T[r][c] = sum_x jac*drdx[r,x] *
    (F_inv - F_visc)[x][c]``, planes ``dim*C + c`` their sum over ``r`` (the scaled normal flux of face 0, stored so
    that a neighbour gathers ONE plane per field whatever face it sees) and the last plane the wave speed
    ``|u| + c``."""
    grad = _make_ns_grad(dim, with_ghost)

    def body(actx, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
        grad.actx = actx
        if ghost is None:
            gq = grad(q, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar)
        else:
            gq = grad(q, ghost, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar)
        C, E, Np = q.shape
        ph = [phys[k] for k in range(4)]
        gamma = ph[0]
        qc = [q[c] for c in range(C)]
        gc = [[gq[x][c] for c in range(C)] for x in range(dim)]
        finv, vel, p = inviscid_flux(actx, qc, gamma, dim)
        fvis = viscous_flux(actx, qc, gc, vel, ph, dim)
        ftot = [[finv[x][c] if fvis[x][c] is None else finv[x][c] - fvis[x][c] for c in range(C)]
                for x in range(dim)]
        fstack = actx.np.stack([actx.np.stack(fx) for fx in ftot])            # (d, C, E, Np)
        T = actx.np.einsum("rxe,e,xcej->rcej", drdx, jac, fstack)
        tsum = T[0] + T[1]
        for r in range(2, dim):
            tsum = tsum + T[r]
        lam = _wavespeed(actx, gamma, qc, vel, p, dim)
        return actx.np.concatenate([actx.np.reshape(T, (dim * C, E, Np)), tsum, actx.np.reshape(lam, (1, E, Np))])

    if with_ghost:
        def dg_ns_flux(q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
            return body(dg_ns_flux.actx, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p,
                        bc_kind, qfar, phys)
    else:
        def dg_ns_flux(q, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
            return body(dg_ns_flux.actx, q, None, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p,
                        bc_kind, qfar, phys)
    return dg_ns_flux


def _make_ns_div(dim, with_ghost):
    """Pass 2 of the flux arrangement: ``rhs = (1/J) (sum_r Sw_r T_r - lift(sJ F*.n))`` with
    ``sJ F-.n = sum_g facemat[g,f] T-[g]`` and ``sJ F+.n = -sum_g facemat[g,f+] T+[g]`` over the ``dim + 1`` plane
    groups of ``dg_ns_flux`` (``T[dim]`` = sum of the others: face 0 selects it, face ``f >= 1`` selects ``-T[f-1]``;
    ``facemat_p`` is ``facemat`` of the neighbour's face, per face)."""
    def body(actx, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p,
             bc_kind, qfar, phys):
        C, E, Np = q.shape
        Nf = dim + 1
        Nfp = lift.shape[1] // Nf
        L = C + (dim + 1) * C + 1
        gamma = phys[0]
        vol = actx.np.einsum("rij,rcej->cei", Sw, actx.np.reshape(T[0:dim * C], (dim, C, E, Np)))
        planes = actx.np.concatenate([q, T])                                   # (L, E, Np)
        gplanes = None if ghost is None else actx.np.concatenate([ghost, Tghost])
        tm, tp = _traces(actx, planes, gplanes, vmap_m, vmap_p, L, E, Np, Nf, Nfp)
        nrm = [normals[x] for x in range(dim)]
        sj = fscale * actx.np.reshape(jac, (E, 1, 1))                          # face Jacobian (E, Nf, 1)
        qm = [tm[c] for c in range(C)]
        qp = [tp[c] for c in range(C)]
        own, nbr = [], []
        for c in range(C):
            o = facemat[0] * tm[C + c]
            n = facemat_p[0] * tp[C + c]
            for r in range(1, dim + 1):
                o = o + facemat[r] * tm[C + r * C + c]
                n = n + facemat_p[r] * tp[C + r * C + c]
            own.append(o)
            nbr.append(n)
        lam_m, lam_p = tm[L - 1], tp[L - 1]
        # boundary faces: inviscid flux of the exterior state, viscous flux of the interior state
        qb = _bc_state(actx, qm, qp, nrm, bc_kind, [qfar[c] for c in range(C)], dim, "noslip")
        fb, vb, pb = inviscid_flux(actx, qb, gamma, dim)
        fi, _, _ = inviscid_flux(actx, qm, gamma, dim)
        fnb = _normal_dot(fb, nrm, dim, range(C))
        fni = _normal_dot(fi, nrm, dim, range(C))
        lam_b = actx.np.maximum(lam_m, _wavespeed(actx, gamma, qb, vb, pb, dim))
        is_bnd = actx.np.not_equal(bc_kind, BC_NONE)
        fstar = []
        for c in range(C):
            f_int = 0.5 * (own[c] - nbr[c]) + 0.5 * sj * actx.np.maximum(lam_m, lam_p) * (qm[c] - qp[c])
            f_bnd = own[c] + 0.5 * sj * (fnb[c] - fni[c]) + 0.5 * sj * lam_b * (qm[c] - qb[c])
            fstar.append(actx.np.where(is_bnd, f_bnd, f_int))
        fs = actx.np.reshape(actx.np.stack(fstar), (C, E, Nf * Nfp))
        return (vol - actx.np.einsum("if,cef->cei", lift, fs)) / actx.np.reshape(jac, (E, 1))

    if with_ghost:
        def dg_ns_div(q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p,
                      bc_kind, qfar, phys):
            return body(dg_ns_div.actx, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat,
                        facemat_p, vmap_m, vmap_p, bc_kind, qfar, phys)
    else:
        def dg_ns_div(q, T, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind,
                      qfar, phys):
            return body(dg_ns_div.actx, q, T, None, None, Sw, jac, lift, normals, fscale, facemat,
                        facemat_p, vmap_m, vmap_p, bc_kind, qfar, phys)
    return dg_ns_div


def _axpby_outputs(rhs, x1, x2, coef):
    """RK stage update fused behind the right-hand side (north-star item 3):
    ``out1 = a1*x1 + b1*rhs``, ``out2 = a2*x2 + b2*rhs`` with ``coef = [a1, b1, a2, b2]``."""
    return {"out1": coef[0] * x1 + coef[1] * rhs, "out2": coef[2] * x2 + coef[3] * rhs}


def _make_euler_rhs_rk(dim, with_ghost):
    inner = _make_euler_rhs(dim, False)

    def dg_euler_rhs_rk(q, x1, x2, coef, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
        inner.actx = dg_euler_rhs_rk.actx
        rhs = inner(q, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys)
        return _axpby_outputs(rhs, x1, x2, coef)
    return dg_euler_rhs_rk


def _make_ns_rhs_rk(dim, with_ghost):
    inner = _make_ns_rhs(dim, False)

    def dg_ns_rhs_rk(q, gq, x1, x2, coef, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys):
        inner.actx = dg_ns_rhs_rk.actx
        rhs = inner(q, gq, Sw, drdx, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, phys)
        return _axpby_outputs(rhs, x1, x2, coef)
    return dg_ns_rhs_rk

def _make_ns_div_rk(dim, with_ghost):
    inner = _make_ns_div(dim, False)

    def dg_ns_div_rk(q, T, x1, x2, coef, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p,
                     bc_kind, qfar, phys):
        inner.actx = dg_ns_div_rk.actx
        rhs = inner(q, T, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar, phys)
        return _axpby_outputs(rhs, x1, x2, coef)
    return dg_ns_div_rk

# }}}


class _OperatorBase:
    def __init__(self, dcoll: DGDiscretization, gamma=1.4, mu=0.0, prandtl=0.72, rgas=1.0,
                 farfield=None):
        self.dcoll = dcoll
        self.actx = actx = dcoll.actx
        self.dim = dim = dcoll.dim
        self.gamma, self.mu, self.rgas = float(gamma), float(mu), float(rgas)
        self.kappa = self.mu * (self.gamma * self.rgas / (self.gamma - 1.0)) / float(prandtl)
        C = dim + 2
        if farfield is None:
            farfield = np.zeros(C)
            farfield[0] = 1.0
            farfield[1] = 1.0 / (self.gamma * (self.gamma - 1.0))
        self.qfar_host = np.asarray(farfield, dtype=np.float64).reshape(C)
        self.qfar = actx.from_numpy(self.qfar_host.reshape(C, 1, 1, 1))
        self.phys_host = np.array([self.gamma, self.mu, self.kappa, self.rgas])
        self.phys = actx.from_numpy(self.phys_host)

    def _outlined(self, maker, with_ghost):
        f = maker(self.dim, with_ghost)
        f.actx = self.actx
        f.dg_dim = self.dim
        return self.actx.outline(f)

    def _common(self):
        d = self.dcoll
        return (d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind, self.qfar)


class EulerOperator(_OperatorBase):
    """``rhs(q)`` of the compressible Euler equations; ``q`` is a ``DOFArray`` ``(C, E, Np)``."""

    def __init__(self, dcoll, gamma=1.4, farfield=None):
        super().__init__(dcoll, gamma=gamma, farfield=farfield)
        self._f = self._outlined(_make_euler_rhs, False)
        self._fg = self._outlined(_make_euler_rhs, True)

    def rhs(self, q: DOFArray, t=0.0, ghost=None) -> DOFArray:
        if ghost is None:
            out = self._f(q.data, *self._common(), self.phys)
        else:
            out = self._fg(q.data, ghost, *self._common(), self.phys)
        return DOFArray(self.actx, out)

    def rhs_rk(self, q: DOFArray, x1: DOFArray, x2: DOFArray, coef, t=0.0):
        """``(a1*x1 + b1*rhs(q), a2*x2 + b2*rhs(q))`` in one fused pass; ``coef = (a1, b1, a2, b2)``."""
        if not hasattr(self, "_frk"):
            self._frk = self._outlined(_make_euler_rhs_rk, False)
        c = self.actx.from_numpy(np.asarray(coef, dtype=np.float64))
        out = self._frk(q.data, x1.data, x2.data, c, *self._common(), self.phys)
        return DOFArray(self.actx, out["out1"]), DOFArray(self.actx, out["out2"])


class NavierStokesOperator(_OperatorBase):
    """Two-pass (BR1) compressible Navier-Stokes right-hand side.

    ``rhs`` / ``rhs_rk`` use the flux arrangement (``dg_ns_flux`` + ``dg_ns_div``, see the module
    docstring); ``rhs_grad_form`` / ``rhs_rk_grad_form`` the gradient arrangement (``dg_ns_grad`` +
    ``dg_ns_rhs``).  Both evaluate the same scheme."""

    def __init__(self, dcoll, gamma=1.4, mu=1e-3, prandtl=0.72, rgas=1.0, farfield=None):
        super().__init__(dcoll, gamma=gamma, mu=mu, prandtl=prandtl, rgas=rgas, farfield=farfield)
        self._g = self._outlined(_make_ns_grad, False)
        self._gg = self._outlined(_make_ns_grad, True)
        self._f = self._outlined(_make_ns_rhs, False)
        self._fg = self._outlined(_make_ns_rhs, True)
        self._flux = self._outlined(_make_ns_flux, False)
        self._fluxg = self._outlined(_make_ns_flux, True)
        self._div = self._outlined(_make_ns_div, False)
        self._divg = self._outlined(_make_ns_div, True)

    def _flux_args(self):
        d = self.dcoll
        return (d.Sw, d.drdx, d.jac, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind, self.qfar,
                self.phys)

    def _div_args(self):
        d = self.dcoll
        return (d.Sw, d.jac, d.lift, d.normals, d.fscale, d.facemat, d.facemat_p, d.vmap_m, d.vmap_p,
                d.bc_kind, self.qfar, self.phys)

    def grad(self, q: DOFArray, ghost=None) -> DOFArray:
        if ghost is None:
            out = self._g(q.data, *self._common())
        else:
            out = self._gg(q.data, ghost, *self._common())
        return DOFArray(self.actx, out)

    def flux(self, q: DOFArray, ghost=None):
        """Pass 1: contravariant total-flux planes + wave speed, ``(dim*C + 1, E, Np)``."""
        if ghost is None:
            return self._flux(q.data, *self._flux_args())
        return self._fluxg(q.data, ghost, *self._flux_args())

    def rhs(self, q: DOFArray, t=0.0, ghost=None, halo_fn=None) -> DOFArray:
        """``halo_fn(DOFArray of the pass-1 result) -> ghost array`` performs the second halo
        exchange on partitioned meshes (flux planes here, ``grad q`` in ``rhs_grad_form``)."""
        T = self.flux(q, ghost)
        if ghost is None:
            out = self._div(q.data, T, *self._div_args())
        else:
            out = self._divg(q.data, T, ghost, halo_fn(DOFArray(self.actx, T)), *self._div_args())
        return DOFArray(self.actx, out)

    def rhs_rk(self, q: DOFArray, x1: DOFArray, x2: DOFArray, coef, t=0.0):
        """``(a1*x1 + b1*rhs(q), a2*x2 + b2*rhs(q))`` with the stage update fused into the second pass."""
        if not hasattr(self, "_divrk"):
            self._divrk = self._outlined(_make_ns_div_rk, False)
        T = self.flux(q)
        c = self.actx.from_numpy(np.asarray(coef, dtype=np.float64))
        out = self._divrk(q.data, T, x1.data, x2.data, c, *self._div_args())
        return DOFArray(self.actx, out["out1"]), DOFArray(self.actx, out["out2"])

    def rhs_grad_form(self, q: DOFArray, t=0.0, ghost=None, halo_fn=None) -> DOFArray:
        gq = self.grad(q, ghost)
        if ghost is None:
            out = self._f(q.data, gq.data, *self._common(), self.phys)
        else:
            gghost = halo_fn(gq)
            out = self._fg(q.data, gq.data, ghost, gghost, *self._common(), self.phys)
        return DOFArray(self.actx, out)

    def rhs_rk_grad_form(self, q: DOFArray, x1: DOFArray, x2: DOFArray, coef, t=0.0):
        if not hasattr(self, "_frk"):
            self._frk = self._outlined(_make_ns_rhs_rk, False)
        gq = self.grad(q)
        c = self.actx.from_numpy(np.asarray(coef, dtype=np.float64))
        out = self._frk(q.data, gq.data, x1.data, x2.data, c, *self._common(), self.phys)
        return DOFArray(self.actx, out["out1"]), DOFArray(self.actx, out["out2"])


# {{{ time stepping

def rk4_step(rhs, q, t, dt):
    """Classical fourth-order Runge-Kutta step in array-context arithmetic
    (the paper's applications step with RK4: /root/reference/PAPER.md:1692)."""
    k1 = rhs(q, t)
    k2 = rhs(q + (0.5 * dt) * k1, t + 0.5 * dt)
    k3 = rhs(q + (0.5 * dt) * k2, t + 0.5 * dt)
    k4 = rhs(q + dt * k3, t + dt)
    return q + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def rk4_step_fused(op, q, t, dt):
    """Classical RK4 with every stage update fused into the right-hand-side pass
    (``op.rhs_rk``): per stage one read of the stage state and of the two update operands and one
    write of each output, instead of separate axpy sweeps.  Same scheme as ``rk4_step``; the final
    combination is accumulated stage by stage."""
    q1, acc = op.rhs_rk(q, q, q, (1.0, 0.5 * dt, 1.0, dt / 6.0), t)
    q2, acc = op.rhs_rk(q1, q, acc, (1.0, 0.5 * dt, 1.0, dt / 3.0), t + 0.5 * dt)
    q3, acc = op.rhs_rk(q2, q, acc, (1.0, dt, 1.0, dt / 3.0), t + 0.5 * dt)
    qn, _ = op.rhs_rk(q3, acc, acc, (1.0, dt / 6.0, 0.0, 0.0), t + dt)
    return qn

# }}}
