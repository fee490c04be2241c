"""Multi-species reactive compressible Navier-Stokes (BASELINE.json configs[4]) -- array-context program.

Nothing in the reference defines a mixture EOS, transport model or reaction mechanism (SURVEY.md §8c:
"parity unpinned"; §8d c4: "a small builder-chosen mechanism"), so the model is fixed HERE and
documented; like ``operators.py`` it is written once against the reference's array-context API
(/root/reference/pkg/src/laze/frontend.py:257-302) and runs unchanged on ``laze.ArrayContext``
(eager and lazy), on the NumPy oracle and on ``B200ArrayContext``.  On B200 the outlined functions
``dg_ms_flux`` / ``dg_ms_div`` / ``dg_ms_rhs`` are dispatched by name to the fused kernels of the flux
arrangement instantiated for ``C = d + 2 + ns`` fields (round 2: ``dgb_ms_flux`` / ``dgb_ms_div``, the same
``k_nsflux3`` / ``k_nsdiv8`` templates with the mixture physics; round 1 ran every op on the generic device
kernels, profiles/r01_multispecies.md).

Model
-----
* conserved state ``q = [rho, rho E, rho u_1..rho u_d, rho Y_1..rho Y_ns]`` stored ``(C, E, Np)``,
  ``C = d + 2 + ns``; ``rho`` is the mixture density and is transported itself;
* thermally perfect mixture with constant species properties: gas constants ``R_k``, heat
  capacities ``cv_k``, formation enthalpies ``h0_k``:
  ``R = sum Y_k R_k``, ``cv = sum Y_k cv_k``,
  ``T = (E/rho - |u|^2/2 - sum Y_k h0_k) / cv``, ``p = rho R T``, ``c^2 = (1 + R/cv) p / rho``;
* transport: constant ``mu``, ``kappa``, species diffusivity ``D`` (Fick, ``J_k = -rho D grad Y_k``, with
  the enthalpy flux ``sum h_k J_k``, ``h_k = h0_k + (cv_k + R_k) T``);
* chemistry: one irreversible Arrhenius step ``species a -> species b``:
  ``omega = A rho Y_a exp(-T_a / T)``, source ``-omega`` / ``+omega`` on ``rho Y_a`` / ``rho Y_b`` (the heat
  release is in ``h0``; total energy needs no source);
* discretisation = the single-species scheme: weak-form nodal DG, Rusanov inviscid flux with the
  mixture wave speed, BR1 (gradient of the conserved variables with the central flux; velocity, mass-fraction and
  temperature gradients by the chain rule; viscous flux central), periodic or prescribed far-field exterior state; partitioned meshes through ghost
  arrays (``rhs(q, ghost, halo_fn)``, ``HaloExchange.ms_rhs``).
"""
from __future__ import annotations

import numpy as np

from .discretization import BC_NONE, DGDiscretization
from .dofarray import DOFArray
from .operators import _traces


class Mixture:
    """Constant-property species set + one Arrhenius step (defaults: a 3-species toy mechanism
    fuel -> product in an inert bath, non-dimensional)."""

    def __init__(self, R=(1.0, 0.8, 1.2), cv=(2.5, 2.0, 3.0), h0=(0.5, -0.5, 0.0), reaction=(0, 1), A=5.0, Ta=2.0):
        self.R, self.cv, self.h0 = (np.asarray(v, dtype=np.float64) for v in (R, cv, h0))
        self.ns = self.R.size
        if not (self.cv.size == self.ns == self.h0.size) or self.ns < 1:
            raise ValueError("species property arrays must have one entry per species")
        self.reaction, self.A, self.Ta = (int(reaction[0]), int(reaction[1])), float(A), float(Ta)


def _thermo(actx, mix, q, dim):
    """Velocity, mass fractions, temperature, pressure, mixture R and cv from conserved fields."""
    rho, ener = q[0], q[1]
    inv_rho = 1.0 / rho
    vel = [q[2 + i] * inv_rho for i in range(dim)]
    Y = [q[2 + dim + k] * inv_rho for k in range(mix.ns)]
    ke = vel[0] * vel[0]
    for i in range(1, dim):
        ke = ke + vel[i] * vel[i]
    R = float(mix.R[0]) * Y[0]
    cv = float(mix.cv[0]) * Y[0]
    hf = float(mix.h0[0]) * Y[0]
    for k in range(1, mix.ns):
        R = R + float(mix.R[k]) * Y[k]
        cv = cv + float(mix.cv[k]) * Y[k]
        hf = hf + float(mix.h0[k]) * Y[k]
    T = (ener * inv_rho - 0.5 * ke - hf) / cv
    p = rho * R * T
    return vel, Y, T, p, R, cv


def _inviscid(actx, mix, q, dim):
    vel, Y, T, p, R, cv = _thermo(actx, mix, q, dim)
    C = len(q)
    flux = []
    for x in range(dim):
        fx = [q[2 + x], vel[x] * (q[1] + p)]
        for i in range(dim):
            mi = q[2 + i] * vel[x]
            fx.append(mi + p if i == x else mi)
        for k in range(mix.ns):
            fx.append(q[2 + dim + k] * vel[x])
        flux.append(fx)
    v2 = vel[0] * vel[0]
    for i in range(1, dim):
        v2 = v2 + vel[i] * vel[i]
    lam = actx.np.sqrt(v2) + actx.np.sqrt((1.0 + R / cv) * p / q[0])
    assert len(flux[0]) == C
    return flux, lam, (vel, Y, T, cv)


def _viscous(actx, mix, q, gq, prim, transport, dim):
    """``Fv[x][c]`` from the state and ``gq[x][c] = d q_c/dx_x``.  Velocity, mass-fraction and temperature gradients
    follow from the gradient of the conserved fields by the chain rule, like the single-species operator
    (``operators.viscous_flux``): ``T cv(Y) = E/rho - |u|^2/2 - sum Y_k h0_k``, so
    ``dT = (d(E/rho) - u.du - sum (h0_k + T cv_k) dY_k) / cv``."""
    mu, kappa, D = transport
    vel, Y, T, cv = prim
    rho = q[0]
    inv_rho = 1.0 / rho
    du = [[(gq[x][2 + i] - vel[i] * gq[x][0]) * inv_rho for x in range(dim)] for i in range(dim)]
    div = du[0][0]
    for i in range(1, dim):
        div = div + du[i][i]
    dY = [[(gq[x][2 + dim + k] - Y[k] * gq[x][0]) * inv_rho for x in range(dim)] for k in range(mix.ns)]
    flux = []
    for x in range(dim):
        tau = []
        for i in range(dim):
            t = mu * (du[i][x] + du[x][i])
            if i == x:
                t = t - (2.0 / 3.0) * mu * div
            tau.append(t)
        work = vel[0] * tau[0]
        for i in range(1, dim):
            work = work + vel[i] * tau[i]
        de = (gq[x][1] - (q[1] * inv_rho) * gq[x][0]) * inv_rho
        for i in range(dim):
            de = de - vel[i] * du[i][x]
        for k in range(mix.ns):
            de = de - (float(mix.h0[k]) + float(mix.cv[k]) * T) * dY[k][x]
        heat = kappa * (de / cv)
        spec = []
        for k in range(mix.ns):
            jk = (rho * D) * dY[k][x]                       # = -J_k
            hk = float(mix.h0[k]) + float(mix.cv[k] + mix.R[k]) * T
            heat = heat + hk * jk
            spec.append(jk)
        flux.append([None, work + heat] + tau + spec)
    return flux


def _ms_pass1(actx, mix, dim, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport):
    """Pass 1 (``dg_ms_flux``): BR1 gradient of ``q`` (central flux), then the total flux at every node, stored
    like ``dg_ns_flux`` of the single-species operator: planes ``r*C + c`` (``r < dim``) hold the contravariant,
    Jacobian-scaled components ``T[r][c] = sum_x jac*drdx[r,x] (F_inv - F_visc)[x][c]``, planes ``dim*C + c`` their sum
    over ``r`` and the last plane the mixture wave speed: shape ``((dim+1)*C + 1, E, Np)`` -- what pass 2 contracts and
    gathers and, on a partitioned mesh, what the second halo exchange carries."""
    C, E, Np = q.shape
    Nf = dim + 1
    Nfp = lift.shape[1] // Nf
    tr = [transport[k] for k in range(3)]
    nrm = [normals[x] for x in range(dim)]
    is_bnd = actx.np.not_equal(bc_kind, BC_NONE)
    qc = [q[c] for c in range(C)]
    finv, lam, prim = _inviscid(actx, mix, qc, dim)
    vol = actx.np.einsum("rij,rxe,cej->xcei", Sw, drdx, q)
    wm, wp = _traces(actx, q, ghost, vmap_m, vmap_p, C, E, Np, Nf, Nfp)
    far = [qfar[c] for c in range(C)]
    wpl = [actx.np.where(is_bnd, far[c], wp[c]) for c in range(C)]
    wstar = [fscale * (0.5 * (wm[c] + wpl[c])) for c in range(C)]
    fs = actx.np.stack([actx.np.stack([nrm[x] * wstar[c] for c in range(C)]) for x in range(dim)])
    gW = actx.np.einsum("if,xcef->xcei", lift, actx.np.reshape(fs, (dim, C, E, Nf * Nfp))) - vol
    gq = [[gW[x][c] for c in range(C)] for x in range(dim)]
    fvis = _viscous(actx, mix, qc, gq, prim, tr, dim)
    ftot = [[finv[x][c] if fvis[x][c] is None else finv[x][c] - fvis[x][c] for c in range(C)] for x in range(dim)]
    fstack = actx.np.stack([actx.np.stack(fx) for fx in ftot])                          # (d, C, E, Np)
    T = actx.np.einsum("rxe,e,xcej->rcej", drdx, jac, fstack)
    tsum = T[0] + T[1]
    for r in range(2, dim):
        tsum = tsum + T[r]
    return actx.np.concatenate([actx.np.reshape(T, (dim * C, E, Np)), tsum, actx.np.reshape(lam, (1, E, Np))])


def _ms_pass2(actx, mix, dim, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p,
              bc_kind, qfar):
    """Pass 2 (``dg_ms_div``): ``rhs = (1/J)(sum_r Sw_r T_r - lift(sJ F*.n)) + chemistry``; the scaled normal flux of
    either side of a face is one plane group of pass 1 (``facemat``, as in ``dg_ns_div``), Rusanov with the mixture
    wave speed; far-field boundary faces: inviscid flux of the exterior state, viscous flux of the interior one."""
    C, E, Np = q.shape
    Nf = dim + 1
    Nfp = lift.shape[1] // Nf
    ns = mix.ns
    L = C + (dim + 1) * C + 1
    nrm = [normals[x] for x in range(dim)]
    is_bnd = actx.np.not_equal(bc_kind, BC_NONE)
    far = [qfar[c] for c in range(C)]
    vol = actx.np.einsum("rij,rcej->cei", Sw, actx.np.reshape(T[0:dim * C], (dim, C, E, Np)))
    planes = actx.np.concatenate([q, T])                                                # q, plane groups, lam
    gplanes = None if ghost is None else actx.np.concatenate([ghost, Tghost])
    tm, tp = _traces(actx, planes, gplanes, vmap_m, vmap_p, L, E, Np, Nf, Nfp)
    sj = fscale * actx.np.reshape(jac, (E, 1, 1))                                       # face Jacobian (E, Nf, 1)
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
    ffar, lam_far, _ = _inviscid(actx, mix, far, dim)
    fmi, _, _ = _inviscid(actx, mix, qm, dim)
    lam_b = actx.np.maximum(lam_m, lam_far)
    fstar = []
    for c in range(C):
        fnb = nrm[0] * (ffar[0][c] - fmi[0][c])
        for x in range(1, dim):
            fnb = fnb + nrm[x] * (ffar[x][c] - fmi[x][c])
        f_int = 0.5 * (own[c] - nbr[c]) + 0.5 * sj * actx.np.maximum(lam_m, lam_p) * (qm[c] - qp[c])
        f_bnd = own[c] + 0.5 * sj * fnb + 0.5 * sj * lam_b * (qm[c] - far[c])
        fstar.append(actx.np.where(is_bnd, f_bnd, f_int))
    fsx = actx.np.reshape(actx.np.stack(fstar), (C, E, Nf * Nfp))
    rhs = (vol - actx.np.einsum("if,cef->cei", lift, fsx)) / actx.np.reshape(jac, (E, 1))
    # chemistry: one Arrhenius step a -> b
    qc = [q[c] for c in range(C)]
    Tn = _thermo(actx, mix, qc, dim)[2]
    a, b = mix.reaction
    omega = mix.A * qc[2 + dim + a] * actx.np.exp((-mix.Ta) / Tn)
    zero = 0.0 * omega
    src = [zero] * (2 + dim) + [(-1.0 * omega) if k == a else (omega if k == b else zero) for k in range(ns)]
    return rhs + actx.np.stack(src)


def _make_ms_functions(dim, mix):
    """The outlined functions -- the plugin boundary of the multi-species operator: ``dg_ms_rhs`` (single domain, both
    passes) and, for partitioned meshes, ``dg_ms_flux`` / ``dg_ms_div`` with ghost arrays (the halo of the flux planes
    is exchanged in between).  On B200 they are dispatched by name to the fused kernels (``fused.py``,
    ``dgb_ms_flux`` / ``dgb_ms_div``); the mixture travels with the function (``f.dg_mix``)."""
    def dg_ms_rhs(q, Sw, drdx, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar, transport):
        actx = dg_ms_rhs.actx
        T = _ms_pass1(actx, mix, dim, q, None, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport)
        return _ms_pass2(actx, mix, dim, q, T, None, None, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m,
                         vmap_p, bc_kind, qfar)

    def dg_ms_flux(q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p, bc_kind, qfar, transport):
        return _ms_pass1(dg_ms_flux.actx, mix, dim, q, ghost, Sw, drdx, jac, lift, normals, fscale, vmap_m, vmap_p,
                         bc_kind, qfar, transport)

    def dg_ms_div(q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat, facemat_p, vmap_m, vmap_p, bc_kind, qfar):
        return _ms_pass2(dg_ms_div.actx, mix, dim, q, T, ghost, Tghost, Sw, jac, lift, normals, fscale, facemat,
                         facemat_p, vmap_m, vmap_p, bc_kind, qfar)
    return dg_ms_rhs, dg_ms_flux, dg_ms_div


class MultispeciesOperator:
    """``rhs(q)`` of the multi-species reactive Navier-Stokes equations; ``q``: ``DOFArray (C, E, Np)``.
    Boundaries: periodic, or far-field (every tagged boundary face takes ``farfield`` as exterior state)."""

    def __init__(self, dcoll: DGDiscretization, mixture: Mixture | None = None, mu=1e-2, kappa=2e-2, diffusivity=1e-2,
                 farfield=None, graph: bool | None = None, fused: bool = True):
        """``fused`` (default): the outlined functions go through ``actx.outline`` -- on B200 that is the by-name
        dispatch to the fused kernels; ``fused=False`` runs their bodies op by op on whatever the context provides
        (the round-1 path, kept as an independent cross-check on the device).  ``graph`` (device contexts only;
        default on) applies to functions that are NOT fused: evaluate them through ``actx.compile(f, graph=True)`` --
        first call eager, second call captured into one CUDA graph, later calls replayed -- instead of ~800
        separately dispatched kernels."""
        self.dcoll, self.actx, self.dim = dcoll, dcoll.actx, dcoll.dim
        self.mix = mixture or Mixture()
        self.ncomp = self.dim + 2 + self.mix.ns
        if farfield is None:
            farfield = self.state_from_primitive(1.0, np.zeros(self.dim), 1.0, np.full(self.mix.ns, 1.0 / self.mix.ns))
        self.qfar_host = np.asarray(farfield, dtype=np.float64).reshape(self.ncomp)
        self.qfar = self.actx.from_numpy(self.qfar_host.reshape(self.ncomp, 1, 1, 1))
        self.transport = self.actx.from_numpy(np.array([mu, kappa, diffusivity], dtype=np.float64))
        if graph is None:
            graph = hasattr(self.actx, "lib")
        fns = []
        for f in _make_ms_functions(self.dim, self.mix):
            f.actx = self.actx
            f.dg_dim = self.dim
            f.dg_mix = self.mix
            g = self.actx.outline(f) if fused else f
            # hand-fused on the device (fused.py); a function that is NOT dispatched to the fused kernels (edited
            # body) runs op by op on the device, where one CUDA graph per right-hand side removes the dispatch cost
            fns.append(self.actx.compile(g, graph=True) if (graph and not getattr(g, "fused", False)) else g)
        self._f, self._flux, self._div = fns

    def state_from_primitive(self, rho, vel, T, Y):
        """Conserved state (any broadcastable shapes) from density, velocity, temperature, mass fractions."""
        mix = self.mix
        Y = [np.asarray(y, dtype=np.float64) for y in Y]
        vel = [np.asarray(v, dtype=np.float64) for v in vel]
        rho = np.asarray(rho, dtype=np.float64)
        cv = sum(mix.cv[k] * Y[k] for k in range(mix.ns))
        hf = sum(mix.h0[k] * Y[k] for k in range(mix.ns))
        e = cv * T + hf + 0.5 * sum(v * v for v in vel)
        parts = [rho, rho * e] + [rho * v for v in vel] + [rho * y for y in Y]
        return np.stack(np.broadcast_arrays(*parts))

    def flux(self, q, ghost):
        """Pass 1 on a partitioned mesh: the flux planes of the owned elements (raw array ``((dim+1)*C + 1, E, Np)``)."""
        d = self.dcoll
        q = q.data if isinstance(q, DOFArray) else q
        return self._flux(q, ghost, d.Sw, d.drdx, d.jac, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p, d.bc_kind,
                          self.qfar, self.transport)

    def div(self, q, T, ghost=None, Tghost=None) -> DOFArray:
        """Pass 2 from the flux planes ``T`` of pass 1 (and, on a partitioned mesh, the ghost arrays of both)."""
        d = self.dcoll
        q = q.data if isinstance(q, DOFArray) else q
        return DOFArray(self.actx, self._div(q, T, ghost, Tghost, d.Sw, d.jac, d.lift, d.normals, d.fscale, d.facemat,
                                             d.facemat_p, d.vmap_m, d.vmap_p, d.bc_kind, self.qfar))

    def rhs(self, q: DOFArray, t=0.0, ghost=None, halo_fn=None) -> DOFArray:
        """Single domain: ``rhs(q)``.  Partitioned: ``ghost`` = halo of ``q`` and ``halo_fn(DOFArray of the flux
        planes) -> their halo`` (second exchange), like ``NavierStokesOperator.rhs``."""
        d = self.dcoll
        maps = (d.vmap_m, d.vmap_p, d.bc_kind, self.qfar)
        if ghost is None:
            return DOFArray(self.actx, self._f(q.data, d.Sw, d.drdx, d.jac, d.lift, d.normals, d.fscale, d.facemat,
                                               d.facemat_p, *maps, self.transport))
        T = self._flux(q.data, ghost, d.Sw, d.drdx, d.jac, d.lift, d.normals, d.fscale, *maps, self.transport)
        return DOFArray(self.actx, self._div(q.data, T, ghost, halo_fn(DOFArray(self.actx, T)), d.Sw, d.jac, d.lift,
                                             d.normals, d.fscale, d.facemat, d.facemat_p, *maps))
