"""Device-resident RK4 driver for the Navier-Stokes / Euler operators.

``rk4_step_fused`` (operators.py) already fuses every stage update into the right-hand-side pass;
it still allocates per stage and goes through the Python dispatch of the array context.  This
driver owns all stage storage, calls the C ABI directly and -- optionally -- captures the whole
step (4 stages x 2 kernels + the work-counter resets) in ONE CUDA graph, so a step is a single
launch: no allocation, no per-kernel Python, no launch gaps.  That is the B200 answer to the
"performance floor" the paper attributes to its dispatch layer
and what the reference's ``CompiledFunction`` (frontend.py:606-679: trace once, replay) stands for.

Scheme = classical RK4, accumulated stage by stage exactly like ``rk4_step_fused``:
    q1 = q + dt/2 k1        acc  = q + dt/6 k1
    q2 = q + dt/2 k2        acc += dt/3 k2
    q3 = q + dt   k3        acc += dt/3 k3
    qn = acc + dt/6 k4
"""
from __future__ import annotations

import numpy as np

from . import _cabi, errors, fused
from .dofarray import DOFArray


class DeviceRK4:
    """``stepper = DeviceRK4(op, q0, dt); stepper.step(); ...; q = stepper.state``.

    ``op``: ``NavierStokesOperator``, ``EulerOperator`` or ``MultispeciesOperator`` (3 species: the fused
    kernels) on a ``B200ArrayContext`` (single partition).  ``use_graph=True`` captures one step into a CUDA graph at construction.
    """

    def __init__(self, op, q0: DOFArray, dt: float, use_graph: bool = True):
        actx = op.actx
        if not hasattr(actx, "lib"):
            raise errors.LazeError("DeviceRK4 drives the B200 context; use rk4_step on other contexts")
        self.op, self.actx, self.dt = op, actx, float(dt)
        import torch
        self._torch = torch
        self.multi = hasattr(op, "mix")
        self.viscous = hasattr(op, "flux")
        shape = tuple(q0.data.shape)
        dim = op.dim
        if self.multi and op.mix.ns not in fused.MS_FUSED_SPECIES:
            raise errors.LazeError("DeviceRK4 needs the fused multi-species kernels (2, 3 or 4 species)")
        self.q = actx.empty(shape)
        self._d2d(self.q, actx._contiguous(q0.data))
        self.s1, self.s2, self.acc = actx.empty(shape), actx.empty(shape), actx.empty(shape)
        npl = fused.ms_flux_planes(dim, op.mix.ns) if self.multi else fused.flux_planes(dim)
        self.T = actx.empty((npl,) + shape[1:]) if self.viscous else None
        d = op.dcoll
        self.disc = fused.get_disc(actx, dim, self.q, 0, d.Sw, d.drdx, d.lift, d.normals, d.fscale, d.vmap_m, d.vmap_p,
                                   d.bc_kind, nspecies=op.mix.ns if self.multi else 0)
        if self.multi:
            mix = op.mix
            self._mix = np.ascontiguousarray(np.concatenate(
                [[mix.ns], mix.R, mix.cv, mix.h0, [mix.A, mix.Ta, mix.reaction[0], mix.reaction[1]]]).astype(np.float64))
            self._tr = np.ascontiguousarray(np.asarray(op.transport.host_value(), dtype=np.float64).reshape(3))
        if self.viscous:
            fused._bind_jacobian(actx, self.disc, d.jac)
            fused._check_facemat(self.disc, d.facemat, d.facemat_p)
        self.nsteps = 0
        self.graph = None
        self._enqueue_step()              # warm-up outside capture (first-launch attribute setup); undone below
        self._d2d(self.q, actx._contiguous(q0.data))
        actx.synchronize()
        if use_graph:
            import torch
            # capture needs a non-default stream: the context launches on a side stream for the duration
            self.graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device=actx.device)
            cap.wait_stream(actx.stream)
            home, actx.stream = actx.stream, cap
            try:
                with torch.cuda.graph(self.graph, stream=cap):
                    self._enqueue_step()
            finally:
                actx.stream = home
            home.wait_stream(cap)
            # capture does not execute: self.q still holds q0; replays run on the context's own stream

    # {{{ one step = 4 fused stages + copy-back, all on the context's stream
    def _d2d(self, dst, src):
        _cabi.check(self.actx.lib.dgb_memcpy_d2d(dst.ptr, src.ptr, dst.size * 8, self.actx._st), "d2d")

    def _stage(self, qin, x1, out1, x2, out2, coef):
        actx, lib, op = self.actx, self.actx.lib, self.op
        rk = np.asarray(coef, dtype=np.float64)
        qf = op.qfar_host
        o2 = out2.ptr if out2 is not None else None
        x2p = x2.ptr if x2 is not None else None
        if self.multi:
            tr, mx = self._tr.ctypes.data, self._mix.ctypes.data
            _cabi.check(lib.dgb_ms_flux_range(self.disc.handle, qin.ptr, None, self.T.ptr, qf.ctypes.data, tr, mx, 0, -1,
                                              actx._st), "dg_ms_flux")
            _cabi.check(lib.dgb_ms_div_rk(self.disc.handle, qin.ptr, self.T.ptr, None, None, x1.ptr, out1.ptr, x2p, o2,
                                          rk.ctypes.data, qf.ctypes.data, tr, mx, actx._st), "dg_ms_div_rk")
            actx.launch_count += 2
            return
        ph = op.phys_host
        if self.viscous:
            _cabi.check(lib.dgb_ns_flux(self.disc.handle, qin.ptr, None, self.T.ptr, qf.ctypes.data, ph.ctypes.data,
                                        actx._st), "dg_ns_flux")
            _cabi.check(lib.dgb_ns_div_rk(self.disc.handle, qin.ptr, self.T.ptr, None, None, x1.ptr, out1.ptr, x2p, o2,
                                          rk.ctypes.data, qf.ctypes.data, ph.ctypes.data, actx._st), "dg_ns_div_rk")
            actx.launch_count += 2
        else:
            _cabi.check(lib.dgb_euler_rhs_rk(self.disc.handle, qin.ptr, None, x1.ptr, out1.ptr, x2p, o2, rk.ctypes.data,
                                             qf.ctypes.data, ph.ctypes.data, actx._st), "dg_euler_rhs_rk")
            actx.launch_count += 1

    def _enqueue_step(self):
        dt, q, s1, s2, acc = self.dt, self.q, self.s1, self.s2, self.acc
        self._stage(q, q, s1, q, acc, (1.0, 0.5 * dt, 1.0, dt / 6.0))
        self._stage(s1, q, s2, acc, acc, (1.0, 0.5 * dt, 1.0, dt / 3.0))
        self._stage(s2, q, s1, acc, acc, (1.0, dt, 1.0, dt / 3.0))
        self._stage(s1, acc, s2, None, None, (1.0, dt / 6.0, 0.0, 0.0))
        self._d2d(q, s2)
    # }}}

    def step(self, nsteps: int = 1):
        for _ in range(nsteps):
            if self.graph is not None:
                with self._torch.cuda.stream(self.actx.stream):
                    self.graph.replay()
            else:
                self._enqueue_step()
        self.nsteps += nsteps
        return self

    @property
    def state(self) -> DOFArray:
        """The current solution (a view of the driver's buffer: copy it before stepping on)."""
        return DOFArray(self.actx, self.q)

    @property
    def time(self) -> float:
        return self.nsteps * self.dt

    # {{{ checkpoint / restart: .npz of the state + step counter + a mesh fingerprint
    def _fingerprint(self) -> np.ndarray:
        d = self.op.dcoll
        vp = np.asarray(d.vmap_p_host).reshape(-1)
        return np.array([d.dim, d.order, d.nelements, d.Np, int(vp.sum() % (1 << 61)), int(vp[::97].sum() % (1 << 61))],
                        dtype=np.int64)

    def _equations(self) -> str:
        return "multispecies" if self.multi else ("ns" if self.viscous else "euler")

    def save(self, path: str) -> None:
        """Write ``q`` (host copy), the step counter and ``dt``; bit-exact restart with ``restore``."""
        np.savez(path, q=self.actx.to_numpy(self.q), nsteps=np.int64(self.nsteps), dt=np.float64(self.dt),
                 mesh=self._fingerprint(), equations=self._equations())

    @classmethod
    def restore(cls, op, path: str, use_graph: bool = True) -> "DeviceRK4":
        """Continue a run saved with ``save`` on the same discretisation (checked by fingerprint)."""
        with np.load(path) as ck:
            q, nsteps, dt, mesh, eq = ck["q"], int(ck["nsteps"]), float(ck["dt"]), ck["mesh"], str(ck["equations"])
        stepper = cls(op, DOFArray(op.actx, op.actx.from_numpy(q)), dt, use_graph=use_graph)
        if not np.array_equal(mesh, stepper._fingerprint()) or eq != stepper._equations():
            raise errors.BindingMismatch("checkpoint was written for another mesh / order / equation set")
        stepper.nsteps = nsteps
        return stepper
    # }}}
