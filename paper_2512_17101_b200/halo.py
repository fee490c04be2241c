"""Face-halo exchange between mesh partitions (north-star item 4).

Message model = the reference's: one array per ``(source, destination, tag)``
(/root/reference/pkg/src/laze/distpart.py:396-411), receives conceptually posted up front, one
communication batch per dependency level -- Euler: one batch (state halos); Navier-Stokes: two
(state halos, then the halos of the pass-1 result -- flux planes, or gradients in the gradient
arrangement -- which depend on received data: distpart.py:168-176).

``TorchCommunicator`` moves the payloads with ``torch.distributed`` point-to-point ops: NCCL
send/recv over NVLink for device arrays, gloo for the CPU oracle context (tests).  All sends and
receives of a batch are posted together (``batch_isend_irecv`` = one ncclGroupStart/End).
"""
from __future__ import annotations

import numpy as np

from . import errors
from .dg.partition import HaloPlan
from .dofarray import DOFArray


class TorchCommunicator:
    """Point-to-point transport over an initialised ``torch.distributed`` process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise errors.CommunicationInSingleProcessGraph("torch.distributed is not initialised")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def exchange(self, sends, recvs):
        """``sends``: list of (tensor, peer, tag); ``recvs``: list of (tensor, peer, tag).
        Posts everything as one batch and waits."""
        dist = self.dist
        if self.backend == "gloo" and any(t.is_cuda for t, _, _ in list(sends) + list(recvs)):
            # test configuration only (two ranks sharing one GPU): gloo has no device send/recv, so the
            # payloads are staged through host memory.  The NCCL path below never does this.
            import torch
            torch.cuda.current_stream().synchronize()
            hs = [(t.detach().cpu(), peer, tag) for t, peer, tag in sends]
            hr = [(torch.empty(t.shape, dtype=t.dtype), peer, tag) for t, peer, tag in recvs]
            self.exchange(hs, hr)
            for (t, _, _), (h, _, _) in zip(recvs, hr):
                t.copy_(h)
            return
        ops = []
        if self.backend == "gloo":
            # gloo matches messages by tag only within a (source, destination) pair and needs dense CPU tensors
            sends = [(t.contiguous(), peer, tag) for t, peer, tag in sends]
        # a deterministic global order keeps NCCL's paired send/recv matching happy: receives and
        # sends are sorted by (tag, peer)
        for t, peer, tag in sorted(recvs, key=lambda x: (x[2], x[1])):
            ops.append(dist.P2POp(dist.irecv, t, peer, self.group, tag))
        for t, peer, tag in sorted(sends, key=lambda x: (x[2], x[1])):
            ops.append(dist.P2POp(dist.isend, t, peer, self.group, tag))
        if not ops:
            return
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class HaloExchange:
    """Packs the elements a peer needs, exchanges, and returns the ghost array of a field."""

    def __init__(self, actx, plan: HaloPlan, comm: TorchCommunicator | None, ndofs: int, transport: str = "nccl"):
        """``transport``: "nccl" = torch.distributed send/recv (NCCL over NVLink; gloo in tests);
        "peer" = the pack kernel stores the halo rows straight into the neighbour's ghost array through
        CUDA-IPC peer-mapped memory (device contexts only; ``comm`` is then used once, for the handles)."""
        self.actx, self.plan, self.comm, self.ndofs = actx, plan, comm, ndofs
        if transport not in ("nccl", "peer"):
            raise ValueError("transport must be 'nccl' or 'peer'")
        self.transport = transport
        self._channels = {}
        self.nghost = plan.nghost
        self.on_device = hasattr(actx, "lib")
        self.send_tags = getattr(plan, "send_tags", plan.tags)
        if plan.nranks > 1 and comm is None:
            raise errors.CommunicationInSingleProcessGraph("a partitioned mesh needs a communicator")
        if self.on_device:
            self._send_idx = [actx.from_numpy(np.ascontiguousarray(s, dtype=np.int64)) for s in plan.send_local]
        self.bytes_per_exchange = 0
        self.messages_per_exchange = len(plan.peers)
        # interior elements first + a communication stream: the exchange hides behind the interior
        # range of each pass (set ``overlap = False`` for the plain exchange-then-compute order)
        self.overlap = True
        # SMs the persistent kernels leave free while a halo is in flight, so that NCCL's send/recv kernel can
        # start at once on the communication stream instead of waiting for a CTA of the interior range to
        # retire (the peer transport has no communication kernel: its pack kernels run on the compute stream)
        self.sm_reserve = 8 if transport == "nccl" else 0

    # {{{ packing
    def _pack(self, data, k):
        """(lead..., E, Np) -> contiguous (lead..., n_k, Np) of the elements peer k needs."""
        sel = self.plan.send_local[k]
        if not self.on_device:
            return np.ascontiguousarray(np.asarray(data)[..., sel, :])
        import math
        from . import _cabi
        actx = self.actx
        src = actx._contiguous(data)
        lead = src.shape[:-2]
        ncomp = math.prod(lead) if lead else 1
        out = actx.empty(lead + (len(sel), self.ndofs))
        _cabi.check(actx.lib.dgb_pack_elements(out.ptr, src.ptr, self._send_idx[k].ptr, ncomp, src.shape[-2],
                                               len(sel), self.ndofs, actx._st), "halo pack")
        actx.launch_count += 1
        return out
    # }}}

    def exchange(self, data):
        """Ghost array ``(lead..., G, Np)`` for the field ``data`` ``(lead..., E, Np)``."""
        plan = self.plan
        if plan.nranks == 1 or not plan.peers:
            return None
        lead = tuple(data.shape[:-2])
        import torch
        if self.on_device and self.transport == "peer":
            from . import _cabi
            ch = self._peer_begin(data)
            shared = self._peer_end(ch)
            ghost = self.actx.empty(lead + (plan.nghost, self.ndofs))       # private copy: the shared array is released at once
            _cabi.check(self.actx.lib.dgb_memcpy_d2d(ghost.ptr, shared.ptr, ghost.size * 8, self.actx._st), "d2d")
            self._peer_release(ch)
            return ghost
        if self.on_device:
            # same transfers as the overlapped path, posted on the context's own stream (the NCCL
            # operations, the pack kernels before them and the consumers after them are then stream-ordered)
            return self.exchange_end(self.exchange_begin(data, stream=self.actx.stream))
        ghost = np.empty(lead + (plan.nghost, self.ndofs))
        sends, recvs, bufs = [], [], []
        for k, (peer, tag) in enumerate(zip(plan.peers, plan.tags)):
            a, b = plan.recv_slots[k]
            buf = torch.empty(lead + (b - a, self.ndofs), dtype=torch.float64)
            recvs.append((buf, peer, tag)); bufs.append((buf, a, b))
            sends.append((torch.from_numpy(self._pack(data, k)), peer, self.send_tags[k]))
        self.comm.exchange(sends, recvs)
        for buf, a, b in bufs:
            ghost[..., a:b, :] = buf.numpy()
        self.bytes_per_exchange = sum(t.numel() * 8 for t, _, _ in sends)
        return self.actx.from_numpy(ghost)

    # {{{ asynchronous exchange on a communication stream (device contexts)
    @property
    def comm_stream(self):
        if getattr(self, "_comm_stream", None) is None:
            import torch
            self._comm_stream = torch.cuda.Stream(device=self.actx.device)
        return self._comm_stream

    # components of a message travel as separate transfers of one batch (one NCCL group): for component c the
    # rows [a, b) of a peer are contiguous both in the packed send buffer (lead, n_k, Np) and in the ghost
    # array (lead, G, Np), so the payload is received IN PLACE -- no staging buffer, no scatter kernel
    _COMP_TAGS = 64

    def exchange_begin(self, data, stream=None):
        """Pack on the compute stream, then post the whole batch on the communication stream
        (NCCL group of sends and receives over NVLink).  Returns a ticket for ``exchange_end``;
        kernels enqueued on the compute stream in between overlap the transfer."""
        import math
        import torch
        plan, actx = self.plan, self.actx
        lead = tuple(data.shape[:-2])
        ncomp = math.prod(lead) if lead else 1
        if ncomp > self._COMP_TAGS:
            raise errors.ShapeMismatch(f"halo messages carry at most {self._COMP_TAGS} components, got {ncomp}")
        ghost = actx.empty(lead + (plan.nghost, self.ndofs))
        gview = ghost.t.view(ncomp, plan.nghost, self.ndofs)
        sends, recvs, keep = [], [], []
        for k, (peer, tag) in enumerate(zip(plan.peers, plan.tags)):
            a, b = plan.recv_slots[k]
            packed = self._pack(data, k)
            keep.append(packed)
            pview = packed.t.view(ncomp, -1, self.ndofs)
            for c in range(ncomp):
                recvs.append((gview[c, a:b], peer, tag * self._COMP_TAGS + c))
                sends.append((pview[c], peer, self.send_tags[k] * self._COMP_TAGS + c))
        cs = self.comm_stream if stream is None else stream
        if cs is not actx.stream:
            packed_ready = torch.cuda.Event()
            packed_ready.record(actx.stream)
            cs.wait_event(packed_ready)
        with torch.cuda.stream(cs):
            if cs is not actx.stream:
                ghost.t.record_stream(cs)
                for pk in keep:
                    pk.t.record_stream(cs)
            self.comm.exchange(sends, recvs)
            done = torch.cuda.Event()
            done.record(cs)
        self.bytes_per_exchange = sum(pk.size * 8 for pk in keep)
        self.transfers_per_exchange = len(sends)
        return ghost, keep, done, cs

    def exchange_end(self, ticket):
        """Make the compute stream wait for the transfer; the ghost array was filled in place."""
        ghost, _keep, done, cs = ticket
        if cs is not self.actx.stream:
            self.actx.stream.wait_event(done)
        return ghost
    # }}}

    # {{{ peer-memory transport: pack kernel -> neighbour's ghost array over NVLink, flags for ordering
    class _Channel:
        pass

    def _peer_channel(self, lead):
        """Ghost array + flags of one message family (state halos, flux-plane halos), created on first use:
        allocate, publish the IPC handles, map the neighbours' arrays, pair the plan entries."""
        import ctypes as C
        import math
        import torch
        from . import _cabi
        key = tuple(lead)
        ch = self._channels.get(key)
        if ch is not None:
            return ch
        actx, plan, lib, dist = self.actx, self.plan, self.actx.lib, self.comm.dist
        ncomp = math.prod(lead) if lead else 1
        npeers = len(plan.peers)
        ch = HaloExchange._Channel()
        ch.lead, ch.ncomp, ch.epoch = key, ncomp, 0
        gh, fl = C.c_void_p(), C.c_void_p()
        hg, hf = C.create_string_buffer(64), C.create_string_buffer(64)
        _cabi.check(lib.dgb_ipc_alloc(C.byref(gh), ncomp * max(plan.nghost, 1) * self.ndofs * 8, hg), "ipc alloc")
        _cabi.check(lib.dgb_ipc_alloc(C.byref(fl), 16 * max(npeers, 1), hf), "ipc alloc")
        ch.ghost_ptr, ch.flags_ptr = gh.value, fl.value            # flags: ready[npeers] then ack[npeers] (u64)

        class _Raw:
            __cuda_array_interface__ = {"shape": key + (plan.nghost, self.ndofs), "typestr": "<f8",
                                        "data": (gh.value, False), "version": 3, "strides": None}
        from .actx import DeviceArray
        ch.ghost = DeviceArray(actx, torch.as_tensor(_Raw(), device=actx.device))
        info = {"rank": plan.rank, "key": key, "ghost": hg.raw, "flags": hf.raw, "nghost": plan.nghost,
                "peers": list(plan.peers), "tags": list(plan.tags), "send_tags": list(self.send_tags),
                "recv_slots": [tuple(x) for x in plan.recv_slots]}
        infos = [None] * self.comm.size
        dist.all_gather_object(infos, info, group=self.comm.group)
        by_rank = {i["rank"]: i for i in infos}
        opened = {}

        def peer_ptrs(r):
            if r not in opened:
                a, b = C.c_void_p(), C.c_void_p()
                if r == plan.rank:
                    a.value, b.value = ch.ghost_ptr, ch.flags_ptr
                else:
                    _cabi.check(lib.dgb_ipc_open(C.byref(a), by_rank[r]["ghost"]), "ipc open")
                    _cabi.check(lib.dgb_ipc_open(C.byref(b), by_rank[r]["flags"]), "ipc open")
                opened[r] = (a.value, b.value)
            return opened[r]

        ch.send = []      # per entry k: (peer ghost ptr, peer nghost, peer slot0, peer ready-flag ptr)
        ch.ack_to = []    # per entry k: ack-flag ptr at the peer for the message RECEIVED through entry k
        for k, peer in enumerate(plan.peers):
            pi = by_rank[peer]
            if pi["key"] != key:
                raise errors.MismatchedCommunication(f"rank {peer} opened channel {pi['key']}, expected {key}")
            np_ = len(pi["peers"])
            j = [jj for jj in range(np_) if pi["peers"][jj] == plan.rank and pi["tags"][jj] == self.send_tags[k]]
            jb = [jj for jj in range(np_) if pi["peers"][jj] == plan.rank and pi["send_tags"][jj] == plan.tags[k]]
            if len(j) != 1 or len(jb) != 1:
                raise errors.MismatchedCommunication(f"no unique partner entry at rank {peer}",
                                                     keys=[(plan.rank, peer, self.send_tags[k])])
            gp, fp = peer_ptrs(peer)
            a, b = pi["recv_slots"][j[0]]
            if b - a != len(plan.send_local[k]):
                raise errors.MismatchedCommunication(f"message to rank {peer}: {len(plan.send_local[k])} elements sent, "
                                                     f"{b - a} expected", keys=[(plan.rank, peer, self.send_tags[k])])
            ch.send.append((gp, pi["nghost"], a, fp + 8 * j[0]))
            ch.ack_to.append(fp + 8 * (np_ + jb[0]))
        ch.keep = opened
        dist.barrier(group=self.comm.group)
        self._channels[key] = ch
        return ch

    def _peer_begin(self, data):
        import math
        from . import _cabi
        actx, lib, plan = self.actx, self.actx.lib, self.plan
        lead = tuple(data.shape[:-2])
        ch = self._peer_channel(lead)
        ch.epoch += 1
        src = actx._contiguous(data)
        npeers = len(plan.peers)
        nbytes = 0
        for k in range(npeers):
            gp, ng, slot0, ready = ch.send[k]
            # the neighbour has consumed what I stored there last time
            _cabi.check(lib.dgb_flag_wait(ch.flags_ptr + 8 * (npeers + k), ch.epoch - 1, actx._st), "halo ack wait")
            _cabi.check(lib.dgb_pack_elements_to(gp, ng, slot0, src.ptr, self._send_idx[k].ptr, ch.ncomp, src.shape[-2],
                                                 len(plan.send_local[k]), self.ndofs, actx._st), "halo pack (peer)")
            _cabi.check(lib.dgb_flag_signal(ready, ch.epoch, actx._st), "halo signal")
            actx.launch_count += 3
            nbytes += ch.ncomp * len(plan.send_local[k]) * self.ndofs * 8
        self.bytes_per_exchange = nbytes
        self._keep_src = src
        return ch

    def _peer_end(self, ch):
        from . import _cabi
        for k in range(len(self.plan.peers)):
            _cabi.check(self.actx.lib.dgb_flag_wait(ch.flags_ptr + 8 * k, ch.epoch, self.actx._st), "halo wait")
            self.actx.launch_count += 1
        return ch.ghost

    def _peer_release(self, ch):
        """Everything enqueued so far has read the ghost array: let the neighbours overwrite it."""
        from . import _cabi
        for k in range(len(self.plan.peers)):
            _cabi.check(self.actx.lib.dgb_flag_signal(ch.ack_to[k], ch.epoch, self.actx._st), "halo ack")
            self.actx.launch_count += 1
    # }}}

    def close(self):
        """Peer transport: wait until every rank is done with everybody's ghost arrays, then unmap and free
        them.  (Call before the process group is destroyed; a no-op for the NCCL transport.)"""
        if not self._channels:
            return
        from . import _cabi
        self.actx.synchronize()
        self.comm.dist.barrier(group=self.comm.group)
        for ch in self._channels.values():
            for r, (gp, fp) in ch.keep.items():
                if r != self.plan.rank:
                    _cabi.check(self.actx.lib.dgb_ipc_close(gp), "ipc close")
                    _cabi.check(self.actx.lib.dgb_ipc_close(fp), "ipc close")
        self.comm.dist.barrier(group=self.comm.group)        # nobody still maps what is freed next
        for ch in self._channels.values():
            ch.ghost = None
            _cabi.check(self.actx.lib.dgb_free(ch.ghost_ptr), "free")
            _cabi.check(self.actx.lib.dgb_free(ch.flags_ptr), "free")
        self._channels = {}

    # {{{ transport-independent begin / end / release
    def _begin(self, data):
        return self._peer_begin(data) if self.transport == "peer" else self.exchange_begin(data)

    def _reserve(self, on: bool):
        if self.on_device and self.sm_reserve:
            from . import _cabi
            _cabi.check(self.actx.lib.dgb_set_sm_reserve(self.sm_reserve if on else 0), "dgb_set_sm_reserve")

    def _ghost_of(self, ticket):
        return ticket.ghost if self.transport == "peer" else ticket[0]

    def _end(self, ticket):
        return self._peer_end(ticket) if self.transport == "peer" else self.exchange_end(ticket)

    def _release(self, ticket):
        if self.transport == "peer":
            self._peer_release(ticket)
    # }}}

    # {{{ partition-aware right-hand sides
    def _can_overlap(self):
        return (self.on_device and self.overlap and self.plan.nranks > 1 and bool(self.plan.peers)
                and self.plan.n_interior is not None)

    def euler_rhs(self, op, q: DOFArray) -> DOFArray:
        if not self._can_overlap():
            return op.rhs(q, ghost=self.exchange(q.data))
        from . import fused
        actx, nI, E = self.actx, self.plan.n_interior, self.plan.nlocal
        t1 = self._begin(q.data)                                        # state halos in flight ...
        out = actx.empty(q.data.shape)
        self._reserve(True)
        fused.euler_rhs_range(actx, op, q.data, self._ghost_of(t1), out, 0, nI)   # ... under the interior elements
        self._reserve(False)
        ghost = self._end(t1)
        fused.euler_rhs_range(actx, op, q.data, ghost, out, nI, E)
        self._release(t1)
        return DOFArray(actx, out)

    def ns_rhs(self, op, q: DOFArray) -> DOFArray:
        if not self._can_overlap():
            ghost = self.exchange(q.data)                                   # batch 1: state halos
            return op.rhs(q, ghost=ghost, halo_fn=lambda T: self.exchange(T.data))   # batch 2: flux-plane halos
        from . import fused
        actx, nI, E = self.actx, self.plan.n_interior, self.plan.nlocal
        dim = op.dim
        t1 = self._begin(q.data)                                            # batch 1 in flight ...
        T = actx.empty((fused.flux_planes(dim),) + tuple(q.data.shape[1:]))
        self._reserve(True)
        fused.ns_flux_range(actx, op, q.data, self._ghost_of(t1), T, 0, nI)  # ... under pass 1 of the interior
        self._reserve(False)
        ghost = self._end(t1)
        fused.ns_flux_range(actx, op, q.data, ghost, T, nI, E)              # pass 1 next to the partition boundary
        t2 = self._begin(T)                                                 # batch 2 in flight ...
        out = actx.empty(q.data.shape)
        self._reserve(True)
        fused.ns_div_range(actx, op, q.data, T, ghost, self._ghost_of(t2), out, 0, nI)   # ... under pass 2 of the interior
        self._reserve(False)
        tghost = self._end(t2)
        fused.ns_div_range(actx, op, q.data, T, ghost, tghost, out, nI, E)
        self._release(t1)
        self._release(t2)
        return DOFArray(actx, out)

    def ns_rhs_rk(self, op, q: DOFArray, x1: DOFArray, x2: DOFArray, coef, t=0.0):
        """``(a1*x1 + b1*rhs(q), a2*x2 + b2*rhs(q))`` on a partitioned mesh, ``coef = (a1, b1, a2, b2)``: the stage update
        is fused into the store of pass 2 (``dgb_ns_div_rk_range``) on the device; elsewhere (oracle context, no
        overlap) it is the exchange-then-compute right-hand side followed by array arithmetic.  Same contract as
        ``NavierStokesOperator.rhs_rk``, so ``rk4_step_fused(PartitionedOperator(halo, op), q, t, dt)`` steps in time."""
        a1, b1, a2, b2 = (float(c) for c in coef)
        if not self._can_overlap():
            r = self.ns_rhs(op, q)
            return a1 * x1 + b1 * r, a2 * x2 + b2 * r
        from . import fused
        actx, nI, E = self.actx, self.plan.n_interior, self.plan.nlocal
        t1 = self._begin(q.data)
        T = actx.empty((fused.flux_planes(op.dim),) + tuple(q.data.shape[1:]))
        self._reserve(True)
        fused.ns_flux_range(actx, op, q.data, self._ghost_of(t1), T, 0, nI)
        self._reserve(False)
        ghost = self._end(t1)
        fused.ns_flux_range(actx, op, q.data, ghost, T, nI, E)
        t2 = self._begin(T)
        o1, o2 = actx.empty(q.data.shape), actx.empty(q.data.shape)
        self._reserve(True)
        fused.ns_div_rk_range(actx, op, q.data, T, ghost, self._ghost_of(t2), x1.data, o1, x2.data, o2, (a1, b1, a2, b2), 0, nI)
        self._reserve(False)
        tghost = self._end(t2)
        fused.ns_div_rk_range(actx, op, q.data, T, ghost, tghost, x1.data, o1, x2.data, o2, (a1, b1, a2, b2), nI, E)
        self._release(t1)
        self._release(t2)
        return DOFArray(actx, o1), DOFArray(actx, o2)

    def ms_rhs(self, op, q: DOFArray) -> DOFArray:
        """Multi-species operator: state halos, then flux-plane halos; with the fused kernels each exchange runs
        under the interior range of its pass, like ``ns_rhs``."""
        if not (self._can_overlap() and getattr(op._flux, "fused", False) and getattr(op._div, "fused", False)):
            ghost = self.exchange(q.data)
            return op.rhs(q, ghost=ghost, halo_fn=lambda FL: self.exchange(FL.data))
        from . import fused
        actx, nI, E = self.actx, self.plan.n_interior, self.plan.nlocal
        t1 = self._begin(q.data)
        T = actx.empty((fused.ms_flux_planes(op.dim, op.mix.ns),) + tuple(q.data.shape[1:]))
        self._reserve(True)
        fused.ms_flux_range(actx, op, q.data, self._ghost_of(t1), T, 0, nI)
        self._reserve(False)
        ghost = self._end(t1)
        fused.ms_flux_range(actx, op, q.data, ghost, T, nI, E)
        t2 = self._begin(T)
        out = actx.empty(q.data.shape)
        self._reserve(True)
        fused.ms_div_range(actx, op, q.data, T, ghost, self._ghost_of(t2), out, 0, nI)
        self._reserve(False)
        tghost = self._end(t2)
        fused.ms_div_range(actx, op, q.data, T, ghost, tghost, out, nI, E)
        self._release(t1)
        self._release(t2)
        return DOFArray(actx, out)

    def ns_rhs_grad_form(self, op, q: DOFArray) -> DOFArray:
        ghost = self.exchange(q.data)
        return op.rhs_grad_form(q, ghost=ghost, halo_fn=lambda gq: self.exchange(gq.data))
    # }}}


class PartitionedOperator:
    """``rhs`` / ``rhs_rk`` of a Navier-Stokes operator on one rank of a partitioned mesh (halo exchanges inside), with
    the interface ``rk4_step`` / ``rk4_step_fused`` expect of an operator."""

    def __init__(self, halo: HaloExchange, op):
        self.halo, self.op, self.actx, self.dim, self.dcoll = halo, op, op.actx, op.dim, op.dcoll

    def rhs(self, q: DOFArray, t=0.0) -> DOFArray:
        return self.halo.ns_rhs(self.op, q)

    def rhs_rk(self, q: DOFArray, x1: DOFArray, x2: DOFArray, coef, t=0.0):
        return self.halo.ns_rhs_rk(self.op, q, x1, x2, coef, t)


def ring_slab_halo(actx, mesh, ncells_x, rank, nranks, order, lo_x=-1.0, hi_x=1.0, transport="nccl"):
    """Weak-scaling helper for bench.py: local mesh + ``HaloExchange`` of one rank of a ring."""
    from .dg.partition import ring_slab
    from .dg.simplex import simplex_element
    from .dg.partition import interior_first
    local, plan = ring_slab(mesh, ncells_x, rank, nranks, lo_x, hi_x)
    if nranks > 1:
        local, plan = interior_first(local, plan)
    comm = TorchCommunicator() if nranks > 1 else None
    return local, HaloExchange(actx, plan, comm, simplex_element(mesh.dim, order).Np, transport=transport)
