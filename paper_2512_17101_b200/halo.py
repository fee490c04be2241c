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

    def exchange(self, sends, recvs):
        """``sends``: list of (tensor, peer, tag); ``recvs``: list of (tensor, peer, tag).
        Posts everything as one batch and waits."""
        dist = self.dist
        ops = []
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

    def __init__(self, actx, plan: HaloPlan, comm: TorchCommunicator | None, ndofs: int):
        self.actx, self.plan, self.comm, self.ndofs = actx, plan, comm, ndofs
        self.nghost = plan.nghost
        self.on_device = hasattr(actx, "lib")
        self.send_tags = getattr(plan, "send_tags", plan.tags)
        if plan.nranks > 1 and comm is None:
            raise errors.CommunicationInSingleProcessGraph("a partitioned mesh needs a communicator")
        if self.on_device:
            self._send_idx = [actx.from_numpy(np.ascontiguousarray(s, dtype=np.int64)) for s in plan.send_local]
        self.bytes_per_exchange = 0
        self.messages_per_exchange = len(plan.peers)

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
        if self.on_device:
            actx = self.actx
            ghost = actx.empty(lead + (plan.nghost, self.ndofs))
            gview = ghost.t.view(-1, plan.nghost, self.ndofs)
            sends, recvs, keep = [], [], []
            for k, (peer, tag) in enumerate(zip(plan.peers, plan.tags)):
                a, b = plan.recv_slots[k]
                # ghosts of one peer are a strided slab of the ghost array: receive into a dense
                # buffer, scatter afterwards
                buf = actx.empty(lead + (b - a, self.ndofs))
                recvs.append((buf.t, peer, tag)); keep.append((buf, a, b))
                packed = self._pack(data, k)
                sends.append((packed.t, peer, self.send_tags[k]))
            actx.synchronize()                 # packed payloads complete before NCCL reads them
            self.comm.exchange(sends, recvs)
            for buf, a, b in keep:
                actx._scatter_into(ghost, ghost.t[..., a:b, :], buf)
            self.bytes_per_exchange = sum(t.numel() * 8 for t, _, _ in sends)
            return ghost
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

    # {{{ partition-aware right-hand sides
    def euler_rhs(self, op, q: DOFArray) -> DOFArray:
        return op.rhs(q, ghost=self.exchange(q.data))

    def ns_rhs(self, op, q: DOFArray) -> DOFArray:
        ghost = self.exchange(q.data)                                   # batch 1: state halos
        return op.rhs(q, ghost=ghost, halo_fn=lambda T: self.exchange(T.data))   # batch 2: flux-plane halos

    def ns_rhs_grad_form(self, op, q: DOFArray) -> DOFArray:
        ghost = self.exchange(q.data)
        return op.rhs_grad_form(q, ghost=ghost, halo_fn=lambda gq: self.exchange(gq.data))
    # }}}


def ring_slab_halo(actx, mesh, ncells_x, rank, nranks, order, lo_x=-1.0, hi_x=1.0):
    """Weak-scaling helper for bench.py: local mesh + ``HaloExchange`` of one rank of a ring."""
    from .dg.partition import ring_slab
    from .dg.simplex import simplex_element
    local, plan = ring_slab(mesh, ncells_x, rank, nranks, lo_x, hi_x)
    comm = TorchCommunicator() if nranks > 1 else None
    return local, HaloExchange(actx, plan, comm, simplex_element(mesh.dim, order).Np)
