"""Mesh partitioning and halo plans (host, NumPy, integer-exact).

The reference's only parallelism is rank-partitioned graphs that exchange arrays point to point
through Send / Receive nodes (/root/reference/pkg/src/laze/adfg.py:380-399,834-869;
/root/reference/pkg/src/laze/distpart.py:97-196).  Here the unit that is partitioned is the
element set of a mesh; what crosses ranks is the nodal data of the elements adjacent to a
partition boundary ("halo" elements), one message per (source, destination, tag) -- the same
keying as the reference's transport (distpart.py:396-411).

A rank-local mesh keeps its ``E`` owned elements first and addresses the remote neighbours as
"ghost" elements ``E .. E+G-1``; face index maps into ``[E*Np, (E+G)*Np)`` therefore refer to the
received halo array.  Ghosts are grouped by owning rank and, inside a group, ordered by GLOBAL
element id, which both sides can compute without talking to each other.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh


@dataclass
class HaloPlan:
    rank: int
    nranks: int
    nlocal: int
    nghost: int
    peers: list[int]                          # ascending peer ranks (a peer may repeat with another tag)
    tags: list[int]                           # message tag per entry of `peers`
    send_local: list[np.ndarray]              # per peer: local element ids to send (int64)
    recv_slots: list[tuple[int, int]]         # per peer: [start, stop) ghost slots filled by its message
    global_ids: np.ndarray | None = None      # (nlocal,) global element id of each local element
    n_interior: int | None = None             # elements [0, n_interior) touch no ghost (interior_first)

    def validate_against(self, other: "HaloPlan") -> None:
        """Symmetric, shape-matched plan check before the first exchange (the reference validates
        pairing and shapes at plan time: distpart.py:143-162)."""
        from ..errors import MismatchedCommunication
        for k, (peer, tag) in enumerate(zip(self.peers, self.tags)):
            if peer != other.rank:
                continue
            match = [j for j, (p2, t2) in enumerate(zip(other.peers, other.tags)) if p2 == self.rank and t2 == tag]
            if len(match) != 1:
                raise MismatchedCommunication(f"rank {self.rank} sends to {peer} with tag {tag} but the peer "
                                              f"has no matching receive", keys=[(self.rank, peer, tag)])
            j = match[0]
            n_recv = other.recv_slots[j][1] - other.recv_slots[j][0]
            if n_recv != len(self.send_local[k]):
                raise MismatchedCommunication(
                    f"message ({self.rank}->{peer}, tag {tag}): {len(self.send_local[k])} elements sent, "
                    f"{n_recv} expected", keys=[(self.rank, peer, tag)])


def partition_elements(mesh: Mesh, nparts: int) -> np.ndarray:
    """Recursive coordinate bisection of element centroids into ``nparts`` equal-size parts."""
    cent = mesh.vertices.mean(axis=1)
    part = np.zeros(mesh.nelements, dtype=np.int64)

    def split(ids, lo, n):
        if n == 1:
            part[ids] = lo
            return
        ext = cent[ids].max(axis=0) - cent[ids].min(axis=0)
        ax = int(np.argmax(ext))
        order = ids[np.argsort(cent[ids, ax], kind="stable")]
        nl = n // 2
        cut = (len(order) * nl) // n
        split(order[:cut], lo, nl)
        split(order[cut:], lo + nl, n - nl)

    split(np.arange(mesh.nelements), 0, int(nparts))
    return part


def rank_mesh(mesh: Mesh, part: np.ndarray, rank: int) -> tuple[Mesh, HaloPlan]:
    """Local mesh + halo plan of one rank of a partitioned global mesh."""
    nranks = int(part.max()) + 1
    mine = np.nonzero(part == rank)[0]                       # ascending global ids
    E = mine.size
    g2l = np.full(mesh.nelements, -1, dtype=np.int64)
    g2l[mine] = np.arange(E)
    nbr_g = mesh.nbr_elem[mine]                              # (E, Nf) global neighbour ids
    nbr_rank = part[nbr_g]
    remote = (nbr_rank != rank) & (mesh.btag[mine] == 0)
    nbr_local = g2l[nbr_g]
    peers, tags, send_local, recv_slots = [], [], [], []
    slot = 0
    for r in sorted(set(nbr_rank[remote].tolist())):
        need = np.unique(nbr_g[remote & (nbr_rank == r)])    # global ids, ascending
        lut = {int(g): slot + k for k, g in enumerate(need)}
        sel = remote & (nbr_rank == r)
        nbr_local[sel] = E + np.array([lut[int(g)] for g in nbr_g[sel]], dtype=np.int64)
        # what r needs from me: my elements adjacent to r, ascending global id (r computes the same list)
        give = np.unique(mine[np.any(sel, axis=1)])
        peers.append(int(r)); tags.append(0)
        send_local.append(g2l[give])
        recv_slots.append((slot, slot + need.size))
        slot += need.size
    local = Mesh(mesh.dim, mesh.vertices[mine], mesh.vertex_ids[mine], nbr_local, mesh.nbr_face[mine].copy(),
                 mesh.nbr_perm[mine].copy(), mesh.btag[mine].copy(), nbr_rank=nbr_rank)
    plan = HaloPlan(rank, nranks, E, slot, peers, tags, send_local, recv_slots, global_ids=mine)
    return local, plan


def ring_slab(mesh: Mesh, ncells_x: int, rank: int, nranks: int, lo_x: float, hi_x: float) -> tuple[Mesh, HaloPlan]:
    """Weak-scaling decomposition without ever building the global mesh: every rank owns an
    identical box mesh that is periodic in all axes; the faces that cross the periodic wrap in x
    are re-targeted at the left / right neighbour rank of a ring (whose local mesh, and hence
    local element numbering, is identical).  The global domain is the ring of ``nranks`` boxes."""
    if nranks == 1:
        return mesh, HaloPlan(0, 1, mesh.nelements, 0, [], [], [], [])
    E = mesh.nelements
    h = (hi_x - lo_x) / ncells_x
    cell_x = np.floor((mesh.vertices[:, :, 0].min(axis=1) - lo_x) / h + 1e-9).astype(np.int64)
    nb_cell = cell_x[mesh.nbr_elem]
    interior = mesh.btag == 0
    to_left = interior & (cell_x[:, None] == 0) & (nb_cell == ncells_x - 1)
    to_right = interior & (cell_x[:, None] == ncells_x - 1) & (nb_cell == 0)
    if ncells_x < 3:
        raise ValueError("ring_slab needs at least 3 cells along x")
    nbr_local = mesh.nbr_elem.copy()
    left, right = (rank - 1) % nranks, (rank + 1) % nranks
    need_left = np.unique(mesh.nbr_elem[to_left])            # peer-local ids == my-local ids of layer n-1
    need_right = np.unique(mesh.nbr_elem[to_right])          # ... of layer 0
    lut = np.full(E, -1, dtype=np.int64)
    lut[need_left] = E + np.arange(need_left.size)
    nbr_local[to_left] = lut[mesh.nbr_elem[to_left]]
    lut[:] = -1
    lut[need_right] = E + need_left.size + np.arange(need_right.size)
    nbr_local[to_right] = lut[mesh.nbr_elem[to_right]]
    # by symmetry the left peer needs my layer-0 elements (= what I need from the right peer) and
    # the right peer my layer n-1 elements; tag 1 = data travelling left, tag 2 = travelling right
    local = Mesh(mesh.dim, mesh.vertices, mesh.vertex_ids, nbr_local, mesh.nbr_face, mesh.nbr_perm, mesh.btag)
    plan = HaloPlan(rank, nranks, E, need_left.size + need_right.size,
                    peers=[left, right], tags=[2, 1],      # receive tags: from the left peer comes tag 2
                    send_local=[need_right, need_left],    # to the left peer goes my layer 0 ...
                    recv_slots=[(0, need_left.size), (need_left.size, need_left.size + need_right.size)])
    plan.send_tags = [1, 2]                                  # ... travelling left (1); to the right peer tag 2
    return local, plan


def interior_first(local: Mesh, plan: HaloPlan) -> tuple[Mesh, HaloPlan]:
    """Renumber a rank's elements as [interior | adjacent to a ghost element] (stable inside each
    group, so the space-filling-curve locality survives).  The interior range needs no halo data:
    the fused kernels run it while the exchange is in flight (halo.py), then the rest.  Ghost slots
    and message contents keep their order (both are defined by ids the peers share), only the
    local ids inside ``send_local`` are translated."""
    E = plan.nlocal
    touches = np.any(local.nbr_elem >= E, axis=1)
    perm = np.concatenate([np.nonzero(~touches)[0], np.nonzero(touches)[0]])     # new -> old
    inv = np.empty(E, dtype=np.int64)
    inv[perm] = np.arange(E)
    nbr = local.nbr_elem[perm].copy()
    loc = nbr < E
    nbr[loc] = inv[nbr[loc]]
    mesh = Mesh(local.dim, local.vertices[perm], local.vertex_ids[perm], nbr, local.nbr_face[perm].copy(),
                local.nbr_perm[perm].copy(), local.btag[perm].copy(),
                nbr_rank=None if local.nbr_rank is None else local.nbr_rank[perm].copy())
    new = HaloPlan(plan.rank, plan.nranks, plan.nlocal, plan.nghost, list(plan.peers), list(plan.tags),
                   [inv[np.asarray(sl, dtype=np.int64)] for sl in plan.send_local], list(plan.recv_slots),
                   global_ids=None if plan.global_ids is None else plan.global_ids[perm],
                   n_interior=int((~touches).sum()))
    if hasattr(plan, "send_tags"):
        new.send_tags = list(plan.send_tags)
    new.local_perm = perm
    return mesh, new
