"""Connectivity, index maps and partition/halo plans: integer-exact host logic."""
import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext, rel_err
from paper_2512_17101_b200 import DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
from paper_2512_17101_b200.dg.mesh import face_index_maps, geometry
from paper_2512_17101_b200.dg.partition import interior_first, partition_elements, rank_mesh, ring_slab
from paper_2512_17101_b200.dg.simplex import simplex_element
from paper_2512_17101_b200.discretization import BC_FARFIELD, BC_WALL
from tests.common import FARFIELD, random_state


@pytest.mark.parametrize("dim,p,n,per", [(2, 3, 4, False), (2, 2, 4, True), (3, 3, 3, False), (3, 4, 3, True), (3, 1, 4, True)])
def test_face_maps_match_coordinates(dim, p, n, per):
    el = simplex_element(dim, p)
    m = box_mesh((n,) * dim, (-1,) * dim, (1,) * dim, periodic=(per,) * dim)
    g = geometry(m, el)
    vm, vp = face_index_maps(m, el)
    assert vm.dtype == np.int64 and vp.dtype == np.int64
    x = g.nodes.reshape(dim, -1)
    dlt = x[:, vm.ravel()] - x[:, vp.ravel()]
    if per:
        dlt = dlt - 2 * np.round(dlt / 2)
    assert np.abs(dlt).max() < 1e-13
    assert (m.btag != 0).sum() == (0 if per else 2 * dim * n ** (dim - 1) * (1 if dim == 2 else 2))
    assert abs(g.jac.sum() * {2: 2.0, 3: 4.0 / 3.0}[dim] - 2.0 ** dim) < 1e-12
    # involution: the neighbour of my neighbour across the shared face is me
    E, Nf = m.nbr_elem.shape
    back_e = m.nbr_elem[m.nbr_elem, m.nbr_face]
    back_f = m.nbr_face[m.nbr_elem, m.nbr_face]
    interior = m.btag == 0
    assert np.array_equal(back_e[interior], np.broadcast_to(np.arange(E)[:, None], (E, Nf))[interior])
    assert np.array_equal(back_f[interior], np.broadcast_to(np.arange(Nf)[None, :], (E, Nf))[interior])


def test_empty_and_degenerate_inputs():
    with pytest.raises(ValueError):
        box_mesh((2, 2, 2), (-1,) * 3, (1,) * 3, periodic=(True,) * 3)     # too coarse for periodic keys
    with pytest.raises(ValueError):
        simplex_element(4, 2)
    m = box_mesh((1, 1), (0, 0), (1, 1))
    assert m.nelements == 2 and (m.btag != 0).sum() == 4


def _loopback(locs, fields, Np):
    out = []
    for r, (m, p) in enumerate(locs):
        g = np.empty(fields[r].shape[:-2] + (p.nghost, Np))
        for k, peer in enumerate(p.peers):
            pp = locs[peer][1]
            j = pp.peers.index(r)
            a, b = p.recv_slots[k]
            g[..., a:b, :] = fields[peer][..., pp.send_local[j], :]
        out.append(g)
    return out


@pytest.mark.parametrize("dim,n,per,nparts", [(3, 3, True, 2), (3, 3, True, 4), (2, 4, False, 3)])
def test_partitioned_rhs_equals_single_domain(dim, n, per, nparts, reorder=False):
    actx = NumpyArrayContext()
    mesh = box_mesh((n,) * dim, (-1,) * dim, (1,) * dim, periodic=(per,) * dim)
    bc = None if per else {k: (BC_WALL if k % 2 else BC_FARFIELD) for k in range(1, 2 * dim + 1)}
    d = DGDiscretization(actx, mesh, 3, bc_map=bc)
    q0 = random_state(dim, d.nelements, d.Np, seed=5)
    part = partition_elements(mesh, nparts)
    assert np.bincount(part).min() >= mesh.nelements // nparts - 1
    locs = [rank_mesh(mesh, part, r) for r in range(nparts)]
    if reorder:       # [interior | next to a ghost] renumbering used for the exchange/compute overlap
        locs = [interior_first(m, p) for m, p in locs]
        for m, p in locs:
            assert not np.any(m.nbr_elem[:p.n_interior] >= p.nlocal)
            assert np.all(np.any(m.nbr_elem[p.n_interior:] >= p.nlocal, axis=1))
            assert sorted(p.global_ids.tolist()) == sorted(np.nonzero(part == p.rank)[0].tolist())
    for a in range(nparts):
        for b in range(nparts):
            if a != b:
                locs[a][1].validate_against(locs[b][1])
    ds = [DGDiscretization(actx, m, 3, bc_map=bc, ghost_elements=p.nghost) for m, p in locs]
    qs = [q0[:, p.global_ids, :] for _, p in locs]
    gh = _loopback(locs, qs, d.Np)
    for Op, kw in [(EulerOperator, {}), (NavierStokesOperator, {"mu": 2e-2})]:
        ref = d.to_numpy(Op(d, farfield=FARFIELD[dim], **kw).rhs(d.from_numpy(q0)))
        ops = [Op(dd, farfield=FARFIELD[dim], **kw) for dd in ds]
        if Op is EulerOperator:
            res = [ds[r].to_numpy(ops[r].rhs(ds[r].from_numpy(qs[r]), ghost=gh[r])) for r in range(nparts)]
        else:
            # gradient arrangement: second exchange carries grad q
            gqs = [ds[r].to_numpy(ops[r].grad(ds[r].from_numpy(qs[r]), gh[r])) for r in range(nparts)]
            ggh = _loopback(locs, gqs, d.Np)
            res = [ds[r].to_numpy(ops[r].rhs_grad_form(ds[r].from_numpy(qs[r]), ghost=gh[r],
                                                       halo_fn=lambda gq, r=r: ggh[r])) for r in range(nparts)]
            full = np.empty_like(ref)
            for r, (m, p) in enumerate(locs):
                full[:, p.global_ids, :] = res[r]
            assert rel_err(full, ref) <= 1e-13
            # flux arrangement (default): second exchange carries the flux planes
            Ts = [np.asarray(actx.to_numpy(ops[r].flux(ds[r].from_numpy(qs[r]), gh[r]))) for r in range(nparts)]
            tgh = _loopback(locs, Ts, d.Np)
            res = [ds[r].to_numpy(ops[r].rhs(ds[r].from_numpy(qs[r]), ghost=gh[r],
                                             halo_fn=lambda T, r=r: tgh[r])) for r in range(nparts)]
        full = np.empty_like(ref)
        for r, (m, p) in enumerate(locs):
            full[:, p.global_ids, :] = res[r]
        assert rel_err(full, ref) <= 1e-13


@pytest.mark.parametrize("dim,n,per,nparts", [(3, 3, True, 2), (2, 4, False, 3)])
def test_interior_first_renumbering(dim, n, per, nparts):
    test_partitioned_rhs_equals_single_domain(dim, n, per, nparts, reorder=True)


def test_mismatched_plan_is_rejected():
    from paper_2512_17101_b200 import errors
    mesh = box_mesh((3,) * 3, (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    part = partition_elements(mesh, 2)
    (m0, p0), (m1, p1) = rank_mesh(mesh, part, 0), rank_mesh(mesh, part, 1)
    p1.recv_slots[0] = (0, p1.recv_slots[0][1] - 1)
    with pytest.raises(errors.MismatchedCommunication) as exc:
        p0.validate_against(p1)
    assert exc.value.keys == ((0, 1, 0),)


def test_ring_slab_equals_global_periodic_mesh():
    """Three identical periodic boxes wired as a ring == one periodic box three times as long."""
    actx = NumpyArrayContext()
    n, R = 3, 3
    glob = box_mesh((n * R, n, n), (-1, -1, -1), (-1 + 2 * R, 1, 1), periodic=(True,) * 3)
    dg_ = DGDiscretization(actx, glob, 2)

    def state(x):
        k = 2 * np.pi / (2 * R)
        rho = 1 + 0.1 * np.sin(k * (x[0] + 1)) * np.cos(np.pi * x[1])
        u = [0.1 * np.cos(k * (x[0] + 1)), 0.05 * np.sin(np.pi * x[2]), 0.02 + 0 * x[0]]
        p = 1 / 1.4 + 0.05 * np.cos(k * (x[0] + 1) + np.pi * x[2])
        return np.stack([rho, p / 0.4 + 0.5 * rho * sum(v * v for v in u)] + [rho * v for v in u])

    op_g = NavierStokesOperator(dg_, mu=2e-2)
    ref = dg_.to_numpy(op_g.rhs(dg_.from_numpy(state(dg_.nodes()))))
    gkey = {tuple(np.round(c, 9)): e for e, c in enumerate(glob.vertices.mean(axis=1))}

    base = box_mesh((n, n, n), (-1,) * 3, (1,) * 3, periodic=(True,) * 3)
    locs = [ring_slab(base, n, r, R, -1.0, 1.0) for r in range(R)]
    ds = [DGDiscretization(actx, m, 2, ghost_elements=p.nghost) for m, p in locs]
    shift = [np.array([2.0 * r, 0, 0])[:, None, None] for r in range(R)]
    qs = [state(ds[r].nodes() + shift[r]) for r in range(R)]

    def exch(fields):
        out = []
        for r, (m, p) in enumerate(locs):
            g = np.empty(fields[r].shape[:-2] + (p.nghost, ds[r].Np))
            for k, peer in enumerate(p.peers):
                pp = locs[peer][1]
                # the message I receive with tag t is the one the peer sends with send_tag t to me
                j = [jj for jj in range(len(pp.peers)) if pp.peers[jj] == r and pp.send_tags[jj] == p.tags[k]][0]
                a, b = p.recv_slots[k]
                g[..., a:b, :] = fields[peer][..., pp.send_local[j], :]
            out.append(g)
        return out

    ops = [NavierStokesOperator(dd, mu=2e-2) for dd in ds]
    gh = exch(qs)
    Ts = [np.asarray(ops[r].flux(ds[r].from_numpy(qs[r]), gh[r])) for r in range(R)]
    tgh = exch(Ts)
    for r in range(R):
        out = ds[r].to_numpy(ops[r].rhs(ds[r].from_numpy(qs[r]), ghost=gh[r], halo_fn=lambda T, r=r: tgh[r]))
        cent = base.vertices.mean(axis=1) + np.array([2.0 * r, 0, 0])
        idx = np.array([gkey[tuple(np.round(c, 9))] for c in cent])
        assert rel_err(out, ref[:, idx, :]) <= 1e-12
