"""Small cases that touch every default kernel (NS flux arrangement incl. RK epilogue, Euler, boundary faces,
ragged tail blocks) for `compute-sanitizer --tool memcheck|racecheck python scripts/sanitize_case.py`."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2512_17101_b200 import B200ArrayContext, EulerOperator, Mixture, MultispeciesOperator, NavierStokesOperator
from tests.common import FARFIELD, make_dcoll, random_state
actx = B200ArrayContext()
for dim, order, n, bc in [(3, 3, 2, "mixed"), (3, 3, 3, "periodic"), (2, 4, 3, "mixed"), (3, 4, 2, "farfield"), (3, 4, 3, "periodic")]:
    d = make_dcoll(actx, dim, order, n, bc)
    q = d.from_numpy(random_state(dim, d.nelements, d.Np, seed=2))
    ns = NavierStokesOperator(d, farfield=FARFIELD[dim], mu=2e-2)
    eu = EulerOperator(d, farfield=FARFIELD[dim])
    r = ns.rhs(q)
    a, b = ns.rhs_rk(q, q, r, (1.0, 0.1, 0.5, 0.2))
    e = eu.rhs(q)
    e1, e2 = eu.rhs_rk(q, q, e, (1.0, 0.1, 0.5, 0.2))
    vals = [float(np.abs(d.to_numpy(x)).max()) for x in (r, a, b, e, e1, e2)]
    assert all(np.isfinite(v) for v in vals)
    if bc in ("periodic", "farfield"):                     # the multi-species instantiation of the same kernels (C = dim + 5)
        from tests.common import MS_MIXTURES
        for nspec in (2, 3, 4):                            # one translation unit per species count
            ms = MultispeciesOperator(d, Mixture(**MS_MIXTURES[nspec]))
            rng = np.random.default_rng(4)
            E, Np = d.nelements, d.Np
            Y = rng.uniform(0.2, 0.5, (nspec, E, Np)); Y /= Y.sum(0)
            qm = d.from_numpy(ms.state_from_primitive(rng.uniform(0.9, 1.1, (E, Np)), [rng.uniform(-0.1, 0.1, (E, Np)) for _ in range(dim)],
                                                      rng.uniform(0.9, 1.1, (E, Np)), list(Y)))
            v = float(np.abs(d.to_numpy(ms.rhs(qm))).max())
            assert np.isfinite(v) and ms._f.fused
    print(dim, order, n, bc, "ok", flush=True)
