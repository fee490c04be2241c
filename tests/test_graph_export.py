"""Export of the traced right-hand side in the reference CLI's JSON program format (SURVEY.md §8f rank 4,
/root/reference/pkg/src/laze/cli.py:434-576): the document must replay through the REAL reference (its loader,
`eager_eval` oracle and compile pipeline -- here, where /root/reference is mounted) to the oracle's values, and
must equal the committed golden document everywhere else."""
import json
import os
import sys

import numpy as np
import pytest

from oracle.laze_port import NumpyArrayContext, rel_err
from paper_2512_17101_b200 import DGDiscretization, EulerOperator, NavierStokesOperator, box_mesh
from paper_2512_17101_b200.export import GraphExportContext, export_rhs_program
from tests.common import random_state

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
CASES = [("ns", 2, 1, 3, {"mu": 2e-2}), ("ns_grad_form", 2, 2, 3, {"mu": 2e-2}), ("euler", 3, 1, 3, {}), ("ns", 3, 2, 3, {"mu": 1e-2}),
         ("multispecies", 2, 2, 3, {})]      # exp / truediv lambdas of the reactive mixture (expr.py:265-289)


def _case(equations, dim, order, n, kw):
    mesh = box_mesh((n,) * dim, (-1.0,) * dim, (1.0,) * dim, periodic=(True,) * dim)
    cpu = NumpyArrayContext()
    d = DGDiscretization(cpu, mesh, order)
    if equations == "multispecies":
        from paper_2512_17101_b200 import MultispeciesOperator
        from tests.test_multispecies import ms_state
        op = MultispeciesOperator(d, **kw)
        q0 = ms_state(op, d.nodes())
        return mesh, q0, d.to_numpy(op.rhs(d.from_numpy(q0)))
    q0 = random_state(dim, d.nelements, d.Np, seed=7)
    op = (EulerOperator if equations == "euler" else NavierStokesOperator)(d, **kw)
    f = op.rhs_grad_form if equations == "ns_grad_form" else op.rhs
    return mesh, q0, d.to_numpy(f(d.from_numpy(q0)))


@pytest.mark.parametrize("equations,dim,order,n,kw", CASES)
def test_exported_program_structure(equations, dim, order, n, kw):
    mesh, q0, _ = _case(equations, dim, order, n, kw)
    doc = export_rhs_program(mesh, order, q0, equations, **kw)
    text = json.dumps(doc)                                     # plain JSON, nothing but lists / numbers / strings
    doc2 = json.loads(text)
    assert set(doc2) >= {"name", "nodes", "outputs", "functions", "bindings"}
    kinds = {spec["kind"] for spec in doc2["nodes"].values()}
    assert {"placeholder", "data", "call"} <= kinds
    names = sorted(f["name"] for f in doc2["functions"].values())
    assert names == {"ns": ["dg_ns_div", "dg_ns_flux"], "ns_grad_form": ["dg_ns_grad", "dg_ns_rhs"],
                     "euler": ["dg_euler_rhs"], "multispecies": ["dg_ms_rhs"]}[equations]
    # definition before use, inside every table (cli.py:160-176)
    for table, pre in [(doc2["nodes"], set())] + [(f["nodes"], set(f["parameters"])) for f in doc2["functions"].values()]:
        seen = set(pre)
        for name, spec in table.items():
            refs = list(spec.get("inputs", [])) + list(spec.get("args", []) if isinstance(spec.get("args"), list) else
                                                      (spec.get("args") or {}).values()) + list(spec.get("arrays", []))
            refs += [spec[k] for k in ("array", "call") if k in spec]
            refs += [s["array"] for s in spec.get("selectors", []) if isinstance(s, dict) and "array" in s]
            assert all(r in seen for r in refs), (name, refs)
            seen.add(name)


def test_exporter_matches_committed_golden_document():
    with open(os.path.join(HERE, "golden", "ns2d_p1_rhs_program.json")) as fh:
        golden = json.load(fh)
    equations, dim, order, n, kw = CASES[0]
    mesh, q0, ref = _case(equations, dim, order, n, kw)
    doc = json.loads(json.dumps(export_rhs_program(mesh, order, q0, equations, **kw)))
    assert doc == golden["program"]
    # the values the reference's own `oracle` evaluation of that document produced (make_program_golden.py)
    assert rel_err(np.asarray(golden["reference_oracle_rhs"]), ref) <= 1e-12


@pytest.mark.skipif(not os.path.isdir(REF), reason="the reference is only mounted in the build container")
@pytest.mark.parametrize("equations,dim,order,n,kw", CASES)
def test_exported_program_replays_through_the_reference(equations, dim, order, n, kw, tmp_path):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from laze import cli, eager_eval
    from laze.adfg import as_dtype
    from laze.pipeline import compile_graph
    mesh, q0, ref = _case(equations, dim, order, n, kw)
    path = tmp_path / "prog.json"
    path.write_text(json.dumps(export_rhs_program(mesh, order, q0, equations, **kw)))
    graphs, bindings_spec, doc = cli.load_program_file(str(path), as_dtype("f64"))
    graph = graphs[0]
    bindings = cli.materialize_bindings(bindings_spec[0], graph, 0)
    got = {name: eager_eval(node, bindings) for name, node in graph.outputs}
    assert rel_err(got["rhs"], ref) <= 1e-12
    if equations == "euler":                                   # the lazy pipeline too (interpreter: small case only)
        out = compile_graph(graph).execute(bindings)
        assert rel_err(out["rhs"], ref) <= 1e-12
    # the reference's serializer reproduces a document its loader accepts again (fixed point of its own format)
    again = cli.graph_to_doc(graph, doc["name"])
    assert set(again["outputs"]) == {"rhs"} and len(again.get("functions", {})) == len(doc["functions"])
    # and its CLI replays the file
    assert cli.main(["oracle", str(path)]) == 0
