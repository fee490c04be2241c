"""tests/golden/ns2d_p1_rhs_program.json: the exported NS right-hand-side program of a 3x3 periodic triangle mesh
(order 1) and the values the REAL reference's oracle (`eager_eval` on the loaded document) computes for it.
Run in the build container only:  python tests/golden/make_program_golden.py"""
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from laze import cli, eager_eval  # noqa: E402
from laze.adfg import as_dtype  # noqa: E402
from paper_2512_17101_b200.export import export_rhs_program  # noqa: E402
from tests.test_graph_export import CASES, _case  # noqa: E402

equations, dim, order, n, kw = CASES[0]
mesh, q0, _ = _case(equations, dim, order, n, kw)
doc = json.loads(json.dumps(export_rhs_program(mesh, order, q0, equations, **kw)))
with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
    json.dump(doc, fh)
graphs, bindings_spec, _ = cli.load_program_file(fh.name, as_dtype("f64"))
bindings = cli.materialize_bindings(bindings_spec[0], graphs[0], 0)
rhs = dict((name, eager_eval(node, bindings)) for name, node in graphs[0].outputs)["rhs"]
with open(os.path.join(HERE, "ns2d_p1_rhs_program.json"), "w") as out:
    json.dump({"program": doc, "reference_oracle_rhs": rhs.tolist()}, out)
print("wrote ns2d_p1_rhs_program.json", os.path.getsize(os.path.join(HERE, "ns2d_p1_rhs_program.json")), "bytes")
