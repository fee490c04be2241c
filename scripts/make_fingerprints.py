"""Regenerate paper_2512_17101_b200/fused_fingerprints.json: the source fingerprints of the outlined DG
functions of operators.py that the fused kernels implement.  Run it ONLY after changing the kernels (and
the operator program) together; tests/test_cabi_and_host.py checks that the shipped program matches."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_17101_b200 import fused, operators  # noqa: E402

MAKERS = {"dg_euler_rhs": operators._make_euler_rhs, "dg_ns_grad": operators._make_ns_grad, "dg_ns_rhs": operators._make_ns_rhs,
          "dg_ns_flux": operators._make_ns_flux, "dg_ns_div": operators._make_ns_div,
          "dg_euler_rhs_rk": operators._make_euler_rhs_rk, "dg_ns_rhs_rk": operators._make_ns_rhs_rk,
          "dg_ns_div_rk": operators._make_ns_div_rk}


def _ms_makers():
    from paper_2512_17101_b200 import multispecies
    out = {}
    for k, name in enumerate(("dg_ms_rhs", "dg_ms_flux", "dg_ms_div")):
        out[name] = lambda dim, ghost, k=k: multispecies._make_ms_functions(dim, multispecies.Mixture())[k]
    return out


def compute():
    MAKERS.update(_ms_makers())
    out = {}
    for name, mk in MAKERS.items():
        fps = set()
        for dim in (2, 3):
            for ghost in (False, True):
                f = mk(dim, ghost)
                assert f.__name__ == name, (f.__name__, name)
                fps.add(fused.fingerprint(f))
        out[name] = sorted(fps)
    return out


if __name__ == "__main__":
    path = os.path.join(ROOT, "paper_2512_17101_b200", "fused_fingerprints.json")
    with open(path, "w") as fh:
        json.dump({"python": "%d.%d" % sys.version_info[:2], "functions": compute()}, fh, indent=1)
        fh.write("\n")
    print("wrote", path)
