"""Writes paper_1803_09948_b200/data/quadrature_rules.npz: the interpolation and quadrature tables the
correction builders take as INPUT (hfmm_correction_rules): Lagrange nodes and reference weights of basis
orders 1 and 2, the 25-point triangle Gauss rule, the Duffy rules centred on every node (self_rule 8) and
the basis values at their points — numbers produced by the reference's geometry.cpp (geom::lagrange_basis,
geom::gauss_rule, geom::duffy_rule), tabulated here by running the compiled reference (oracle/_ref), so that
the product ships the tables a caller without the reference at hand would otherwise have to supply.
Run in the authoring container only (needs /root/reference)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from checkers import Ref

out = {}
ref = Ref()
for order in (1, 2):
    t = ref.correction_tables(order, near_rule=25, self_rule=8)
    for k, v in t.items():
        out[f"order{order}_{k}"] = np.asarray(v)
path = os.path.join(ROOT, "paper_1803_09948_b200", "data", "quadrature_rules.npz")
np.savez_compressed(path, **out)
print(path, {k: v.shape for k, v in out.items()})
