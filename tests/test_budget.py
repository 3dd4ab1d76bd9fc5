"""The layer-wise budget allocation behind the non-uniform k sweep (BASELINE configs[4]) against
golden vectors of the reference's own dbf.budget.allocate (tests/golden/make_golden_budget.py)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2505_11076_b200.budget import allocate_middle_dims

GOLD = Path(__file__).resolve().parent / "golden" / "golden_budget.npz"


def test_allocate_matches_reference_golden():
    with np.load(GOLD) as z:
        for ci in range(int(z["count"])):
            names = [str(s) for s in z[f"c{ci}_names"]]
            shapes = z[f"c{ci}_shapes"]
            target, floor, gran = z[f"c{ci}_params"]
            layers = [(nm, int(n), int(m)) for nm, (n, m) in zip(names, shapes)]
            scores = {nm: z[f"c{ci}_{nm}_scores"] for nm in names}
            k = allocate_middle_dims(layers, scores, float(target), float(floor), int(gran))
            assert [k[nm] for nm in names] == list(z[f"c{ci}_k"]), ci


def test_allocate_rejects_infeasible_floor():
    with pytest.raises(ValueError, match="infeasible"):
        allocate_middle_dims([("a", 64, 64)], {"a": np.ones(64)}, 0.5, floor_bpw=1.0)
