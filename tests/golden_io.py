"""Load tests/golden fixtures (made by tests/golden/make_golden.py from the reference)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    return dict(history=z["history"], final_norms=z["final_norms"], x_rows=z["x_rows"],
                x_sample=z["x_sample"], meta=meta)


def names(full=False):
    """Fixture names.  full=True returns EVERY full-size case declared in
    cases.FULL_CASES whether or not its fixture exists, so a missing fixture
    fails its test (load() raises) instead of silently dropping out."""
    from cases import FULL_NAMES
    if full:
        return sorted(FULL_NAMES)
    all_ = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))
    return [n for n in all_ if n not in FULL_NAMES]


def missing_full():
    """FULL_CASES whose fixture has not been generated."""
    return [n for n in names(full=True) if not os.path.exists(os.path.join(GOLDEN, f"{n}.npz"))]
