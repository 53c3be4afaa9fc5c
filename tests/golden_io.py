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
    """Fixture names; full-size BASELINE configs only when full=True."""
    from cases import FULL_NAMES
    all_ = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))
    return [n for n in all_ if (n in FULL_NAMES) == full]
