"""Helpers to load the committed golden fixtures (generated from the real
reference by tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

STAGES = ("y0s", "aeqs", "rhoE_c", "rhoE_fy", "fW", "fE", "fS", "fN", "vol", "psi",
          "quiet", "DW", "DE", "DS", "DN")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_case(name):
    z = np.load(os.path.join(GOLDEN, f"case_{name}.npz"))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    meta = json.loads(str(z["meta"]))
    return meta, arrays


def case_names():
    return sorted(f[5:-4] for f in os.listdir(GOLDEN) if f.startswith("case_"))


def same(a, b):
    """Bit-level equality: every double has the same bit pattern (so +0 and -0
    differ); NaNs match NaNs of any payload."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype.kind == "f":
        a64 = np.ascontiguousarray(a, dtype=np.float64)
        b64 = np.ascontiguousarray(b, dtype=np.float64)
        eq = a64.view(np.int64) == b64.view(np.int64)
        if not eq.all():
            eq |= np.isnan(a64) & np.isnan(b64)
        return bool(eq.all())
    return bool(np.array_equal(a, b))
