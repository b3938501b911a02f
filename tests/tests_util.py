import hashlib

import numpy as np


def sha(*arrays):
    """SHA-256 of the float64 bytes (matches tests/golden/make_golden.py)."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()
