"""Degenerate CQK instances shared by tests/test_gpu_degenerate.py and the
golden generator tests/golden/make_par_golden.py (plain numpy)."""
import numpy as np

N = 300_000  # >= 2 x 65536: every rank of a 2- or 3-way split is on the TMA engine


def plateau(n, side, seed):
    """d = b = 1, l = 0, u = 1, a = +-10 + jitter: phi is flat (= n/2) for
    lambda in about (-8.5, 9.5), and the formula start lambda0 lands on that
    plateau.  side 'right': r = 0.75 n, the root lies right of the plateau;
    'left': r = 0.25 n, left of it."""
    rng = np.random.default_rng(seed)
    m = n // 2
    a = np.concatenate([10.0 + rng.uniform(0, 0.5, m), -10.0 + rng.uniform(0, 0.5, n - m)])
    rng.shuffle(a)
    one = np.ones(n)
    r = 0.75 * n if side == "right" else 0.25 * n
    return one.copy(), a, one.copy(), np.zeros(n), one.copy(), r


def pinned_box(n):
    """box([1]*n, [0]*n, [1]*n, [0]*n, [0]*n, 1): every variable pinned at 0."""
    one = np.ones(n)
    return one.copy(), np.zeros(n), one.copy(), np.zeros(n), np.zeros(n), 1.0


def pinned_blocks(n, seed):
    """A random instance with every third variable pinned (l == u)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(0.5, 3.0, n)
    a = rng.normal(0.0, 2.0, n)
    b = rng.uniform(0.5, 3.0, n)
    lo = rng.normal(0.0, 1.0, n)
    hi = lo + rng.uniform(0.0, 2.0, n)
    hi[::3] = lo[::3]
    r = float(b @ lo + 0.4 * (b @ hi - b @ lo))
    return d, a, b, lo, hi, r


CASES = {
    "plateau-right": lambda: plateau(N, "right", 1),
    "plateau-left": lambda: plateau(N, "left", 2),
    "pinned-box": lambda: pinned_box(N),
    "pinned-blocks": lambda: pinned_blocks(N, 3),
}


