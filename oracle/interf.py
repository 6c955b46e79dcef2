"""C3 interference-model oracle (ORACLE — test infrastructure only).

PAPER.md §4.4: interference_factor = c1*l2_m1 + c2*l2_m2 +
c3*mem_m1 + c4*mem_m2 + c5 (eq. at), where l2/mem are the solo-run L2
and DRAM-bandwidth utilisations of the victim (m1) and its partner (m2) at
their gpu-let sizes; "parameters ... are searched with linear
regression" on 1,750 training / 750 validation samples.

Readings: OLS in float64 via numpy.linalg.lstsq;
prediction clamped below at 1.0; error = |max(1, f_hat) - f| / f on a
seeded 70/30 split.  Pinned in tests/test_oracle_interf.py (planted recovery,
rank error, residual orthogonality, the S:170 arithmetic example).
"""
import numpy as np


class RankError(ValueError):
    pass


def design(l2_v, l2_u, mem_v, mem_u):
    """Feature rows x = (l2_v, l2_u, mem_v, mem_u, 1)."""
    l2_v, l2_u, mem_v, mem_u = map(lambda a: np.asarray(a, np.float64), (l2_v, l2_u, mem_v, mem_u))
    return np.stack([l2_v, l2_u, mem_v, mem_u, np.ones_like(l2_v)], axis=-1)


def fit(X, y):
    """OLS min ||X c - y||^2; raises RankError for a rank-deficient design."""
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.float64)
    if X.shape[0] < 5 or np.linalg.matrix_rank(X) < 5:
        raise RankError("rank-deficient design: need more diverse co-run samples")
    c, *_ = np.linalg.lstsq(X, y, rcond=None)
    return c


def predict_raw(c, l2_v, l2_u, mem_v, mem_u):
    return c[0] * l2_v + c[1] * l2_u + c[2] * mem_v + c[3] * mem_u + c[4]


def predict(c, l2_v, l2_u, mem_v, mem_u):
    """Factor clamped below at 1.0 (a co-run never speeds a victim up)."""
    return np.maximum(1.0, predict_raw(c, l2_v, l2_u, mem_v, mem_u))


def overhead(c, L, l2_v, l2_u, mem_v, mem_u):
    """Additional latency L * (factor - 1)."""
    return L * (predict(c, l2_v, l2_u, mem_v, mem_u) - 1.0)


def split(n, seed=0, train_frac=0.7):
    """Seeded train/validation index split (1,750 / 750 of 2,500)."""
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n)
    k = int(round(train_frac * n))
    return np.sort(perm[:k]), np.sort(perm[k:])


def rel_errors(c, X, y):
    f_hat = np.maximum(1.0, X @ c)
    return np.abs(f_hat - y) / y
