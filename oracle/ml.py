"""ML-ensemble oracle, serial fp64 (TEST INFRASTRUCTURE ONLY).

PAPER.md §V-B: "an ML pipeline that combines Categorical Naive Bayes
and Ridge Regression classifiers by applying softmax normalization and
averaging scores. The input matrix has 200 features."  Node names from
Fig. 6 (L719-728) and Fig. 10 (L1292-1307): NORM, MMUL x2, MAX, LSE, EXP,
ADDV, SOFTMAX x2, ARGMAX.  Formulas are SURVEY §8(c2) ML readings
(DESIGN.md R-ML): the NB branch is the multinomial-form dot product the
figure draws (MMUL), not a per-category table lookup.

    NB: r1 = X theta^T + prior;  m = max_c r1;  l = m + ln sum_c e^(r1-m);
        r1 = e^(r1 - l);  r1 = softmax(r1)
    RR: mu_f = mean_i X, sd_f = sqrt(mean_i (X - mu_f)^2) (population, sd=0 -> 1);
        Z = (X - mu)/sd;  r2 = Z W^T;  r2 += b;  r2 = softmax(r2)
    r[i] = lowest c maximising r1[i,c] + r2[i,c]

Pins (tests/test_oracle_ml.py): MMULs against numpy.matmul (the oracle's
MMUL is an explicit per-feature accumulation); EXP rows sum to 1 and equal
scipy.special.softmax of the NB scores; softmax rows sum to 1 and equal
scipy.special.softmax; Z columns mean 0 / std 1; argmax by brute force.
"""
import numpy as np

N_CLASSES = 10   # reading; parity unpinned (constant)
N_FEATURES = 200


def norm_stats(X, chunk=1 << 20):
    """Per-feature population mean and standard deviation, the textbook
    two-pass definition in fp64 (reading R-ML: population std,
    sd = 0 -> 1):  mu_f = (1/N) sum_i x_if;  sd_f = sqrt((1/N) sum_i (x_if - mu_f)^2).
    Chunked over rows only to bound memory (fp64 sums are per chunk, then
    added in row order)."""
    X = np.asarray(X)
    n = X.shape[0]
    S = np.zeros(X.shape[1])
    for i in range(0, n, chunk):
        S += X[i:i + chunk].astype(np.float64).sum(axis=0)
    mu = S / n
    D = np.zeros(X.shape[1])
    for i in range(0, n, chunk):
        d = X[i:i + chunk].astype(np.float64) - mu
        D += (d * d).sum(axis=0)
    sd = np.sqrt(D / n)
    return mu, np.where(sd > 0, sd, 1.0)


def apply_norm(X, mu, sd):
    return (np.asarray(X, dtype=np.float64) - mu) / sd


def norm(X):
    """NORM: per-feature standardisation over rows (population std)."""
    return apply_norm(X, *norm_stats(X))


def mmul(A, Wt):
    """MMUL: out[i,c] = sum_f A[i,f] Wt[c,f], accumulated feature by feature."""
    A = np.asarray(A, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    out = np.zeros((A.shape[0], Wt.shape[0]))
    for f in range(A.shape[1]):
        out += A[:, f:f + 1] * Wt[None, :, f]
    return out


def nb_mmul(X, theta, prior):
    """NB MMUL with the class prior added (prior is a const input)."""
    return mmul(X, theta) + np.asarray(prior, dtype=np.float64)[None, :]


def rowmax(r):
    return np.max(r, axis=1)


def lse(r, m):
    return m + np.log(np.sum(np.exp(r - m[:, None]), axis=1))


def exp_sub(r, l):
    return np.exp(r - l[:, None])


def addv(r, b):
    return r + np.asarray(b, dtype=np.float64)[None, :]


def softmax(r):
    m = np.max(r, axis=1, keepdims=True)
    e = np.exp(r - m)
    return e / e.sum(axis=1, keepdims=True)


def argmax(r1, r2):
    """ARGMAX of the averaged scores; ties go to the lowest class index."""
    s = np.asarray(r1, np.float64) + np.asarray(r2, np.float64)
    return np.argmax(s, axis=1).astype(np.int32)  # numpy returns the first maximum


def ml(X, theta, prior, W, b):
    """The ML DAG in program order (SURVEY §8(c2) launch order)."""
    Z = norm(X)
    r1 = nb_mmul(X, theta, prior)
    r2 = mmul(Z, W)
    amax = rowmax(r1)
    l = lse(r1, amax)
    r2 = addv(r2, b)
    r1e = exp_sub(r1, l)
    r2s = softmax(r2)
    r1s = softmax(r1e)
    r = argmax(r1s, r2s)
    return dict(Z=Z, r1_scores=r1, amax=amax, l=l, r1_exp=r1e, r1=r1s, r2=r2s, r=r)


def top2_gap(r1, r2):
    """Oracle top-2 margin of the averaged score per row (for the near-tie rule)."""
    s = np.sort(np.asarray(r1, np.float64) + np.asarray(r2, np.float64), axis=1)
    return s[:, -1] - s[:, -2]
