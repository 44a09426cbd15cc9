"""R36 on the host: GICP plane-regularised scan covariances, as they reach the
library (fp32 entries), have their two largest eigenvalues within 2^-21 of the largest, so
every point of the synthetic scans is plane-form and the sweep's plane instantiation runs; the
plane form lam3 I + a (I - n n^T), a = (l1 + l2) / 2 - lam3, reproduces the fp32 covariance to
the size of its own rounding.  Random SPD covariances are not plane-form."""
import numpy as np

import synth

TOL = 2.0 ** -21


def _mats(c6):
    c = c6.astype(np.float64)
    A = np.empty((len(c), 3, 3))
    for k, (a, b) in enumerate([(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]):
        A[:, a, b] = c[:, k]
        A[:, b, a] = c[:, k]
    return A


def _split(A):
    w = np.linalg.eigvalsh(A)  # ascending
    return (w[:, 2] - w[:, 1]) / np.abs(w[:, 2]), w


def test_synthetic_scans_are_plane_form():
    for s in (synth.c1(), synth.c2(N=10)):
        r, _ = _split(_mats(s.scan_cov6))
        assert r.max() <= TOL / 4, r.max()  # well inside the rule: fp32 rounding only


def test_plane_form_reconstructs_the_fp32_covariance():
    s = synth.c2(N=10)
    A = _mats(s.scan_cov6)
    w, V = np.linalg.eigh(A)
    a = 0.5 * (w[:, 1] + w[:, 2]) - w[:, 0]
    n = V[:, :, 0]
    P = w[:, 0, None, None] * np.eye(3) + a[:, None, None] * (
        np.eye(3) - np.einsum("ni,nj->nij", n, n))
    # the merge moves l1, l2 by at most half their split: at the fp32 input rounding
    err = np.abs(P - A).max(axis=(1, 2)) / w[:, 2]
    assert err.max() <= TOL / 2, err.max()
    # and the [x]x^T [x]x form with x = sqrt(a) n is the same matrix
    x = np.sqrt(a)[:, None] * n
    X = np.zeros((len(x), 3, 3))
    X[:, 0, 1], X[:, 0, 2], X[:, 1, 2] = -x[:, 2], x[:, 1], -x[:, 0]
    X = X - np.transpose(X, (0, 2, 1))
    Q = w[:, 0, None, None] * np.eye(3) + np.einsum("nki,nkj->nij", X, X)
    assert np.abs(Q - P).max() <= 1e-12


def test_random_spd_covariances_are_general():
    rng = np.random.default_rng(36)
    lam = np.exp(rng.uniform(np.log(1e-3), 0.0, (2000, 3)))
    V, _ = np.linalg.qr(rng.standard_normal((2000, 3, 3)))
    A = np.einsum("nij,nj,nkj->nik", V, lam, V).astype(np.float32).astype(np.float64)
    r, _ = _split(A)
    assert (r > TOL).mean() > 0.99
