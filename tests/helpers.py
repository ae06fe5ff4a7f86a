"""Shared numerics helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np


def with_spectrum(w, seed, oracle):
    """Symmetric matrix V diag(w) V^T, V from the QR of a seeded Gaussian
    matrix (the construction of ref tests/test_rsvd.cpp:27-46, with the
    oracle's Householder QR standing in for Eigen's)."""
    n = len(w)
    a = oracle.fill_gaussian(seed, n * n).reshape(n, n)
    v = oracle.thin_orthonormal(a)
    g = v @ np.diag(np.asarray(w, float)) @ v.T
    return np.ascontiguousarray((g + g.T) / 2.0)


def rel_err(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) if a.size else 0.0


def sin_subspace(u1, u2):
    """sin of the largest principal angle between span(u1) and span(u2)
    (both with orthonormal columns), as ||(I - U1 U1^T) U2||_2 (SURVEY §8d:
    the arccos form has a sqrt(eps) floor)."""
    q1, _ = np.linalg.qr(u1)
    q2, _ = np.linalg.qr(u2)
    r = q2 - q1 @ (q1.T @ q2)
    return np.linalg.norm(r, 2)


def coords_match_up_to_sign(a, b):
    """max |a - s b| over columns with the best per-column sign s."""
    if a.shape != b.shape:
        return np.inf
    worst = 0.0
    for c in range(a.shape[1]):
        d = min(np.max(np.abs(a[:, c] - b[:, c])), np.max(np.abs(a[:, c] + b[:, c])))
        worst = max(worst, d)
    return worst
