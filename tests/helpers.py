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


def sym_fingerprint(rows, row0):
    """numpy restatement of the sharded gram's antisymmetric symmetry
    fingerprint (k1_shard.cu SymFp) over a block of full rows starting at
    global row row0: two 32-bit sums over (i, j) of sgn(j - i) times a mix of
    each half of bits(d_ij) with the unordered position {i, j}. Summed over
    all shards (mod 2^32) both are 0 iff D is exactly symmetric.
    Returns (lo, hi)."""
    import numpy as np
    m32 = np.uint64(0xFFFFFFFF)
    v = np.ascontiguousarray(rows, dtype=np.float64).view(np.uint64)
    vl, vh = v & m32, v >> np.uint64(32)
    i = (np.arange(rows.shape[0], dtype=np.uint64) + np.uint64(row0))[:, None]
    j = np.arange(rows.shape[1], dtype=np.uint64)[None, :]
    lo_, hi_ = np.minimum(i, j), np.maximum(i, j)
    key = (lo_ * np.uint64(0x9E3779B1) + hi_ * np.uint64(0x85EBCA77)) & m32
    xl = (((vl ^ key) & m32) * np.uint64(0xC2B2AE3D)) & m32
    xh = (((vh ^ key ^ np.uint64(0x165667B1)) & m32) * np.uint64(0x27D4EB2F)) & m32
    out = []
    for x in (xl, xh):
        pos = int(np.sum(np.where(j > i, x, np.uint64(0)), dtype=np.uint64))
        neg = int(np.sum(np.where(j < i, x, np.uint64(0)), dtype=np.uint64))
        out.append((pos - neg) % 2**32)
    return tuple(out)
