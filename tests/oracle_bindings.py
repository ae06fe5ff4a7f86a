"""ctypes bindings for the CPU oracles — TEST INFRASTRUCTURE ONLY.

* ``Oracle``   -> oracle/liboracle.so      (restatement, always built)
* ``RefLib``   -> oracle/_ref/libdivscope_ref.so (the reference's own sources
                  compiled against oracle/eigen_shim; present only where it was
                  built from /root/reference, so tests using it skip otherwise)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libdivscope_ref.so"

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_u64 = C.c_uint64


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _threads() -> int:
    return max(1, os.cpu_count() or 1)


class Oracle:
    """CPU restatement of the reference path (oracle/divscope_oracle.cpp)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_fill_gaussian.argtypes = [_u64, _dp, _sz]
        L.orc_gram_stats.argtypes = [_dp, _sz, _sz, C.c_int, C.c_uint, _dp, _dp]
        L.orc_gram.argtypes = [_dp, _sz, _sz, C.c_int, C.c_uint, _dp]
        L.orc_multiply_sym.argtypes = [_dp, _sz, _dp, _sz, C.c_uint, _dp]
        L.orc_multiply_gram_otf.argtypes = [_dp, _sz, _dp, C.c_double, _dp, _sz, C.c_uint, _dp]
        L.orc_frobenius_sq.argtypes = [_dp, _sz, C.c_uint]
        L.orc_frobenius_sq.restype = C.c_double
        L.orc_thin_orthonormal.argtypes = [_dp, _sz, _sz, _dp]
        L.orc_sym_evd.argtypes = [_dp, _sz, _dp, _dp]
        L.orc_eigs.argtypes = [_dp, _dp, _dp, C.c_double, _sz, _sz, _sz, _sz, _u64, C.c_uint,
                               _dp, _dp, C.POINTER(_sz), _dp]
        L.orc_embed.argtypes = [_dp, _dp, _dp, C.c_double, _sz, _sz, _sz, _sz, _u64, C.c_uint,
                                _dp, _dp, C.POINTER(_sz), _dp, C.POINTER(C.c_int), _dp]
        L.orc_hamming_counts.argtypes = [C.c_char_p, _sz, _sz, C.POINTER(C.c_uint32)]
        L.orc_euclidean_matrix.argtypes = [_dp, _sz, _sz, _dp]
        L.orc_euclidean_matrix_mt.argtypes = [_dp, _sz, _sz, C.c_uint, _dp]
        L.orc_reconstruction_error.argtypes = [_dp, _sz, _dp, _sz]
        L.orc_reconstruction_error.restype = C.c_double
        L.orc_stable_rank.argtypes = [_dp, _sz, C.c_uint, _dp]
        L.orc_synth_points.argtypes = [C.c_int, _sz, _u64, _dp, C.POINTER(_sz)]
        L.orc_multiply_gram_otf_rows.argtypes = [_dp, _sz, _dp, C.c_double, _dp, _sz, _sz, _sz,
                                                 C.c_uint, _dp]
        L.orc_multiply_gram_otf_rows.restype = None
        L.orc_hamming_matrix_mt.argtypes = [C.c_char_p, _sz, _sz, C.c_uint, _dp]
        L.orc_synth_reads.argtypes = [_sz, _sz, _sz, C.c_double, _u64, C.c_char_p]
        L.orc_synth_reads.restype = None
        L.orc_sw_align.argtypes = [C.c_char_p, _sz, C.c_char_p, _sz, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_longlong)]
        L.orc_sw_distance.argtypes = [C.c_char_p, _sz, C.c_char_p, _sz, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_int)]

    def fill_gaussian(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.lib.orc_fill_gaussian(seed, _ptr(out), count)
        return out

    def gram_stats(self, d: np.ndarray, sym: bool = True):
        n = d.shape[0]
        rm = np.empty(n, np.float64)
        grand = C.c_double(0.0)
        st = self.lib.orc_gram_stats(_ptr(d), d.shape[0], d.shape[1], int(sym), _threads(),
                                     _ptr(rm), C.byref(grand))
        return st, rm, grand.value

    def gram(self, d: np.ndarray, sym: bool = True):
        g = np.empty((d.shape[0], d.shape[0]), np.float64)
        st = self.lib.orc_gram(_ptr(d), d.shape[0], d.shape[1], int(sym), _threads(), _ptr(g))
        return st, g

    def multiply_sym(self, g: np.ndarray, m: np.ndarray) -> np.ndarray:
        n, k = m.shape
        out = np.empty((n, k), np.float64)
        self.lib.orc_multiply_sym(_ptr(g), n, _ptr(np.ascontiguousarray(m)), k, _threads(), _ptr(out))
        return out

    def multiply_gram_otf(self, d, row_mean, grand, m, threads: int | None = None):
        n, k = m.shape
        out = np.empty((n, k), np.float64)
        self.lib.orc_multiply_gram_otf(_ptr(d), n, _ptr(row_mean), grand,
                                       _ptr(np.ascontiguousarray(m)), k, threads or _threads(),
                                       _ptr(out))
        return out

    def frobenius_sq(self, g: np.ndarray) -> float:
        return self.lib.orc_frobenius_sq(_ptr(g), g.shape[0], _threads())

    def thin_orthonormal(self, y: np.ndarray) -> np.ndarray:
        n, k = y.shape
        q = np.empty((n, k), np.float64)
        self.lib.orc_thin_orthonormal(_ptr(np.ascontiguousarray(y)), n, k, _ptr(q))
        return q

    def sym_evd(self, a: np.ndarray):
        n = a.shape[0]
        vals = np.empty(n); vecs = np.empty((n, n))
        st = self.lib.orc_sym_evd(_ptr(np.ascontiguousarray(a)), n, _ptr(vals), _ptr(vecs))
        return st, vals, vecs

    def eigs(self, rank, p, q, seed, g=None, d=None, row_mean=None, grand=0.0, vectors=True):
        n = (g if g is not None else d).shape[0]
        vals = np.zeros(max(rank, 1)); keep = _sz(0); resid = C.c_double(0)
        vecs = np.zeros((n, max(rank, 1))) if vectors else None
        st = self.lib.orc_eigs(_ptr(g), _ptr(d), _ptr(row_mean), grand, n, rank, p, q, seed,
                               _threads(), _ptr(vals), _ptr(vecs), C.byref(keep), C.byref(resid))
        k = keep.value
        v = None if vecs is None else np.ascontiguousarray(vecs.reshape(-1)[: n * k].reshape(n, k))
        return st, vals[:k].copy(), v, resid.value

    def embed(self, rank, p, q, seed, g=None, d=None, row_mean=None, grand=0.0):
        n = (g if g is not None else d).shape[0]
        coords = np.zeros(n * max(rank, 1)); ev = np.zeros(max(rank, 1))
        r = _sz(0); mass = C.c_double(0); tr = C.c_int(0); resid = C.c_double(0)
        st = self.lib.orc_embed(_ptr(g), _ptr(d), _ptr(row_mean), grand, n, rank, p, q, seed,
                                _threads(), _ptr(coords), _ptr(ev), C.byref(r), C.byref(mass),
                                C.byref(tr), C.byref(resid))
        rr = r.value
        return dict(status=st, r=rr, coords=coords[: n * rr].reshape(n, rr).copy(),
                    eigenvalues=ev[:rr].copy(), dropped_negative_mass=mass.value,
                    truncated=bool(tr.value), resid=resid.value)

    def hamming_counts(self, reads: bytes, count: int, length: int):
        out = np.empty((count, count), np.uint32)
        st = self.lib.orc_hamming_counts(reads, count, length,
                                         out.ctypes.data_as(C.POINTER(C.c_uint32)))
        return st, out

    def euclidean_matrix(self, pts: np.ndarray) -> np.ndarray:
        n, dim = pts.shape
        out = np.empty((n, n))
        self.lib.orc_euclidean_matrix(_ptr(np.ascontiguousarray(pts)), n, dim, _ptr(out))
        return out

    def multiply_gram_otf_rows(self, d, row_mean, grand, m, row_begin, row_end,
                               threads: int | None = None):
        n, k = m.shape
        out = np.empty((row_end - row_begin, k), np.float64)
        self.lib.orc_multiply_gram_otf_rows(_ptr(d), n, _ptr(row_mean), grand,
                                            _ptr(np.ascontiguousarray(m)), k, row_begin, row_end,
                                            threads or _threads(), _ptr(out))
        return out

    def hamming_matrix_mt(self, reads, length: int, threads: int | None = None) -> np.ndarray:
        n = len(reads)
        out = np.empty((n, n))
        st = self.lib.orc_hamming_matrix_mt(b"".join(reads), n, length, threads or _threads(),
                                            _ptr(out))
        assert st == 0, "non-ACGT read"
        return out

    def synth_points(self, config: int, n: int, seed: int) -> np.ndarray:
        dims = {1: 20, 2: 50, 3: 100, 4: 64}
        out = np.empty((n, dims[config]))
        dim = _sz(0)
        st = self.lib.orc_synth_points(config, n, seed, _ptr(out), C.byref(dim))
        assert st == 0 and dim.value == dims[config]
        return out

    def synth_reads(self, count: int, length: int = 400, ancestors: int = 50,
                    sub_rate: float = 0.05, seed: int = 0) -> list:
        buf = C.create_string_buffer(count * length)
        self.lib.orc_synth_reads(count, length, ancestors, C.c_double(sub_rate), seed, buf)
        raw = buf.raw
        return [raw[i * length:(i + 1) * length] for i in range(count)]

    def euclidean_matrix_mt(self, pts: np.ndarray, threads: int | None = None) -> np.ndarray:
        n, dim = pts.shape
        out = np.empty((n, n))
        self.lib.orc_euclidean_matrix_mt(_ptr(np.ascontiguousarray(pts)), n, dim,
                                         threads or _threads(), _ptr(out))
        return out

    def reconstruction_error(self, g, coords):
        n, r = coords.shape
        return self.lib.orc_reconstruction_error(_ptr(g), n, _ptr(np.ascontiguousarray(coords)), r)

    def sw_align(self, a: bytes, b: bytes, scheme=(1, -1, -2)):
        out = (C.c_longlong * 6)()
        st = self.lib.orc_sw_align(a, len(a), b, len(b), *scheme, out)
        return st, tuple(out)

    def sw_distance(self, a: bytes, b: bytes, scheme=(1, -1, -2)):
        out = C.c_int(0)
        st = self.lib.orc_sw_distance(a, len(a), b, len(b), *scheme, C.byref(out))
        return st, out.value

    def stable_rank(self, g):
        out = C.c_double(0)
        st = self.lib.orc_stable_rank(_ptr(g), g.shape[0], _threads(), C.byref(out))
        return st, out.value


class RefLib:
    """The reference's own sources compiled into oracle/_ref (see oracle/Makefile)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (built only where /root/reference exists)")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_fill_gaussian.argtypes = [_u64, _dp, _sz]
        L.ref_mt19937_64.argtypes = [_u64, C.POINTER(C.c_uint64), _sz]
        L.ref_uniform_box.argtypes = [_sz, _sz, _u64, _dp]
        L.ref_euclidean_matrix.argtypes = [_dp, _sz, _sz, _dp]
        L.ref_random_reads.argtypes = [_sz, _sz, _u64, C.c_char_p]
        L.ref_gram.argtypes = [_dp, _sz, _sz, C.c_int, C.c_uint, _dp]
        L.ref_multiply_sym.argtypes = [_dp, _sz, _dp, _sz, C.c_uint, _dp]
        L.ref_frobenius_sq.argtypes = [_dp, _sz, C.c_uint]
        L.ref_frobenius_sq.restype = C.c_double
        L.ref_randomized_range.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, C.c_uint, _dp]
        L.ref_eigs_sym.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, C.c_uint, _dp, _dp,
                                   C.POINTER(_sz), _dp]
        L.ref_stable_rank.argtypes = [_dp, _sz, C.c_uint, _dp]
        L.ref_write_matrix_tsv.argtypes = [C.c_char_p, _dp, _sz, _sz, C.c_int]
        L.ref_sw_align.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_longlong)]
        L.ref_sw_distance.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_int)]
        L.ref_pairwise_self.argtypes = [C.c_char_p, C.POINTER(_sz), _sz, C.c_int, C.c_int,
                                        C.c_int, C.c_uint, _dp]
        L.ref_pairwise_cross.argtypes = [C.c_char_p, C.POINTER(_sz), _sz, C.c_char_p,
                                         C.POINTER(_sz), _sz, C.c_int, C.c_int, C.c_int,
                                         C.c_uint, _dp]
        L.ref_embed.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, C.c_uint, _dp, _dp,
                                C.POINTER(_sz), _dp, C.POINTER(C.c_int)]
        L.ref_reconstruction_error.argtypes = [_dp, _sz, _dp, _sz, C.c_uint]
        L.ref_reconstruction_error.restype = C.c_double
        L.ref_write_matrix.argtypes = [C.c_char_p, _dp, _sz, _sz, C.c_int]
        L.ref_read_matrix.argtypes = [C.c_char_p, _dp, C.POINTER(_sz), C.POINTER(_sz),
                                      C.POINTER(C.c_int)]

    def fill_gaussian(self, seed, count):
        out = np.empty(count); self.lib.ref_fill_gaussian(seed, _ptr(out), count); return out

    def mt19937_64(self, seed, count):
        out = np.empty(count, np.uint64)
        self.lib.ref_mt19937_64(seed, out.ctypes.data_as(C.POINTER(C.c_uint64)), count)
        return out

    def uniform_box(self, n, dim, seed):
        out = np.empty((n, dim)); self.lib.ref_uniform_box(n, dim, seed, _ptr(out)); return out

    def euclidean_matrix(self, pts):
        n, dim = pts.shape
        out = np.empty((n, n))
        self.lib.ref_euclidean_matrix(_ptr(np.ascontiguousarray(pts)), n, dim, _ptr(out))
        return out

    def random_reads(self, count, length, seed) -> bytes:
        buf = C.create_string_buffer(count * length)
        self.lib.ref_random_reads(count, length, seed, buf)
        return buf.raw

    def gram(self, d, sym=True, threads=None):
        g = np.empty((d.shape[0], d.shape[0]))
        st = self.lib.ref_gram(_ptr(d), d.shape[0], d.shape[1], int(sym), threads or _threads(), _ptr(g))
        return st, g

    def multiply_sym(self, g, m, threads=None):
        n, k = m.shape
        out = np.empty((n, k))
        self.lib.ref_multiply_sym(_ptr(g), n, _ptr(np.ascontiguousarray(m)), k,
                                  threads or _threads(), _ptr(out))
        return out

    def frobenius_sq(self, g):
        return self.lib.ref_frobenius_sq(_ptr(g), g.shape[0], _threads())

    def randomized_range(self, g, rank, p, q, seed):
        n = g.shape[0]
        out = np.empty((n, rank + p))
        st = self.lib.ref_randomized_range(_ptr(g), n, rank, p, q, seed, _threads(), _ptr(out))
        return st, out

    def eigs(self, g, rank, p, q, seed, threads=None):
        n = g.shape[0]
        vals = np.zeros(max(rank, 1)); vecs = np.zeros(n * max(rank, 1))
        keep = _sz(0); resid = C.c_double(0)
        st = self.lib.ref_eigs_sym(_ptr(g), n, rank, p, q, seed, threads or _threads(), _ptr(vals),
                                   _ptr(vecs), C.byref(keep), C.byref(resid))
        k = keep.value
        return st, vals[:k].copy(), vecs[: n * k].reshape(n, k).copy(), resid.value

    def write_matrix_tsv(self, path, v, sym=True):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.lib.ref_write_matrix_tsv(str(path).encode(), _ptr(v), v.shape[0], v.shape[1],
                                             int(sym))

    def sw_align(self, a: bytes, b: bytes, scheme=(1, -1, -2)):
        out = (C.c_longlong * 6)()
        st = self.lib.ref_sw_align(a, b, *scheme, out)
        return st, tuple(out)

    def sw_distance(self, a: bytes, b: bytes, scheme=(1, -1, -2)):
        out = C.c_int(0)
        st = self.lib.ref_sw_distance(a, b, *scheme, C.byref(out))
        return st, out.value

    @staticmethod
    def _concat(seqs):
        offs = [0]
        for s in seqs:
            offs.append(offs[-1] + len(s))
        return b"".join(seqs), (C.c_size_t * len(offs))(*offs)

    def pairwise_self(self, seqs, scheme=(1, -1, -2), threads=None):
        cat, offs = self._concat(seqs)
        out = np.zeros((len(seqs), len(seqs)))
        st = self.lib.ref_pairwise_self(cat, offs, len(seqs), *scheme, threads or _threads(),
                                        _ptr(out))
        return st, out

    def pairwise_cross(self, q, r, scheme=(1, -1, -2), threads=None):
        qc, qo = self._concat(q)
        rc, ro = self._concat(r)
        out = np.zeros((len(q), len(r)))
        st = self.lib.ref_pairwise_cross(qc, qo, len(q), rc, ro, len(r), *scheme,
                                         threads or _threads(), _ptr(out))
        return st, out

    def stable_rank(self, g):
        out = C.c_double(0)
        st = self.lib.ref_stable_rank(_ptr(g), g.shape[0], _threads(), C.byref(out))
        return st, out.value

    def embed(self, g, rank, p, q, seed, threads=None):
        n = g.shape[0]
        coords = np.zeros(n * max(rank, 1)); ev = np.zeros(max(rank, 1))
        r = _sz(0); mass = C.c_double(0); tr = C.c_int(0)
        st = self.lib.ref_embed(_ptr(g), n, rank, p, q, seed, threads or _threads(), _ptr(coords),
                                _ptr(ev), C.byref(r), C.byref(mass), C.byref(tr))
        rr = r.value
        return dict(status=st, r=rr, coords=coords[: n * rr].reshape(n, rr).copy(),
                    eigenvalues=ev[:rr].copy(), dropped_negative_mass=mass.value,
                    truncated=bool(tr.value))

    def reconstruction_error(self, g, coords):
        n, r = coords.shape
        return self.lib.ref_reconstruction_error(_ptr(g), n, _ptr(np.ascontiguousarray(coords)), r, 1)

    def write_matrix(self, path, v, sym=True):
        return self.lib.ref_write_matrix(str(path).encode(), _ptr(np.ascontiguousarray(v)),
                                         v.shape[0], v.shape[1], int(sym))

    def read_matrix(self, path):
        rows = _sz(0); cols = _sz(0); sym = C.c_int(0)
        st = self.lib.ref_read_matrix(str(path).encode(), None, C.byref(rows), C.byref(cols), C.byref(sym))
        if st:
            return st, None, False
        v = np.empty((rows.value, cols.value))
        st = self.lib.ref_read_matrix(str(path).encode(), _ptr(v), C.byref(rows), C.byref(cols), C.byref(sym))
        return st, v, bool(sym.value)


def ref_available() -> bool:
    return REF_SO.exists()
