"""divscope-b200: B200-native drop-in for the randomized classical-MDS path of
the reference ``divscope`` toolkit (arXiv:1803.02272).

This module is the Python (ctypes) binding of the C ABI in
``include/divscope.h`` — the same binding a maintainer of the reference would
write against its shared library. Names, argument meaning
and error behaviour follow the reference's C API
(/root/reference/proj/include/divscope.h:130-185, src/capi.cpp:286-414):

* every failing call raises :class:`DivscopeError` carrying the reference
  status code and the thread-local message (``divscope_last_error``);
* ``threads`` arguments are accepted and ignored (the GPU path is
  thread-count independent);
* there is no CPU fallback: importing fails loudly when the CUDA library has
  not been built, and compute calls fail with ``DIVSCOPE_ERR_INTERNAL`` when
  no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from pathlib import Path
from typing import Sequence

import numpy as np

__all__ = [
    "Status", "DivscopeError", "SolverOptions", "Matrix", "Embedding", "Stats", "lib",
    "matrix_from_host", "matrix_from_host_f32", "matrix_read", "matrix_euclidean",
    "matrix_hamming", "matrix_hamming_rows", "hamming_counts", "gram", "eigs", "embed", "stable_rank",
    "randomized_range", "embedding_load", "synth_points", "synth_reads", "solver_options_init",
    "stats_enable_timing", "stats_reset", "set_product_path", "set_sdig_cache", "matrix_read_rows", "reconstruction_error", "Scoring", "Alignment",
    "align", "distance", "pairwise_self", "pairwise_cross", "stats_get", "set_device", "LIB_PATH",
    "fp64_tensor_peak_tflops", "stream_ptr", "eigs_vectors", "debug_omega_panel",
    "debug_fill_gaussian",
]

LIB_PATH = Path(os.environ.get("DSB_LIB_OVERRIDE") or Path(__file__).resolve().parent / "libdivscope_b200.so")


class Status(enum.IntEnum):
    """ref include/divscope.h:22-42"""
    OK = 0
    ERR_IO = 1
    ERR_EMPTY_INPUT = 2
    ERR_INVALID_CHARACTER = 3
    ERR_DUPLICATE_ID = 4
    ERR_SAMPLE_TOO_LARGE = 5
    ERR_EMPTY_SEQUENCE = 6
    ERR_BAD_FORMAT = 7
    ERR_TRUNCATED = 8
    ERR_NOT_SYMMETRIC = 9
    ERR_RANK_TOO_LARGE = 10
    ERR_ZERO_MATRIX = 11
    ERR_BAD_GAP = 12
    ERR_SHAPE_MISMATCH = 13
    ERR_MISSING_LABEL = 14
    ERR_JOIN_ERROR = 15
    ERR_BAD_AXIS = 16
    ERR_INVALID_ARGUMENT = 17
    ERR_INTERNAL = 18


class DivscopeError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = Status(status)
        self.message = message
        super().__init__(f"{self.status.name}: {message}")


class SolverOptions(C.Structure):
    """ref include/divscope.h:132-137"""
    _fields_ = [("rank", C.c_size_t), ("oversampling", C.c_size_t),
                ("power_iters", C.c_size_t), ("seed", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("product_launches", C.c_uint64),
                ("product_ms", C.c_double), ("stats_launches", C.c_uint64),
                ("stats_ms", C.c_double), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("last_evd_sweeps", C.c_int32), ("last_orth_shifted", C.c_int32),
                ("last_power_iters", C.c_int32), ("last_product_kernel", C.c_int32),
                ("last_product_groups", C.c_int32), ("last_product_sdigits", C.c_int32),
                ("last_product_pair", C.c_int32), ("last_product_sdig", C.c_int32),
                ("product_first_launches", C.c_uint64), ("product_first_ms", C.c_double),
                ("last_product_stream_cl", C.c_int32)]


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_vp = C.c_void_p
_sz = C.c_size_t
_st = C.c_int


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA library must be built first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    sig = {
        "divscope_status_name": ([_st], C.c_char_p),
        "divscope_last_error": ([], C.c_char_p),
        "divscope_version": ([], C.c_char_p),
        "divscope_readset_from_ids": ([C.POINTER(C.c_char_p), _sz, C.POINTER(_vp)], _st),
        "divscope_readset_size": ([_vp], _sz),
        "divscope_readset_id": ([_vp, _sz], C.c_char_p),
        "divscope_readset_free": ([_vp], None),
        "divscope_readset_from_sequences": ([C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), _sz,
                                             C.POINTER(_vp)], _st),
        "divscope_readset_sequence": ([_vp, _sz], C.c_char_p),
        "divscope_scoring_init": ([C.c_void_p], None),
        "divscope_align": ([C.c_char_p, C.c_char_p, C.c_void_p, C.c_void_p], _st),
        "divscope_distance": ([C.c_char_p, C.c_char_p, C.c_void_p, C.POINTER(C.c_int)], _st),
        "divscope_pairwise_self": ([_vp, C.c_void_p, C.c_uint, C.POINTER(_vp)], _st),
        "divscope_pairwise_cross": ([_vp, _vp, C.c_void_p, C.c_uint, C.POINTER(_vp)], _st),
        "divscope_matrix_from_host": ([_dp, _sz, _sz, C.c_int, C.POINTER(_vp)], _st),
        "divscope_matrix_from_host_f32": ([_fp, _sz, _sz, C.c_int, C.POINTER(_vp)], _st),
        "divscope_matrix_rows": ([_vp], _sz),
        "divscope_matrix_cols": ([_vp], _sz),
        "divscope_matrix_symmetric": ([_vp], C.c_int),
        "divscope_matrix_get": ([_vp, _sz, _sz], C.c_double),
        "divscope_matrix_copy_to_host": ([_vp, _dp], _st),
        "divscope_matrix_write": ([_vp, C.c_char_p], _st),
        "divscope_matrix_read": ([C.c_char_p, C.POINTER(_vp)], _st),
        "divscope_matrix_read_rows": ([C.c_char_p, _sz, _sz, C.POINTER(_vp)], _st),
        "divscope_matrix_write_tsv": ([_vp, _vp, _vp, C.c_char_p], _st),
        "divscope_reconstruction_error": ([_vp, _vp, C.c_uint, _dp], _st),
        "divscope_matrix_free": ([_vp], None),
        "divscope_dvs_read_host": ([C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(C.c_int),
                                    _dp], _st),
        "divscope_matrix_euclidean": ([_dp, _sz, _sz, C.c_int, C.POINTER(_vp)], _st),
        "divscope_matrix_hamming": ([C.c_char_p, _sz, _sz, C.POINTER(_vp)], _st),
        "divscope_hamming_counts": ([C.c_char_p, _sz, _sz, C.POINTER(C.c_uint32)], _st),
        "divscope_solver_options_init": ([C.POINTER(SolverOptions)], None),
        "divscope_gram": ([_vp, C.c_uint, C.POINTER(_vp)], _st),
        "divscope_eigs": ([_vp, C.POINTER(SolverOptions), C.c_uint, _dp, C.POINTER(_sz), _dp], _st),
        "divscope_eigs_vectors": ([_vp, C.POINTER(SolverOptions), C.c_uint, _dp, _dp,
                                   C.POINTER(_sz), _dp], _st),
        "divscope_debug_omega_panel": ([C.c_uint64, _sz, _sz, _dp], C.c_int),
        "divscope_debug_fill_gaussian": ([C.c_uint64, _sz, _dp], C.c_int),
        "divscope_stable_rank": ([_vp, C.c_uint, _dp], _st),
        "divscope_embed": ([_vp, C.POINTER(SolverOptions), C.c_uint, _vp, C.POINTER(_vp)], _st),
        "divscope_embedding_rows": ([_vp], _sz),
        "divscope_embedding_dims": ([_vp], _sz),
        "divscope_embedding_id": ([_vp, _sz], C.c_char_p),
        "divscope_embedding_get": ([_vp, _sz, _sz], C.c_double),
        "divscope_embedding_eigenvalues": ([_vp, _dp, _sz], _sz),
        "divscope_embedding_dropped_negative_mass": ([_vp], C.c_double),
        "divscope_embedding_truncated": ([_vp], C.c_int),
        "divscope_embedding_coords": ([_vp], _dp),
        "divscope_embedding_resid": ([_vp], C.c_double),
        "divscope_embedding_write": ([_vp, C.c_char_p, C.c_char_p], _st),
        "divscope_embedding_load": ([C.c_char_p, C.POINTER(_vp)], _st),
        "divscope_embedding_free": ([_vp], None),
        "divscope_randomized_range": ([_vp, C.POINTER(SolverOptions), _dp], _st),
        "divscope_synth_points": ([C.c_int, _sz, C.c_uint64, _dp, C.POINTER(_sz)], _st),
        "divscope_synth_reads": ([_sz, _sz, _sz, C.c_double, C.c_uint64, C.c_char_p], _st),
        "divscope_set_device": ([C.c_int], _st),
        "divscope_comm_unique_id": ([_vp], _st),
        "divscope_comm_init": ([C.c_int, C.c_int, _vp], _st),
        "divscope_comm_destroy": ([], _st),
        "divscope_shard_range": ([_sz, C.c_int, C.c_int, C.POINTER(_sz), C.POINTER(_sz)], _st),
        "divscope_matrix_from_host_rows": ([_dp, _sz, _sz, _sz, C.c_int, C.POINTER(_vp)], _st),
        "divscope_matrix_from_host_rows_f32": ([_fp, _sz, _sz, _sz, C.c_int, C.POINTER(_vp)], _st),
        "divscope_matrix_euclidean_rows": ([_dp, _sz, _sz, C.c_int, _sz, _sz, C.POINTER(_vp)], _st),
        "divscope_matrix_hamming_rows": ([C.c_char_p, _sz, _sz, _sz, _sz, C.POINTER(_vp)], _st),
        "divscope_stats_enable_timing": ([C.c_int], None),
        "divscope_set_product_path": ([C.c_int], C.c_int),
        "divscope_set_sdig_cache": ([C.c_int], C.c_int),
        "divscope_stats_reset": ([], None),
        "divscope_stats_get": ([C.POINTER(Stats)], None),
        "divscope_stream": ([], _vp),
        "divscope_fp64_tensor_peak_tflops": ([C.c_int], C.c_double),
        "divscope_bench_product": ([_vp, C.c_int, C.c_int, C.c_int], C.c_double),
        "divscope_bench_product": ([_vp, C.c_int, C.c_int, C.c_int], C.c_double),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()

def _check(status: int) -> None:
    if status != 0:
        raise DivscopeError(status, (lib.divscope_last_error() or b"").decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def solver_options_init() -> SolverOptions:
    """ref capi.cpp:288-294 (rank 50, oversampling 10, power_iters 2, seed 0)"""
    o = SolverOptions()
    lib.divscope_solver_options_init(C.byref(o))
    return o


def _opts(rank=None, oversampling=None, power_iters=None, seed=None, opts=None) -> SolverOptions:
    o = opts if opts is not None else solver_options_init()
    if rank is not None:
        o.rank = rank
    if oversampling is not None:
        o.oversampling = oversampling
    if power_iters is not None:
        o.power_iters = power_iters
    if seed is not None:
        o.seed = seed
    return o


class Matrix:
    """Owning wrapper of a ``divscope_matrix*`` (device resident)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.divscope_matrix_free(h)
            self._h = C.c_void_p()

    @property
    def rows(self) -> int:
        return lib.divscope_matrix_rows(self._h)

    @property
    def cols(self) -> int:
        return lib.divscope_matrix_cols(self._h)

    @property
    def symmetric(self) -> bool:
        return bool(lib.divscope_matrix_symmetric(self._h))

    def get(self, i: int, j: int) -> float:
        return lib.divscope_matrix_get(self._h, i, j)

    def to_numpy(self) -> np.ndarray:
        out = np.empty((self.rows, self.cols), np.float64)
        _check(lib.divscope_matrix_copy_to_host(self._h, out.ctypes.data_as(_dp)))
        return out

    def write(self, path) -> None:
        _check(lib.divscope_matrix_write(self._h, str(path).encode()))

    def write_tsv(self, path, row_ids=None, col_ids=None) -> None:
        """ref divscope_matrix_write_tsv (ids default to 0-based indices)."""
        def rs(ids):
            if ids is None:
                return None, None
            arr = (C.c_char_p * len(ids))(*[str(i).encode() for i in ids])
            h = _vp()
            _check(lib.divscope_readset_from_ids(arr, len(ids), C.byref(h)))
            return h, arr
        (rh, ra), (ch, ca) = rs(row_ids), rs(col_ids)
        try:
            _check(lib.divscope_matrix_write_tsv(self._h, rh, ch, str(path).encode()))
        finally:
            for h in (rh, ch):
                if h is not None and h.value:
                    lib.divscope_readset_free(h)


def _new_matrix(fn, *args) -> Matrix:
    h = _vp()
    _check(fn(*args, C.byref(h)))
    return Matrix(h.value)


def matrix_from_host(values: np.ndarray, symmetric: bool = True) -> Matrix:
    a = _f64(values)
    rows, cols = a.shape
    return _new_matrix(lib.divscope_matrix_from_host, a.ctypes.data_as(_dp), rows, cols,
                       int(symmetric))


def matrix_from_host_f32(values: np.ndarray, symmetric: bool = True) -> Matrix:
    a = np.ascontiguousarray(values, dtype=np.float32)
    rows, cols = a.shape
    return _new_matrix(lib.divscope_matrix_from_host_f32, a.ctypes.data_as(_fp), rows, cols,
                       int(symmetric))


def matrix_read(path) -> Matrix:
    return _new_matrix(lib.divscope_matrix_read, str(path).encode())


def matrix_read_rows(path, row_begin: int, row_end: int) -> Matrix:
    """Rows [row_begin, row_end) of a symmetric DVS1 file as a row-shard handle."""
    return _new_matrix(lib.divscope_matrix_read_rows, str(path).encode(), row_begin, row_end)


def dvs_read_host(path) -> tuple[np.ndarray, bool]:
    """DVS1 file -> (values, symmetric) on the host (no device needed)."""
    rows, cols, sym = _sz(0), _sz(0), C.c_int(0)
    _check(lib.divscope_dvs_read_host(str(path).encode(), C.byref(rows), C.byref(cols),
                                      C.byref(sym), None))
    out = np.empty((rows.value, cols.value), np.float64)
    _check(lib.divscope_dvs_read_host(str(path).encode(), C.byref(rows), C.byref(cols),
                                      C.byref(sym), out.ctypes.data_as(_dp)))
    return out, bool(sym.value)


def matrix_euclidean(points: np.ndarray, store_f32: bool = False) -> Matrix:
    p = _f64(points)
    n, dim = p.shape
    return _new_matrix(lib.divscope_matrix_euclidean, p.ctypes.data_as(_dp), n, dim,
                       int(store_f32))


def _reads_bytes(reads) -> tuple[bytes, int, int]:
    if isinstance(reads, (bytes, bytearray)):
        raise TypeError("pass a list of equal-length reads")
    if isinstance(reads, np.ndarray):
        # count x length uint8 array (e.g. pinned host memory): passed in place
        if reads.dtype != np.uint8 or reads.ndim != 2 or not reads.flags["C_CONTIGUOUS"]:
            raise TypeError("reads array must be C-contiguous uint8, count x length")
        return reads.ctypes.data_as(C.c_char_p), reads.shape[0], reads.shape[1]
    reads = [r.encode() if isinstance(r, str) else bytes(r) for r in reads]
    if not reads:
        return b"", 0, 0
    length = len(reads[0])
    if any(len(r) != length for r in reads):
        raise DivscopeError(Status.ERR_SHAPE_MISMATCH, "reads must have equal length")
    return b"".join(reads), len(reads), length


def matrix_hamming(reads: Sequence[str | bytes]) -> Matrix:
    buf, count, length = _reads_bytes(reads)
    return _new_matrix(lib.divscope_matrix_hamming, buf, count, length)


def matrix_hamming_rows(reads: Sequence[str | bytes], row_begin: int, row_end: int) -> Matrix:
    """NEW divscope_matrix_hamming_rows: this rank's rows of the Hamming D (K7)."""
    buf, count, length = _reads_bytes(reads)
    return _new_matrix(lib.divscope_matrix_hamming_rows, buf, count, length, row_begin, row_end)


def hamming_counts(reads: Sequence[str | bytes]) -> np.ndarray:
    buf, count, length = _reads_bytes(reads)
    out = np.empty((count, count), np.uint32)
    _check(lib.divscope_hamming_counts(buf, count, length, out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out


def gram(dist: Matrix, threads: int = 1) -> Matrix:
    """ref divscope_gram (capi.cpp:296-307): lazy gram handle."""
    return _new_matrix(lib.divscope_gram, dist.handle, threads)


def eigs(g: Matrix, rank=None, oversampling=None, power_iters=None, seed=None, opts=None,
         threads: int = 1) -> tuple[np.ndarray, float]:
    """ref divscope_eigs (capi.cpp:309-325): (eigenvalues[count], resid)."""
    o = _opts(rank, oversampling, power_iters, seed, opts)
    vals = np.zeros(max(int(o.rank), 1), np.float64)
    count = _sz(0)
    resid = C.c_double(-1.0)
    _check(lib.divscope_eigs(g.handle, C.byref(o), threads, vals.ctypes.data_as(_dp),
                             C.byref(count), C.byref(resid)))
    return vals[: count.value].copy(), resid.value


def eigs_vectors(g: Matrix, rank=None, oversampling=None, power_iters=None, seed=None,
                 opts=None, threads: int = 1) -> tuple[np.ndarray, np.ndarray, float]:
    """divscope_eigs_vectors — the reference's C++ eigs_sym (rsvd.hpp:43-62)
    with Spectrum::vectors: (eigenvalues[count], vectors n x count, resid)."""
    o = _opts(rank, oversampling, power_iters, seed, opts)
    n = g.rows
    k = max(int(o.rank), 1)
    vals = np.zeros(k, np.float64)
    vecs = np.zeros(n * k, np.float64)
    count = _sz(0)
    resid = C.c_double(-1.0)
    _check(lib.divscope_eigs_vectors(g.handle, C.byref(o), threads, vals.ctypes.data_as(_dp),
                                     vecs.ctypes.data_as(_dp), C.byref(count), C.byref(resid)))
    c = count.value
    return vals[:c].copy(), vecs[: n * c].reshape(n, c).copy(), resid.value


def debug_omega_panel(seed: int, n: int, w: int) -> np.ndarray:
    """Test hook: Omega (n x w) exactly as a solve uploads it to the device."""
    out = np.zeros(n * w, np.float64)
    _check(lib.divscope_debug_omega_panel(seed, n, w, out.ctypes.data_as(_dp)))
    return out.reshape(n, w)


def debug_fill_gaussian(seed: int, count: int) -> np.ndarray:
    """Test hook (host only): the product's fill_gaussian over mt19937_64(seed)."""
    out = np.zeros(count, np.float64)
    _check(lib.divscope_debug_fill_gaussian(seed, count, out.ctypes.data_as(_dp)))
    return out


def stable_rank(g: Matrix, threads: int = 1) -> float:
    out = C.c_double(0.0)
    _check(lib.divscope_stable_rank(g.handle, threads, C.byref(out)))
    return out.value


def randomized_range(g: Matrix, rank=None, oversampling=None, power_iters=None, seed=None,
                     opts=None) -> np.ndarray:
    o = _opts(rank, oversampling, power_iters, seed, opts)
    n = g.rows
    out = np.zeros((n, int(o.rank + o.oversampling)), np.float64)
    _check(lib.divscope_randomized_range(g.handle, C.byref(o), out.ctypes.data_as(_dp)))
    return out


class Embedding:
    """Owning wrapper of a ``divscope_embedding*`` (coordinates stay on the device
    until first read, then are cached on the host)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.divscope_embedding_free(h)
            self._h = C.c_void_p()

    @property
    def rows(self) -> int:
        return lib.divscope_embedding_rows(self._h)

    @property
    def dims(self) -> int:
        return lib.divscope_embedding_dims(self._h)

    def id(self, i: int) -> str | None:
        s = lib.divscope_embedding_id(self._h, i)
        return None if s is None else s.decode()

    def get(self, i: int, c: int) -> float:
        return lib.divscope_embedding_get(self._h, i, c)

    @property
    def coords(self) -> np.ndarray:
        n, r = self.rows, self.dims
        if n * r == 0:
            return np.zeros((n, r))
        p = lib.divscope_embedding_coords(self._h)
        return np.ctypeslib.as_array(p, shape=(n * r,)).reshape(n, r).copy()

    @property
    def eigenvalues(self) -> np.ndarray:
        k = lib.divscope_embedding_eigenvalues(self._h, None, 0)
        out = np.zeros(max(k, 1))
        lib.divscope_embedding_eigenvalues(self._h, out.ctypes.data_as(_dp), k)
        return out[:k].copy()

    @property
    def dropped_negative_mass(self) -> float:
        return lib.divscope_embedding_dropped_negative_mass(self._h)

    @property
    def truncated(self) -> bool:
        return bool(lib.divscope_embedding_truncated(self._h))

    @property
    def resid(self) -> float:
        return lib.divscope_embedding_resid(self._h)

    def write(self, tsv_path, meta_path=None) -> None:
        _check(lib.divscope_embedding_write(self._h, str(tsv_path).encode(),
                                            None if meta_path is None else str(meta_path).encode()))


def embed(g: Matrix, rank=None, oversampling=None, power_iters=None, seed=None, opts=None,
          ids: Sequence[str] | None = None, threads: int = 1) -> Embedding:
    """ref divscope_embed (capi.cpp:337-354)."""
    o = _opts(rank, oversampling, power_iters, seed, opts)
    rs = _vp()
    try:
        if ids is not None:
            arr = (C.c_char_p * len(ids))(*[s.encode() for s in ids])
            _check(lib.divscope_readset_from_ids(arr, len(ids), C.byref(rs)))
        h = _vp()
        _check(lib.divscope_embed(g.handle, C.byref(o), threads, rs, C.byref(h)))
        return Embedding(h.value)
    finally:
        if rs.value:
            lib.divscope_readset_free(rs)


def reconstruction_error(g: Matrix, e: "Embedding", threads: int = 1) -> float:
    """ref mds.cpp:126-150 (sqrt of sum_ij (g_ij - x_i . x_j)^2)."""
    out = C.c_double(0.0)
    _check(lib.divscope_reconstruction_error(g.handle, e._h, threads, C.byref(out)))
    return out.value


class Scoring(C.Structure):
    """ref divscope_scoring (divscope.h:75-79); defaults 1 / -1 / -2."""
    _fields_ = [("match", C.c_int), ("mismatch", C.c_int), ("gap", C.c_int)]

    def __init__(self, match=1, mismatch=-1, gap=-2):
        super().__init__(match, mismatch, gap)


class Alignment(C.Structure):
    _fields_ = [("score", C.c_int), ("distance", C.c_int), ("a_begin", _sz), ("a_end", _sz),
                ("b_begin", _sz), ("b_end", _sz)]


def _seq(s) -> bytes:
    return s.encode() if isinstance(s, str) else bytes(s)


def align(a, b, scoring: Scoring | None = None) -> Alignment:
    """ref divscope_align: Smith-Waterman with the deterministic traceback (GPU)."""
    out = Alignment()
    _check(lib.divscope_align(_seq(a), _seq(b), C.byref(scoring) if scoring else None,
                              C.byref(out)))
    return out


def distance(a, b, scoring: Scoring | None = None) -> int:
    """ref divscope_distance (canonical operand order)."""
    out = C.c_int(0)
    _check(lib.divscope_distance(_seq(a), _seq(b), C.byref(scoring) if scoring else None,
                                 C.byref(out)))
    return out.value


class _Readset:
    def __init__(self, seqs, ids=None):
        seqs = [_seq(s) for s in seqs]
        sa = (C.c_char_p * len(seqs))(*seqs)
        ia = None
        if ids is not None:
            ia = (C.c_char_p * len(ids))(*[_seq(i) for i in ids])
        self.h = _vp()
        _check(lib.divscope_readset_from_sequences(ia, sa, len(seqs), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.divscope_readset_free(self.h)


def pairwise_self(seqs, scoring: Scoring | None = None, ids=None) -> Matrix:
    """ref divscope_pairwise_self: n x n Smith-Waterman distance matrix (GPU)."""
    rs = _Readset(seqs, ids)
    return _new_matrix(lib.divscope_pairwise_self, rs.h, C.byref(scoring) if scoring else None,
                       1)


def pairwise_cross(queries, refs, scoring: Scoring | None = None) -> Matrix:
    """ref divscope_pairwise_cross: queries x refs distance matrix (GPU)."""
    q, r = _Readset(queries), _Readset(refs)
    return _new_matrix(lib.divscope_pairwise_cross, q.h, r.h,
                       C.byref(scoring) if scoring else None, 1)


def embedding_load(path) -> Embedding:
    h = _vp()
    _check(lib.divscope_embedding_load(str(path).encode(), C.byref(h)))
    return Embedding(h.value)


def synth_points(config: int, n: int, seed: int) -> np.ndarray:
    dims = {1: 20, 2: 50, 3: 100, 4: 64}
    out = np.empty((n, dims[config]), np.float64)
    d = _sz(0)
    _check(lib.divscope_synth_points(config, n, seed, out.ctypes.data_as(_dp), C.byref(d)))
    return out


def synth_reads(count: int, length: int = 400, ancestors: int = 50, sub_rate: float = 0.05,
                seed: int = 0) -> list[bytes]:
    buf = C.create_string_buffer(count * length)
    _check(lib.divscope_synth_reads(count, length, ancestors, sub_rate, seed, buf))
    raw = buf.raw
    return [raw[i * length:(i + 1) * length] for i in range(count)]


# ---- multi-GPU -----------------------------------------------------------

def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.divscope_comm_unique_id(buf))
    return buf.raw


def comm_init(world: int, rank: int, uid: bytes) -> None:
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(lib.divscope_comm_init(world, rank, buf))


def comm_destroy() -> None:
    _check(lib.divscope_comm_destroy())


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    b, e = _sz(0), _sz(0)
    _check(lib.divscope_shard_range(n, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def matrix_from_host_rows(rows: np.ndarray, n: int, row_begin: int, row_end: int,
                          symmetric: bool = True) -> Matrix:
    a = _f64(rows)
    return _new_matrix(lib.divscope_matrix_from_host_rows, a.ctypes.data_as(_dp), n, row_begin,
                       row_end, int(symmetric))


def matrix_from_host_rows_f32(rows: np.ndarray, n: int, row_begin: int, row_end: int,
                              symmetric: bool = True) -> Matrix:
    a = np.ascontiguousarray(rows, dtype=np.float32)
    return _new_matrix(lib.divscope_matrix_from_host_rows_f32, a.ctypes.data_as(_fp), n,
                       row_begin, row_end, int(symmetric))


def matrix_euclidean_rows(points: np.ndarray, row_begin: int, row_end: int,
                          store_f32: bool = False) -> Matrix:
    p = _f64(points)
    n, dim = p.shape
    return _new_matrix(lib.divscope_matrix_euclidean_rows, p.ctypes.data_as(_dp), n, dim,
                       int(store_f32), row_begin, row_end)


def set_device(device: int) -> None:
    _check(lib.divscope_set_device(device))


def set_product_path(mode: int) -> None:
    """0 auto, 1 fp64 DMMA only, 2 int8 slice product whenever supported."""
    _check(lib.divscope_set_product_path(int(mode)))


def set_sdig_cache(mode: int) -> None:
    """S-digit cache of the int8 product: 0 off, 1 auto, 2 whenever it fits."""
    _check(lib.divscope_set_sdig_cache(int(mode)))


def stats_enable_timing(on: bool = True) -> None:
    lib.divscope_stats_enable_timing(int(on))


def stats_reset() -> None:
    lib.divscope_stats_reset()


def fp64_tensor_peak_tflops(iters: int = 20000) -> float:
    return lib.divscope_fp64_tensor_peak_tflops(iters)


def bench_product(m: "Matrix", wp: int, mode: int = 1, iters: int = 5) -> float:
    """mean device ms of one K2 streaming-product launch (kernel tuning aid)"""
    return lib.divscope_bench_product(m.handle, wp, mode, iters)


def bench_product(m: "Matrix", wp: int, mode: int = 1, iters: int = 5) -> float:
    """mean device ms of one K2 streaming-product launch (kernel tuning aid)"""
    return lib.divscope_bench_product(m.handle, wp, mode, iters)


def stream_ptr() -> int:
    return lib.divscope_stream() or 0


def stats_get() -> Stats:
    s = Stats()
    lib.divscope_stats_get(C.byref(s))
    return s
