/* divscope-b200 — B200-native drop-in for the randomized classical-MDS path
 * of the reference `divscope` toolkit (arXiv:1803.02272).
 *
 * This is the C ABI the reference's own FFI binds for the MDS path. The
 * status enum, handle types, option struct and the semantics of every entry
 * point that also exists in the reference are kept exactly; each declaration
 * cites the reference declaration it replaces
 * (/root/reference/proj/include/divscope.h = "ref divscope.h", and
 * /root/reference/proj/src/capi.cpp = "ref capi.cpp").
 *
 * Conventions (ref divscope.h:1-9, ref capi.cpp:66-87):
 *  - every call returns divscope_status; nothing throws across the ABI;
 *  - NULL required arguments -> DIVSCOPE_ERR_INVALID_ARGUMENT ("null argument");
 *  - the failure message is thread-local (divscope_last_error);
 *  - out-handles are written only on success; the caller frees them;
 *  - handles are immutable once created and may be shared across threads.
 *
 * Device model: matrices live in the HBM of the calling process's CUDA
 * device (one process per GPU). divscope_gram returns a *lazy* gram handle:
 * it keeps the distance matrix resident plus its row means / grand mean and
 * never materializes G = -1/2 J D^2 J; divscope_matrix_get / _write evaluate
 * G on demand. The `threads` arguments are accepted for ABI compatibility and
 * ignored (the GPU path is not thread-count dependent). There is no CPU
 * fallback: without a usable CUDA device every compute call fails with
 * DIVSCOPE_ERR_INTERNAL.
 */
#ifndef DIVSCOPE_H
#define DIVSCOPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ref divscope.h:22-42 (values mirror errc, ref src/error.hpp:10-30) */
typedef enum divscope_status {
    DIVSCOPE_OK = 0,
    DIVSCOPE_ERR_IO,
    DIVSCOPE_ERR_EMPTY_INPUT,
    DIVSCOPE_ERR_INVALID_CHARACTER,
    DIVSCOPE_ERR_DUPLICATE_ID,
    DIVSCOPE_ERR_SAMPLE_TOO_LARGE,
    DIVSCOPE_ERR_EMPTY_SEQUENCE,
    DIVSCOPE_ERR_BAD_FORMAT,
    DIVSCOPE_ERR_TRUNCATED,
    DIVSCOPE_ERR_NOT_SYMMETRIC,
    DIVSCOPE_ERR_RANK_TOO_LARGE,
    DIVSCOPE_ERR_ZERO_MATRIX,
    DIVSCOPE_ERR_BAD_GAP,
    DIVSCOPE_ERR_SHAPE_MISMATCH,
    DIVSCOPE_ERR_MISSING_LABEL,
    DIVSCOPE_ERR_JOIN_ERROR,
    DIVSCOPE_ERR_BAD_AXIS,
    DIVSCOPE_ERR_INVALID_ARGUMENT,
    DIVSCOPE_ERR_INTERNAL
} divscope_status;

/* ref divscope.h:44 */
const char* divscope_status_name(divscope_status s);
/* ref divscope.h:49 */
const char* divscope_last_error(void);
/* ref divscope.h:51 */
const char* divscope_version(void);

/* ---- read-set ids (only what divscope_embed needs) ---------------------- */

/* ref divscope.h:55 (opaque type). FASTA ingestion is out of scope for this
 * path; a readset here is an ordered list of row ids. */
typedef struct divscope_readset divscope_readset;
/* NEW: build a readset of `count` ids (copied). */
divscope_status divscope_readset_from_ids(const char* const* ids, size_t count,
                                          divscope_readset** out);
/* ref divscope.h:62, :64, :71 */
/* NEW. A readset with sequences (ids NULL -> "0".."count-1"); sequences are
 * copied. (The reference builds readsets from FASTA, seqio.cpp; FASTA parsing
 * is out of scope here.) */
divscope_status divscope_readset_from_sequences(const char* const* ids,
                                                const char* const* sequences, size_t count,
                                                divscope_readset** out);
/* ref divscope.h:65 (NULL for ids-only readsets) */
const char* divscope_readset_sequence(const divscope_readset* rs, size_t i);
size_t divscope_readset_size(const divscope_readset* rs);
const char* divscope_readset_id(const divscope_readset* rs, size_t i);
void divscope_readset_free(divscope_readset* rs);

/* ---- matrices ------------------------------------------------------------ */

/* ref divscope.h:103 */
/* ---- Smith-Waterman alignment distances, on the GPU (ref divscope.h:73-112;
 * src/align.cpp:28-106, src/distmat.cpp:45-128): bit-exact distances, same
 * error codes. `threads` is accepted and ignored. */
typedef struct divscope_scoring {
    int match;    /* > 0 */
    int mismatch; /* < 0 */
    int gap;      /* < 0 */
} divscope_scoring;

/* 1 / -1 / -2 */
void divscope_scoring_init(divscope_scoring* s);

typedef struct divscope_alignment {
    int score;
    int distance;
    size_t a_begin, a_end; /* half-open spans of the locally aligned regions */
    size_t b_begin, b_end;
} divscope_alignment;

/* scoring == NULL selects the defaults */
divscope_status divscope_align(const char* a, const char* b, const divscope_scoring* scoring,
                               divscope_alignment* out);
/* Symmetric alignment distance (operands are ordered canonically first). */
divscope_status divscope_distance(const char* a, const char* b, const divscope_scoring* scoring,
                                  int* out);

typedef struct divscope_matrix divscope_matrix;

/* ref divscope.h:105-112: all pairs of a readset (symmetric n x n, zero
 * diagonal) / queries x refs; readsets must carry sequences. */
divscope_status divscope_pairwise_self(const divscope_readset* rs, const divscope_scoring* scoring,
                                       unsigned threads, divscope_matrix** out);
divscope_status divscope_pairwise_cross(const divscope_readset* queries,
                                        const divscope_readset* refs,
                                        const divscope_scoring* scoring, unsigned threads,
                                        divscope_matrix** out);

/* NEW (in-memory constructor a cgo/ctypes binding needs; the reference only
 * builds matrices via pairwise alignment or DVS files): copy a row-major
 * rows x cols float64 host buffer into device memory. Pinned host memory
 * gives the fastest upload. */
divscope_status divscope_matrix_from_host(const double* values, size_t rows, size_t cols,
                                          int symmetric, divscope_matrix** out);
/* NEW: float32 storage (BASELINE config 4). All arithmetic on it is fp64
 * (d is widened before squaring, so d^2 is exact). */
divscope_status divscope_matrix_from_host_f32(const float* values, size_t rows, size_t cols,
                                              int symmetric, divscope_matrix** out);
/* ref divscope.h:114-117 */
size_t divscope_matrix_rows(const divscope_matrix* m);
size_t divscope_matrix_cols(const divscope_matrix* m);
int divscope_matrix_symmetric(const divscope_matrix* m);
double divscope_matrix_get(const divscope_matrix* m, size_t i, size_t j);
/* NEW: copy the whole matrix (materializing G for a lazy gram) to a host
 * row-major buffer of rows*cols doubles. */
divscope_status divscope_matrix_copy_to_host(const divscope_matrix* m, double* out);
/* ref divscope.h:118-121 (DVS1 container, ref src/distmat.hpp:42-44) */
divscope_status divscope_matrix_write(const divscope_matrix* m, const char* dvs_path);
/* ref divscope.h:122-128: tab-separated export with an id header row; ids
 * from the given readsets (NULL -> 0-based index ids); a gram handle writes G */
divscope_status divscope_matrix_write_tsv(const divscope_matrix* m, const divscope_readset* row_ids,
                                          const divscope_readset* col_ids, const char* tsv_path);
divscope_status divscope_matrix_read(const char* dvs_path, divscope_matrix** out);

/* NEW. Rows [row_begin, row_end) of a symmetric DVS1 file as a row-shard
 * handle (the multi-GPU layout of divscope_shard_range): each rank reads only
 * its own rows, streamed from the file through pinned staging buffers into
 * HBM. Same errors as divscope_matrix_read; a non-symmetric file gives
 * DIVSCOPE_ERR_NOT_SYMMETRIC. (ref src/distmat.cpp:189-222 reads the whole
 * payload on one host.) */
divscope_status divscope_matrix_read_rows(const char* dvs_path, size_t row_begin,
                                          size_t row_end, divscope_matrix** out);
/* ref divscope.h:128 */
void divscope_matrix_free(divscope_matrix* m);
/* NEW: host-only DVS1 header / payload check (no device needed): shape and
 * symmetric flag of a DVS file, with read_matrix's error codes
 * (ref src/distmat.cpp:189-222). If values != NULL it receives rows*cols
 * doubles. */
divscope_status divscope_dvs_read_host(const char* dvs_path, size_t* rows, size_t* cols,
                                       int* symmetric, double* values);

/* ---- distance builders that feed the path (no reference equivalent) ----- */

/* NEW (BASELINE configs 1-4 input): exact Euclidean distances of `n` points
 * in R^dim (row-major host buffer), computed on the GPU with the reference
 * fixture's operation order (ref tests/testdata.cpp:165-184: sequential
 * coordinate sum, no FMA contraction, sqrt), so the result is bit-identical
 * to the CPU formula and exactly symmetric. store_f32 != 0 rounds the
 * stored distances to float32. */
divscope_status divscope_matrix_euclidean(const double* points, size_t n, size_t dim,
                                          int store_f32, divscope_matrix** out);
/* NEW (BASELINE config 5): normalized Hamming distance of `count` DNA reads
 * of equal `length` over {A,C,G,T} (concatenated, no separators): D_ij =
 * h_ij / length, h_ij = number of differing positions, computed on the GPU
 * from a 2-bit packed copy (XOR / fold / popcount). Reads containing any
 * other character fail with DIVSCOPE_ERR_INVALID_CHARACTER. */
divscope_status divscope_matrix_hamming(const char* reads, size_t count, size_t length,
                                        divscope_matrix** out);
/* NEW: the integer counts h (count x count, uint32) of the same computation,
 * for bit-exact checks. */
divscope_status divscope_hamming_counts(const char* reads, size_t count, size_t length,
                                        uint32_t* out);

/* ---- spectra and embeddings --------------------------------------------- */

/* ref divscope.h:132-137 */
typedef struct divscope_solver_options {
    size_t rank;
    size_t oversampling; /* clamped so rank + oversampling <= n for embed */
    size_t power_iters;
    uint64_t seed;
} divscope_solver_options;

/* ref divscope.h:140: rank 50, oversampling 10, power_iters 2, seed 0 */
void divscope_solver_options_init(divscope_solver_options* o);

/* ref divscope.h:144-145. Validates (square + symmetric flag, n > 0,
 * |d_ij - d_ji| <= 1e-12 max(1, max|d|)) and computes the row means of D^2
 * and the grand mean in one streaming pass over D (kernel K1). Returns a lazy
 * gram handle (G is never materialized). */
divscope_status divscope_gram(const divscope_matrix* dist, unsigned threads,
                              divscope_matrix** out);

/* ref divscope.h:151-154. Works on a lazy gram or on any explicit symmetric
 * matrix (symmetry checked to 1e-10 max(1, max|g|), ref rsvd.cpp:46-60). */
divscope_status divscope_eigs(const divscope_matrix* gram, const divscope_solver_options* opts,
                              unsigned threads, double* eigenvalues, size_t* count,
                              double* resid);

/* ref divscope.h:157-158: ||G||_F^2 / ||G||_S^2 (power iteration on the GPU). */
/* NEW (the reference has it in C++ only: eigs_sym's Spectrum::vectors,
 * src/rsvd.hpp:29-33, :43-62): divscope_eigs plus the Ritz vectors, row-major
 * n x count into `vectors` (n * opts->rank doubles), column a pairing with
 * eigenvalues[a]; sign as the eigensolver leaves it. Unsharded handles only. */
divscope_status divscope_eigs_vectors(const divscope_matrix* gram,
                                      const divscope_solver_options* opts, unsigned threads,
                                      double* eigenvalues, double* vectors, size_t* count,
                                      double* resid);
divscope_status divscope_stable_rank(const divscope_matrix* gram, unsigned threads,
                                     double* out);

/* ref divscope.h:160 */
typedef struct divscope_embedding divscope_embedding;

/* ref divscope.h:165-168 */
divscope_status divscope_embed(const divscope_matrix* gram, const divscope_solver_options* opts,
                               unsigned threads, const divscope_readset* ids,
                               divscope_embedding** out);
/* ref divscope.h:169-178 */
size_t divscope_embedding_rows(const divscope_embedding* e);
size_t divscope_embedding_dims(const divscope_embedding* e);
const char* divscope_embedding_id(const divscope_embedding* e, size_t i);
double divscope_embedding_get(const divscope_embedding* e, size_t i, size_t c);
size_t divscope_embedding_eigenvalues(const divscope_embedding* e, double* out, size_t cap);
double divscope_embedding_dropped_negative_mass(const divscope_embedding* e);
int divscope_embedding_truncated(const divscope_embedding* e);
/* NEW: pointer to the n x dims row-major coordinates (valid for the life of
 * the handle; NULL when dims == 0). divscope_embed leaves the coordinates in
 * device memory; the first host access (this call, _get, _write) downloads
 * them once. */
const double* divscope_embedding_coords(const divscope_embedding* e);
/* NEW: Frobenius-gap residual of the spectrum the embedding came from. */
double divscope_embedding_resid(const divscope_embedding* e);
/* ref divscope.h:180-185 (TSV `id dim1..dimr` + key=value meta sidecar) */
divscope_status divscope_embedding_write(const divscope_embedding* e, const char* tsv_path,
                                         const char* meta_path);
divscope_status divscope_embedding_load(const char* tsv_path, divscope_embedding** out);
void divscope_embedding_free(divscope_embedding* e);

/* NEW (ports the C++-only reference entry randomized_range, ref
 * src/rsvd.hpp:43-44, for its orthonormality / subspace KATs): writes the
 * n x (rank + oversampling) basis, row-major. Numerically rank-deficient
 * directions come back as zero columns (K3). */
/* NEW (the reference has it in C++ only, src/mds.hpp:54-58 / mds.cpp:126-150).
 * sqrt(sum_ij (g_ij - x_i . x_j)^2) of an embedding against its gram (lazy:
 * G evaluated on the fly from the upper triangle of D; explicit: stored
 * entries). DIVSCOPE_ERR_SHAPE_MISMATCH when the sizes differ. */
divscope_status divscope_reconstruction_error(const divscope_matrix* gram,
                                              const divscope_embedding* e, unsigned threads,
                                              double* out);

divscope_status divscope_randomized_range(const divscope_matrix* gram,
                                          const divscope_solver_options* opts, double* q_out);

/* ---- multi-GPU: one process per GPU, NCCL over NVLink (NEW) ------------ */

/* 128-byte NCCL unique id (create on rank 0, share out of band). */
divscope_status divscope_comm_unique_id(void* id128);
/* Join the communicator (collective over all ranks). While active, gram /
 * eigs / embed on row-sharded handles run the distributed algorithm. */
divscope_status divscope_comm_init(int world, int rank, const void* id128);
divscope_status divscope_comm_destroy(void);
/* Row shard [begin, end) of `rank` for an n x n matrix: the reference chunk
 * formula (ref src/parallel.hpp:33-34) over 256-row blocks. Host-only. */
divscope_status divscope_shard_range(size_t n, int world, int rank, size_t* begin, size_t* end);
/* This rank's rows [row_begin, row_end) of an n x n symmetric distance matrix
 * (row-major host buffer of (row_end-row_begin) x n). */
divscope_status divscope_matrix_from_host_rows(const double* rows, size_t n, size_t row_begin,
                                               size_t row_end, int symmetric,
                                               divscope_matrix** out);
divscope_status divscope_matrix_from_host_rows_f32(const float* rows, size_t n, size_t row_begin,
                                                   size_t row_end, int symmetric,
                                                   divscope_matrix** out);
/* This rank's rows [row_begin, row_end) of the Hamming distance matrix of
 * all `count` reads (K7 row shard; same values as divscope_matrix_hamming). */
divscope_status divscope_matrix_hamming_rows(const char* reads, size_t count, size_t length,
                                            size_t row_begin, size_t row_end,
                                            divscope_matrix** out);
/* This rank's rows of the exact Euclidean distance matrix of all n points. */
divscope_status divscope_matrix_euclidean_rows(const double* points, size_t n, size_t dim,
                                               int store_f32, size_t row_begin, size_t row_end,
                                               divscope_matrix** out);

/* ---- seeded workload synthesis (NEW; BASELINE.json configs) ------------ */

/* Points of BASELINE config `config` (1..4), n x dim row-major into `out`
 * (dim = 20, 50, 100, 64). Every draw follows the reference RNG conventions
 * (ref src/rng.hpp:16-48, std::mt19937_64(seed)); the recipe per config is
 * in DESIGN.md "Synthetic inputs". Returns the dimension via *dim_out. */
divscope_status divscope_synth_points(int config, size_t n, uint64_t seed, double* out,
                                      size_t* dim_out);
/* Config 5 reads: `count` reads of `length` bases copied from `ancestors`
 * seeded random ancestors with independent `sub_rate` substitutions,
 * concatenated into `out` (count * length chars, no terminator). */
divscope_status divscope_synth_reads(size_t count, size_t length, size_t ancestors,
                                     double sub_rate, uint64_t seed, char* out);

/* ---- device / instrumentation (NEW) ------------------------------------- */

/* NEW. Product-pass kernel: 0 = auto (int8 slice product on the integer
 * tensor cores for lazy grams with rank + oversampling <= 64 and n >= 4096,
 * else fp64 DMMA), 1 = fp64 DMMA only, 2 = int8 whenever supported. */
divscope_status divscope_set_product_path(int mode);

/* NEW. S-digit cache of the int8 product: 0 = off (a slot already filled
 * stays in the library's workspace until a failed allocation evicts it),
 * 1 = auto (default: on when the device has room for it next to a reserve of
 * max(1 GB, 2 %)), 2 = on whenever it fits. With it, divscope_gram (f64 D,
 * n >= 4096) also writes the exact digit bytes of D o D, or else a solve's
 * first product pass stores them, and the product passes read those instead
 * of D. Results equal the uncached path's to fp64 rounding (Hamming D and a
 * solve that stores its own: bit-identical). */
divscope_status divscope_set_sdig_cache(int mode);

/* Select the CUDA device used by this process (default: current device). */
divscope_status divscope_set_device(int device);

typedef struct divscope_stats {
    uint64_t kernel_launches;   /* kernels this library launched */
    uint64_t product_launches;  /* K2 launches (streaming product passes) */
    double product_ms;          /* summed K2 device time (CUDA events), when timing on */
    uint64_t stats_launches;    /* K1 launches (pass 0) */
    double stats_ms;            /* summed K1 device time, when timing on */
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    int32_t last_evd_sweeps;    /* Jacobi sweeps of the last Rayleigh-Ritz EVD */
    int32_t last_orth_shifted;  /* 1 if a shifted CholeskyQR step was needed */
    int32_t last_power_iters;   /* power iterations of the last stable_rank */
    int32_t last_product_kernel; /* 0 fp64 DMMA (k2_product), 1 int8 slice product */
    int32_t last_product_groups; /* int8 path: column groups = reads of D per product pass */
    int32_t last_product_sdigits; /* int8 path: bytes per S element (7; 3 for Hamming D) */
    int32_t last_product_pair;    /* int8 path: 1 when a CTA pair shared each D tile (64 < WP <= 96:
                                     both column groups in ONE read of D) */
    int32_t last_product_sdig;    /* int8 path: 1 when the S-digit cache was used (the first pass
                                     stored each element's SD digit bytes, the later passes read
                                     those instead of D) */
    uint64_t product_first_launches; /* the first product pass of each solve (also counted in
                                        product_launches): the storing pass with the cache on */
    double product_first_ms;          /* its summed device time, when timing on */
    int32_t last_product_stream_cl;   /* CTAs sharing each streamed digit item (0: no cache) */
} divscope_stats;

/* timing on => CUDA events are recorded around K1/K2 on the library stream */
void divscope_stats_enable_timing(int on);
void divscope_stats_reset(void);
void divscope_stats_get(divscope_stats* out);
/* stream the library enqueues on (cudaStream_t as void*) */
void* divscope_stream(void);
/* measured FP64 tensor-core (DMMA) throughput of this device in TFLOP/s
 * (roofline denominator of the FP64-bound product pass); < 0 on failure */
double divscope_fp64_tensor_peak_tflops(int iters);

#ifdef __cplusplus
}
#endif

#endif /* DIVSCOPE_H */
