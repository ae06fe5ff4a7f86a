// Launch interface of the divscope-b200 kernels (host side). Every launcher
// enqueues on the given stream and never synchronizes.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

namespace dsb {

constexpr int kRowPad = 256;  // panels / row blocks are padded to a multiple of this
constexpr int kMaxWP = 128;   // widest panel (rank + oversampling, padded to 8)

// indices into the K1 scalar block (double[16])
enum Scalar : int {
    S_GRAND = 0,       // grand mean of d^2 (mds.cpp:39-41)
    S_FRO2_LAZY = 1,   // ||G||_F^2 by the closed form 1/4 (sum d^4 - 2 n |r|^2 + n^2 g^2)
    S_FRO2_EXPL = 2,   // sum_ij a_ij^2 (explicit matrices, rsvd.cpp:64-79)
    S_MAXABS = 3,      // max |a_ij| over all entries (mds.cpp:21-22)
    S_MAXABS_UP = 4,   // max |a_ij| over i <= j (rsvd.cpp:50-54)
    S_MAXASYM = 5,     // max |a_ij - a_ji|
    S_SUM4 = 6,        // sum a^4
    S_SUMR = 7,        // sum_i r_i
    S_SUMR2 = 8,       // sum_i r_i^2
    S_ROWRATIO = 9,    // max_i 2^e_i / r_i (row max of d^2 over row mean, bound)
    S_SDIG_BAD = 10,   // K1 digits: 1 when a bound exponent is below a row's true
                       // exponent or more than 3 above it (the digits are unused)
    S_COUNT = 16,
};

enum class DType { F64 = 0, F32 = 1 };

// ---- K1: one streaming pass over D (tile pairs): row sums of squares,
// sum of fourth powers, max |d| and max |d_ij - d_ji| -----------------------
struct K1Work {
    double* part;        // [nbt][n_pad64] per-tile-column row partial sums
    int* pexp;           // [nbt][n_pad64] per-tile-column row exponents of max d^2
    double* cta_stats;   // [grid][4]
    double* blk_stats;   // [nblk][4]
    int* blk_bad;        // [nblk] S-digit bound violations per row block
    int grid;
};
size_t k1_part_elems(size_t n);
int k1_grid(size_t n, int sms);
// tmap64: TMA descriptor of D with 64-row x 128-byte boxes (SWIZZLE_128B)
// row_exp[i]: smallest e with d_ij^2 < 2^e for all j (the int8 slice scale)
// K1 writing the S-digit cache (f64 D): sd = 7 with row exponents row_eb
// (a bound from row 0, launch_row0_bound) or sd = 3 for Hamming D (hlen = L);
// nks = ceil(n / 32) k-steps per row block
struct K1Digits {
    unsigned char* sdig = nullptr;
    int* row_eb = nullptr;
    int nks = 0;
    int sd = 0;
    double hlen = 0.0;
};
void launch_k1(const CUtensorMap* tmap64, DType dt, size_t n, const K1Work& w, double* row_mean,
               int* row_exp, double* scalars, int sms, cudaStream_t st,
               const K1Digits* dig = nullptr);
// row_eb[i] = smallest e with (|d_0i| + max_j |d_0j|)^2 < 2^e, rounded up: by
// the triangle inequality a bound on row i's max d_ij^2 for a metric D (K1
// verifies it: scalars[S_SDIG_BAD])
void launch_row0_bound(const double* d, size_t n, int* row_eb, cudaStream_t st);

// ---- K1 for a row shard (rectangular rows x cols block): row sums of d^2,
// sum d^4 and max |d| (deterministic per-CTA partials), plus the shard's
// antisymmetric symmetry fingerprint (atomically added into *sym_fp; the
// sum over all shards is zero iff D is exactly symmetric)
int k1_rows_grid(size_t rows, int sms);
// row_exp[r]: smallest e with d_rj^2 < 2^e over the row (int8 slice product)
void launch_k1_rows(const void* d, DType dt, size_t ld, size_t rows, size_t cols, size_t row0,
                    double* rowsum, double* row_mean, double* cta_stats, int grid,
                    cudaStream_t st, int* row_exp, unsigned long long* sym_fp);
// fold of the K1-rows CTA partials (3 per CTA): red[0] sum d^4, red[1] max |d|,
// red[3] int8 admission ratio
void launch_shard_fold(const double* cta, int grid, double* red, cudaStream_t st);
// sums[0] = sum r_i, sums[1] = sum r_i^2 over the full row means (fixed order)
void launch_rowmean_sums(const double* row_mean, size_t n, double* sums, cudaStream_t st);
// max |A[i][j] - B[j][i]| over an m x p block A (lda) and p x m block B (ldb),
// atomically max-ed (non-negative doubles as u64) into *out
void launch_asym_block(const void* a, size_t lda, const void* b, size_t ldb, DType dt, size_t m,
                       size_t p, double* out, cudaStream_t st);

// ---- K2: centered skinny product Y = G X (stream-K, DMMA f64) -------------
struct K2Plan {
    int wp = 0;
    int cw = 8, bm = 128;   // consumer warps, rows per tile (16 per warp)
    int n = 0, nb = 0, nk = 0;
    long long total = 0;
    int grid = 0, maxseg = 0, stages = 0;
    int ks = 1;             // 128-byte D boxes per stage
    size_t smem = 0;
    size_t part_elems = 0;   // doubles needed for the partial workspace
};
K2Plan k2_plan(size_t n, int wp, DType dt, int sms);
// rows (output rows, D rows) != ncols (reduction length = panel rows used)
K2Plan k2_plan_rect(size_t rows, size_t ncols, int wp, DType dt, int sms);
// mode: 0 = explicit matrix (Y = A X), 1 = gram of D (D squared on the fly,
// then rank-3 centering).
// e0/e1 (may be null) are recorded around the streaming kernel only
int k2_warps(int wp);
int k2_ks(int wp, DType dt);
void launch_k2(const CUtensorMap* tmap, DType dt, int mode, const K2Plan& p, const double* x,
               double* part, const double* row_mean, const double* scalars,
               const double* colsums, double* y, size_t n_pad, cudaStream_t st,
               cudaEvent_t e0 = nullptr, cudaEvent_t e1 = nullptr, const int* skip = nullptr);

// k2_reduce for an explicit row-block height (bm = 128 or 256)
// slot table of a stream-K split (k2_reduce), uploaded once per split and
// kept in the workspace arena; call before a graph capture
const int* k2_slot_table(int nb, int nk, long long total, int P, int maxseg);
// one stream-K split of a product launch: nk k-steps per row block, `total`
// items over P work units, its partial slots start at slot `slot_base`
struct K2Split {
    int nk;
    long long total;
    int P, maxseg;
    long long slot_base;
};
const int* k2_slot_table_multi(int nb, const std::vector<K2Split>& splits);
// one reduce over several splits' partial slots (summed split by split)
void launch_k2_reduce_multi(int wp, int bm, const double* part, const std::vector<K2Split>& splits,
                            int n, int mode, const double* row_mean, const double* scalars,
                            const double* colsums, double* y, cudaStream_t st, const int* skip);
void launch_k2_reduce(int wp, int bm, const double* part, int maxseg, int nk, long long total,
                      int P, int n, int mode, const double* row_mean, const double* scalars,
                      const double* colsums, double* y, cudaStream_t st, const int* skip);

// ---- K2 on the integer tensor cores (k2i_product.cu): exact 7x7-digit
// slice product of D o D and the panel on tcgen05 kind::i8 (lazy grams,
// WP <= 64). row_exp from K1.
struct K2iPlan {
    static constexpr int kMaxGroups = 4;
    int nb = 0;             // padded panel width covered by the column groups (>= WP)
    int ngroups = 0;        // launches per pass (each streams D once)
    int gc0[kMaxGroups] = {};  // first panel column of each group
    int gnb[kMaxGroups] = {};  // MMA N per digit of each group (32 or 64)
    int nrows = 0, nblk = 0, nks = 0;
    long long total = 0;
    int grid = 0, maxseg = 0, colmax_grid = 0;  // grid: work units (CTAs, or CTA pairs)
    size_t part_elems = 0;  // doubles
    size_t bdig_bytes = 0;  // panel digit planes
    bool pair = false;      // w > 64: one pass by CTA pairs (a column group per CTA)
    size_t bdig_stride = 0; // pair: bytes between the two groups' digit planes
    int cl = 1;             // CTAs per work unit (2: the pair; streaming plans up to 4)
};
bool k2i_supported(int wp);
K2iPlan k2i_plan(size_t nrows, size_t ncols, int wp, int sms);
// the plan of the passes that stream the S-digit cache: WP <= 32 as
// k2i_plan, wider panels on clusters of ceil(WP / 32) <= 4 CTAs sharing every
// digit item, one 32-column group per CTA (sdigits: 7, or 3 for Hamming)
K2iPlan k2i_stream_plan(size_t nrows, size_t ncols, int wp, int sms, int sdigits);
// the sharded product over k-step ranges of D's columns (panel all-gather
// overlapped: ranges[0] needs only the local panel rows, the rest wait on
// `gathered`), one stream-K split and slot set per range, one reduce
size_t k2i_ranges_part_elems(const K2iPlan& full, int wp,
                             const std::vector<std::pair<int, int>>& ranges, int sms);
void launch_k2i_ranges(const CUtensorMap* tmap128, const CUtensorMap* tmap64, DType dt,
                       const K2iPlan& full, int wp, const double* x, const int* row_exp,
                       const int* col_exp, unsigned char* bdig, double* part,
                       const double* row_mean, const double* scalars, const double* colsums,
                       double* y, size_t y_rows_pad, cudaStream_t st, cudaEvent_t gathered,
                       const std::vector<std::pair<int, int>>& ranges, int sms, cudaEvent_t e0,
                       cudaEvent_t e1, int hamming_len, unsigned char* sdig = nullptr,
                       int sdig_mode = 0);
// pmax: colmax_grid * wp doubles; col_exp: nb ints (<= 128); bdig: bdig_bytes
// tmap64: 64-row boxes of the same D (the pair kernel's multicast halves)
void launch_k2i(const CUtensorMap* tmap128, const CUtensorMap* tmap64, DType dt, const K2iPlan& p,
                int wp, const double* x, size_t x_rows_pad, const int* row_exp, double* pmax,
                int* col_exp, unsigned char* bdig, double* part, const double* row_mean,
                const double* scalars, const double* colsums, double* y, size_t y_rows_pad,
                cudaStream_t st, cudaEvent_t e0 = nullptr, cudaEvent_t e1 = nullptr,
                const int* skip = nullptr, int hamming_len = 0, unsigned char* sdig = nullptr,
                int sdig_mode = 0, const K2iPlan* stream_plan = nullptr);
// bytes of the S-digit cache of a plan (sdigits: 7, or 3 for Hamming slices):
// the solve's first product pass stores every (row block, k-step) item's
// digit planes there (sdig_mode 1), the later passes stream them (mode 2)
size_t k2i_sdig_bytes(const K2iPlan& p, int sdigits);

// out[0] = sum of `count` doubles in a fixed order
void launch_sum_fixed(const double* partial, size_t count, double* out, cudaStream_t st);

// reconstruction_error (recon.cu, ref mds.cpp:126-150): out[0] = sum_ij
// (g_ij - x_i . x_j)^2 over a lazy gram of D (upper tiles only) or an explicit
// matrix; x: n x r row-major; partial: recon_blocks(n, lazy) doubles
size_t recon_blocks(size_t n, bool lazy);
void launch_recon(const void* d, DType dt, size_t ld, size_t n, bool lazy, const double* row_mean,
                  const double* scalars, const double* x, int r, double* partial, double* out,
                  cudaStream_t st);

// ---- Smith-Waterman distances (sw.cu) ----------------------------------------
struct SwPlan {
    int nstr_max = 0;        // 8-column strips of the longest read
    long long threads = 0;   // persistent threads (each owns scratch columns)
    size_t dirs_elems = 0;   // u16 traceback codes
    size_t hb_elems = 0;     // int boundary columns
    bool forward_only = false;  // k_sw_e: events carried forward, no traceback codes
};
SwPlan sw_plan(int max_len, int sms, int mode, int match, int mismatch, int gap);
// mode 0: pairs i < j of n_a reads (D symmetric, both halves written);
// 1: n_a queries x n_b refs; 2: one pair (reads 0, 1) as given -> aux[6]
void launch_sw(const unsigned char* seq, const long long* off, const int* len, int mode,
               long long n_a, long long n_b, long long npairs, int match, int mismatch, int gap,
               const SwPlan& p, unsigned short* dirs, int* hb, double* dout, size_t ld,
               long long* aux, cudaStream_t st);

// ---- panel kernels (n_pad x WP, k4-interleaved) -----------------------------
int panel_grid(size_t n_pad, int sms);
void launch_panel_from_rowmajor(const double* src, size_t n, int w, int wp, size_t n_pad,
                                double* dst, cudaStream_t st);
void launch_panel_to_rowmajor(const double* src, size_t n, int w, int wp, double* dst,
                              cudaStream_t st);
// colsums[0..wp) = 1^T X, colsums[wp..2wp) = r^T X (deterministic 2-level)
// With pmax/col_exp (int8 product): also the column max partials [P][wp] and
// the column exponents col_exp[0..nb) of the panel digits.
void launch_colsums(const double* x, const double* row_mean, size_t n, size_t n_pad, int wp,
                    double* partial, double* colsums, int sms, cudaStream_t st,
                    double* pmax = nullptr, int nb = 0, int* col_exp = nullptr);
// per-column max |x| from launch_colsums' pmax partials (P of them), and the
// int8 column exponents from such maxima (sharded product: local maxima are
// reduced over the ranks in between)
void launch_colmax(const double* pmax, int P, int wp, double* cmax, cudaStream_t st);
void launch_colexp(const double* cmax, int wp, int nb, int* col_exp, cudaStream_t st);
// out (wp x wp) = A^T B (deterministic 2-level). gate (nullable): skip the
// kernels unless gate[0] & 1 (the shift flag: a third CholeskyQR pass is only
// needed after a shifted first pass)
void launch_panel_dot(const double* a, const double* b, size_t n_pad, int wp, double* partial,
                      double* out, int sms, cudaStream_t st, const int* gate = nullptr);
// stable_rank power iteration, device side (ref rsvd.cpp:160-176): state =
// {sigma, norm, done, zero, iters, active}; norm of Y column 0, v = w / norm,
// convergence |norm - sigma| <= 1e-13 norm.
struct SrState {
    double sigma, norm;
    int done, zero, iters, active;
};
void launch_sr_step(const double* y, size_t n, int wp, double* partial, SrState* state, double* x,
                    int sms, cudaStream_t st);

// CholQR step on W = Y^T Y: rinv = R^{-1} with breakdown handling (shift /
// drop, K3); flags[0] |= 1 when shifted.
void launch_chol_inv(const double* w_mat, int wp, int w, size_t n, int allow_shift, double* rinv,
                     int* flags, cudaStream_t st);
// the fused kernel's L D L^T elimination (carrying L^{-1}) as one CTA, WP <= 64:
// rinv = R^{-1} with the shift (pass 0) / drop (later passes) rules; false
// when WP is not supported (use launch_chol_inv)
// With y (apply mode): q = y R^{-1} on the panel rows as well, one CTA per
// SM each computing the factor (rinv, nullable, written once); false when the
// rows per CTA do not fit shared memory (use the factor + apply kernels).
bool launch_chol_inv_elim(const double* w_mat, int wp, int w, size_t n, int pass, double* rinv,
                          int* flags, cudaStream_t st, const int* gate = nullptr,
                          const double* y = nullptr, double* q = nullptr, size_t n_pad = 0,
                          int sms = 0);
// q = y * rinv (row-wise, upper-triangular rinv); gated off: q = y
void launch_panel_apply(const double* y, const double* rinv, size_t n_pad, int wp, double* q,
                        cudaStream_t st, const int* gate = nullptr);

// K3 fast path for wp <= 32: the three CholeskyQR passes y -> t -> y -> out
// in one cooperative launch (returns false when not applicable / launch
// refused, in which case the caller uses the multi-kernel path).
int orth_fused_grid(size_t n_pad, int sms);
// cstat (nullable): per CTA [3][WP] column statistics of the result for the
// next product pass (1^T Q, r^T Q with row_mean (nullable -> 0), max |Q|);
// reduce with launch_colstats_final over orth_fused_grid() CTAs
bool launch_orth_fused(double* y, double* t, double* out, size_t n_pad, int wp, int w, size_t n,
                       double* partial, double* wsum, int* flags, int sms, cudaStream_t st,
                       const double* row_mean = nullptr, double* cstat = nullptr);
// colsums[0..wp) = sum_c s, [wp..2wp) = sum_c t; col_exp (nullable) from the
// maxima (int8 panel digits), over P per-CTA [3][wp] statistics
void launch_colstats_final(const double* cstat, int P, int wp, int nb, double* colsums,
                           int* col_exp, cudaStream_t st);

// ---- K5: Rayleigh-Ritz EVD + |lambda| ordering + embed filter (1 CTA) -----
struct EvdOut {
    double* vals;      // [w] eigenvalues in reference order (|lambda| desc, + first)
    double* vkeep;     // [w][r] eigenvectors of the embed-kept eigenvalues
    double* kept_vals; // [r]
    double* dmeta;     // [0]=resid [1]=dropped_negative_mass [2]=sum lambda^2
    int* imeta;        // [0]=keep [1]=r [2]=truncated [3]=sweeps [4]=converged
};
void launch_evd(const double* b, int wp, int w, int rank, int requested_rank,
                const double* scalars, int fro_index, const EvdOut& o, cudaStream_t st);

// ---- K6: lift U = Q V_keep, sign rule (mds.cpp:65-77), scale by sqrt(lambda)
void launch_lift(const double* q, size_t n, int wp, int w, const double* vkeep,
                 const double* kept_vals, const int* imeta, int rmax, double* coords,
                 double* partial, int sms, cudaStream_t st);
int lift_grid(size_t n, int sms);
// partial: P x rmax x (value, global row index); row_off = global index of local row 0
void launch_lift_partial(const double* q, size_t n, int wp, int w, const double* vkeep,
                         const int* imeta, int rmax, double* coords, double* partial,
                         long long row_off, int P, cudaStream_t st);
void launch_lift_finish(size_t n, const int* imeta, int P, int rmax, const double* kept_vals,
                        const double* partial, double* scale, double* coords, cudaStream_t st);

// ---- K9 / K7: distance builders --------------------------------------------
void launch_euclid(const double* pts, size_t n, int dim, void* d, DType dt, size_t ld,
                   cudaStream_t st);
// rows [row0, row0 + nrows) of the n x n matrix into d (row-major, local rows)
void launch_euclid_rows(const double* pts, size_t n, int dim, void* d, DType dt, size_t ld,
                        size_t row0, size_t nrows, cudaStream_t st);
// reads (count x length bytes, device) -> two bit planes lo/hi (count x words
// uint32 each, 32 bases per word); *bad = smallest linear index of a non-ACGT
// byte (preset to ~0)
void launch_pack_reads(const unsigned char* reads, size_t count, int length, int words,
                       uint32_t* lo, uint32_t* hi, unsigned long long* bad, int sms,
                       cudaStream_t st);
// K7: rows [row0, row0 + nrows) of the Hamming matrix from the bit planes:
// d (f64, D = h / L, leading dimension ld) and/or counts (u32, n x n);
// the full matrix is built from its upper-triangle tiles
void launch_hamming(const uint32_t* lo, const uint32_t* hi, size_t count, int words, int length,
                    double* d, size_t ld, uint32_t* counts, cudaStream_t st, size_t row0 = 0,
                    size_t nrows = static_cast<size_t>(-1));

// K7 on the int8 tensor cores (D only): false when not applicable (disabled
// by DSB_HAMMING_TC=0, or row0 not a multiple of 128), nothing launched
bool launch_hamming_tc(const uint32_t* lo, const uint32_t* hi, size_t count, int words, int length,
                       double* d, size_t ld, cudaStream_t st, size_t row0, size_t nrows);
bool hamming_tc_enabled();

// ---- misc ------------------------------------------------------------------
// Opt a kernel into the full shared-memory carve-out once (dynamic limit =
// 227 KB minus its static shared memory), so static + dynamic may exceed the
// 48 KB default.
void allow_dyn_smem(const void* kernel);
// dynamic shared memory >= bytes for `kernel` on the current device
void ensure_dyn_smem(const void* kernel, size_t bytes);
uint64_t kernel_launch_count();
// cudaEventRecord, as an event node when the stream is being captured into a
// graph (a plain record there only marks a capture dependency)
void record_timing_event(cudaEvent_t e, cudaStream_t st);
void count_launch(int k = 1);

}  // namespace dsb
