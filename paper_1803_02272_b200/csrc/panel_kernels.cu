// Panel kernels of the range finder and Rayleigh-Ritz step:
//   * layout conversion of Omega (host row-major -> k4-interleaved panel),
//   * column sums 1^T X and r^T X for the rank-3 centering of K2,
//   * K3: CholeskyQR with shift / drop breakdown handling — panel Gram
//     A^T B on the f64 tensor cores, single-CTA Cholesky + triangular
//     inverse, and the row-wise apply Q = Y R^{-1}
//     (replaces thin_orthonormal = Eigen HouseholderQR, ref rsvd.cpp:38-44),
//   * K4: the Ritz Gram Q^T (G Q) is launch_panel_dot on (Q, GQ)
//     (ref rsvd.cpp:109-110).
// All reductions are two-level with a fixed CTA order, so results are
// bit-identical run to run.
#include <algorithm>
#include <stdexcept>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace dsb {

namespace {

__global__ void k_panel_from_rowmajor(const double* __restrict__ src, size_t n, int w, int wp,
                                      size_t n_pad, double* __restrict__ dst) {
    const size_t total = n_pad * wp;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        // e enumerates the destination in memory order
        const size_t q = e / (static_cast<size_t>(wp) * 4);
        const int rem = static_cast<int>(e % (static_cast<size_t>(wp) * 4));
        const int c = rem / 4;
        const size_t i = q * 4 + (rem & 3);
        dst[e] = (i < n && c < w) ? src[i * w + c] : 0.0;
    }
}

__global__ void k_panel_to_rowmajor(const double* __restrict__ src, size_t n, int w, int wp,
                                    double* __restrict__ dst) {
    const size_t total = n * w;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t i = e / w;
        const int c = static_cast<int>(e % w);
        dst[e] = src[pidx(i, c, wp)];
    }
}

// colsum partials: CTA c handles k4 row blocks [nq c / P, nq (c+1) / P);
// optionally also the column max |x| (int8 product: column exponents)
__global__ void __launch_bounds__(256) k_colsum_partial(const double* __restrict__ x,
                                                        const double* __restrict__ row_mean,
                                                        size_t n, size_t n_pad, int wp,
                                                        double* __restrict__ partial,
                                                        double* __restrict__ pmax) {
    extern __shared__ double sh[];  // [3][wp*4]
    const size_t nq = n_pad / 4;
    const size_t q0 = nq * blockIdx.x / gridDim.x, q1 = nq * (blockIdx.x + 1) / gridDim.x;
    const int per = wp * 4;
    for (int e = threadIdx.x; e < per; e += blockDim.x) {
        double s = 0.0, t = 0.0, m = 0.0;
        const int rr = e & 3;
        for (size_t q = q0; q < q1; ++q) {
            const double v = x[q * per + e];
            const size_t i = q * 4 + rr;
            s += v;
            m = fmax(m, fabs(v));
            if (i < n) t += row_mean[i] * v;
        }
        sh[e] = s;
        sh[per + e] = t;
        sh[2 * per + e] = m;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < wp; c += blockDim.x) {
        const double s = ((sh[4 * c] + sh[4 * c + 1]) + sh[4 * c + 2]) + sh[4 * c + 3];
        const double t =
            ((sh[per + 4 * c] + sh[per + 4 * c + 1]) + sh[per + 4 * c + 2]) + sh[per + 4 * c + 3];
        partial[static_cast<size_t>(blockIdx.x) * 2 * wp + c] = s;
        partial[static_cast<size_t>(blockIdx.x) * 2 * wp + wp + c] = t;
        if (pmax) {
            const double* mm = sh + 2 * per + 4 * c;
            pmax[static_cast<size_t>(blockIdx.x) * wp + c] =
                fmax(fmax(mm[0], mm[1]), fmax(mm[2], mm[3]));
        }
    }
}

// out[e] = sum_c partial[c][e]. A block owns 32 consecutive e (one per lane);
// its 32 warps take fixed strided subsets of c, combined in warp order, so the
// result is deterministic for a fixed P.
__global__ void __launch_bounds__(1024) k_sum_partials(const double* __restrict__ partial, int P,
                                                       int m, double* __restrict__ out,
                                                       const int* __restrict__ gate = nullptr) {
    if (gate && !(gate[0] & 1)) return;  // shift-gated third CholeskyQR pass
    __shared__ double sh[32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * 32 + lane;
    double s = 0.0;
    if (e < m) {
#pragma unroll 4
        for (int c = warp; c < P; c += 32) s += partial[static_cast<size_t>(c) * m + e];
    }
    sh[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && e < m) {
        double t = sh[0][lane];
#pragma unroll
        for (int w = 1; w < 32; ++w) t += sh[w][lane];
        out[e] = t;
    }
}

// column exponents f_c for the int8 panel digits: max |X_c| 2^-f_c < 1/4
// (one warp per column; max is exact in any order)
__global__ void __launch_bounds__(1024) k_colexp_final(const double* __restrict__ pmax, int P,
                                                       int wp, int nb, int* __restrict__ col_exp) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = warp; c < nb; c += blockDim.x >> 5) {
        double m = 0.0;
        if (c < wp)
    #pragma unroll 8
            for (int b = lane; b < P; b += 32) m = fmax(m, pmax[static_cast<size_t>(b) * wp + c]);
        m = warp_max(m);
        if (lane == 0) {
            int f = -1100;
            if (m > 0.0) {
                int e;
                frexp(m, &e);  // m < 2^e
                f = e + 2;
            }
            col_exp[c] = f;
        }
    }
}

// A^T B partials with the f64 MMA: warp w owns output 8x8 tiles t = w, w+8, ..
// (t -> (ta, tb) = (t / NF, t % NF)) and walks all k4 row blocks of the CTA.
// Fragments come straight from the interleaved layout: the A operand
// (A^T)[a][i] of a tile and the B operand B[i][b] are both 32 consecutive
// doubles.
template <int WP>
__global__ void __launch_bounds__(256) k_panel_dot_partial(const double* __restrict__ a,
                                                           const double* __restrict__ b,
                                                           size_t n_pad,
                                                           double* __restrict__ partial,
                                                           const int* __restrict__ gate) {
    if (gate && !(gate[0] & 1)) return;
    constexpr int NF = WP / 8;
    constexpr int NT = NF * NF;
    constexpr int TPW = (NT + 7) / 8;  // tiles per warp
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t nq = n_pad / 4;
    const size_t q0 = nq * blockIdx.x / gridDim.x, q1 = nq * (blockIdx.x + 1) / gridDim.x;
    double acc[TPW][2];
#pragma unroll
    for (int j = 0; j < TPW; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (size_t q = q0; q < q1; ++q) {
        const double* ab = a + q * WP * 4;
        const double* bb = b + q * WP * 4;
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
            const int t = warp + 8 * j;
            if (t < NT) {
                const int ta = t / NF, tb = t % NF;
                const double av = ab[(8 * ta) * 4 + lane];
                const double bv = bb[(8 * tb) * 4 + lane];
                dmma884(acc[j][0], acc[j][1], av, bv);
            }
        }
    }
    double* out = partial + static_cast<size_t>(blockIdx.x) * WP * WP;
    const int rq = lane >> 2, kq = lane & 3;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
        const int t = warp + 8 * j;
        if (t < NT) {
            const int ta = t / NF, tb = t % NF;
            out[(8 * ta + rq) * WP + 8 * tb + 2 * kq] = acc[j][0];
            out[(8 * ta + rq) * WP + 8 * tb + 2 * kq + 1] = acc[j][1];
        }
    }
}

// ---- K3 Cholesky of W (wp x wp) with breakdown handling ---------------------
// Pass with allow_shift: if some pivot falls below kShiftTrig times its
// column's squared norm (column condition ~1e5+), refactor W + sigma I with
// the shifted-CholeskyQR shift sigma = 11 (n w + w (w+1)) u tr(W)
// (Fukaya et al. 2020); then only all-zero columns are dropped.
// Pass without shift: a column whose pivot is <= kDropTol * max diag (or
// not positive) is numerically dependent and is dropped: its row and column
// of R^{-1} are zeroed, so the orthonormalized panel gets a zero column there.
constexpr double kShiftTrig = 1e-10;
constexpr double kDropTol = 1e-20;

__global__ void __launch_bounds__(128) k_chol_inv(const double* __restrict__ wmat, int wp, int w,
                                                  double nrows, int allow_shift,
                                                  double* __restrict__ rinv,
                                                  int* __restrict__ flags) {
    extern __shared__ double sm[];
    const int ld = wp + 1;
    double* A = sm;               // [wp][ld] working matrix, becomes R (upper)
    double* diag0 = A + wp * ld;  // [wp]
    __shared__ int dropped[kMaxWP];
    __shared__ int need_shift;
    __shared__ double sigma_s;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int e = tid; e < wp; e += nt) diag0[e] = e < w ? wmat[e * wp + e] : 0.0;
    __syncthreads();
    double trace = 0.0, maxdiag = 0.0;
    for (int j = 0; j < w; ++j) {
        trace += diag0[j];
        maxdiag = fmax(maxdiag, diag0[j]);
    }
    double sigma = 0.0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (int e = tid; e < wp * wp; e += nt) {
            const int i = e / wp, j = e % wp;
            double v = (i < w && j < w) ? wmat[i * wp + j] : 0.0;
            if (i == j && i < w && diag0[i] > 0.0) v += sigma;
            A[i * ld + j] = v;
        }
        for (int e = tid; e < wp; e += nt) dropped[e] = 0;
        if (tid == 0) need_shift = 0;
        __syncthreads();
        for (int j = 0; j < wp; ++j) {
            if (tid == 0) {
                const double p = A[j * ld + j];
                int drop = 0;
                if (j >= w || diag0[j] <= 0.0 || !(p > 0.0)) {
                    drop = 1;
                } else if (allow_shift && attempt == 0 && p <= kShiftTrig * diag0[j]) {
                    need_shift = 1;
                } else if (!allow_shift && p <= kDropTol * maxdiag) {
                    drop = 1;
                }
                if (allow_shift && attempt == 0 && drop && j < w && diag0[j] > 0.0) {
                    need_shift = 1;  // non-positive pivot on a nonzero column: shift instead
                    drop = 0;
                }
                dropped[j] = drop;
                sigma_s = drop ? 1.0 : sqrt(fmax(p, 0.0));
                A[j * ld + j] = sigma_s;
            }
            __syncthreads();
            if (need_shift) break;
            const double rjj = sigma_s;
            const int dj = dropped[j];
            for (int k = j + 1 + tid; k < wp; k += nt) A[j * ld + k] = dj ? 0.0 : A[j * ld + k] / rjj;
            __syncthreads();
            const int m = wp - j - 1;
            for (int e = tid; e < m * m; e += nt) {
                const int k = j + 1 + e / m, l = j + 1 + e % m;
                if (l >= k) A[k * ld + l] -= A[j * ld + k] * A[j * ld + l];
            }
            __syncthreads();
        }
        if (!need_shift) break;
        sigma = 11.0 * (nrows * w + static_cast<double>(w) * (w + 1)) * 0x1.0p-53 * trace;
        if (tid == 0) flags[0] |= 1;
        __syncthreads();
    }
    // in-place inverse of the upper-triangular R held in A (column by column,
    // LAPACK trti2 order): T = R^{-1} on columns 0..j-1 is used to form column j
    __shared__ double inv_jj;
    for (int j = 0; j < wp; ++j) {
        if (tid == 0) inv_jj = 1.0 / A[j * ld + j];
        double t = 0.0;
        const int i = tid;
        if (i < j) {
            for (int k = i; k < j; ++k) t += A[i * ld + k] * A[k * ld + j];
        }
        __syncthreads();
        if (i < j) A[i * ld + j] = -t * inv_jj;
        if (tid == 0) A[j * ld + j] = inv_jj;
        __syncthreads();
    }
    for (int e = tid; e < wp * wp; e += nt) {
        const int i = e / wp, j = e % wp;
        rinv[e] = (i > j || dropped[i] || dropped[j]) ? 0.0 : A[i * ld + j];
    }
}

// q = y * rinv, rinv upper triangular (wp x wp). CTA stages rinv in smem and
// walks k4 row blocks; thread (block, column) computes 4 rows.
template <int WP>
__global__ void __launch_bounds__(256) k_panel_apply(const double* __restrict__ y,
                                                     const double* __restrict__ rinv,
                                                     size_t n_pad, double* __restrict__ q,
                                                     const int* __restrict__ gate) {
    const size_t nq = n_pad / 4;
    if (gate && !(gate[0] & 1)) {
        // gated-off pass: the panel passes through unchanged
        for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < nq * WP;
             e += static_cast<size_t>(gridDim.x) * blockDim.x)
            reinterpret_cast<double4*>(q)[e] = reinterpret_cast<const double4*>(y)[e];
        return;
    }
    extern __shared__ double R[];  // [WP * WP]
    for (int e = threadIdx.x; e < WP * WP; e += blockDim.x) R[e] = rinv[e];
    __syncthreads();
    for (size_t item = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
         item < nq * WP; item += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t qb = item / WP;
        const int c = static_cast<int>(item % WP);
        const double* yb = y + qb * WP * 4;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        for (int k = 0; k <= c; ++k) {
            const double r = R[k * WP + c];
            const double4 v = *reinterpret_cast<const double4*>(yb + k * 4);
            s0 += v.x * r;
            s1 += v.y * r;
            s2 += v.z * r;
            s3 += v.w * r;
        }
        double4 o;
        o.x = s0;
        o.y = s1;
        o.z = s2;
        o.w = s3;
        *reinterpret_cast<double4*>(q + qb * WP * 4 + c * 4) = o;
    }
}

template <int WP>
void panel_dot_wp(const double* a, const double* b, size_t n_pad, double* partial, int P,
                  cudaStream_t st, const int* gate) {
    k_panel_dot_partial<WP><<<P, 256, 0, st>>>(a, b, n_pad, partial, gate);
}

template <int WP>
void panel_apply_wp(const double* y, const double* rinv, size_t n_pad, double* q, int grid,
                    cudaStream_t st, const int* gate) {
    constexpr size_t smem = static_cast<size_t>(WP) * WP * sizeof(double);
    allow_dyn_smem(reinterpret_cast<const void*>(k_panel_apply<WP>));
    k_panel_apply<WP><<<grid, 256, smem, st>>>(y, rinv, n_pad, q, gate);
}


// ---- stable_rank power iteration step (ref rsvd.cpp:160-176) --------------
// partial[b] = sum of y(i,0)^2 over CTA b's rows (fixed order)
__global__ void __launch_bounds__(256) k_sr_norm_partial(const double* __restrict__ y, size_t n,
                                                         int wp, const SrState* __restrict__ st,
                                                         double* __restrict__ partial) {
    if (st->done) return;
    __shared__ double red[8];
    const size_t i0 = n * blockIdx.x / gridDim.x, i1 = n * (blockIdx.x + 1) / gridDim.x;
    double s = 0.0;
    for (size_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double v = y[pidx(i, 0, wp)];
        s += v * v;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        partial[blockIdx.x] = t;
    }
}

// one thread: norm, restart flag, convergence (same tests as the reference)
__global__ void k_sr_update(const double* __restrict__ partial, int P, SrState* __restrict__ st) {
    if (st->done) {
        st->active = 0;
        return;
    }
    double ss = 0.0;
    for (int b = 0; b < P; ++b) ss += partial[b];
    const double norm = sqrt(ss);
    st->active = 1;
    st->iters += 1;
    st->norm = norm;
    if (norm == 0.0) {  // start vector in the kernel: the host redraws it
        st->zero = 1;
        st->done = 1;
        return;
    }
    if (st->sigma != 0.0 && fabs(norm - st->sigma) <= 1e-13 * norm) st->done = 1;
    st->sigma = norm;
}

// v = w / norm (column 0; the other panel columns stay zero)
__global__ void __launch_bounds__(256) k_sr_scale(const double* __restrict__ y, size_t n, int wp,
                                                  const SrState* __restrict__ st,
                                                  double* __restrict__ x) {
    if (!st->active || st->zero) return;
    const double norm = st->norm;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        x[pidx(i, 0, wp)] = y[pidx(i, 0, wp)] / norm;
}

// one warp per output: e < 2 wp sums (s, then t), e >= 2 wp the column
// exponents from the maxima; lanes stride over the P CTA statistics in a
// fixed order, xor-tree combine => deterministic
__global__ void __launch_bounds__(256) k_colstats_final(const double* __restrict__ cstat, int P,
                                                        int wp, int nb, double* __restrict__ colsums,
                                                        int* __restrict__ col_exp) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nsum = 2 * wp;
    if (gw < nsum) {
        double v = 0.0;
        for (int b = lane; b < P; b += 32) v += cstat[static_cast<size_t>(b) * 3 * wp + gw];
        v = warp_sum(v);
        if (lane == 0) colsums[gw] = v;
    } else if (col_exp && gw < nsum + nb) {
        const int c = gw - nsum;
        double m = 0.0;
        if (c < wp)
            for (int b = lane; b < P; b += 32)
                m = fmax(m, cstat[static_cast<size_t>(b) * 3 * wp + 2 * wp + c]);
        m = warp_max(m);
        if (lane == 0) {
            int f = -1100;
            if (m > 0.0) {
                int e;
                frexp(m, &e);  // m < 2^e
                f = e + 2;
            }
            col_exp[c] = f;
        }
    }
}

}  // namespace

int panel_grid(size_t n_pad, int sms) {
    const size_t nq = n_pad / 4;
    const size_t g = std::min<size_t>(static_cast<size_t>(sms) * 2, std::max<size_t>(nq / 8, 1));
    return static_cast<int>(g);
}

void launch_panel_from_rowmajor(const double* src, size_t n, int w, int wp, size_t n_pad,
                                double* dst, cudaStream_t st) {
    const size_t total = n_pad * wp;
    const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 4096));
    k_panel_from_rowmajor<<<grid, 256, 0, st>>>(src, n, w, wp, n_pad, dst);
    count_launch();
}

void launch_panel_to_rowmajor(const double* src, size_t n, int w, int wp, double* dst,
                              cudaStream_t st) {
    const size_t total = n * w;
    const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256 + 1, 4096));
    k_panel_to_rowmajor<<<grid, 256, 0, st>>>(src, n, w, wp, dst);
    count_launch();
}

void launch_colsums(const double* x, const double* row_mean, size_t n, size_t n_pad, int wp,
                    double* partial, double* colsums, int sms, cudaStream_t st, double* pmax,
                    int nb, int* col_exp) {
    const int P = panel_grid(n_pad, sms);
    k_colsum_partial<<<P, 256, 3 * wp * 4 * sizeof(double), st>>>(x, row_mean, n, n_pad, wp,
                                                                  partial, pmax);
    k_sum_partials<<<(2 * wp + 31) / 32, 1024, 0, st>>>(partial, P, 2 * wp, colsums);
    count_launch(2);
    if (pmax && col_exp) {
        k_colexp_final<<<1, 1024, 0, st>>>(pmax, P, wp, nb, col_exp);
        count_launch(1);
    }
}

// column maxima of the colsum partials' pmax (P x wp) -> cmax (wp)
__global__ void __launch_bounds__(256) k_colmax_final(const double* __restrict__ pmax, int P,
                                                      int wp, double* __restrict__ cmax) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < wp; c += gridDim.x * blockDim.x) {
        double m = 0.0;
        for (int b = 0; b < P; ++b) m = fmax(m, pmax[static_cast<size_t>(b) * wp + c]);
        cmax[c] = m;
    }
}

void launch_colmax(const double* pmax, int P, int wp, double* cmax, cudaStream_t st) {
    k_colmax_final<<<1, 256, 0, st>>>(pmax, P, wp, cmax);
    count_launch();
}

void launch_colexp(const double* cmax, int wp, int nb, int* col_exp, cudaStream_t st) {
    k_colexp_final<<<1, 1024, 0, st>>>(cmax, 1, wp, nb, col_exp);
    count_launch();
}

void launch_panel_dot(const double* a, const double* b, size_t n_pad, int wp, double* partial,
                      double* out, int sms, cudaStream_t st, const int* gate) {
    const int P = panel_grid(n_pad, sms);
    switch (wp) {
#define DSB_WP(W)                                         \
    case W:                                               \
        panel_dot_wp<W>(a, b, n_pad, partial, P, st, gate); \
        break;
        DSB_WP(8) DSB_WP(16) DSB_WP(24) DSB_WP(32) DSB_WP(40) DSB_WP(48) DSB_WP(56) DSB_WP(64)
        DSB_WP(72) DSB_WP(80) DSB_WP(88) DSB_WP(96) DSB_WP(104) DSB_WP(112) DSB_WP(120)
        DSB_WP(128)
#undef DSB_WP
        default:
            throw std::invalid_argument("unsupported panel width");
    }
    k_sum_partials<<<(wp * wp + 31) / 32, 1024, 0, st>>>(partial, P, wp * wp, out, gate);
    count_launch(2);
}

void launch_chol_inv(const double* w_mat, int wp, int w, size_t n, int allow_shift, double* rinv,
                     int* flags, cudaStream_t st) {
    const size_t smem = (static_cast<size_t>(wp) * (wp + 1) + wp) * sizeof(double);
    allow_dyn_smem(reinterpret_cast<const void*>(k_chol_inv));
    k_chol_inv<<<1, 128, smem, st>>>(w_mat, wp, w, static_cast<double>(n), allow_shift, rinv,
                                     flags);
    count_launch();
}

void launch_panel_apply(const double* y, const double* rinv, size_t n_pad, int wp, double* q,
                        cudaStream_t st, const int* gate) {
    const size_t items = n_pad / 4 * wp;
    const int grid = static_cast<int>(std::min<size_t>((items + 255) / 256, 148 * 8));
    switch (wp) {
#define DSB_WP(W)                                               \
    case W:                                                     \
        panel_apply_wp<W>(y, rinv, n_pad, q, grid, st, gate);   \
        break;
        DSB_WP(8) DSB_WP(16) DSB_WP(24) DSB_WP(32) DSB_WP(40) DSB_WP(48) DSB_WP(56) DSB_WP(64)
        DSB_WP(72) DSB_WP(80) DSB_WP(88) DSB_WP(96) DSB_WP(104) DSB_WP(112) DSB_WP(120)
        DSB_WP(128)
#undef DSB_WP
        default:
            throw std::invalid_argument("unsupported panel width");
    }
    count_launch();
}

}  // namespace dsb

namespace dsb {
void launch_sr_step(const double* y, size_t n, int wp, double* partial, SrState* state, double* x,
                    int sms, cudaStream_t st) {
    const int P = sms;
    k_sr_norm_partial<<<P, 256, 0, st>>>(y, n, wp, state, partial);
    k_sr_update<<<1, 1, 0, st>>>(partial, P, state);
    k_sr_scale<<<sms, 256, 0, st>>>(y, n, wp, state, x);
    count_launch(3);
}
}  // namespace dsb

namespace dsb {
// out[0] = sum of count doubles, fixed order (deterministic)
void launch_sum_fixed(const double* partial, size_t count, double* out, cudaStream_t st) {
    k_sum_partials<<<1, 1024, 0, st>>>(partial, static_cast<int>(count), 1, out);
    count_launch(1);
}
}  // namespace dsb

namespace dsb {
void launch_colstats_final(const double* cstat, int P, int wp, int nb, double* colsums,
                           int* col_exp, cudaStream_t st) {
    const int warps = 2 * wp + (col_exp ? nb : 0);
    k_colstats_final<<<(warps * 32 + 255) / 256, 256, 0, st>>>(cstat, P, wp, nb, colsums, col_exp);
    count_launch(1);
}
}  // namespace dsb
