// K3 fast path (panel width WP <= 64): the whole CholeskyQR2/3 of one
// orthonormalization in ONE cooperative launch (replaces thin_orthonormal,
// ref src/rsvd.cpp:38-44).
//
// Per pass (pass 0 may shift; a third pass only when it did):
//   1. each CTA forms the partial Gram Y_c^T Y_c of its contiguous row range
//      (resident in shared memory) on the f64 tensor cores;
//   2. grid sync; fixed-order reduction of the partials (warp per element);
//      grid sync;
//   3. every CTA factors W = L D L^T redundantly (identical inputs and code =>
//      identical factors), carrying E = L^{-1} along the elimination, with
//      the shift / drop rules of launch_chol_inv; T = L^{-T} D^{-1/2};
//   4. Q = Y T on the f64 tensor cores, in place, right to left.
// Rows never leave their CTA between passes, so a pass needs only the two
// grid syncs around the Gram reduction. The same single-CTA elimination is
// exported for the multi-kernel (sharded) path: launch_chol_inv_elim.
#include <cooperative_groups.h>

#include <algorithm>
#include <stdexcept>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace dsb {

namespace {

constexpr double kShiftTrigF = 1e-10;  // same rules as k_chol_inv
long long* g_orth_prof = nullptr;      // debug: per-phase cycle counts of CTA 0
constexpr double kDropTolF = 1e-20;
#ifndef DSB_ORTH_FAST_RCP
#define DSB_ORTH_FAST_RCP 1
#endif

// CTA-wide elimination W = L D L^T (A in shared memory, upper triangle used)
// that also carries E = L^{-1} along (Gauss-Jordan style, same steps), so the
// inverse Cholesky factor T = R^{-1} = L^{-T} D^{-1/2} comes out without a
// second sequential sweep; the apply Q = Y T is then a small GEMM.
// Step k: thread 0 takes the pivot decision (shift / drop rules of
// k_chol_inv); one barrier; the trailing update of A and the new column
// entries of E are spread over the CTA; one barrier.
// Returns true when the first (shift-allowed) attempt asks for a shift.
template <int WP>
__device__ bool cta_chol_inverse(double* __restrict__ A, double* __restrict__ E, int w,
                                 const double* __restrict__ d0s, double maxdiag,
                                 bool first_shifting, bool drop_mode, int* __restrict__ dropped_s,
                                 double* __restrict__ dpiv, const unsigned short* __restrict__ tri,
                                 const int* __restrict__ tri_off) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < WP * WP; e += nt) E[e] = (e / WP == e % WP) ? 1.0 : 0.0;
    __syncthreads();
    for (int k = 0; k < WP; ++k) {
        // every thread takes the (identical) pivot decision from the same
        // shared values: no barrier between the decision and the update
        const double p = A[k * WP + k];
        const double d0k = d0s[k];
        bool drop = (k >= w) || !(d0k > 0.0) || !(p > 0.0);
        bool shift = false;
        if (first_shifting) {
            if (k < w && d0k > 0.0 && (drop || p <= kShiftTrigF * d0k)) shift = true;
            drop = drop && !(k < w && d0k > 0.0);
        } else if (drop_mode && p <= kDropTolF * maxdiag) {
            drop = true;
        }
        if (shift) {  // uniform across the CTA; the caller rewrites A next
            __syncthreads();
            return true;
        }
        if (tid == 0) {
            dropped_s[k] = drop;
            dpiv[k] = drop ? 0.0 : p;
        }
        // 0 for a dropped column: no elimination with it. The reciprocal is
        // the MUFU seed + two Newton steps (<= 1 ulp): the IEEE division's
        // slow-path check sits on this loop's critical path
        double invp = 0.0;
        if (!drop) {
#if DSB_ORTH_FAST_RCP
            double r;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
            r = fma(r, fma(-p, r, 1.0), r);
            invp = fma(r, fma(-p, r, 1.0), r);
#else
            invp = 1.0 / p;
#endif
        }
        const double* rowk = A + k * WP;
        // trailing upper triangle {(i, j): k < i <= j}: a suffix of `tri`
        const int t0 = tri_off[k + 1], t1 = tri_off[WP];
        for (int t = t0 + tid; t < t1; t += nt) {
            const int i = tri[t] >> 8, j = tri[t] & 0xff;
            A[i * WP + j] -= rowk[i] * rowk[j] * invp;
        }
        // E rows i > k, columns c <= k: E[i][c] -= l_ik E[k][c], l_ik = a_ki / d_k
        const int cols = k + 1, nrow = WP - k - 1;
        for (int e = tid; e < nrow * cols; e += nt) {
            const int i = k + 1 + e / cols, cc = e % cols;
            E[i * WP + cc] -= rowk[i] * invp * E[k * WP + cc];
        }
        __syncthreads();
    }
    return false;
}

// The same elimination blocked by 4 pivots (right-looking LDL^T): warp 0
// factors the block's 4 pivot rows in order (the per-pivot shift / drop
// decisions and updates of k_chol_inv, restricted to the block's rows and
// their E rows, with __syncwarp between pivots), then the whole CTA applies
// the 4 pivots to the trailing rows of A and E as one rank-4 update (one
// barrier) — 8 CTA barriers instead of 32 per 32 x 32 factor. Every entry
// receives the same updates with the same pivot-row values as in the
// one-pivot-at-a-time order (the panel rows are final before the trailing
// update reads them); only the order of independent writes changes.
template <int WP>
__device__ bool cta_chol_inverse_b4(double* __restrict__ A, double* __restrict__ E, int w,
                                    const double* __restrict__ d0s, double maxdiag,
                                    bool first_shifting, bool drop_mode, int* __restrict__ dropped_s,
                                    double* __restrict__ dpiv, const unsigned short* __restrict__ tri,
                                    const int* __restrict__ tri_off) {
    __shared__ double invs[4];
    __shared__ int shift_req;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < WP * WP; e += nt) E[e] = (e / WP == e % WP) ? 1.0 : 0.0;
    if (tid == 0) shift_req = 0;
    __syncthreads();
    for (int k0 = 0; k0 < WP; k0 += 4) {
        if (tid < 32) {
            const int lane = tid;
            for (int kk = k0; kk < k0 + 4; ++kk) {
                const double p = A[kk * WP + kk];
                const double d0k = d0s[kk];
                bool drop = (kk >= w) || !(d0k > 0.0) || !(p > 0.0);
                bool shift = false;
                if (first_shifting) {
                    if (kk < w && d0k > 0.0 && (drop || p <= kShiftTrigF * d0k)) shift = true;
                    drop = drop && !(kk < w && d0k > 0.0);
                } else if (drop_mode && p <= kDropTolF * maxdiag) {
                    drop = true;
                }
                if (shift) {  // warp-uniform
                    if (lane == 0) shift_req = 1;
                    break;
                }
                double invp = 0.0;
                if (!drop) {
                    double r;
                    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
                    r = fma(r, fma(-p, r, 1.0), r);
                    invp = fma(r, fma(-p, r, 1.0), r);
                }
                if (lane == 0) {
                    dropped_s[kk] = drop;
                    dpiv[kk] = drop ? 0.0 : p;
                    invs[kk - k0] = invp;
                }
                const double* rowk = A + kk * WP;
                // the block's later pivot rows (at most 3), every column
                // j >= i, and their E rows: all multipliers and row-k values
                // are read first, then the (independent) row updates run side
                // by side instead of one row after another
                double f[3];
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const int i = kk + 1 + t;
                    f[t] = i < k0 + 4 ? rowk[i] * invp : 0.0;
                }
                for (int jj = lane; jj < WP; jj += 32) {
                    const double rj = rowk[jj];
#pragma unroll
                    for (int t = 0; t < 3; ++t) {
                        const int i = kk + 1 + t;
                        if (i < k0 + 4 && jj >= i) A[i * WP + jj] -= f[t] * rj;
                    }
                }
                for (int c = lane; c <= kk; c += 32) {
                    const double ek = E[kk * WP + c];
#pragma unroll
                    for (int t = 0; t < 3; ++t) {
                        const int i = kk + 1 + t;
                        if (i < k0 + 4) E[i * WP + c] -= f[t] * ek;
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (shift_req) return true;  // uniform: the caller rewrites A next
        // trailing rows i >= k0 + 4 of A (upper part) and of E: rank-4 update
        const double i0 = invs[0], i1 = invs[1], i2 = invs[2], i3 = invs[3];
        const double* r0 = A + k0 * WP;
        const double* r1 = r0 + WP;
        const double* r2 = r1 + WP;
        const double* r3 = r2 + WP;
        const int t0 = tri_off[k0 + 4], t1 = tri_off[WP];
        for (int t = t0 + tid; t < t1; t += nt) {
            const int i = tri[t] >> 8, j = tri[t] & 0xff;
            A[i * WP + j] -= ((r0[i] * i0) * r0[j] + (r1[i] * i1) * r1[j]) +
                             ((r2[i] * i2) * r2[j] + (r3[i] * i3) * r3[j]);
        }
        const int ncol = k0 + 4, nrow = WP - k0 - 4;
        for (int e = tid; e < nrow * ncol; e += nt) {
            const int i = k0 + 4 + e / ncol, cc = e % ncol;
            E[i * WP + cc] -= ((r0[i] * i0) * E[k0 * WP + cc] + (r1[i] * i1) * E[(k0 + 1) * WP + cc]) +
                              ((r2[i] * i2) * E[(k0 + 2) * WP + cc] +
                               (r3[i] * i3) * E[(k0 + 3) * WP + cc]);
        }
        __syncthreads();
    }
    return false;
}

#ifndef DSB_ORTH_BLOCKED
#define DSB_ORTH_BLOCKED 1
#endif
template <int WP>
__device__ __forceinline__ bool chol_inverse(double* __restrict__ A, double* __restrict__ E, int w,
                                             const double* __restrict__ d0s, double maxdiag,
                                             bool first_shifting, bool drop_mode,
                                             int* __restrict__ dropped_s, double* __restrict__ dpiv,
                                             const unsigned short* __restrict__ tri,
                                             const int* __restrict__ tri_off) {
    if constexpr (DSB_ORTH_BLOCKED != 0)
        return cta_chol_inverse_b4<WP>(A, E, w, d0s, maxdiag, first_shifting, drop_mode,
                                       dropped_s, dpiv, tri, tri_off);
    else
        return cta_chol_inverse<WP>(A, E, w, d0s, maxdiag, first_shifting, drop_mode, dropped_s,
                                    dpiv, tri, tri_off);
}

// WP <= 32: the factor on ONE warp, the matrix in registers (lane j holds
// column j's upper part A[0..j][j]); step k broadcasts the pivot and, lane
// by lane, row k (A[k][i] from lane i's register k), and every lane applies
// the same update as cta_chol_inverse — A[i][j] -= A[k][i] A[k][j] / p —
// with the same shift / drop decisions. No barriers, no shared-memory
// round trips on the pivot chain (the CTA elimination spends ~800 cycles per
// pivot on them). Writes L (Lm[j][k] = A[k][j] / p_k below the diagonal,
// zero for a dropped pivot), dpiv and dropped_s; the caller applies
// Q = Y L^-T D^-1/2 by forward substitution, so no inverse is formed.
// Returns true when the first (shift-allowed) attempt asks for a shift.
#ifndef DSB_ORTH_WARP_LDL
#define DSB_ORTH_WARP_LDL 1
#endif
template <int WP>
__device__ bool warp_ldl(const double* __restrict__ A, double* __restrict__ Lm, int w,
                         const double* __restrict__ d0s, double maxdiag, bool first_shifting,
                         bool drop_mode, int* __restrict__ dropped_s,
                         double* __restrict__ dpiv) {
    static_assert(WP <= 32, "one row per lane");
    const int lane = threadIdx.x & 31;
    constexpr unsigned FULL = 0xffffffffu;
    double a[WP];
#pragma unroll
    for (int i = 0; i < WP; ++i) a[i] = (lane < WP && i <= lane) ? A[i * WP + lane] : 0.0;
#pragma unroll
    for (int k = 0; k < WP; ++k) {
        const double p = __shfl_sync(FULL, a[k], k);
        const double d0k = d0s[k];
        bool drop = (k >= w) || !(d0k > 0.0) || !(p > 0.0);
        bool shift = false;
        if (first_shifting) {
            if (k < w && d0k > 0.0 && (drop || p <= kShiftTrigF * d0k)) shift = true;
            drop = drop && !(k < w && d0k > 0.0);
        } else if (drop_mode && p <= kDropTolF * maxdiag) {
            drop = true;
        }
        if (shift) return true;  // uniform
        if (lane == 0) {
            dropped_s[k] = drop;
            dpiv[k] = drop ? 0.0 : p;
        }
        double invp = 0.0;
        if (!drop) {
            double r;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
            r = fma(r, fma(-p, r, 1.0), r);
            invp = fma(r, fma(-p, r, 1.0), r);
        }
        const double akj = a[k];  // A[k][j] of this lane's column j
        // (fixed trip counts: the inner loops unroll before the outer one,
        // so every register index stays static)
#pragma unroll
        for (int i = 0; i < WP; ++i) {
            if (i > k) {
                const double aki = __shfl_sync(FULL, a[k], i);  // A[k][i] from lane i
                if (lane >= i) a[i] -= aki * akj * invp;
            }
        }
        // L[j][k] (lanes j > k), once every lane has read A[k][j]
        if (lane > k) a[k] = akj * invp;
    }
    if (lane < WP) {
#pragma unroll
        for (int k = 0; k < WP; ++k) Lm[lane * WP + k] = k < lane ? a[k] : 0.0;
    }
    return false;
}

template <int WP>
__global__ void __launch_bounds__(256, 1)
    k_orth_fused(const double* __restrict__ y, double* __restrict__ out, size_t n_pad, int w,
                 double nrows, int ldr, double* __restrict__ partial, double* __restrict__ wsum,
                 int* __restrict__ flags, long long* __restrict__ prof,
                 const double* __restrict__ row_mean, double* __restrict__ cstat) {
    long long t_last = clock64();
    int prof_i = 0;
    auto mark = [&]() {
        if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
            const long long t = clock64();
            prof[prof_i] = t - t_last;
            t_last = t;
        }
        ++prof_i;
    };
    constexpr int NF = WP / 8;
    constexpr int NT = NF * NF;
    constexpr int TPW = (NT + 7) / 8;
    cg::grid_group grid = cg::this_grid();
    __shared__ int dropped_s[WP];
    __shared__ double d0s[WP];
    __shared__ double dpiv[WP];
    __shared__ double tr_s[2];
    __shared__ unsigned short tri[WP * (WP + 1) / 2];
    __shared__ int tri_off[WP + 1];
    __shared__ int skip_third;
    __shared__ int shift_flag;
    // the warp factor + forward-substitution apply up to WP = 24 (C1, w = 20:
    // factor 18.5k -> 12.1k cycles per pass); at WP = 32 the fully unrolled
    // code (255 registers, ~1k shuffles) lost to the CTA elimination
    // (factor 32k / 17k vs 26k / 26k cycles, apply 21k / 8.5k vs 9.4k / 9.0k)
    constexpr bool kWarpLdl = DSB_ORTH_WARP_LDL != 0 && WP <= 24;
    // the CTA's rows stay in shared memory for all passes, column-major with
    // leading dimension ldr = 4 (mod 16): conflict-free MMA fragments and
    // conflict-free thread-per-row access
    extern __shared__ double ps[];  // [WP][ldr], then R [WP*WP], E [WP*WP]
    double* R = ps + static_cast<size_t>(WP) * ldr;  // W, eliminated in place; then T
    double* E = R + WP * WP;                         // L^{-1}
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = gridDim.x, c = blockIdx.x;
    const size_t nq = n_pad / 4;
    const size_t q0 = nq * c / P, q1 = nq * (c + 1) / P;
    const int nrow = static_cast<int>((q1 - q0) * 4);
    {
        // the CTA's rows (contiguous in the interleaved panel) into shared
        // memory, column-major: 8 independent loads in flight per thread
        // (a load-store loop serialized on the global latency, ~5 us)
        const double* src = y + q0 * WP * 4;
        const int ne = nrow * WP, nt = blockDim.x;
        for (int e0 = threadIdx.x; e0 < ne; e0 += 8 * nt) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * nt;
                v[u] = e < ne ? __ldg(src + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * nt;
                if (e < ne) {
                    const int qb = e / (WP * 4), cc = (e / 4) % WP, rr = e & 3;
                    ps[cc * ldr + 4 * qb + rr] = v[u];
                }
            }
        }
    }
    if (threadIdx.x == 0) {
        skip_third = 0;
        shift_flag = 0;
    }
    for (int i = threadIdx.x; i <= WP; i += blockDim.x) {  // upper-triangle list sorted by row
        const int off = i * WP - (i * (i - 1)) / 2;
        tri_off[i] = off;
        for (int j = i; j < WP && i < WP; ++j)
            tri[off + j - i] = static_cast<unsigned short>((i << 8) | j);
    }
    __syncthreads();
    mark();
    // pass 0 may shift; when it did not, CholQR2 suffices (same decision in
    // every CTA: identical factorization)
    for (int pass = 0; pass < 3; ++pass) {
        if (pass == 2 && skip_third) break;
        // ---- 1. partial Gram of this CTA's rows (f64 MMA from shared memory)
        {
            double acc[TPW][2];
#pragma unroll
            for (int j = 0; j < TPW; ++j) acc[j][0] = acc[j][1] = 0.0;
            const int rq = lane >> 2, kq = lane & 3;
            for (int q = 0; q < nrow / 4; ++q) {
#pragma unroll
                for (int j = 0; j < TPW; ++j) {
                    const int tt = warp + 8 * j;
                    if (tt < NT) {
                        const int ta = tt / NF, tb = tt % NF;
                        dmma884(acc[j][0], acc[j][1], ps[(8 * ta + rq) * ldr + 4 * q + kq],
                                ps[(8 * tb + rq) * ldr + 4 * q + kq]);
                    }
                }
            }
            double* o = partial + static_cast<size_t>(c) * WP * WP;
#pragma unroll
            for (int j = 0; j < TPW; ++j) {
                const int tt = warp + 8 * j;
                if (tt < NT) {
                    const int ta = tt / NF, tb = tt % NF;
                    o[(8 * ta + rq) * WP + 8 * tb + 2 * kq] = acc[j][0];
                    o[(8 * ta + rq) * WP + 8 * tb + 2 * kq + 1] = acc[j][1];
                }
            }
        }
        mark();
        grid.sync();
        mark();
        // ---- 2. W = sum of partials: one warp per element, lanes stride over
        // the P partials, fixed shuffle tree => deterministic
        {
            const int gw = (c * 256 + threadIdx.x) >> 5, nw = P * 8;
            for (int e = gw; e < WP * WP; e += nw) {
                double s = 0.0;
                for (int k = lane; k < P; k += 32) s += partial[static_cast<size_t>(k) * WP * WP + e];
                s = warp_sum(s);
                if (lane == 0) wsum[e] = s;
            }
        }
        mark();
        grid.sync();
        mark();
        // ---- 3. Cholesky of W, every CTA (identical inputs and code)
        {
            const int tid = threadIdx.x;
            if (tid < WP) d0s[tid] = tid < w ? wsum[tid * WP + tid] : 0.0;
            __syncthreads();
            if (tid == 0) {
                double tr = 0.0, mx = 0.0;
                for (int j = 0; j < w; ++j) {
                    tr += d0s[j];
                    mx = fmax(mx, d0s[j]);
                }
                tr_s[0] = tr;
                tr_s[1] = mx;
            }
            double sigma = 0.0;
            bool shifted = false;
            for (int attempt = 0; attempt < 2; ++attempt) {
                for (int e = tid; e < WP * WP; e += blockDim.x) {
                    const int i = e / WP, j = e % WP;
                    double v = (i < w && j < w) ? wsum[e] : 0.0;
                    if (i == j && i < w && d0s[i] > 0.0) v += sigma;
                    R[e] = v;
                }
                __syncthreads();
                const bool first_shifting = pass == 0 && attempt == 0;
                const bool drop_mode = pass != 0;
                if constexpr (kWarpLdl) {
                    // warp 0 factors into E (= L); the CTA waits for it
                    if (threadIdx.x < 32 &&
                        warp_ldl<WP>(R, E, w, d0s, tr_s[1], first_shifting, drop_mode, dropped_s,
                                     dpiv) &&
                        threadIdx.x == 0)
                        shift_flag = 1;
                    __syncthreads();
                    const bool sh = shift_flag != 0;
                    __syncthreads();
                    if (threadIdx.x == 0) shift_flag = 0;
                    if (!sh) break;
                } else if (!chol_inverse<WP>(R, E, w, d0s, tr_s[1], first_shifting, drop_mode,
                                             dropped_s, dpiv, tri, tri_off)) {
                    break;
                }
                sigma = 11.0 * (nrows * w + static_cast<double>(w) * (w + 1)) * 0x1.0p-53 * tr_s[0];
                shifted = true;
            }
            if (tid == 0) {
                if (shifted && c == 0) flags[0] |= 1;
                if (pass == 0) skip_third = shifted ? 0 : 1;
            }
        }
        __syncthreads();
        mark();
        if constexpr (kWarpLdl) {
            // ---- 4'. Q = Y L^-T D^-1/2 row by row: x L^T = y by forward
            // substitution (L from the warp factor, broadcast from shared
            // memory), x_k / sqrt(d_k); each thread owns whole rows
            for (int r = threadIdx.x; r < nrow; r += blockDim.x) {
                double x[WP];
#pragma unroll
                for (int k = 0; k < WP; ++k) x[k] = ps[k * ldr + r];
#pragma unroll
                for (int k = 1; k < WP; ++k) {
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int i = 0; i < WP; ++i) {
                        if (i < k) {
                            if (i & 1)
                                s1 = fma(E[k * WP + i], x[i], s1);
                            else
                                s0 = fma(E[k * WP + i], x[i], s0);
                        }
                    }
                    x[k] -= s0 + s1;
                }
#pragma unroll
                for (int k = 0; k < WP; ++k) {
                    const double dk = dpiv[k];
                    ps[k * ldr + r] = dk > 0.0 ? x[k] * rsqrt(dk) : 0.0;
                }
            }
            __syncthreads();
            mark();
            continue;
        }
        // ---- 4. T = R^{-1} = L^{-T} D^{-1/2} (into R), then Q = Y T for this
        // CTA's rows: outputs kept in registers until every thread has read
        // its inputs, then written back in place
        for (int e = threadIdx.x; e < WP * WP; e += blockDim.x) {
            const int i = e / WP, j = e % WP;
            const double dj = dpiv[j];
            R[e] = (i <= j && dj > 0.0) ? E[j * WP + i] * rsqrt(dj) : 0.0;
        }
        __syncthreads();
        {
            // Q = Y T on the f64 tensor cores, in place: column c of Q needs
            // columns k <= c of Y only (T upper triangular), so the 8-column
            // tiles are produced right to left — each tile's rows are computed
            // into registers, then written over Y's (no longer needed) columns.
            // Fragments come straight from shared memory (ps column-major,
            // ldr = 4 mod 16: conflict-free A fragments).
            constexpr int NFT = WP / 8;
            constexpr int kMaxRT = 16;  // row tiles per warp (rows per CTA <= 1024)
            const int ntm = (nrow + 7) / 8;
            const int rq = lane >> 2, kq = lane & 3;
            for (int tn = NFT - 1; tn >= 0; --tn) {
                double acc[kMaxRT][2];
#pragma unroll
                for (int j = 0; j < kMaxRT; ++j) {
                    acc[j][0] = acc[j][1] = 0.0;
                    const int tm = warp + 8 * j;
                    if (tm < ntm) {
                        for (int kk = 0; kk < 2 * tn + 2; ++kk) {  // k <= 8 tn + 7
                            const double av = ps[(4 * kk + kq) * ldr + 8 * tm + rq];
                            const double bv = R[(4 * kk + kq) * WP + 8 * tn + rq];
                            dmma884(acc[j][0], acc[j][1], av, bv);
                        }
                    }
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kMaxRT; ++j) {
                    const int tm = warp + 8 * j;
                    const int row = 8 * tm + rq, col = 8 * tn + 2 * kq;
                    if (tm < ntm && row < nrow) {
                        ps[col * ldr + row] = acc[j][0];
                        ps[(col + 1) * ldr + row] = acc[j][1];
                    }
                }
                __syncthreads();
            }
        }
        __syncthreads();
        mark();
    }
    {
        double* dst = out + q0 * WP * 4;
        for (int e = threadIdx.x; e < nrow * WP; e += blockDim.x) {
            const int qb = e / (WP * 4), cc = (e / 4) % WP, rr = e & 3;
            dst[e] = ps[cc * ldr + 4 * qb + rr];
        }
    }
    if (cstat) {
        // the next product pass's column statistics of this CTA's rows:
        // 1^T Q, r^T Q (centering) and max |Q| (int8 column exponents).
        // Thread (slice, column): rows slice, slice + S, ...; the S slice
        // partials are combined in slice order (fixed) in shared memory
        // (reusing the Gram scratch R, free after the last pass).
        // S slices per column, bounded by the threads and by the 2 WP^2
        // doubles of R and E that hold the [3][S][WP] partials
        constexpr int S = (256 / WP < (2 * WP) / 3) ? 256 / WP : (2 * WP) / 3;
        const size_t i0 = q0 * 4;
        double* red = R;
        const int cc = threadIdx.x % WP, sl = threadIdx.x / WP;
        static_assert(3 * S * WP <= 2 * WP * WP && S >= 1, "partials fit in R and E");
        if (sl < S) {
            double sv = 0.0, tv = 0.0, mv = 0.0;
            for (int r = sl; r < nrow; r += S) {
                const double v = ps[cc * ldr + r];
                sv += v;
                if (row_mean && i0 + r < static_cast<size_t>(nrows)) tv += row_mean[i0 + r] * v;
                mv = fmax(mv, fabs(v));
            }
            red[(0 * S + sl) * WP + cc] = sv;
            red[(1 * S + sl) * WP + cc] = tv;
            red[(2 * S + sl) * WP + cc] = mv;
        }
        __syncthreads();
        if (threadIdx.x < WP) {
            double sv = 0.0, tv = 0.0, mv = 0.0;
            for (int k = 0; k < S; ++k) {
                sv += red[(0 * S + k) * WP + cc];
                tv += red[(1 * S + k) * WP + cc];
                mv = fmax(mv, red[(2 * S + k) * WP + cc]);
            }
            double* o = cstat + static_cast<size_t>(c) * 3 * WP;
            o[cc] = sv;
            o[WP + cc] = tv;
            o[2 * WP + cc] = mv;
        }
    }
}

template <int WP>
bool launch_wp(double* y, double* out, size_t n_pad, int w, size_t n, double* partial,
               double* wsum, int* flags, int sms, cudaStream_t st, const double* row_mean,
               double* cstat) {
    const int P = std::min<int>(sms, static_cast<int>(std::max<size_t>(n_pad / 4 / 8, 1)));
    const size_t nq = n_pad / 4;
    const int rows_max = static_cast<int>(((nq + P - 1) / P) * 4);
    const int ldr = (rows_max + 15) / 16 * 16 + 4;
    const size_t smem = (static_cast<size_t>(WP) * ldr + 2 * WP * WP) * sizeof(double);
    // DMMA apply: ceil(rows / 8) row tiles over 8 warps, <= 16 per warp
    if (smem > 220 * 1024 || (rows_max + 7) / 8 > 8 * 16) return false;
    allow_dyn_smem(reinterpret_cast<const void*>(k_orth_fused<WP>));
    static size_t occ_smem = 0;
    static int per_sm = 0;
    if (occ_smem != smem) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_orth_fused<WP>, 256, smem);
        occ_smem = smem;
    }
    if (per_sm < 1) return false;
    double nr = static_cast<double>(n);
    int ldr_a = ldr;
    const double* yc = y;
    long long* prof = g_orth_prof;
    void* args[] = {&yc,   &out,   &n_pad, &w,    &nr,       &ldr_a,
                    &partial, &wsum, &flags, &prof, &row_mean, &cstat};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_orth_fused<WP>), dim3(P),
                                       dim3(256), args, smem, st) == cudaSuccess;
}

// W -> T = R^{-1} for the multi-kernel / sharded CholeskyQR (same
// elimination and pivot rules as the fused kernel's step 3 and 4a). With y
// (apply mode, one CTA per SM) every CTA computes the identical T and applies
// it to its own 4-row groups of the panel, q = y T, staged through shared
// memory (loaded while the factor is computed) — one launch instead of the
// factor kernel plus an apply kernel; CTA 0 writes rinv (nullable) and the
// flags. Gated off (third pass after an unshifted first one): q = y.
template <int WP>
__global__ void __launch_bounds__(256) k_chol_inv_elim(const double* __restrict__ wmat, int w,
                                                       double nrows, int pass,
                                                       double* __restrict__ rinv,
                                                       int* __restrict__ flags,
                                                       const int* __restrict__ gate,
                                                       const double* __restrict__ y,
                                                       double* __restrict__ q, size_t n_pad) {
    const size_t nq = n_pad / 4;
    const size_t g0 = nq * blockIdx.x / gridDim.x, g1 = nq * (blockIdx.x + 1) / gridDim.x;
    if (gate && !(gate[0] & 1)) {
        if (y)
            for (size_t e = g0 * WP + threadIdx.x; e < g1 * WP; e += blockDim.x)
                reinterpret_cast<double4*>(q)[e] = reinterpret_cast<const double4*>(y)[e];
        return;
    }
    __shared__ int dropped_s[WP];
    __shared__ double d0s[WP];
    __shared__ double dpiv[WP];
    __shared__ double tr_s[2];
    __shared__ unsigned short tri[WP * (WP + 1) / 2];
    __shared__ int tri_off[WP + 1];
    extern __shared__ double ce[];  // R [WP*WP], E [WP*WP], apply mode: the CTA's y rows
    double* R = ce;
    double* E = R + WP * WP;
    double* ys = E + WP * WP;
    const int tid = threadIdx.x;
    if (y)  // coalesced copy of this CTA's panel rows, in flight during the factor
        for (size_t e = tid; e < (g1 - g0) * WP; e += blockDim.x)
            reinterpret_cast<double4*>(ys)[e] = reinterpret_cast<const double4*>(y)[g0 * WP + e];
    for (int i = tid; i <= WP; i += blockDim.x) {
        const int off = i * WP - (i * (i - 1)) / 2;
        tri_off[i] = off;
        for (int j = i; j < WP && i < WP; ++j)
            tri[off + j - i] = static_cast<unsigned short>((i << 8) | j);
    }
    if (tid < WP) d0s[tid] = tid < w ? wmat[tid * WP + tid] : 0.0;
    __syncthreads();
    if (tid == 0) {
        double tr = 0.0, mx = 0.0;
        for (int j = 0; j < w; ++j) {
            tr += d0s[j];
            mx = fmax(mx, d0s[j]);
        }
        tr_s[0] = tr;
        tr_s[1] = mx;
    }
    double sigma = 0.0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (int e = tid; e < WP * WP; e += blockDim.x) {
            const int i = e / WP, j = e % WP;
            double v = (i < w && j < w) ? wmat[e] : 0.0;
            if (i == j && i < w && d0s[i] > 0.0) v += sigma;
            R[e] = v;
        }
        __syncthreads();
        if (!chol_inverse<WP>(R, E, w, d0s, tr_s[1], pass == 0 && attempt == 0, pass != 0,
                                  dropped_s, dpiv, tri, tri_off))
            break;
        sigma = 11.0 * (nrows * w + static_cast<double>(w) * (w + 1)) * 0x1.0p-53 * tr_s[0];
        if (tid == 0 && blockIdx.x == 0) {
            flags[0] |= 1;  // any shift in this solve (reported)
            flags[1] = 1;   // this orthonormalization shifted: its third pass runs
        }
        __syncthreads();
    }
    __syncthreads();
    for (int e = tid; e < WP * WP; e += blockDim.x) {
        const int i = e / WP, j = e % WP;
        const double dj = dpiv[j];
        const double t = (i <= j && dj > 0.0) ? E[j * WP + i] * rsqrt(dj) : 0.0;
        if (rinv && blockIdx.x == 0) rinv[e] = t;
        R[e] = t;  // E is no longer read: R's slot holds T
    }
    if (!y) return;
    __syncthreads();
    // q = y T on this CTA's 4-row groups (T upper triangular), from shared memory
    for (size_t item = tid; item < (g1 - g0) * WP; item += blockDim.x) {
        const size_t qb = item / WP;
        const int c = static_cast<int>(item % WP);
        const double* yb = ys + qb * WP * 4;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        for (int k = 0; k <= c; ++k) {
            const double r = R[k * WP + c];
            const double4 v = *reinterpret_cast<const double4*>(yb + k * 4);
            s0 += v.x * r;
            s1 += v.y * r;
            s2 += v.z * r;
            s3 += v.w * r;
        }
        *reinterpret_cast<double4*>(q + (g0 + qb) * WP * 4 + c * 4) = make_double4(s0, s1, s2, s3);
    }
}

}  // namespace

extern "C" void divscope_debug_orth_prof(long long* dev_buf) { g_orth_prof = dev_buf; }

int orth_fused_grid(size_t n_pad, int sms) {
    return std::min<int>(sms, static_cast<int>(std::max<size_t>(n_pad / 4 / 8, 1)));
}

bool launch_orth_fused(double* y, double* t, double* out, size_t n_pad, int wp, int w, size_t n,
                       double* partial, double* wsum, int* flags, int sms, cudaStream_t st,
                       const double* row_mean, double* cstat) {
    (void)t;
    bool ok = false;
    switch (wp) {
        case 8: ok = launch_wp<8>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 16: ok = launch_wp<16>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 24: ok = launch_wp<24>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 32: ok = launch_wp<32>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 40: ok = launch_wp<40>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 48: ok = launch_wp<48>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 56: ok = launch_wp<56>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        case 64: ok = launch_wp<64>(y, out, n_pad, w, n, partial, wsum, flags, sms, st, row_mean, cstat); break;
        default: return false;
    }
    if (ok) count_launch();
    return ok;
}

bool launch_chol_inv_elim(const double* w_mat, int wp, int w, size_t n, int pass, double* rinv,
                          int* flags, cudaStream_t st, const int* gate, const double* y,
                          double* q, size_t n_pad, int sms) {
    // apply mode: one CTA per SM, its panel rows staged in shared memory
    const size_t nq = n_pad / 4;
    int grid = 1;
    size_t smem = static_cast<size_t>(2) * wp * wp * sizeof(double);
    if (y) {
        grid = static_cast<int>(std::max<size_t>(1, std::min<size_t>(sms, nq)));
        const size_t rows_per_cta = (nq + grid - 1) / grid * 4;
        const size_t stage = rows_per_cta * wp * sizeof(double);
        if (smem + stage > 200 * 1024) return false;  // caller falls back to the two kernels
        smem += stage;
    }
    const double nr = static_cast<double>(n);
    switch (wp) {
#define DSB_CE(W)                                                                              \
    case W:                                                                                    \
        allow_dyn_smem(reinterpret_cast<const void*>(k_chol_inv_elim<W>));                     \
        k_chol_inv_elim<W><<<grid, 256, smem, st>>>(w_mat, w, nr, pass, rinv, flags, gate, y, \
                                                    q, n_pad);                               \
        break;
        DSB_CE(8) DSB_CE(16) DSB_CE(24) DSB_CE(32) DSB_CE(40) DSB_CE(48) DSB_CE(56) DSB_CE(64)
#undef DSB_CE
        default:
            return false;
    }
    count_launch();
    return true;
}

}  // namespace dsb
