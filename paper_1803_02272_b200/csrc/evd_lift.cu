// K5 — the projected eigenproblem on the device (replaces the Eigen
// SelfAdjointEigenSolver call, the |lambda| ordering and the resid of
// eigs_sym, ref src/rsvd.cpp:109-145, plus the eigenvalue filter of
// embed_from_spectrum, ref src/mds.cpp:81-100).
// K6 — lift U = Q V_keep, sign normalization and sqrt(lambda) scaling
// (ref rsvd.cpp:129-138; mds.cpp:62-77, :102-112).
//
// K5 runs in one CTA: B = 1/2 (B + B^T) is stored packed (upper triangle) in
// shared memory next to the w x w eigenvector matrix, and diagonalized by
// parallel cyclic Jacobi: each round applies w/2 disjoint rotations
// (round-robin tournament ordering), updating every 2x2 block of B and
// every row pair of V independently — two barriers per round, no atomics.
#include <algorithm>
#include <cstdlib>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace dsb {

namespace {

__device__ __forceinline__ int pk(int a, int b, int w) {
    if (a > b) {
        const int t = a;
        a = b;
        b = t;
    }
    return a * w - (a * (a - 1)) / 2 + (b - a);
}

// Rotation of pair (p, q) annihilating a_pq (Rutishauser's formulas, as the
// oracle's Jacobi; jacobi_rot2 below): J = [[c, s], [-s, c]] on (p, q).
// theta = (a_qq - a_pp) / (2 a_pq), t = sgn(theta) / (|theta| + sqrt(theta^2+1)),
// c = 1 / sqrt(t^2 + 1), s = t c. The reciprocals / square roots use the
// MUFU seeds plus Newton steps (a few ulps): any c, s with c^2 + s^2 = 1 to
// rounding is an orthogonal rotation, and a slightly imperfect annihilation is
// removed by the next sweep.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return r;
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y = rsqrt(x);  // MUFU.RSQ64H + refinement in libdevice
    return y;
}

// Rotation from d = a_qq - a_pp and a_pq without forming theta:
// t = 2 a_pq sgn(d) / (|d| + sqrt(d^2 + 4 a_pq^2)) (the same angle as
// jacobi_rot: t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)) with theta =
// d / (2 a_pq)), one reciprocal and two reciprocal square roots on the
// dependent chain instead of two and two.
__device__ __forceinline__ void jacobi_rot2(double app, double aqq, double apq, double& c,
                                            double& s) {
    c = 1.0;
    s = 0.0;
    if (fabs(apq) >= 1e-300) {
        const double d = aqq - app;
        const double a2 = apq + apq;
        const double h2 = fma(d, d, a2 * a2);
        const double r = h2 * rsqrt_nr(h2);  // sqrt(d^2 + 4 a_pq^2)
        double t = a2 * rcp_nr(fabs(d) + r);
        if (d < 0.0) t = -t;
        c = rsqrt_nr(fma(t, t, 1.0));
        s = t * c;
    }
}

// (i, j) block of J_i^T A J_j for the 2x2 blocks of the round's pairs
__device__ __forceinline__ void block_update(const double* __restrict__ Ain, double* __restrict__ Aout,
                                             int w, int pi, int qi, int pj, int qj, double ci,
                                             double si, double cj, double sj, bool diag) {
    const bool vqi = qi < w, vqj = qj < w;
    const double a11 = Ain[pk(pi, pj, w)];
    const double a12 = vqj ? Ain[pk(pi, qj, w)] : 0.0;
    const double a21 = vqi ? Ain[pk(qi, pj, w)] : 0.0;
    const double a22 = (vqi && vqj) ? Ain[pk(qi, qj, w)] : 0.0;
    const double b11 = cj * a11 - sj * a12, b12 = sj * a11 + cj * a12;
    const double b21 = cj * a21 - sj * a22, b22 = sj * a21 + cj * a22;
    const double n11 = ci * b11 - si * b21, n21 = si * b11 + ci * b21;
    const double n12 = ci * b12 - si * b22, n22 = si * b12 + ci * b22;
    if (diag) {
        Aout[pk(pi, pi, w)] = n11;
        if (vqi) {
            Aout[pk(qi, qi, w)] = n22;
            Aout[pk(pi, qi, w)] = 0.0;
        }
    } else {
        Aout[pk(pi, pj, w)] = n11;
        if (vqj) Aout[pk(pi, qj, w)] = n12;
        if (vqi) Aout[pk(qi, pj, w)] = n21;
        if (vqi && vqj) Aout[pk(qi, qj, w)] = n22;
    }
}

// round-robin tournament: players 0..m-1, player 0 fixed
__device__ __forceinline__ void pair_at(int r, int k, int m, int& p, int& q) {
    const int x = (k == 0) ? 0 : 1 + ((k - 1 + r) % (m - 1));
    const int y = 1 + ((m - 2 - k + r) % (m - 1));
    p = min(x, y);
    q = max(x, y);
}

// off-diagonal / diagonal energy of packed A -> done flag (block reduce)
__device__ int jacobi_converged(const double* __restrict__ A, int w, double* red) {
    const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31;
    double off = 0.0, dg = 0.0;
    for (int a = tid; a < w; a += nt) {
        const double* row = A + pk(a, a, w);
        dg += row[0] * row[0];
        for (int b = 1; b < w - a; ++b) off += row[b] * row[b];
    }
    off = warp_sum(off);
    dg = warp_sum(dg);
    if (lane == 0) {
        red[warp] = off;
        red[32 + warp] = dg;
    }
    __syncthreads();
    double so = 0.0, sd = 0.0;
    for (int k = 0; k < nt / 32; ++k) {
        so += red[k];
        sd += red[32 + k];
    }
    __syncthreads();
    return (so == 0.0 || so <= 1e-34 * sd) ? 1 : 0;
}

// Shared tail: reference ordering (rsvd.cpp:118-127), keep / resid
// (rsvd.cpp:129-142), embed filter (mds.cpp:85-99), V_keep.
// dg: the w eigenvalues (diagonal of the converged A); V row-major with
// leading dimension ldv
__device__ void evd_finish_dg(const double* __restrict__ dg, const double* __restrict__ V,
                              int ldv, int w, int rank, int requested,
                              const double* __restrict__ scalars, int fro_index, const EvdOut& o,
                              int sweeps, int done, int* __restrict__ order,
                              int* __restrict__ kept);

__device__ void evd_finish(const double* __restrict__ A, const double* __restrict__ V, int w,
                           int rank, int requested, const double* __restrict__ scalars,
                           int fro_index, const EvdOut& o, int sweeps, int done,
                           int* __restrict__ order, int* __restrict__ kept) {
    __shared__ double dg[kMaxWP];
    for (int a = threadIdx.x; a < w; a += blockDim.x) dg[a] = A[pk(a, a, w)];
    __syncthreads();
    evd_finish_dg(dg, V, w, w, rank, requested, scalars, fro_index, o, sweeps, done, order, kept);
}

__device__ void evd_finish_dg(const double* __restrict__ dg, const double* __restrict__ V,
                              int ldv, int w, int rank, int requested,
                              const double* __restrict__ scalars, int fro_index, const EvdOut& o,
                              int sweeps, int done, int* __restrict__ order,
                              int* __restrict__ kept) {
    const int tid = threadIdx.x, nt = blockDim.x;
    // Reference order (rsvd.cpp:118-127 applied to Eigen's ascending output):
    // ascending stable sort, then stable sort by |lambda| desc, positive first.
    // Equivalent total order on (lambda, index): a before b iff
    //   |la| > |lb|, or |la| == |lb| and la > lb, or la == lb and a < b
    // (equal values keep the ascending sort's index order). Each thread
    // computes its element's rank by counting predecessors.
    // NaN eigenvalues (non-finite input) sort last by index, so the ranks
    // always form a permutation
    for (int a = tid; a < w; a += nt) {
        const double la = dg[a];
        const bool na = isnan(la);
        int pos = 0;
        for (int b = 0; b < w; ++b) {
            if (b == a) continue;
            const double lb = dg[b];
            const bool nb = isnan(lb);
            bool b_first;
            if (na || nb)
                b_first = (na && nb) ? (b < a) : na;
            else
                b_first = (fabs(lb) != fabs(la)) ? (fabs(lb) > fabs(la))
                          : (lb != la)           ? (lb > la)
                                                 : (b < a);
            pos += b_first ? 1 : 0;
        }
        order[pos] = a;
    }
    __syncthreads();
    if (tid == 0) {
        // "positive first on equal |lambda|" (rsvd.cpp:118-127) also for twins
        // equal to rounding (|la| and |lb| within 4 ulps): the reference's
        // exact tie comes out of Eigen's EVD; ours can differ in the last bit.
        for (int a = 0; a + 1 < w; ++a) {
            const double x = dg[order[a]], y = dg[order[a + 1]];
            if (x < 0.0 && y > 0.0 && fabs(fabs(x) - y) <= 4.0 * 0x1.0p-52 * fabs(x)) {
                const int t = order[a];
                order[a] = order[a + 1];
                order[a + 1] = t;
            }
        }
        const int keep = min(rank, w);
        double sumsq = 0.0, maxabs = 0.0;
        for (int a = 0; a < w; ++a) o.vals[a] = dg[order[a]];
        for (int a = 0; a < keep; ++a) {
            const double lam = o.vals[a];
            sumsq += lam * lam;
            maxabs = fmax(maxabs, fabs(lam));
        }
        const double fro2 = scalars[fro_index];
        const double eps = 1e-9 * maxabs;
        int cnt = 0;
        double mass = 0.0;
        for (int a = 0; a < keep; ++a) {
            const double lam = o.vals[a];
            if (requested < 0)  // eigenvector mode: the first keep, any sign
                kept[cnt++] = order[a];
            else if (lam > eps && cnt < requested)
                kept[cnt++] = order[a];
            else if (lam < 0.0)
                mass += -lam;
        }
        o.dmeta[0] = sqrt(fmax(0.0, fro2 - sumsq));
        o.dmeta[1] = mass;
        o.dmeta[2] = sumsq;
        o.imeta[0] = keep;
        o.imeta[1] = cnt;
        o.imeta[2] = requested >= 0 && cnt < requested ? 1 : 0;
        o.imeta[3] = sweeps;
        o.imeta[4] = done;
        for (int c = 0; c < cnt; ++c) o.kept_vals[c] = dg[kept[c]];
    }
    __syncthreads();
    const int r = o.imeta[1];
    const int rq = requested < 0 ? o.imeta[0] : requested;  // columns of vkeep
    for (int e = tid; e < w * rq; e += nt) {
        const int x = e / rq, c = e % rq;
        o.vkeep[e] = c < r ? V[x * ldv + kept[c]] : 0.0;
    }
}

constexpr int kEvdThreads = 512;
__device__ long long g_evd_prof[16];

// General kernel (any w <= 128): packed A single-buffered, rotations of a
// round computed first (barrier), then all 2x2 blocks and V row pairs.
__global__ void __launch_bounds__(kEvdThreads) k_evd(const double* __restrict__ bmat, int wp, int w,
                                                     int rank, int requested,
                                                     const double* __restrict__ scalars,
                                                     int fro_index, EvdOut o) {
    extern __shared__ double sm[];
    const int npk = w * (w + 1) / 2;
    double* A = sm;       // packed upper triangle
    double* V = A + npk;  // [w][w]
    __shared__ double cs[kMaxWP / 2 + 1], sn[kMaxWP / 2 + 1];
    __shared__ int pp[kMaxWP / 2 + 1], qq[kMaxWP / 2 + 1];
    __shared__ double red[64];
    __shared__ int order[kMaxWP], kept[kMaxWP];
    __shared__ unsigned char blk_i[(kMaxWP / 2) * (kMaxWP / 2 + 1) / 2];
    __shared__ unsigned char blk_j[(kMaxWP / 2) * (kMaxWP / 2 + 1) / 2];
    __shared__ unsigned short sched[(kMaxWP - 1) * (kMaxWP / 2)];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < w * w; e += nt) {
        const int a = e / w, b = e % w;
        if (b >= a) A[pk(a, b, w)] = 0.5 * (bmat[a * wp + b] + bmat[b * wp + a]);
        V[e] = (a == b) ? 1.0 : 0.0;
    }
    const int m = w + (w & 1), h = m / 2, nblk = h * (h + 1) / 2;
    for (int i = tid; i < h; i += nt) {
        const int base = i * h - (i * (i - 1)) / 2;
        for (int j = i; j < h; ++j) {
            blk_i[base + j - i] = static_cast<unsigned char>(i);
            blk_j[base + j - i] = static_cast<unsigned char>(j);
        }
    }
    // tournament schedule of every round, precomputed (no modulo in the loop)
    for (int e = tid; e < (m - 1) * h; e += nt) {
        const int r = e / h, k = e % h;
        int p, q;
        pair_at(r, k, m, p, q);
        sched[e] = static_cast<unsigned short>((p << 8) | q);
    }
    // V rotation mapping: thread -> (pair vi, first row vk0), rows stride vks.
    // With enough threads the block updates (first half) and the V row pairs
    // (second half) run on different warps, side by side
    const int vbase = (nt >= 256 && nblk <= nt / 2) ? nt / 2 : 0;
    const int nbt = vbase ? vbase : nt;  // threads of the block-update phase
    const int tv = tid - vbase, ntv = nt - vbase;
    const int vact = (ntv / h) * h;  // active threads in the V phase
    const int vi = tv >= 0 ? tv % h : 0, vk0 = tv >= 0 ? tv / h : 0, vks = ntv / h;
    __syncthreads();
    // a thread's own block (when every block has one) is fixed for the
    // whole solve: its pair indices stay in registers
    const bool one_block = nblk <= nbt;
    const int my_i = (one_block && tid < nblk) ? blk_i[tid] : 0;
    const int my_j = (one_block && tid < nblk) ? blk_j[tid] : 0;
    int done = (w <= 1), sweeps = 0;
    long long t_a = clock64(), acc1 = 0, acc2 = 0, acc3 = 0;
    for (; sweeps < 60 && !done; ++sweeps) {
        for (int r = 0; r < m - 1; ++r) {
            const long long t0 = clock64();
            for (int k = tid; k < h; k += nt) {
                const int pq = sched[r * h + k];
                const int p = pq >> 8, q = pq & 0xff;
                double c = 1.0, s = 0.0;
                if (q < w) jacobi_rot2(A[pk(p, p, w)], A[pk(q, q, w)], A[pk(p, q, w)], c, s);
                pp[k] = p;
                qq[k] = q;
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            const long long t1 = clock64();
            acc1 += t1 - t0;
            if (one_block) {
                if (tid < nblk)
                    block_update(A, A, w, pp[my_i], qq[my_i], pp[my_j], qq[my_j], cs[my_i],
                                 sn[my_i], cs[my_j], sn[my_j], my_i == my_j);
            } else {
                for (int e = tid; e < nblk && tid < nbt; e += nbt) {
                    const int i = blk_i[e], j = blk_j[e];
                    block_update(A, A, w, pp[i], qq[i], pp[j], qq[j], cs[i], sn[i], cs[j], sn[j],
                                 i == j);
                }
            }
            if (tv >= 0 && tv < vact && qq[vi] < w) {
                const int p = pp[vi], q = qq[vi];
                const double c = cs[vi], s = sn[vi];
                // the rows' loads first, then the rotations and stores (the
                // row pairs are disjoint; 4 in flight per thread)
                for (int k0 = vk0; k0 < w; k0 += 4 * vks) {
                    double vp[4], vq[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int k = k0 + u * vks;
                        vp[u] = k < w ? V[k * w + p] : 0.0;
                        vq[u] = k < w ? V[k * w + q] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int k = k0 + u * vks;
                        if (k < w) {
                            V[k * w + p] = c * vp[u] - s * vq[u];
                            V[k * w + q] = s * vp[u] + c * vq[u];
                        }
                    }
                }
            }
            __syncthreads();
            acc2 += clock64() - t1;
        }
        const long long t2 = clock64();
        done = jacobi_converged(A, w, red);
        acc3 += clock64() - t2;
    }
    const long long t_b = clock64();
    evd_finish(A, V, w, rank, requested, scalars, fro_index, o, sweeps, done, order, kept);
    if (tid == 0) {
        g_evd_prof[0] = t_b - t_a;
        g_evd_prof[1] = acc1;
        g_evd_prof[2] = acc2;
        g_evd_prof[3] = acc3;
        g_evd_prof[4] = clock64() - t_b;
        g_evd_prof[5] = sweeps;
    }
}

// Small problems (w <= 16): one warp, the matrix in registers. Lane i holds
// row i of A (full storage) and row i of V. The tournament is run on fixed
// positions — pairs (k, M-1-k) every round — and the data moves instead
// (circle method: position 0 fixed, position j -> j+1, M-1 -> 1), so every
// register index is a compile-time constant: column updates and the column
// move are register operations, rotation inputs, the partner row and the row
// move are shuffles. No shared memory and no barriers in the sweep. Same
// rotations (jacobi_rot2), same convergence test, same tail (evd_finish_dg
// with eigenvalues in original index order). Padded positions (w odd) keep
// a_pq = 0, so their rotations are exact identities.
template <int M>
__global__ void __launch_bounds__(32, 1) k_evd_warp(const double* __restrict__ bmat, int wp, int w,
                                                    int rank, int requested,
                                                    const double* __restrict__ scalars,
                                                    int fro_index, EvdOut o) {
    constexpr int H = M / 2;
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ double dg[32], Vs[32 * 32];
    __shared__ int order[32], kept[32];
    const int lane = threadIdx.x;
    const long long t_a = clock64();
    double a[M], v[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
        a[j] = (lane < w && j < w) ? 0.5 * (bmat[lane * wp + j] + bmat[j * wp + lane]) : 0.0;
        v[j] = (j == lane) ? 1.0 : 0.0;
    }
    const bool isp = lane < H;
    const int partner = lane < M ? M - 1 - lane : lane;
    const int from = lane == 0 ? 0 : (lane == 1 ? M - 1 : (lane < M ? lane - 1 : lane));
    int done = __all_sync(FULL, w <= 1) ? 1 : 0, sweeps = 0;
    long long rounds = 0;
    for (; sweeps < 60 && !done; ++sweeps) {
#pragma unroll 1
        for (int r = 0; r < M - 1; ++r, ++rounds) {
            // rotation of this lane's pair (lanes < H): A[k][k], A[q][q], A[k][q]
            double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double x = __shfl_sync(FULL, a[k], k);
                const double y = __shfl_sync(FULL, a[M - 1 - k], M - 1 - k);
                const double z = __shfl_sync(FULL, a[M - 1 - k], k);
                if (lane == k) {
                    app = x;
                    aqq = y;
                    apq = z;
                }
            }
            double c, s;
            jacobi_rot2(app, aqq, apq, c, s);
            // A J and V J: columns (k, M-1-k) of every row
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double ck = __shfl_sync(FULL, c, k), sk = __shfl_sync(FULL, s, k);
                const double ap = a[k], aq = a[M - 1 - k];
                a[k] = ck * ap - sk * aq;
                a[M - 1 - k] = sk * ap + ck * aq;
                const double vp = v[k], vq = v[M - 1 - k];
                v[k] = ck * vp - sk * vq;
                v[M - 1 - k] = sk * vp + ck * vq;
            }
            // J^T (A J): rows p' = c p - s q, q' = s p + c q with the own pair's rotation
            const double co = __shfl_sync(FULL, c, isp ? lane : partner);
            const double so = __shfl_sync(FULL, s, isp ? lane : partner);
#pragma unroll
            for (int j = 0; j < M; ++j) {
                const double t = __shfl_sync(FULL, a[j], partner);
                a[j] = isp ? co * a[j] - so * t : so * t + co * a[j];
            }
#pragma unroll
            for (int k = 0; k < H; ++k) {  // the annihilated pair, exactly
                if (lane == k) a[M - 1 - k] = 0.0;
                if (lane == M - 1 - k) a[k] = 0.0;
            }
            // move the data one tournament step: columns in registers, rows by shuffle
            {
                const double al = a[M - 1], vl = v[M - 1];
#pragma unroll
                for (int j = M - 1; j >= 2; --j) {
                    a[j] = a[j - 1];
                    v[j] = v[j - 1];
                }
                if (M > 1) {
                    a[1] = al;
                    v[1] = vl;
                }
            }
#pragma unroll
            for (int j = 0; j < M; ++j) a[j] = __shfl_sync(FULL, a[j], from);
        }
        // convergence: off-diagonal vs diagonal energy (as jacobi_converged)
        double off = 0.0, dgs = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            if (j == lane) dgs += a[j] * a[j];
            else off += a[j] * a[j];
        }
        off = warp_sum(off);
        dgs = warp_sum(dgs);
        // a vote keeps the loop condition warp-uniform for the compiler (no
        // collective fallback around the shuffles)
        done = __all_sync(FULL, off == 0.0 || off <= 1e-34 * dgs) ? 1 : 0;
    }
    const long long t_b = clock64();
    // position j holds original index 1 + (j - 1 - rounds) mod (M - 1) (0 stays)
    const int sh = M > 1 ? static_cast<int>(rounds % (M - 1)) : 0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const int oj = j == 0 ? 0 : 1 + ((j - 1 - sh + (M - 1)) % (M - 1));
        if (oj < w) {
            if (lane == j) dg[oj] = a[j];
            if (lane < w) Vs[lane * w + oj] = v[j];
        }
    }
    __syncwarp();
    evd_finish_dg(dg, Vs, w, w, rank, requested, scalars, fro_index, o, sweeps, done, order, kept);
    if (lane == 0) {
        g_evd_prof[0] = t_b - t_a;
        g_evd_prof[1] = 0;
        g_evd_prof[2] = 0;
        g_evd_prof[3] = 0;
        g_evd_prof[4] = clock64() - t_b;
        g_evd_prof[5] = sweeps;
    }
}

template <int M>
void launch_evd_warp_m(int m, const double* b, int wp, int w, int rank, int requested_rank,
                       const double* scalars, int fro_index, const EvdOut& o, cudaStream_t st) {
    if constexpr (M <= 16) {
        if (m == M) {
            k_evd_warp<M><<<1, 32, 0, st>>>(b, wp, w, rank, requested_rank, scalars, fro_index, o);
            return;
        }
        launch_evd_warp_m<M + 2>(m, b, wp, w, rank, requested_rank, scalars, fro_index, o, st);
    }
}

// rows of the panel staged per chunk by k_lift (<= 64 KB of shared memory)
__host__ __device__ constexpr int lift_chunk_rows(int wp) { return wp <= 64 ? 128 : 64; }

// U = Q V_keep (n x r, row-major into coords). CTA c owns rows
// [n c / P, n (c+1) / P); thread t owns column t % r and rows t / r + k * (256 / r),
// keeping a running (value at max |u|, first index) that is merged in thread
// (= row) order into the CTA partial — the sign rule of ref mds.cpp:65-77.
__global__ void __launch_bounds__(256) k_lift(const double* __restrict__ q, int n, int wp, int w,
                                              const double* __restrict__ vkeep,
                                              const int* __restrict__ imeta, int rmax,
                                              double* __restrict__ coords,
                                              double* __restrict__ partial, long long row_off) {
    extern __shared__ double sm_lift[];
    double* sv = sm_lift;             // [w][rmax]
    double* sq = sm_lift + w * rmax;  // staged panel rows (4-row groups)
    __shared__ double best_v[256];
    __shared__ int best_i[256];
    const int r = imeta[1];
    if (r == 0) return;
    for (int e = threadIdx.x; e < w * rmax; e += blockDim.x) sv[e] = vkeep[e];
    const int row0 = static_cast<int>(static_cast<long long>(n) * blockIdx.x / gridDim.x);
    const int row1 = static_cast<int>(static_cast<long long>(n) * (blockIdx.x + 1) / gridDim.x);
    const int per = 256 / r;  // rows in flight per sweep (r <= 128)
    const int t = threadIdx.x;
    const int ch = lift_chunk_rows(wp);
    double bv = 0.0;
    int bi = -1;
    // the CTA's panel rows are staged chunk by chunk with coalesced copies
    // (their interleaved 4-row groups are contiguous), then every thread's
    // w-term dot products read shared memory
    for (int a = row0; a < row1; a += ch) {
        const int b = min(row1, a + ch);
        const int g0 = a / 4, g1 = (b + 3) / 4;
        const size_t base = static_cast<size_t>(g0) * wp * 4;
        for (int e = threadIdx.x; e < (g1 - g0) * wp * 4; e += blockDim.x) sq[e] = q[base + e];
        __syncthreads();
        if (t < per * r) {
            const int c = t % r;
            for (int i = a + t / r; i < b; i += per) {
                const double* qi = sq + static_cast<size_t>(i / 4 - g0) * wp * 4 + (i & 3);
                double s = 0.0;
                for (int k = 0; k < w; ++k) s += qi[k * 4] * sv[k * rmax + c];
                coords[static_cast<size_t>(i) * r + c] = s;
                if (bi < 0 || fabs(s) > fabs(bv)) {
                    bv = s;
                    bi = i;
                }
            }
        }
        __syncthreads();
    }
    best_v[t] = bv;
    best_i[t] = bi;
    __syncthreads();
    if (t < r) {
        double v = 0.0;
        int ix = -1;
        for (int k = 0; k < per; ++k) {  // threads t + k r own column t, rows in order
            const int ti = best_i[t + k * r];
            if (ti < 0) continue;
            const double tv = best_v[t + k * r];
            if (ix < 0 || fabs(tv) > fabs(v) || (fabs(tv) == fabs(v) && ti < ix)) {
                v = tv;
                ix = ti;
            }
        }
        partial[(static_cast<size_t>(blockIdx.x) * rmax + t) * 2 + 0] = v;
        partial[(static_cast<size_t>(blockIdx.x) * rmax + t) * 2 + 1] =
            ix < 0 ? -1.0 : static_cast<double>(ix + row_off);
    }
}

// per column: merge the CTA partials (warp per column, any order gives the
// same winner: larger |u|, then smaller index), scale = sign * sqrt(lambda)
__global__ void __launch_bounds__(256) k_lift_signs(const int* __restrict__ imeta, int P, int rmax,
                                                    const double* __restrict__ kept_vals,
                                                    const double* __restrict__ partial,
                                                    double* __restrict__ scale) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int r = imeta[1];
    if (warp >= r) return;
    double v = 0.0;
    long long ix = -1;
    for (int b = lane; b < P; b += 32) {
        const double iv = partial[(static_cast<size_t>(b) * rmax + warp) * 2 + 1];
        if (!(iv >= 0.0)) continue;  // empty CTA / rank (or NaN fill)
        const double tv = partial[(static_cast<size_t>(b) * rmax + warp) * 2 + 0];
        const long long ti = static_cast<long long>(iv);
        if (ix < 0 || fabs(tv) > fabs(v) || (fabs(tv) == fabs(v) && ti < ix)) {
            v = tv;
            ix = ti;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, ix, o);
        if (oi >= 0 && (ix < 0 || fabs(ov) > fabs(v) || (fabs(ov) == fabs(v) && oi < ix))) {
            v = ov;
            ix = oi;
        }
    }
    if (lane == 0) scale[warp] = (v < 0.0 ? -1.0 : 1.0) * sqrt(kept_vals[warp]);
}

__global__ void k_lift_scale(int n, const int* __restrict__ imeta,
                             const double* __restrict__ scale_g, double* __restrict__ coords) {
    __shared__ double scale[kMaxWP];
    const int r = imeta[1];
    if (threadIdx.x < r) scale[threadIdx.x] = scale_g[threadIdx.x];
    __syncthreads();
    const size_t total = static_cast<size_t>(n) * r;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x)
        coords[e] *= scale[e % r];
}


}  // namespace

extern "C" void divscope_debug_evd_prof(long long* host16) {
    cudaMemcpyFromSymbol(host16, g_evd_prof, 16 * sizeof(long long));
}

void launch_evd(const double* b, int wp, int w, int rank, int requested_rank,
                const double* scalars, int fro_index, const EvdOut& o, cudaStream_t st) {
    static const bool warp_evd = [] {
        const char* e = std::getenv("DSB_EVD_WARP");
        return !(e && std::atoi(e) == 0);
    }();
    // the register kernel wins up to w = 16 (measured against the CTA kernel
    // with its split block / V warps: w = 12 63k vs 97k cycles, w = 16 95k vs
    // 127k, w = 20 even — 162k vs 159k, one sweep more); wider, its single
    // warp is latency-bound (w = 30: 867k vs 292k)
    if (warp_evd && w >= 1 && w <= 16) {
        launch_evd_warp_m<2>(w + (w & 1), b, wp, w, rank, requested_rank, scalars, fro_index, o,
                             st);
        count_launch();
        return;
    }
    {
        const size_t smem = (static_cast<size_t>(w) * (w + 1) / 2 + static_cast<size_t>(w) * w) *
                            sizeof(double);
        allow_dyn_smem(reinterpret_cast<const void*>(k_evd));
        static const int forced = [] {
            const char* e = std::getenv("DSB_EVD_THREADS");
            return e ? std::atoi(e) : 0;
        }();
        const int threads = forced > 0 ? forced : (w <= 64 ? 256 : kEvdThreads);
        k_evd<<<1, threads, smem, st>>>(b, wp, w, rank, requested_rank, scalars, fro_index, o);
    }
    count_launch();
}

void launch_lift(const double* q, size_t n, int wp, int w, const double* vkeep,
                 const double* kept_vals, const int* imeta, int rmax, double* coords,
                 double* partial, int sms, cudaStream_t st) {
    const int P = lift_grid(n, sms);
    launch_lift_partial(q, n, wp, w, vkeep, imeta, rmax, coords, partial, 0, P, st);
    double* scale = partial + static_cast<size_t>(P) * rmax * 2;
    launch_lift_finish(n, imeta, P, rmax, kept_vals, partial, scale, coords, st);
}

int lift_grid(size_t n, int sms) {
    return static_cast<int>(std::min<size_t>(static_cast<size_t>(sms) * 2, std::max<size_t>(n / 64, 1)));
}

void launch_lift_partial(const double* q, size_t n, int wp, int w, const double* vkeep,
                         const int* imeta, int rmax, double* coords, double* partial,
                         long long row_off, int P, cudaStream_t st) {
    const size_t smem =
        (static_cast<size_t>(w) * rmax +
         static_cast<size_t>(lift_chunk_rows(wp) / 4 + 2) * wp * 4) * sizeof(double);
    allow_dyn_smem(reinterpret_cast<const void*>(k_lift));
    k_lift<<<P, 256, smem, st>>>(q, static_cast<int>(n), wp, w, vkeep, imeta, rmax, coords,
                                 partial, row_off);
    count_launch();
}

// signs from `P` partials (any number of CTAs / ranks, merged order-free),
// then coords (n local rows) *= sign * sqrt(lambda); scale -> rmax doubles
void launch_lift_finish(size_t n, const int* imeta, int P, int rmax, const double* kept_vals,
                        const double* partial, double* scale, double* coords, cudaStream_t st) {
    k_lift_signs<<<(rmax * 32 + 255) / 256, 256, 0, st>>>(imeta, P, rmax, kept_vals, partial,
                                                         scale);
    const int sg = static_cast<int>(std::min<size_t>((n * rmax + 255) / 256, 148 * 8));
    k_lift_scale<<<std::max(sg, 1), 256, 0, st>>>(static_cast<int>(n), imeta, scale, coords);
    count_launch(2);
}

}  // namespace dsb
