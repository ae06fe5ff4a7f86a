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

constexpr int kEvdThreads = 512;

__global__ void __launch_bounds__(kEvdThreads) k_evd(const double* __restrict__ bmat, int wp, int w,
                                                     int rank, int requested,
                                                     const double* __restrict__ scalars,
                                                     int fro_index, EvdOut o) {
    extern __shared__ double sm[];
    const int npk = w * (w + 1) / 2;
    double* A = sm;            // packed upper triangle
    double* V = A + npk;       // [w][w]
    __shared__ double cs[kMaxWP / 2 + 1], sn[kMaxWP / 2 + 1];
    __shared__ int pp[kMaxWP / 2 + 1], qq[kMaxWP / 2 + 1];
    __shared__ double red[2][kEvdThreads / 32];
    __shared__ int done;
    __shared__ int order[kMaxWP];
    __shared__ int kept[kMaxWP];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;

    for (int a = tid; a < w; a += nt)
        for (int b = a; b < w; ++b)
            A[pk(a, b, w)] = 0.5 * (bmat[a * wp + b] + bmat[b * wp + a]);
    for (int e = tid; e < w * w; e += nt) V[e] = (e / w == e % w) ? 1.0 : 0.0;
    if (tid == 0) done = (w <= 1);
    __syncthreads();

    const int m = w + (w & 1);  // players (w odd -> one dummy)
    const int h = m / 2;
    const int nblk = h * (h + 1) / 2;
    int sweeps = 0;
    for (; sweeps < 60 && !done; ++sweeps) {
        for (int r = 0; r < m - 1; ++r) {
            // phase 1: rotations of this round's pairs
            for (int k = tid; k < h; k += nt) {
                const int x = (k == 0) ? 0 : 1 + ((k - 1 + r) % (m - 1));
                const int kk = m - 1 - k;
                const int y = 1 + ((kk - 1 + r) % (m - 1));
                const int p = min(x, y), q = max(x, y);
                double c = 1.0, s = 0.0;
                if (q < w) {
                    const double apq = A[pk(p, q, w)];
                    if (fabs(apq) >= 1e-300) {
                        const double app = A[pk(p, p, w)], aqq = A[pk(q, q, w)];
                        const double theta = (aqq - app) / (2.0 * apq);
                        const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                                         (fabs(theta) + sqrt(theta * theta + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                pp[k] = p;
                qq[k] = q;
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // phase 2a: 2x2 blocks of A (J_i^T A J_j)
            for (int e = tid; e < nblk; e += nt) {
                // decode e -> (i, j), i <= j over h pairs (row-major upper)
                int i = 0, rem = e;
                while (rem >= h - i) {
                    rem -= h - i;
                    ++i;
                }
                const int j = i + rem;
                const int pi = pp[i], qi = qq[i], pj = pp[j], qj = qq[j];
                const double ci = cs[i], si = sn[i], cj = cs[j], sj = sn[j];
                const bool vqi = qi < w, vqj = qj < w;
                const double a11 = A[pk(pi, pj, w)];
                const double a12 = vqj ? A[pk(pi, qj, w)] : 0.0;
                const double a21 = vqi ? A[pk(qi, pj, w)] : 0.0;
                const double a22 = (vqi && vqj) ? A[pk(qi, qj, w)] : 0.0;
                const double b11 = cj * a11 - sj * a12, b12 = sj * a11 + cj * a12;
                const double b21 = cj * a21 - sj * a22, b22 = sj * a21 + cj * a22;
                const double n11 = ci * b11 - si * b21, n21 = si * b11 + ci * b21;
                const double n12 = ci * b12 - si * b22, n22 = si * b12 + ci * b22;
                if (i == j) {
                    A[pk(pi, pi, w)] = n11;
                    if (vqi) {
                        A[pk(qi, qi, w)] = n22;
                        A[pk(pi, qi, w)] = 0.0;
                    }
                } else {
                    A[pk(pi, pj, w)] = n11;
                    if (vqj) A[pk(pi, qj, w)] = n12;
                    if (vqi) A[pk(qi, pj, w)] = n21;
                    if (vqi && vqj) A[pk(qi, qj, w)] = n22;
                }
            }
            // phase 2b: columns of V
            for (int e = tid; e < w * h; e += nt) {
                const int k = e / h, i = e % h;
                const int p = pp[i], q = qq[i];
                if (q < w) {
                    const double c = cs[i], s = sn[i];
                    const double vp = V[k * w + p], vq = V[k * w + q];
                    V[k * w + p] = c * vp - s * vq;
                    V[k * w + q] = s * vp + c * vq;
                }
            }
            __syncthreads();
        }
        // convergence: off-diagonal energy vs diagonal energy
        double off = 0.0, dg = 0.0;
        for (int e = tid; e < npk; e += nt) {
            // decode packed index e -> (a, b)
            int a = 0, rem = e;
            while (rem >= w - a) {
                rem -= w - a;
                ++a;
            }
            const double v = A[e];
            if (rem == 0)
                dg += v * v;
            else
                off += v * v;
        }
        off = warp_sum(off);
        dg = warp_sum(dg);
        if (lane == 0) {
            red[0][warp] = off;
            red[1][warp] = dg;
        }
        __syncthreads();
        if (tid == 0) {
            double so = 0.0, sd = 0.0;
            for (int k = 0; k < nt / 32; ++k) {
                so += red[0][k];
                sd += red[1][k];
            }
            done = (so == 0.0 || so <= 1e-34 * sd) ? 1 : 0;
        }
        __syncthreads();
    }

    if (tid == 0) {
        // ascending (stable on index), then stable by |lambda| desc, + first
        // (the reference sorts Eigen's ascending output, rsvd.cpp:118-127)
        for (int a = 0; a < w; ++a) order[a] = a;
        for (int a = 1; a < w; ++a) {
            const int x = order[a];
            const double vx = A[pk(x, x, w)];
            int b = a - 1;
            while (b >= 0 && A[pk(order[b], order[b], w)] > vx) {
                order[b + 1] = order[b];
                --b;
            }
            order[b + 1] = x;
        }
        for (int a = 1; a < w; ++a) {
            const int x = order[a];
            const double vx = A[pk(x, x, w)];
            int b = a - 1;
            while (b >= 0) {
                const double vb = A[pk(order[b], order[b], w)];
                const bool x_before =
                    (fabs(vx) != fabs(vb)) ? (fabs(vx) > fabs(vb)) : (vx > vb);
                if (!x_before) break;
                order[b + 1] = order[b];
                --b;
            }
            order[b + 1] = x;
        }
        const int keep = min(rank, w);
        double sumsq = 0.0, maxabs = 0.0;
        for (int a = 0; a < w; ++a) o.vals[a] = A[pk(order[a], order[a], w)];
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
            if (lam > eps && cnt < requested)
                kept[cnt++] = order[a];
            else if (lam < 0.0)
                mass += -lam;
        }
        o.dmeta[0] = sqrt(fmax(0.0, fro2 - sumsq));
        o.dmeta[1] = mass;
        o.dmeta[2] = sumsq;
        o.imeta[0] = keep;
        o.imeta[1] = cnt;
        o.imeta[2] = cnt < requested ? 1 : 0;
        o.imeta[3] = sweeps;
        o.imeta[4] = done;
        for (int c = 0; c < cnt; ++c) o.kept_vals[c] = A[pk(kept[c], kept[c], w)];
    }
    __syncthreads();
    // V_keep [w][requested]
    int r = o.imeta[1];
    for (int e = tid; e < w * requested; e += nt) {
        const int x = e / requested, c = e % requested;
        o.vkeep[e] = c < r ? V[x * w + kept[c]] : 0.0;
    }
}

// U = Q V_keep for a CTA-contiguous row range, written to coords (n x r),
// plus the CTA's per-column (|u| max, first index) partial.
__global__ void __launch_bounds__(256) k_lift(const double* __restrict__ q, int n, int wp, int w,
                                              const double* __restrict__ vkeep,
                                              const int* __restrict__ imeta, int rmax,
                                              double* __restrict__ coords,
                                              double* __restrict__ partial) {
    extern __shared__ double sv[];  // [w][rmax] then [4 * wp] staging
    const int r = imeta[1];
    for (int e = threadIdx.x; e < w * rmax; e += blockDim.x) sv[e] = vkeep[e];
    __syncthreads();
    const int row0 = static_cast<int>(static_cast<long long>(n) * blockIdx.x / gridDim.x);
    const int row1 = static_cast<int>(static_cast<long long>(n) * (blockIdx.x + 1) / gridDim.x);
    // per column: threads stride over the CTA's rows keeping a running
    // (value at max |u|, first index); merged in thread order below
    __shared__ double best_v[256];
    __shared__ int best_i[256];
    for (int c = 0; c < r; ++c) {
        double bv = 0.0;
        int bi = -1;
        for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < w; ++k) s += q[pidx(i, k, wp)] * sv[k * rmax + c];
            coords[static_cast<size_t>(i) * r + c] = s;
            if (bi < 0 || fabs(s) > fabs(bv)) {
                bv = s;
                bi = i;
            }
        }
        best_v[threadIdx.x] = bv;
        best_i[threadIdx.x] = bi;
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = 0.0;
            int ix = -1;
            for (int t = 0; t < blockDim.x; ++t) {
                const int ti = best_i[t];
                if (ti < 0) continue;
                const double tv = best_v[t];
                if (ix < 0 || fabs(tv) > fabs(v) || (fabs(tv) == fabs(v) && ti < ix)) {
                    v = tv;
                    ix = ti;
                }
            }
            partial[(static_cast<size_t>(blockIdx.x) * rmax + c) * 2 + 0] = v;
            partial[(static_cast<size_t>(blockIdx.x) * rmax + c) * 2 + 1] = static_cast<double>(ix);
        }
        __syncthreads();
    }
}

__global__ void k_lift_scale(int n, const int* __restrict__ imeta, int P, int rmax,
                             const double* __restrict__ kept_vals,
                             const double* __restrict__ partial, double* __restrict__ coords) {
    __shared__ double scale[kMaxWP];
    const int r = imeta[1];
    if (threadIdx.x < r) {
        const int c = threadIdx.x;
        double v = 0.0;
        long long ix = -1;
        for (int b = 0; b < P; ++b) {
            const double iv = partial[(static_cast<size_t>(b) * rmax + c) * 2 + 1];
            if (iv < 0) continue;
            const double tv = partial[(static_cast<size_t>(b) * rmax + c) * 2 + 0];
            const long long ti = static_cast<long long>(iv);
            if (ix < 0 || fabs(tv) > fabs(v) || (fabs(tv) == fabs(v) && ti < ix)) {
                v = tv;
                ix = ti;
            }
        }
        const double sg = (v < 0.0) ? -1.0 : 1.0;
        scale[c] = sg * sqrt(kept_vals[c]);
    }
    __syncthreads();
    const size_t total = static_cast<size_t>(n) * r;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x)
        coords[e] *= scale[e % r];
}

}  // namespace

void launch_evd(const double* b, int wp, int w, int rank, int requested_rank,
                const double* scalars, int fro_index, const EvdOut& o, cudaStream_t st) {
    const size_t smem = (static_cast<size_t>(w) * (w + 1) / 2 + static_cast<size_t>(w) * w) *
                        sizeof(double);
    static size_t set_for = 0;
    if (smem > 48 * 1024 && smem > set_for) {
        cudaFuncSetAttribute(k_evd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        set_for = smem;
    }
    k_evd<<<1, kEvdThreads, smem, st>>>(b, wp, w, rank, requested_rank, scalars, fro_index, o);
    count_launch();
}

void launch_lift(const double* q, size_t n, int wp, int w, const double* vkeep,
                 const double* kept_vals, const int* imeta, int rmax, double* coords,
                 double* partial, int sms, cudaStream_t st) {
    const int P = static_cast<int>(std::min<size_t>(static_cast<size_t>(sms) * 2,
                                                    std::max<size_t>(n / 64, 1)));
    const size_t smem = static_cast<size_t>(w) * rmax * sizeof(double);
    static size_t set_for = 0;
    if (smem > 48 * 1024 && smem > set_for) {
        cudaFuncSetAttribute(k_lift, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        set_for = smem;
    }
    k_lift<<<P, 256, smem, st>>>(q, static_cast<int>(n), wp, w, vkeep, imeta, rmax, coords,
                                 partial);
    k_lift_scale<<<std::min(P, 1024), 256, 0, st>>>(static_cast<int>(n), imeta, P, rmax,
                                                    kept_vals, partial, coords);
    count_launch(2);
}

}  // namespace dsb
