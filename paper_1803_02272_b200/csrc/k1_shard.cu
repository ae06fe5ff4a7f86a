// K1 for a row shard of D (multi-GPU pass 0): a warp streams one full row at
// a time (16-byte loads, 8 in flight per lane), giving the row sum of d^2 in a
// fixed order, the row mean and int8 row exponent, per-CTA sum d^4 / max |d|
// / admission ratio, and the shard's antisymmetric symmetry fingerprint
// (SymFp below) — one read of the shard. The exact max |d_ij - d_ji| on
// exchanged blocks (k_asym_block) runs only when the all-reduced fingerprint
// is nonzero (ref src/mds.cpp:21-41).
#include <algorithm>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace dsb {

namespace {

template <typename T>
struct V2;
template <>
struct V2<double> {
    using type = double2;
};
template <>
struct V2<float> {
    using type = float2;
};

// Antisymmetric fingerprint of D: sum over (i, j) of sgn(j - i) h(d_ij, {i, j})
// where h mixes the value bits with the UNORDERED position through a
// bijection of each 32-bit half of the value (two independent 32-bit sums,
// `lo` and `hi`). Over a whole matrix both sums are zero (mod 2^32) iff every
// mirrored pair has identical bits: one differing pair is always detected,
// several cancel only by a ~2^-64 accident. Each rank sums over its own rows
// inside the K1 pass (32-bit integer ops only, ~12 per element, so the pass
// stays HBM-bound) and one all-reduce decides the symmetry of the whole
// sharded matrix.
struct SymFp {
    uint32_t lo = 0, hi = 0;
    __device__ __forceinline__ void add(double v, uint32_t i, uint32_t j) {
        const uint32_t key = j > i ? i * 0x9E3779B1u + j * 0x85EBCA77u
                                   : j * 0x9E3779B1u + i * 0x85EBCA77u;
        const uint32_t s = j > i ? 1u : (j < i ? 0xFFFFFFFFu : 0u);
        const uint32_t vl = static_cast<uint32_t>(__double2loint(v));
        const uint32_t vh = static_cast<uint32_t>(__double2hiint(v));
        lo += ((vl ^ key) * 0xC2B2AE3Du) * s;
        hi += ((vh ^ key ^ 0x165667B1u) * 0x27D4EB2Fu) * s;
    }
};

template <typename T>
__global__ void __launch_bounds__(256) k1_rows_kernel(const T* __restrict__ d, size_t ld,
                                                      size_t rows, size_t cols, size_t row0,
                                                      double* __restrict__ rowsum,
                                                      double* __restrict__ row_mean,
                                                      double* __restrict__ cta_stats,
                                                      int* __restrict__ row_exp,
                                                      unsigned long long* __restrict__ fp_out) {
    __shared__ double red[3][8];
    __shared__ uint32_t fred[2][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t gw = static_cast<size_t>(blockIdx.x) * 8 + warp;
    const size_t nw = static_cast<size_t>(gridDim.x) * 8;
    double sum4 = 0.0, maxabs = 0.0, ratio = 0.0;
    const double nf = static_cast<double>(cols);
    SymFp fp;
    for (size_t r = gw; r < rows; r += nw) {
        const T* row = d + r * ld;
        const uint32_t gi = static_cast<uint32_t>(row0 + r);
        double s = 0.0;
        uint32_t hmx = 0u;  // max over the row of the high word of d^2 (>= 0)
        size_t c = 2 * lane;
        // main body: 8 independent 2-element loads per lane per iteration
        for (; c + 448 + 1 < cols; c += 512) {
            typename V2<T>::type v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = __ldg(reinterpret_cast<const typename V2<T>::type*>(row + c + 64 * u));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double a0 = v[u].x, a1 = v[u].y;
                const uint32_t j = static_cast<uint32_t>(c + 64 * u);
                fp.add(a0, gi, j);
                fp.add(a1, gi, j + 1);
                const double s0 = a0 * a0, s1 = a1 * a1;
                s += s0 + s1;
                sum4 += s0 * s0 + s1 * s1;
                // NaN-ignoring select, as the reference's std::max scan
                const double m01 = fabs(a1) > fabs(a0) ? fabs(a1) : fabs(a0);
                maxabs = m01 > maxabs ? m01 : maxabs;
                hmx = max(hmx, max(static_cast<uint32_t>(__double2hiint(s0)),
                                   static_cast<uint32_t>(__double2hiint(s1))));
            }
        }
        for (; c < cols; c += 64) {
            const double a0 = static_cast<double>(row[c]);
            const double a1 = (c + 1 < cols) ? static_cast<double>(row[c + 1]) : 0.0;
            fp.add(a0, gi, static_cast<uint32_t>(c));
            if (c + 1 < cols) fp.add(a1, gi, static_cast<uint32_t>(c + 1));
            const double s0 = a0 * a0, s1 = a1 * a1;
            s += s0 + s1;
            sum4 += s0 * s0 + s1 * s1;
            const double m01 = fabs(a1) > fabs(a0) ? fabs(a1) : fabs(a0);
            maxabs = m01 > maxabs ? m01 : maxabs;
            hmx = max(hmx, max(static_cast<uint32_t>(__double2hiint(s0)),
                               static_cast<uint32_t>(__double2hiint(s1))));
        }
        s = warp_sum(s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hmx = max(hmx, __shfl_xor_sync(0xffffffffu, hmx, o));
        if (lane == 0) {
            rowsum[r] = s;
            const double rm = s / nf;
            if (row_mean) row_mean[r] = rm;
            // smallest e with d^2 < 2^e over the row (int8 slice scale; K1 rule)
            const int be = static_cast<int>((hmx >> 20) & 0x7ffu);
            const int e = hmx == 0u ? -1100 : (be == 0 ? -1022 : be - 1022);
            row_exp[r] = e;
            // int8 admission bound 2^e_i / r_i (K1 rule)
            if (e > -1100) ratio = fmax(ratio, rm > 0.0 ? ldexp(1.0, e) / rm : 1e300);
        }
    }
    sum4 = warp_sum(sum4);
    maxabs = warp_max(maxabs);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        fp.lo += __shfl_xor_sync(0xffffffffu, fp.lo, o);
        fp.hi += __shfl_xor_sync(0xffffffffu, fp.hi, o);
    }
    if (lane == 0) {
        red[0][warp] = sum4;
        red[1][warp] = maxabs;
        red[2][warp] = ratio;
        fred[0][warp] = fp.lo;
        fred[1][warp] = fp.hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, m = 0.0, q = 0.0;
        uint32_t fl = 0, fh = 0;
        for (int w = 0; w < 8; ++w) {
            a += red[0][w];
            m = fmax(m, red[1][w]);
            q = fmax(q, red[2][w]);
            fl += fred[0][w];
            fh += fred[1][w];
        }
        cta_stats[blockIdx.x * 3 + 0] = a;
        cta_stats[blockIdx.x * 3 + 1] = m;
        cta_stats[blockIdx.x * 3 + 2] = q;
        // each half as a 64-bit addend (< 2^32): the sums stay exact, the
        // verdict reads them mod 2^32
        if (fp_out) {
            if (fl) atomicAdd(fp_out, static_cast<unsigned long long>(fl));
            if (fh) atomicAdd(fp_out + 1, static_cast<unsigned long long>(fh));
        }
    }
}

// Fold of the K1-rows CTA partials, fixed order: red[0] = sum d^4,
// red[1] = max |d|, red[3] = max_i 2^e_i / r_i (int8 admission bound).
__global__ void __launch_bounds__(32) k_shard_fold(const double* __restrict__ cta, int grid,
                                                   double* __restrict__ red) {
    const int lane = threadIdx.x;
    double a = 0.0, m = 0.0, q = 0.0;
    for (int b = lane; b < grid; b += 32) {  // lane-strided, then a fixed tree
        a += cta[3 * b];
        m = fmax(m, cta[3 * b + 1]);
        q = fmax(q, cta[3 * b + 2]);
    }
    a = warp_sum(a);
    m = warp_max(m);
    q = warp_max(q);
    if (lane == 0) {
        red[0] = a;
        red[1] = m;
        red[3] = q;
    }
}

// Grand mean terms over the full (all-gathered) row means in a fixed order
// independent of the rank count: sums[0] = sum r_i, sums[1] = sum r_i^2.
__global__ void __launch_bounds__(1024) k_rowmean_sums(const double* __restrict__ r, size_t n,
                                                       double* __restrict__ sums) {
    __shared__ double a[1024], b[1024];
    double s = 0.0, s2 = 0.0;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
        s += r[i];
        s2 += r[i] * r[i];
    }
    a[threadIdx.x] = s;
    b[threadIdx.x] = s2;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (static_cast<int>(threadIdx.x) < o) {
            a[threadIdx.x] += a[threadIdx.x + o];
            b[threadIdx.x] += b[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sums[0] = a[0];
        sums[1] = b[0];
    }
}

// 32x32 tiles: A tile read row-wise, B tile read row-wise into smem and
// compared transposed
template <typename T>
__global__ void __launch_bounds__(256) k_asym_block(const T* __restrict__ a, size_t lda,
                                                    const T* __restrict__ b, size_t ldb, size_t m,
                                                    size_t p, unsigned long long* __restrict__ out) {
    __shared__ double bt[32][33];
    const size_t i0 = static_cast<size_t>(blockIdx.y) * 32, j0 = static_cast<size_t>(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    // B rows j0.., cols i0..
    for (int r = ty; r < 32; r += 8) {
        const size_t j = j0 + r, i = i0 + tx;
        bt[r][tx] = (j < p && i < m) ? static_cast<double>(b[j * ldb + i]) : 0.0;
    }
    __syncthreads();
    double mx = 0.0;
    for (int r = ty; r < 32; r += 8) {
        const size_t i = i0 + r, j = j0 + tx;
        if (i < m && j < p) mx = fmax(mx, fabs(static_cast<double>(a[i * lda + j]) - bt[tx][r]));
    }
    mx = warp_max(mx);
    if (tx == 0 && mx > 0.0) atomicMax(out, __double_as_longlong(mx));
}

}  // namespace

int k1_rows_grid(size_t rows, int sms) {
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>((rows + 7) / 8, sms * 8)));
}

void launch_k1_rows(const void* d, DType dt, size_t ld, size_t rows, size_t cols, size_t row0,
                    double* rowsum, double* row_mean, double* cta_stats, int grid,
                    cudaStream_t st, int* row_exp, unsigned long long* sym_fp) {
    if (dt == DType::F64)
        k1_rows_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(d), ld, rows, cols,
                                                     row0, rowsum, row_mean, cta_stats, row_exp,
                                                     sym_fp);
    else
        k1_rows_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(d), ld, rows, cols,
                                                    row0, rowsum, row_mean, cta_stats, row_exp,
                                                    sym_fp);
    count_launch();
}

void launch_shard_fold(const double* cta, int grid, double* red, cudaStream_t st) {
    k_shard_fold<<<1, 32, 0, st>>>(cta, grid, red);
    count_launch();
}

void launch_rowmean_sums(const double* row_mean, size_t n, double* sums, cudaStream_t st) {
    k_rowmean_sums<<<1, 1024, 0, st>>>(row_mean, n, sums);
    count_launch();
}

void launch_asym_block(const void* a, size_t lda, const void* b, size_t ldb, DType dt, size_t m,
                       size_t p, double* out, cudaStream_t st) {
    if (m == 0 || p == 0) return;
    dim3 grid(static_cast<unsigned>((p + 31) / 32), static_cast<unsigned>((m + 31) / 32));
    auto* o = reinterpret_cast<unsigned long long*>(out);
    if (dt == DType::F64)
        k_asym_block<double><<<grid, 256, 0, st>>>(static_cast<const double*>(a), lda,
                                                   static_cast<const double*>(b), ldb, m, p, o);
    else
        k_asym_block<float><<<grid, 256, 0, st>>>(static_cast<const float*>(a), lda,
                                                  static_cast<const float*>(b), ldb, m, p, o);
    count_launch();
}


}  // namespace dsb
