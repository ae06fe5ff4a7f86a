// K1 for a row shard of D (multi-GPU pass 0): a warp streams one full row at
// a time (16-byte loads, 8 in flight per lane), giving the row sum of d^2 in a
// fixed order, plus per-CTA sum d^4 / max |d|; and the cross-shard symmetry
// check max |d_ij - d_ji| on exchanged blocks (ref src/mds.cpp:21-41).
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

template <typename T>
__global__ void __launch_bounds__(256) k1_rows_kernel(const T* __restrict__ d, size_t ld,
                                                      size_t rows, size_t cols,
                                                      double* __restrict__ rowsum,
                                                      double* __restrict__ cta_stats,
                                                      int* __restrict__ row_exp) {
    __shared__ double red[2][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t gw = static_cast<size_t>(blockIdx.x) * 8 + warp;
    const size_t nw = static_cast<size_t>(gridDim.x) * 8;
    double sum4 = 0.0, maxabs = 0.0;
    for (size_t r = gw; r < rows; r += nw) {
        const T* row = d + r * ld;
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
            // smallest e with d^2 < 2^e over the row (int8 slice scale; K1 rule)
            const int be = static_cast<int>((hmx >> 20) & 0x7ffu);
            row_exp[r] = hmx == 0u ? -1100 : (be == 0 ? -1022 : be - 1022);
        }
    }
    sum4 = warp_sum(sum4);
    maxabs = warp_max(maxabs);
    if (lane == 0) {
        red[0][warp] = sum4;
        red[1][warp] = maxabs;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, m = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += red[0][w];
            m = fmax(m, red[1][w]);
        }
        cta_stats[blockIdx.x * 2 + 0] = a;
        cta_stats[blockIdx.x * 2 + 1] = m;
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

// Order-independent 64-bit fingerprint of a block of D: sum over its entries
// of a mix of (value bits, global row, global column), exact mod 2^64 (so
// the result does not depend on the launch shape). With swap the positions
// enter as (column, row): the fingerprint of a block equals that of the
// transposed partner block iff (up to a 2^-64 collision) they are transposes.
__device__ __forceinline__ unsigned long long fp_mix(unsigned long long v, unsigned long long i,
                                                     unsigned long long j) {
    unsigned long long x = v ^ (i * 0x9E3779B97F4A7C15ull) ^ (j * 0xC2B2AE3D27D4EB4Full);
    x ^= x >> 31;
    x *= 0x7FB5D329728EA185ull;
    x ^= x >> 27;
    x *= 0x81DADEF4BC2DD44Dull;
    x ^= x >> 33;
    return x;
}

template <typename T>
__global__ void __launch_bounds__(256) k_block_fingerprint(const T* __restrict__ d, size_t ld,
                                                           size_t m, size_t col0, size_t ncols,
                                                           size_t row0, int swap,
                                                           unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    const size_t total = m * ncols;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t r = e / ncols, c = e % ncols;
        const double v = static_cast<double>(d[r * ld + col0 + c]);
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
        const unsigned long long gi = row0 + r, gj = col0 + c;
        acc += swap ? fp_mix(bits, gj, gi) : fp_mix(bits, gi, gj);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

}  // namespace

int k1_rows_grid(size_t rows, int sms) {
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>((rows + 7) / 8, sms * 8)));
}

void launch_k1_rows(const void* d, DType dt, size_t ld, size_t rows, size_t cols, double* rowsum,
                    double* cta_stats, int grid, cudaStream_t st, int* row_exp) {
    if (dt == DType::F64)
        k1_rows_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(d), ld, rows, cols,
                                                     rowsum, cta_stats, row_exp);
    else
        k1_rows_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(d), ld, rows, cols,
                                                    rowsum, cta_stats, row_exp);
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

void launch_block_fingerprint(const void* d, DType dt, size_t ld, size_t m, size_t col0,
                              size_t ncols, size_t row0, bool swap, unsigned long long* out,
                              int sms, cudaStream_t st) {
    if (m == 0 || ncols == 0) return;
    const int grid = static_cast<int>(std::min<size_t>((m * ncols + 255) / 256, sms * 8));
    if (dt == DType::F64)
        k_block_fingerprint<double><<<grid, 256, 0, st>>>(static_cast<const double*>(d), ld, m, col0,
                                                          ncols, row0, swap ? 1 : 0, out);
    else
        k_block_fingerprint<float><<<grid, 256, 0, st>>>(static_cast<const float*>(d), ld, m, col0,
                                                         ncols, row0, swap ? 1 : 0, out);
    count_launch();
}

}  // namespace dsb
