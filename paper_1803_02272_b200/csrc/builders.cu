// Distance builders feeding the MDS path (no reference kernel exists):
//   K9 euclid  — exact Euclidean D from points, with the reference fixture's
//                operation order (ref tests/testdata.cpp:165-184): sequential
//                coordinate sum, explicit round-to-nearest sub/mul/add (no FMA
//                contraction), IEEE sqrt. (x_i - x_j)^2 == (x_j - x_i)^2 exactly,
//                so computing every (i, j) independently gives an exactly
//                symmetric D, bit-identical to the CPU formula. HBM-write bound.
//   K7 hamming — D_ij = h_ij / L, h = popcount of the nonzero 2-bit groups of
//                a_i XOR a_j over 2-bit packed reads (BASELINE config 5).
#include <algorithm>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace dsb {

namespace {

constexpr int kET = 64;  // output tile edge

template <bool F32>
__global__ void __launch_bounds__(256) k_euclid(const double* __restrict__ pts, int n, int dim,
                                                void* __restrict__ dout, size_t ld, int row0,
                                                int nrows) {
    extern __shared__ double sp[];
    const int ldp = dim + 1;  // odd stride: conflict-free column reads
    double* ri = sp;               // [64][ldp]
    double* cj = sp + kET * ldp;   // [64][ldp]
    const int i0 = row0 + blockIdx.y * kET, j0 = blockIdx.x * kET;
    const int iend = row0 + nrows;
    for (int e = threadIdx.x; e < kET * dim; e += blockDim.x) {
        const int r = e / dim, c = e % dim;
        ri[r * ldp + c] = (i0 + r < iend) ? pts[static_cast<size_t>(i0 + r) * dim + c] : 0.0;
        cj[r * ldp + c] = (j0 + r < n) ? pts[static_cast<size_t>(j0 + r) * dim + c] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int c = 0; c < dim; ++c) {
        double xi[4], xj[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xi[a] = ri[(ty + 16 * a) * ldp + c];
#pragma unroll
        for (int b = 0; b < 4; ++b) xj[b] = cj[(tx + 16 * b) * ldp + c];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double diff = __dsub_rn(xi[a], xj[b]);
                acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(diff, diff));
            }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int i = i0 + ty + 16 * a;
        if (i >= iend) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = j0 + tx + 16 * b;
            if (j >= n) continue;
            const double dist = (i == j) ? 0.0 : __dsqrt_rn(acc[a][b]);
            const size_t li = static_cast<size_t>(i - row0);
            if (F32)
                static_cast<float*>(dout)[li * ld + j] = __double2float_rn(dist);
            else
                static_cast<double*>(dout)[li * ld + j] = dist;
        }
    }
}

__global__ void __launch_bounds__(256) k_hamming(const unsigned long long* __restrict__ packed,
                                                 int count, int words, int length,
                                                 double* __restrict__ d, size_t ld,
                                                 uint32_t* __restrict__ counts) {
    extern __shared__ unsigned long long sw[];
    unsigned long long* ra = sw;                 // [64][words]
    unsigned long long* rb = sw + kET * words;   // [64][words]
    const int i0 = blockIdx.y * kET, j0 = blockIdx.x * kET;
    for (int e = threadIdx.x; e < kET * words; e += blockDim.x) {
        const int r = e / words, c = e % words;
        ra[e] = (i0 + r < count) ? packed[static_cast<size_t>(i0 + r) * words + c] : 0ull;
        rb[e] = (j0 + r < count) ? packed[static_cast<size_t>(j0 + r) * words + c] : 0ull;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    unsigned h[4][4] = {};
    for (int c = 0; c < words; ++c) {
        unsigned long long a[4], b[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k] = ra[(ty + 16 * k) * words + c];
            b[k] = rb[(tx + 16 * k) * words + c];
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const unsigned long long z = a[x] ^ b[y];
                h[x][y] += static_cast<unsigned>(__popcll((z | (z >> 1)) & 0x5555555555555555ull));
            }
    }
    const double L = static_cast<double>(length);
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const int i = i0 + ty + 16 * x;
        if (i >= count) continue;
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int j = j0 + tx + 16 * y;
            if (j >= count) continue;
            if (d) d[static_cast<size_t>(i) * ld + j] = static_cast<double>(h[x][y]) / L;
            if (counts) counts[static_cast<size_t>(i) * count + j] = h[x][y];
        }
    }
}

}  // namespace

void launch_euclid(const double* pts, size_t n, int dim, void* d, DType dt, size_t ld,
                   cudaStream_t st) {
    launch_euclid_rows(pts, n, dim, d, dt, ld, 0, n, st);
}

void launch_euclid_rows(const double* pts, size_t n, int dim, void* d, DType dt, size_t ld,
                        size_t row0, size_t nrows, cudaStream_t st) {
    if (nrows == 0) return;
    const size_t smem = 2 * static_cast<size_t>(kET) * (dim + 1) * sizeof(double);
    dim3 grid(static_cast<unsigned>((n + kET - 1) / kET), static_cast<unsigned>((nrows + kET - 1) / kET));
    if (dt == DType::F32) {
        allow_dyn_smem(reinterpret_cast<const void*>(k_euclid<true>));
        k_euclid<true><<<grid, 256, smem, st>>>(pts, static_cast<int>(n), dim, d, ld,
                                                static_cast<int>(row0), static_cast<int>(nrows));
    } else {
        allow_dyn_smem(reinterpret_cast<const void*>(k_euclid<false>));
        k_euclid<false><<<grid, 256, smem, st>>>(pts, static_cast<int>(n), dim, d, ld,
                                                 static_cast<int>(row0), static_cast<int>(nrows));
    }
    count_launch();
}

void launch_hamming(const unsigned long long* packed, size_t count, int words, int length,
                    double* d, size_t ld, uint32_t* counts, cudaStream_t st) {
    const int nb = static_cast<int>((count + kET - 1) / kET);
    const size_t smem = 2 * static_cast<size_t>(kET) * words * sizeof(unsigned long long);
    allow_dyn_smem(reinterpret_cast<const void*>(k_hamming));
    dim3 grid(nb, nb);
    k_hamming<<<grid, 256, smem, st>>>(packed, static_cast<int>(count), words, length, d, ld,
                                       counts);
    count_launch();
}

}  // namespace dsb
