// reconstruction_error (ref src/mds.cpp:126-150): sqrt(sum_ij (g_ij - x_i . x_j)^2)
// — the diagnostic n^2 r pass of SURVEY §8f row 4, on the device.
//
// A lazy gram is evaluated on the fly with the reference's expression and
// operand choice, g_ij = -1/2 (d d - r_i - r_j + g_bar) from the upper
// triangle d_ij (ref mds.cpp:43-58, mirrored). Both g and x_i . x_j are
// symmetric in (i, j) bit for bit (mirrored d; the dot is accumulated over c
// in the same order either way), so only the upper 64 x 64 tiles I <= J of D
// are read — half the bytes of the reference's full scan — and the strictly
// upper tiles count twice. Explicit matrices are scanned in full (their g_ij
// is the stored entry). One CTA per tile: the two 64 x r coordinate blocks
// are staged in shared memory, each thread owns one column j and 16 rows,
// fp64 FMAs for the dots (2 n^2 r flops; FP64-pipe / HBM bound), per-CTA
// partial sums reduced in a fixed order.
#include <algorithm>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace dsb {

namespace {

constexpr int kRT = 64;  // tile edge

__device__ __forceinline__ void upper_pair(long long p, int nbt, int& I, int& J) {
    // p -> (I, J), I <= J, row-major over the upper triangle of tiles
    double nf = nbt + 0.5;
    int i = static_cast<int>(nf - sqrt(nf * nf - 2.0 * static_cast<double>(p)));
    if (i < 0) i = 0;
    if (i > nbt - 1) i = nbt - 1;
    auto off = [&](long long r) { return r * nbt - r * (r - 1) / 2; };
    while (i > 0 && off(i) > p) --i;
    while (i + 1 < nbt && off(i + 1) <= p) ++i;
    I = i;
    J = static_cast<int>(i + (p - off(i)));
}

template <typename T, bool LAZY>
__global__ void __launch_bounds__(256) k_recon(const T* __restrict__ d, size_t ld, int n,
                                               const double* __restrict__ row_mean,
                                               const double* __restrict__ scalars,
                                               const double* __restrict__ x, int r,
                                               double* __restrict__ partial) {
    extern __shared__ double xs[];  // [2][kRT][r + 1]
    __shared__ double red[8];
    const int nbt = (n + kRT - 1) / kRT;
    int I, J;
    if (LAZY) {
        upper_pair(blockIdx.x, nbt, I, J);
    } else {
        I = static_cast<int>(blockIdx.x / nbt);
        J = static_cast<int>(blockIdx.x % nbt);
    }
    const int rp = r + 1;
    double* xi = xs;
    double* xj = xs + kRT * rp;
    for (int e = threadIdx.x; e < kRT * r; e += blockDim.x) {
        const int a = e / r, c = e % r;
        const int gi = I * kRT + a, gj = J * kRT + a;
        xi[a * rp + c] = gi < n ? x[static_cast<size_t>(gi) * r + c] : 0.0;
        xj[a * rp + c] = gj < n ? x[static_cast<size_t>(gj) * r + c] : 0.0;
    }
    __syncthreads();
    const double grand = LAZY ? scalars[S_GRAND] : 0.0;
    const int tx = threadIdx.x & (kRT - 1), ty = threadIdx.x / kRT;
    const int j = J * kRT + tx;
    double acc = 0.0;
    if (j < n) {
        const double rj = LAZY ? row_mean[j] : 0.0;
        for (int a = ty; a < kRT; a += 4) {
            const int i = I * kRT + a;
            if (i >= n) break;
            double g;
            if (LAZY) {
                // upper-triangle d_ij (mirrored below the diagonal)
                const double dij = (i <= j) ? static_cast<double>(d[static_cast<size_t>(i) * ld + j])
                                            : static_cast<double>(d[static_cast<size_t>(j) * ld + i]);
                g = -0.5 * (dij * dij - row_mean[i] - rj + grand);
            } else {
                g = static_cast<double>(d[static_cast<size_t>(i) * ld + j]);
            }
            double dot = 0.0;
            for (int c = 0; c < r; ++c) dot += xi[a * rp + c] * xj[tx * rp + c];
            const double diff = g - dot;
            acc += diff * diff;
        }
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += red[w];
        partial[blockIdx.x] = (LAZY && I != J) ? 2.0 * s : s;
    }
}

}  // namespace

size_t recon_blocks(size_t n, bool lazy) {
    const size_t nbt = (n + kRT - 1) / kRT;
    return lazy ? nbt * (nbt + 1) / 2 : nbt * nbt;
}

void launch_recon(const void* d, DType dt, size_t ld, size_t n, bool lazy, const double* row_mean,
                  const double* scalars, const double* x, int r, double* partial, double* out,
                  cudaStream_t st) {
    const size_t nblk = recon_blocks(n, lazy);
    const size_t smem = static_cast<size_t>(2) * kRT * (r + 1) * sizeof(double);
    const int ni = static_cast<int>(n);
#define DSB_RECON(T, L)                                                                        \
    do {                                                                                       \
        allow_dyn_smem(reinterpret_cast<const void*>(k_recon<T, L>));                          \
        k_recon<T, L><<<static_cast<unsigned>(nblk), 256, smem, st>>>(                         \
            static_cast<const T*>(d), ld, ni, row_mean, scalars, x, r, partial);               \
    } while (0)
    if (dt == DType::F64) {
        if (lazy) DSB_RECON(double, true); else DSB_RECON(double, false);
    } else {
        if (lazy) DSB_RECON(float, true); else DSB_RECON(float, false);
    }
#undef DSB_RECON
    launch_sum_fixed(partial, nblk, out, st);
    count_launch(1);
}

}  // namespace dsb
