// Validation of the tcgen05 kind::i8 path used by the K2 int8 slice product:
// one CTA, A = 7 u8 digit tiles (128 x 32), B = 7 s8 digit tiles (N x 32),
// per digit t one MMA against the concatenation of B digits 1..8-t written to
// TMEM columns (t-1)*N.. (the diagonal accumulators), K steps accumulated.
// Compares every TMEM value against a CPU evaluation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1803_02272_b200/csrc umma_i8_test.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace dsb;

constexpr int M = 128, KSTEP = 32, T = 7;

template <int N>
__global__ void k_test(const uint8_t* __restrict__ A, const int8_t* __restrict__ B, int ksteps,
                       int32_t* __restrict__ out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned char* sa = sm;                       // [T][M x 32]
    unsigned char* sb = sm + T * M * KSTEP;       // [T][N x 32]
    constexpr int NCOL = (T * N <= 256) ? 256 : 512;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tbase, NCOL);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    uint32_t phase = 0;
    for (int ks = 0; ks < ksteps; ++ks) {
        // stage digits (global row-major [t][r][k]) into the canonical layout
        for (int e = threadIdx.x; e < T * M * KSTEP; e += blockDim.x) {
            const int t = e / (M * KSTEP), r = (e / KSTEP) % M, k = e % KSTEP;
            sa[t * M * KSTEP + umma_tile_off(r, k)] =
                A[(static_cast<size_t>(t) * M + r) * (ksteps * KSTEP) + ks * KSTEP + k];
        }
        for (int e = threadIdx.x; e < T * N * KSTEP; e += blockDim.x) {
            const int u = e / (N * KSTEP), c = (e / KSTEP) % N, k = e % KSTEP;
            sb[u * N * KSTEP + umma_tile_off(c, k)] = static_cast<unsigned char>(
                B[(static_cast<size_t>(u) * N + c) * (ksteps * KSTEP) + ks * KSTEP + k]);
        }
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
            tc_fence_after();
            for (int t = 1; t <= T; ++t) {
                // u = 1 .. 8 - t, in chunks of at most 256 columns
                const int umax = 8 - t;
                const int per = 256 / N;
                for (int u0 = 1; u0 <= umax; u0 += per) {
                    const int nu = (umax - u0 + 1 < per) ? (umax - u0 + 1) : per;
                    const uint64_t ad =
                        umma_desc_k_interleave(smem_u32(sa + (t - 1) * M * KSTEP));
                    const uint64_t bd =
                        umma_desc_k_interleave(smem_u32(sb + (u0 - 1) * N * KSTEP));
                    const int acc = (ks > 0 || t > 1) ? 1 : 0;
                    umma_i8(tmem + (t + u0 - 2) * N, ad, bd, umma_idesc_i8(nu * N, false, true),
                            acc);
                }
            }
            umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        __syncthreads();
    }
    // read back: warps 0..3 own lanes 0..127
    if (warp < 4) {
        const int row = warp * 32 + (threadIdx.x & 31);
        for (int c0 = 0; c0 < T * N; c0 += 32) {
            int32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j)
                if (c0 + j < T * N) out[row * (T * N) + c0 + j] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, NCOL);
}

template <int N>
__global__ void k_test_ts(const uint8_t* __restrict__ A, const int8_t* __restrict__ B, int ksteps,
                          int32_t* __restrict__ out);

template <int N>
int run(int ksteps, bool ts = false) {
    const int K = ksteps * KSTEP;
    std::vector<uint8_t> A(static_cast<size_t>(T) * M * K);
    std::vector<int8_t> B(static_cast<size_t>(T) * N * K);
    srand(1234 + N);
    for (auto& a : A) a = static_cast<uint8_t>(rand() & 255);
    for (auto& b : B) b = static_cast<int8_t>((rand() & 255) - 128);
    uint8_t* dA;
    int8_t* dB;
    int32_t* dO;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dO, sizeof(int32_t) * M * T * N);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, sizeof(int32_t) * M * T * N);
    const int smem = T * M * KSTEP + T * N * KSTEP;
    if (ts) {
        cudaFuncSetAttribute(k_test_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_test_ts<N><<<1, 256, smem>>>(dA, dB, ksteps, dO);
    } else {
        cudaFuncSetAttribute(k_test<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_test<N><<<1, 256, smem>>>(dA, dB, ksteps, dO);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e));
        return 1;
    }
    std::vector<int32_t> O(static_cast<size_t>(M) * T * N);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int r = 0; r < M; ++r)
        for (int d = 2; d <= 8; ++d)
            for (int c = 0; c < N; ++c) {
                long long want = 0;
                for (int t = 1; t <= T; ++t) {
                    const int u = d - t;
                    if (u < 1 || u > T) continue;
                    for (int k = 0; k < K; ++k)
                        want += static_cast<long long>(A[(static_cast<size_t>(t - 1) * M + r) * K + k]) *
                                B[(static_cast<size_t>(u - 1) * N + c) * K + k];
                }
                const int32_t got = O[r * (T * N) + (d - 2) * N + c];
                if (got != static_cast<int32_t>(want)) {
                    if (bad < 5)
                        printf("  mismatch r=%d d=%d c=%d got %d want %lld\n", r, d, c, got, want);
                    ++bad;
                }
            }
    printf("%s N=%d ksteps=%d: %s (%ld mismatches)\n", ts ? "TS" : "SS", N, ksteps,
           bad ? "FAIL" : "OK", bad);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
    return bad ? 1 : 0;
}

// Same product with the A digits in tensor memory (written by tcgen05.st,
// row r = lane r, byte k of the 32-byte K slice in column k/4).
template <int N>
__global__ void k_test_ts(const uint8_t* __restrict__ A, const int8_t* __restrict__ B, int ksteps,
                          int32_t* __restrict__ out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned char* sb = sm;  // [T][N x 32]
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tbase, 512);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t ta = tmem + 256;  // A digits: 7 x 8 columns
    uint32_t phase = 0;
    for (int ks = 0; ks < ksteps; ++ks) {
        if (warp < 4) {
            const int r = threadIdx.x;
            for (int t = 0; t < T; ++t)
                for (int c = 0; c < 8; c += 2) {
                    uint32_t w[2];
                    for (int h = 0; h < 2; ++h) {
                        uint32_t v = 0;
                        for (int b = 0; b < 4; ++b)
                            v |= static_cast<uint32_t>(
                                     A[(static_cast<size_t>(t) * M + r) * (ksteps * KSTEP) +
                                       ks * KSTEP + (c + h) * 4 + b])
                                 << (8 * b);
                        w[h] = v;
                    }
                    tmem_st2(ta + (static_cast<uint32_t>(warp * 32) << 16) + t * 8 + c, w[0], w[1]);
                }
            tmem_st_wait();
        }
        for (int e = threadIdx.x; e < T * N * KSTEP; e += blockDim.x) {
            const int u = e / (N * KSTEP), c = (e / KSTEP) % N, k = e % KSTEP;
            sb[u * N * KSTEP + umma_tile_off(c, k)] = static_cast<unsigned char>(
                B[(static_cast<size_t>(u) * N + c) * (ksteps * KSTEP) + ks * KSTEP + k]);
        }
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();
        if (threadIdx.x == 0) {
            tc_fence_after();
            for (int t = 1; t <= T; ++t) {
                const int umax = 8 - t;
                const int per = 256 / N;
                for (int u0 = 1; u0 <= umax; u0 += per) {
                    const int nu = (umax - u0 + 1 < per) ? (umax - u0 + 1) : per;
                    const uint64_t bd = umma_desc_k_interleave(smem_u32(sb + (u0 - 1) * N * KSTEP));
                    umma_i8_ts(tmem + (t + u0 - 2) * N, ta + (t - 1) * 8, bd,
                               umma_idesc_i8(nu * N, false, true), (ks > 0 || t > 1) ? 1 : 0);
                }
            }
            umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        __syncthreads();
    }
    if (warp < 4) {
        const int row = warp * 32 + (threadIdx.x & 31);
        for (int c0 = 0; c0 < T * N; c0 += 32) {
            int32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j)
                if (c0 + j < T * N) out[row * (T * N) + c0 + j] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    int rc = 0;
    rc |= run<32>(1);
    rc |= run<32>(3);
    rc |= run<64>(2);
    rc |= run<16>(2);
    rc |= run<32>(1, true);
    rc |= run<32>(3, true);
    return rc;
}
