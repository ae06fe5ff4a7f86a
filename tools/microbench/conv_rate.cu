// Throughput of the int8 slice product's digit conversion (k2i_product.cu
// converters) without memory traffic: each thread turns 8 fp64 d values per
// iteration into the 7 byte planes of the 56-bit fixed-point d^2, with
//   mode 0: d*d*sc -> F2I.U64.F64 (the product kernel's path)
//   mode 1: d*d*sc -> mantissa shift on the integer pipe (no F2I)
//   mode 2: d*d -> F2I.U64.F64 only (the conversion instruction's rate)
//   mode 3: byte-plane packing only (PRMT)
// 16 warps per SM (the converter count). Prints cycles per element per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/conv_rate \
//        tools/microbench/conv_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned long long fix56_int(double v) {
    // floor(v) for 0 <= v < 2^56 from the bits: mantissa shifted by the exponent
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const int e = static_cast<int>((b >> 52) & 0x7FF) - 1075;  // v = m * 2^e, m 53-bit
    const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | (1ull << 52);
    if (e >= 0) return m << e;
    if (e <= -53) return 0ull;
    return m >> (-e);
}

template <int MODE>
__global__ void k_conv(int iters, double sc, uint32_t* sink, unsigned long long* cycles) {
    double d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = 1.0 + 1e-3 * (threadIdx.x * 8 + j);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            unsigned long long m;
            if (MODE == 0) m = __double2ull_rz((d[j] * d[j]) * sc);
            else if (MODE == 1) m = fix56_int((d[j] * d[j]) * sc);
            else if (MODE == 2) m = __double2ull_rz(d[j]);
            else m = static_cast<unsigned long long>(__double_as_longlong(d[j]));
            lo[j] = static_cast<uint32_t>(m);
            hi[j] = static_cast<uint32_t>(m >> 32);
        }
        uint32_t w[7][2];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int e = 4 * g;
            const uint32_t p45 = __byte_perm(lo[e], lo[e + 1], 0x6273);
            const uint32_t q45 = __byte_perm(lo[e + 2], lo[e + 3], 0x6273);
            w[3][g] = __byte_perm(p45, q45, 0x5410);
            w[4][g] = __byte_perm(p45, q45, 0x7632);
            const uint32_t p67 = __byte_perm(lo[e], lo[e + 1], 0x4051);
            const uint32_t q67 = __byte_perm(lo[e + 2], lo[e + 3], 0x4051);
            w[5][g] = __byte_perm(p67, q67, 0x5410);
            w[6][g] = __byte_perm(p67, q67, 0x7632);
            const uint32_t p12 = __byte_perm(hi[e], hi[e + 1], 0x5162);
            const uint32_t q12 = __byte_perm(hi[e + 2], hi[e + 3], 0x5162);
            w[0][g] = __byte_perm(p12, q12, 0x5410);
            w[1][g] = __byte_perm(p12, q12, 0x7632);
            const uint32_t p3 = __byte_perm(hi[e], hi[e + 1], 0x0040);
            const uint32_t q3 = __byte_perm(hi[e + 2], hi[e + 3], 0x0040);
            w[2][g] = __byte_perm(p3, q3, 0x5410);
        }
#pragma unroll
        for (int t = 0; t < 7; ++t) acc += w[t][0] ^ (w[t][1] << 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = __longlong_as_double(__double_as_longlong(d[j]) + (acc & 1));
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = c1 - c0;
}

template <int MODE>
void run(const char* name, int sms, uint32_t* sink, unsigned long long* dc) {
    const int iters = 2000, threads = 512;
    k_conv<MODE><<<sms, threads>>>(10, 0x1p10, sink, dc);
    k_conv<MODE><<<sms, threads>>>(iters, 0x1p10, sink, dc);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    const double per_elem = static_cast<double>(cyc) / iters / (threads * 8);
    printf("%-48s %s  %.4f cycles/element/SM  (%.0f cycles per 128x32 tile)\n", name,
           err == cudaSuccess ? "ok " : cudaGetErrorString(err), per_elem, per_elem * 4096);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink;
    unsigned long long* dc;
    cudaMalloc(&sink, sms * 512 * 4);
    cudaMalloc(&dc, 8);
    run<0>("DMUL x2 + F2I.U64.F64 + byte planes", sms, sink, dc);
    run<1>("DMUL x2 + integer mantissa shift + byte planes", sms, sink, dc);
    run<2>("F2I.U64.F64 + byte planes", sms, sink, dc);
    run<3>("byte planes only", sms, sink, dc);
    return 0;
}
