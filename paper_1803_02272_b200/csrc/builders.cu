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
#include <type_traits>

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

// Reads -> two bit planes on the device (A=00, C=01, G=10, T=11): lo[r][w]
// bit t = code bit 0 of base 32 w + t, hi[r][w] its bit 1; positions past
// the read length are 0 in every read. One thread per 32-base word; the
// smallest linear index of a non-ACGT byte goes to *bad (atomicMin).
__global__ void __launch_bounds__(256) k_pack_reads(const unsigned char* __restrict__ reads,
                                                    long long count, int length, int words,
                                                    uint32_t* __restrict__ lo,
                                                    uint32_t* __restrict__ hi,
                                                    unsigned long long* __restrict__ bad) {
    const long long total = count * words;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = e / words;
        const int w = static_cast<int>(e % words);
        const unsigned char* src = reads + r * length + w * 32;
        const int nb = min(32, length - w * 32);
        uint32_t l = 0, h = 0;
        for (int t = 0; t < nb; ++t) {
            const unsigned char ch = src[t];
            uint32_t code;
            switch (ch) {
                case 'A': code = 0; break;
                case 'C': code = 1; break;
                case 'G': code = 2; break;
                case 'T': code = 3; break;
                default:
                    atomicMin(bad, static_cast<unsigned long long>(r * length + w * 32 + t));
                    code = 0;
            }
            l |= (code & 1u) << t;
            h |= (code >> 1) << t;
        }
        lo[e] = l;
        hi[e] = h;
    }
}

// K7: Hamming counts h_ij = popcount((lo_i ^ lo_j) | (hi_i ^ hi_j)) over the
// 32-base words (two LOP3 + POPC + add per 32 positions). 64x64 output tile
// per CTA of 256 threads, 4x4 outputs per thread from planes staged in
// shared memory (measured at n = 50k: 7.7 ms; 4x8 outputs on 128 threads
// 8.6 ms, 128x128 tiles with 8x8 per thread 14.9 ms — register-limited to
// one CTA per SM). SYM (a full matrix): only tiles I <= J
// are computed and the mirror tile is written through a shared-memory
// transpose, so the popcount work halves and both writes stay coalesced;
// otherwise (a row shard) every tile of the row band. OUT = double writes
// D = h / L, OUT = uint32_t writes h.
constexpr int kHT = 64;  // Hamming output tile edge
constexpr int kHThreads = 256;
__device__ __forceinline__ void tile_pair_of(long long p, int nbt, int& I, int& J) {
    const double nf = static_cast<double>(nbt);
    double g = (2.0 * nf + 1.0 - sqrt((2.0 * nf + 1.0) * (2.0 * nf + 1.0) - 8.0 * (double)p)) / 2.0;
    long long i = g <= 0.0 ? 0 : static_cast<long long>(g);
    if (i > nbt - 1) i = nbt - 1;
    auto start = [&](long long r) { return r * nbt - r * (r - 1) / 2; };
    while (i > 0 && start(i) > p) --i;
    while (i + 1 < nbt && start(i + 1) <= p) ++i;
    I = static_cast<int>(i);
    J = static_cast<int>(i + (p - start(i)));
}

template <typename OUT, bool SYM>
__global__ void __launch_bounds__(kHThreads) k_hamming(const uint32_t* __restrict__ plo,
                                                       const uint32_t* __restrict__ phi, int count,
                                                       int words, int length,
                                                       OUT* __restrict__ out, size_t ld, int row0,
                                                       int nrows) {
    extern __shared__ uint32_t sw[];
    uint32_t* alo = sw;                      // [64][words]
    uint32_t* ahi = alo + kHT * words;
    uint32_t* blo = ahi + kHT * words;
    uint32_t* bhi = blo + kHT * words;
    OUT* tr = reinterpret_cast<OUT*>(bhi + kHT * words);  // [64][65] mirror tile (SYM)
    int i0, j0;
    if constexpr (SYM) {
        int I, J;
        tile_pair_of(blockIdx.x, (count + kHT - 1) / kHT, I, J);
        i0 = I * kHT;
        j0 = J * kHT;
    } else {
        i0 = row0 + blockIdx.y * kHT;
        j0 = blockIdx.x * kHT;
    }
    const int iend = SYM ? count : row0 + nrows;
    for (int e = threadIdx.x; e < kHT * words; e += blockDim.x) {
        const int r = e / words, c = e % words;
        const bool ia = i0 + r < iend, jb = j0 + r < count;
        const size_t oa = static_cast<size_t>(i0 + r) * words + c;
        const size_t ob = static_cast<size_t>(j0 + r) * words + c;
        alo[e] = ia ? plo[oa] : 0u;
        ahi[e] = ia ? phi[oa] : 0u;
        blo[e] = jb ? plo[ob] : 0u;
        bhi[e] = jb ? phi[ob] : 0u;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    uint32_t h[4][4] = {};
    for (int c = 0; c < words; ++c) {
        uint32_t al[4], ah[4], bl[4], bh[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            al[k] = alo[(ty + 16 * k) * words + c];
            ah[k] = ahi[(ty + 16 * k) * words + c];
            bl[k] = blo[(tx + 16 * k) * words + c];
            bh[k] = bhi[(tx + 16 * k) * words + c];
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) h[x][y] += __popc((al[x] ^ bl[y]) | (ah[x] ^ bh[y]));
    }
    const double L = static_cast<double>(length);
    auto val = [&](uint32_t v) -> OUT {
        if constexpr (sizeof(OUT) == 8)
            return static_cast<double>(v) / L;
        else
            return v;
    };
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const int i = i0 + ty + 16 * x;
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int j = j0 + tx + 16 * y;
            if (i < iend && j < count)
                out[static_cast<size_t>(i - (SYM ? 0 : row0)) * ld + j] = val(h[x][y]);
            if constexpr (SYM) tr[(tx + 16 * y) * 65 + ty + 16 * x] = val(h[x][y]);
        }
    }
    if constexpr (SYM) {
        if (i0 == j0) return;  // diagonal tile: written once
        __syncthreads();
        // mirror: rows j0.., columns i0.. (coalesced along the columns)
        for (int e = threadIdx.x; e < kHT * kHT; e += blockDim.x) {
            const int r = e / kHT, cc = e % kHT;
            const int j = j0 + r, i = i0 + cc;
            if (j < count && i < count) out[static_cast<size_t>(j) * ld + i] = tr[r * 65 + cc];
        }
    }
}

}  // namespace

void launch_pack_reads(const unsigned char* reads, size_t count, int length, int words,
                       uint32_t* lo, uint32_t* hi, unsigned long long* bad, int sms,
                       cudaStream_t st) {
    const long long total = static_cast<long long>(count) * words;
    if (total == 0) return;
    const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, sms * 8));
    k_pack_reads<<<grid, 256, 0, st>>>(reads, static_cast<long long>(count), length, words, lo, hi,
                                       bad);
    count_launch();
}

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

void launch_hamming(const uint32_t* lo, const uint32_t* hi, size_t count, int words, int length,
                    double* d, size_t ld, uint32_t* counts, cudaStream_t st, size_t row0,
                    size_t nrows) {
    if (nrows == static_cast<size_t>(-1)) nrows = count;
    if (nrows == 0 || count == 0) return;
    const int nb = static_cast<int>((count + kHT - 1) / kHT);
    const bool sym = row0 == 0 && nrows == count;
    auto go = [&](auto* out, size_t ldo, auto sym_tag) {
        using O = std::remove_pointer_t<decltype(out)>;
        constexpr bool S = decltype(sym_tag)::value;
        const size_t smem = 4 * static_cast<size_t>(kHT) * words * sizeof(uint32_t) +
                            (S ? kHT * 65 * sizeof(O) : 0);
        allow_dyn_smem(reinterpret_cast<const void*>(k_hamming<O, S>));
        if constexpr (S) {
            const long long pairs = static_cast<long long>(nb) * (nb + 1) / 2;
            k_hamming<O, true><<<static_cast<unsigned>(pairs), kHThreads, smem, st>>>(
                lo, hi, static_cast<int>(count), words, length, out, ldo, 0,
                static_cast<int>(count));
        } else {
            dim3 grid(nb, static_cast<unsigned>((nrows + kHT - 1) / kHT));
            k_hamming<O, false><<<grid, kHThreads, smem, st>>>(lo, hi, static_cast<int>(count), words,
                                                         length, out, ldo,
                                                         static_cast<int>(row0),
                                                         static_cast<int>(nrows));
        }
    };
    // D on the int8 tensor cores (hamming_tc.cu) unless disabled or the row
    // band is not 128-aligned
    if (d && launch_hamming_tc(lo, hi, count, words, length, d, ld, st, row0, nrows)) d = nullptr;
    if (d) {
        if (sym) go(d, ld, std::true_type{});
        else go(d, ld, std::false_type{});
    }
    if (counts) {
        if (sym) go(counts, count, std::true_type{});
        else go(counts, count, std::false_type{});
    }
    count_launch();
}

}  // namespace dsb
