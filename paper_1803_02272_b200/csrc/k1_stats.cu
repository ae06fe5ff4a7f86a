// K1 — pass 0 over the distance matrix (replaces the validation / row-mean
// part of gram_from_distances, ref src/mds.cpp:14-41, and frobenius_sq,
// ref src/rsvd.cpp:64-79).
//
// One read of D. The grid walks the upper-triangular pairs of 64x64 tiles
// (I <= J); each CTA loads tile (I,J) and its mirror (J,I) with coalesced
// 16-byte loads and produces, from that single read:
//   * partial row sums of d^2 of both tiles -> part[J][rows of I] and
//     part[I][rows of J] (disjoint slots, so no atomics; k1_rowmeans sums the
//     slots of a row in tile order => deterministic),
//   * sum of d^4 (closed-form ||G||_F^2), max |d| (all entries and the upper
//     triangle), and max |d_ij - d_ji| by comparing the tile with the
//     transposed mirror through shared memory.
// HBM roofline: n^2 * sizeof(T) bytes read once (+ n^2/64 * 8 partial bytes).
#include <cfloat>

#include "device_utils.cuh"
#include "kernels.cuh"
#include "sdig.cuh"

namespace dsb {

namespace {

constexpr int kT = 64;          // tile edge
#ifndef DSB_K1_NCH32
#define DSB_K1_NCH32 2  // f32 tiles: independent accumulation chains per lane (2: 0.7 % over 4)
#endif

template <typename T>
struct Pair2;
template <>
struct Pair2<double> {
    using V = double2;
};
template <>
struct Pair2<float> {
    using V = float2;
};

// load d[row][col], d[row][col+1] (zeros outside [0,n)), widened to double
template <typename T>
__device__ __forceinline__ void load2(const T* __restrict__ d, size_t ld, size_t n, size_t row,
                                      size_t col, double& a0, double& a1) {
    a0 = 0.0;
    a1 = 0.0;
    if (row >= n || col >= n) return;
    const T* p = d + row * ld + col;
    if (col + 1 < n) {
        const typename Pair2<T>::V v = __ldg(reinterpret_cast<const typename Pair2<T>::V*>(p));
        a0 = static_cast<double>(v.x);
        a1 = static_cast<double>(v.y);
    } else {
        a0 = static_cast<double>(__ldg(p));
    }
}

// (I, J) with I <= J from the linear index over the upper triangle, row-major
__device__ __forceinline__ void pair_of(long long p, int nbt, int& I, int& J) {
    const double nf = static_cast<double>(nbt);
    double g = (2.0 * nf + 1.0 - sqrt((2.0 * nf + 1.0) * (2.0 * nf + 1.0) - 8.0 * (double)p)) / 2.0;
    long long i = g <= 0.0 ? 0 : static_cast<long long>(g);
    if (i > nbt - 1) i = nbt - 1;
    auto off = [&](long long r) { return r * nbt - r * (r - 1) / 2; };
    while (i > 0 && off(i) > p) --i;
    while (i + 1 < nbt && off(i + 1) <= p) ++i;
    I = static_cast<int>(i);
    J = static_cast<int>(i + (p - off(i)));
}

// ---- TMA-fed version: tiles arrive as NB boxes of 64 rows x 128 bytes
// (SWIZZLE_128B) on a 3..6-stage mbarrier ring filled by a producer warp; 8
// consumer warps each own 8 rows of both tiles: lane (row r = l % 8, quarter
// q = l / 8) reads its 16-element row segment with 16-byte shared loads,
// sums it sequentially, and two xor-shuffles complete the 64-column row sum.
template <typename T>
struct K1Cfg {
    // consumer warps: 8 for f64 tiles (HBM-bound), 16 for f32 tiles (twice the
    // elements per byte: more warps to hide the FP64 / conversion latency).
    // Warp w owns rows 8 (w % 8) .. +7 and column part w / 8 (H parts of 64 / H
    // columns); each lane (row l % 8, quarter l / 8) EL consecutive columns.
    static constexpr int CW = sizeof(T) == 4 ? 16 : 8;
    static constexpr int H = CW / 8;
    static constexpr int EL = 16 / H;
    static constexpr int THREADS = CW * 32 + 32;
    static constexpr int E = sizeof(T);
    static constexpr int BC = 128 / E;           // columns per 128-byte box row
    static constexpr int NB = kT / BC;           // boxes per 64-column tile
    static constexpr int TILE = NB * kT * 128;   // bytes per tile
    static constexpr int STAGE = 2 * TILE;
    static constexpr int STAGES = (192 * 1024) / STAGE;
};

template <typename T>
struct C_EL_IS_16 {
    static constexpr bool value = K1Cfg<T>::EL == 16 && K1Cfg<T>::H == 1;
};

// element (r, c) of a swizzled tile (box-major)
template <typename T>
__device__ __forceinline__ const T* tile_at(const unsigned char* tile, int r, int c) {
    using C = K1Cfg<T>;
    const int b = c / C::BC, cc = c % C::BC;
    const int byte = cc * C::E;
    return reinterpret_cast<const T*>(tile + b * (kT * 128) + r * 128 +
                                      ((((byte >> 4) ^ (r & 7))) << 4) + (byte & 15));
}

// Smallest e with x < 2^e for the largest x >= 0 of a set, from the max of
// the high 32 bits of the doubles (for non-negative doubles the bit patterns
// order like the values; integer max keeps this off the FP64 pipe).
// kExpZero when all are zero.
constexpr int kExpZero = -1100;
__device__ __forceinline__ double max_keep(double m, double x) { return x > m ? x : m; }
__device__ __forceinline__ uint32_t hi_bits(double x) {
    return static_cast<uint32_t>(__double2hiint(x));
}
__device__ __forceinline__ int exp_above_hi(uint32_t hmax) {
    if (hmax == 0u) return kExpZero;
    const int be = static_cast<int>((hmax >> 20) & 0x7ffu);
    if (be == 0) return -1022;  // subnormal: x < 2^-1022
    return be - 1022;
}

// K1 writing the S-digit cache: the 16 values v of tile row r, tile columns
// 16 q .. 16 q + 15, of the 64 x 64 tile (tr, tc) -> item (tr / 2, 2 tc +
// q / 2), half tr % 2, converter parts 2 (q % 2) + {0, 1} (sdig.cuh layout).
// DG = 7: the 56-bit fixed point of v^2 relative to 2^e (sc = 2^(56 - e)),
// as the product's converters form it; DG = 3: the bytes of h^2, h = L v.
template <int DG>
__device__ __forceinline__ void k1_write_digits(unsigned char* __restrict__ sdig, int nks, int tr,
                                                int tc, int r, int q, const double (&v)[16],
                                                double sc, double hlen) {
    const int ks = 2 * tc + (q >> 1);
    if (ks >= nks) return;  // the last tile's padding columns past the last k-step
    const size_t item = static_cast<size_t>(tr >> 1) * nks + ks;
    unsigned char* base =
        sdig + item * sdig_item_bytes<DG>() + (tr & 1) * DG * 2048 + r * 8 + (q & 1) * 2 * 512;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        uint32_t w[DG][2];
        if constexpr (DG == 7) {
            uint32_t lo[8], hi[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const unsigned long long m = __double2ull_rz((v[8 * g + j] * v[8 * g + j]) * sc);
                lo[j] = static_cast<uint32_t>(m);
                hi[j] = static_cast<uint32_t>(m >> 32);
            }
            pack_digits(lo, hi, w);
        } else {
            uint32_t s2[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t h = static_cast<uint32_t>(__double2int_rn(v[8 * g + j] * hlen));
                s2[j] = h * h;
            }
            pack_digits3(s2, w);
        }
#pragma unroll
        for (int t = 1; t <= DG; ++t)
            *reinterpret_cast<uint2*>(base + ((t - 1) * 4 + g) * 512) = make_uint2(w[t - 1][0],
                                                                                  w[t - 1][1]);
    }
}

template <typename T, int DG>
__global__ void __launch_bounds__(K1Cfg<T>::THREADS, 1)
    k1_tile_pairs(const __grid_constant__ CUtensorMap tm, int n, int nbt,
                  double* __restrict__ part, int* __restrict__ pexp, size_t part_ld,
                  double* __restrict__ cta_stats, unsigned char* __restrict__ sdig,
                  const int* __restrict__ row_eb, int nks, double hlen) {
    static_assert(DG == 0 || (sizeof(T) == 8 && C_EL_IS_16<T>::value), "digits: f64 tiles");
    using C = K1Cfg<T>;
    extern __shared__ __align__(1024) unsigned char k1_raw[];
    unsigned char* sm = k1_raw + ((1024u - (smem_u32(k1_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    // tile-pair coordinates of each stage, written by the producer before its
    // expect_tx arrival (release) and read after the full wait (acquire), so
    // the consumers do not each re-derive them (a double sqrt per pair)
    int2* stage_ij = reinterpret_cast<int2*>(empty + C::STAGES);
    __shared__ double red[4][C::CW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long npairs = static_cast<long long>(nbt) * (nbt + 1) / 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == C::CW) {  // producer
        if (lane == 0) {
            prefetch_tmap(&tm);
            int s = 0;
            uint32_t ph = 0;
            long long it = 0;
            for (long long p = blockIdx.x; p < npairs; p += gridDim.x, ++it) {
                if (it >= C::STAGES) mbar_wait(&empty[s], ph ^ 1);
                int I, J;
                pair_of(p, nbt, I, J);
                unsigned char* st = sm + s * C::STAGE;
                if constexpr (sizeof(T) == 4) stage_ij[s] = make_int2(I, J);
                mbar_arrive_expect_tx(&full[s], (I != J ? 2 : 1) * C::TILE);
                for (int b = 0; b < C::NB; ++b)
                    tma_load_2d(st + b * (kT * 128), &tm, J * kT + b * C::BC, I * kT, &full[s]);
                if (I != J)
                    for (int b = 0; b < C::NB; ++b)
                        tma_load_2d(st + C::TILE + b * (kT * 128), &tm, I * kT + b * C::BC, J * kT,
                                    &full[s]);
                if (++s == C::STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }
    double sum4 = 0.0, maxabs = 0.0, maxabs_up = 0.0, maxasym = 0.0;
    float maxf = 0.0f, maxup_f = 0.0f;  // f32 tiles: the maxima in the float domain
    const int r = (warp & 7) * 8 + (lane & 7), q = lane >> 3, h = warp >> 3;
    const int col0 = h * (kT / C::H) + q * C::EL;  // first tile column of this lane
    int s = 0;
    uint32_t ph = 0;
    for (long long p = blockIdx.x; p < npairs; p += gridDim.x) {
        int I, J;
        if constexpr (sizeof(T) == 4) {
            mbar_wait(&full[s], ph);
            const int2 ij = stage_ij[s];
            I = ij.x;
            J = ij.y;
        } else {
            // f64 tiles: deriving (I, J) overlaps the wait (measured faster)
            pair_of(p, nbt, I, J);
        }
        // the digits' row exponents, loaded ahead (their global latency
        // otherwise stalled the conversion: 22 % of the stall samples)
        int ebA = kExpZero, ebB = kExpZero;
        if constexpr (DG == 7) {
            const int ga = I * kT + r, gb = J * kT + r;
            if (ga < n) ebA = __ldg(row_eb + ga);
            if (gb < n) ebB = __ldg(row_eb + gb);
        }
        if constexpr (sizeof(T) == 8) mbar_wait(&full[s], ph);
        const unsigned char* A = sm + s * C::STAGE;
        const unsigned char* B = (I != J) ? A + C::TILE : A;
        double a[C::EL];
        T av[C::EL];  // the raw row segment (f32: two 16-byte loads per 8 values)
        if constexpr (sizeof(T) == 4) {
#pragma unroll
            for (int j = 0; j < C::EL; j += 4) {
                const float4 v = *reinterpret_cast<const float4*>(tile_at<T>(A, r, col0 + j));
                av[j] = v.x;
                av[j + 1] = v.y;
                av[j + 2] = v.z;
                av[j + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < C::EL; ++j) av[j] = *tile_at<T>(A, r, col0 + j);
        }
#pragma unroll
        for (int j = 0; j < C::EL; ++j) a[j] = static_cast<double>(av[j]);
        // f32 tiles: DSB_K1_NCH32 independent accumulation chains (a 16-long dependent
        // DADD chain left the FP64 latency exposed); f64 tiles: one (faster there)
        constexpr int NCH = sizeof(T) == 4 ? DSB_K1_NCH32 : 1;
        double rsp[4] = {0.0, 0.0, 0.0, 0.0}, s4p[4] = {0.0, 0.0, 0.0, 0.0};
        uint32_t rmx = 0u;
        float rmaxf = 0.0f;  // f32 tiles: max |d| of the row segment
        T mtv[C::EL];        // f32 tiles: the mirror entries B[c][r] of the segment
        uint32_t diff = 0u;  // f32 tiles: OR of the pairs' bit differences
#pragma unroll
        for (int j = 0; j < C::EL; ++j) {
            const double sq = a[j] * a[j];
            rsp[j % NCH] += sq;
            s4p[j % NCH] += sq * sq;
            const bool upper = I != J || col0 + j >= r;
            // (x > m ? x : m): NaN is never selected, as std::max(m, x) in the
            // reference's scans (mds.cpp:21-27, rsvd.cpp:50-54); cheaper than fmax
            if constexpr (sizeof(T) == 4) {
                // max |d| in the float domain (widening is monotonic, so the
                // widened max is the max of the widened values); the row
                // exponent follows from the row max: max d^2 = (max |d|)^2.
                // fmaxf (one FMNMX) never returns a NaN operand over a
                // non-NaN one, as (x > m ? x : m) in the reference's scans;
                // off the diagonal every entry is upper: the segment max
                // covers it below
                const float af = fabsf(av[j]);
                rmaxf = fmaxf(rmaxf, af);
                if (I == J && upper) maxup_f = fmaxf(maxup_f, af);
            } else {
                rmx = max(rmx, hi_bits(sq));
                if (upper) maxabs_up = max_keep(maxabs_up, fabs(a[j]));
            }
            // symmetry: A[r][c] vs B[c][r] (d_ij vs d_ji)
            if constexpr (sizeof(T) == 4) {
                // identical bits (the symmetric case) give 0: only the bit
                // difference is accumulated here; a segment with any
                // differing pair takes the f64 differences below
                mtv[j] = *tile_at<T>(B, col0 + j, r);
                diff |= __float_as_uint(mtv[j]) ^ __float_as_uint(av[j]);
            } else {
                const T mt = *tile_at<T>(B, col0 + j, r);
                maxasym = max_keep(maxasym, fabs(a[j] - mt));
            }
        }
        if constexpr (sizeof(T) == 4) {
            if (diff != 0u) {  // rare: the reference's f64 difference per pair
#pragma unroll
                for (int j = 0; j < C::EL; ++j)
                    if (__float_as_uint(mtv[j]) != __float_as_uint(av[j]))
                        maxasym = max_keep(maxasym, fabs(a[j] - static_cast<double>(mtv[j])));
            }
        }
        if constexpr (sizeof(T) == 4) {
            const double m = static_cast<double>(rmaxf);
            rmx = hi_bits(m * m);
            if (I == J) maxf = fmaxf(maxf, rmaxf);
            else maxup_f = fmaxf(maxup_f, rmaxf);
        } else if (I == J) {  // diagonal tile: maxabs_up saw only its upper part
#pragma unroll
            for (int j = 0; j < C::EL; ++j) maxabs = max_keep(maxabs, fabs(a[j]));
        }
        double rs = (rsp[0] + rsp[1]) + (rsp[2] + rsp[3]);
        sum4 += (s4p[0] + s4p[1]) + (s4p[2] + s4p[3]);
        if constexpr (DG != 0) {
            double sc = 0.0;
            if constexpr (DG == 7) sc = ebA > kExpZero ? ldexp(1.0, 56 - ebA) : 0.0;
            k1_write_digits<DG>(sdig, nks, I, J, r, q, a, sc, hlen);
        }
        rs += __shfl_xor_sync(0xffffffffu, rs, 8);
        rs += __shfl_xor_sync(0xffffffffu, rs, 16);
        rmx = max(rmx, __shfl_xor_sync(0xffffffffu, rmx, 8));
        rmx = max(rmx, __shfl_xor_sync(0xffffffffu, rmx, 16));
        if (q == 0 && I * kT + r < n) {
            part[static_cast<size_t>(J * C::H + h) * part_ld + I * kT + r] = rs;
            pexp[static_cast<size_t>(J * C::H + h) * part_ld + I * kT + r] = exp_above_hi(rmx);
        }
        if (I != J) {
            double rbp[4] = {0.0, 0.0, 0.0, 0.0}, b4p[4] = {0.0, 0.0, 0.0, 0.0};
            uint32_t bmx = 0u;
            float bmaxf = 0.0f;
            T bv[C::EL];
            if constexpr (sizeof(T) == 4) {
#pragma unroll
                for (int j = 0; j < C::EL; j += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(tile_at<T>(B, r, col0 + j));
                    bv[j] = v.x;
                    bv[j + 1] = v.y;
                    bv[j + 2] = v.z;
                    bv[j + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < C::EL; ++j) bv[j] = *tile_at<T>(B, r, col0 + j);
            }
#pragma unroll
            for (int j = 0; j < C::EL; ++j) {
                const T bt = bv[j];
                const double b = static_cast<double>(bt);
                const double sq = b * b;
                rbp[j % NCH] += sq;
                b4p[j % NCH] += sq * sq;
                if constexpr (sizeof(T) == 4) {
                    bmaxf = fmaxf(bmaxf, fabsf(bt));
                } else {
                    bmx = max(bmx, hi_bits(sq));
                    maxabs = max_keep(maxabs, fabs(b));
                }
            }
            if constexpr (sizeof(T) == 4) {
                const double m = static_cast<double>(bmaxf);
                bmx = hi_bits(m * m);
                maxf = fmaxf(maxf, bmaxf);
            }
            if constexpr (DG != 0) {
                double bd[C::EL];
#pragma unroll
                for (int j = 0; j < C::EL; ++j) bd[j] = static_cast<double>(bv[j]);
                double sc = 0.0;
                if constexpr (DG == 7) sc = ebB > kExpZero ? ldexp(1.0, 56 - ebB) : 0.0;
                k1_write_digits<DG>(sdig, nks, J, I, r, q, bd, sc, hlen);
            }
            double rb = (rbp[0] + rbp[1]) + (rbp[2] + rbp[3]);
            sum4 += (b4p[0] + b4p[1]) + (b4p[2] + b4p[3]);
            rb += __shfl_xor_sync(0xffffffffu, rb, 8);
            rb += __shfl_xor_sync(0xffffffffu, rb, 16);
            bmx = max(bmx, __shfl_xor_sync(0xffffffffu, bmx, 8));
            bmx = max(bmx, __shfl_xor_sync(0xffffffffu, bmx, 16));
            if (q == 0 && J * kT + r < n) {
                part[static_cast<size_t>(I * C::H + h) * part_ld + J * kT + r] = rb;
                pexp[static_cast<size_t>(I * C::H + h) * part_ld + J * kT + r] = exp_above_hi(bmx);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
        }
    }
    if constexpr (sizeof(T) == 4) {
        maxabs = static_cast<double>(maxf);
        maxabs_up = static_cast<double>(maxup_f);
    }
    // every off-diagonal A tile entry is an upper entry: max|a| over all
    // entries = max(max over upper entries, B tiles, diagonal tiles)
    maxabs = max_keep(maxabs, maxabs_up);
    // fixed-order block reduction (deterministic for a fixed grid)
    sum4 = warp_sum(sum4);
    maxabs = warp_max(maxabs);
    maxabs_up = warp_max(maxabs_up);
    maxasym = warp_max(maxasym);
    if (lane == 0) {
        red[0][warp] = sum4;
        red[1][warp] = maxabs;
        red[2][warp] = maxabs_up;
        red[3][warp] = maxasym;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(C::CW * 32));  // consumers only
    if (threadIdx.x == 0) {
        double su = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0;
        for (int w = 0; w < C::CW; ++w) {
            su += red[0][w];
            m1 = fmax(m1, red[1][w]);
            m2 = fmax(m2, red[2][w]);
            m3 = fmax(m3, red[3][w]);
        }
        cta_stats[blockIdx.x * 4 + 0] = su;
        cta_stats[blockIdx.x * 4 + 1] = m1;
        cta_stats[blockIdx.x * 4 + 2] = m2;
        cta_stats[blockIdx.x * 4 + 3] = m3;
    }
}

template <typename T>
size_t k1_smem() {
    return static_cast<size_t>(K1Cfg<T>::STAGES) * K1Cfg<T>::STAGE + 1024 + 16 * K1Cfg<T>::STAGES;
}

// r_i = (sum over tile columns of part[J][i]) / n, plus per-block sums of
// the raw row sums, r and r^2. Also the row exponent e_i (max over the tile
// partials: every d_ij^2 of row i is < 2^e_i) and the block max of the
// dynamic-range bound 2^e_i / r_i used to admit the int8 slice product.
// A block owns 32 rows; its 8 warps stride over the tile columns J (warp w:
// J = w, w + 8, ...) and the 8 partials are added in warp order (fixed).
constexpr int kRmRows = 32;
// row_eb (K1 writing the S-digit cache): the bound exponents its digits
// used; blk_bad[b] = 1 when a row of block b is not covered by its bound or
// the bound is more than 3 bits above the row's exponent (k1_finalize ORs
// them into scalars[S_SDIG_BAD])
__global__ void __launch_bounds__(256) k1_rowmeans(const double* __restrict__ part,
                                                   const int* __restrict__ pexp, size_t part_ld,
                                                   int nbt, int n, double* __restrict__ row_mean,
                                                   int* __restrict__ row_exp,
                                                   double* __restrict__ blk_stats,
                                                   const int* __restrict__ row_eb,
                                                   int* __restrict__ blk_bad) {
    __shared__ double ps[8][kRmRows];
    __shared__ int pe[8][kRmRows];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * kRmRows + lane;
    double acc = 0.0;
    int e = kExpZero;
    if (i < n) {
        for (int J = warp; J < nbt; J += 8) {
            acc += part[static_cast<size_t>(J) * part_ld + i];
            e = max(e, pexp[static_cast<size_t>(J) * part_ld + i]);
        }
    }
    ps[warp][lane] = acc;
    pe[warp][lane] = e;
    __syncthreads();
    if (warp == 0) {
        double rowsum = 0.0, r = 0.0, ratio = 0.0;
        int bad = 0;
        if (i < n) {
            int ee = kExpZero;
            for (int w = 0; w < 8; ++w) {
                rowsum += ps[w][lane];
                ee = max(ee, pe[w][lane]);
            }
            r = rowsum / static_cast<double>(n);
            row_mean[i] = r;
            row_exp[i] = ee;
            if (row_eb) {
                const int eb = row_eb[i];
                bad = (ee > eb || (ee > kExpZero && eb - ee > 3)) ? 1 : 0;
            }
            if (ee > kExpZero) ratio = (r > 0.0) ? ldexp(1.0, ee) / r : 1e300;
        }
        const double v0 = warp_sum(rowsum), v1 = warp_sum(r), v2 = warp_sum(r * r),
                     v3 = warp_max(ratio);
        bad = __any_sync(0xffffffffu, bad != 0) ? 1 : 0;
        if (lane == 0) {
            blk_bad[blockIdx.x] = bad;
            blk_stats[blockIdx.x * 4 + 0] = v0;
            blk_stats[blockIdx.x * 4 + 1] = v1;
            blk_stats[blockIdx.x * 4 + 2] = v2;
            blk_stats[blockIdx.x * 4 + 3] = v3;
        }
    }
}

// One block: thread t reduces entries t, t+256, ... (fixed order), then a
// fixed-order tree over the 256 threads — deterministic.
__global__ void __launch_bounds__(256) k1_finalize(const double* __restrict__ cta_stats, int ncta,
                                                   const double* __restrict__ blk_stats, int nblk,
                                                   int n, double* __restrict__ scalars,
                                                   const int* __restrict__ blk_bad) {
    __shared__ double sh[8][256];
    const int t = threadIdx.x;
    double sum4 = 0, m1 = 0, m2 = 0, m3 = 0, rows = 0, sr = 0, sr2 = 0, rr = 0;
    for (int c = t; c < ncta; c += 256) {
        sum4 += cta_stats[c * 4 + 0];
        m1 = fmax(m1, cta_stats[c * 4 + 1]);
        m2 = fmax(m2, cta_stats[c * 4 + 2]);
        m3 = fmax(m3, cta_stats[c * 4 + 3]);
    }
    int bad = 0;
    for (int b = t; b < nblk; b += 256) {
        bad |= blk_bad[b];
        rows += blk_stats[b * 4 + 0];
        sr += blk_stats[b * 4 + 1];
        sr2 += blk_stats[b * 4 + 2];
        rr = fmax(rr, blk_stats[b * 4 + 3]);
    }
    sh[0][t] = sum4; sh[1][t] = m1; sh[2][t] = m2; sh[3][t] = m3;
    sh[4][t] = rows; sh[5][t] = sr; sh[6][t] = sr2; sh[7][t] = rr;
    bad = __syncthreads_or(bad);
    for (int off = 128; off > 0; off >>= 1) {
        if (t < off) {
            sh[0][t] += sh[0][t + off];
            sh[1][t] = fmax(sh[1][t], sh[1][t + off]);
            sh[2][t] = fmax(sh[2][t], sh[2][t + off]);
            sh[3][t] = fmax(sh[3][t], sh[3][t + off]);
            sh[4][t] += sh[4][t + off];
            sh[5][t] += sh[5][t + off];
            sh[6][t] += sh[6][t + off];
            sh[7][t] = fmax(sh[7][t], sh[7][t + off]);
        }
        __syncthreads();
    }
    if (t == 0) {
        const double nf = static_cast<double>(n);
        const double grand = sh[5][0] / nf;
        scalars[S_GRAND] = grand;
        scalars[S_FRO2_LAZY] = 0.25 * (sh[0][0] - 2.0 * nf * sh[6][0] + nf * nf * grand * grand);
        scalars[S_FRO2_EXPL] = sh[4][0];
        scalars[S_MAXABS] = sh[1][0];
        scalars[S_MAXABS_UP] = sh[2][0];
        scalars[S_MAXASYM] = sh[3][0];
        scalars[S_SUM4] = sh[0][0];
        scalars[S_SUMR] = sh[5][0];
        scalars[S_SUMR2] = sh[6][0];
        scalars[S_ROWRATIO] = sh[7][0];
        scalars[S_SDIG_BAD] = bad ? 1.0 : 0.0;
    }
}

// row_eb from row 0 of D: max_j d_ij <= d_i0 + d_0j <= |d_0i| + M0 (triangle
// inequality, d_i0 = d_0i), M0 = max_j |d_0j| (NaN-ignoring selects, as K1);
// the sum and square rounded up. Every CTA forms M0 itself (4 loads in
// flight per thread), then bounds its own 1024 rows
__global__ void __launch_bounds__(1024) k_row0_bound(const double* __restrict__ d0, int n,
                                                     int* __restrict__ row_eb) {
    __shared__ double red[32];
    double m[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j0 = threadIdx.x; j0 < n; j0 += 4 * blockDim.x) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * blockDim.x;
            if (j < n) m[u] = max_keep(m[u], fabs(__ldg(d0 + j)));
        }
    }
    double mm = max_keep(max_keep(m[0], m[1]), max_keep(m[2], m[3]));
    mm = warp_max(mm);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mm;
    __syncthreads();
    double m0 = 0.0;
    for (int w = 0; w < 32; ++w) m0 = max_keep(m0, red[w]);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double b = __dadd_ru(fabs(d0[i]), m0);
        row_eb[i] = exp_above_hi(hi_bits(__dmul_ru(b, b)));
    }
}

}  // namespace

size_t k1_part_elems(size_t n) {
    const size_t nbt = (n + kT - 1) / kT;
    return nbt * nbt * kT * 2;  // up to 2 column parts per tile (f32: K1Cfg<float>::H)
}

int k1_grid(size_t n, int sms) {
    const long long nbt = static_cast<long long>((n + kT - 1) / kT);
    const long long npairs = nbt * (nbt + 1) / 2;
    const long long cap = static_cast<long long>(sms);
    return static_cast<int>(npairs < cap ? npairs : cap);
}

void launch_k1(const CUtensorMap* tmap64, DType dt, size_t n, const K1Work& w, double* row_mean,
               int* row_exp, double* scalars, int sms, cudaStream_t st, const K1Digits* dig) {
    (void)sms;
    const int nbt = static_cast<int>((n + kT - 1) / kT);
    const size_t part_ld = static_cast<size_t>(nbt) * kT;
    const int dg = (dig && dig->sdig && dt == DType::F64) ? dig->sd : 0;
    auto run64 = [&](auto kern) {
        ensure_dyn_smem(reinterpret_cast<const void*>(kern), k1_smem<double>());
        kern<<<w.grid, K1Cfg<double>::THREADS, k1_smem<double>(), st>>>(
            *tmap64, static_cast<int>(n), nbt, w.part, w.pexp, part_ld, w.cta_stats,
            dg ? dig->sdig : nullptr, dg == 7 ? dig->row_eb : nullptr, dg ? dig->nks : 0,
            dg == 3 ? dig->hlen : 0.0);
    };
    if (dt == DType::F64) {
        if (dg == 7)
            run64(k1_tile_pairs<double, 7>);
        else if (dg == 3)
            run64(k1_tile_pairs<double, 3>);
        else
            run64(k1_tile_pairs<double, 0>);
    } else {
        ensure_dyn_smem(reinterpret_cast<const void*>(k1_tile_pairs<float, 0>), k1_smem<float>());
        k1_tile_pairs<float, 0><<<w.grid, K1Cfg<float>::THREADS, k1_smem<float>(), st>>>(
            *tmap64, static_cast<int>(n), nbt, w.part, w.pexp, part_ld, w.cta_stats, nullptr,
            nullptr, 0, 0.0);
    }
    const int nblk = static_cast<int>((n + kRmRows - 1) / kRmRows);
    const int nparts = nbt * (dt == DType::F64 ? K1Cfg<double>::H : K1Cfg<float>::H);
    k1_rowmeans<<<nblk, 256, 0, st>>>(w.part, w.pexp, part_ld, nparts, static_cast<int>(n),
                                      row_mean, row_exp, w.blk_stats,
                                      dg == 7 ? dig->row_eb : nullptr, w.blk_bad);
    k1_finalize<<<1, 256, 0, st>>>(w.cta_stats, w.grid, w.blk_stats, nblk, static_cast<int>(n),
                                   scalars, w.blk_bad);
    count_launch(3);
}

void launch_row0_bound(const double* d, size_t n, int* row_eb, cudaStream_t st) {
    k_row0_bound<<<static_cast<unsigned>((n + 1023) / 1024), 1024, 0, st>>>(
        d, static_cast<int>(n), row_eb);
    count_launch(1);
}

}  // namespace dsb
