// S-digit layout shared by the int8 product (k2i_product.cu) and the K1
// pass that can write the cache (k1_stats.cu).
#pragma once
#include <cstdint>

namespace dsb {

// ---- S-digit cache -----------------------------------------------------------
// The S digits of a (128-row block, 32-column k-step) item depend only on D
// and the row exponents, which every product pass of a solve shares. With
// the cache on, either K1 writes every item's digit planes (SD x 4 KB) while
// it reads D for the gram (row exponents from a triangle-inequality bound,
// verified against the true ones; Hamming slices need none), or the solve's
// first product pass (DM = 1) stores them; the other passes (DM = 2) stream
// the planes with one bulk copy per item instead of the D tile: SD bytes per
// element instead of 8 (Hamming: 3), and no conversion.
// Item layout (bytes): half h = row / 64, plane t, converter column part p
// (8 columns), row % 64, 8 digit bytes: h SD 2048 + ((t-1) 4 + p) 512 +
// (row % 64) 8 — a converter warp's 32 rows are 256 contiguous bytes per
// plane, and each 64-row half is contiguous (the pair's multicast halves).
template <int SD>
constexpr int sdig_item_bytes() {
    return SD * 4 * 128 * 8;  // SD planes x 128 rows x 32 columns
}
__device__ __forceinline__ uint32_t sdig_off(int row, int part, int t, int sd) {
    return static_cast<uint32_t>((row >> 6) * sd * 2048 + ((t - 1) * 4 + part) * 512 +
                                 (row & 63) * 8);
}

// Digit planes of 8 fixed-point values (lo/hi 32-bit halves): w[t-1][g] holds
// digit t (byte 7 - t of the 56-bit value) of elements 4g..4g+3, byte j =
// element 4g+j. Two bytes of two planes are gathered per first-level
// byte_perm, so a pair of planes costs 4 permutes instead of 6.
__device__ __forceinline__ void pack_digits(const uint32_t (&lo)[8], const uint32_t (&hi)[8],
                                            uint32_t (&w)[7][2]) {
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const int e = 4 * g;
        // lo bytes 3,2 -> digits 4,5 ; lo bytes 1,0 -> digits 6,7
        const uint32_t p45 = __byte_perm(lo[e], lo[e + 1], 0x6273);
        const uint32_t q45 = __byte_perm(lo[e + 2], lo[e + 3], 0x6273);
        w[3][g] = __byte_perm(p45, q45, 0x5410);
        w[4][g] = __byte_perm(p45, q45, 0x7632);
        const uint32_t p67 = __byte_perm(lo[e], lo[e + 1], 0x4051);
        const uint32_t q67 = __byte_perm(lo[e + 2], lo[e + 3], 0x4051);
        w[5][g] = __byte_perm(p67, q67, 0x5410);
        w[6][g] = __byte_perm(p67, q67, 0x7632);
        // hi bytes 2,1 -> digits 1,2 ; hi byte 0 -> digit 3
        const uint32_t p12 = __byte_perm(hi[e], hi[e + 1], 0x5162);
        const uint32_t q12 = __byte_perm(hi[e + 2], hi[e + 3], 0x5162);
        w[0][g] = __byte_perm(p12, q12, 0x5410);
        w[1][g] = __byte_perm(p12, q12, 0x7632);
        const uint32_t p3 = __byte_perm(hi[e], hi[e + 1], 0x0040);
        const uint32_t q3 = __byte_perm(hi[e + 2], hi[e + 3], 0x0040);
        w[2][g] = __byte_perm(p3, q3, 0x5410);
    }
}


// Hamming slices: the three bytes (high first) of S' = h^2 < 2^24 of 8
// elements: plane t, word g holds byte (3 - t) of elements 4 g .. 4 g + 3
__device__ __forceinline__ void pack_digits3(const uint32_t (&s2)[8], uint32_t (&w)[3][2]) {
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const int e = 4 * g;
        const uint32_t h01 = __byte_perm(s2[e], s2[e + 1], 0x0062);
        const uint32_t h23 = __byte_perm(s2[e + 2], s2[e + 3], 0x0062);
        const uint32_t m01 = __byte_perm(s2[e], s2[e + 1], 0x0051);
        const uint32_t m23 = __byte_perm(s2[e + 2], s2[e + 3], 0x0051);
        const uint32_t l01 = __byte_perm(s2[e], s2[e + 1], 0x0040);
        const uint32_t l23 = __byte_perm(s2[e + 2], s2[e + 3], 0x0040);
        w[0][g] = __byte_perm(h01, h23, 0x5410);
        w[1][g] = __byte_perm(m01, m23, 0x5410);
        w[2][g] = __byte_perm(l01, l23, 0x5410);
    }
}

}  // namespace dsb
