// mx8.cuh — the MX8 weight format (FDIRW_W_MX8): layout and quantiser shared
// by its writer (dedup.cu: expand_mx8_kernel, mx8_diag_kernel), the superposition
// (superpose.cu: superpose_mx8_kernel) and the exporter.
//
// A gather block = the 8 weights one superposition thread loads for one slot (8 consecutive
// targets x0..x0+7 of a row, one window offset o; sources x0−ox … x0+7−ox).  Each weight is an
// unsigned 8-bit mantissa m; the block has one power-of-two scale s = 2^(E−127) (E an 8-bit
// biased exponent): w = m·s.  s is the smallest power of two with max_block(w)/s ≤ 255;
// m = RNE(w/s), negative weights (Chebyshev round-off, |w| ≲ 1e-10) clamp to 0.  The fp32
// diagonal restores each source's mass from the decoded weights (reading A10 unchanged).
//
// Layout per tile of T chunks, stored row i (i = 0: centre row, L − 1 slots; i ≥ 1: L slots,
// slot order of layout.cuh) at byte (first slot of row i)·9T:
//   mantissas [n_i][T][8] u8, then scales [n_i][T] u8
// so one stored row (n_i·9T bytes, a multiple of 16) is one contiguous bulk copy, and the
// whole tile is (K − 1)·9T bytes.
#pragma once
#include <cstddef>
#include <cstdint>

namespace fdirw {

__host__ __device__ __forceinline__ int mx8_row_first(int i, int L) { return i == 0 ? 0 : (L - 1) + (i - 1) * L; }

// (slot k, chunk e, target j) of tile `tile` → byte offsets of its mantissa and its block scale
__host__ __device__ __forceinline__ void mx8_addr(size_t tile, int k, int e, int j, int L, int K, int T, size_t* mant,
                                                  size_t* scale)
{
    const int i = k < L - 1 ? 0 : 1 + (k - (L - 1)) / L;
    const int f = mx8_row_first(i, L), n = i == 0 ? L - 1 : L, kin = k - f;
    const size_t base = tile * (size_t)(K - 1) * 9 * T + (size_t)f * 9 * T;
    *mant = base + (size_t)kin * 8 * T + (size_t)e * 8 + j;
    *scale = base + (size_t)n * 8 * T + (size_t)kin * T + e;
}

// Quantise one gather block: 8 fp32 weights → 8 mantissas (little-endian in a uint2) + E.
__device__ __forceinline__ void mx8_quant(const float v[8], uint2* mant, uint32_t* Eout)
{
    float M = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) M = fmaxf(M, v[j]);
    int E = 1;
    if (M > 0.f) {
        int e = ilogbf(M) - 7;                // M·2^−e ∈ [128, 256)
        if (ldexpf(M, -e) > 255.f) e += 1;    // smallest e with M·2^−e ≤ 255
        E = e + 127;
        if (E < 1) E = 1;                     // M < 255·2^−126: m ≤ 255 still holds
    }
    const float inv = __uint_as_float((uint32_t)(254 - E) << 23);  // 2^(127 − E) = 1/s
    uint32_t m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float q = rintf(fmaxf(v[j], 0.f) * inv);
        m[j] = (uint32_t)fminf(q, 255.f);
    }
    mant->x = m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24);
    mant->y = m[4] | (m[5] << 8) | (m[6] << 16) | (m[7] << 24);
    *Eout = (uint32_t)E;
}

// Decode weight j of a block exactly: s = 2^(E−127), m·s (8-bit m, normal s: exact in fp32).
__device__ __forceinline__ float mx8_decode(uint32_t m, uint32_t E)
{
    return (float)m * __uint_as_float(E << 23);
}

}  // namespace fdirw
