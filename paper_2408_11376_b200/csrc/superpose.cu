// superpose.cu — a5: the FDiRW superposition step in gather form, plus the small
// state kernels (pack/unpack of the padded state, fp64 mass reduction, kernel export).
//
//   C_new(x) = d_x·C_old(x) + Σ_{o≠0} Wt[o][x]·C_old(x − o)
//
// = P:101 Eq.8 / P:131 Eq.14 with the per-source kernels W_s(o) = p_{s+o,s}
// read in gather order (closed domain: no p_BC term, reading A3).
// Weights are fp32/fp16/bf16 (§3.3; reading A9: reduced-precision
// storage, fp32 products and accumulation).
//
// B200 mapping: HBM-bound weight streaming.
//  * one thread = 8 consecutive x targets of one row; one CTA = one tile of
//    `tile` such chunks; the tile's weights for one slot are `tile`·8 contiguous
//    values, so a warp reads 512 B (bf16) per slot with 128-bit loads, and the
//    whole tile streams one contiguous (K−1)·tile·8·b_w region;
//  * weights: ld.global.nc.L1::no_allocate + L2 evict_first policy (read once);
//  * C_old: the padded state (zero halo of R planes/rows, 8 columns), read with
//    128-bit L1-cached loads: per (oz, oy) row a thread loads the aligned
//    24-float segment [x−8, x+16) once and reuses it for all 2R+1 x-offsets
//    × 8 targets (register blocking: 6 loads per 8·(2R+1) FMAs);
//  * bf16 → fp32 is a shift/mask, fp16 → fp32 a cvt; accumulation: fp32 FMA per row, rows combined
//    error-free into an fp32 (hi, lo) pair, in a fixed order (diag, centre row, rows (oz, oy) ascending), so the result is
//    bitwise independent of the slab decomposition.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "bulk.cuh"
#include "fdirw_internal.h"
#include "layout.cuh"
#include "mx8.cuh"
#include <cstdlib>

namespace fdirw {

__device__ __forceinline__ uint64_t evict_first_policy()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint4 ld_stream(const void* ptr, uint64_t pol)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ float4 ld_c(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// The diagonal term of 8 targets, d·C_old(x) with d = dh + dl an fp32 pair (reading A10), in two
// parts: head (first, DESIGN §6 order) hi = RN(dh·C), lo = 0; tail (last, before acc = hi + lo)
// lo += (dh·C − RN(dh·C)) + dl·C, the head product's exact error (FMA) and the low part.  (With the
// whole pair in the head, lo starting non-zero made the one-wave register-prefetch launch 24 %
// slower at cfg2 for reasons ncu does not show — same instructions, more long-scoreboard stalls;
// the tail form measures as before.)  dp = 8 float2 (64 B, 16-byte aligned), c = C_old(x .. x+7).
__device__ __forceinline__ void diag_pair_head(const float2* dp, const float* c, float hi[8], float lo[8])
{
    const float4 v0 = ld_c(c), v1 = ld_c(c + 4);
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 d = __ldg(reinterpret_cast<const float4*>(dp) + k);  // (dh, dl) of targets 2k, 2k+1
        hi[2 * k] = __fmul_rn(d.x, v[2 * k]);
        hi[2 * k + 1] = __fmul_rn(d.z, v[2 * k + 1]);
        lo[2 * k] = lo[2 * k + 1] = 0.f;
    }
}
__device__ __forceinline__ void diag_pair_tail(const float2* dp, const float* c, float lo[8])
{
    const float4 v0 = ld_c(c), v1 = ld_c(c + 4);
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 d = __ldg(reinterpret_cast<const float4*>(dp) + k);
        lo[2 * k] = __fadd_rn(lo[2 * k], fmaf(d.y, v[2 * k], fmaf(d.x, v[2 * k], -__fmul_rn(d.x, v[2 * k]))));
        lo[2 * k + 1] =
            __fadd_rn(lo[2 * k + 1], fmaf(d.w, v[2 * k + 1], fmaf(d.z, v[2 * k + 1], -__fmul_rn(d.z, v[2 * k + 1]))));
    }
}
// the same with one pair d for all 8 targets (N4: a uniform chunk's class diagonal)
__device__ __forceinline__ void diag_pair_head1(float2 d, const float* c, float hi[8], float lo[8])
{
    const float4 v0 = ld_c(c), v1 = ld_c(c + 4);
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        hi[j] = __fmul_rn(d.x, v[j]);
        lo[j] = 0.f;
    }
}
__device__ __forceinline__ void diag_pair_tail1(float2 d, const float* c, float lo[8])
{
    const float4 v0 = ld_c(c), v1 = ld_c(c + 4);
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) lo[j] = __fadd_rn(lo[j], fmaf(d.y, v[j], fmaf(d.x, v[j], -__fmul_rn(d.x, v[j]))));
}

template <typename WT>
struct WLoad;

template <>
struct WLoad<float> {
    static __device__ __forceinline__ void load(const float* p, uint64_t pol, float w[8])
    {
        const uint4 a = ld_stream(p, pol), b = ld_stream(p + 4, pol);
        w[0] = __uint_as_float(a.x); w[1] = __uint_as_float(a.y); w[2] = __uint_as_float(a.z); w[3] = __uint_as_float(a.w);
        w[4] = __uint_as_float(b.x); w[5] = __uint_as_float(b.y); w[6] = __uint_as_float(b.z); w[7] = __uint_as_float(b.w);
    }
};

template <>
struct WLoad<__nv_bfloat16> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, uint64_t pol, float w[8])
    {
        const uint4 a = ld_stream(p, pol);
        const unsigned u[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[2 * i] = __uint_as_float(u[i] << 16);
            w[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
        }
    }
};

template <>
struct WLoad<__half> {
    static __device__ __forceinline__ void load(const __half* p, uint64_t pol, float w[8])
    {
        const uint4 a = ld_stream(p, pol);
        const unsigned u[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u[i]));
            w[2 * i] = f.x;
            w[2 * i + 1] = f.y;
        }
    }
};

// Raw 128-bit words of one weight slot (8 targets): 2 for fp32, 1 for fp16/bf16.
template <typename WT>
struct RawW {
    static constexpr int N = sizeof(WT) == 4 ? 2 : 1;
};

__device__ __forceinline__ void decode_w(const uint4 (&r)[2], float w[8])
{
    w[0] = __uint_as_float(r[0].x); w[1] = __uint_as_float(r[0].y); w[2] = __uint_as_float(r[0].z);
    w[3] = __uint_as_float(r[0].w); w[4] = __uint_as_float(r[1].x); w[5] = __uint_as_float(r[1].y);
    w[6] = __uint_as_float(r[1].z); w[7] = __uint_as_float(r[1].w);
}
template <typename WT>
__device__ __forceinline__ void decode_w(const uint4 (&r)[1], float w[8])
{
    const unsigned u[4] = {r[0].x, r[0].y, r[0].z, r[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if constexpr (std::is_same<WT, __nv_bfloat16>::value) {
            w[2 * i] = __uint_as_float(u[i] << 16);
            w[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
        } else {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u[i]));
            w[2 * i] = f.x;
            w[2 * i + 1] = f.y;
        }
    }
}

// Error-free addition (Knuth TwoSum): s + e == a + b exactly.
__device__ __forceinline__ void two_sum(float a, float b, float& s, float& e)
{
    s = __fadd_rn(a, b);
    const float bb = __fsub_rn(s, a);
    e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
}

// One (oz, oy) row: 2R+1 x-offsets (all of them, or all but the centre).  The row's
// products are summed in an fp32 FMA chain from 0 (a partial ~1/L² of the total), and
// the partial is added to the (hi, lo) fp32 pair error-free.  Without the pair, fp32
// round-off is systematic over homogeneous regions (identical kernels, identical C):
// −6.8e-6 relative mass per step at 192³ R5 bf16.
template <int R, typename WT, bool CENTRE_ROW>
__device__ __forceinline__ void do_row(const float* srow, const WT* wp, size_t wstride, uint64_t pol,
                                       float hi[8], float lo[8])
{
    float seg[24];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const float4 v = ld_c(srow + 4 * i);
        seg[4 * i] = v.x; seg[4 * i + 1] = v.y; seg[4 * i + 2] = v.z; seg[4 * i + 3] = v.w;
    }
    float w[2 * R + 1][8];
#pragma unroll
    for (int ox = -R; ox <= R; ++ox) {
        if (CENTRE_ROW && ox == 0) continue;
        const int k = CENTRE_ROW ? (ox < 0 ? ox + R : ox + R - 1) : ox + R;
        WLoad<WT>::load(wp + (size_t)k * wstride, pol, w[ox + R]);
    }
    float p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = 0.f;
#pragma unroll
    for (int ox = -R; ox <= R; ++ox) {
        if (CENTRE_ROW && ox == 0) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = fmaf(w[ox + R][j], seg[j - ox + 8], p[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s, e;
        two_sum(hi[j], p[j], s, e);
        hi[j] = s;
        lo[j] = __fadd_rn(lo[j], e);
    }
}

// Staged form (superpose_bulk_kernel): the row's weights were copied into shared memory by
// the TMA engine; thread e's 8 weights of slot k sit at wb + k·slotB (16 B, or 2 × 16 B for
// fp32).  Decode and arithmetic are do_row's exactly (identical bits).
__device__ __forceinline__ void load_seg(const float* srow, float seg[24])
{
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const float4 v = ld_c(srow + 4 * i);
        seg[4 * i] = v.x; seg[4 * i + 1] = v.y; seg[4 * i + 2] = v.z; seg[4 * i + 3] = v.w;
    }
}

template <int R, typename WT, bool CENTRE_ROW>
__device__ __forceinline__ void do_row_s(const float seg[24], const unsigned char* wb, uint32_t slotB, float hi[8],
                                         float lo[8])
{
    float p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = 0.f;
#pragma unroll
    for (int ox = -R; ox <= R; ++ox) {
        if (CENTRE_ROW && ox == 0) continue;
        const int k = CENTRE_ROW ? (ox < 0 ? ox + R : ox + R - 1) : ox + R;
        uint4 raw[RawW<WT>::N];
        raw[0] = *reinterpret_cast<const uint4*>(wb + (size_t)k * slotB);
        if constexpr (RawW<WT>::N == 2) raw[1] = *reinterpret_cast<const uint4*>(wb + (size_t)k * slotB + 16);
        float w[8];
        if constexpr (RawW<WT>::N == 2) decode_w(raw, w);
        else decode_w<WT>(raw, w);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = fmaf(w[j], seg[j - ox + 8], p[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s, e;
        two_sum(hi[j], p[j], s, e);
        hi[j] = s;
        lo[j] = __fadd_rn(lo[j], e);
    }
}

// Prefetching form (small grids): the raw weight words of a row are loaded into
// registers one row ahead, so each thread keeps two rows of weight loads in flight.  The
// arithmetic (seg, FMA chain in ox order from 0, TwoSum into (hi, lo)) is do_row's exactly.
template <int R, typename WT, int NS>
__device__ __forceinline__ void load_row_raw(const WT* wp, size_t wstride, uint64_t pol,
                                             uint4 (&raw)[2 * R + 1][RawW<WT>::N])
{
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        raw[k][0] = ld_stream(wp + (size_t)k * wstride, pol);
        if constexpr (RawW<WT>::N == 2) raw[k][1] = ld_stream(wp + (size_t)k * wstride + 4, pol);
    }
}

template <int R, typename WT, bool CENTRE_ROW>
__device__ __forceinline__ void fma_row_raw(const float* srow, const uint4 (&raw)[2 * R + 1][RawW<WT>::N],
                                            float hi[8], float lo[8])
{
    float seg[24];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const float4 v = ld_c(srow + 4 * i);
        seg[4 * i] = v.x; seg[4 * i + 1] = v.y; seg[4 * i + 2] = v.z; seg[4 * i + 3] = v.w;
    }
    float p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = 0.f;
#pragma unroll
    for (int ox = -R; ox <= R; ++ox) {
        if (CENTRE_ROW && ox == 0) continue;
        const int k = CENTRE_ROW ? (ox < 0 ? ox + R : ox + R - 1) : ox + R;
        float w[8];
        if constexpr (RawW<WT>::N == 2) decode_w(raw[k], w);
        else decode_w<WT>(raw[k], w);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = fmaf(w[j], seg[j - ox + 8], p[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s, e;
        two_sum(hi[j], p[j], s, e);
        hi[j] = s;
        lo[j] = __fadd_rn(lo[j], e);
    }
}

// N4: one (oz, oy) row with the weights of a uniform chunk — the class kernel's value for
// this slot, shared by all 8 targets, read from shared memory.  The same fmaf sequence and
// (hi, lo) update as do_row, so the result is bitwise the dense path's.
template <int R, bool CENTRE_ROW>
__device__ __forceinline__ void do_row_u(const float* srow, const float* ws, float hi[8], float lo[8])
{
    float seg[24];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const float4 v = ld_c(srow + 4 * i);
        seg[4 * i] = v.x; seg[4 * i + 1] = v.y; seg[4 * i + 2] = v.z; seg[4 * i + 3] = v.w;
    }
    float p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = 0.f;
#pragma unroll
    for (int ox = -R; ox <= R; ++ox) {
        if (CENTRE_ROW && ox == 0) continue;
        const int k = CENTRE_ROW ? (ox < 0 ? ox + R : ox + R - 1) : ox + R;
        const float w = ws[k];
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = fmaf(w, seg[j - ox + 8], p[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s, e;
        two_sum(hi[j], p[j], s, e);
        hi[j] = s;
        lo[j] = __fadd_rn(lo[j], e);
    }
}

// N4: a CTA = up to 256 uniform chunks of ONE class u; the class kernel (slot order, fp32
// values decoded from the storage format) is staged once in shared memory.  No weight bytes
// come from HBM: the chunk's cost is FMAs + L1-resident C reads.
template <int R>
__device__ __forceinline__ void uniform_body(const UniArgs& a, int blk, float* ws)
{
    constexpr int L = 2 * R + 1, K = L * L * L;
    const int4 b = a.blocks[blk];  // {start, count, u, -}
    for (int i = threadIdx.x; i < K - 1; i += blockDim.x) ws[i] = a.ukf[(size_t)b.z * (K - 1) + i];
    __syncthreads();
    if ((int)threadIdx.x >= b.y) return;
    const int chunk = a.list[b.x + threadIdx.x];
    const int tile = chunk / a.tile, e = chunk % a.tile;
    const int zl = tile / a.tpp, tp = tile % a.tpp;
    const int q = tp * a.tile + e;
    const int y = q / a.nxq, x = (q % a.nxq) * 8;
    const long nxp = a.nxp, plane = (long)a.nyp * nxp;
    const float* c0 = a.cpad + (zl + R) * plane + (long)(y + R) * nxp + kPadX + x;
    float hi[8], lo[8];
    const float2* dpt = a.udiag_t ? a.udiag_t + (size_t)(b.x + threadIdx.x) * 8 : nullptr;
    if (dpt) diag_pair_head(dpt, c0, hi, lo);  // MX8: per-target diagonal
    else diag_pair_head1(a.udiag[b.z], c0, hi, lo);  // the class's diagonal for all 8 targets
    do_row_u<R, true>(c0 - 8, ws, hi, lo);
    const float* wr = ws + (L - 1);
#pragma unroll 1
    for (int r = 0; r < L * L; ++r) {
        if (r == R * L + R) continue;
        const int oz = r / L - R, oy = r % L - R;
        do_row_u<R, false>(c0 - (long)oz * plane - (long)oy * nxp - 8, wr, hi, lo);
        wr += L;
    }
    if (dpt) diag_pair_tail(dpt, c0, lo);
    else diag_pair_tail1(a.udiag[b.z], c0, lo);
    float* out = a.out + (long)zl * a.out_ps + (long)y * a.out_rs + x;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(hi[j], lo[j]);
    if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        reinterpret_cast<float4*>(out)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        reinterpret_cast<float4*>(out)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) out[j] = acc[j];
    }
}

template <int R>
__global__ void __launch_bounds__(256) superpose_uniform_kernel(const UniArgs a)
{
    __shared__ float ws[(2 * R + 1) * (2 * R + 1) * (2 * R + 1) - 1];
    uniform_body<R>(a, blockIdx.x, ws);
}

template <int R>
static cudaError_t launch_uniform_r(const UniArgs& a, cudaStream_t s)
{
    if (a.n_blocks <= 0) return cudaSuccess;
    superpose_uniform_kernel<R><<<a.n_blocks, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_superpose_uniform(const UniArgs& a, int R, cudaStream_t s)
{
    switch (R) {
        case 1: return launch_uniform_r<1>(a, s);
        case 2: return launch_uniform_r<2>(a, s);
        case 3: return launch_uniform_r<3>(a, s);
        case 4: return launch_uniform_r<4>(a, s);
        case 5: return launch_uniform_r<5>(a, s);
        case 6: return launch_uniform_r<6>(a, s);
        case 7: return launch_uniform_r<7>(a, s);
        case 8: return launch_uniform_r<8>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

// Deterministic fp64 sum over the CTA (≤ 1024 threads): shuffle tree, then warps in order.
__device__ __forceinline__ double tile_block_sum(double s)
{
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    return t;  // valid in thread 0
}

// The tile a CTA works on, and thread e's chunk in it.
struct TileCtx {
    int tile, zl, y, x;
    bool real;          // false: dummy chunk past the end of the plane (or of the N4 list)
    const float* c0;    // C_old(z, y, x) in the padded state
    long nxp, plane;
};

template <int R>
__device__ __forceinline__ TileCtx tile_ctx(const SuperArgs& a, int blk, int e)
{
    TileCtx t;
    int tile = a.t_begin + blk;  // weight tile (compact tile when a.list, N4)
    if (a.gap_len) {
        const int nb = a.t_end - a.t_begin - a.gap_len;  // CTAs of the two outer bands
        if (a.gap_last && blk >= nb) tile = a.gap_at + (blk - nb);
        else if (tile >= a.gap_at) tile += a.gap_len;
    }
    int zl, q;
    bool real;
    if (a.list) {  // N4: tiles hold only the non-uniform chunks, in chunk order
        const long idx = (long)tile * a.tile + e;
        real = idx < a.n_list;
        const int chunk = real ? a.list[idx] : 0;
        const int ot = chunk / a.tile;
        zl = ot / a.tpp;
        q = (ot % a.tpp) * a.tile + chunk % a.tile;
    } else {
        zl = tile / a.tpp;
        q = (tile % a.tpp) * a.tile + e;
        real = q < a.ny * a.nxq;  // false: dummy chunk at the end of the plane
    }
    t.tile = tile;
    t.zl = zl;
    t.real = real;
    t.y = real ? q / a.nxq : 0;
    t.x = real ? (q % a.nxq) * 8 : 0;  // dummies: harmless reads
    t.nxp = a.nxp;
    t.plane = (long)a.nyp * t.nxp;
    t.c0 = a.cpad + (zl + R) * t.plane + (long)(t.y + R) * t.nxp + kPadX + t.x;
    return t;
}

// (hi, lo) = d·C_old(x) (the diagonal term first, DESIGN §6 order)
__device__ __forceinline__ void diag_init(const SuperArgs& a, const TileCtx& t, int e, float hi[8], float lo[8])
{
#pragma unroll
    for (int j = 0; j < 8; ++j) hi[j] = lo[j] = 0.f;
    if (!t.real) return;
    diag_pair_head(a.diag + ((size_t)t.tile * a.tile + e) * 8, t.c0, hi, lo);
}

// Stored row i of a tile (i = 0: the centre row, L − 1 slots; i ≥ 1: row r of (oz, oy)
// ascending with the centre skipped, L slots) → its source row pointer (C_old − 8).
template <int R>
__device__ __forceinline__ const float* row_src(const TileCtx& t, int i)
{
    constexpr int L = 2 * R + 1;
    if (i == 0) return t.c0 - 8;
    const int r = (i - 1) < R * L + R ? i - 1 : i;
    const int oz = r / L - R, oy = r % L - R;
    return t.c0 - (long)oz * t.plane - (long)oy * t.nxp - 8;
}

// acc = hi + lo; N2 boundary term; store; P2P halo pushes; N2 per-tile Σ.  Every thread of
// the CTA calls it (tile_sum's reduction is CTA-wide).
__device__ __forceinline__ void tile_epilogue(const SuperArgs& a, const TileCtx& t, int e, const float hi[8],
                                              const float lo[8])
{
    const int x = t.x, y = t.y, zl = t.zl, tile = t.tile;
    const bool real = t.real;
    const long nxp = t.nxp, plane = t.plane;
    float acc[8];
    float lo2[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) lo2[j] = lo[j];
    if (real) diag_pair_tail(a.diag + ((size_t)tile * a.tile + e) * 8, t.c0, lo2);  // the diagonal's tail
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(hi[j], lo2[j]);
    if (a.pbc) {  // N2: + p_BC(x)·c_far(t)  (Eq.8 boundary term; 0 on far-field targets)
        const float cf = (float)a.far_state[0];
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(a.pbc + ((size_t)tile * a.tile + e) * 8));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(a.pbc + ((size_t)tile * a.tile + e) * 8 + 4));
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(b[j], cf, acc[j]);
    }
    if (real) {
        float* out = a.out + (long)zl * a.out_ps + (long)y * a.out_rs + x;
        if (x + 8 <= a.nx && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            reinterpret_cast<float4*>(out)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            reinterpret_cast<float4*>(out)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (x + j < a.nx) out[j] = acc[j];
        }
        // a6 over peer memory: the first / last R planes also go straight into the
        // neighbours' halo planes (P2P stores over NVLink), fenced before the step's signal
        float* pd[2] = {nullptr, nullptr};
        if (a.push_lo && zl < a.pR) pd[0] = a.push_lo + (long)zl * plane + (long)y * nxp + x;
        if (a.push_hi && zl >= a.nzl - a.pR) pd[1] = a.push_hi + (long)(zl - (a.nzl - a.pR)) * plane + (long)y * nxp + x;
        if (pd[0] || pd[1]) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!pd[h]) continue;
                if (x + 8 <= a.nx) {
                    reinterpret_cast<float4*>(pd[h])[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                    reinterpret_cast<float4*>(pd[h])[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (x + j < a.nx) pd[h][j] = acc[j];
                }
            }
            __threadfence_system();
        }
    }
    if (a.tile_sum) {  // N2: this tile's Σ C_new (fp64, fixed order) for Eq.7
        double s = 0.0;
        if (real) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (x + j < a.nx) s += (double)acc[j];
        }
        s = tile_block_sum(s);
        if (threadIdx.x == 0) a.tile_sum[tile] = s;
    }
}

template <int R, typename WT, bool PF = false>
__device__ __forceinline__ void dense_body(const SuperArgs& a, int blk)
{
    constexpr int L = 2 * R + 1, K = L * L * L;
    const int e = threadIdx.x;
    const TileCtx t = tile_ctx<R>(a, blk, e);
    if (!t.real && a.tile_sum == nullptr) return;
    size_t wstride = (size_t)a.tile * 8;
    const WT* wt = reinterpret_cast<const WT*>(a.Wt) + ((size_t)t.tile * (K - 1) * a.tile + e) * 8;
    uint64_t pol = evict_first_policy();
    const float* c0 = t.c0;
    const long nxp = t.nxp, plane = t.plane;

    float hi[8], lo[8];
    diag_init(a, t, e, hi, lo);
    if (t.real) {
        if constexpr (PF) {
            // same rows in the same order, each row's weights loaded while the previous row
            // computes (ping-pong register buffers; L² − 1 is even)
            uint4 ra[L][RawW<WT>::N], rb[L][RawW<WT>::N];
            const WT* wr = wt + (size_t)(L - 1) * wstride;
            load_row_raw<R, WT, L - 1>(wt, wstride, pol, ra);
            load_row_raw<R, WT, L>(wr, wstride, pol, rb);
            fma_row_raw<R, WT, true>(c0 - 8, ra, hi, lo);
            constexpr int NR = L * L - 1, RC = R * L + R;
#pragma unroll 1
            for (int i = 0; i < NR; i += 2) {
                const int r0 = i < RC ? i : i + 1, r1 = i + 1 < RC ? i + 1 : i + 2;
                if (i + 1 < NR) load_row_raw<R, WT, L>(wr + (size_t)L * wstride, wstride, pol, ra);
                fma_row_raw<R, WT, false>(c0 - (long)(r0 / L - R) * plane - (long)(r0 % L - R) * nxp - 8, rb, hi, lo);
                wr += (size_t)L * wstride;
                if (i + 1 >= NR) break;
                if (i + 2 < NR) load_row_raw<R, WT, L>(wr + (size_t)L * wstride, wstride, pol, rb);
                fma_row_raw<R, WT, false>(c0 - (long)(r1 / L - R) * plane - (long)(r1 % L - R) * nxp - 8, ra, hi, lo);
                wr += (size_t)L * wstride;
            }
        } else {
        // centre row (oz = oy = 0): slots [0, L−1)
        do_row<R, WT, true>(c0 - 8, wt, wstride, pol, hi, lo);
        // remaining rows, ascending (oz, oy); source row of target row (z, y) is (z − oz, y − oy)
        const WT* wr = wt + (size_t)(L - 1) * wstride;
#pragma unroll 1
        for (int r = 0; r < L * L; ++r) {
            if (r == R * L + R) continue;
            const int oz = r / L - R, oy = r % L - R;
            const float* srow = c0 - (long)oz * plane - (long)oy * nxp - 8;
            do_row<R, WT, false>(srow, wr, wstride, pol, hi, lo);
            wr += (size_t)L * wstride;
        }
        }
    }

    tile_epilogue(a, t, e, hi, lo);
}

template <int R, typename WT, bool PF>
__global__ void __launch_bounds__(256) superpose_kernel(const SuperArgs a)
{
    dense_body<R, WT, PF>(a, blockIdx.x);
}

// TMA-staged weight stream (default for dense tiles of 256 chunks).  A CTA = one tile:
// warps 0-7 compute (thread e = chunk e, exactly dense_body's arithmetic), warp 8's lane 0
// streams the tile's contiguous weight region row by row (one stored row = L or L − 1 slots
// of tile·8 weights: 44 KB at R5 bf16) with cp.async.bulk into a ring of S shared-memory
// stages.  full[st] completes when a row's bytes have landed (expect_tx), empty[st] when all 8
// compute warps have read it; the producer refills stage st for row i + S only after that.
// The weight bytes in flight no longer depend on how many warps are waiting on loads: each
// SM keeps up to 2 CTAs × S rows outstanding with one thread issuing them.
constexpr int kBulkWarps = 8;  // at most: a tile of ≤ 256 chunks = a.tile/32 compute warps
// sub = chunks per CTA: the whole tile (sub = a.tile), or a part of it (a.tile / sub CTAs per
// tile, CTA blk → tile blk / nsub, part blk % nsub) so that short launches quantise into
// smaller units (wave balance, see launch_superpose_r).  A part's weights for one slot are a
// contiguous sub·8 run inside the tile's slot block: the producer copies them slot by slot.
// fdirw_debug_stage_canary: compare this thread's 16 / 32 B of every slot of stored row i in the
// stage with the same bytes in global memory (plain coherent loads).  Row i starts at slot 0 for
// i = 0 (the centre row, L − 1 slots) and at slot (L − 1) + (i − 1)·L otherwise.
template <typename WT>
__device__ __noinline__ void stage_canary(const SuperArgs& a, const TileCtx& t, int e, int i, int L,
                                          const unsigned char* wb, uint32_t subB)
{
    const int n = i == 0 ? L - 1 : L, k0 = i == 0 ? 0 : (L - 1) + (i - 1) * L;
    const size_t slotE = (size_t)a.tile * 8;  // elements per slot of the whole tile
    const WT* g = reinterpret_cast<const WT*>(a.Wt) + ((size_t)t.tile * (a.K - 1) + k0) * slotE + (size_t)e * 8;
    unsigned long long bad = 0;
    for (int k = 0; k < n; ++k) {
        const uint4* gs = reinterpret_cast<const uint4*>(g + (size_t)k * slotE);
        const uint4* ss = reinterpret_cast<const uint4*>(wb + (size_t)k * subB);
        for (int w = 0; w < RawW<WT>::N; ++w) {
            const uint4 x = gs[w], y = ss[w];
            bad += (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
        }
    }
    atomicAdd(a.canary, (unsigned long long)n * RawW<WT>::N);
    if (bad) atomicAdd(a.canary + 1, bad);
}

template <int R, typename WT>
__device__ __forceinline__ void bulk_body(const SuperArgs& a, int blk, int S, int sub, unsigned char* smem_b)
{
    constexpr int L = 2 * R + 1, K = L * L * L, NROW = L * L;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_b);
    uint64_t* empty = full + S;
    unsigned char* stg = smem_b + 128;
    const int nsub = a.tile / sub, part = blk % nsub;
    const uint32_t slotB = (uint32_t)a.tile * 8 * sizeof(WT);  // one slot of the whole tile
    const uint32_t subB = (uint32_t)sub * 8 * sizeof(WT), stageB = (uint32_t)L * subB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = sub >> 5;  // compute warps
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(smem_u32(full + i), 1);
            mbar_init(smem_u32(empty + i), nw);
        }
        mbar_init_fence();
    }
    __syncthreads();
    const bool producer = warp == nw;
    const int e = part * sub + (producer ? 0 : (int)threadIdx.x);
    TileCtx t = tile_ctx<R>(a, blk / nsub, e);
    float hi[8], lo[8];
    if (producer) {
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            const unsigned char* src = reinterpret_cast<const unsigned char*>(a.Wt) +
                                       (size_t)t.tile * (K - 1) * slotB + (size_t)part * subB;
            for (int i = 0; i < NROW; ++i) {
                const int st = i % S, u = i / S;
                const int n = i == 0 ? L - 1 : L;
                if (u > 0) mbar_wait(smem_u32(empty + st), (u - 1) & 1);
                mbar_expect_tx(smem_u32(full + st), (uint32_t)n * subB);
                if (nsub == 1) {
                    bulk_g2s(smem_u32(stg + (size_t)st * stageB), src, (uint32_t)n * subB, smem_u32(full + st), pol);
                } else {
                    for (int k = 0; k < n; ++k)
                        bulk_g2s(smem_u32(stg + (size_t)st * stageB + (size_t)k * subB), src + (size_t)k * slotB, subB,
                                 smem_u32(full + st), pol);
                }
                src += (size_t)n * slotB;
            }
        }
        t.real = false;  // joins the epilogue only for tile_sum's CTA-wide reduction
#pragma unroll
        for (int j = 0; j < 8; ++j) hi[j] = lo[j] = 0.f;
    } else {
        diag_init(a, t, e, hi, lo);
        const unsigned char* wb = stg + (size_t)threadIdx.x * 8 * sizeof(WT);
        // the row's C segment is loaded before waiting for its weights (the L1/L2 latency
        // overlaps the stage's arrival)
        float seg[24];
        for (int i = 0; i < NROW; ++i) {
            const int st = i % S, u = i / S;
            if (t.real) load_seg(row_src<R>(t, i), seg);
            mbar_wait(smem_u32(full + st), u & 1);
            if (a.canary && t.real) stage_canary<WT>(a, t, e, i, L, wb + (size_t)st * stageB, subB);
            if (t.real) {
                if (i == 0) do_row_s<R, WT, true>(seg, wb + (size_t)st * stageB, subB, hi, lo);
                else do_row_s<R, WT, false>(seg, wb + (size_t)st * stageB, subB, hi, lo);
            }
            if (a.canary && t.real) stage_canary<WT>(a, t, e, i, L, wb + (size_t)st * stageB, subB);
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(empty + st));
        }
    }
    tile_epilogue(a, t, e, hi, lo);
}

template <int R, typename WT>
__global__ void __launch_bounds__((kBulkWarps + 1) * 32) superpose_bulk_kernel(const SuperArgs a, int S, int sub)
{
    extern __shared__ __align__(128) unsigned char smem_b[];
    bulk_body<R, WT>(a, blockIdx.x, S, sub, smem_b);
}

// FDIRW_W_MX8 (mx8.cuh): one stored row of the tile = n slots × (T·8 mantissa bytes)
// then n × T scale bytes, staged like bulk_body's rows (whole tiles only).  Per slot thread e
// reads its 8 mantissas (LDS.64) and its block's exponent byte; weight j is decoded exactly as
// fma(2^23 + m_j, s, −2^23·s) = m_j·s, with 2^23 + m_j built by one byte permute
// (0x4B0000·m_j as fp32 bits), then the FMA chain and TwoSum of do_row_s.  The kernel is
// issue-bound (ncu: ~74 % issue slots at the first version), so everything per row that is not
// decode + FMA is kept out of the loop: TT = the tile width as a compile-time constant (256, the
// closed-domain default; 0 = runtime), stage/phase counters instead of divisions, row pointers
// stepped instead of recomputed.
__device__ __forceinline__ unsigned long long pk2f(float a, float b)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2f(unsigned long long v, float& a, float& b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long fma2f(unsigned long long a, unsigned long long b, unsigned long long c)
{
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// One stored row's slots into the partial sums p (FMA chain in slot order).  The decode runs
// two weights per FFMA2 (each lane an ordinary fp32 fma: exact here, the scale and bias as
// broadcast operands); the accumulation stays scalar: an FFMA2 there needs the C pairs
// (seg[i], seg[i+1]) at odd i, which are not register pairs (measured: the re-pairing moves
// cost more than the FFMA2 saves).
template <int R, bool CENTRE_ROW, int TT>
__device__ __forceinline__ void row_mx8(const float seg[24], const unsigned char* mb, const unsigned char* sb, int T_,
                                        float p[8])
{
    const int T = TT ? TT : T_;
#pragma unroll
    for (int ox = -R; ox <= R; ++ox) {
        if (CENTRE_ROW && ox == 0) continue;
        const int k = CENTRE_ROW ? (ox < 0 ? ox + R : ox + R - 1) : ox + R;
        const uint2 m = *reinterpret_cast<const uint2*>(mb + k * 8 * T);
        const uint32_t E = sb[k * T];
        const float sc = __uint_as_float(E << 23), bias = __uint_as_float(((E + 23u) << 23) | 0x80000000u);
        const unsigned long long sc2 = pk2f(sc, sc), b2 = pk2f(bias, bias);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const unsigned wd = h < 2 ? m.x : m.y;
            const float f0 = __uint_as_float(__byte_perm(wd, 0x4B000000u, 0x7440u | (unsigned)((2 * h) & 3)));
            const float f1 = __uint_as_float(__byte_perm(wd, 0x4B000000u, 0x7440u | (unsigned)((2 * h + 1) & 3)));
            float w0, w1;
            upk2f(fma2f(pk2f(f0, f1), sc2, b2), w0, w1);
            p[2 * h] = fmaf(w0, seg[2 * h - ox + 8], p[2 * h]);
            p[2 * h + 1] = fmaf(w1, seg[2 * h + 1 - ox + 8], p[2 * h + 1]);
        }
    }
}

// (hi, lo) += p error-free (Knuth TwoSum), p = 0
__device__ __forceinline__ void flush_mx8(float p[8], float hi[8], float lo[8])
{
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s, e2;
        two_sum(hi[j], p[j], s, e2);
        hi[j] = s;
        lo[j] = __fadd_rn(lo[j], e2);
        p[j] = 0.f;
    }
}

// rows per fp32 partial before the error-free add: the most rows of ≤ 44 slots in all that
// divide L² − 1 (R5: 4 rows; R8: 2).  A partial's fp32 round-off is systematic over
// homogeneous regions, so it is bounded in slots, not rows (cfg5 mass drift: DESIGN §15)
constexpr int mx8_rows(int R)
{
    int g = 44 / (2 * R + 1);
    while (g > 1 && ((2 * R + 1) * (2 * R + 1) - 1) % g != 0) --g;
    return g < 1 ? 1 : g;
}
template <int R, int TT>
__device__ __forceinline__ void mx8_body(const SuperArgs& a, int blk, int S, unsigned char* smem_b, int nsub = 1)
{
    // nsub > 1 (one-wave launches): the CTA takes part blk % nsub of tile blk / nsub, T chunks of
    // the tile's Tf; its stage holds the part's runs of every slot in the same [n][T][8] +
    // [n][T] layout (2 bulk copies per slot instead of 1 per row).  Same arithmetic per thread.
    constexpr int L = 2 * R + 1, K = L * L * L, NROW = L * L;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_b);
    uint64_t* empty = full + S;
    unsigned char* stg = smem_b + 128;
    const int Tf = a.tile;
    const int T = TT ? TT : Tf / nsub;
    const int part = blk % nsub;
    blk /= nsub;
    const uint32_t slotB = (uint32_t)T * 9, stageB = (uint32_t)L * slotB, slotBf = (uint32_t)Tf * 9;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = T >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(smem_u32(full + i), 1);
            mbar_init(smem_u32(empty + i), nw);
        }
        mbar_init_fence();
    }
    __syncthreads();
    const bool producer = warp == nw;
    const int e = part * T + (producer ? 0 : (int)threadIdx.x);
    TileCtx t = tile_ctx<R>(a, blk, e);
    float hi[8], lo[8];
    if (producer) {
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            const unsigned char* src = reinterpret_cast<const unsigned char*>(a.Wt) + (size_t)t.tile * (K - 1) * slotBf;
            int st = 0;
            uint32_t ph = 0;  // parity of the empty barrier to wait for (from the second lap)
            for (int i = 0; i < NROW; ++i) {
                const int n = i == 0 ? L - 1 : L;
                if (i >= S) mbar_wait(smem_u32(empty + st), ph);
                mbar_expect_tx(smem_u32(full + st), (uint32_t)n * slotB);
                unsigned char* dst = stg + (size_t)st * stageB;
                if (nsub == 1) {
                    bulk_g2s(smem_u32(dst), src, (uint32_t)n * slotB, smem_u32(full + st), pol);
                } else {
                    for (int k = 0; k < n; ++k) {
                        bulk_g2s(smem_u32(dst + (size_t)k * 8 * T), src + (size_t)k * 8 * Tf + (size_t)part * 8 * T,
                                 (uint32_t)(8 * T), smem_u32(full + st), pol);
                        bulk_g2s(smem_u32(dst + (size_t)n * 8 * T + (size_t)k * T),
                                 src + (size_t)n * 8 * Tf + (size_t)k * Tf + (size_t)part * T, (uint32_t)T,
                                 smem_u32(full + st), pol);
                    }
                }
                src += (size_t)n * slotBf;
                if (++st == S) {
                    st = 0;
                    if (i >= S) ph ^= 1u;
                }
            }
        }
        t.real = false;
#pragma unroll
        for (int j = 0; j < 8; ++j) hi[j] = lo[j] = 0.f;
    } else {
        diag_init(a, t, e, hi, lo);
        float seg[24], p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = 0.f;
        const unsigned char* m0 = stg + (size_t)threadIdx.x * 8;     // this thread's mantissas in stage 0
        const unsigned char* s0 = stg + (size_t)8 * T + threadIdx.x;  // its scales (after n·8T bytes; n folded below)
        int st = 0;
        uint32_t ph = 0;
        // row i = 0: the centre row; then (oz, oy) ascending without the centre (row_src order)
        // source row of stored row i: C_old − oz·plane − oy·nxp − 8 (32-bit offsets: the padded
        // state is < 2^31 elements)
        const int pl = (int)t.plane, nx_ = (int)t.nxp;
        int oz = 0, oy = 0;
        for (int i = 0; i < NROW; ++i) {
            if (t.real) load_seg(t.c0 + (-oz * pl - oy * nx_ - 8), seg);
            mbar_wait(smem_u32(full + st), ph);
            if (t.real) {
                // partial sums over the centre row, then over groups of mx8_rows(R) rows (L² − 1 =
                // 4R(R+1) is a multiple of 8), each added to (hi, lo) error-free
                const unsigned char* mb = m0 + st * stageB;
                if (i == 0) {
                    row_mx8<R, true, TT>(seg, mb, s0 + st * stageB + (L - 2) * 8 * T, T, p);
                    flush_mx8(p, hi, lo);
                } else {
                    row_mx8<R, false, TT>(seg, mb, s0 + st * stageB + (L - 1) * 8 * T, T, p);
                    if (i % mx8_rows(R) == 0) flush_mx8(p, hi, lo);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(empty + st));
            if (++st == S) {
                st = 0;
                ph ^= 1u;
            }
            if (i == 0) {  // after the centre row: (oz, oy) = (−R, −R), then ascending, centre skipped
                oz = -R;
                oy = -R;
            } else {
                if (++oy > R) {
                    oy = -R;
                    ++oz;
                }
                if (oz == 0 && oy == 0) oy = 1;
            }
        }
    }
    tile_epilogue(a, t, e, hi, lo);
}

template <int R, int TT>
__global__ void __launch_bounds__((kBulkWarps + 1) * 32, 3) superpose_mx8_kernel(const SuperArgs a, int S, int nsub)
{
    extern __shared__ __align__(128) unsigned char smem_b[];
    mx8_body<R, TT>(a, blockIdx.x, S, smem_b, nsub);
}

// MX8 uniform blocks: uniform_body's work with the MX8 body's summation grouping (the centre
// row, then groups of mx8_rows(R) rows into one fp32 partial before the TwoSum).  The decoded
// weights are the dense MX8 layout's, so the field is bitwise the dense MX8 path's.
template <int R>
__device__ __forceinline__ void uniform_body_mx8(const UniArgs& a, int blk, float* ws)
{
    constexpr int L = 2 * R + 1, K = L * L * L, G = mx8_rows(R);
    const int4 b = a.blocks[blk];  // {start, count, u, -}
    for (int i = threadIdx.x; i < K - 1; i += blockDim.x) ws[i] = a.ukf[(size_t)b.z * (K - 1) + i];
    __syncthreads();
    if ((int)threadIdx.x >= b.y) return;
    const int chunk = a.list[b.x + threadIdx.x];
    const int tile = chunk / a.tile, e = chunk % a.tile;
    const int zl = tile / a.tpp, tp = tile % a.tpp;
    const int q = tp * a.tile + e;
    const int y = q / a.nxq, x = (q % a.nxq) * 8;
    const long nxp = a.nxp, plane = (long)a.nyp * nxp;
    const float* c0 = a.cpad + (zl + R) * plane + (long)(y + R) * nxp + kPadX + x;
    float hi[8], lo[8], p[8];
    diag_pair_head(a.udiag_t + (size_t)(b.x + threadIdx.x) * 8, c0, hi, lo);
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = 0.f;
    float seg[24];
    int n = 0;  // stored row index (0: the centre row)
    const float* wr = ws;
    for (int oz = -R - 1; oz <= R; ++oz) {  // oz = −R − 1 stands for the centre row
#pragma unroll 1
        for (int oy = -R; oy <= R; ++oy) {
            const bool centre = oz == -R - 1;
            if (centre && oy > -R) break;
            if (!centre && oz == 0 && oy == 0) continue;
            load_seg(centre ? c0 - 8 : c0 - (long)oz * plane - (long)oy * nxp - 8, seg);
#pragma unroll
            for (int ox = -R; ox <= R; ++ox) {
                if (centre && ox == 0) continue;
                const int k = centre ? (ox < 0 ? ox + R : ox + R - 1) : ox + R;
                const float w = wr[k];
#pragma unroll
                for (int j = 0; j < 8; ++j) p[j] = fmaf(w, seg[j - ox + 8], p[j]);
            }
            wr += centre ? L - 1 : L;
            if (n == 0 || n % G == 0) flush_mx8(p, hi, lo);
            ++n;
        }
    }
    diag_pair_tail(a.udiag_t + (size_t)(b.x + threadIdx.x) * 8, c0, lo);
    float* out = a.out + (long)zl * a.out_ps + (long)y * a.out_rs + x;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(hi[j], lo[j]);
    if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        reinterpret_cast<float4*>(out)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        reinterpret_cast<float4*>(out)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) out[j] = acc[j];
    }
}

// MX8 with N4 storage: the mixed launch of superpose_mixed_bulk_kernel with MX8 dense tiles.
template <int R>
__global__ void __launch_bounds__((kBulkWarps + 1) * 32, 3) superpose_mx8_mixed_kernel(const SuperArgs a,
                                                                                      const UniArgs u, int S)
{
    extern __shared__ __align__(128) unsigned char smem_b[];
    const long T = gridDim.x, U = u.n_blocks, b = blockIdx.x;
    const long u0 = b * U / T, u1 = (b + 1) * U / T;
    if (u1 > u0) uniform_body_mx8<R>(u, (int)u0, reinterpret_cast<float*>(smem_b + 128));
    else mx8_body<R, 256>(a, (int)(b - u0), S, smem_b);
}

// N4 with the staged stream: the mixed launch's dense tiles run bulk_body, its uniform blocks
// uniform_body with the class kernel in the (otherwise unused) stage memory.
template <int R, typename WT>
__global__ void __launch_bounds__((kBulkWarps + 1) * 32) superpose_mixed_bulk_kernel(const SuperArgs a, const UniArgs u,
                                                                                     int S)
{
    extern __shared__ __align__(128) unsigned char smem_b[];
    const long T = gridDim.x, U = u.n_blocks, b = blockIdx.x;
    const long u0 = b * U / T, u1 = (b + 1) * U / T;
    if (u1 > u0) uniform_body<R>(u, (int)u0, reinterpret_cast<float*>(smem_b + 128));
    else bulk_body<R, WT>(a, (int)(b - u0), S, a.tile, smem_b);
}

// stages of the bulk kernel: 2 CTAs per SM with ≥ 2 stages each, else 1 CTA with ≥ 2; 0 = the
// row does not fit twice (register path)
static int bulk_stages(int R, int b_w, int tile, int* ctas_per_sm)
{
    const size_t row = (size_t)(2 * R + 1) * tile * 8 * b_w, avail = 227 * 1024 - 128;
    const size_t half = (228 * 1024) / 2 - 1024 - 128;  // per CTA at 2 CTAs/SM (1 KB reserved each)
    int S = (int)(half / row);
    if (S >= 2) {
        *ctas_per_sm = 2;
        return S > 8 ? 8 : S;
    }
    S = (int)(avail / row);
    *ctas_per_sm = 1;
    return S >= 2 ? (S > 8 ? 8 : S) : 0;
}

// N4: ONE launch mixing the HBM-bound dense tiles and the FMA-bound uniform blocks, the U
// uniform blocks spread evenly over the grid (block b is uniform iff ⌊(b+1)U/T⌋ > ⌊bU/T⌋),
// so every SM streams weights and runs uniform FMAs at the same time.
template <int R, typename WT>
__global__ void __launch_bounds__(256) superpose_mixed_kernel(const SuperArgs a, const UniArgs u)
{
    __shared__ float ws[(2 * R + 1) * (2 * R + 1) * (2 * R + 1) - 1];
    const long T = gridDim.x, U = u.n_blocks, b = blockIdx.x;
    const long u0 = b * U / T, u1 = (b + 1) * U / T;
    if (u1 > u0) uniform_body<R>(u, (int)u0, ws);
    else dense_body<R, WT>(a, (int)(b - u0));
}

// prefetch buffers are 2·L·(1 or 2) 128-bit words: only where they fit the registers
template <int R, typename WT>
struct PfOK {
    static constexpr bool v = (2 * R + 1) * RawW<WT>::N <= 18;
};
template <int R>
constexpr bool kPrefetchOK(int fmt)
{
    return fmt == 0 ? PfOK<R, float>::v : PfOK<R, __half>::v;
}

template <int R>
static cudaError_t launch_superpose_r(const SuperArgs& a, int fmt, cudaStream_t s)
{
    const int nblk = a.t_end - a.t_begin - (a.gap_last ? 0 : a.gap_len);
    if (nblk <= 0) return cudaSuccess;
    if (fmt == FDIRW_W_MX8) {  // staged stream only (whole tiles), at any launch size
        if (a.tile % 32 != 0 || a.tile > kBulkWarps * 32) return cudaErrorInvalidValue;
        const size_t row = (size_t)(2 * R + 1) * a.tile * 9, half = (228 * 1024) / 2 - 1024 - 128;
        int S = (int)(half / row);
        if (S < 2) S = (int)((227 * 1024 - 128) / row);
        if (S > 3) S = 3;  // measured at cfg3: 3 stages 1.74 ms, 4: 1.79, 2 (3 CTAs/SM): 1.76
        // wave balance (the tile stays 256 for MX8, see make_geometry's caller): 2 stages give
        // 3 CTAs/SM; take them when waves × CTAs-per-SM (∝ time when bandwidth-shared) drops,
        // e.g. a 24-plane slab (432 tiles) fits one wave of 444 instead of 1.5 of 296
        if (S == 3 && (long)3 * ((nblk + 443) / 444) < (long)2 * ((nblk + 295) / 296)) S = 2;
        if (const char* ev = getenv("FDIRW_MX8_STAGES")) S = atoi(ev);  // A/B of the stage count
        if (S < 2 || S > 8) return cudaErrorInvalidValue;  // the 128-byte barrier header holds 8 + 8
        // Tile split (FDIRW_MX8_NSUB = 2 / 4, A/B only): parts of a tile as separate CTAs, for
        // one-wave launches.  Measured slower at cfg2 (128 tiles: whole 0.059 ms, auto-split
        // into 256 CTAs 0.073 ms — 2 copies per slot and the runtime-width body cost more than
        // the 20 idle SMs), so whole tiles stay the default.
        int nsub = 1;
        if (const char* ev = getenv("FDIRW_MX8_NSUB")) nsub = atoi(ev);
        if (nsub < 1 || a.tile % nsub != 0 || (a.tile / nsub) % 32 != 0 || (nsub > 1 && a.tile_sum))
            return cudaErrorInvalidValue;
        const size_t smem = 128 + (size_t)S * (row / nsub);
        const bool t256 = a.tile == 256 && nsub == 1;
        const void* f = t256 ? (const void*)superpose_mx8_kernel<R, 256> : (const void*)superpose_mx8_kernel<R, 0>;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (t256) superpose_mx8_kernel<R, 256><<<nblk, a.tile + 32, smem, s>>>(a, S, 1);
        else superpose_mx8_kernel<R, 0><<<nblk * nsub, a.tile / nsub + 32, smem, s>>>(a, S, nsub);
        return cudaGetLastError();
    }
    // a launch of fewer than two CTAs per SM cannot keep enough weight loads in flight
    // through occupancy: those threads prefetch one row ahead instead (identical bits)
    // TMA-staged weight stream for launches of ≥ 2 CTAs per SM (the common case); the
    // register-prefetching body below for smaller launches (one wave: no CTA to overlap the
    // pipeline fill with) or FDIRW_F_NO_BULK_STREAM.  Identical bits either way.
    const int b_w = fmt == 0 ? 4 : 2;
    int cps = 0;
    const int S1 = (a.tile % 32 == 0 && a.tile <= kBulkWarps * 32) ? bulk_stages(R, b_w, a.tile, &cps) : 0;
    // Wave balance (e.g. the compacted tiles of an open domain, N2/N3): split each tile into
    // nsub ∈ {1, 2, 4} parts of a.tile/nsub chunks (≥ 64), at the same CTAs per SM, when the
    // modelled time waves·(chunks per CTA) drops; a split launch must still fill the GPU once
    // (2 CTAs/SM × 148) so the stage pipelines' fill overlaps.  Not with in-kernel per-tile
    // sums (N2 multi-rank Eq.7), which need the whole tile.
    // Parts keep ≥ 128 chunks (measured: 64-chunk parts, 1 KB per slot copy, lose to the
    // register-prefetch body at cfg2 and to whole tiles at cfg3), and only launches of < 4
    // waves are split at all.
    int nsub = 0;
    if (!a.no_bulk && S1 > 0) {
        const long slots = (long)cps * 148;
        const int dmax = (a.tile_sum || nblk >= 4 * slots) ? 1 : 4;
        long best = -1;
        for (int d = 1; d <= dmax && a.tile / d >= 128 && (a.tile / d) % 32 == 0; d *= 2) {
            if ((long)nblk * d < 2 * 148) continue;
            const long cost = (((long)nblk * d + slots - 1) / slots) * (a.tile / d);
            if (best < 0 || cost < best) { best = cost; nsub = d; }
        }
    }
    if (nsub > 0) {
        {
            const int sub = a.tile / nsub;
            int S = S1 * nsub;  // same shared memory per CTA: stages of a part are nsub× smaller
            if (S > 8) S = 8;
            const size_t smem = 128 + (size_t)S * (2 * R + 1) * sub * 8 * b_w;
            const void* f = fmt == 0 ? (const void*)superpose_bulk_kernel<R, float>
                          : fmt == 1 ? (const void*)superpose_bulk_kernel<R, __half>
                                     : (const void*)superpose_bulk_kernel<R, __nv_bfloat16>;
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            const int nt = sub + 32;
            const int grid = nblk * nsub;
            if (fmt == 0) superpose_bulk_kernel<R, float><<<grid, nt, smem, s>>>(a, S, sub);
            else if (fmt == 1) superpose_bulk_kernel<R, __half><<<grid, nt, smem, s>>>(a, S, sub);
            else superpose_bulk_kernel<R, __nv_bfloat16><<<grid, nt, smem, s>>>(a, S, sub);
            return cudaGetLastError();
        }
    }
    const bool pf = nblk < 2 * 148 && kPrefetchOK<R>(fmt);
    if (pf) {
        if (fmt == 0) superpose_kernel<R, float, PfOK<R, float>::v><<<nblk, a.tile, 0, s>>>(a);
        else if (fmt == 1) superpose_kernel<R, __half, PfOK<R, __half>::v><<<nblk, a.tile, 0, s>>>(a);
        else superpose_kernel<R, __nv_bfloat16, PfOK<R, __nv_bfloat16>::v><<<nblk, a.tile, 0, s>>>(a);
    } else {
        if (fmt == 0) superpose_kernel<R, float, false><<<nblk, a.tile, 0, s>>>(a);
        else if (fmt == 1) superpose_kernel<R, __half, false><<<nblk, a.tile, 0, s>>>(a);
        else superpose_kernel<R, __nv_bfloat16, false><<<nblk, a.tile, 0, s>>>(a);
    }
    return cudaGetLastError();
}

template <int R>
static cudaError_t launch_mixed_r(const SuperArgs& a, const UniArgs& u, int fmt, cudaStream_t s)
{
    const int nblk = (a.t_end - a.t_begin) + u.n_blocks;
    if (nblk <= 0) return cudaSuccess;
    if (a.tile != 256) return cudaErrorInvalidValue;  // uniform blocks are 256 chunks
    if (fmt == FDIRW_W_MX8) {  // staged MX8 stream for the dense tiles, at any launch size
        const size_t row = (size_t)(2 * R + 1) * a.tile * 9, half = (228 * 1024) / 2 - 1024 - 128;
        int S = (int)(half / row);
        if (S < 2) S = (int)((227 * 1024 - 128) / row);
        if (S > 3) S = 3;
        if (const char* ev = getenv("FDIRW_MX8_STAGES")) S = atoi(ev);  // A/B of the stage count
        if (S < 2 || S > 8) return cudaErrorInvalidValue;  // the 128-byte barrier header holds 8 + 8
        size_t smem = 128 + (size_t)S * row;
        const size_t need = 128 + (size_t)((2 * R + 1) * (2 * R + 1) * (2 * R + 1) - 1) * 4;  // uniform kernel
        if (smem < need) smem = need;
        cudaError_t e = cudaFuncSetAttribute(superpose_mx8_mixed_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        superpose_mx8_mixed_kernel<R><<<nblk, a.tile + 32, smem, s>>>(a, u, S);
        return cudaGetLastError();
    }
    if (!a.no_bulk && nblk >= 2 * 148) {
        const int b_w = fmt == 0 ? 4 : 2;
        int cps = 0;
        const int S = bulk_stages(R, b_w, a.tile, &cps);
        const size_t smem = 128 + (size_t)S * (2 * R + 1) * a.tile * 8 * b_w;
        if (S > 0 && smem >= 128 + (size_t)(2 * R + 1) * (2 * R + 1) * (2 * R + 1) * 4) {
            const void* f = fmt == 0 ? (const void*)superpose_mixed_bulk_kernel<R, float>
                          : fmt == 1 ? (const void*)superpose_mixed_bulk_kernel<R, __half>
                                     : (const void*)superpose_mixed_bulk_kernel<R, __nv_bfloat16>;
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            const int nt = (kBulkWarps + 1) * 32;
            if (fmt == 0) superpose_mixed_bulk_kernel<R, float><<<nblk, nt, smem, s>>>(a, u, S);
            else if (fmt == 1) superpose_mixed_bulk_kernel<R, __half><<<nblk, nt, smem, s>>>(a, u, S);
            else superpose_mixed_bulk_kernel<R, __nv_bfloat16><<<nblk, nt, smem, s>>>(a, u, S);
            return cudaGetLastError();
        }
    }
    if (fmt == 0) superpose_mixed_kernel<R, float><<<nblk, 256, 0, s>>>(a, u);
    else if (fmt == 1) superpose_mixed_kernel<R, __half><<<nblk, 256, 0, s>>>(a, u);
    else superpose_mixed_kernel<R, __nv_bfloat16><<<nblk, 256, 0, s>>>(a, u);
    return cudaGetLastError();
}

cudaError_t launch_superpose_mixed(const SuperArgs& a, const UniArgs& u, int R, int fmt, cudaStream_t s)
{
    switch (R) {
        case 1: return launch_mixed_r<1>(a, u, fmt, s);
        case 2: return launch_mixed_r<2>(a, u, fmt, s);
        case 3: return launch_mixed_r<3>(a, u, fmt, s);
        case 4: return launch_mixed_r<4>(a, u, fmt, s);
        case 5: return launch_mixed_r<5>(a, u, fmt, s);
        case 6: return launch_mixed_r<6>(a, u, fmt, s);
        case 7: return launch_mixed_r<7>(a, u, fmt, s);
        case 8: return launch_mixed_r<8>(a, u, fmt, s);
        default: return cudaErrorInvalidValue;
    }
}

// Read-stream probe (fdirw_read_ceiling): the HBM read bandwidth this box gives a kernel that
// does nothing but stream a buffer with the superposition's load (128-bit, L1 no-allocate, L2
// evict-first), grid-stride over 4 CTAs of 256 threads per SM, 8 loads in flight per thread.
__global__ void __launch_bounds__(256) read_stream_kernel(const uint4* __restrict__ p, size_t n16, unsigned* sink)
{
    const uint64_t pol = evict_first_policy();
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(p + i + u * stride, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        const uint4 v = ld_stream(p + i, pol);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;  // keeps the loads; practically never taken
}

cudaError_t launch_read_stream(const void* p, size_t bytes, unsigned* sink, int sms, cudaStream_t s)
{
    read_stream_kernel<<<sms * 4, 256, 0, s>>>(reinterpret_cast<const uint4*>(p), bytes / 16, sink);
    return cudaGetLastError();
}

// Identity rows: chunk ch (tile·tile + e) of the slab, 8 targets, C_new = C_old (bitwise what
// the dense path computes for them: d = 1, every other weight 0, p_BC = 0).
__global__ void copy_chunks_kernel(const float* __restrict__ cpad, float* __restrict__ out, long out_ps, long out_rs,
                                   const int* __restrict__ list, long n, int nx, int nxq, int tile, int tpp, int nxp,
                                   int nyp, int R)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int ch = list[i];
        const int t = ch / tile, e = ch % tile;
        const int zl = t / tpp, q = (t % tpp) * tile + e;
        const int y = q / nxq, x = (q % nxq) * 8;
        const float* src = cpad + ((long)(zl + R) * nyp + (y + R)) * nxp + kPadX + x;
        float* dst = out + (long)zl * out_ps + (long)y * out_rs + x;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (x + j < nx) dst[j] = src[j];
    }
}

cudaError_t launch_copy_chunks(const float* cpad, float* out, long out_ps, long out_rs, const int* list, long n,
                               const Geometry& g, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const long blocks = (n + 255) / 256;
    copy_chunks_kernel<<<(unsigned)(blocks < 148L * 8 ? blocks : 148L * 8), 256, 0, s>>>(
        cpad, out, out_ps, out_rs, list, n, g.nx, g.nxq, g.tile, g.tpp, g.nxp, g.nyp, g.R);
    return cudaGetLastError();
}

cudaError_t launch_superpose(const SuperArgs& a, int R, int fmt, cudaStream_t s)
{
    switch (R) {
        case 1: return launch_superpose_r<1>(a, fmt, s);
        case 2: return launch_superpose_r<2>(a, fmt, s);
        case 3: return launch_superpose_r<3>(a, fmt, s);
        case 4: return launch_superpose_r<4>(a, fmt, s);
        case 5: return launch_superpose_r<5>(a, fmt, s);
        case 6: return launch_superpose_r<6>(a, fmt, s);
        case 7: return launch_superpose_r<7>(a, fmt, s);
        case 8: return launch_superpose_r<8>(a, fmt, s);
        default: return cudaErrorInvalidValue;
    }
}

// ---- state kernels ------------------------------------------------------------------
__global__ void pack_kernel(const float* __restrict__ c, float* __restrict__ cpad, int nx, int ny, long n,
                            int R, int nxp, int nyp, const uint8_t* __restrict__ farmask)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int x = (int)(i % nx);
        const long r = i / nx;
        const int y = (int)(r % ny);
        const long z = r / ny;
        // N2: far-field voxels carry no fine value (theirs is the scalar c_far)
        cpad[((z + R) * nyp + (y + R)) * (long)nxp + kPadX + x] = (farmask && farmask[i]) ? 0.f : c[i];
    }
}

// ---- N2 far field --------------------------------------------------------------------
static unsigned grid_for(long n, int threads);
__global__ void tile_mass_kernel(const float* __restrict__ c, long ps, long rs, const uint8_t* __restrict__ farmask,
                                 int nx, int ny, int nxq, int tile, int tpp, double* __restrict__ tile_sum)
{
    const int t = blockIdx.x, zl = t / tpp, tp = t % tpp;
    const int q = tp * tile + threadIdx.x;
    double s = 0.0;
    if (q < ny * nxq) {
        const int y = q / nxq, x = (q % nxq) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (x + j >= nx) continue;
            const long i = ((long)zl * ny + y) * nx + x + j;  // dense index of the far mask
            s += (farmask && farmask[i]) ? 0.0 : (double)c[(long)zl * ps + (long)y * rs + x + j];
        }
    }
    s = tile_block_sum(s);
    if (threadIdx.x == 0) tile_sum[t] = s;
}

cudaError_t launch_tile_mass(const float* c, const uint8_t* farmask, const Geometry& g, double* tile_sum,
                             cudaStream_t s)
{
    if (g.n_tiles <= 0) return cudaSuccess;
    tile_mass_kernel<<<g.n_tiles, g.tile, 0, s>>>(c, (long)g.nx * g.ny, g.nx, farmask, g.nx, g.ny, g.nxq, g.tile,
                                                  g.tpp, tile_sum);
    return cudaGetLastError();
}

cudaError_t launch_tile_mass_padded(const float* c_interior, const uint8_t* farmask, const Geometry& g,
                                    double* tile_sum, cudaStream_t s)
{
    if (g.n_tiles <= 0) return cudaSuccess;
    tile_mass_kernel<<<g.n_tiles, g.tile, 0, s>>>(c_interior, (long)g.plane_elems, g.nxp, farmask, g.nx, g.ny,
                                                  g.nxq, g.tile, g.tpp, tile_sum);
    return cudaGetLastError();
}

__global__ void ones_kernel(const uint8_t* __restrict__ mask, int mz0, int nx, int ny, int nz, int z0, int R,
                            int nzl, int nxp, int nyp, float* __restrict__ cpad)
{
    const long n = (long)nx * ny * (nzl + 2 * R);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int x = (int)(i % nx), y = (int)((i / nx) % ny);
        const int pz = (int)(i / ((long)nx * ny));  // padded plane
        const int z = z0 - R + pz;
        float v = 0.f;
        if (z >= 0 && z < nz) v = mask[((long)(z - mz0) * ny + y) * nx + x] == 2 ? 0.f : 1.f;
        cpad[((long)pz * nyp + (y + R)) * nxp + kPadX + x] = v;
    }
}

cudaError_t launch_ones(const uint8_t* mask, int mz0, const Geometry& g, float* cpad, cudaStream_t s)
{
    const long n = (long)g.nx * g.ny * (g.nzl + 2 * g.R);
    ones_kernel<<<grid_for(n, 256), 256, 0, s>>>(mask, mz0, g.nx, g.ny, g.nz, g.z0, g.R, g.nzl, g.nxp, g.nyp, cpad);
    return cudaGetLastError();
}

__global__ void pbc_kernel(const float* __restrict__ rowsum, const uint8_t* __restrict__ farmask, int nx, int ny,
                           int nxq, int tile, int tpp, long n_elems, float* __restrict__ pbc,
                           const int* __restrict__ list, long n_list, int direct)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n_elems; i += (long)gridDim.x * blockDim.x) {
        const int j = (int)(i & 7);
        long te = i >> 3;
        bool ok = true;
        if (list) {  // N2 compaction: element te of the compact layout is chunk list[te]
            ok = te < n_list;
            te = ok ? list[te] : 0;
        }
        const int e = (int)(te % tile);
        const long t = te / tile;
        const int zl = (int)(t / tpp), tp = (int)(t % tpp);
        const int q = tp * tile + e;
        float v = 0.f;
        if (ok && q < ny * nxq) {
            const int y = q / nxq, x = (q % nxq) * 8 + j;
            if (x < nx) {
                const long k = ((long)zl * ny + y) * nx + x;
                // reading A26: p_BC = 1 − Σ_s W̃_s(x−s); direct: the reservoir FD's response itself
                v = farmask[k] ? 0.f : direct ? rowsum[k] : 1.f - rowsum[k];
            }
        }
        pbc[i] = v;
    }
}

cudaError_t launch_pbc(const float* rowsum, const uint8_t* farmask, const Geometry& g, float* pbc, cudaStream_t s,
                       const int* list, long n_list, int n_list_tiles, bool direct)
{
    const long n = list ? (long)n_list_tiles * g.tile * kChunk : (long)g.diag_elems;
    if (n <= 0) return cudaSuccess;
    pbc_kernel<<<grid_for(n, 256), 256, 0, s>>>(rowsum, farmask, g.nx, g.ny, g.nxq, g.tile, g.tpp, n, pbc, list,
                                                n_list, direct ? 1 : 0);
    return cudaGetLastError();
}

// One explicit FD substep over the whole grid (dense layout): far-field voxels (mask 2) held at 1,
// faces between non-far voxels and far ones as between fast cells (kgen's rule, face_lambda);
// faces summed in the order −x, +x, −y, +y, −z, +z
__global__ void reservoir_fd_kernel(const uint8_t* __restrict__ mask, const float* __restrict__ cin,
                                    float* __restrict__ cout, int nx, int ny, int nz, float lff, float lfs, float lss)
{
    const long n = (long)nx * ny * nz;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((long)nx * ny));
        const unsigned p = mask[i];
        if (p == 2u) { cout[i] = 1.f; continue; }
        const float c = cin[i];
        float acc = c;
        const long d[3] = {1, nx, (long)nx * ny};
        const bool inb[6] = {x > 0, x < nx - 1, y > 0, y < ny - 1, z > 0, z < nz - 1};
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            if (!inb[f]) continue;
            const long j = i + (f & 1 ? d[f >> 1] : -d[f >> 1]);
            const unsigned q = mask[j];
            const bool fp = p == 1u, fq = q != 0u;  // far counts as fast
            const float lam = fp && fq ? lff : (fp || fq ? lfs : lss);
            acc = fmaf(lam, cin[j] - c, acc);
        }
        cout[i] = acc;
    }
}

__global__ void reservoir_init_kernel(const uint8_t* __restrict__ mask, float* __restrict__ c, long n)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        c[i] = mask[i] == 2 ? 1.f : 0.f;
}

cudaError_t launch_reservoir_fd(const uint8_t* mask, const Geometry& g, float lff, float lfs, float lss, int n_fd,
                                float* out, float* tmp, cudaStream_t s)
{
    const long n = (long)g.nx * g.ny * g.nz;
    if (g.mz0 != 0 || g.mz1 != g.nz) return cudaErrorInvalidValue;  // needs every mask plane (world 1)
    float* a = (n_fd & 1) ? tmp : out;  // so the last substep lands in out
    float* b = (n_fd & 1) ? out : tmp;
    reservoir_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(mask, a, n);
    for (int k = 0; k < n_fd; ++k) {
        reservoir_fd_kernel<<<grid_for(n, 256), 256, 0, s>>>(mask, a, b, g.nx, g.ny, g.nz, lff, lfs, lss);
        float* t = a; a = b; b = t;
    }
    return cudaGetLastError();
}

// One warp: lane l sums the tile partials whose GLOBAL tile index ≡ l (mod 32) in increasing
// order, then a fixed shuffle tree — the same sequence for every slab decomposition.
__global__ void far_reduce_kernel(const double* __restrict__ gathered, int world, long stride,
                                  double* __restrict__ far_state, double v_far, double c_far0, int mode)
{
    const int lane = threadIdx.x;
    double s = 0.0;
    long g0 = 0;
    for (int r = 0; r < world; ++r) {
        const double* blk = gathered + (long)r * stride;
        const long n = (long)blk[0];
        long t = ((lane - g0) % 32 + 32) % 32;
        for (; t < n; t += 32) s += blk[1 + t];
        g0 += n;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        if (mode == 0) {
            far_state[0] = (far_state[1] - s) / v_far;  // Eq.7
        } else {
            far_state[1] = s + c_far0 * v_far;          // M0 = Σc_{S+L}(t0)
            far_state[0] = c_far0;
        }
    }
}

cudaError_t launch_far_reduce(const double* gathered, int world, long stride, double* far_state, double v_far,
                              double c_far0, int mode, cudaStream_t s)
{
    far_reduce_kernel<<<1, 32, 0, s>>>(gathered, world, stride, far_state, v_far, c_far0, mode);
    return cudaGetLastError();
}

__global__ void unpack_kernel(const float* __restrict__ cpad, float* __restrict__ c, int nx, int ny, long n,
                              int R, int nxp, int nyp)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int x = (int)(i % nx);
        const long r = i / nx;
        const int y = (int)(r % ny);
        const long z = r / ny;
        c[i] = cpad[((z + R) * nyp + (y + R)) * (long)nxp + kPadX + x];
    }
}

static unsigned grid_for(long n, int threads)
{
    long b = (n + threads - 1) / threads;
    if (b > 148L * 16) b = 148L * 16;
    if (b < 1) b = 1;
    return (unsigned)b;
}

cudaError_t launch_pack(const float* c, float* cpad, const Geometry& g, cudaStream_t s, const uint8_t* farmask)
{
    const long n = (long)g.nx * g.ny * g.nzl;
    if (n == 0) return cudaSuccess;
    pack_kernel<<<grid_for(n, 256), 256, 0, s>>>(c, cpad, g.nx, g.ny, n, g.R, g.nxp, g.nyp, farmask);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const float* cpad, float* c, const Geometry& g, cudaStream_t s)
{
    const long n = (long)g.nx * g.ny * g.nzl;
    if (n == 0) return cudaSuccess;
    unpack_kernel<<<grid_for(n, 256), 256, 0, s>>>(cpad, c, g.nx, g.ny, n, g.R, g.nxp, g.nyp);
    return cudaGetLastError();
}

// CUDA 12 loads kernels lazily at their first launch, and loading can wait for the device.
// Steps whose kernels spin on a neighbour's flags (P2P transport, several contexts on one
// device) must not trigger a load mid-run: load the step's kernels up front.
cudaError_t preload_step_kernels()
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, pack_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, unpack_kernel);
    return e;
}

// fp64 sum, two passes with a fixed order (deterministic).
__global__ void mass_partial_kernel(const float* __restrict__ c, size_t n, double* __restrict__ partial)
{
    __shared__ double red[32];
    double v = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        v += (double)c[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = v;
    }
}

__global__ void mass_final_kernel(const double* __restrict__ partial, int n, double* __restrict__ out)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double v = 0.0;
        for (int i = 0; i < n; ++i) v += partial[i];
        *out = v;
    }
}

cudaError_t launch_mass(const float* c, size_t n, double* partial, int nblk, double* out, cudaStream_t s)
{
    mass_partial_kernel<<<nblk, 256, 0, s>>>(c, n, partial);
    mass_final_kernel<<<1, 32, 0, s>>>(partial, nblk, out);
    return cudaGetLastError();
}

// Decode the stored kernels of the sources in `box` back to per-source fp64 arrays.
__global__ void export_kernel(const void* __restrict__ Wt, const float2* __restrict__ diag, Geometry g, int fmt,
                              int bx0, int bx, int by0, int by, int bz0, int bz, double* __restrict__ out,
                              const int* __restrict__ chunk_pos)
{
    const long total = (long)bx * by * bz * g.K;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int o = (int)(i % g.K);
        const long n = i / g.K;
        const int sx = bx0 + (int)(n % bx), sy = by0 + (int)((n / bx) % by), sz = bz0 + (int)(n / ((long)bx * by));
        const int ox = o % g.L - g.R, oy = (o / g.L) % g.L - g.R, oz = o / (g.L * g.L) - g.R;
        const int x = sx + ox, y = sy + oy, z = sz + oz;
        double v = 0.0;
        if (x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= g.z0 && z < g.z1 && sx >= 0 && sx < g.nx &&
            sy >= 0 && sy < g.ny && sz >= 0 && sz < g.nz) {
            const int q = y * g.nxq + (x >> 3);
            size_t tile = (size_t)(z - g.z0) * g.tpp + q / g.tile;
            int e = q % g.tile;
            const int j = x & 7;
            const int cp = chunk_pos ? chunk_pos[tile * g.tile + e] : 0;  // N2 compaction
            if (chunk_pos && cp >= 0) {
                tile = cp / g.tile;
                e = cp % g.tile;
            }
            if (chunk_pos && cp < 0) {
                // an all-far chunk (−1): no weights stored (they are 0); an identity chunk (−2,
                // impermeable solid targets): the centre weight is 1, every other 0
                v = (cp == -2 && o == g.K / 2) ? 1.0 : 0.0;
            } else if (o == g.K / 2) {
                const float2 d = diag[(tile * g.tile + e) * 8 + j];
                v = (double)d.x + (double)d.y;  // the fp32 pair (reading A10), exact in fp64
            } else if (fmt == FDIRW_W_MX8) {
                size_t mo, so;
                mx8_addr(tile, slot_of(ox, oy, oz, g.R), e, j, g.L, g.K, g.tile, &mo, &so);
                const unsigned char* wq = reinterpret_cast<const unsigned char*>(Wt);
                v = mx8_decode(wq[mo], wq[so]);
            } else {
                const size_t idx = ((tile * (size_t)(g.K - 1) + slot_of(ox, oy, oz, g.R)) * g.tile + e) * 8 + j;
                if (fmt == 0) v = reinterpret_cast<const float*>(Wt)[idx];
                else if (fmt == 1) v = __half2float(reinterpret_cast<const __half*>(Wt)[idx]);
                else v = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(Wt)[idx]);
            }
        }
        out[i] = v;
    }
}

cudaError_t launch_export(const void* Wt, const float2* diag, const Geometry& g, int fmt, const int32_t* box,
                          double* out, cudaStream_t s, const int* chunk_pos)
{
    const int bx = box[1] - box[0], by = box[3] - box[2], bz = box[5] - box[4];
    const long total = (long)bx * by * bz * g.K;
    if (total <= 0) return cudaSuccess;
    export_kernel<<<grid_for(total, 256), 256, 0, s>>>(Wt, diag, g, fmt, box[0], bx, box[2], by, box[4], bz, out,
                                                       chunk_pos);
    return cudaGetLastError();
}

}  // namespace fdirw
