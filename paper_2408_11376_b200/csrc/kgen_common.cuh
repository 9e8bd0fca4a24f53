// kgen_common.cuh — device helpers shared by the kgen kernels (kgen.cu, kgen_bal.cu):
// deterministic fp64 block sums, packed fp32x2 arithmetic (FADD2/FFMA2) and the face numbers
// of the explicit-FD stencil (reading A4: harmonic-mean faces precomputed per phase pair).
#pragma once

#include <cuda_runtime.h>

namespace fdirw {

__device__ __forceinline__ double warp_sum_f64(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block reduction (fixed shuffle tree + fixed warp order).
template <int NW>
__device__ __forceinline__ double block_sum_f64(double v, double* red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum_f64(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = lane < NW ? red[lane] : 0.0;
        w = warp_sum_f64(w);
        if (lane == 0) red[NW] = w;
    }
    __syncthreads();
    const double r = red[NW];
    __syncthreads();
    return r;
}

// Packed fp32x2 arithmetic (sm_100a FADD2/FFMA2): two cells per instruction, each
// lane an ordinary IEEE fp32 add / fma — bitwise identical to the scalar form.
__device__ __forceinline__ unsigned long long pk2(float a, float b)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long v, float& a, float& b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b)
{
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c)
{
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

__device__ __forceinline__ float face_lambda(unsigned p, unsigned q, float ff, float fs, float ss)
{
    // p, q ∈ {0 slow, 1 fast, 2 outside the domain, 3 far-field reservoir (N2)}.  A far
    // cell is a fast-phase Dirichlet cell held at 0: faces into it carry flux, its own
    // value never changes (p = 3 → no update).
    if (p > 1u || q == 2u) return 0.f;
    if (q == 3u) q = 1u;
    return (p & q) ? ff : ((p | q) ? fs : ss);
}

// Face-number lookup tables, built once per CTA in shared memory (64 floats): for the literal
// substeps (set 0: λ) and the Chebyshev passes (set 1: 2μ), tab[32·set + p·4 + q] = face_lambda(p,
// q) and tab[32·set + 16 + p·4 + q] = the z-face form (p ≤ 1 ? face_lambda(p, q) : face_lambda(q,
// p)): one shared load per face instead of face_lambda's branches (bitwise the same values).
__device__ __forceinline__ void build_face_tables(float* tab, float lff, float lfs, float lss, float mff, float mfs,
                                                  float mss)
{
    for (int i = threadIdx.x; i < 64; i += blockDim.x) {  // (R ≤ 2 windows run 32 threads)
        const int set = i >> 5, sym = (i >> 4) & 1;
        const unsigned p = (i >> 2) & 3, q = i & 3;
        const float ff = set ? mff : lff, fs = set ? mfs : lfs, ss = set ? mss : lss;
        tab[i] = sym ? (p <= 1u ? face_lambda(p, q, ff, fs, ss) : face_lambda(q, p, ff, fs, ss))
                     : face_lambda(p, q, ff, fs, ss);
    }
}

}  // namespace fdirw
