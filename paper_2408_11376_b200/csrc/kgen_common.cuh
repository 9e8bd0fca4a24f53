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

// CTA barriers for warp-specialised kernels (kgen_bal.cu), where each segment's warps run their own
// instantiation and so reach the CTA barrier from different code.
//  CLEAN = false (default): named barrier 1 with the CTA's thread count, `bar.sync 1, NT` /
//    `bar.red.or.pred`, issued inline — the CUTLASS NamedBarrier form; every thread executes the
//    same barriers in the same order.  compute-sanitizer synccheck reports these ("divergent
//    threads in block": it expects one PC per CTA barrier).
//  CLEAN = true (FDIRW_KGEN_SYNCCHECK=1): the barrier lives in one non-inlined function every
//    thread calls, so all threads execute the same `bar.sync` instruction; synccheck-clean,
//    measured 15 % slower at R5 (the call per pass).
template <int NT, bool CLEAN>
__device__ __forceinline__ void cta_sync_any_pc();
template <int NT, bool CLEAN>
__device__ __forceinline__ bool cta_or_any_pc(bool v);

static __device__ __noinline__ void cta_sync_call() { __syncthreads(); }
static __device__ __noinline__ int cta_or_call(int v) { return __syncthreads_or(v); }

template <int NT, bool CLEAN>
__device__ __forceinline__ void cta_sync_any_pc()
{
    if constexpr (CLEAN) cta_sync_call();
    else asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
template <int NT, bool CLEAN>
__device__ __forceinline__ bool cta_or_any_pc(bool v)
{
    if constexpr (CLEAN) {
        return cta_or_call(v ? 1 : 0) != 0;
    } else {
        unsigned r;
        asm volatile(
            "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, 1, %2, p;\n selp.u32 %0, 1, 0, q;\n}"
            : "=r"(r)
            : "r"((unsigned)v), "n"(NT)
            : "memory");
        return r != 0;
    }
}

// Deterministic block reduction (fixed shuffle tree + fixed warp order).  ANY_PC: the barriers
// are cta_sync_any_pc<NW·32, CLEAN> (for warp-specialised callers), else __syncthreads.
template <int NW, bool ANY_PC = false, bool CLEAN = false>
__device__ __forceinline__ double block_sum_f64(double v, double* red)
{
    auto sync = [] {
        if constexpr (ANY_PC) cta_sync_any_pc<NW * 32, CLEAN>();
        else __syncthreads();
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum_f64(v);
    if (lane == 0) red[warp] = v;
    sync();
    if (warp == 0) {
        double w = lane < NW ? red[lane] : 0.0;
        w = warp_sum_f64(w);
        if (lane == 0) red[NW] = w;
    }
    sync();
    const double r = red[NW];
    sync();
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

// An isolated source: every face of the window's centre cell has face number 0 (a slow-phase
// voxel with D_slow = 0, the N3 loop's impermeable solid).  Its kernel is exactly δ_s — each literal
// substep leaves it unchanged — so kgen runs no pass for it.  (The Chebyshev recurrence would give
// Σ fp32(c_k)·δ = (1 − ~6e-8)·δ: renormalisation hides that in a closed window, but an open (N2)
// window keeps its kernel's own mass, and that would make the identity row of a solid voxel
// leak.)  T: the λ face table (build_face_tables set 0); faces are ≥ 0.
__device__ __forceinline__ bool isolated_source(const unsigned char* ph, const float* T, int KC, int L, int LL)
{
    const unsigned pc = ph[KC];
    const float f = T[(pc << 2) | ph[KC - 1]] + T[(pc << 2) | ph[KC + 1]] + T[(pc << 2) | ph[KC - L]] +
                    T[(pc << 2) | ph[KC + L]] + T[16 + ((ph[KC - LL] << 2) | pc)] + T[16 + ((pc << 2) | ph[KC + LL])];
    return f == 0.f;
}

}  // namespace fdirw
