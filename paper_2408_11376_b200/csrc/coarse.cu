// coarse.cu — NEXT row N1: coarse-mesh FDiRW (§3.1, Eqs.10-15) on B200,
// with the far-field boundary term of NEXT row N2 (P_BC, Eq.7) when v_far > 0.
//
// Build (one-time, "preconditioned" P):
//   groups      Ω_L ∩ b³ blocks (P:113 N = N_L/125 ⇔ b = 5): used-block flags → scan → ids;
//               group CSR (stable radix sort of (group, voxel)) for the mapping step
//   columns     explicit FD over Ω_L from the group-uniform sources 1_J,
//               all columns of a chunk at once: X[row][j] with j fastest, so the 7-point
//               stencil reads whole neighbour rows (coalesced 16-byte loads, neighbour
//               table read once per row, rows of 3 z-planes of the region stay in L2).
//               Faces into far-field voxels (region value 2) are Dirichlet: 0 for the P
//               columns, 1 for the extra P_BC column
//   P           group means of the FD result (Eq.11/13), fp64, then RNE to the storage
//               format with an fp32 diagonal keeping each column's mass Σ_I N_I P_IJ
// Step (the paper's three kernels, §3.2 / Fig.2, captured in a CUDA graph for run):
//   map_kernel     one warp per group, fp32 sum over its voxels ("mapping ... FP32")
//   gemv_kernel    one warp per row I of P̃ (row-major, L2-resident: N² b_w bytes), 128-bit
//                  loads, fp32 FMA + fixed shuffle tree ("accumulation ... FP32"),
//                  + P_BC_I·c_far (Eq.14)
//   remap_kernel   c'_i = C'_{I(i)} for every Ω_L voxel (Eq.15)
//   far_kernel     Eq.7: c_far = (K0 − Σ_I N_I C'_I)/V_far (voxels outside Ω_L are not
//                  touched by the coarse step, so their mass is a constant folded into K0)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "bulk.cuh"
#include "fdirw_internal.h"

using namespace fdirw;

struct fdirw_coarse {
    fdirw_params p;
    int n_fd = 0, b = 5, fmt = 0, b_w = 4, device = 0;
    int fd_passes = 0;        // stencil passes per P column: n_fd, or kCheb_pre + Chebyshev degree
    double lam = 0;
    long nvox = 0, NL = 0, N = 0;
    long ldp = 0;             // row stride of P: N rounded up to 8 (16-byte rows, zero padding)
    int bulk_m = 0;           // > 0: bulk-copy GEMV with GEMV_NW·bulk_m row stages per CTA
    size_t bulk_smem = 0;
    int n_sm = 148;
    int* group_of = nullptr;  // [nvox]
    int* rows = nullptr;      // [NL] voxel of each region row (voxel order)
    int* grp_ptr = nullptr;   // [N+1]
    int* grp_vox = nullptr;   // [NL] voxels sorted by group
    int* sizes = nullptr;     // [N]
    void* P = nullptr;        // [N][ldp] storage format, diagonal slot 0, zero padding
    float* Pdiag = nullptr;   // [N]
    float* C = nullptr;       // [ldp], zero padding
    float* C2 = nullptr;      // [ldp]
    cudaStream_t cap = nullptr;
    cudaGraphExec_t graph = nullptr;
    cudaGraphExec_t graph2 = nullptr;  // fdirw_coarse_run: two coarse-space steps C → C2 → C
    float* graph_c = nullptr;
    // N2
    bool far = false;
    double v_far = 0;
    float* Pbc = nullptr;        // [N] fp32
    double* far_state = nullptr; // {c_far, K0}
};

namespace fdirw {
const char* coarse_set_error(const std::string& m);
}

static fdirw_status cfail(fdirw_status s, const std::string& m)
{
    coarse_set_error(m);
    return s;
}

#define CK(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) return cfail(FDIRW_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

static unsigned gridn(long n, int t = 256)
{
    long b = (n + t - 1) / t;
    if (b > 148L * 32) b = 148L * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

#define GRID_STRIDE(i, n) for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (n); i += (long)gridDim.x * blockDim.x)

// region codes: 1 = Ω_L, 2 = far-field reservoir (N2), anything else = outside
__global__ void k_mark_blocks(const uint8_t* reg, long nvox, int nx, int ny, int b, int bx, int by, int* used)
{
    GRID_STRIDE(v, nvox)
    {
        if (reg[v] != 1) continue;
        const int x = (int)(v % nx), y = (int)((v / nx) % ny), z = (int)(v / ((long)nx * ny));
        used[((z / b) * by + (y / b)) * bx + (x / b)] = 1;
    }
}

__global__ void k_group_of(const uint8_t* reg, long nvox, int nx, int ny, int b, int bx, int by, const int* bid,
                           int* group_of, int* sizes, int* row_flag)
{
    GRID_STRIDE(v, nvox)
    {
        int g = -1;
        if (reg[v] == 1) {
            const int x = (int)(v % nx), y = (int)((v / nx) % ny), z = (int)(v / ((long)nx * ny));
            g = bid[((z / b) * by + (y / b)) * bx + (x / b)];
            atomicAdd(&sizes[g], 1);
        }
        group_of[v] = g;
        row_flag[v] = g >= 0 ? 1 : 0;
    }
}

__global__ void k_rows(const int* row_flag, const int* row_pos, long nvox, int* rows, int* row_of, const int* group_of,
                       int* row_group)
{
    GRID_STRIDE(v, nvox)
    {
        if (row_flag[v]) {
            const int r = row_pos[v];
            rows[r] = (int)v;
            row_group[r] = group_of[v];
            row_of[v] = r;
        } else {
            row_of[v] = -1;
        }
    }
}

// neighbour rows in the order −x, +x, −y, +y, −z, +z: a row index, −2 = far-field (Dirichlet),
// −1 = no flux
__global__ void k_neighbours(const int* rows, long NL, const int* row_of, const uint8_t* reg, int nx, int ny, int nz,
                             int* nb)
{
    GRID_STRIDE(r, NL)
    {
        const int v = rows[r];
        const int x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
        const long pl = (long)nx * ny;
        const long q[6] = {x > 0 ? v - 1 : -1L, x < nx - 1 ? v + 1 : -1L, y > 0 ? v - nx : -1L,
                           y < ny - 1 ? v + nx : -1L, z > 0 ? v - pl : -1L, z < nz - 1 ? v + pl : -1L};
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            int code = -1;
            if (q[f] >= 0) code = row_of[q[f]] >= 0 ? row_of[q[f]] : (reg[q[f]] == 2 ? -2 : -1);
            nb[r * 6 + f] = code;
        }
    }
}

__global__ void k_init_cols(const int* row_group, long NL, int CB, int J0, float* X)
{
    GRID_STRIDE(i, NL * (long)CB)
    {
        const long r = i / CB;
        const int j = (int)(i % CB);
        X[i] = row_group[r] == J0 + j ? 1.f : 0.f;  // column N (P_BC) has no group: starts at 0
    }
}

// One FD substep for CB columns at once: one warp per row, lanes over float4 column quads.
// A far-field face adds λ·(b_j − c) with b_j = 1 for the P_BC column (global index Nbc), else 0.
__global__ void __launch_bounds__(256) k_fd_cols(const float* __restrict__ X, float* __restrict__ Y,
                                                 const int* __restrict__ nb, long NL, int CB, float lam, int J0,
                                                 int Nbc)
{
    const int lane = threadIdx.x & 31;
    const long warps = (long)gridDim.x * (blockDim.x >> 5);
    const int q4 = CB >> 2;
    for (long r = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < NL; r += warps) {
        int n[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) n[f] = __ldg(nb + r * 6 + f);
        const float4* xr = reinterpret_cast<const float4*>(X + r * (long)CB);
        float4* yr = reinterpret_cast<float4*>(Y + r * (long)CB);
        for (int q = lane; q < q4; q += 32) {
            const float4 c = xr[q];
            float4 a = c;
            const int j0 = J0 + 4 * q;
            const float4 bv = make_float4(j0 == Nbc ? 1.f : 0.f, j0 + 1 == Nbc ? 1.f : 0.f, j0 + 2 == Nbc ? 1.f : 0.f,
                                          j0 + 3 == Nbc ? 1.f : 0.f);
#pragma unroll
            for (int f = 0; f < 6; ++f) {
                if (n[f] == -1) continue;
                const float4 m = n[f] >= 0 ? reinterpret_cast<const float4*>(X + (long)n[f] * CB)[q] : bv;
                a.x = fmaf(lam, m.x - c.x, a.x);
                a.y = fmaf(lam, m.y - c.y, a.y);
                a.z = fmaf(lam, m.z - c.z, a.z);
                a.w = fmaf(lam, m.w - c.w, a.w);
            }
            yr[q] = a;
        }
    }
}

// One Chebyshev pass for CB columns (reading A30; the same recurrence as kgen's): with
// Â = I + Σ_f μ_f (t_f − t) (μ = 2λ/(1 − a), far-field faces Dirichlet 0),
//   prv ← 2·Â·cur − prv  (first pass: Â·cur, prv unread),  acc ← acc + c_k·prv
// (first pass: acc ← c_0·cur + c_1·prv).  mu2 = 2μ.  One warp per row, float4 column quads.
__global__ void __launch_bounds__(256) k_cheb_cols(const float* __restrict__ cur, float* __restrict__ prv,
                                                   float* __restrict__ acc, const int* __restrict__ nb, long NL,
                                                   int CB, float mu2, float c0, float ck, int first)
{
    const int lane = threadIdx.x & 31;
    const long warps = (long)gridDim.x * (blockDim.x >> 5);
    const int q4 = CB >> 2;
    for (long r = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < NL; r += warps) {
        int n[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) n[f] = __ldg(nb + r * 6 + f);
        const float4* cr = reinterpret_cast<const float4*>(cur + r * (long)CB);
        float4* pr = reinterpret_cast<float4*>(prv + r * (long)CB);
        float4* ar = reinterpret_cast<float4*>(acc + r * (long)CB);
        for (int q = lane; q < q4; q += 32) {
            const float4 c = cr[q];
            float4 v;
            if (first) {
                v = make_float4(2.f * c.x, 2.f * c.y, 2.f * c.z, 2.f * c.w);
            } else {
                const float4 p = pr[q];
                v = make_float4(fmaf(2.f, c.x, -p.x), fmaf(2.f, c.y, -p.y), fmaf(2.f, c.z, -p.z), fmaf(2.f, c.w, -p.w));
            }
#pragma unroll
            for (int f = 0; f < 6; ++f) {
                if (n[f] == -1) continue;
                const float4 m = n[f] >= 0 ? reinterpret_cast<const float4*>(cur + (long)n[f] * CB)[q]
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                v.x = fmaf(mu2, m.x - c.x, v.x);
                v.y = fmaf(mu2, m.y - c.y, v.y);
                v.z = fmaf(mu2, m.z - c.z, v.z);
                v.w = fmaf(mu2, m.w - c.w, v.w);
            }
            if (first) v = make_float4(0.5f * v.x, 0.5f * v.y, 0.5f * v.z, 0.5f * v.w);
            const float4 a0 = first ? make_float4(c0 * c.x, c0 * c.y, c0 * c.z, c0 * c.w) : ar[q];
            pr[q] = v;
            ar[q] = make_float4(fmaf(ck, v.x, a0.x), fmaf(ck, v.y, a0.y), fmaf(ck, v.z, a0.z), fmaf(ck, v.w, a0.w));
        }
    }
}

// P64[I][J0 + j] = Σ_{v∈I} X[row(v)][j] / N_I (fp64, CSR order); stride Ncol.  Entries are
// clamped at 0 (A^n·1_J ≥ 0; only the Chebyshev path's rounding noise can dip below).
__global__ void k_map_cols(const float* X, const int* grp_ptr, const int* grp_vox, const int* row_of, long N,
                           long Ncol, int CB, int J0, int Jn, double* P64)
{
    GRID_STRIDE(i, N * (long)Jn)
    {
        const long I = i / Jn;
        const int j = (int)(i % Jn);
        double s = 0.0;
        for (int k = grp_ptr[I]; k < grp_ptr[I + 1]; ++k) s += (double)fmaxf(X[(long)row_of[grp_vox[k]] * CB + j], 0.f);
        P64[I * Ncol + J0 + j] = s / (double)(grp_ptr[I + 1] - grp_ptr[I]);
    }
}

template <typename WT>
__device__ __forceinline__ WT enc(float f);
template <>
__device__ __forceinline__ float enc<float>(float f) { return f; }
template <>
__device__ __forceinline__ __half enc<__half>(float f) { return __float2half_rn(f); }
template <>
__device__ __forceinline__ __nv_bfloat16 enc<__nv_bfloat16>(float f) { return __float2bfloat16_rn(f); }
__device__ __forceinline__ float dec(float v) { return v; }
__device__ __forceinline__ float dec(__half v) { return __half2float(v); }
__device__ __forceinline__ float dec(__nv_bfloat16 v) { return __bfloat162float(v); }

// one block per column J: quantise off-diagonal entries; the fp32 diagonal keeps the column's
// fp64 mass M_J = Σ_I N_I P_IJ (N_J when closed)
template <typename WT>
__global__ void k_quantize(const double* P64, long Ncol, const int* sizes, long N, long ldp, WT* P, float* Pdiag)
{
    __shared__ double red[32], redm[32];
    const long J = blockIdx.x;
    double s = 0.0, m = 0.0;
    for (long I = threadIdx.x; I < N; I += blockDim.x) {
        const double pv = P64[I * Ncol + J];
        WT q = enc<WT>((float)pv);
        if (I == J) q = enc<WT>(0.f);
        P[I * ldp + J] = q;
        s += (double)sizes[I] * (double)dec(q);
        m += (double)sizes[I] * pv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = s; redm[threadIdx.x >> 5] = m; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, tm = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += red[w]; tm += redm[w]; }
        Pdiag[J] = (float)((tm - t) / (double)sizes[J]);
    }
}

// Closed region, Chebyshev-evaluated columns: the recurrence's fp32 rounding moves a column's
// mass Σ_I N_I P_IJ off its exact value N_J (FD conserves mass; ~6e-7 relative), so each
// column is rescaled in fp64 to N_J before quantisation — kgen's renormalisation of closed
// windows (§7), here by the group size (reading A30).  One block per column, fixed order.
__global__ void k_renorm_cols(double* P64, long Ncol, const int* sizes, long N)
{
    __shared__ double red[32];
    __shared__ double scale;
    const long J = blockIdx.x;
    double m = 0.0;
    for (long I = threadIdx.x; I < N; I += blockDim.x) m += (double)sizes[I] * P64[I * Ncol + J];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        scale = t > 0.0 ? (double)sizes[J] / t : 1.0;
    }
    __syncthreads();
    for (long I = threadIdx.x; I < N; I += blockDim.x) P64[I * Ncol + J] *= scale;
}

__global__ void k_pbc(const double* P64, long Ncol, long N, float* Pbc)
{
    GRID_STRIDE(I, N) Pbc[I] = (float)P64[I * Ncol + N];
}

// ---- step kernels -------------------------------------------------------------------
__global__ void k_map(const float* __restrict__ c, const int* __restrict__ grp_ptr, const int* __restrict__ grp_vox,
                      long N, float* __restrict__ C)
{
    const int lane = threadIdx.x & 31;
    const long warps = (long)gridDim.x * (blockDim.x >> 5);
    for (long I = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); I < N; I += warps) {
        const int a = grp_ptr[I], b = grp_ptr[I + 1];
        float s = 0.f;
        for (int k = a + lane; k < b; k += 32) s += c[grp_vox[k]];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) C[I] = s / (float)(b - a);
    }
}

// C (fp32, zero-padded to ldp) is read as float4 through L1; each lane keeps GU 16-byte loads
// of its row in flight before the FMAs.  Rows of P̃ bypass L1 and carry an L2 evict_last hint:
// P̃ is re-read every step and (N² b_w ≤ ~100 MB) can stay resident in the 126 MB L2.
__device__ __forceinline__ uint4 ld_row(const uint4* p, uint64_t pol)
{
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

template <typename WT>
__device__ __forceinline__ float dot16(const uint4& u, const float (&cv)[16 / sizeof(WT)])
{
    constexpr int V = 16 / sizeof(WT);
    const WT* w = reinterpret_cast<const WT*>(&u);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < V; ++k) acc = fmaf(dec(w[k]), cv[k], acc);
    return acc;
}

// One warp per GEMV_RW consecutive rows: every C quad read from L1 serves GEMV_RW rows (the
// single-row form was L1-throughput bound on the C reads, ncu 94% of peak).  Per row the lane
// partition (q ≡ lane mod 32, increasing q) and the FMA order are fixed.
constexpr int GEMV_RW = 4;

// SMC: C (ldp floats, zero past N) staged in shared memory once per block, so its reads leave the
// L1/TEX pipe to the P̃ stream (identical values and order: identical bits).  Measured (round 2,
// bf16, R50 near field): 22.7 → 20.6 µs per coarse step; with C in smem (RW, GU) = (4, 4) stays
// best — (2, 4) 24.0, (2, 8) 22.7, (4, 2) 22.7, (4, 8) 26.2, (8, 2) 26.8, (8, 4) 38.3 µs.
// cfine (closed domains): the remap fused into the epilogue — the warp that computed C'_I stores it
// into every fine voxel of group I (lane 0's value, broadcast), so no k_remap launch follows
template <typename WT, bool SMC = false>
__global__ void __launch_bounds__(512) k_gemv(const WT* __restrict__ P, const float* __restrict__ Pdiag,
                                              const float* __restrict__ C, long N, long ldp,
                                              float* __restrict__ Cout, const float* __restrict__ Pbc,
                                              const double* __restrict__ far_state,
                                              const int* __restrict__ grp_ptr = nullptr,
                                              const int* __restrict__ grp_vox = nullptr,
                                              float* __restrict__ cfine = nullptr)
{
    extern __shared__ __align__(16) float Csm[];
    if constexpr (SMC) {
        for (long i = threadIdx.x; i < ldp / 4; i += blockDim.x)
            reinterpret_cast<float4*>(Csm)[i] = __ldg(reinterpret_cast<const float4*>(C) + i);
        __syncthreads();
    }
    constexpr int V = 16 / sizeof(WT);  // elements per 128-bit load
    constexpr int GU = 4;
    const int lane = threadIdx.x & 31;
    const long warps = (long)gridDim.x * (blockDim.x >> 5);
    const int nv = (int)(ldp / V);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    // row group j = (warp w of block b) = w·gridDim + b: consecutive groups go to different
    // blocks (one block per SM), so every SM gets ⌈groups/SMs⌉ or one less (the first form,
    // 186 blocks of 8 warps on 148 SMs, left 38 SMs with twice the rows: 16.7 µs → see §11)
    for (long I0 = ((threadIdx.x >> 5) * (long)gridDim.x + blockIdx.x) * GEMV_RW; I0 < N;
         I0 += warps * GEMV_RW) {
        const int nrow = (int)min((long)GEMV_RW, N - I0);
        float acc[GEMV_RW];
#pragma unroll
        for (int r = 0; r < GEMV_RW; ++r) acc[r] = 0.f;
        for (int q0 = lane; q0 < nv; q0 += 32 * GU) {
            uint4 u[GEMV_RW][GU];
#pragma unroll
            for (int r = 0; r < GEMV_RW; ++r)
#pragma unroll
                for (int k = 0; k < GU; ++k)
                    u[r][k] = (r < nrow && q0 + 32 * k < nv)
                                  ? ld_row(reinterpret_cast<const uint4*>(P + (I0 + r) * ldp) + q0 + 32 * k, pol)
                                  : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int k = 0; k < GU; ++k) {
                if (q0 + 32 * k < nv) {
                    float cv[V];
#pragma unroll
                    for (int h = 0; h < V / 4; ++h) {
                        const float4 c4 = SMC ? reinterpret_cast<const float4*>(Csm + (long)(q0 + 32 * k) * V)[h]
                                              : __ldg(reinterpret_cast<const float4*>(C + (long)(q0 + 32 * k) * V) + h);
                        cv[4 * h] = c4.x; cv[4 * h + 1] = c4.y; cv[4 * h + 2] = c4.z; cv[4 * h + 3] = c4.w;
                    }
#pragma unroll
                    for (int r = 0; r < GEMV_RW; ++r) acc[r] += dot16<WT>(u[r][k], cv);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < GEMV_RW; ++r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
            if (lane == 0 && r < nrow) {
                const long I = I0 + r;
                float v = fmaf(Pdiag[I], C[I], acc[r]);
                if (Pbc) v = fmaf(Pbc[I], (float)far_state[0], v);  // Eq.14 boundary term
                Cout[I] = v;
                acc[r] = v;
            }
            if (cfine && r < nrow) {
                const float v = __shfl_sync(0xffffffffu, acc[r], 0);
                const long I = I0 + r;
                for (int k = grp_ptr[I] + lane; k < grp_ptr[I + 1]; k += 32) cfine[grp_vox[k]] = v;
            }
        }
    }
}

// ---- bulk-copy GEMV (opt-in, FDIRW_COARSE_GEMV=1; measured slower than k_gemv) ----
// Persistent: one CTA per SM owns a contiguous range of rows, cut into groups of GEMV_RB
// consecutive rows.  A producer warp streams each group (one contiguous run of P̃) into a
// ring of shared-memory stages with cp.async.bulk (TMA engine, no registers held per byte in
// flight) signalled through mbarriers; GEMV_NW consumer warps each own bulk_m stages and take
// groups g ≡ w (mod GEMV_NW) — a warp's stage is refilled only after that warp released it,
// so every wait is on the next phase of its own barrier.  C is staged in shared memory once
// per CTA and each C quad read serves GEMV_RB rows.  Per row, lane partition and FMA order
// are those of k_gemv, so the two kernels give identical bits.
constexpr int GEMV_NW = 4, GEMV_RB = 2;

template <typename WT>
__global__ void __launch_bounds__((GEMV_NW + 1) * 32) k_gemv_bulk(const WT* __restrict__ P,
                                                                  const float* __restrict__ Pdiag,
                                                                  const float* __restrict__ C, long N, long ldp,
                                                                  float* __restrict__ Cout, const float* __restrict__ Pbc,
                                                                  const double* __restrict__ far_state, int m)
{
    constexpr int V = 16 / sizeof(WT);
    extern __shared__ __align__(128) unsigned char sm[];
    const int S = GEMV_NW * m;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + S;
    float* Cs = reinterpret_cast<float*>(sm + ((16 * S + 127) / 128) * 128);
    unsigned char* stage = reinterpret_cast<unsigned char*>(Cs) + ((ldp * 4 + 127) / 128) * 128;
    const uint32_t rowB = (uint32_t)(ldp * sizeof(WT));
    const long r0 = blockIdx.x * N / gridDim.x, r1 = (blockIdx.x + 1) * N / gridDim.x;
    const int nr = (int)(r1 - r0), ng = (nr + GEMV_RB - 1) / GEMV_RB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(smem_u32(full + i), 1);
            mbar_init(smem_u32(empty + i), 1);
        }
        mbar_init_fence();
    }
    for (long i = threadIdx.x; i < ldp / 4; i += blockDim.x)
        reinterpret_cast<float4*>(Cs)[i] = __ldg(reinterpret_cast<const float4*>(C) + i);
    __syncthreads();
    if (warp == GEMV_NW) {  // producer
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            for (int g = 0; g < ng; ++g) {
                const int j = g / GEMV_NW, st = (g % GEMV_NW) * m + j % m, u = j / m;
                const int rows = min(GEMV_RB, nr - g * GEMV_RB);
                if (u > 0) mbar_wait(smem_u32(empty + st), (u - 1) & 1);
                mbar_expect_tx(smem_u32(full + st), rows * rowB);
                bulk_g2s(smem_u32(stage + (size_t)st * GEMV_RB * rowB), P + (r0 + (long)g * GEMV_RB) * ldp,
                         rows * rowB, smem_u32(full + st), pol);
            }
        }
        return;
    }
    const int nv = (int)(ldp / V);
    for (int g = warp, j = 0; g < ng; g += GEMV_NW, ++j) {
        const int st = warp * m + j % m, u = j / m;
        const int rows = min(GEMV_RB, nr - g * GEMV_RB);
        mbar_wait(smem_u32(full + st), u & 1);
        const uint4* base = reinterpret_cast<const uint4*>(stage + (size_t)st * GEMV_RB * rowB);
        float acc[GEMV_RB];
#pragma unroll
        for (int r = 0; r < GEMV_RB; ++r) acc[r] = 0.f;
        for (int q = lane; q < nv; q += 32) {
            float cv[V];
#pragma unroll
            for (int h = 0; h < V / 4; ++h) {
                const float4 c4 = reinterpret_cast<const float4*>(Cs + (long)q * V)[h];
                cv[4 * h] = c4.x; cv[4 * h + 1] = c4.y; cv[4 * h + 2] = c4.z; cv[4 * h + 3] = c4.w;
            }
#pragma unroll
            for (int r = 0; r < GEMV_RB; ++r) {
                if (r < rows) {
                    const uint4 uu = base[(long)r * nv + q];
                    const WT* w = reinterpret_cast<const WT*>(&uu);
                    float d = 0.f;
#pragma unroll
                    for (int k = 0; k < V; ++k) d = fmaf(dec(w[k]), cv[k], d);
                    acc[r] += d;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(empty + st));
#pragma unroll
        for (int r = 0; r < GEMV_RB; ++r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
            if (lane == 0 && r < rows) {
                const long I = r0 + (long)g * GEMV_RB + r;
                float v = fmaf(Pdiag[I], Cs[I], acc[r]);
                if (Pbc) v = fmaf(Pbc[I], (float)far_state[0], v);  // Eq.14 boundary term
                Cout[I] = v;
            }
        }
    }
}

// Eq.7 on the coarse mesh, one block of 256 threads: thread-strided fp64 partials, fixed
// shared-memory tree (deterministic)
__device__ void far_block(const float* __restrict__ C, const int* __restrict__ sizes, long N, double* far_state,
                          double v_far, int init, double c_far0)
{
    __shared__ double red[256];
    double s = 0.0;
    for (long I = threadIdx.x; I < N; I += 256) s += (double)sizes[I] * (double)C[I];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        s = red[0];
        if (init) {
            far_state[1] = s + c_far0 * v_far;  // K0 = Σ_{Ω_L} c(t0) + c_far(t0)·V_far
            far_state[0] = c_far0;
        } else {
            far_state[0] = (far_state[1] - s) / v_far;
        }
    }
}

__global__ void __launch_bounds__(256) k_far(const float* __restrict__ C, const int* __restrict__ sizes, long N,
                                             double* far_state, double v_far, int init, double c_far0)
{
    far_block(C, sizes, N, far_state, v_far, init, c_far0);
}

// c'_i = C'_{I(i)} over the Ω_L rows; with a far field block 0 does Eq.7 instead (it
// reads only C', so it runs beside the remap rather than as a fourth launch)
__global__ void __launch_bounds__(256) k_remap(const int* __restrict__ rows, long NL, const int* __restrict__ group_of,
                                               const float* __restrict__ C, float* __restrict__ c,
                                               const int* __restrict__ sizes, long N, double* far_state, double v_far)
{
    const unsigned f = far_state ? 1 : 0;
    if (f && blockIdx.x == 0) {  // first block: scheduled first, its serial reduction overlaps the remap
        far_block(C, sizes, N, far_state, v_far, 0, 0.0);
        return;
    }
    const unsigned nb = gridDim.x - f;
    for (long r = (blockIdx.x - f) * (long)blockDim.x + threadIdx.x; r < NL; r += (long)nb * blockDim.x) {
        const int v = rows[r];
        c[v] = C[group_of[v]];
    }
}

static void coarse_free(fdirw_coarse* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->graph2) cudaGraphExecDestroy(c->graph2);
    if (c->cap) cudaStreamDestroy(c->cap);
    cudaFree(c->group_of); cudaFree(c->rows); cudaFree(c->grp_ptr); cudaFree(c->grp_vox); cudaFree(c->sizes);
    cudaFree(c->P); cudaFree(c->Pdiag); cudaFree(c->C); cudaFree(c->C2); cudaFree(c->Pbc); cudaFree(c->far_state);
    delete c;
}

extern "C" fdirw_status fdirw_coarse_build(const fdirw_params* p, const uint8_t* region_host, int32_t block,
                                           void* cuda_stream, fdirw_coarse** out)
{
    if (!p || !region_host || !out) return cfail(FDIRW_E_INVALID, "NULL argument");
    *out = nullptr;
    if (p->nx < 1 || p->ny < 1 || p->nz < 1 || block < 1) return cfail(FDIRW_E_INVALID, "dims and block must be >= 1");
    if (!(p->dh > 0) || !(p->dt > 0) || !(p->D_fast > 0) || p->n_fd < 0)
        return cfail(FDIRW_E_INVALID, "need dh, dt, D_fast > 0 and n_fd >= 0");
    if (p->weights < 0 || p->weights > 2) return cfail(FDIRW_E_INVALID, "bad weight format");
    if (!(p->v_far >= 0)) return cfail(FDIRW_E_INVALID, "v_far must be >= 0");
    const long nvox = (long)p->nx * p->ny * p->nz;
    bool has_far = false;
    for (long i = 0; i < nvox && !has_far; ++i) has_far = region_host[i] == 2;
    if (has_far && !(p->v_far > 0)) return cfail(FDIRW_E_INVALID, "far-field voxels (2) need v_far > 0");
    // a1 for the fast phase (reading A5)
    long n = p->n_fd;
    if (n == 0) {
        const double x = p->D_fast * p->dt / (0.1 * p->dh * p->dh);
        const double cc = std::ceil(x * (1.0 - 1e-9));
        if (!(cc < 2.0e9)) return cfail(FDIRW_E_INVALID, "derived n_fd too large");
        n = cc < 1.0 ? 1 : (long)cc;
    }
    const double lam = (p->dt / (double)n) * p->D_fast / (p->dh * p->dh);
    if (lam > 1.0 / 6.0) return cfail(FDIRW_E_UNSTABLE, "explicit FD unstable: lambda > 1/6");

    fdirw_coarse* c = new fdirw_coarse();
    c->p = *p;
    c->n_fd = (int)n;
    c->lam = lam;
    c->b = block;
    c->fmt = p->weights;
    c->b_w = c->fmt == FDIRW_W_FP32 ? 4 : 2;
    c->far = p->v_far > 0;
    c->v_far = p->v_far;
    cudaGetDevice(&c->device);
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const int nx = p->nx, ny = p->ny, nz = p->nz, b = block;
    c->nvox = nvox;
    const int bx = (nx + b - 1) / b, by = (ny + b - 1) / b, bz = (nz + b - 1) / b;
    const long nblk = (long)bx * by * bz;

    uint8_t* reg = nullptr;
    int *used = nullptr, *bid = nullptr, *row_flag = nullptr, *row_pos = nullptr, *row_of = nullptr;
    int *row_group = nullptr, *row_group2 = nullptr, *nb = nullptr;
    float *X = nullptr, *Y = nullptr, *Z = nullptr;
    double* P64 = nullptr;
    void* tmp = nullptr;
    auto cleanup = [&]() {
        cudaFree(reg); cudaFree(used); cudaFree(bid); cudaFree(row_flag); cudaFree(row_pos); cudaFree(row_of);
        cudaFree(row_group); cudaFree(row_group2); cudaFree(nb); cudaFree(X); cudaFree(Y); cudaFree(Z); cudaFree(P64);
        cudaFree(tmp);
    };
    cudaError_t e = cudaSuccess;
#define T(call)                                                                     \
    do {                                                                            \
        e = (call);                                                                 \
        if (e != cudaSuccess) {                                                     \
            std::string m_ = std::string(#call) + ": " + cudaGetErrorString(e);     \
            cleanup();                                                              \
            coarse_free(c);                                                         \
            return cfail(e == cudaErrorMemoryAllocation ? FDIRW_E_OOM : FDIRW_E_CUDA, m_); \
        }                                                                           \
    } while (0)
    T(cudaMalloc(&reg, nvox));
    T(cudaMemcpyAsync(reg, region_host, nvox, cudaMemcpyHostToDevice, s));
    T(cudaMalloc(&used, (nblk + 1) * 4));
    T(cudaMalloc(&bid, (nblk + 1) * 4));
    T(cudaMemsetAsync(used, 0, (nblk + 1) * 4, s));
    k_mark_blocks<<<gridn(nvox), 256, 0, s>>>(reg, nvox, nx, ny, b, bx, by, used);
    T(cudaGetLastError());
    size_t tb = 0, tb2 = 0;
    T(cub::DeviceScan::ExclusiveSum(nullptr, tb, used, bid, (int)(nblk + 1), s));
    T(cub::DeviceScan::ExclusiveSum(nullptr, tb2, used, bid, (int)nvox, s));
    if (tb2 > tb) tb = tb2;
    T(cudaMalloc(&tmp, tb));
    T(cub::DeviceScan::ExclusiveSum(tmp, tb, used, bid, (int)(nblk + 1), s));
    int N = 0;
    T(cudaMemcpyAsync(&N, bid + nblk, 4, cudaMemcpyDeviceToHost, s));
    T(cudaStreamSynchronize(s));
    if (N == 0) {
        cleanup();
        coarse_free(c);
        return cfail(FDIRW_E_INVALID, "empty region");
    }
    c->N = N;
    T(cudaMalloc(&c->group_of, nvox * 4));
    T(cudaMalloc(&c->sizes, (long)N * 4));
    T(cudaMemsetAsync(c->sizes, 0, (long)N * 4, s));
    T(cudaMalloc(&row_flag, nvox * 4));
    T(cudaMalloc(&row_pos, nvox * 4));
    k_group_of<<<gridn(nvox), 256, 0, s>>>(reg, nvox, nx, ny, b, bx, by, bid, c->group_of, c->sizes, row_flag);
    T(cudaGetLastError());
    T(cub::DeviceScan::ExclusiveSum(tmp, tb, row_flag, row_pos, (int)nvox, s));
    int last[2];
    T(cudaMemcpyAsync(&last[0], row_pos + nvox - 1, 4, cudaMemcpyDeviceToHost, s));
    T(cudaMemcpyAsync(&last[1], row_flag + nvox - 1, 4, cudaMemcpyDeviceToHost, s));
    T(cudaStreamSynchronize(s));
    const long NL = (long)last[0] + last[1];
    c->NL = NL;
    T(cudaMalloc(&c->rows, NL * 4));
    T(cudaMalloc(&row_of, nvox * 4));
    T(cudaMalloc(&row_group, NL * 4));
    T(cudaMalloc(&row_group2, NL * 4));
    k_rows<<<gridn(nvox), 256, 0, s>>>(row_flag, row_pos, nvox, c->rows, row_of, c->group_of, row_group);
    T(cudaGetLastError());
    // group CSR: stable sort of (group, voxel) over the region rows
    T(cudaMalloc(&c->grp_vox, NL * 4));
    T(cudaMalloc(&c->grp_ptr, ((long)N + 1) * 4));
    size_t ts = 0;
    T(cub::DeviceRadixSort::SortPairs(nullptr, ts, row_group, row_group2, c->rows, c->grp_vox, (int)NL, 0, 32, s));
    if (ts > tb) {
        cudaFree(tmp);
        tmp = nullptr;
        T(cudaMalloc(&tmp, ts));
        tb = ts;
    }
    T(cub::DeviceRadixSort::SortPairs(tmp, tb, row_group, row_group2, c->rows, c->grp_vox, (int)NL, 0, 32, s));
    T(cudaMemsetAsync(c->grp_ptr, 0, 4, s));
    T(cub::DeviceScan::InclusiveSum(tmp, tb, c->sizes, c->grp_ptr + 1, N, s));
    T(cudaMalloc(&nb, NL * 6 * 4));
    k_neighbours<<<gridn(NL), 256, 0, s>>>(c->rows, NL, row_of, reg, nx, ny, nz, nb);
    T(cudaGetLastError());

    // P (and P_BC as column N) by batched FD over Ω_L, CB columns per pass
    const long Ncol = (long)N + (c->far ? 1 : 0);
    // 512 columns per chunk: 3 z-planes of the region's rows stay in L2 (measured: 512 beats
    // 1024-2048 by 3-8 %); three buffers (cur, prev, acc) for the Chebyshev recurrence
    const long budget = 6L << 30;
    long CB = budget / (3L * 4 * NL);
    if (CB > 512) CB = 512;
    CB = CB < 4 ? 4 : (CB / 4) * 4;
    const long Npad = (Ncol + 3) / 4 * 4;
    if (CB > Npad) CB = Npad;
    T(cudaMalloc(&X, NL * CB * 4));
    T(cudaMalloc(&Y, NL * CB * 4));
    T(cudaMalloc(&Z, NL * CB * 4));
    T(cudaMalloc(&P64, (long)N * Ncol * 8));
    const int Nbc = c->far ? N : -1;
    // P columns of a closed region: kCheb_pre literal substeps, then the Chebyshev recurrence
    // for the remaining n_fd − kCheb_pre (reading A30), columns renormalised to their exact mass
    // N_J.  Literal substeps instead with FDIRW_F_KGEN_DIRECT, a small n_fd, or a far field:
    // there most of a column's mass leaks to the reservoir, and the recurrence's rounding — on
    // the scale of the source, not of what remains — would cost the remaining mass its fp32
    // accuracy (measured 1.8e-5 relative vs 2e-6 for the substeps).  The P_BC column
    // (inhomogeneous: its far faces see the Dirichlet value 1) runs in a chunk of its own.
    std::vector<float> cheb;
    // (with a far field and fp16 / bf16 storage the recurrence too, FDIRW_COARSE_OPEN_LITERAL=1: literal)
    const bool far_lit = c->far && (c->fmt == 0 || getenv("FDIRW_COARSE_OPEN_LITERAL"));
    const int m = (p->flags & FDIRW_F_KGEN_DIRECT) || c->n_fd <= 2 * kCheb_pre || far_lit
                      ? 0 : cheb_plan(c->n_fd - kCheb_pre, lam, &cheb);
    c->fd_passes = m > 0 ? kCheb_pre + m : c->n_fd;
    const float mu2 = (float)(lam * 4.0 / (12.0 * lam));  // 2μ = 4λ/(1 − a), 1 − a = 12λ: 1/3
    auto direct = [&](float*& a, float*& bb, int cb, int j0, int passes) {
        for (int k = 0; k < passes; ++k) {
            k_fd_cols<<<gridn(NL * 32), 256, 0, s>>>(a, bb, nb, NL, cb, (float)lam, j0, Nbc);
            float* t = a; a = bb; bb = t;
        }
    };
    for (long J0 = 0; J0 < N; J0 += CB) {
        const int Jn = (int)((N - J0) < CB ? (N - J0) : CB);
        k_init_cols<<<gridn(NL * CB), 256, 0, s>>>(row_group, NL, (int)CB, (int)J0, X);
        T(cudaGetLastError());
        float *a = X, *bb = Y;
        if (m == 0) {
            direct(a, bb, (int)CB, (int)J0, c->n_fd);
        } else {
            direct(a, bb, (int)CB, (int)J0, kCheb_pre);  // a = v = A^pre·1_J
            k_cheb_cols<<<gridn(NL * 32), 256, 0, s>>>(a, bb, Z, nb, NL, (int)CB, mu2, cheb[0], cheb[1], 1);
            for (int k = 1; k < m; ++k) {  // bb = t_k, a = t_{k−1} ← t_{k+1}
                k_cheb_cols<<<gridn(NL * 32), 256, 0, s>>>(bb, a, Z, nb, NL, (int)CB, mu2, 0.f, cheb[k + 1], 0);
                float* t = a; a = bb; bb = t;
            }
            a = Z;
        }
        T(cudaGetLastError());
        k_map_cols<<<gridn((long)N * Jn), 256, 0, s>>>(a, c->grp_ptr, c->grp_vox, row_of, N, Ncol, (int)CB, (int)J0,
                                                       Jn, P64);
        T(cudaGetLastError());
    }
    if (c->far) {  // P_BC = column N, literal substeps (4-wide chunk)
        k_init_cols<<<gridn(NL * 4), 256, 0, s>>>(row_group, NL, 4, N, X);
        T(cudaGetLastError());
        float *a = X, *bb = Y;
        direct(a, bb, 4, N, c->n_fd);
        T(cudaGetLastError());
        k_map_cols<<<gridn((long)N), 256, 0, s>>>(a, c->grp_ptr, c->grp_vox, row_of, N, Ncol, 4, N, 1, P64);
        T(cudaGetLastError());
    }
    if (m > 0 && !c->far) {
        k_renorm_cols<<<N, 256, 0, s>>>(P64, Ncol, c->sizes, N);
        T(cudaGetLastError());
    }
    c->ldp = ((long)N + 7) / 8 * 8;
    T(cudaMalloc(&c->P, (long)N * c->ldp * c->b_w));
    T(cudaMemsetAsync(c->P, 0, (long)N * c->ldp * c->b_w, s));
    T(cudaMalloc(&c->Pdiag, (long)N * 4));
    if (c->fmt == 0) k_quantize<float><<<N, 256, 0, s>>>(P64, Ncol, c->sizes, N, c->ldp, (float*)c->P, c->Pdiag);
    else if (c->fmt == 1) k_quantize<__half><<<N, 256, 0, s>>>(P64, Ncol, c->sizes, N, c->ldp, (__half*)c->P, c->Pdiag);
    else k_quantize<__nv_bfloat16><<<N, 256, 0, s>>>(P64, Ncol, c->sizes, N, c->ldp, (__nv_bfloat16*)c->P, c->Pdiag);
    T(cudaGetLastError());
    if (c->far) {
        T(cudaMalloc(&c->Pbc, (long)N * 4));
        T(cudaMalloc(&c->far_state, 16));
        T(cudaMemsetAsync(c->far_state, 0, 16, s));
        k_pbc<<<gridn(N), 256, 0, s>>>(P64, Ncol, N, c->Pbc);
        T(cudaGetLastError());
    }
    T(cudaMalloc(&c->C, c->ldp * 4));
    T(cudaMalloc(&c->C2, c->ldp * 4));
    T(cudaMemsetAsync(c->C, 0, c->ldp * 4, s));
    T(cudaMemsetAsync(c->C2, 0, c->ldp * 4, s));
    T(cudaStreamSynchronize(s));
    T(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
    {  // bulk-copy GEMV: as many row-group stages per consumer warp (≤ 4) as shared memory allows
        int dev_smem = 0;
        T(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
        T(cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, c->device));
        const size_t rowB = (size_t)c->ldp * c->b_w, cB = ((size_t)c->ldp * 4 + 127) / 128 * 128;
        const int fl = getenv("FDIRW_COARSE_GEMV") ? atoi(getenv("FDIRW_COARSE_GEMV")) : 0;  // 1 = bulk GEMV
        for (int m = 4; m >= 1 && fl == 1; --m) {
            const size_t need = ((16 * GEMV_NW * m + 127) / 128) * 128 + cB + (size_t)GEMV_NW * m * GEMV_RB * rowB;
            if (need <= (size_t)dev_smem) {
                c->bulk_m = m;
                c->bulk_smem = need;
                break;
            }
        }
        if (c->bulk_m > 0) {
            const void* f = c->fmt == 0 ? (const void*)k_gemv_bulk<float>
                          : c->fmt == 1 ? (const void*)k_gemv_bulk<__half> : (const void*)k_gemv_bulk<__nv_bfloat16>;
            T(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->bulk_smem));
        }
    }
#undef T
    cleanup();
    *out = c;
    return FDIRW_OK;
}

// GEMV launch: one block per SM, ⌈row groups / SMs⌉ warps each (≤ 16; more groups loop)
static unsigned gemv_grid(const fdirw_coarse* c) { return (unsigned)c->n_sm; }
static unsigned gemv_block(const fdirw_coarse* c)
{
    const long groups = (c->N + GEMV_RW - 1) / GEMV_RW;
    long w = (groups + c->n_sm - 1) / c->n_sm;
    if (w < 1) w = 1;
    if (w > 16) w = 16;
    return (unsigned)(32 * w);
}

// One coarse GEMV C' = P̃·Cin + diag∘Cin (+ P_BC·c_far): the bulk form, or the register form with
// C staged in shared memory; fine ≠ null (closed domain) fuses the remap of C' into cbuf.
static cudaError_t coarse_gemv(fdirw_coarse* c, const float* Cin, float* Cout, float* fine, cudaStream_t s)
{
    const long N = c->N;
    if (c->bulk_m > 0) {
        const dim3 g((unsigned)(N < c->n_sm ? N : c->n_sm)), bl((GEMV_NW + 1) * 32);
        if (c->fmt == 0)
            k_gemv_bulk<float><<<g, bl, c->bulk_smem, s>>>((const float*)c->P, c->Pdiag, Cin, N, c->ldp, Cout,
                                                          c->Pbc, c->far_state, c->bulk_m);
        else if (c->fmt == 1)
            k_gemv_bulk<__half><<<g, bl, c->bulk_smem, s>>>((const __half*)c->P, c->Pdiag, Cin, N, c->ldp, Cout,
                                                           c->Pbc, c->far_state, c->bulk_m);
        else
            k_gemv_bulk<__nv_bfloat16><<<g, bl, c->bulk_smem, s>>>((const __nv_bfloat16*)c->P, c->Pdiag, Cin, N,
                                                                  c->ldp, Cout, c->Pbc, c->far_state, c->bulk_m);
        return cudaGetLastError();
    }
    // C in shared memory when it fits (FDIRW_COARSE_GEMV_L1=1: the L1 form, A/B)
    static const bool l1 = getenv("FDIRW_COARSE_GEMV_L1") != nullptr;
    const size_t csm = (size_t)c->ldp * 4;
    const bool smc = !l1 && csm <= 96 * 1024;
    auto go = [&](auto wt) -> cudaError_t {
        using WT = decltype(wt);
        const WT* P = (const WT*)c->P;
        if (smc) {
            cudaError_t e = cudaFuncSetAttribute(k_gemv<WT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)csm);
            if (e != cudaSuccess) return e;
            k_gemv<WT, true><<<gemv_grid(c), gemv_block(c), csm, s>>>(P, c->Pdiag, Cin, N, c->ldp, Cout, c->Pbc,
                                                                     c->far_state, c->grp_ptr, c->grp_vox, fine);
        } else {
            k_gemv<WT, false><<<gemv_grid(c), gemv_block(c), 0, s>>>(P, c->Pdiag, Cin, N, c->ldp, Cout, c->Pbc,
                                                                      c->far_state, c->grp_ptr, c->grp_vox, fine);
        }
        return cudaGetLastError();
    };
    return c->fmt == 0 ? go(float{}) : c->fmt == 1 ? go(__half{}) : go(__nv_bfloat16{});
}

// One whole coarse step on the fine field cbuf: map, GEMV, remap (+ Eq.7 with a far
// field, in the remap's first block).  Closed domains with the register GEMV fuse the remap.
static cudaError_t coarse_enqueue(fdirw_coarse* c, float* cbuf, cudaStream_t s)
{
    const long N = c->N;
    k_map<<<gridn(N * 32), 256, 0, s>>>(cbuf, c->grp_ptr, c->grp_vox, N, c->C);
    const bool fuse = !c->far && c->bulk_m == 0;
    cudaError_t e = coarse_gemv(c, c->C, c->C2, fuse ? cbuf : nullptr, s);
    if (e != cudaSuccess) return e;
    if (!fuse)
        k_remap<<<gridn(c->NL) + (c->far ? 1 : 0), 256, 0, s>>>(c->rows, c->NL, c->group_of, c->C2, cbuf, c->sizes, N,
                                                               c->far ? c->far_state : nullptr, c->v_far);
    return cudaGetLastError();
}

extern "C" fdirw_status fdirw_coarse_step(fdirw_coarse* c, const float* cin, float* cout, void* cuda_stream)
{
    if (!c || !cin || !cout) return cfail(FDIRW_E_INVALID, "NULL argument");
    if (cin == cout) return cfail(FDIRW_E_ALIAS, "c_in == c_out");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    CK(cudaMemcpyAsync(cout, cin, c->nvox * 4, cudaMemcpyDeviceToDevice, s));
    CK(coarse_enqueue(c, cout, s));
    return FDIRW_OK;
}

// n steps (round 2): between steps the fine field inside Ω_L is the remap of C' — constant over
// each group — so the next map would only re-average equal values.  The run therefore maps once,
// steps the group values (C ↔ C2 ping-pong; Eq.7 after each GEMV with a far field), and remaps
// once at the end: the same operator sequence without the n − 1 intermediate map/remap pairs
// (whose re-averaging only adds fp32 rounding).  Two steps are one captured graph, replayed.
extern "C" fdirw_status fdirw_coarse_run(fdirw_coarse* c, float* cbuf, int32_t n, void* cuda_stream)
{
    if (!c || !cbuf) return cfail(FDIRW_E_INVALID, "NULL argument");
    if (n < 0) return cfail(FDIRW_E_INVALID, "n_steps must be >= 0");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    if (n == 0) return FDIRW_OK;
    const long N = c->N;
    const bool per_step = getenv("FDIRW_COARSE_PER_STEP_REMAP") != nullptr;  // (A/B: map/remap each step; read per call)
    if (per_step) {
        if (!c->graph || c->graph_c != cbuf) {
            if (c->graph) cudaGraphExecDestroy(c->graph);
            c->graph = nullptr;
            CK(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = coarse_enqueue(c, cbuf, c->cap);
            cudaGraph_t g = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(c->cap, &g);
            if (e != cudaSuccess || e2 != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                return cfail(FDIRW_E_CUDA, std::string("coarse graph capture: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
            }
            e = cudaGraphInstantiate(&c->graph, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) { c->graph = nullptr; return cfail(FDIRW_E_CUDA, std::string("graph: ") + cudaGetErrorString(e)); }
            c->graph_c = cbuf;
        }
        for (int i = 0; i < n; ++i) CK(cudaGraphLaunch(c->graph, s));
        return FDIRW_OK;
    }
    auto step = [&](const float* Cin, float* Cout, cudaStream_t ss) -> cudaError_t {
        cudaError_t e = coarse_gemv(c, Cin, Cout, nullptr, ss);
        if (e != cudaSuccess) return e;
        if (c->far) k_far<<<1, 256, 0, ss>>>(Cout, c->sizes, N, c->far_state, c->v_far, 0, 0.0);  // Eq.7
        return cudaGetLastError();
    };
    k_map<<<gridn(N * 32), 256, 0, s>>>(cbuf, c->grp_ptr, c->grp_vox, N, c->C);
    CK(cudaGetLastError());
    if (n >= 2) {
        if (!c->graph2) {  // C → C2 → C
            CK(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = step(c->C, c->C2, c->cap);
            if (e == cudaSuccess) e = step(c->C2, c->C, c->cap);
            cudaGraph_t g = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(c->cap, &g);
            if (e != cudaSuccess || e2 != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                return cfail(FDIRW_E_CUDA, std::string("coarse graph capture: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
            }
            e = cudaGraphInstantiate(&c->graph2, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) { c->graph2 = nullptr; return cfail(FDIRW_E_CUDA, std::string("graph: ") + cudaGetErrorString(e)); }
        }
        for (int i = 0; i < n / 2; ++i) CK(cudaGraphLaunch(c->graph2, s));
    }
    const float* last = c->C;
    if (n & 1) {
        CK(step(c->C, c->C2, s));
        last = c->C2;
    }
    k_remap<<<gridn(c->NL), 256, 0, s>>>(c->rows, c->NL, c->group_of, last, cbuf, c->sizes, N, nullptr, 0.0);
    CK(cudaGetLastError());
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_coarse_far_init(fdirw_coarse* c, const float* c_dev, double c_far0, double* M_out,
                                              void* cuda_stream)
{
    if (!c || !c_dev) return cfail(FDIRW_E_INVALID, "NULL argument");
    if (!c->far) return cfail(FDIRW_E_STATE, "closed-domain coarse context (v_far = 0)");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    // Σ_{Ω_L} c(t0) as Σ_I N_I C_I of the mapped field (the coarse step's own conserved form)
    k_map<<<gridn(c->N * 32), 256, 0, s>>>(c_dev, c->grp_ptr, c->grp_vox, c->N, c->C2);
    k_far<<<1, 256, 0, s>>>(c->C2, c->sizes, c->N, c->far_state, c->v_far, 1, c_far0);
    CK(cudaGetLastError());
    double fs[2];
    CK(cudaMemcpyAsync(fs, c->far_state, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (M_out) *M_out = fs[1];
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_coarse_far_get(fdirw_coarse* c, double* c_far_out, void* cuda_stream)
{
    if (!c || !c_far_out) return cfail(FDIRW_E_INVALID, "NULL argument");
    if (!c->far) return cfail(FDIRW_E_STATE, "closed-domain coarse context (v_far = 0)");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    CK(cudaMemcpyAsync(c_far_out, c->far_state, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_coarse_query(const fdirw_coarse* c, fdirw_coarse_info* info)
{
    if (!c || !info) return cfail(FDIRW_E_INVALID, "NULL argument");
    info->n_fd = c->n_fd;
    info->block = c->b;
    info->n_groups = c->N;
    info->n_region = c->NL;
    info->p_bytes = (uint64_t)c->N * c->ldp * c->b_w + (uint64_t)c->N * 4 * (c->far ? 2 : 1);
    info->flops_per_step = (uint64_t)c->N * (c->N + 1) + 2ull * c->NL;
    info->fd_passes = c->fd_passes;
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_coarse_export(const fdirw_coarse* c, double* P_host, int32_t* group_of_host)
{
    if (!c) return cfail(FDIRW_E_INVALID, "NULL argument");
    CK(cudaSetDevice(c->device));
    const long N = c->N;
    if (P_host) {
        const long ld = c->ldp;
        std::vector<unsigned char> raw((size_t)N * ld * c->b_w);
        std::vector<float> dg(N);
        CK(cudaMemcpy(raw.data(), c->P, raw.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(dg.data(), c->Pdiag, N * 4, cudaMemcpyDeviceToHost));
        for (long I = 0; I < N; ++I)
            for (long J = 0; J < N; ++J) {
                const long i = I * ld + J;
                double v;
                if (c->fmt == 0) { float f; memcpy(&f, &raw[i * 4], 4); v = f; }
                else if (c->fmt == 1) { __half h; memcpy(&h, &raw[i * 2], 2); v = __half2float(h); }
                else { __nv_bfloat16 h; memcpy(&h, &raw[i * 2], 2); v = __bfloat162float(h); }
                P_host[I * N + J] = v;
            }
        for (long I = 0; I < N; ++I) P_host[I * N + I] = dg[I];
    }
    if (group_of_host) CK(cudaMemcpy(group_of_host, c->group_of, c->nvox * 4, cudaMemcpyDeviceToHost));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_coarse_export_pbc(const fdirw_coarse* c, double* pbc_host)
{
    if (!c || !pbc_host) return cfail(FDIRW_E_INVALID, "NULL argument");
    if (!c->far) return cfail(FDIRW_E_STATE, "closed-domain coarse context (v_far = 0)");
    CK(cudaSetDevice(c->device));
    std::vector<float> v(c->N);
    CK(cudaMemcpy(v.data(), c->Pbc, c->N * 4, cudaMemcpyDeviceToHost));
    for (long i = 0; i < c->N; ++i) pbc_host[i] = v[i];
    return FDIRW_OK;
}

extern "C" void fdirw_coarse_destroy(fdirw_coarse* c) { coarse_free(c); }
