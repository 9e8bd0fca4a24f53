// kgen.cu — a3/a4: batched-window explicit FD kernel generation + quantising epilogue.
//
// For every source s (§3.1: column j of p "obtained directly by solving the
// governing diffusion equation with an initial single point source ... using the
// explicit Finite Difference Method"), run n_fd Jacobi substeps of the 7-point
// variable-coefficient stencil inside the source's (2R+1)^3 window (north_star;
// readings A1-A4, A21 in DESIGN.md):
//     c⁰ = δ_s,  c^{k+1}_i = c^k_i + Σ_{j∈nb(i)∩Ω_s} λ_ij (c^k_j − c^k_i)
// with λ_ij = Δt_fd·H(D_i, D_j)/Δh² (harmonic mean H), no flux across window or
// domain edges.  Then (a4): renormalise by the fp64 sum, round every off-centre
// weight to fp32 then to the storage format (RNE, §3.3), set the fp32
// diagonal d_s = 1 − Σ_{o≠0} W̃_s(o) (fp64 sum; reading A10) and scatter the
// weights into the gather layout Wt[tile(x)][slot(o)][e(x)][j(x)], x = s + o.
//
// Mapping: one CTA per window at a time (persistent grid, sources x-fastest so
// the CTAs in flight write neighbouring targets and L2 merges the 2-byte writes).
// Thread t < L² owns the z-column (ox, oy) = (t % L − R, t / L − R) of the window
// in registers: the ±z neighbours are register reads; the ±x/±y neighbours come
// from a double-buffered shared-memory copy of the window (one barrier per
// substep).  The 6 face numbers of every owned cell live in registers.
// Bound: shared-memory bandwidth (4 LDS + 1 STS per cell-update).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <type_traits>

#include "fdirw_internal.h"
#include "kgen_common.cuh"
#include "layout.cuh"

namespace fdirw {

template <int R, bool F64 = false>
struct KgenShape {
    static constexpr int L = 2 * R + 1;
    static constexpr int LL = L * L;
    static constexpr int LLL = L * L * L;
    static constexpr int NT = ((LL + 31) / 32) * 32;
    static constexpr int NW = NT / 32;
    static constexpr int Lp = (L + 3) / 4 * 4;                             // column padded to float4s
    static constexpr size_t smem_floats = 2 * (size_t)NT * Lp;             // double-buffered, column-major
    static constexpr size_t buf_bytes = smem_floats * (F64 ? 8 : 4);
    static constexpr size_t tab_off = buf_bytes + ((LLL + 15) / 16) * 16 + NW * 8 + 16;  // face tables
    static constexpr size_t smem_bytes = tab_off + 64 * 4;
    static constexpr size_t cheb_off = smem_bytes;  // Chebyshev coefficients c_0..c_m (fp32) follow
    // CTAs per SM the register allocation is sized for: ~128 registers per thread (R5 measured
    // 3 → 4 CTAs: −2.5 % kernel time; R7 would spill 212 B at 2 CTAs, so it keeps 1)
    static constexpr int kMinBlocks = (R != 7 && 65536 / (NT * 128) > 1) ? 65536 / (NT * 128) : 1;
};

__device__ __forceinline__ double face_lambda_d(unsigned p, unsigned q, const double* lam)
{
    if (p > 1u || q == 2u) return 0.0;
    if (q == 3u) q = 1u;
    return (p & q) ? lam[0] : ((p | q) ? lam[1] : lam[2]);
}

// F64 = true: FDIRW_F_KGEN_FP64 (reading A22, debugging).  The same window, thread mapping
// and epilogue, but the substeps run in fp64 in the oracle's operation order
// (acc = c; acc += λ_f·(c_f − c) for f = −x,+x,−y,+y,−z,+z, separate multiply and add, no
// FMA) and the result is not renormalised (fp64 FD keeps Σ = 1 to rounding), so the
// off-centre weights are the oracle's O2 kernels rounded exactly as O5 rounds them.
template <int R, bool F64>
__global__ void __launch_bounds__(KgenShape<R, F64>::NT, F64 ? 1 : KgenShape<R, F64>::kMinBlocks) kgen_kernel(const KgenArgs a)
{
    using S = KgenShape<R, F64>;
    using T = typename std::conditional<F64, double, float>::type;
    constexpr int L = S::L, LL = S::LL, LLL = S::LLL, NT = S::NT;
    constexpr int KC = LLL / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* buf = reinterpret_cast<T*>(smem_raw);
    unsigned char* ph = smem_raw + S::buf_bytes;
    double* red = reinterpret_cast<double*>(smem_raw + S::buf_bytes + ((LLL + 15) / 16) * 16);

    const int t = threadIdx.x;
    const bool col = t < LL;
    const int cx = t % L, cy = t / L;
    const int oxm = (col && cx > 0) ? -1 : 0, oxp = (col && cx < L - 1) ? 1 : 0;
    const int oym = (col && cy > 0) ? -L : 0, oyp = (col && cy < L - 1) ? L : 0;
    // smem read offsets of the ±x neighbours: a column on the window's x edge has no neighbour
    // there (face number 0), but reading its own slot would leave a hole in the warp's run of
    // consecutive float4s at every row boundary, which splits an 8-lane LDS.128 phase over two
    // bank rounds (ncu: 5.4 % of the shared wavefronts were conflicts).  It reads the adjacent
    // row's edge column instead (a written, finite window value; 0·(v − c) adds ±0).
    const int axm = (col && (cx > 0 || t > 0)) ? -1 : 0, axp = (col && (cx < L - 1 || t + 1 < LL)) ? 1 : 0;
    const int nx = a.nx, ny = a.ny, nz = a.nz;
    const long nsrc = a.src_list ? a.n_list : (long)nx * ny * (a.sz1 - a.sz0);

    float* ftab = reinterpret_cast<float*>(smem_raw + S::tab_off);
    if (!F64) build_face_tables(ftab, a.lam_ff, a.lam_fs, a.lam_ss, a.mu2_ff, a.mu2_fs, a.mu2_ss);
    if (!F64 && a.cheb_m) {
        float* cc = reinterpret_cast<float*>(smem_raw + S::cheb_off);
        for (int i = t; i <= a.cheb_m; i += NT) cc[i] = a.cheb_c[i];
        // (the first window's __syncthreads below orders these stores before any read)
    }
    for (long it = blockIdx.x; it < nsrc; it += gridDim.x) {
        const long src = a.src_list ? (long)a.src_list[it] : it;
        const int sx = (int)(src % nx);
        const int sy = (int)((src / nx) % ny);
        const int sz = a.sz0 + (int)(src / ((long)nx * ny));

        // window phases → smem (2 = outside the domain, 3 = far field)
        __syncthreads();  // the previous source's readers of ph are done
        int far_here = 0;
        for (int i = t; i < LLL; i += NT) {
            const int gx = sx + i % L - R, gy = sy + (i / L) % L - R, gz = sz + i / LL - R;
            const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz;
            unsigned char v = in ? a.mask[((size_t)(gz - a.mz0) * ny + gy) * nx + gx] : (unsigned char)2;
            if (in && v == 2) v = 3;
            far_here |= v == 3;
            ph[i] = v;
        }
        const bool open = __syncthreads_or(far_here) != 0;  // window touches the reservoir
        if (ph[KC] == 3) continue;  // far-field voxels are not sources (their value is c_far)

        constexpr int Lp = S::Lp;
        T c[Lp];
        if constexpr (F64) {
#pragma unroll
            for (int z = 0; z < Lp; ++z) c[z] = (col && t == R * L + R && z == R) ? 1.0 : 0.0;
            for (int k = 0; k < a.n_fd; ++k) {
                double* b = buf + (k & 1) * (NT * Lp);
                if (col) {
#pragma unroll
                    for (int z = 0; z < Lp; ++z) b[t * Lp + z] = c[z];
                }
                __syncthreads();
                if (col) {
                    double nw[L];
#pragma unroll
                    for (int z = 0; z < L; ++z) {
                        const int i = z * LL + t;
                        const unsigned p = ph[i];
                        double acc = c[z];
                        const double cz = c[z];
                        // −x, +x, −y, +y, −z, +z (the oracle's face order)
                        if (oxm) acc = __dadd_rn(acc, __dmul_rn(face_lambda_d(p, ph[i + oxm], a.lam_d),
                                                                __dsub_rn(b[(t + oxm) * Lp + z], cz)));
                        if (oxp) acc = __dadd_rn(acc, __dmul_rn(face_lambda_d(p, ph[i + oxp], a.lam_d),
                                                                __dsub_rn(b[(t + oxp) * Lp + z], cz)));
                        if (oym) acc = __dadd_rn(acc, __dmul_rn(face_lambda_d(p, ph[i + oym], a.lam_d),
                                                                __dsub_rn(b[(t + oym) * Lp + z], cz)));
                        if (oyp) acc = __dadd_rn(acc, __dmul_rn(face_lambda_d(p, ph[i + oyp], a.lam_d),
                                                                __dsub_rn(b[(t + oyp) * Lp + z], cz)));
                        if (z > 0) acc = __dadd_rn(acc, __dmul_rn(face_lambda_d(p, ph[i - LL], a.lam_d),
                                                                  __dsub_rn(c[z - 1], cz)));
                        if (z < L - 1) acc = __dadd_rn(acc, __dmul_rn(face_lambda_d(p, ph[i + LL], a.lam_d),
                                                                      __dsub_rn(c[z + 1], cz)));
                        nw[z] = acc;
                    }
#pragma unroll
                    for (int z = 0; z < L; ++z) c[z] = nw[z];
                }
            }
        } else {
        // Face numbers in registers: λ for the direct substeps; 2μ = 4λ/(1 − a) (rounded once
        // from fp64 on the host) for the Chebyshev recurrence, which steps the mapped operator
        // Â = (2A − (1 + a)I)/(1 − a) = I + Σ μ_f (c_f − c).
        // z faces: fz[z] = the face between cells z and z + 1, as seen from its active side
        // (face_lambda is symmetric except towards a reservoir cell, whose own faces are 0):
        // both cells read the same register, 17 fewer per thread at R8 than separate −z / +z
        // arrays.  A reservoir cell (open windows, N2) then picks up z fluxes, so the literal
        // substeps reset it to its Dirichlet 0 (rmask); closed windows have none.
        float fz[L > 1 ? L - 1 : 1];
        unsigned rmask = 0;
        // Lateral face numbers: cells (2h, 2h+1) packed for FFMA2/FADD2, h < NPR; the odd last
        // cell L − 1 on its own (L = 2R + 1 is odd).
        constexpr int NPR = (L - 1) / 2;
        unsigned long long lxm2[NPR > 0 ? NPR : 1], lxp2[NPR > 0 ? NPR : 1], lym2[NPR > 0 ? NPR : 1],
            lyp2[NPR > 0 ? NPR : 1];
        float lxm1, lxp1, lym1, lyp1;
        // Chebyshev passes (reading A30) in the operator's row form: 2Â t = D∘t + Σ_f F_f t_f with
        // F_f = 2μ_f and the cell's own coefficient D = 2 − Σ_f F_f (fp64 sum, rounded once), so Â
        // keeps constants as stored.  Packed like the lateral numbers (dg2 pairs, dg1 the last cell).
        unsigned long long dg2[NPR > 0 ? NPR : 1];
        float dg1 = 0.f;
        auto faces = [&](const float* T, const bool row_form) {  // T: face table set (λ or 2μ)
            float v[4][L];
#pragma unroll
            for (int z = 0; z < L; ++z) {
                const int i = z * LL + t;
                const unsigned p = col ? ph[i] : 2u;
                v[0][z] = (col && oxm) ? T[(p << 2) | ph[i + oxm]] : 0.f;
                v[1][z] = (col && oxp) ? T[(p << 2) | ph[i + oxp]] : 0.f;
                v[2][z] = (col && oym) ? T[(p << 2) | ph[i + oym]] : 0.f;
                v[3][z] = (col && oyp) ? T[(p << 2) | ph[i + oyp]] : 0.f;
                if (z < L - 1) {
                    const unsigned q = col ? ph[i + LL] : 2u;
                    fz[z] = col ? T[16 + ((p << 2) | q)] : 0.f;
                }
                if (col && p == 3u) rmask |= 1u << z;
            }
            if (row_form) {
                float d[L];
#pragma unroll
                for (int z = 0; z < L; ++z) {
                    double f = (double)v[0][z] + (double)v[1][z] + (double)v[2][z] + (double)v[3][z];
                    if (z > 0) f += (double)fz[z - 1];
                    if (z < L - 1) f += (double)fz[z];
                    d[z] = col ? (float)(2.0 - f) : 0.f;
                }
#pragma unroll
                for (int h = 0; h < NPR; ++h) dg2[h] = pk2(d[2 * h], d[2 * h + 1]);
                dg1 = d[L - 1];
            }
#pragma unroll
            for (int h = 0; h < NPR; ++h) {
                lxm2[h] = pk2(v[0][2 * h], v[0][2 * h + 1]);
                lxp2[h] = pk2(v[1][2 * h], v[1][2 * h + 1]);
                lym2[h] = pk2(v[2][2 * h], v[2][2 * h + 1]);
                lyp2[h] = pk2(v[3][2 * h], v[3][2 * h + 1]);
            }
            lxm1 = v[0][L - 1];
            lxp1 = v[1][L - 1];
            lym1 = v[2][L - 1];
            lyp1 = v[3][L - 1];
        };
        faces(ftab, false);
#pragma unroll
        for (int z = 0; z < Lp; ++z) c[z] = (col && t == R * L + R && z == R) ? 1.f : 0.f;

        // The window in smem, one buffer of NT·L floats per parity: each column's first 4·NH
        // cells as float4 quads laid out quad-major (quad q of column t at q·NT + t), the
        // remaining NTL (1 or 3) cells as scalars (cell 4·NH + j at j·NT + t).  Consecutive
        // threads touch consecutive 16 / 4 bytes: conflict-free, and no padding cell moves.
        constexpr int NH = L / 4, NTL = L - 4 * NH;
        auto store_col = [&](float* b, const float (&v)[Lp]) {
            float4* b4 = reinterpret_cast<float4*>(b);
#pragma unroll
            for (int q = 0; q < NH; ++q) b4[q * NT + t] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
#pragma unroll
            for (int j = 0; j < NTL; ++j) b[4 * NH * NT + j * NT + t] = v[4 * NH + j];
        };
        auto load_col = [&](const float* b, const int tt, float (&v)[L]) {
            const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
            for (int q = 0; q < NH; ++q) {
                const float4 w = b4[q * NT + tt];
                v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
            }
#pragma unroll
            for (int j = 0; j < NTL; ++j) v[4 * NH + j] = b[4 * NH * NT + j * NT + tt];
        };
        // nw += Σ over −x,+x,−y,+y of λ_f (c_f − c), cells in pairs (FADD2/FFMA2) and the last alone;
        // then the two z faces from registers (one difference per face, used by both cells:
        // c_{z−1} − c_z is exactly −(c_z − c_{z−1}) in IEEE arithmetic).
        auto flux = [&](const float* b, const float (&cur)[Lp], float (&nw)[Lp]) {
            float xm[L], xp[L], ym[L], yp[L];
            load_col(b, t + axm, xm);
            load_col(b, t + axp, xp);
            load_col(b, t + oym, ym);
            load_col(b, t + oyp, yp);
            // z faces from registers: for R ≤ 5 before the lateral faces, so they run while the
            // neighbours' shared-memory loads are in flight (cfg3 kgen 140 → 135 ms); for larger
            // R after them (the other order measured 4 % slower at R8).  Either order is fixed
            // per R, so every path (dedup or not, any decomposition) gives the same bits.
            auto zfaces = [&]() {
                float dz[L > 1 ? L - 1 : 1];
#pragma unroll
                for (int z = 0; z + 1 < L; ++z) dz[z] = cur[z + 1] - cur[z];
#pragma unroll
                for (int z = 0; z < L; ++z) {
                    float v = nw[z];
                    if (z > 0) v = fmaf(fz[z - 1], -dz[z - 1], v);
                    if (z < L - 1) v = fmaf(fz[z], dz[z], v);
                    nw[z] = v;
                }
            };
            if constexpr (R <= 5) zfaces();
#pragma unroll
            for (int h = 0; h < NPR; ++h) {
                const unsigned long long c2 = pk2(cur[2 * h], cur[2 * h + 1]);
                unsigned long long s2 = pk2(nw[2 * h], nw[2 * h + 1]);
                s2 = fma2(lxm2[h], sub2(pk2(xm[2 * h], xm[2 * h + 1]), c2), s2);
                s2 = fma2(lxp2[h], sub2(pk2(xp[2 * h], xp[2 * h + 1]), c2), s2);
                s2 = fma2(lym2[h], sub2(pk2(ym[2 * h], ym[2 * h + 1]), c2), s2);
                s2 = fma2(lyp2[h], sub2(pk2(yp[2 * h], yp[2 * h + 1]), c2), s2);
                upk2(s2, nw[2 * h], nw[2 * h + 1]);
            }
            {
                const float c1 = cur[L - 1];
                float s1 = nw[L - 1];
                s1 = fmaf(lxm1, xm[L - 1] - c1, s1);
                s1 = fmaf(lxp1, xp[L - 1] - c1, s1);
                s1 = fmaf(lym1, ym[L - 1] - c1, s1);
                s1 = fmaf(lyp1, yp[L - 1] - c1, s1);
                nw[L - 1] = s1;
            }
            if constexpr (R > 5) zfaces();
        };

        // n_fd Jacobi substeps; lateral faces summed −x,+x,−y,+y, the z faces before (R ≤ 5) or
        // after them (see flux).
        // Direct: all n_fd substeps.  Chebyshev: the first cheb_pre substeps (the peaked start,
        // whose large entries would otherwise feed the recurrence's rounding), then the recurrence.
        // Windows touching the far-field reservoir (N2) keep the literal substeps: their kernel
        // keeps only the mass M_s that did not leak, and the recurrence's rounding is on the
        // scale of the source, not of M_s (measured: M_s relative error 7e-5 vs 5e-6).
        // act: run the step on this thread.  For R ≥ 6 every thread runs it (threads without a
        // column, t ≥ L², compute zeros: face numbers and neighbour offsets 0, own smem slot
        // only), which removes the divergent branches; measured faster there (cfg5 R8 967 →
        // 908 ms) and slower at R5 (140 → 155 ms), so R ≤ 5 keep the guard.
        const bool act = R >= 6 || col;
        const bool iso = !F64 && isolated_source(ph, ftab, KC, L, LL);  // kernel δ_s: no pass
        const bool cheb = !iso && a.cheb_m && (!open || a.cheb_open);
        const int n_direct = iso ? 0 : cheb ? a.cheb_pre : a.n_fd;
        for (int k = 0; k < n_direct; ++k) {
            float* b = buf + (k & 1) * (NT * Lp);
            if (act) store_col(b, c);
            __syncthreads();
            if (act) {
                float nw[Lp];
#pragma unroll
                for (int z = 0; z < L; ++z) nw[z] = c[z];
                flux(b, c, nw);
#pragma unroll
                for (int z = 0; z < L; ++z) c[z] = (rmask >> z) & 1u ? 0.f : nw[z];
            }
        }
        if (cheb) {
            // Chebyshev evaluation of the rest, A^{n_fd − pre} v with v = A^{pre} δ_s (DESIGN.md
            // §7, reading A30): x^n' = Σ_k c_k T_k(y) on the spectrum [a, 1] of A,
            // y = (2x − 1 − a)/(1 − a), all c_k ≥ 0 with Σ c_k = 1, truncated at degree m where the
            // tail Σ_{k>m} c_k ≤ 1e-10 (so ‖p_m(A)v − A^n' v‖₂ ≤ 1e-10 ‖v‖₂).  Three-term recurrence
            // t_{k+1} = 2Â t_k − t_{k−1}, t_0 = v, t_1 = Â v; p = Σ c_k t_k.  Each step is one stencil
            // pass of the direct substep's cost (+2 FMA): pre + m ≈ 8 + 157 passes instead of
            // n_fd = 1000 at Table 1's λ = 0.1.
            // State: c[] = t (A), pv[] = t_{k−1} (B) overwritten in place by t_{k+1}, acc[] = p.
            faces(ftab + 32, true);
            const float* cc = reinterpret_cast<const float*>(smem_raw + S::cheb_off);
            float pv[Lp], acc[L];
#pragma unroll
            for (int z = 0; z < Lp; ++z) pv[z] = 0.f;
#pragma unroll
            for (int z = 0; z < L; ++z) acc[z] = c[z] * cc[0];
            // prv ← κ·Â·cur − prv, κ = 2 (κ = 1, prv = 0 on the first step: 2Âδ·½, exact)
            auto step = [&](float (&cur)[Lp], float (&prv)[Lp], const int k, const bool first) {
                float* b = buf + ((k + n_direct) & 1) * (NT * Lp);
                if (act) store_col(b, cur);
                __syncthreads();
                const float ck = cc[k + 1];
                if (act) {
                    // nw = D∘t − t_{k−1}, then the z faces (registers: they run while the
                    // neighbours' loads are in flight), then −x, +x, −y, +y: 8 lane-FMAs per
                    // cell-pass with p's update (the flux form took 13)
                    float xm[L], xp[L], ym[L], yp[L];
                    load_col(b, t + axm, xm);
                    load_col(b, t + axp, xp);
                    load_col(b, t + oym, ym);
                    load_col(b, t + oyp, yp);
                    float nw[Lp];
#pragma unroll
                    for (int h = 0; h < NPR; ++h) {
                        const unsigned long long s2 =
                            fma2(dg2[h], pk2(cur[2 * h], cur[2 * h + 1]), pk2(-prv[2 * h], -prv[2 * h + 1]));
                        upk2(s2, nw[2 * h], nw[2 * h + 1]);
                    }
                    nw[L - 1] = fmaf(dg1, cur[L - 1], -prv[L - 1]);
#pragma unroll
                    for (int z = 0; z < L; ++z) {
                        float v = nw[z];
                        if (z > 0) v = fmaf(fz[z - 1], cur[z - 1], v);
                        if (z < L - 1) v = fmaf(fz[z], cur[z + 1], v);
                        nw[z] = v;
                    }
#pragma unroll
                    for (int h = 0; h < NPR; ++h) {
                        unsigned long long s2 = pk2(nw[2 * h], nw[2 * h + 1]);
                        s2 = fma2(lxm2[h], pk2(xm[2 * h], xm[2 * h + 1]), s2);
                        s2 = fma2(lxp2[h], pk2(xp[2 * h], xp[2 * h + 1]), s2);
                        s2 = fma2(lym2[h], pk2(ym[2 * h], ym[2 * h + 1]), s2);
                        s2 = fma2(lyp2[h], pk2(yp[2 * h], yp[2 * h + 1]), s2);
                        if (first) s2 = fma2(s2, pk2(0.5f, 0.5f), pk2(-0.f, -0.f));  // exact halving
                        upk2(s2, prv[2 * h], prv[2 * h + 1]);
                        if (rmask) {  // reservoir cells (open windows, A30): Dirichlet 0 in every t_k
                            if ((rmask >> (2 * h)) & 1u) prv[2 * h] = 0.f;
                            if ((rmask >> (2 * h + 1)) & 1u) prv[2 * h + 1] = 0.f;
                            s2 = pk2(prv[2 * h], prv[2 * h + 1]);
                        }
                        const unsigned long long a2 = fma2(pk2(ck, ck), s2, pk2(acc[2 * h], acc[2 * h + 1]));
                        upk2(a2, acc[2 * h], acc[2 * h + 1]);
                    }
                    {
                        float v = nw[L - 1];
                        v = fmaf(lxm1, xm[L - 1], v);
                        v = fmaf(lxp1, xp[L - 1], v);
                        v = fmaf(lym1, ym[L - 1], v);
                        v = fmaf(lyp1, yp[L - 1], v);
                        if (first) v *= 0.5f;
                        if ((rmask >> (L - 1)) & 1u) v = 0.f;
                        prv[L - 1] = v;
                        acc[L - 1] = fmaf(ck, v, acc[L - 1]);
                    }
                }
            };
            const int m = a.cheb_m;
            step(c, pv, 0, true);  // pv = t_1
            for (int k = 1; k < m; k += 2) {
                step(pv, c, k, false);                  // c  = t_{k+1}
                if (k + 1 < m) step(c, pv, k + 1, false);  // pv = t_{k+2}
            }
            // A^n δ ≥ 0 (maximum principle, λ_max ≤ 1/6): clamping the truncation / rounding
            // noise of tiny entries at 0 can only move them closer to it
#pragma unroll
            for (int z = 0; z < Lp; ++z) c[z] = z < L ? fmaxf(acc[z < L ? z : 0], 0.f) : 0.f;
            // an open window keeps its own mass (no renormalisation): divide out p(1) = Σ fp32(c_k)
            // so a conserved mode (a pore the reservoir cannot reach) keeps it exactly (A30)
            if (open)
#pragma unroll
                for (int z = 0; z < L; ++z) c[z] *= a.cheb_scale;
        }
        }  // fp32 substeps

        // ---- epilogue (a4) ----
        double s = 0.0;
        if (col) {
#pragma unroll
            for (int z = 0; z < L; ++z) s += (double)c[z];
        }
        const double S_ = block_sum_f64<S::NW>(s, red);
        // closed window: renormalise to mass 1 (fp32 FD drift); open window (N2): the kernel
        // keeps its own mass M = S, the rest went to the reservoir
        const double inv = (open || F64) ? 1.0 : 1.0 / S_;
        const double M = open ? S_ : 1.0;
        double qsum = 0.0;
        float centre_q = 0.f;
        if (col) {
            const int ox = cx - R, oy = cy - R;
            // gather target and slot of this weight: x = s + o in slot o, or with the symmetric
            // rule (reading A24, exact regime P = Pᵀ) the source's own target x = s in slot −o
            const int gx = a.symmetric ? sx : sx + ox, gy = a.symmetric ? sy : sy + oy;
#pragma unroll
            for (int z = 0; z < L; ++z) {
                const int o = z * LL + t;
                const int oz = z - R, gz = a.symmetric ? sz : sz + oz;
                const bool active = ph[o] <= 1;
                const float wf = (float)((double)c[z] * inv);
                float qd;
                unsigned short bits = 0;
                if (a.fmt == 1) {
                    const __half h = __float2half_rn(wf);
                    bits = __half_as_ushort(h);
                    qd = __half2float(h);
                } else if (a.fmt == 2) {
                    const __nv_bfloat16 h = __float2bfloat16_rn(wf);
                    bits = __bfloat16_as_ushort(h);
                    qd = __bfloat162float(h);
                } else {
                    qd = wf;
                }
                if (a.class_w) {  // class-major store (dedup path): every slot written
                    const size_t ci = (size_t)it * LLL + o;
                    const bool keep = active && o != KC;
                    if (a.fmt == 0) reinterpret_cast<float*>(a.class_w)[ci] = keep ? wf : 0.f;
                    else reinterpret_cast<unsigned short*>(a.class_w)[ci] = keep ? bits : (unsigned short)0;
                }
                if (o == KC) {
                    centre_q = qd;
                    continue;
                }
                if (!active) continue;
                qsum += (double)qd;
                if (a.class_w || gz < a.z0 || gz >= a.z1) continue;
                const int zl = gz - a.z0;
                const int q = gy * a.nxq + (gx >> 3);
                const size_t tile = (size_t)zl * a.tpp + q / a.tile;
                const int e = q % a.tile, j = gx & 7;
                const int sl = a.symmetric ? slot_of(-ox, -oy, -oz, R) : slot_of(ox, oy, oz, R);
                const size_t idx = ((tile * (size_t)(a.K - 1) + sl) * a.tile + e) * 8 + j;
                if (a.fmt == 0) reinterpret_cast<float*>(a.Wt)[idx] = wf;
                else reinterpret_cast<unsigned short*>(a.Wt)[idx] = bits;
            }
        }
        const double off = block_sum_f64<S::NW>(qsum, red);
        if (t == R * L + R && a.class_w) {
            a.class_diag[it] = a.mass_fix ? fp32_pair(M - off) : make_float2(centre_q, 0.f);
            if (a.class_mass) a.class_mass[it] = M;
        } else if (t == R * L + R && sz >= a.z0 && sz < a.z1) {
            const float2 d = a.mass_fix ? fp32_pair(M - off) : make_float2(centre_q, 0.f);
            const int zl = sz - a.z0;
            const int q = sy * a.nxq + (sx >> 3);
            const size_t tile = (size_t)zl * a.tpp + q / a.tile;
            a.diag[(tile * a.tile + q % a.tile) * 8 + (sx & 7)] = d;
        }
        // (the block_sum barriers separate this source's smem use from the next one's)
    }
}

template <int R, bool F64>
static cudaError_t launch_kgen_r(const KgenArgs& a, cudaStream_t s)
{
    using S = KgenShape<R, F64>;
    const long nsrc = a.src_list ? a.n_list : (long)a.nx * a.ny * (a.sz1 - a.sz0);
    if (nsrc <= 0) return cudaSuccess;
    const size_t smem = S::smem_bytes + (F64 || !a.cheb_m ? 0 : ((size_t)(a.cheb_m + 1) * 4 + 15) / 16 * 16);
    cudaError_t e = cudaFuncSetAttribute(kgen_kernel<R, F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kgen_kernel<R, F64>, S::NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    long grid = (long)sms * per_sm;
    if (grid > nsrc) grid = nsrc;
    kgen_kernel<R, F64><<<(unsigned)grid, S::NT, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_kgen(const KgenArgs& a, int R, cudaStream_t s)
{
    // R = 5 (cfg3/cfg4) and R = 8 (cfg5): two columns per thread over balanced z segments
    // (kgen_bal.cu) unless FDIRW_F_KGEN_COLUMNS (A/B)
    if (!a.columns && (R == 5 || R == 8) && !a.fp64 && !a.symmetric) return launch_kgen_bal(a, R, s);
    if (a.fp64) {
        switch (R) {
            case 1: return launch_kgen_r<1, true>(a, s);
            case 2: return launch_kgen_r<2, true>(a, s);
            case 3: return launch_kgen_r<3, true>(a, s);
            case 4: return launch_kgen_r<4, true>(a, s);
            case 5: return launch_kgen_r<5, true>(a, s);
            case 6: return launch_kgen_r<6, true>(a, s);
            case 7: return launch_kgen_r<7, true>(a, s);
            case 8: return launch_kgen_r<8, true>(a, s);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (R) {
        case 1: return launch_kgen_r<1, false>(a, s);
        case 2: return launch_kgen_r<2, false>(a, s);
        case 3: return launch_kgen_r<3, false>(a, s);
        case 4: return launch_kgen_r<4, false>(a, s);
        case 5: return launch_kgen_r<5, false>(a, s);
        case 6: return launch_kgen_r<6, false>(a, s);
        case 7: return launch_kgen_r<7, false>(a, s);
        case 8: return launch_kgen_r<8, false>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fdirw
