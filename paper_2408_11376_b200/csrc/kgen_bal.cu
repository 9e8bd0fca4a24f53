// kgen_bal.cu — a3 + a4 for R = 5 and 8 with TWO window columns per thread over balanced z
// segments (DESIGN.md §7 "Round 2, continued").  Same method and per-cell arithmetic as kgen.cu's
// column kernel (FDIRW_F_KGEN_COLUMNS selects that one for A/B).
//
// Why pairs: the column kernel moves 20 B of shared memory per cell-pass (a thread owns one
// z-column; its 4 lateral neighbours come from smem).  A thread owning the linear columns 2p and
// 2p + 1 reads the x face between them from registers, so it loads 3 neighbour ranges per
// column; splitting z into segments keeps a thread at ~11 cells and 128 registers (R5: 4 CTAs
// × 4 warps per SM; R8: 15 warps per window instead of the column kernel's 10).
// Why balanced: with both columns in the same 6-cell segments (the first version, in git
// history) the lower R5 thread owned 12 cells and 50 wavefronts per warp-pass, the upper 10 and
// 42, and every pass waited for the heavier one (cfg3 114 ms).  Here column A (2p) is split at
// [6s, 6s + 6) and column B (2p + 1) at [6s − 1, 6s + 5) (the first [0, 5)): at L = 11 each thread
// owns 11 cells and moves 46 / 47 wavefronts (cfg3 104 ms); at L = 17 the middle thread keeps 12
// (53 wavefronts; cfg5 652 vs 655 ms).
//
// Shared layout (per pass buffer): every column side stores its cells in the same z items —
// for each segment s: Q_s = cells 6s … 6s + 3 (float4), S4_s = cell 6s + 4, S5_s = cell 6s + 5
// (scalar, absent for the last segment) — each item an array over the pairs [pair + PAD].  A
// thread's own cells and every neighbour range it reads are whole items, in the same grouping,
// so the 16-byte loads land in the register pairs the FFMA2s use.  One extra scalar array X_s
// (s ≥ 1) duplicates cell 6s of column A, the cell below it needs as its z neighbour (it sits
// inside the quad Q_s otherwise).  Each warp access is a run of consecutive 4 / 16 B words.
//
// Thread (pair p, segment s) loads, per pass: the B-side items over its A cells for the −x, −y, +y
// neighbours of A (pairs p − 1, p − R − 1, p + R), the A-side items over its B cells for the +x,
// −y, +y neighbours of B (pairs p + 1, p − R, p + R + 1), and the boundary cells of the
// neighbouring segments (own pair); A's +x and B's −x neighbours are the other column's registers.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <type_traits>

#include "fdirw_internal.h"
#include "kgen_common.cuh"
#include "layout.cuh"

namespace fdirw {

namespace {

template <int R>
struct BalShape {
    static constexpr int L = 2 * R + 1, LL = L * L, LLL = LL * L;
    static constexpr int NSEG = (L + 1) / 6;
    static_assert(NSEG * 6 == L + 1, "L = 6·NSEG − 1");
    static constexpr int NP = (LL + 1) / 2;
    static constexpr int NPW = (NP + 31) / 32 * 32;
    static constexpr int NT = NSEG * NPW;
    static constexpr int NW = NT / 32;
    static constexpr int PAD = (R + 2 + 3) / 4 * 4;
    static constexpr int NPP = (NPW + 2 * PAD + 3) / 4 * 4;
    // item float offsets within a pass buffer: side-major, then segment, then Q (4·NPP), S4, S5
    static constexpr int off(int side, int s, int kind) { return ((side * NSEG + s) * 6 + kind) * NPP; }
    static constexpr int KQ = 0, KS4 = 4, KS5 = 5;
    static constexpr int offX(int s) { return (12 * NSEG + s) * NPP; }
    static constexpr int BUFF = 13 * NSEG * NPP;
    static constexpr size_t buf_bytes = 2 * (size_t)BUFF * 4;
    static constexpr size_t tab_off = buf_bytes + ((LLL + 15) / 16) * 16 + NW * 8 + 16;
    static constexpr size_t smem_bytes = tab_off + 64 * 4;
    static constexpr size_t cheb_off = smem_bytes;
    static constexpr int kMinBlocks = 65536 / (NT * 128) > 0 ? 65536 / (NT * 128) : 1;
};

// per segment: column A cells [zA, zA + NA), column B cells [zB, zB + NB); packed cell pairs
template <int R, int SEG>
struct BalSeg {
    using S = BalShape<R>;
    static constexpr bool last = SEG == S::NSEG - 1;
    static constexpr int zA = 6 * SEG, NA = last ? S::L - 6 * SEG : 6;
    static constexpr int zB = SEG ? 6 * SEG - 1 : 0, NB = SEG ? 6 : 5;
    static constexpr int offB = zA - zB;  // B's local index of the z at A's local 0
    static constexpr int N(int sd) { return sd ? NB : NA; }
    static constexpr int Z0(int sd) { return sd ? zB : zA; }
    // cell pairs (local indices) matching the item grouping; a 5-cell column has a single cell
    static constexpr int NPR(int sd) { return N(sd) == 6 ? 3 : 2; }
    static constexpr int PA(int sd, int h) { return (sd == 1 && SEG > 0) ? (h == 2 ? 0 : 2 * h + 1) : 2 * h; }
    static constexpr int PB(int sd, int h) { return (sd == 1 && SEG > 0) ? (h == 2 ? 5 : 2 * h + 2) : 2 * h + 1; }
    static constexpr int SGL(int sd) { return N(sd) == 6 ? -1 : 4; }
};

}  // namespace

// CO: the build lets windows touching the N2 reservoir take the recurrence (a.cheb_open); a
// separate instantiation, so closed-domain builds keep the code (and registers) without the
// reservoir masks
template <int R, int SEG, bool CLEAN, bool CO>
__device__ __forceinline__ void bal_body(const KgenArgs& a)
{
    using S = BalShape<R>;
    using G = BalSeg<R, SEG>;
    constexpr int L = S::L, LL = S::LL, LLL = S::LLL, NPP = S::NPP;
    constexpr int KC = LLL / 2;
    constexpr int NA = G::NA, NB = G::NB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* buf = reinterpret_cast<float*>(smem_raw);
    unsigned char* ph = smem_raw + S::buf_bytes;
    double* red = reinterpret_cast<double*>(smem_raw + S::buf_bytes + ((LLL + 15) / 16) * 16);

    const int t = threadIdx.x;
    const int p = t - SEG * S::NPW;
    const bool real = p < S::NP;
    const int col[2] = {2 * p, 2 * p + 1};
    const bool has[2] = {real, real && 2 * p + 1 < LL};
    const int pp = p + S::PAD;
    const int nx = a.nx, ny = a.ny, nz = a.nz;
    const long nsrc = a.src_list ? a.n_list : (long)nx * ny * (a.sz1 - a.sz0);

    for (int i = t; i < 2 * S::BUFF; i += S::NT) buf[i] = 0.f;
    float* ftab = reinterpret_cast<float*>(smem_raw + S::tab_off);
    build_face_tables(ftab, a.lam_ff, a.lam_fs, a.lam_ss, a.mu2_ff, a.mu2_fs, a.mu2_ss);
    if (a.cheb_m) {
        float* cc = reinterpret_cast<float*>(smem_raw + S::cheb_off);
        for (int i = t; i <= a.cheb_m; i += S::NT) cc[i] = a.cheb_c[i];
    }

    auto sc = [](float* b, int side, int s, int kind) { return b + S::off(side, s, kind); };
    auto qd = [](float* b, int side, int s) { return reinterpret_cast<float4*>(b + S::off(side, s, S::KQ)); };
    // own cells → the buffer
    auto store_own = [&](float* b, const float (&cA)[6], const float (&cB)[6]) {
        qd(b, 0, SEG)[pp] = make_float4(cA[0], cA[1], cA[2], cA[3]);
        sc(b, 0, SEG, S::KS4)[pp] = cA[4];
        if constexpr (NA == 6) sc(b, 0, SEG, S::KS5)[pp] = cA[5];
        if constexpr (SEG > 0) (b + S::offX(SEG))[pp] = cA[0];
        if constexpr (SEG > 0) {
            sc(b, 1, SEG - 1, S::KS5)[pp] = cB[0];
            qd(b, 1, SEG)[pp] = make_float4(cB[1], cB[2], cB[3], cB[4]);
            sc(b, 1, SEG, S::KS4)[pp] = cB[5];
        } else {
            qd(b, 1, 0)[pp] = make_float4(cB[0], cB[1], cB[2], cB[3]);
            sc(b, 1, 0, S::KS4)[pp] = cB[4];
        }
    };
    // B-side cells over A's z range of pair slot q (A's −x / ±y neighbours)
    auto load_Brange = [&](float* b, int q, float (&v)[6]) {
        const float4 w = qd(b, 1, SEG)[q];
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
        v[4] = sc(b, 1, SEG, S::KS4)[q];
        v[5] = NA == 6 ? sc(b, 1, SEG, S::KS5)[q] : 0.f;
    };
    // A-side cells over B's z range of pair slot q (B's +x / ±y neighbours)
    auto load_Arange = [&](float* b, int q, float (&v)[6]) {
        if constexpr (SEG > 0) {
            v[0] = sc(b, 0, SEG - 1, S::KS5)[q];
            const float4 w = qd(b, 0, SEG)[q];
            v[1] = w.x; v[2] = w.y; v[3] = w.z; v[4] = w.w;
            v[5] = sc(b, 0, SEG, S::KS4)[q];
        } else {
            const float4 w = qd(b, 0, 0)[q];
            v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
            v[4] = sc(b, 0, 0, S::KS4)[q];
            v[5] = 0.f;
        }
    };
    // neighbouring segments' boundary cells of the own pair: A below (6s − 1), A above (6s + 6),
    // B below (6s − 2), B above (6s + 5); absent ones read a finite own value nobody uses
    auto load_halo = [&](float* b, float& hAdn, float& hAup, float& hBdn, float& hBup) {
        hAdn = SEG > 0 ? sc(b, 0, SEG > 0 ? SEG - 1 : 0, S::KS5)[pp] : 0.f;
        hAup = !G::last ? (b + S::offX(G::last ? SEG : SEG + 1))[pp] : 0.f;
        hBdn = SEG > 0 ? sc(b, 1, SEG > 0 ? SEG - 1 : 0, S::KS4)[pp] : 0.f;
        hBup = !G::last ? sc(b, 1, SEG, S::KS5)[pp] : 0.f;
    };
    const int qxmA = pp - 1, qymA = pp - (R + 1), qypA = pp + R;
    const int qxpB = pp + 1, qymB = pp - R, qypB = pp + R + 1;

    for (long it = blockIdx.x; it < nsrc; it += gridDim.x) {
        const long src = a.src_list ? (long)a.src_list[it] : it;
        const int sx = (int)(src % nx);
        const int sy = (int)((src / nx) % ny);
        const int sz = a.sz0 + (int)(src / ((long)nx * ny));

        cta_sync_any_pc<S::NT, CLEAN>();  // (each segment's warps run their own instantiation:
                                          // the CTA barriers of kgen_common.cuh)
        int far_here = 0;
        for (int i = t; i < LLL; i += S::NT) {
            const int gx = sx + i % L - R, gy = sy + (i / L) % L - R, gz = sz + i / LL - R;
            const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz;
            unsigned char v = in ? a.mask[((size_t)(gz - a.mz0) * ny + gy) * nx + gx] : (unsigned char)2;
            if (in && v == 2) v = 3;
            far_here |= v == 3;
            ph[i] = v;
        }
        const bool open = cta_or_any_pc<S::NT, CLEAN>(far_here != 0);
        if (ph[KC] == 3) continue;

        // ---- face numbers: fl[sd][f][h] packed pairs, fl1[sd][f] the single cell; fz[sd][j] the
        // face between the column's local cells j − 1 and j (j = 0..N, halos at both ends) ----
        unsigned long long fl[2][4][3], dg2[2][3];
        float fl1[2][4], dg1[2], fz[2][7];
        unsigned rmask[2] = {0u, 0u};
        auto faces = [&](const float* T, const bool row_form) {
            auto side = [&](auto sdc) {
                constexpr int sd = decltype(sdc)::value;
                constexpr int N = G::N(sd), Z0 = G::Z0(sd);
                const int c = col[sd], cx = c % L, cy = c / L;
                float v[4][6], d[6];
#pragma unroll
                for (int j = 0; j <= N; ++j) {
                    const int z = Z0 + j;
                    float f = 0.f;
                    if (has[sd] && z >= 1 && z < L) f = T[16 + ((ph[(z - 1) * LL + c] << 2) | ph[z * LL + c])];
                    fz[sd][j] = f;
                }
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    const int z = Z0 + i, o = z * LL + c;
                    const bool cell = has[sd];
                    const unsigned pc = cell ? ph[o] : 2u;
                    v[0][i] = (cell && cx > 0) ? T[(pc << 2) | ph[o - 1]] : 0.f;
                    v[1][i] = (cell && cx < L - 1) ? T[(pc << 2) | ph[o + 1]] : 0.f;
                    v[2][i] = (cell && cy > 0) ? T[(pc << 2) | ph[o - L]] : 0.f;
                    v[3][i] = (cell && cy < L - 1) ? T[(pc << 2) | ph[o + L]] : 0.f;
                    if (cell && pc == 3u) rmask[sd] |= 1u << i;
                    if (row_form) {
                        double f = (double)v[0][i] + (double)v[1][i] + (double)v[2][i] + (double)v[3][i];
                        if (z > 0) f += (double)fz[sd][i];
                        if (z < L - 1) f += (double)fz[sd][i + 1];
                        d[i] = cell ? (float)(2.0 - f) : 0.f;
                    }
                }
#pragma unroll
                for (int h = 0; h < G::NPR(sd); ++h) {
#pragma unroll
                    for (int f = 0; f < 4; ++f) fl[sd][f][h] = pk2(v[f][G::PA(sd, h)], v[f][G::PB(sd, h)]);
                    if (row_form) dg2[sd][h] = pk2(d[G::PA(sd, h)], d[G::PB(sd, h)]);
                }
                if constexpr (G::SGL(sd) >= 0) {
#pragma unroll
                    for (int f = 0; f < 4; ++f) fl1[sd][f] = v[f][G::SGL(sd)];
                    if (row_form) dg1[sd] = d[G::SGL(sd)];
                }
            };
            side(std::integral_constant<int, 0>{});
            side(std::integral_constant<int, 1>{});
        };
        faces(ftab, false);

        float c[2][6];
#pragma unroll
        for (int sd = 0; sd < 2; ++sd)
#pragma unroll
            for (int i = 0; i < 6; ++i)
                c[sd][i] = (real && sd == 0 && col[0] == R * L + R && G::zA + i == R && i < NA) ? 1.f : 0.f;

        // the 4 lateral neighbour values of every own cell: nb[sd][f][i]
        auto gather = [&](float* b, const float (&cur)[2][6], float (&nb)[2][4][6], float (&h)[4]) {
            load_Brange(b, qxmA, nb[0][0]);
            load_Brange(b, qymA, nb[0][2]);
            load_Brange(b, qypA, nb[0][3]);
            load_Arange(b, qxpB, nb[1][1]);
            load_Arange(b, qymB, nb[1][2]);
            load_Arange(b, qypB, nb[1][3]);
            load_halo(b, h[0], h[1], h[2], h[3]);
#pragma unroll
            for (int i = 0; i < NA; ++i) nb[0][1][i] = i + G::offB < NB ? cur[1][i + G::offB] : h[3];
#pragma unroll
            for (int i = 0; i < NB; ++i) nb[1][0][i] = i - G::offB >= 0 ? cur[0][i - G::offB] : h[0];
        };
        // z neighbour values of local cell i (below / above) and whether the term exists
        auto zdn = [&](const float (&cur)[2][6], const float (&h)[4], int sd, int i) {
            return i > 0 ? cur[sd][i > 0 ? i - 1 : 0] : (sd ? h[2] : h[0]);
        };
        auto zup = [&](const float (&cur)[2][6], const float (&h)[4], int sd, int i) {
            return i < G::N(sd) - 1 ? cur[sd][i < 5 ? i + 1 : 5] : (sd ? h[3] : h[1]);
        };
        auto below = [](int sd, int i) { return G::Z0(sd) + i > 0; };
        auto above = [](int sd, int i) { return G::Z0(sd) + i < L - 1; };

        const bool act = real;
        const bool iso = isolated_source(ph, ftab, KC, L, LL);  // kernel δ_s: no pass
        const bool cheb = !iso && a.cheb_m && (!open || (CO && a.cheb_open));
        const int n_direct = iso ? 0 : cheb ? a.cheb_pre : a.n_fd;
        unsigned ps = 0;
        // ---- literal substeps, flux form in the column kernel's order (z faces first for R ≤ 5) ----
        for (int k = 0; k < n_direct; ++k, ++ps) {
            float* b = buf + (ps & 1u) * S::BUFF;
            if (act) store_own(b, c[0], c[1]);
            cta_sync_any_pc<S::NT, CLEAN>();
            if (act) {
                float nb[2][4][6], h[4];
                gather(b, c, nb, h);
                float nw[2][6];
                auto side = [&](auto sdc) {
                    constexpr int sd = decltype(sdc)::value;
                    constexpr int N = G::N(sd);
                    auto zterms = [&]() {
#pragma unroll
                        for (int i = 0; i < N; ++i) {
                            float v = nw[sd][i];
                            if (below(sd, i)) v = fmaf(fz[sd][i], -(c[sd][i] - zdn(c, h, sd, i)), v);
                            if (above(sd, i)) v = fmaf(fz[sd][i + 1], zup(c, h, sd, i) - c[sd][i], v);
                            nw[sd][i] = v;
                        }
                    };
#pragma unroll
                    for (int i = 0; i < N; ++i) nw[sd][i] = c[sd][i];
                    if constexpr (R <= 5) zterms();
#pragma unroll
                    for (int hh = 0; hh < G::NPR(sd); ++hh) {
                        const int i0 = G::PA(sd, hh), i1 = G::PB(sd, hh);
                        const unsigned long long c2 = pk2(c[sd][i0], c[sd][i1]);
                        unsigned long long s2 = pk2(nw[sd][i0], nw[sd][i1]);
#pragma unroll
                        for (int f = 0; f < 4; ++f)
                            s2 = fma2(fl[sd][f][hh], sub2(pk2(nb[sd][f][i0], nb[sd][f][i1]), c2), s2);
                        upk2(s2, nw[sd][i0], nw[sd][i1]);
                    }
                    if constexpr (G::SGL(sd) >= 0) {
                        constexpr int i = G::SGL(sd);
                        float v = nw[sd][i];
#pragma unroll
                        for (int f = 0; f < 4; ++f) v = fmaf(fl1[sd][f], nb[sd][f][i] - c[sd][i], v);
                        nw[sd][i] = v;
                    }
                    if constexpr (R > 5) zterms();
                };
                side(std::integral_constant<int, 0>{});
                side(std::integral_constant<int, 1>{});
#pragma unroll
                for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                    for (int i = 0; i < G::N(sd); ++i) c[sd][i] = (rmask[sd] >> i) & 1u ? 0.f : nw[sd][i];
            }
        }
        if (cheb) {
            // ---- Chebyshev passes, row form (reading A30) ----
            faces(ftab + 32, true);
            const float* cc = reinterpret_cast<const float*>(smem_raw + S::cheb_off);
            float pv[2][6], acc[2][6];
#pragma unroll
            for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    pv[sd][i] = 0.f;
                    acc[sd][i] = c[sd][i] * cc[0];
                }
            auto step = [&](auto openc, float (&cur)[2][6], float (&prv)[2][6], const int k, const bool first) {
                constexpr bool OPEN = decltype(openc)::value;
                float* b = buf + (ps & 1u) * S::BUFF;
                if (act) store_own(b, cur[0], cur[1]);
                cta_sync_any_pc<S::NT, CLEAN>();
                ++ps;
                const float ck = cc[k + 1];
                if (act) {
                    float nb[2][4][6], h[4];
                    gather(b, cur, nb, h);
                    auto side = [&](auto sdc) {
                        constexpr int sd = decltype(sdc)::value;
                        constexpr int N = G::N(sd);
                        float nw[6];
#pragma unroll
                        for (int hh = 0; hh < G::NPR(sd); ++hh) {
                            const int i0 = G::PA(sd, hh), i1 = G::PB(sd, hh);
                            const unsigned long long s2 = fma2(dg2[sd][hh], pk2(cur[sd][i0], cur[sd][i1]),
                                                               pk2(-prv[sd][i0], -prv[sd][i1]));
                            upk2(s2, nw[i0], nw[i1]);
                        }
                        if constexpr (G::SGL(sd) >= 0) {
                            constexpr int i = G::SGL(sd);
                            nw[i] = fmaf(dg1[sd], cur[sd][i], -prv[sd][i]);
                        }
#pragma unroll
                        for (int i = 0; i < N; ++i) {
                            float v = nw[i];
                            if (below(sd, i)) v = fmaf(fz[sd][i], zdn(cur, h, sd, i), v);
                            if (above(sd, i)) v = fmaf(fz[sd][i + 1], zup(cur, h, sd, i), v);
                            nw[i] = v;
                        }
#pragma unroll
                        for (int hh = 0; hh < G::NPR(sd); ++hh) {
                            const int i0 = G::PA(sd, hh), i1 = G::PB(sd, hh);
                            unsigned long long s2 = pk2(nw[i0], nw[i1]);
#pragma unroll
                            for (int f = 0; f < 4; ++f) s2 = fma2(fl[sd][f][hh], pk2(nb[sd][f][i0], nb[sd][f][i1]), s2);
                            if (first) s2 = fma2(s2, pk2(0.5f, 0.5f), pk2(-0.f, -0.f));
                            upk2(s2, prv[sd][i0], prv[sd][i1]);
                            if constexpr (OPEN) {  // reservoir cells (open windows, A30): Dirichlet 0 in every t_k
                                if ((rmask[sd] >> i0) & 1u) prv[sd][i0] = 0.f;
                                if ((rmask[sd] >> i1) & 1u) prv[sd][i1] = 0.f;
                                s2 = pk2(prv[sd][i0], prv[sd][i1]);
                            }
                            const unsigned long long a2 = fma2(pk2(ck, ck), s2, pk2(acc[sd][i0], acc[sd][i1]));
                            upk2(a2, acc[sd][i0], acc[sd][i1]);
                        }
                        if constexpr (G::SGL(sd) >= 0) {
                            constexpr int i = G::SGL(sd);
                            float v = nw[i];
#pragma unroll
                            for (int f = 0; f < 4; ++f) v = fmaf(fl1[sd][f], nb[sd][f][i], v);
                            if (first) v *= 0.5f;
                            if constexpr (OPEN)
                                if ((rmask[sd] >> i) & 1u) v = 0.f;
                            prv[sd][i] = v;
                            acc[sd][i] = fmaf(ck, v, acc[sd][i]);
                        }
                    };
                    side(std::integral_constant<int, 0>{});
                    side(std::integral_constant<int, 1>{});
                }
            };
            const int m = a.cheb_m;
            // (open windows, which take the recurrence only with reduced-precision storage, run
            // their own instantiation with the reservoir masks: closed windows keep the unmasked
            // code and its registers)
            auto recur = [&](auto openc) {
                step(openc, c, pv, 0, true);
                for (int k = 1; k < m; k += 2) {
                    step(openc, pv, c, k, false);
                    if (k + 1 < m) step(openc, c, pv, k + 1, false);
                }
            };
            if (!open) recur(std::integral_constant<bool, false>{});
            else if constexpr (CO) recur(std::integral_constant<bool, true>{});
#pragma unroll
            for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                for (int i = 0; i < 6; ++i) c[sd][i] = fmaxf(acc[sd][i], 0.f);
            // an open window keeps its own mass (no renormalisation): divide out p(1) = Σ fp32(c_k)
            // so a conserved mode (a pore the reservoir cannot reach) keeps it exactly (A30)
            if (open)
#pragma unroll
                for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                    for (int i = 0; i < 6; ++i) c[sd][i] *= a.cheb_scale;
        }

        // ---- epilogue (a4): as kgen.cu's, per owned cell ----
        double s = 0.0;
#pragma unroll
        for (int sd = 0; sd < 2; ++sd)
#pragma unroll
            for (int i = 0; i < G::N(sd); ++i)
                if (has[sd]) s += (double)c[sd][i];
        const double S_ = block_sum_f64<S::NW, true, CLEAN>(s, red);
        const double inv = open ? 1.0 : 1.0 / S_;
        const double M = open ? S_ : 1.0;
        double qsum = 0.0;
        float centre_q = 0.f;
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            if (!has[sd]) continue;
            const int cx = col[sd] % L, cy = col[sd] / L;
            const int ox = cx - R, oy = cy - R;
            const int gx = sx + ox, gy = sy + oy;
#pragma unroll
            for (int i = 0; i < G::N(sd); ++i) {
                const int z = G::Z0(sd) + i;
                const int o = z * LL + col[sd];
                const int oz = z - R, gz = sz + oz;
                const bool active = ph[o] <= 1;
                const float wf = (float)((double)c[sd][i] * inv);
                float qv;
                unsigned short bits = 0;
                if (a.fmt == 1) {
                    const __half hv = __float2half_rn(wf);
                    bits = __half_as_ushort(hv);
                    qv = __half2float(hv);
                } else if (a.fmt == 2) {
                    const __nv_bfloat16 hv = __float2bfloat16_rn(wf);
                    bits = __bfloat16_as_ushort(hv);
                    qv = __bfloat162float(hv);
                } else {
                    qv = wf;
                }
                if (a.class_w) {
                    const size_t ci = (size_t)it * LLL + o;
                    const bool keep = active && o != KC;
                    if (a.fmt == 0) reinterpret_cast<float*>(a.class_w)[ci] = keep ? wf : 0.f;
                    else reinterpret_cast<unsigned short*>(a.class_w)[ci] = keep ? bits : (unsigned short)0;
                }
                if (o == KC) {
                    centre_q = qv;
                    continue;
                }
                if (!active) continue;
                qsum += (double)qv;
                if (a.class_w || gz < a.z0 || gz >= a.z1) continue;
                const int zl = gz - a.z0;
                const int q = gy * a.nxq + (gx >> 3);
                const size_t tile = (size_t)zl * a.tpp + q / a.tile;
                const int e = q % a.tile, j = gx & 7;
                const size_t idx = ((tile * (size_t)(a.K - 1) + slot_of(ox, oy, oz, R)) * a.tile + e) * 8 + j;
                if (a.fmt == 0) reinterpret_cast<float*>(a.Wt)[idx] = wf;
                else reinterpret_cast<unsigned short*>(a.Wt)[idx] = bits;
            }
        }
        const double off = block_sum_f64<S::NW, true, CLEAN>(qsum, red);
        const bool centre = real && col[0] == R * L + R && R >= G::zA && R < G::zA + NA;
        if (centre && a.class_w) {
            a.class_diag[it] = a.mass_fix ? fp32_pair(M - off) : make_float2(centre_q, 0.f);
            if (a.class_mass) a.class_mass[it] = M;
        } else if (centre && sz >= a.z0 && sz < a.z1) {
            const float2 d = a.mass_fix ? fp32_pair(M - off) : make_float2(centre_q, 0.f);
            const int zl = sz - a.z0;
            const int q = sy * a.nxq + (sx >> 3);
            const size_t tile = (size_t)zl * a.tpp + q / a.tile;
            a.diag[(tile * a.tile + q % a.tile) * 8 + (sx & 7)] = d;
        }
    }
}

template <int R, bool CLEAN, bool CO>
__global__ void __launch_bounds__(BalShape<R>::NT, BalShape<R>::kMinBlocks) kgen_bal_kernel(const KgenArgs a)
{
    constexpr int NPW = BalShape<R>::NPW;
    if constexpr (BalShape<R>::NSEG == 2) {
        if (threadIdx.x < NPW) bal_body<R, 0, CLEAN, CO>(a);
        else bal_body<R, 1, CLEAN, CO>(a);
    } else {
        static_assert(BalShape<R>::NSEG == 3, "R = 5, 8");
        if (threadIdx.x < NPW) bal_body<R, 0, CLEAN, CO>(a);
        else if (threadIdx.x < 2 * NPW) bal_body<R, 1, CLEAN, CO>(a);
        else bal_body<R, 2, CLEAN, CO>(a);
    }
}

template <int R, bool CLEAN, bool CO>
static cudaError_t launch_bal_r(const KgenArgs& a, cudaStream_t s)
{
    using S = BalShape<R>;
    const long nsrc = a.src_list ? a.n_list : (long)a.nx * a.ny * (a.sz1 - a.sz0);
    if (nsrc <= 0) return cudaSuccess;
    const size_t smem = S::smem_bytes + (!a.cheb_m ? 0 : ((size_t)(a.cheb_m + 1) * 4 + 15) / 16 * 16);
    cudaError_t e = cudaFuncSetAttribute(kgen_bal_kernel<R, CLEAN, CO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kgen_bal_kernel<R, CLEAN, CO>, S::NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    long grid = (long)sms * per_sm;
    if (grid > nsrc) grid = nsrc;
    kgen_bal_kernel<R, CLEAN, CO><<<(unsigned)grid, S::NT, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_kgen_bal(const KgenArgs& a, int R, cudaStream_t s)
{
    if (a.fp64 || a.symmetric) return cudaErrorNotSupported;
    // FDIRW_KGEN_SYNCCHECK=1: the synccheck-clean barrier form (kgen_common.cuh), for sanitizer runs
    static const bool clean = [] {
        const char* ev = getenv("FDIRW_KGEN_SYNCCHECK");
        return ev && ev[0] == '1';
    }();
    const bool co = a.cheb_m && a.cheb_open;
    if (R == 5)
        return clean ? (co ? launch_bal_r<5, true, true>(a, s) : launch_bal_r<5, true, false>(a, s))
                     : (co ? launch_bal_r<5, false, true>(a, s) : launch_bal_r<5, false, false>(a, s));
    if (R == 8)
        return clean ? (co ? launch_bal_r<8, true, true>(a, s) : launch_bal_r<8, true, false>(a, s))
                     : (co ? launch_bal_r<8, false, true>(a, s) : launch_bal_r<8, false, false>(a, s));
    return cudaErrorNotSupported;
}

}  // namespace fdirw
