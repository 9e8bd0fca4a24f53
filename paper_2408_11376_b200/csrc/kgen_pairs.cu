// kgen_pairs.cu — a3 + a4 (the same method and arithmetic as kgen.cu's column kernel) for
// R = 5 with TWO window columns per thread, halved in z (DESIGN.md §7 "round 2, pairs").
//
// Why: the column kernel moves 20 B of shared memory per cell-pass (a thread owns one z-column;
// its 4 lateral neighbour columns are read from smem and its own column written back), and ncu
// shows that stream as the binding resource.  Here a thread owns the columns 2p and 2p + 1
// (linear column order t = cy·L + cx) over one half of the window's z range: the x face
// between the two columns is a register read, so per pass a thread loads 6 neighbour segments
// (−x of the left column, +x of the right one, ±y of both) and the other half's boundary cell
// of both columns, and stores its 2 segments: 4.17 accesses per cell instead of 5 (16.7 B).
// Halving z keeps the per-thread state at 12 cells (about the column kernel's 11), so the
// occupancy (4 CTAs × 4 warps per SM) is unchanged.
//
// Layout of one pass buffer (per parity): for each z segment s (cells zb = 6s … zb + 5; the
// upper segment's last cell 11 is a phantom outside the window) three arrays indexed by
// [side][pair + PAD]: H = cell zb (scalar), Q = cells zb+1 … zb+4 (float4), T = cell zb + 5
// (scalar; none for the phantom).  Lanes of a warp hold consecutive pairs, and every neighbour
// is at a fixed pair offset on a fixed side, so all accesses are consecutive 4 / 16 B words
// (conflict-free).  PAD slots on both sides stay 0 and stand in for neighbours outside the
// window (their face numbers are 0).
//
// Per-cell arithmetic is the column kernel's, operation for operation (literal substeps in flux
// form with the z faces first; Chebyshev passes in row form, reading A30), so the substep and
// recurrence values are bitwise the column kernel's; only the fp64 epilogue sums group cells
// per thread differently.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "fdirw_internal.h"
#include "kgen_common.cuh"
#include "layout.cuh"

namespace fdirw {

namespace {

template <int R>
struct PairShape {
    static constexpr int L = 2 * R + 1, LL = L * L, LLL = LL * L;
    static constexpr int NC = 6;                         // cells per z segment (head, quad, tail)
    static constexpr int NSEG = (L + 1) / NC;            // z segments; the last one's tail is a phantom
    static_assert(NSEG * NC == L + 1, "L = 6·NSEG − 1 (R = 2, 5, 8)");
    static constexpr int NP = (LL + 1) / 2;              // column pairs (the last may hold a dummy)
    static constexpr int NPW = (NP + 31) / 32 * 32;      // threads per z segment
    static constexpr int NT = NSEG * NPW;
    static constexpr int NW = NT / 32;
    static constexpr int PAD = (R + 2 + 3) / 4 * 4;      // > the largest pair offset, R + 1
    static constexpr int NPP = (NPW + 2 * PAD + 3) / 4 * 4;  // slots per side
    static constexpr int SEGF = 2 * NPP * 6;             // floats per segment: H, Q (×4), T
    static constexpr int BUFF = NSEG * SEGF;             // floats per parity
    // ~128 registers per thread: R5 4 CTAs (16 warps) per SM, R8 1 CTA (15 warps)
    static constexpr int kMinBlocks = 65536 / (NT * 128) > 0 ? 65536 / (NT * 128) : 1;
    static constexpr size_t buf_bytes = 2 * (size_t)BUFF * 4;
    static constexpr size_t tab_off = buf_bytes + ((LLL + 15) / 16) * 16 + NW * 8 + 16;  // face tables
    static constexpr size_t smem_bytes = tab_off + 64 * 4;
    static constexpr size_t cheb_off = smem_bytes;       // Chebyshev c_0..c_m (fp32) follow
};

}  // namespace

// One z segment's threads (cells 6·SEG … 6·SEG + 5; the last segment's cell L is a phantom).
// The segments' warps run separate instantiations and meet at the same CTA barriers (each warp
// is uniform; every path executes the identical barrier sequence).
template <int R, int SEG>
__device__ __forceinline__ void pair_body(const KgenArgs& a)
{
    using S = PairShape<R>;
    constexpr int L = S::L, LL = S::LL, LLL = S::LLL, NC = S::NC, NPP = S::NPP, SEGF = S::SEGF;
    constexpr int KC = LLL / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* buf = reinterpret_cast<float*>(smem_raw);
    unsigned char* ph = smem_raw + S::buf_bytes;
    double* red = reinterpret_cast<double*>(smem_raw + S::buf_bytes + ((LLL + 15) / 16) * 16);

    const int t = threadIdx.x;
    constexpr int seg = SEG;
    const int p = t - seg * S::NPW;             // column pair
    constexpr int zb = seg * NC;
    const bool real = p < S::NP;
    const int col[2] = {2 * p, 2 * p + 1};
    const bool has[2] = {real, real && 2 * p + 1 < LL};
    const int pp = p + S::PAD;
    // neighbour slots (side, pair) of the two columns; see the header
    const int jxmA = 1 * NPP + pp - 1, jymA = 1 * NPP + pp - (R + 1), jypA = 1 * NPP + pp + R;
    const int jxpB = 0 * NPP + pp + 1, jymB = 0 * NPP + pp - R, jypB = 0 * NPP + pp + R + 1;
    const int jA = pp, jB = NPP + pp;
    constexpr bool top = seg == S::NSEG - 1;     // its tail cell is the phantom
    constexpr bool hb = seg > 0, ha = !top;      // halo cells below / above
    const int nx = a.nx, ny = a.ny, nz = a.nz;
    const long nsrc = a.src_list ? a.n_list : (long)nx * ny * (a.sz1 - a.sz0);

    // zero both pass buffers once: PAD and dummy slots are read, never written
    for (int i = t; i < 2 * S::BUFF; i += S::NT) buf[i] = 0.f;
    // one __syncthreads per pass (a neighbour-only sync through per-warp mbarriers, which lets
    // warps drift up to a pass apart, was measured slower: cfg3 150 vs 114 ms, cfg5 852 vs 654 ms)
    auto pass_sync = [&](unsigned) { __syncthreads(); };
    unsigned ps = 0;  // passes so far (all windows): buffer parity and mbarrier phase
    float* ftab = reinterpret_cast<float*>(smem_raw + S::tab_off);
    build_face_tables(ftab, a.lam_ff, a.lam_fs, a.lam_ss, a.mu2_ff, a.mu2_fs, a.mu2_ss);
    if (a.cheb_m) {
        float* cc = reinterpret_cast<float*>(smem_raw + S::cheb_off);
        for (int i = t; i <= a.cheb_m; i += S::NT) cc[i] = a.cheb_c[i];
    }

    // segment buffers of parity b: H, Q, T of segment s
    auto Hp = [&](float* b, int s) { return b + s * SEGF; };
    auto Qp = [&](float* b, int s) { return reinterpret_cast<float4*>(b + s * SEGF + 2 * NPP); };
    auto Tp = [&](float* b, int s) { return b + s * SEGF + 10 * NPP; };
    auto store_seg = [&](float* b, int j, const float (&v)[NC]) {
        Hp(b, seg)[j] = v[0];
        Qp(b, seg)[j] = make_float4(v[1], v[2], v[3], v[4]);
        if (!top) Tp(b, seg)[j] = v[5];
    };
    auto load_seg = [&](const float* b, int j, float (&v)[NC]) {
        float* bb = const_cast<float*>(b);
        v[0] = Hp(bb, seg)[j];
        const float4 q = Qp(bb, seg)[j];
        v[1] = q.x; v[2] = q.y; v[3] = q.z; v[4] = q.w;
        v[5] = !top ? Tp(bb, seg)[j] : 0.f;
    };
    // the neighbouring segments' boundary cells of column slot j: below = segment SEG − 1's
    // tail (cell zb − 1), above = segment SEG + 1's head (cell zb + 6)
    // (unconditional loads: an edge segment reads its own slot, a finite value that no z term
    // uses — the below / above guards skip the window's first and last cells)
    constexpr int sb = hb ? seg - 1 : seg, sa = ha ? seg + 1 : seg;
    auto load_below = [&](const float* b, int j) { return Tp(const_cast<float*>(b), sb)[j]; };
    auto load_above = [&](const float* b, int j) { return Hp(const_cast<float*>(b), sa)[j]; };

    for (long it = blockIdx.x; it < nsrc; it += gridDim.x) {
        const long src = a.src_list ? (long)a.src_list[it] : it;
        const int sx = (int)(src % nx);
        const int sy = (int)((src / nx) % ny);
        const int sz = a.sz0 + (int)(src / ((long)nx * ny));

        __syncthreads();  // the previous source's readers of ph are done (and the zero fill)
        int far_here = 0;
        for (int i = t; i < LLL; i += S::NT) {
            const int gx = sx + i % L - R, gy = sy + (i / L) % L - R, gz = sz + i / LL - R;
            const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz;
            unsigned char v = in ? a.mask[((size_t)(gz - a.mz0) * ny + gy) * nx + gx] : (unsigned char)2;
            if (in && v == 2) v = 3;
            far_here |= v == 3;
            ph[i] = v;
        }
        const bool open = __syncthreads_or(far_here) != 0;
        if (ph[KC] == 3) continue;

        // ---- face numbers of the owned cells (cell i of side s: z = zb + i, column col[s]) ----
        // lateral, packed for FFMA2 in the cell pairs (0,5), (1,2), (3,4): fl[s][f][h], f = −x, +x,
        // −y, +y; the x face between the two columns is A's +x = B's −x (face_lambda symmetric
        // for closed windows; open windows run the literal path, where each side keeps its own)
        unsigned long long fl[2][4][3];
        auto FL = [&](int sd, int f, int h) { return (sd == 1 && f == 0) ? fl[0][1][h] : fl[sd][f][h]; };
        // z faces: fz[s][j] = the face between cells zb + j − 1 and zb + j, j = 0..6
        float fz[2][NC + 1];
        unsigned long long dg2[2][3];
        unsigned rmask[2] = {0u, 0u};
        auto faces = [&](const float* T, const bool row_form) {  // T: face table set (λ or 2μ)
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
                const int c = col[sd], cx = c % L, cy = c / L;
                float v[4][NC], d[NC];
#pragma unroll
                for (int j = 0; j <= NC; ++j) {
                    const int z = zb + j;
                    float f = 0.f;
                    if (has[sd] && z >= 1 && z < L) {
                        const unsigned pl = ph[(z - 1) * LL + c], pu = ph[z * LL + c];
                        f = T[16 + ((pl << 2) | pu)];
                    }
                    fz[sd][j] = f;
                }
#pragma unroll
                for (int i = 0; i < NC; ++i) {
                    const int z = zb + i, o = z * LL + c;
                    const bool cell = has[sd] && z < L;
                    const unsigned pc = cell ? ph[o] : 2u;
                    v[0][i] = (cell && cx > 0) ? T[(pc << 2) | ph[o - 1]] : 0.f;
                    // side A's +x is the pair's shared x face, as seen from its active side (as fz)
                    v[1][i] = (cell && cx < L - 1) ? T[(sd == 0 ? 16 : 0) + ((pc << 2) | ph[o + 1])] : 0.f;
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
                for (int f = 0; f < 4; ++f) {
                    if (sd == 1 && f == 0) continue;  // B's −x face is A's +x (FL)
                    fl[sd][f][0] = pk2(v[f][0], v[f][5]);
                    fl[sd][f][1] = pk2(v[f][1], v[f][2]);
                    fl[sd][f][2] = pk2(v[f][3], v[f][4]);
                }
                if (row_form) {
                    dg2[sd][0] = pk2(d[0], d[5]);
                    dg2[sd][1] = pk2(d[1], d[2]);
                    dg2[sd][2] = pk2(d[3], d[4]);
                }
            }
        };
        faces(ftab, false);

        // state: c[s][i]
        float c[2][NC];
#pragma unroll
        for (int sd = 0; sd < 2; ++sd)
#pragma unroll
            for (int i = 0; i < NC; ++i)
                c[sd][i] = (real && sd == 0 && col[0] == R * L + R && zb + i == R) ? 1.f : 0.f;

        // which z terms exist for cell i (the column kernel's z > 0 / z < L − 1 guards)
        auto below = [&](int i) { return zb + i > 0; };
        auto above = [&](int i) { return zb + i < L - 1; };
        // cell pairs for the packed lanes
        constexpr int PA[3] = {0, 1, 3}, PB[3] = {5, 2, 4};

        // neighbour values of side sd's lateral faces, f = −x, +x, −y, +y
        auto gather = [&](const float* b, float (&nb)[2][4][NC], float (&hlb)[2], float (&hla)[2]) {
            load_seg(b, jxmA, nb[0][0]);
            load_seg(b, jymA, nb[0][2]);
            load_seg(b, jypA, nb[0][3]);
            load_seg(b, jxpB, nb[1][1]);
            load_seg(b, jymB, nb[1][2]);
            load_seg(b, jypB, nb[1][3]);
            hlb[0] = load_below(b, jA);
            hlb[1] = load_below(b, jB);
            hla[0] = load_above(b, jA);
            hla[1] = load_above(b, jB);
        };

        const bool act = real;
        const bool cheb = a.cheb_m && !open;
        const int n_direct = cheb ? a.cheb_pre : a.n_fd;
        // ---- literal substeps: flux form (the column kernel's operation order) ----
        for (int k = 0; k < n_direct; ++k, ++ps) {
            float* b = buf + (ps & 1u) * S::BUFF;
            if (act) {
                store_seg(b, jA, c[0]);
                store_seg(b, jB, c[1]);
            }
            pass_sync(ps);
            if (act) {
                float nb[2][4][NC], hlb[2], hla[2];
                gather(b, nb, hlb, hla);
#pragma unroll
                for (int i = 0; i < NC; ++i) {  // the x face between the pair: registers
                    nb[0][1][i] = c[1][i];
                    nb[1][0][i] = c[0][i];
                }
                float nw[2][NC];
#pragma unroll
                for (int sd = 0; sd < 2; ++sd) {
                    // dz[j] = cur(zb + j) − cur(zb + j − 1), j = 0..6 (halo cells at both ends)
                    float dz[NC + 1];
#pragma unroll
                    for (int j = 0; j <= NC; ++j) {
                        const float up = j < NC ? c[sd][j] : hla[sd];
                        const float dn = j > 0 ? c[sd][j - 1] : hlb[sd];
                        dz[j] = up - dn;
                    }
                    // the z faces before the lateral ones for R ≤ 5, after them for R > 5: the
                    // column kernel's order per R, so both kernels give the same bits
                    auto zterms = [&]() {
#pragma unroll
                        for (int i = 0; i < NC; ++i) {
                            float v = nw[sd][i];
                            if (below(i)) v = fmaf(fz[sd][i], -dz[i], v);
                            if (above(i)) v = fmaf(fz[sd][i + 1], dz[i + 1], v);
                            nw[sd][i] = v;
                        }
                    };
#pragma unroll
                    for (int i = 0; i < NC; ++i) nw[sd][i] = c[sd][i];
                    if constexpr (R <= 5) zterms();
#pragma unroll
                    for (int h = 0; h < 3; ++h) {
                        const int i0 = PA[h], i1 = PB[h];
                        const unsigned long long c2 = pk2(c[sd][i0], c[sd][i1]);
                        unsigned long long s2 = pk2(nw[sd][i0], nw[sd][i1]);
#pragma unroll
                        for (int f = 0; f < 4; ++f)
                            s2 = fma2(FL(sd, f, h), sub2(pk2(nb[sd][f][i0], nb[sd][f][i1]), c2), s2);
                        upk2(s2, nw[sd][i0], nw[sd][i1]);
                    }
                    if constexpr (R > 5) zterms();
                }
#pragma unroll
                for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                    for (int i = 0; i < NC; ++i) c[sd][i] = (rmask[sd] >> i) & 1u ? 0.f : nw[sd][i];
            }
        }
        if (cheb) {
            // ---- Chebyshev passes in row form (reading A30): t_{k+1} = D∘t + Σ F_f t_f − t_{k−1} ----
            faces(ftab + 32, true);
            const float* cc = reinterpret_cast<const float*>(smem_raw + S::cheb_off);
            float pv[2][NC], acc[2][NC];
#pragma unroll
            for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                for (int i = 0; i < NC; ++i) {
                    pv[sd][i] = 0.f;
                    acc[sd][i] = c[sd][i] * cc[0];
                }
            auto step = [&](float (&cur)[2][NC], float (&prv)[2][NC], const int k, const bool first) {
                float* b = buf + (ps & 1u) * S::BUFF;
                if (act) {
                    store_seg(b, jA, cur[0]);
                    store_seg(b, jB, cur[1]);
                }
                pass_sync(ps);
                ++ps;
                const float ck = cc[k + 1];
                if (act) {
                    float nb[2][4][NC], hlb[2], hla[2];
                    gather(b, nb, hlb, hla);
#pragma unroll
                    for (int i = 0; i < NC; ++i) {
                        nb[0][1][i] = cur[1][i];
                        nb[1][0][i] = cur[0][i];
                    }
#pragma unroll
                    for (int sd = 0; sd < 2; ++sd) {
                        float nw[NC];
#pragma unroll
                        for (int h = 0; h < 3; ++h) {
                            const int i0 = PA[h], i1 = PB[h];
                            const unsigned long long s2 =
                                fma2(dg2[sd][h], pk2(cur[sd][i0], cur[sd][i1]), pk2(-prv[sd][i0], -prv[sd][i1]));
                            upk2(s2, nw[i0], nw[i1]);
                        }
#pragma unroll
                        for (int i = 0; i < NC; ++i) {
                            float v = nw[i];
                            const float dn = i > 0 ? cur[sd][i - 1] : hlb[sd];
                            const float up = i < NC - 1 ? cur[sd][i + 1] : hla[sd];
                            if (below(i)) v = fmaf(fz[sd][i], dn, v);
                            if (above(i)) v = fmaf(fz[sd][i + 1], up, v);
                            nw[i] = v;
                        }
#pragma unroll
                        for (int h = 0; h < 3; ++h) {
                            const int i0 = PA[h], i1 = PB[h];
                            unsigned long long s2 = pk2(nw[i0], nw[i1]);
#pragma unroll
                            for (int f = 0; f < 4; ++f)
                                s2 = fma2(FL(sd, f, h), pk2(nb[sd][f][i0], nb[sd][f][i1]), s2);
                            if (first) s2 = fma2(s2, pk2(0.5f, 0.5f), pk2(-0.f, -0.f));
                            upk2(s2, prv[sd][i0], prv[sd][i1]);
                            const unsigned long long a2 = fma2(pk2(ck, ck), s2, pk2(acc[sd][i0], acc[sd][i1]));
                            upk2(a2, acc[sd][i0], acc[sd][i1]);
                        }
                    }
                }
            };
            const int m = a.cheb_m;
            step(c, pv, 0, true);
            for (int k = 1; k < m; k += 2) {
                step(pv, c, k, false);
                if (k + 1 < m) step(c, pv, k + 1, false);
            }
#pragma unroll
            for (int sd = 0; sd < 2; ++sd)
#pragma unroll
                for (int i = 0; i < NC; ++i) c[sd][i] = fmaxf(acc[sd][i], 0.f);
        }

        // ---- epilogue (a4): as kgen.cu's, per owned cell ----
        double s = 0.0;
#pragma unroll
        for (int sd = 0; sd < 2; ++sd)
#pragma unroll
            for (int i = 0; i < NC; ++i)
                if (has[sd] && zb + i < L) s += (double)c[sd][i];
        const double S_ = block_sum_f64<S::NW>(s, red);
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
            for (int i = 0; i < NC; ++i) {
                const int z = zb + i;
                if (z >= L) continue;
                const int o = z * LL + col[sd];
                const int oz = z - R, gz = sz + oz;
                const bool active = ph[o] <= 1;
                const float wf = (float)((double)c[sd][i] * inv);
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
                if (a.class_w) {
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
                const size_t idx = ((tile * (size_t)(a.K - 1) + slot_of(ox, oy, oz, R)) * a.tile + e) * 8 + j;
                if (a.fmt == 0) reinterpret_cast<float*>(a.Wt)[idx] = wf;
                else reinterpret_cast<unsigned short*>(a.Wt)[idx] = bits;
            }
        }
        const double off = block_sum_f64<S::NW>(qsum, red);
        // the centre cell: column R·L + R (a pair's left column: R·L + R is even), z = R
        const bool centre = real && seg == R / NC && col[0] == R * L + R;
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

// One instantiation per segment (measured faster than a single code path with the segment taken
// at run time: cfg3 112 vs 124 ms, cfg5 693 vs 735 ms, despite R8's three paths' I-cache misses)
template <int R>
__global__ void __launch_bounds__(PairShape<R>::NT, PairShape<R>::kMinBlocks) kgen_pair_kernel(const KgenArgs a)
{
    constexpr int NPW = PairShape<R>::NPW;
    if constexpr (PairShape<R>::NSEG == 1) {
        pair_body<R, 0>(a);
    } else if constexpr (PairShape<R>::NSEG == 2) {
        if (threadIdx.x < NPW) pair_body<R, 0>(a);
        else pair_body<R, 1>(a);
    } else {
        static_assert(PairShape<R>::NSEG == 3, "R = 2, 5, 8");
        if (threadIdx.x < NPW) pair_body<R, 0>(a);
        else if (threadIdx.x < 2 * NPW) pair_body<R, 1>(a);
        else pair_body<R, 2>(a);
    }
}

template <int R>
static cudaError_t launch_pairs_r(const KgenArgs& a, cudaStream_t s)
{
    using S = PairShape<R>;
    const long nsrc = a.src_list ? a.n_list : (long)a.nx * a.ny * (a.sz1 - a.sz0);
    if (nsrc <= 0) return cudaSuccess;
    const size_t smem = S::smem_bytes + (!a.cheb_m ? 0 : ((size_t)(a.cheb_m + 1) * 4 + 15) / 16 * 16);
    cudaError_t e = cudaFuncSetAttribute(kgen_pair_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kgen_pair_kernel<R>, S::NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    long grid = (long)sms * per_sm;
    if (grid > nsrc) grid = nsrc;
    kgen_pair_kernel<R><<<(unsigned)grid, S::NT, smem, s>>>(a);
    return cudaGetLastError();
}

// R = 5 and 8 (L = 6·NSEG − 1), fp32 substeps, no symmetric rule; cudaErrorNotSupported
// otherwise (the caller keeps the column kernel).
cudaError_t launch_kgen_pairs(const KgenArgs& a, int R, cudaStream_t s)
{
    if (a.fp64 || a.symmetric) return cudaErrorNotSupported;
    if (R == 5) return launch_pairs_r<5>(a, s);
    if (R == 8) return launch_pairs_r<8>(a, s);
    return cudaErrorNotSupported;
}

}  // namespace fdirw
