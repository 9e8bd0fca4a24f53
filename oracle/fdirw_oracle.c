/*
 * fdirw_oracle.c — CPU fp64 ORACLE for the FDiRW hot path (arXiv 2408.11376).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2408_11376_b200/) never links, imports or calls it,
 * and shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C99 in fp64.  OpenMP only parallelises the
 * independent per-source loop (each source's kernel is computed by one thread
 * with the same arithmetic, so results do not depend on the thread count).
 *
 * Paper references are "P:<line> §<sec>" into PAPER.md; readings of the paper
 * that the paper leaves open are the "A<n>" entries of DESIGN.md §3.
 *
 * Conventions:
 *   grid [nz][ny][nx], x fastest; voxel index v = (z*ny + y)*nx + x.
 *   mask[v] = 1 fast phase (liquid), 0 slow phase (solid)
 *   window of source s = cube s + [-R,R]^3 (Chebyshev radius R), K=(2R+1)^3 (A1)
 *   window slot o = ((oz+R)*L + (oy+R))*L + (ox+R), L = 2R+1.
 *
 * Parity status of each function is listed in DESIGN.md §4; every function
 * here is pinned by a -m "not gpu" test in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_UNSTABLE 2

typedef struct {
    int32_t nx, ny, nz;
    double dh;
    double D_fast, D_slow; /* effective diffusivities D*A/RT (Eqs.1-3, A6) */
    double dt;             /* macro step Δt (Table 1)                       */
    int32_t R;
    int32_t n_fd;          /* 0 = derive (a1)                                        */
} oracle_params;

typedef struct {
    int32_t n_fd;
    double dt_fd;
    double lam_ff, lam_fs, lam_ss; /* face numbers λ = Δt_fd·D_face/Δh² */
} oracle_derived;

/* ---------------------------------------------------------------------------
 * a1. Parameter derivation.
 * Table 1: Δt = 500 µs, Δt_fd = 0.5 µs, D_L·A_L/RT = 2e-11 m²/s,
 * Δh = 1e-8 m, i.e. λ* = D_L_eff·Δt_fd/Δh² = 0.1 and n_fd = Δt/Δt_fd = 1000.
 * We keep λ* = 0.1 and derive n_fd = ceil(x·(1-1e-9)), x = D_max·Δt/(λ*·Δh²)
 * (reading A5); Δt_fd = Δt/n_fd.  Explicit FD stability: λ_max ≤ 1/6.
 * Face diffusivity between phases: harmonic mean (reading A4).
 * ------------------------------------------------------------------------- */
static double harmonic(double a, double b) { return (a + b) == 0.0 ? 0.0 : 2.0 * a * b / (a + b); }

int oracle_derive(const oracle_params* p, oracle_derived* d)
{
    if (!p || !d) return OR_INVALID;
    if (p->nx < 1 || p->ny < 1 || p->nz < 1 || p->R < 1 || !(p->dh > 0) || !(p->dt > 0) ||
        !(p->D_fast > 0) || !(p->D_slow >= 0) || p->n_fd < 0)
        return OR_INVALID;
    double Dmax = p->D_fast > p->D_slow ? p->D_fast : p->D_slow;
    int n = p->n_fd;
    if (n == 0) {
        double x = Dmax * p->dt / (0.1 * p->dh * p->dh);
        double c = ceil(x * (1.0 - 1e-9));
        n = c < 1.0 ? 1 : (int)c;
    }
    d->n_fd = n;
    d->dt_fd = p->dt / (double)n;
    double s = d->dt_fd / (p->dh * p->dh);
    d->lam_ff = s * p->D_fast;
    d->lam_ss = s * p->D_slow;
    d->lam_fs = s * harmonic(p->D_fast, p->D_slow);
    if (d->lam_ff > 1.0 / 6.0 || d->lam_ss > 1.0 / 6.0) return OR_UNSTABLE;
    return OR_OK;
}

/* phase codes: 0 slow, 1 fast, 2 far-field liquid reservoir (NEXT row N2: a fast-phase
 * Dirichlet cell) — for the face number it counts as fast. */
static double face_lambda(const oracle_derived* d, int pi, int pj)
{
    pi = pi != 0;
    pj = pj != 0;
    if (pi && pj) return d->lam_ff;
    if (!pi && !pj) return d->lam_ss;
    return d->lam_fs;
}

/* ---------------------------------------------------------------------------
 * a3. One source's window kernel, fp64 (§3.1: "the elements of j-th
 * column in p can be obtained directly by solving the governing diffusion
 * equation with an initial single point source ... using the explicit Finite
 * Difference Method"; windowed per north_star, readings A1, A2, A7, A8, A21).
 *
 *   c⁰ = δ_s (unit mass at the source voxel, A7)
 *   c^{k+1}_i = c^k_i + Σ_{j ∈ nb(i)} λ_ij (c^k_j − c^k_i),  k = 0..n_fd-1
 * nb(i): the 6 face neighbours, in the order −x,+x,−y,+y,−z,+z, that lie in the
 * window AND in the domain; faces leaving either carry no flux (A2, A3, A21).
 * Jacobi: every flux uses the previous iterate.  Output W[o] = c^{n_fd}(s+o),
 * 0 for window cells outside the domain.
 * N2 (open domain): window cells with mask 2 are the far-field reservoir held at 0
 * (absorbing Dirichlet: the kernel is the response to c(t0) with
 * c_far = 0; the c_far part is p_BC): their value stays 0 and faces into them
 * carry flux λ(p_i, fast)·(0 − c_i).  A source on a far-field cell has W = 0.
 * ------------------------------------------------------------------------- */
void oracle_kernel(const oracle_params* p, const oracle_derived* d, const uint8_t* mask,
                   int sx, int sy, int sz, double* W)
{
    const int R = p->R, L = 2 * R + 1, K = L * L * L;
    double* cur = (double*)calloc((size_t)K, sizeof(double));
    double* nxt = (double*)calloc((size_t)K, sizeof(double));
    uint8_t* act = (uint8_t*)calloc((size_t)K, 1);
    uint8_t* res = (uint8_t*)calloc((size_t)K, 1); /* far-field reservoir cell */
    uint8_t* ph = (uint8_t*)calloc((size_t)K, 1);
    double* lam = (double*)calloc((size_t)K * 6, sizeof(double)); /* per cell, per face */
    int* nbr = (int*)malloc((size_t)K * 6 * sizeof(int));
    static const int DX[6] = {-1, 1, 0, 0, 0, 0}, DY[6] = {0, 0, -1, 1, 0, 0}, DZ[6] = {0, 0, 0, 0, -1, 1};

    for (int oz = -R; oz <= R; ++oz)
        for (int oy = -R; oy <= R; ++oy)
            for (int ox = -R; ox <= R; ++ox) {
                int i = ((oz + R) * L + (oy + R)) * L + (ox + R);
                int x = sx + ox, y = sy + oy, z = sz + oz;
                int in = x >= 0 && x < p->nx && y >= 0 && y < p->ny && z >= 0 && z < p->nz;
                ph[i] = in ? mask[((size_t)z * p->ny + y) * p->nx + x] : 0;
                res[i] = (uint8_t)(in && ph[i] == 2);
                act[i] = (uint8_t)(in && ph[i] != 2);
            }
    for (int oz = -R; oz <= R; ++oz)
        for (int oy = -R; oy <= R; ++oy)
            for (int ox = -R; ox <= R; ++ox) {
                int i = ((oz + R) * L + (oy + R)) * L + (ox + R);
                for (int f = 0; f < 6; ++f) {
                    int qx = ox + DX[f], qy = oy + DY[f], qz = oz + DZ[f];
                    int j = -1;
                    if (qx >= -R && qx <= R && qy >= -R && qy <= R && qz >= -R && qz <= R)
                        j = ((qz + R) * L + (qy + R)) * L + (qx + R);
                    if (j >= 0 && act[i] && (act[j] || res[j])) {
                        nbr[i * 6 + f] = j;
                        lam[i * 6 + f] = face_lambda(d, ph[i], ph[j]);
                    } else {
                        nbr[i * 6 + f] = -1;
                        lam[i * 6 + f] = 0.0;
                    }
                }
            }
    if (act[(R * L + R) * L + R]) cur[(R * L + R) * L + R] = 1.0;
    for (int k = 0; k < d->n_fd; ++k) {
        for (int i = 0; i < K; ++i) {
            if (!act[i]) { nxt[i] = 0.0; continue; }
            double acc = cur[i];
            for (int f = 0; f < 6; ++f) {
                int j = nbr[i * 6 + f];
                if (j >= 0) acc += lam[i * 6 + f] * (cur[j] - cur[i]);
            }
            nxt[i] = acc;
        }
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(W, cur, (size_t)K * sizeof(double));
    free(cur); free(nxt); free(act); free(res); free(ph); free(lam); free(nbr);
}

/* Kernels of every source in the box [x0,x1)×[y0,y1)×[z0,z1) (clipped to the
 * domain by the caller), stored W[((sz-z0)*(y1-y0) + (sy-y0))*(x1-x0) + (sx-x0)][K]. */
void oracle_build_kernels(const oracle_params* p, const oracle_derived* d, const uint8_t* mask,
                          const int32_t* box, double* W)
{
    const int L = 2 * p->R + 1, K = L * L * L;
    const int bx = box[1] - box[0], by = box[3] - box[2], bz = box[5] - box[4];
    const long nsrc = (long)bx * by * bz;
#pragma omp parallel for schedule(dynamic, 1)
    for (long n = 0; n < nsrc; ++n) {
        int sx = box[0] + (int)(n % bx);
        int sy = box[2] + (int)((n / bx) % by);
        int sz = box[4] + (int)(n / ((long)bx * by));
        oracle_kernel(p, d, mask, sx, sy, sz, W + (size_t)n * K);
    }
}

/* ---------------------------------------------------------------------------
 * a5 (oracle form O4). Superposition in SCATTER form, fp64 (Eq.8,
 * P:109 "p_ij is the mass proportion moving from node j to node i", Eq.14,
 * closed domain so no p_BC term, reading A3):
 *      C_new[s+o] += W_s(o) · C_old[s]   for ascending s, then ascending o.
 * Sources: the box `sbox` (kernels W laid out as oracle_build_kernels writes
 * them).  Targets: the box `tbox`; Cout has tbox's shape and is overwritten.
 * Only targets whose every source lies in sbox are complete — the caller
 * passes sbox ⊇ (tbox expanded by R) ∩ domain.
 * ------------------------------------------------------------------------- */
void oracle_step_scatter(const oracle_params* p, const double* W, const int32_t* sbox,
                         const double* Cold /* full grid */, const int32_t* tbox, double* Cout)
{
    const int R = p->R, L = 2 * R + 1, K = L * L * L;
    const int sbx = sbox[1] - sbox[0], sby = sbox[3] - sbox[2], sbz = sbox[5] - sbox[4];
    const int tbx = tbox[1] - tbox[0], tby = tbox[3] - tbox[2], tbz = tbox[5] - tbox[4];
    memset(Cout, 0, sizeof(double) * (size_t)tbx * tby * tbz);
    for (int sz = sbox[4]; sz < sbox[5]; ++sz)
        for (int sy = sbox[2]; sy < sbox[3]; ++sy)
            for (int sx = sbox[0]; sx < sbox[1]; ++sx) {
                size_t n = ((size_t)(sz - sbox[4]) * sby + (sy - sbox[2])) * sbx + (sx - sbox[0]);
                const double* Ws = W + n * K;
                double cs = Cold[((size_t)sz * p->ny + sy) * p->nx + sx];
                for (int oz = -R; oz <= R; ++oz)
                    for (int oy = -R; oy <= R; ++oy)
                        for (int ox = -R; ox <= R; ++ox) {
                            int x = sx + ox, y = sy + oy, z = sz + oz;
                            if (x < tbox[0] || x >= tbox[1] || y < tbox[2] || y >= tbox[3] ||
                                z < tbox[4] || z >= tbox[5])
                                continue;
                            int o = ((oz + R) * L + (oy + R)) * L + (ox + R);
                            Cout[((size_t)(z - tbox[4]) * tby + (y - tbox[2])) * tbx + (x - tbox[0])] +=
                                Ws[o] * cs;
                        }
            }
    (void)sbz;
}

/* O4 with OpenMP, for timing on all host cores: the same scatter, the target
 * planes split between threads; each thread walks ALL sources in ascending order and adds
 * only into its own planes, so every target receives its terms in exactly the sequential
 * order above (bitwise the same result, pinned in tests/test_oracle_pins.py). */
void oracle_step_scatter_omp(const oracle_params* p, const double* W, const int32_t* sbox,
                             const double* Cold, const int32_t* tbox, double* Cout)
{
    const int R = p->R, L = 2 * R + 1, K = L * L * L;
    const int sbx = sbox[1] - sbox[0], sby = sbox[3] - sbox[2];
    const int tbx = tbox[1] - tbox[0], tby = tbox[3] - tbox[2], tbz = tbox[5] - tbox[4];
    memset(Cout, 0, sizeof(double) * (size_t)tbx * tby * tbz);
#pragma omp parallel for schedule(static, 1)
    for (int tz = tbox[4]; tz < tbox[5]; ++tz)
        for (int sz = sbox[4]; sz < sbox[5]; ++sz) {
            if (tz - sz < -R || tz - sz > R) continue;
            const int oz = tz - sz;
            for (int sy = sbox[2]; sy < sbox[3]; ++sy)
                for (int sx = sbox[0]; sx < sbox[1]; ++sx) {
                    size_t n = ((size_t)(sz - sbox[4]) * sby + (sy - sbox[2])) * sbx + (sx - sbox[0]);
                    const double* Ws = W + n * K;
                    double cs = Cold[((size_t)sz * p->ny + sy) * p->nx + sx];
                    for (int oy = -R; oy <= R; ++oy)
                        for (int ox = -R; ox <= R; ++ox) {
                            int x = sx + ox, y = sy + oy;
                            if (x < tbox[0] || x >= tbox[1] || y < tbox[2] || y >= tbox[3]) continue;
                            int o = ((oz + R) * L + (oy + R)) * L + (ox + R);
                            Cout[((size_t)(tz - tbox[4]) * tby + (y - tbox[2])) * tbx + (x - tbox[0])] +=
                                Ws[o] * cs;
                        }
                }
        }
}

/* ---------------------------------------------------------------------------
 * a4 (oracle form O5). Reduced-precision weight storage (§3.3: "The
 * coefficient matrix P is stored in FP16 precision"; reading A9: weights only,
 * fp32 accumulate; reading A10: fp32 diagonal fix-up for mass conservation, the
 * role Eq.7 plays in the paper).  IEEE 754 round-to-nearest-even (ref 26,
 * P:151; A11).
 *   for o ≠ centre:  Wq[o] = RNE_fmt( RNE_fp32( W[o] ) )
 *   d               = M − Σ_{o≠centre, ascending o} Wq[o]               (fp64 sum)
 *   diag            = d_hi + d_lo,  d_hi = RNE_fp32(d),  d_lo = RNE_fp32(d − d_hi)
 *   (reading A10 as revised in round 2: the diagonal is stored as an fp32 PAIR, so a column
 *   sums to M within ~2^-48 instead of half an fp32 ulp; one fp32 diagonal rounded the same
 *   way for every member of a large class of identical windows, which biased the total
 *   mass by ~1e-8 per step on long runs)
 *   M = 1 for a closed window (Σ_o W = 1, reading A2); with a far field (N2) the
 *   kernel keeps M = Σ_o W (ascending o) and the rest went to the reservoir
 *   (mass_fix = 0:  diag = RNE_fmt(RNE_fp32(W[centre])))
 * Wq[centre] ← diag, so oracle_step_scatter applies the stored operator.
 * fmt: 0 fp32, 1 fp16 (binary16), 2 bf16.
 * ------------------------------------------------------------------------- */
static uint32_t f32_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* binary32 -> binary16, round to nearest, ties to even; subnormals; overflow -> inf */
uint16_t oracle_f32_to_f16(float f)
{
    uint32_t u = f32_bits(f);
    uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
    uint32_t exp = (u >> 23) & 0xFFu, man = u & 0x7FFFFFu;
    if (exp == 0xFFu) return (uint16_t)(sign | 0x7C00u | (man ? 0x200u : 0u)); /* inf / qNaN */
    int e = (int)exp - 127;                  /* unbiased exponent */
    if (e > 15) return (uint16_t)(sign | 0x7C00u);
    if (exp == 0) return sign;               /* fp32 subnormals are far below fp16's range */
    uint32_t m = man | 0x800000u;            /* 24-bit significand, value = m·2^(e-23) */
    int shift;                               /* bits to drop from m */
    uint32_t base;
    if (e >= -14) { shift = 13; base = (uint32_t)(e + 15) << 10; m &= 0x7FFFFFu; }
    else {                                   /* fp16 subnormal: value = q·2^-24 */
        shift = -e - 1;                      /* m·2^(e-23) / 2^-24 = m >> (-(e+1)) */
        if (shift > 24) return sign;
        base = 0;
    }
    uint32_t q = m >> shift;
    uint32_t rem = m & ((1u << shift) - 1u);
    uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) q += 1u;
    uint32_t h = base + q;                   /* a carry into the exponent is the right result */
    if (h >= 0x7C00u) h = 0x7C00u;
    return (uint16_t)(sign | h);
}

double oracle_f16_to_f64(uint16_t h)
{
    int s = (h >> 15) & 1, e = (h >> 10) & 0x1F, m = h & 0x3FF;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(m | 0x400), e - 25);
    return s ? -v : v;
}

/* binary32 -> bfloat16 (8-bit exponent, 7-bit mantissa), RNE */
uint16_t oracle_f32_to_bf16(float f)
{
    uint32_t u = f32_bits(f);
    if (((u >> 23) & 0xFFu) == 0xFFu) return (uint16_t)((u >> 16) | ((u & 0x7FFFFFu) ? 0x40u : 0u));
    uint32_t keep = u >> 16, rem = u & 0xFFFFu;
    if (rem > 0x8000u || (rem == 0x8000u && (keep & 1u))) keep += 1u;
    return (uint16_t)keep;
}

double oracle_bf16_to_f64(uint16_t b) { return (double)bits_f32((uint32_t)b << 16); }

double oracle_round_fmt(double w, int fmt)
{
    float f = (float)w; /* C99 6.3.1.5: conversion under the default rounding mode = RNE */
    if (fmt == 1) return oracle_f16_to_f64(oracle_f32_to_f16(f));
    if (fmt == 2) return oracle_bf16_to_f64(oracle_f32_to_bf16(f));
    return (double)f;
}

void oracle_quantize(const oracle_params* p, const double* W, long nsrc, int fmt, int mass_fix, double* Wq,
                     const uint8_t* open_window)
{
    const int L = 2 * p->R + 1, K = L * L * L, c = K / 2;
    for (long n = 0; n < nsrc; ++n) {
        const double* w = W + (size_t)n * K;
        double* q = Wq + (size_t)n * K;
        double M = 1.0, sum = 0.0;
        if (open_window && open_window[n]) {
            M = 0.0;
            for (int o = 0; o < K; ++o) M += w[o];
        }
        for (int o = 0; o < K; ++o) {
            if (o == c) continue;
            q[o] = oracle_round_fmt(w[o], fmt);
            sum += q[o];
        }
        if (mass_fix) {
            const double d = M - sum;
            const float hi = (float)d, lo = (float)(d - (double)hi);
            q[c] = (double)hi + (double)lo;
        } else {
            q[c] = oracle_round_fmt(w[c], fmt);
        }
    }
}

/* ---------------------------------------------------------------------------
 * O6. Whole-grid explicit FD (the paper's fine-mesh FD solver, §4.1,
 * as a brute-force reference): the same 7-point Jacobi update as
 * oracle_kernel, on the whole closed domain, for nsub substeps.  Far-field
 * cells (mask 2, N2) are held at c_far (Dirichlet, P:76 / SPEC S:190).
 * ------------------------------------------------------------------------- */
void oracle_fd_whole_grid(const oracle_params* p, const oracle_derived* d, const uint8_t* mask,
                          const double* C0, int nsub, double c_far, double* Cout)
{
    const int nx = p->nx, ny = p->ny, nz = p->nz;
    const size_t N = (size_t)nx * ny * nz;
    double* cur = (double*)malloc(N * sizeof(double));
    double* nxt = (double*)malloc(N * sizeof(double));
    memcpy(cur, C0, N * sizeof(double));
    for (size_t i = 0; i < N; ++i)
        if (mask[i] == 2) cur[i] = c_far;
    static const int DX[6] = {-1, 1, 0, 0, 0, 0}, DY[6] = {0, 0, -1, 1, 0, 0}, DZ[6] = {0, 0, 0, 0, -1, 1};
    for (int k = 0; k < nsub; ++k) {
#pragma omp parallel for
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    size_t i = ((size_t)z * ny + y) * nx + x;
                    if (mask[i] == 2) { nxt[i] = c_far; continue; }
                    double acc = cur[i];
                    for (int f = 0; f < 6; ++f) {
                        int qx = x + DX[f], qy = y + DY[f], qz = z + DZ[f];
                        if (qx < 0 || qx >= nx || qy < 0 || qy >= ny || qz < 0 || qz >= nz) continue;
                        size_t j = ((size_t)qz * ny + qy) * nx + qx;
                        acc += face_lambda(d, mask[i], mask[j]) * (cur[j] - cur[i]);
                    }
                    nxt[i] = acc;
                }
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(Cout, cur, N * sizeof(double));
    free(cur); free(nxt);
}

/* O7. Metrics: relL2 = ||g−o||₂/||o||₂ and sums, accumulated in fp64. */
double oracle_rel_l2(const double* g, const double* o, long n)
{
    double num = 0.0, den = 0.0;
    for (long i = 0; i < n; ++i) { double e = g[i] - o[i]; num += e * e; den += o[i] * o[i]; }
    return den > 0 ? sqrt(num / den) : sqrt(num);
}
