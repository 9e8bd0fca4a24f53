// fdirw_api.cu — the C ABI of include/fdirw.h: validation, parameter derivation (a1),
// memory plan, kernel generation driver (a2-a4), step / run loop with CUDA graphs
// (a5-a7), NCCL slab exchange (a6) and test-support entry points.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "fdirw_internal.h"
#include "layout.cuh"

using namespace fdirw;

// device bytes of `elems` stored weights (elems is a multiple of 8: whole gather blocks)
static size_t wbytes(int fmt, size_t elems)
{
    return fmt == FDIRW_W_FP32 ? elems * 4 : fmt == FDIRW_W_MX8 ? elems / 8 * 9 : elems * 2;
}

struct fdirw_ctx {
    fdirw_params p;
    Derived d;
    Geometry g;
    int rank = 0, world = 1, device = 0;
    bool is_virtual = false;
    int fmt = 0, b_w = 4;
    void* Wt = nullptr;
    float2* diag = nullptr;       // fp32 pair (hi, lo) per target (reading A10)
    float* cpad[2] = {nullptr, nullptr};
    double* mass_partial = nullptr;
    double* mass_out = nullptr;
    int mass_blocks = 0;
    cudaStream_t comm_stream = nullptr, capture_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_comm = nullptr;
    cudaGraphExec_t graph2 = nullptr;
    Nccl* nccl = nullptr;
    void* comm = nullptr;
    uint64_t kgen_sources = 0, kgen_windows = 0;
    int kgen_steps = 0;  // stencil passes per window: Chebyshev degree m, or n_fd (direct)
    bool no_bulk = false;  // FDIRW_F_NO_BULK_STREAM
    float* cheb_d = nullptr;  // kgen's Chebyshev coefficients (build only)
    cudaEvent_t kev[2] = {nullptr, nullptr};
    float kgen_ms = 0.f;      // device time of the kgen launch (CUDA events on the build stream)
    // N4 uniform-chunk weight dedup (FDIRW_F_DEDUP_STORAGE)
    UniformTables ut;
    // N2 far field
    bool far = false;
    double v_far = 0.0;
    uint8_t* farmask = nullptr;   // slab planes [z0, z1): 1 = far-field voxel
    float* pbc = nullptr;         // p_BC in the diag layout
    double* tile_buf = nullptr;   // [tile_stride]: n_tiles, then per-tile Σ C_new
    double* gathered = nullptr;   // [world · tile_stride] (NCCL all-gather target)
    double* far_state = nullptr;  // {c_far, M0}
    long tile_stride = 0;
    // N2, world == 1: chunks whose 8 targets are all far-field voxels get no gather weights;
    // Wt / diag / p_BC hold the other chunks compacted (ut.dense_list), chunk_pos maps a
    // chunk (tile·tile + e) to its compact position or −1
    bool compact = false;
    int* chunk_pos = nullptr;
    // ... and with D_slow = 0 (the N3 loop's liquid step) chunks whose non-far
    // targets are all solid: those rows are the identity (W_s = δ for an isolated solid source,
    // no liquid source reaches a solid target, diag = 1, p_BC = 0), so they carry no weights
    // either and the step copies C_old → C_new for them (chunk_pos −2)
    int* ident_list = nullptr;
    long n_ident = 0;
    // N3 integrated loop / precision modes (world == 1)
    int prec_mode = 0;            // 0 = default kernel; 1/2/3 = §3.3 study modes (absorb.cu)
    uint8_t* phase_pp = nullptr;  // padded phase map (255 outside)
    float* alpha = nullptr;       // padded scratch for the reaction clamp
    double* kin_part = nullptr;   // 4·kAbsorbMaxBlocks doubles: sweep partials, interface partials
    IfaceList iface;              // built on the first fdirw_absorb_run
    double* kin_rec = nullptr;
    int kin_cap = 0;
    // N3 loop replay: two macro steps captured once (graph_abs), the kinetics record slot taken
    // from a device counter; recaptured when the loop's parameters or record buffer change
    cudaGraphExec_t graph_abs = nullptr;
    int* abs_ctr = nullptr;
    AbsorbArgs abs_key{};
    const double* abs_rec_key = nullptr;
    double n_solid = 0;
    // a6 over peer memory (FDIRW_TRANSPORT_P2P)
    int transport = FDIRW_TRANSPORT_NCCL;
    unsigned long long* p2p_flags = nullptr;   // [4]: from lo, from hi, own epoch, timed out
    float* peer_lo[2] = {nullptr, nullptr};    // the neighbours' padded state buffers
    float* peer_hi[2] = {nullptr, nullptr};
    unsigned long long* peer_lo_flag = nullptr;  // lo neighbour's flags[1]
    unsigned long long* peer_hi_flag = nullptr;  // hi neighbour's flags[0]
    int nzl_lo = 0;
    bool p2p_ready = false;
    std::vector<void*> ipc_opened;
    // fdirw_step_host: device staging of the caller's host slab (allocated on first use)
    float* host_stage[2] = {nullptr, nullptr};
    unsigned long long* canary = nullptr;  // fdirw_debug_stage_canary: {checks, mismatches}
    // fdirw_step_host's plane-chunk pipeline (world 1, dense closed path): copy streams and
    // per-chunk events, created on first use
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    std::vector<cudaEvent_t> hx_ev;  // [3·nch + 1]: H2D done, step done, D2H done per chunk, start
};

static fdirw_status build_pbc(fdirw_ctx* c, const uint8_t* mask_d, cudaStream_t s);
static cudaError_t virtual_gather(fdirw_ctx* const* ctxs, int n, cudaStream_t s, int mode, double c_far0);

static thread_local std::string g_err;

static fdirw_status fail(fdirw_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

namespace fdirw {
const char* coarse_set_error(const std::string& m)  // coarse.cu shares the thread-local message
{
    g_err = m;
    return g_err.c_str();
}
}  // namespace fdirw

#define CUDA_TRY(call)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(FDIRW_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

namespace fdirw {

Geometry make_geometry(int nx, int ny, int nz, int R, int z0, int z1, bool balance)
{
    Geometry g{};
    g.nx = nx; g.ny = ny; g.nz = nz; g.R = R;
    g.L = 2 * R + 1;
    g.K = g.L * g.L * g.L;
    g.z0 = z0; g.z1 = z1; g.nzl = z1 - z0;
    g.nxq = (nx + kChunk - 1) / kChunk;
    g.cpp = ny * g.nxq;
    int tile = ((g.cpp + 31) / 32) * 32;
    g.tile = tile > 256 ? 256 : tile;
    if (balance && g.tile == 256) {
        // Wave balance for slabs of a few waves (strong scaling: 192³ over 8 ranks is 432 tiles
        // of 256 chunks = 1.46 waves of the 296 CTAs a B200 runs at once, measured 0.92 of the
        // ideal per-rank time): among tiles of 256, 224, 192, 160 or 128 chunks take the one
        // whose model time waves·tile is least (ties: the larger tile).  Only for launches of
        // < 4 waves; results do not depend on the tiling (each target is one thread's sum).
        const long slots = 2L * 148;
        long best_t = 256, best_cost = -1;
        const long n256 = (long)g.nzl * ((g.cpp + 255) / 256);
        if (n256 < 4 * slots) {
            for (int t = 256; t >= 128; t -= 32) {
                const long n = (long)g.nzl * ((g.cpp + t - 1) / t);
                const long cost = ((n + slots - 1) / slots) * t;
                if (best_cost < 0 || cost < best_cost) { best_cost = cost; best_t = t; }
            }
            g.tile = (int)best_t;
        }
    }
    g.tpp = (g.cpp + g.tile - 1) / g.tile;
    g.n_tiles = g.nzl * g.tpp;
    g.nxp = g.nxq * kChunk + 2 * kPadX;
    g.nyp = ny + 2 * R;
    g.nzp = g.nzl + 2 * R;
    g.plane_elems = (size_t)g.nyp * g.nxp;
    g.state_elems = (size_t)g.nzp * g.plane_elems;
    g.w_elems = (size_t)g.n_tiles * (g.K - 1) * g.tile * kChunk;
    g.diag_elems = (size_t)g.n_tiles * g.tile * kChunk;
    g.mz0 = z0 - 2 * R < 0 ? 0 : z0 - 2 * R;
    g.mz1 = z1 + 2 * R > nz ? nz : z1 + 2 * R;
    g.sz0 = z0 - R < 0 ? 0 : z0 - R;
    g.sz1 = z1 + R > nz ? nz : z1 + R;
    return g;
}

HaloPlan make_halo_plan(const Geometry& g, int rank, int world)
{
    HaloPlan h{};
    h.count = (long)g.R * (long)g.plane_elems;
    h.peer_lo = rank > 0 ? rank - 1 : -1;
    h.peer_hi = rank < world - 1 ? rank + 1 : -1;
    h.send_lo = h.peer_lo >= 0 ? (long)g.R * (long)g.plane_elems : -1;
    h.recv_lo = h.peer_lo >= 0 ? 0 : -1;
    h.send_hi = h.peer_hi >= 0 ? (long)g.nzl * (long)g.plane_elems : -1;
    h.recv_hi = h.peer_hi >= 0 ? (long)(g.nzl + g.R) * (long)g.plane_elems : -1;
    return h;
}

}  // namespace fdirw

// a1: n_fd = ceil(x·(1 − 1e-9)), x = D_max·Δt/(λ*·Δh²), λ* = 0.1 (Table 1, P:84-91;
// reading A5); face numbers λ = Δt_fd·D/Δh² with the harmonic mean across phases (A4).
static fdirw_status derive(const fdirw_params& p, Derived* d)
{
    const double dmax = p.D_fast > p.D_slow ? p.D_fast : p.D_slow;
    long n = p.n_fd;
    if (n == 0) {
        const double x = dmax * p.dt / (0.1 * p.dh * p.dh);
        const double c = std::ceil(x * (1.0 - 1e-9));
        if (!(c < 2.0e9)) return fail(FDIRW_E_INVALID, "derived n_fd too large (" + std::to_string(c) + ")");
        n = c < 1.0 ? 1 : (long)c;
    }
    d->n_fd = (int)n;
    d->dt_fd = p.dt / (double)n;
    const double s = d->dt_fd / (p.dh * p.dh);
    const double hm = (p.D_fast + p.D_slow) == 0.0 ? 0.0 : 2.0 * p.D_fast * p.D_slow / (p.D_fast + p.D_slow);
    d->lam_ff = s * p.D_fast;
    d->lam_ss = s * p.D_slow;
    d->lam_fs = s * hm;
    if (d->lam_ff > 1.0 / 6.0 || d->lam_ss > 1.0 / 6.0) {
        char buf[160];
        snprintf(buf, sizeof buf, "explicit FD unstable: lambda_max = %.6g > 1/6 (n_fd = %d)",
                 d->lam_ff > d->lam_ss ? d->lam_ff : d->lam_ss, d->n_fd);
        return fail(FDIRW_E_UNSTABLE, buf);
    }
    return FDIRW_OK;
}

// Chebyshev plan for kgen (reading A30).  Every window operator A (7-point
// stencil, symmetric face numbers λ_ij, no-flux or absorbing edges) is symmetric with its
// spectrum in [a, 1], a = 1 − 12·λ_max (Gershgorin: centre 1 − Λ_i, radius ≤ Λ_i ≤ 6λ_max).
// With x = αy + β (α = 6λ_max, β = 1 − 6λ_max), x^n = Σ_k c_k T_k(y) where every c_k ≥ 0
// (binomial expansion in y, and y^j's Chebyshev coefficients are ≥ 0) and Σ_k c_k = 1^n = 1,
// so |x^n − Σ_{k≤m} c_k T_k(y)| ≤ 1 − Σ_{k≤m} c_k on [a, 1] and, A being symmetric,
// ‖p_m(A)δ − A^n δ‖₂ ≤ that tail.  The c_k come from an M-point discrete Chebyshev
// transform of x^n (fp64; aliasing is below the tail once M ≥ 4m).  Returns m (0 = the
// recurrence would not save work: keep the n_fd direct substeps).
int fdirw::cheb_plan(int n, double lam_max, std::vector<float>* coef)
{
    const double tol = 1e-10;
    const int kmax = 2048;  // coefficients live in the kgen CTA's shared memory
    if (n < 8 || !(lam_max > 0)) return 0;
    const double al = 6.0 * lam_max, be = 1.0 - 6.0 * lam_max;
    const int kk = n < kmax ? n : kmax;
    const int M = 4 * kk + 64;
    std::vector<double> f(M), th(M);
    for (int j = 0; j < M; ++j) {
        th[j] = M_PI * (j + 0.5) / M;
        f[j] = std::pow(al * std::cos(th[j]) + be, (double)n);
    }
    std::vector<double> c;
    double sum = 0.0;
    int m = -1;
    for (int k = 0; k <= kk; ++k) {
        double v = 0.0;
        for (int j = 0; j < M; ++j) v += f[j] * std::cos(k * th[j]);
        v *= (k == 0 ? 1.0 : 2.0) / M;
        c.push_back(v);
        sum += v;
        if (1.0 - sum <= tol) { m = k; break; }
    }
    // one pass costs the direct substep + 2 FMA (14 vs 12 lane-ops, same shared-memory traffic)
    if (m < 1 || 14.0 * m > 0.8 * 12.0 * n) return 0;
    coef->assign(c.begin(), c.end());
    return m;
}

// kgen's plan for these params: kCheb_pre direct substeps first (the peaked start: its entries
// of size ~1 would otherwise enter the recurrence and its rounding), then the Chebyshev degree
// for the remaining n_fd − kCheb_pre.  Returns that degree (0 = all n_fd substeps direct).
static int kgen_cheb(const fdirw_params& p, const Derived& d, std::vector<float>* coef)
{
    if (p.flags & (FDIRW_F_KGEN_FP64 | FDIRW_F_KGEN_DIRECT)) return 0;
    if (d.n_fd <= 2 * kCheb_pre) return 0;
    return cheb_plan(d.n_fd - kCheb_pre, std::max(d.lam_ff, std::max(d.lam_fs, d.lam_ss)), coef);
}

// NVTX ranges (header-only nvtx3: no-ops unless a profiler injects a tool) around the
// C-ABI's entry points, so a timeline shows the build phases and the steps by name.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// FDIRW_TRACE=1: host-side phase timings of fdirw_build_kernels on stderr (the stream is
// synchronised at each mark only when tracing, so an untraced build is unaffected).  Every
// mark is also an NVTX marker inside the "fdirw_build_kernels" range.
struct BuildTrace {
    bool on = getenv("FDIRW_TRACE") != nullptr;
    cudaStream_t s = nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), t = t0;
    NvtxRange range{"fdirw_build_kernels"};
    void mark(const char* what)
    {
        nvtxMarkA(what);
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "fdirw trace: build %-22s %9.2f ms  (total %9.2f ms)\n", what,
                std::chrono::duration<double, std::milli>(n - t).count(),
                std::chrono::duration<double, std::milli>(n - t0).count());
        t = n;
    }
};

static fdirw_status validate(const fdirw_params* p, const uint8_t* phase, const fdirw_dist* dist,
                             fdirw_ctx** out, bool scan_phase = true)
{
    if (!p || !phase || !out) return fail(FDIRW_E_INVALID, "NULL argument");
    if (p->nx < 1 || p->ny < 1 || p->nz < 1) return fail(FDIRW_E_INVALID, "grid dims must be >= 1");
    if (p->radius < 1 || p->radius > kMaxR) return fail(FDIRW_E_INVALID, "radius must be in [1, 8]");
    if (!(p->dh > 0) || !(p->dt > 0)) return fail(FDIRW_E_INVALID, "dh and dt must be > 0");
    if (!(p->D_fast > 0) || !(p->D_slow >= 0)) return fail(FDIRW_E_INVALID, "need D_fast > 0, D_slow >= 0");
    if (p->n_fd < 0) return fail(FDIRW_E_INVALID, "n_fd must be >= 0");
    if (p->weights < 0 || p->weights > 3) return fail(FDIRW_E_INVALID, "weights must be FP32, FP16, BF16 or MX8");
    if (p->weights == FDIRW_W_MX8) {
        if (p->flags & (FDIRW_F_NO_MASS_FIX | FDIRW_F_NO_DEDUP | FDIRW_F_SYMMETRIC_RULE | FDIRW_F_KGEN_FP64))
            return fail(FDIRW_E_INVALID, "MX8 weights are not combined with NO_MASS_FIX, NO_DEDUP, SYMMETRIC_RULE or "
                                         "KGEN_FP64");
    }
    if (p->flags & ~(FDIRW_F_NO_MASS_FIX | FDIRW_F_NO_DEDUP | FDIRW_F_DEDUP_STORAGE | FDIRW_F_KGEN_FP64 |
                     FDIRW_F_SYMMETRIC_RULE | FDIRW_F_KGEN_DIRECT | FDIRW_F_NO_BULK_STREAM | FDIRW_F_KGEN_COLUMNS |
                     FDIRW_F_PBC_RESERVOIR))
        return fail(FDIRW_E_INVALID, "unknown flags");
    if ((p->flags & FDIRW_F_PBC_RESERVOIR) && p->v_far > 0 && dist && dist->world > 1)
        return fail(FDIRW_E_INVALID, "FDIRW_F_PBC_RESERVOIR needs world == 1 (the reservoir FD spans the whole grid)");
    if ((p->flags & FDIRW_F_SYMMETRIC_RULE) && (p->flags & FDIRW_F_DEDUP_STORAGE))
        return fail(FDIRW_E_INVALID, "FDIRW_F_SYMMETRIC_RULE is not combined with FDIRW_F_DEDUP_STORAGE");
    if ((p->flags & FDIRW_F_NO_DEDUP) && (p->flags & FDIRW_F_DEDUP_STORAGE))
        return fail(FDIRW_E_INVALID, "FDIRW_F_DEDUP_STORAGE needs the window de-duplication");
    if (!(p->v_far >= 0)) return fail(FDIRW_E_INVALID, "v_far must be >= 0");
    if (dist && dist->world > 1 && (p->flags & FDIRW_F_DEDUP_STORAGE))
        return fail(FDIRW_E_INVALID, "FDIRW_F_DEDUP_STORAGE needs world == 1");
    if (p->v_far > 0 && (p->flags & FDIRW_F_DEDUP_STORAGE))
        return fail(FDIRW_E_INVALID, "FDIRW_F_DEDUP_STORAGE is not combined with a far field (v_far > 0)");
    if (scan_phase) {
        const size_t n = (size_t)p->nx * p->ny * p->nz;
        uint8_t mx = 0;
        for (size_t i = 0; i < n; ++i) mx = phase[i] > mx ? phase[i] : mx;
        if (mx > 2) return fail(FDIRW_E_INVALID, "phase values must be 0 (slow), 1 (fast) or 2 (far field)");
        if (mx == 2 && !(p->v_far > 0)) return fail(FDIRW_E_INVALID, "far-field voxels (2) need v_far > 0");
    }
    if ((long long)p->nx * p->ny * p->nz > (1LL << 40)) return fail(FDIRW_E_INVALID, "grid too large");
    {   // the window dedup (CUB sorts/scans, int source ids) and the N3 loop index the voxels of
        // one rank's mask planes [z_begin − 2R, z_end + 2R) with 32-bit ints
        const int zb = dist ? dist->z_begin : 0, ze = dist ? dist->z_end : p->nz;
        const long long planes = (long long)std::min(p->nz, ze + 2 * p->radius) - std::max(0, zb - 2 * p->radius);
        if ((long long)p->nx * p->ny * planes >= (1LL << 31))
            return fail(FDIRW_E_INVALID, "slab too large: nx*ny*(mask planes of the slab) must be < 2^31 voxels "
                                         "(split the grid over more ranks)");
    }
    if (dist) {
        if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)
            return fail(FDIRW_E_INVALID, "bad rank/world");
        if (dist->transport != FDIRW_TRANSPORT_NCCL && dist->transport != FDIRW_TRANSPORT_P2P)
            return fail(FDIRW_E_INVALID, "transport must be FDIRW_TRANSPORT_NCCL or FDIRW_TRANSPORT_P2P");
        if (dist->transport == FDIRW_TRANSPORT_P2P && p->v_far > 0)
            return fail(FDIRW_E_INVALID, "FDIRW_TRANSPORT_P2P supports the closed domain only (v_far == 0)");
        if (dist->z_begin < 0 || dist->z_end > p->nz || dist->z_begin >= dist->z_end)
            return fail(FDIRW_E_INVALID, "bad slab [z_begin, z_end)");
        if (dist->world == 1 && (dist->z_begin != 0 || dist->z_end != p->nz))
            return fail(FDIRW_E_INVALID, "world == 1 must own [0, nz)");
        if (dist->world > 1) {
            if (dist->z_end - dist->z_begin < p->radius)
                return fail(FDIRW_E_INVALID, "slab thinner than the window radius R");
            if (dist->rank == 0 && dist->z_begin != 0) return fail(FDIRW_E_INVALID, "rank 0 must start at z = 0");
            if (dist->rank == dist->world - 1 && dist->z_end != p->nz)
                return fail(FDIRW_E_INVALID, "last rank must end at z = nz");
        }
    }
    return FDIRW_OK;
}

static void free_ctx(fdirw_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->graph2) cudaGraphExecDestroy(c->graph2);
    cudaFree(c->cheb_d);
    for (cudaEvent_t e : c->kev)
        if (e) cudaEventDestroy(e);
    if (c->comm) nccl_comm_destroy(c->nccl, c->comm);
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    cudaFree(c->p2p_flags);
    cudaFree(c->Wt);
    cudaFree(c->diag);
    cudaFree(c->cpad[0]);
    cudaFree(c->cpad[1]);
    cudaFree(c->host_stage[0]);
    cudaFree(c->host_stage[1]);
    cudaFree(c->canary);
    for (cudaEvent_t e : c->hx_ev)
        if (e) cudaEventDestroy(e);
    if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    cudaFree(c->mass_partial);
    cudaFree(c->mass_out);
    cudaFree(c->farmask);
    cudaFree(c->pbc);
    cudaFree(c->tile_buf);
    cudaFree(c->gathered);
    cudaFree(c->far_state);
    cudaFree(c->chunk_pos);
    cudaFree(c->ident_list);
    cudaFree(c->phase_pp);
    cudaFree(c->alpha);
    cudaFree(c->kin_part);
    cudaFree(c->iface.list);
    cudaFree(c->iface.tmp);
    cudaFree(c->iface.nf_list);
    cudaFree(c->kin_rec);
    cudaFree(c->abs_ctr);
    if (c->graph_abs) cudaGraphExecDestroy(c->graph_abs);
    cudaFree(c->ut.chunk_u);
    cudaFree(c->ut.dense_list);
    cudaFree(c->ut.ukf);
    cudaFree(c->ut.udiag);
    cudaFree(c->ut.list);
    cudaFree(c->ut.blocks);
    cudaFree(c->ut.udiag_t);
    cudaFree(c->ut.chunk_map);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_comm) cudaEventDestroy(c->ev_comm);
    delete c;
}

static fdirw_status alloc(void** ptr, size_t bytes, const char* what)
{
    cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 16);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        char buf[200];
        snprintf(buf, sizeof buf, "out of device memory allocating %s: %zu bytes required, %zu free", what, bytes, fr);
        return fail(FDIRW_E_OOM, buf);
    }
    if (e != cudaSuccess) return fail(FDIRW_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_nccl_unique_id(void* out128)
{
    if (!out128) return fail(FDIRW_E_INVALID, "NULL argument");
    std::string err;
    Nccl* n = nccl_load(&err);
    if (!n) return fail(FDIRW_E_NCCL, err);
    if (nccl_unique_id(n, out128, &err)) return fail(FDIRW_E_NCCL, err);
    return FDIRW_OK;
}

// N2 (world == 1): list the chunks (tile·tile + e, ascending) holding at least one non-far
// target; the rest carry no weights.  With D_slow = 0, chunks whose non-far targets are all
// solid are identity rows: listed apart (ident_list, chunk_pos −2), no weights either.
// Fills c->ut.{dense_list, n_dense, nd_tiles}, chunk_pos, ident_list.
static fdirw_status far_compact(fdirw_ctx* c, const uint8_t* phase_host, cudaStream_t s)
{
    const Geometry& g = c->g;
    const size_t nch = (size_t)g.n_tiles * g.tile;
    const bool ident = c->p.D_slow == 0.0;
    std::vector<int> pos(nch, -1), list, idl;
    list.reserve(nch);
    for (int zl = 0; zl < g.nzl; ++zl)
        for (int q = 0; q < g.ny * g.nxq; ++q) {
            const int y = q / g.nxq, x0 = (q % g.nxq) * 8;
            const uint8_t* row = phase_host + ((size_t)(g.z0 + zl) * g.ny + y) * g.nx;
            bool any = false, liquid = false;
            for (int j = 0; j < 8 && x0 + j < g.nx; ++j) {
                any |= row[x0 + j] != 2;
                liquid |= row[x0 + j] == 1;
            }
            if (!any) continue;
            const int ch = (zl * g.tpp + q / g.tile) * g.tile + q % g.tile;
            if (ident && !liquid) {
                pos[ch] = -2;
                idl.push_back(ch);
                continue;
            }
            pos[ch] = (int)list.size();
            list.push_back(ch);
        }
    fdirw_status st;
    if (!idl.empty()) {
        if ((st = alloc((void**)&c->ident_list, idl.size() * 4, "identity chunks")) != FDIRW_OK) return st;
        CUDA_TRY(cudaMemcpyAsync(c->ident_list, idl.data(), idl.size() * 4, cudaMemcpyHostToDevice, s));
        c->n_ident = (long)idl.size();
    }
    if ((st = alloc((void**)&c->ut.dense_list, (list.size() + 1) * 4, "far compaction list")) != FDIRW_OK) return st;
    if ((st = alloc((void**)&c->chunk_pos, nch * 4, "far compaction map")) != FDIRW_OK) return st;
    if (!list.empty()) CUDA_TRY(cudaMemcpyAsync(c->ut.dense_list, list.data(), list.size() * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->chunk_pos, pos.data(), nch * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->ut.n_dense = (long)list.size();
    c->ut.nd_tiles = (int)((list.size() + g.tile - 1) / g.tile);
    c->compact = true;
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_build_kernels(const fdirw_params* params, const uint8_t* phase_host,
                                            const fdirw_dist* dist, void* cuda_stream, fdirw_ctx** out)
{
    BuildTrace tr;
    fdirw_status st = validate(params, phase_host, dist, out);
    if (st != FDIRW_OK) return st;
    *out = nullptr;
    tr.mark("validate");
    Derived d;
    if ((st = derive(*params, &d)) != FDIRW_OK) return st;
    if ((params->flags & FDIRW_F_SYMMETRIC_RULE) && d.n_fd > params->radius)
        return fail(FDIRW_E_INVALID, "FDIRW_F_SYMMETRIC_RULE needs the exact regime n_fd <= R (reading A24); n_fd = " +
                                         std::to_string(d.n_fd));

    fdirw_ctx* c = new fdirw_ctx();
    c->p = *params;
    c->d = d;
    c->fmt = params->weights;
    c->b_w = c->fmt == FDIRW_W_FP32 ? 4 : 2;  // MX8: the fp32 class kernels it quantises
    if (c->fmt == FDIRW_W_MX8) c->b_w = 4;
    int z0 = 0, z1 = params->nz;
    if (dist) {
        c->rank = dist->rank;
        c->world = dist->world;
        c->device = dist->device;
        z0 = dist->z_begin;
        z1 = dist->z_end;
        c->transport = dist->transport;
        c->is_virtual = dist->world > 1 && dist->nccl_id == nullptr && dist->transport == FDIRW_TRANSPORT_NCCL;
        if (cudaSetDevice(c->device) != cudaSuccess) {
            delete c;
            return fail(FDIRW_E_INVALID, "cudaSetDevice failed for dist->device");
        }
    } else {
        cudaGetDevice(&c->device);
    }
    c->g = make_geometry(params->nx, params->ny, params->nz, params->radius, z0, z1,
                         !(params->flags & FDIRW_F_DEDUP_STORAGE) && !(params->v_far > 0) &&
                             params->weights != FDIRW_W_MX8);  // MX8: tile 256, waves via stages
    const Geometry& g = c->g;
    if (params->weights == FDIRW_W_MX8 && (params->flags & FDIRW_F_DEDUP_STORAGE) && g.tile != 256) {
        // the small-tile N4 path sums uniform chunks with the bf16 body's grouping, not the MX8
        // body's: the field would no longer be bitwise the dense MX8 field
        delete c;
        return fail(FDIRW_E_INVALID, "MX8 weights with FDIRW_F_DEDUP_STORAGE need planes of >= 256 x-chunks "
                                     "(ny * ceil(nx/8) >= 256)");
    }
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    tr.s = s;

    auto bail = [&](fdirw_status e) {
        std::string keep = g_err;
        free_ctx(c);
        g_err = keep;
        return e;
    };
#define BAIL_CUDA(call)                                                                               \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) {                                                                      \
            g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                               \
            return bail(FDIRW_E_CUDA);                                                                \
        }                                                                                             \
    } while (0)

    // a2: mask planes [mz0, mz1) → device (the face number is a function of the two phases only)
    uint8_t* mask_d = nullptr;
    const size_t plane = (size_t)g.nx * g.ny;
    const size_t mbytes = (size_t)(g.mz1 - g.mz0) * plane;
    if ((st = alloc((void**)&mask_d, mbytes, "mask")) != FDIRW_OK) return bail(st);
    for (int i = 0; i < 2; ++i)
        if ((st = alloc((void**)&c->cpad[i], g.state_elems * 4, "state")) != FDIRW_OK) { cudaFree(mask_d); return bail(st); }
    c->mass_blocks = 148 * 4;
    if ((st = alloc((void**)&c->mass_partial, c->mass_blocks * 8, "mass")) != FDIRW_OK) { cudaFree(mask_d); return bail(st); }
    if ((st = alloc((void**)&c->mass_out, 8, "mass")) != FDIRW_OK) { cudaFree(mask_d); return bail(st); }

    BAIL_CUDA(cudaMemcpyAsync(mask_d, phase_host + (size_t)g.mz0 * plane, mbytes, cudaMemcpyHostToDevice, s));
    BAIL_CUDA(cudaMemsetAsync(c->cpad[0], 0, g.state_elems * 4, s));
    BAIL_CUDA(cudaMemsetAsync(c->cpad[1], 0, g.state_elems * 4, s));
    tr.mark("alloc state + mask");

    // a3 + a4
    KgenArgs ka{};
    ka.mask = mask_d;
    ka.mz0 = g.mz0;
    ka.nx = g.nx; ka.ny = g.ny; ka.nz = g.nz;
    ka.sz0 = g.sz0; ka.sz1 = g.sz1;
    ka.z0 = g.z0; ka.z1 = g.z1;
    ka.lam_ff = (float)d.lam_ff; ka.lam_fs = (float)d.lam_fs; ka.lam_ss = (float)d.lam_ss;
    ka.lam_d[0] = d.lam_ff; ka.lam_d[1] = d.lam_fs; ka.lam_d[2] = d.lam_ss;
    ka.fp64 = (params->flags & FDIRW_F_KGEN_FP64) ? 1 : 0;
    ka.symmetric = (params->flags & FDIRW_F_SYMMETRIC_RULE) ? 1 : 0;
    if (ka.symmetric) {  // every rank generates its own targets' kernels only: no halo sources
        ka.sz0 = g.z0;
        ka.sz1 = g.z1;
    }
    ka.n_fd = d.n_fd;
    c->kgen_steps = d.n_fd;
    c->no_bulk = (params->flags & FDIRW_F_NO_BULK_STREAM) != 0;
    std::vector<float> cheb;
    {
        const double lmax = std::max(d.lam_ff, std::max(d.lam_fs, d.lam_ss));
        const int m = kgen_cheb(*params, d, &cheb);
        if (m > 0) {
            if ((st = alloc((void**)&c->cheb_d, cheb.size() * 4, "chebyshev coefficients")) != FDIRW_OK) {
                cudaFree(mask_d);
                return bail(st);
            }
            BAIL_CUDA(cudaMemcpyAsync(c->cheb_d, cheb.data(), cheb.size() * 4, cudaMemcpyHostToDevice, s));
            const double sc = 4.0 / (12.0 * lmax);  // 2μ = 4λ/(1 − a), 1 − a = 12 λ_max
            ka.cheb_m = m;
            ka.cheb_pre = kCheb_pre;
            double p1 = 0.0;  // p(1) of the fp32 coefficients the passes use
            for (float ck : cheb) p1 += (double)ck;
            ka.cheb_scale = (float)(1.0 / p1);
            ka.cheb_c = c->cheb_d;
            ka.mu2_ff = (float)(d.lam_ff * sc);
            ka.mu2_fs = (float)(d.lam_fs * sc);
            ka.mu2_ss = (float)(d.lam_ss * sc);
            c->kgen_steps = kCheb_pre + m;
        }
    }
    ka.fmt = c->fmt == FDIRW_W_MX8 ? FDIRW_W_FP32 : c->fmt;  // MX8: quantised by the expand pass
    // open windows (N2) and the recurrence (reading A30): with fp32 storage they keep the literal
    // substeps (the recurrence's rounding, on the source's scale, would cost a near-empty window's
    // kept mass its fp32 accuracy); fp16 / bf16 / MX8 storage rounds every weight at 2^-11 … 2^-8
    // relative, far above that, so those windows take the recurrence too (FDIRW_KGEN_OPEN_LITERAL=1:
    // literal for A/B)
    ka.cheb_open = (c->fmt != FDIRW_W_FP32 && params->v_far > 0 && !getenv("FDIRW_KGEN_OPEN_LITERAL")) ? 1 : 0;
    ka.mass_fix = (params->flags & FDIRW_F_NO_MASS_FIX) ? 0 : 1;
    ka.columns = (params->flags & FDIRW_F_KGEN_COLUMNS) ? 1 : 0;
    ka.nxq = g.nxq; ka.tile = g.tile; ka.tpp = g.tpp; ka.K = g.K;
    c->kgen_sources = (uint64_t)g.nx * g.ny * (ka.sz1 - ka.sz0);
    c->kgen_windows = c->kgen_sources;
    // (the symmetric rule writes through the direct path: the expand kernel scatters forward)
    bool dedup = !(params->flags & (FDIRW_F_NO_DEDUP | FDIRW_F_SYMMETRIC_RULE));
    if (dedup) {
        // identical windows ⇒ identical kernels: compute each distinct window once (dedup.cu)
        int* class_pad = nullptr;
        void* class_w = nullptr;
        float2* class_diag = nullptr;
        double* class_mass = nullptr;  // MX8: each class kernel's own mass (N2 open windows < 1)
        DedupResult dr;
        auto dfree = [&]() {
            cudaFree(class_pad); cudaFree(class_w); cudaFree(class_diag); cudaFree(class_mass); cudaFree(dr.rep);
        };
        if ((st = alloc((void**)&class_pad, g.state_elems * 4, "class map")) != FDIRW_OK) { cudaFree(mask_d); return bail(st); }
        cudaError_t e = cudaMemsetAsync(class_pad, 0xff, g.state_elems * 4, s);
        DedupArgs da{mask_d, g.mz0, g.nx, g.ny, g.nz, g.R, g.sz0, g.sz1, g.z0, g.nxp, g.nyp, class_pad};
        if (e == cudaSuccess) e = dedup_classify(da, &dr, s);
        tr.mark("dedup classify");
        if (e != cudaSuccess) { dfree(); cudaFree(mask_d); g_err = std::string("dedup: ") + cudaGetErrorString(e); return bail(FDIRW_E_CUDA); }
        if (dr.collision) {
            dedup = false;  // hash collision detected by the exact check: take the direct path
        } else {
            if ((st = alloc(&class_w, (size_t)dr.n_class * g.K * c->b_w, "class kernels")) != FDIRW_OK ||
                (st = alloc((void**)&class_diag, (size_t)dr.n_class * 8, "class diagonal")) != FDIRW_OK ||
                (c->fmt == FDIRW_W_MX8 &&
                 (st = alloc((void**)&class_mass, (size_t)dr.n_class * 8, "class mass")) != FDIRW_OK)) {
                dfree(); cudaFree(mask_d); return bail(st);
            }
            ka.src_list = dr.rep;
            ka.n_list = dr.n_class;
            ka.class_w = class_w;
            ka.class_diag = class_diag;
            ka.class_mass = class_mass;
            if (e == cudaSuccess) e = cudaEventCreate(&c->kev[0]);
            if (e == cudaSuccess) e = cudaEventCreate(&c->kev[1]);
            if (e == cudaSuccess) e = cudaEventRecord(c->kev[0], s);
            if (e == cudaSuccess) e = launch_kgen(ka, g.R, s);
            if (e == cudaSuccess) e = cudaEventRecord(c->kev[1], s);
            tr.mark("kgen (distinct windows)");
            ExpandArgs ea{class_pad, class_w, class_diag, nullptr, nullptr, g.nx, g.ny, g.nxq, g.tile, g.tpp,
                          g.n_tiles, g.nxp, g.nyp};
            size_t w_elems = g.w_elems, d_elems = g.diag_elems;
            if (e == cudaSuccess && (params->flags & FDIRW_F_DEDUP_STORAGE)) {
                // N4: uniform chunks get no gather weights; the others are compacted into tiles
                e = build_uniform(ea, g.R, c->fmt == FDIRW_W_MX8 ? FDIRW_W_FP32 : c->fmt, dr.n_class, &c->ut, s);
                if (c->fmt == FDIRW_W_MX8) ea.ut = &c->ut;
                ea.list = c->ut.dense_list;
                ea.n_list = c->ut.n_dense;
                ea.n_tiles = c->ut.nd_tiles;
                w_elems = (size_t)c->ut.nd_tiles * (g.K - 1) * g.tile * kChunk;
                d_elems = (size_t)c->ut.nd_tiles * g.tile * kChunk;
            } else if (e == cudaSuccess && params->v_far > 0 && c->world == 1) {
                // N2: all-far chunks (no targets) get no gather weights either
                if ((st = far_compact(c, phase_host, s)) != FDIRW_OK) { dfree(); cudaFree(mask_d); return bail(st); }
                ea.list = c->ut.dense_list;
                ea.n_list = c->ut.n_dense;
                ea.n_tiles = c->ut.nd_tiles;
                w_elems = (size_t)c->ut.nd_tiles * (g.K - 1) * g.tile * kChunk;
                d_elems = (size_t)c->ut.nd_tiles * g.tile * kChunk;
            }
            if (e == cudaSuccess) {
                if ((st = alloc(&c->Wt, wbytes(c->fmt, w_elems ? w_elems : 8), "weights")) != FDIRW_OK ||
                    (st = alloc((void**)&c->diag, (d_elems ? d_elems : 1) * 8, "diagonal")) != FDIRW_OK) {
                    dfree(); cudaFree(mask_d); return bail(st);
                }
                ea.Wt = c->Wt;
                ea.diag = c->diag;
                ea.nzl = g.nzl;
                ea.class_mass = class_mass;
                if (c->fmt == FDIRW_W_MX8 && c->compact) ea.far_pos = c->chunk_pos;
                ea.z0 = g.z0;
                ea.nz = g.nz;
                tr.mark("compact + alloc weights");
                e = launch_expand(ea, g.R, c->fmt, s);
                tr.mark("expand");
            }
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) { dfree(); cudaFree(mask_d); g_err = std::string("kgen: ") + cudaGetErrorString(e); return bail(FDIRW_E_CUDA); }
            c->kgen_windows = (uint64_t)dr.n_class;
        }
        dfree();
    }
    if (!dedup && c->fmt == FDIRW_W_MX8) {
        cudaFree(mask_d);
        g_err = "MX8 weights need the window de-duplication (hash collision fallback not supported)";
        return bail(FDIRW_E_STATE);
    }
    if (!dedup) {
        ka.src_list = nullptr; ka.n_list = 0; ka.class_w = nullptr; ka.class_diag = nullptr;
        if ((st = alloc(&c->Wt, g.w_elems * c->b_w, "weights")) != FDIRW_OK ||
            (st = alloc((void**)&c->diag, g.diag_elems * 8, "diagonal")) != FDIRW_OK) {
            cudaFree(mask_d);
            return bail(st);
        }
        ka.Wt = c->Wt;
        ka.diag = c->diag;
        BAIL_CUDA(cudaMemsetAsync(c->Wt, 0, g.w_elems * c->b_w, s));
        BAIL_CUDA(cudaMemsetAsync(c->diag, 0, g.diag_elems * 8, s));
        if (!c->kev[0]) BAIL_CUDA(cudaEventCreate(&c->kev[0]));
        if (!c->kev[1]) BAIL_CUDA(cudaEventCreate(&c->kev[1]));
        BAIL_CUDA(cudaEventRecord(c->kev[0], s));
        BAIL_CUDA(launch_kgen(ka, g.R, s));
        BAIL_CUDA(cudaEventRecord(c->kev[1], s));
        tr.mark("kgen (every source)");
    }
    BAIL_CUDA(cudaStreamSynchronize(s));
    cudaFree(c->cheb_d);
    c->cheb_d = nullptr;
    BAIL_CUDA(cudaEventElapsedTime(&c->kgen_ms, c->kev[0], c->kev[1]));

    tr.mark("sync");
    c->v_far = params->v_far;
    c->far = params->v_far > 0;
    if (c->far) {  // N2: far-field mask of the slab, p_BC, Eq.7 reduction buffers
        const size_t ns = (size_t)g.nx * g.ny * g.nzl;
        std::vector<uint8_t> fm(ns);
        for (size_t i = 0; i < ns; ++i) fm[i] = phase_host[(size_t)g.z0 * plane + i] == 2 ? 1 : 0;
        c->tile_stride = 1 + (long)g.nz * g.tpp;
        if ((st = alloc((void**)&c->farmask, ns, "far mask")) != FDIRW_OK ||
            (st = alloc((void**)&c->pbc, (c->compact ? (size_t)c->ut.nd_tiles * g.tile * kChunk + 8 : g.diag_elems) * 4,
                        "p_BC")) != FDIRW_OK ||
            (st = alloc((void**)&c->tile_buf, c->tile_stride * 8, "tile sums")) != FDIRW_OK ||
            (st = alloc((void**)&c->gathered, (size_t)c->world * c->tile_stride * 8, "gathered sums")) != FDIRW_OK ||
            (st = alloc((void**)&c->far_state, 16, "far state")) != FDIRW_OK) {
            cudaFree(mask_d);
            return bail(st);
        }
        const double nt = (double)g.n_tiles;
        BAIL_CUDA(cudaMemcpy(c->farmask, fm.data(), ns, cudaMemcpyHostToDevice));
        BAIL_CUDA(cudaMemset(c->tile_buf, 0, c->tile_stride * 8));
        BAIL_CUDA(cudaMemcpy(c->tile_buf, &nt, 8, cudaMemcpyHostToDevice));
        BAIL_CUDA(cudaMemset(c->far_state, 0, 16));
        if ((st = build_pbc(c, mask_d, s)) != FDIRW_OK) {
            cudaFree(mask_d);
            return bail(st);
        }
    }
    if (c->world == 1) {  // N3: padded phase map for the integrated loop (mask_d holds the whole grid)
        for (size_t i = 0; i < plane * g.nz; ++i) c->n_solid += phase_host[i] == 0;
        if ((st = alloc((void**)&c->phase_pp, g.state_elems, "phase map")) != FDIRW_OK) {
            cudaFree(mask_d);
            return bail(st);
        }
        BAIL_CUDA(launch_phase_pad(mask_d, g, c->phase_pp, s));
        BAIL_CUDA(cudaStreamSynchronize(s));
    }
    cudaFree(mask_d);

    BAIL_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    BAIL_CUDA(cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking));
    BAIL_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    BAIL_CUDA(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));

    if (c->world > 1 && c->transport == FDIRW_TRANSPORT_P2P) {
        if ((st = alloc((void**)&c->p2p_flags, 32, "p2p flags")) != FDIRW_OK) return bail(st);
        BAIL_CUDA(cudaMemset(c->p2p_flags, 0, 32));
    } else if (c->world > 1 && !c->is_virtual) {
        std::string err;
        c->nccl = nccl_load(&err);
        if (!c->nccl) { g_err = err; return bail(FDIRW_E_NCCL); }
        c->comm = nccl_comm_init(c->nccl, c->world, c->rank, dist->nccl_id, &err);
        if (!c->comm) { g_err = err; return bail(FDIRW_E_NCCL); }
        // NCCL connects peers lazily on first use; do that here, outside any stream capture
        // (fdirw_run captures the halo exchange and the Eq.7 all-gather into a CUDA graph).
        // The state buffers are still zero, so the exchange moves zeros.
        if (nccl_halo(c->nccl, c->comm, c->cpad[0], make_halo_plan(g, c->rank, c->world), c->comm_stream, &err) ||
            (c->far && nccl_allgather_f64(c->nccl, c->comm, c->tile_buf, c->tile_stride, c->gathered, c->comm_stream, &err)) ||
            nccl_allreduce_sum_f64(c->nccl, c->comm, c->mass_out, c->comm_stream, &err)) {
            g_err = err;
            return bail(FDIRW_E_NCCL);
        }
        BAIL_CUDA(cudaStreamSynchronize(c->comm_stream));
    }
#undef BAIL_CUDA
    tr.mark("far field / comm / end");
    *out = c;
    return FDIRW_OK;
}

// Superpose tiles [t0, t1) of `src` (padded) into `out` with strides (ps, rs).  With a far
// field (N2) and far_terms: + p_BC·c_far and the per-tile Σ C_new for Eq.7.
static cudaError_t superpose(fdirw_ctx* c, const float* src, float* out, long ps, long rs, int t0, int t1,
                             cudaStream_t s, bool far_terms = true, int push_parity = -1, int gap0 = 0, int gap1 = 0,
                             bool gap_last = false)
{
    const Geometry& g = c->g;
    SuperArgs a{};
    a.cpad = src;
    a.Wt = c->Wt;
    a.diag = c->diag;
    a.out = out;
    a.out_ps = ps;
    a.out_rs = rs;
    a.nx = g.nx; a.ny = g.ny; a.nxq = g.nxq; a.tile = g.tile; a.tpp = g.tpp; a.K = g.K;
    a.nxp = g.nxp; a.nyp = g.nyp;
    a.t_begin = t0;
    a.t_end = t1;
    if (gap1 > gap0) {  // tiles [t0, gap0) ∪ [gap1, t1) in one launch
        a.gap_at = gap0;
        a.gap_len = gap1 - gap0;
        a.gap_last = gap_last;
    }
    a.no_bulk = c->no_bulk;
    a.canary = c->canary;
    a.list = c->ut.dense_list;  // N4 (null unless FDIRW_F_DEDUP_STORAGE): compacted non-uniform chunks
    a.n_list = c->ut.n_dense;
    if (c->far && far_terms) {
        a.pbc = c->pbc;
        a.far_state = c->far_state;
        // compacted tiles are not the global tiles of Eq.7: the sums come from tile_mass then
        a.tile_sum = c->compact ? nullptr : c->tile_buf + 1;
    }
    if (push_parity >= 0) {  // a6 over peer memory: boundary planes also into the neighbours' halos
        const long pe = (long)g.plane_elems, row0 = (long)g.R * g.nxp + kPadX;
        if (c->peer_lo[push_parity]) a.push_lo = c->peer_lo[push_parity] + (long)(c->nzl_lo + g.R) * pe + row0;
        if (c->peer_hi[push_parity]) a.push_hi = c->peer_hi[push_parity] + row0;
        a.nzl = g.nzl;
        a.pR = g.R;
    }
    return launch_superpose(a, g.R, c->fmt, s);
}

// N4: the uniform chunks (one CTA per ≤ 256 chunks of one class, class kernel in smem).
static cudaError_t superpose_uniform(fdirw_ctx* c, const float* src, float* out, long ps, long rs, cudaStream_t s)
{
    if (!c->ut.chunk_u || c->ut.n_blocks == 0) return cudaSuccess;
    const Geometry& g = c->g;
    UniArgs u{};
    u.cpad = src;
    u.out = out;
    u.out_ps = ps;
    u.out_rs = rs;
    u.nx = g.nx; u.ny = g.ny; u.nxq = g.nxq; u.tile = g.tile; u.tpp = g.tpp; u.nxp = g.nxp; u.nyp = g.nyp;
    u.list = c->ut.list;
    u.blocks = c->ut.blocks;
    u.n_blocks = c->ut.n_blocks;
    u.ukf = c->ut.ukf;
    u.udiag = c->ut.udiag;
    u.udiag_t = c->ut.udiag_t;
    return launch_superpose_uniform(u, g.R, s);
}

// N4: the compacted dense tiles and the uniform blocks in one mixed launch.
static cudaError_t superpose_n4_mixed(fdirw_ctx* c, const float* src, float* out, long ps, long rs, cudaStream_t s)
{
    const Geometry& g = c->g;
    if (c->ut.n_blocks == 0)  // no uniform chunk at all: the plain dense launch over the compacted tiles
        return superpose(c, src, out, ps, rs, 0, c->ut.nd_tiles, s, false);
    SuperArgs a{};
    a.cpad = src;
    a.Wt = c->Wt;
    a.diag = c->diag;
    a.out = out;
    a.out_ps = ps;
    a.out_rs = rs;
    a.nx = g.nx; a.ny = g.ny; a.nxq = g.nxq; a.tile = g.tile; a.tpp = g.tpp; a.K = g.K;
    a.nxp = g.nxp; a.nyp = g.nyp;
    a.t_begin = 0;
    a.t_end = c->ut.nd_tiles;
    a.no_bulk = c->no_bulk;
    a.list = c->ut.dense_list;
    a.n_list = c->ut.n_dense;
    UniArgs u{};
    u.cpad = src;
    u.out = out;
    u.out_ps = ps;
    u.out_rs = rs;
    u.nx = g.nx; u.ny = g.ny; u.nxq = g.nxq; u.tile = g.tile; u.tpp = g.tpp; u.nxp = g.nxp; u.nyp = g.nyp;
    u.list = c->ut.list;
    u.blocks = c->ut.blocks;
    u.n_blocks = c->ut.n_blocks;
    u.ukf = c->ut.ukf;
    u.udiag = c->ut.udiag;
    u.udiag_t = c->ut.udiag_t;
    return launch_superpose_mixed(a, u, g.R, c->fmt, s);
}

// N2: p_BC(x) = 1 − Σ_s W̃_s(x−s) (reading A26) = 1 − (stored operator applied to the
// indicator of the non-far voxels); computed once after kgen with the superposition itself.
static fdirw_status build_pbc(fdirw_ctx* c, const uint8_t* mask_d, cudaStream_t s)
{
    const Geometry& g = c->g;
    float* rowsum = nullptr;
    const size_t n = (size_t)g.nx * g.ny * g.nzl;
    fdirw_status st = alloc((void**)&rowsum, n * 4, "p_BC scratch");
    if (st != FDIRW_OK) return st;
    cudaError_t e = cudaSuccess;
    const bool reservoir = (c->p.flags & FDIRW_F_PBC_RESERVOIR) && c->world == 1;
    if (reservoir) {  // the reservoir's held-Dirichlet FD response (A26 alternative), into rowsum
        float* tmp = nullptr;
        if ((st = alloc((void**)&tmp, n * 4, "p_BC reservoir FD")) != FDIRW_OK) { cudaFree(rowsum); return st; }
        e = launch_reservoir_fd(mask_d, g, (float)c->d.lam_ff, (float)c->d.lam_fs, (float)c->d.lam_ss, c->d.n_fd,
                                rowsum, tmp, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(tmp);
    } else {
        e = launch_ones(mask_d, g.mz0, g, c->cpad[1], s);
        if (e == cudaSuccess)
            e = superpose(c, c->cpad[1], rowsum, (long)g.nx * g.ny, g.nx, 0, c->compact ? c->ut.nd_tiles : g.n_tiles, s,
                          false);
    }
    if (e == cudaSuccess)
        e = launch_pbc(rowsum, c->farmask, g, c->pbc, s, c->compact ? c->ut.dense_list : nullptr, c->ut.n_dense,
                       c->ut.nd_tiles, reservoir);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->cpad[1], 0, g.state_elems * 4, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(rowsum);
    if (e != cudaSuccess) return fail(FDIRW_E_CUDA, std::string("p_BC: ") + cudaGetErrorString(e));
    return FDIRW_OK;
}

// N2: Eq.7 after a step (or M0 at init, mode 1): tile sums of every rank in global tile order.
static fdirw_status far_reduce(fdirw_ctx* c, cudaStream_t s, int mode, double c_far0)
{
    if (c->world == 1 || c->is_virtual) {
        if (c->is_virtual) return FDIRW_OK;  // fdirw_step_virtual gathers across the contexts
        CUDA_TRY(launch_far_reduce(c->tile_buf, 1, c->tile_stride, c->far_state, c->v_far, c_far0, mode, s));
        return FDIRW_OK;
    }
    std::string err;
    if (nccl_allgather_f64(c->nccl, c->comm, c->tile_buf, c->tile_stride, c->gathered, s, &err))
        return fail(FDIRW_E_NCCL, err);
    CUDA_TRY(launch_far_reduce(c->gathered, c->world, c->tile_stride, c->far_state, c->v_far, c_far0, mode, s));
    return FDIRW_OK;
}

// Interior tiles are those whose targets read no halo plane: z_local ∈ [R, nzl − R).
static void split_tiles(const Geometry& g, int* int0, int* int1)
{
    if (g.nzl <= 2 * g.R) { *int0 = *int1 = 0; return; }
    *int0 = g.R * g.tpp;
    *int1 = (g.nzl - g.R) * g.tpp;
}

// Phase events of one step (fdirw_profile_phases; null on the normal path).  Recorded on the
// compute stream unless noted: t0 start, halo0/halo1 the halo phase (P2P: the wait kernel;
// NCCL: the exchange, both on the comm stream), sup the interior (or only) superposition done,
// bnd0/bnd1 the boundary-band launch (NCCL), t1 the end of the step (P2P signal / Eq.7 done).
struct PhaseEv {
    cudaEvent_t t0, halo0, halo1, sup, bnd0, bnd1, t1;
};
#define PHASE(field, stream) \
    do { if (pe) CUDA_TRY(cudaEventRecord(pe->field, stream)); } while (0)

// One step src (padded, slab planes filled) → out; exchanges the halo planes of src first.
// eq7 = false (the N3 loop): skip the compacted path's Eq.7 sums and c_far update after the liquid
// step — the loop's kinetics pass sets c_far from the whole step's totals (oracle/integrated.py
// run(), component (4) after (1)-(3)), which overwrites it before any kernel reads it.
// copy_ident = false (the N3 loop's nf path): skip the identity-chunk copy — the loop's solid pass
// writes every solid voxel of the output from the input
static fdirw_status enqueue_step(fdirw_ctx* c, float* src, float* out, long ps, long rs, cudaStream_t s,
                                 int dst_parity = 1, PhaseEv* pe = nullptr, bool eq7 = true, bool copy_ident = true)
{
    const Geometry& g = c->g;
    PHASE(t0, s);
    if (c->world > 1 && c->transport == FDIRW_TRANSPORT_P2P) {
        // wait for the neighbours' previous step (their stores into my halo are complete and
        // they are done reading the halo I overwrite) → ONE launch over every tile, boundary
        // bands first so their stores into the neighbours' halos start early → signal.
        // (No transfer phase is left to overlap, so the interior is not split off: one
        // launch keeps the SMs evenly loaded at strong-scaling slab sizes.)
        int i0, i1;
        split_tiles(g, &i0, &i1);
        PHASE(halo0, s);
        CUDA_TRY(p2p_wait(c->p2p_flags, c->peer_lo_flag != nullptr, c->peer_hi_flag != nullptr, s));
        PHASE(halo1, s);
        if (i1 > i0)
            CUDA_TRY(superpose(c, src, out, ps, rs, 0, g.n_tiles, s, true, dst_parity, i0, i1, true));
        else
            CUDA_TRY(superpose(c, src, out, ps, rs, 0, g.n_tiles, s, true, dst_parity));
        PHASE(sup, s);
        PHASE(bnd0, s);
        PHASE(bnd1, s);
        CUDA_TRY(p2p_signal(c->p2p_flags, c->peer_lo_flag, c->peer_hi_flag, s));
        PHASE(t1, s);
        return FDIRW_OK;
    }
    if (pe && c->world == 1 && (c->prec_mode != 0 || c->ut.chunk_u || c->compact))
        return fail(FDIRW_E_STATE, "phase profile: the dense superposition path only");
    if (c->world == 1 && c->prec_mode != 0) {  // N3 §3.3 study modes: padded output only
        StudyArgs a{src, out - ((size_t)g.R * g.plane_elems + (size_t)g.R * g.nxp + kPadX), c->Wt, c->diag,
                    g.nx, g.ny, g.nzl, g.nxq, g.tile, g.tpp, g.nxp, g.nyp, g.R, c->pbc, c->far_state,
                    c->compact ? c->chunk_pos : nullptr};
        if (ps != (long)g.plane_elems) return fail(FDIRW_E_STATE, "precision study modes run through fdirw_run");
        CUDA_TRY(launch_superpose_study(a, c->prec_mode, s));
        if (c->far && eq7) {  // study kernel has no tile sums: Eq.7 from a separate pass
            CUDA_TRY(launch_tile_mass_padded(out, c->farmask, g, c->tile_buf + 1, s));
            return far_reduce(c, s, 0, 0.0);
        }
        return FDIRW_OK;
    }
    if (c->world == 1) {
        if (c->ut.chunk_u && g.tile == 256) {  // N4: one launch mixing dense and uniform blocks
            CUDA_TRY(superpose_n4_mixed(c, src, out, ps, rs, s));
            return FDIRW_OK;
        }
        if (c->ut.chunk_u) {  // N4 (small tiles): dense and uniform kernels on two streams
            CUDA_TRY(cudaEventRecord(c->ev_fork, s));
            CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
            CUDA_TRY(superpose_uniform(c, src, out, ps, rs, c->comm_stream));
            CUDA_TRY(cudaEventRecord(c->ev_comm, c->comm_stream));
            CUDA_TRY(superpose(c, src, out, ps, rs, 0, c->ut.nd_tiles, s));
            CUDA_TRY(cudaStreamWaitEvent(s, c->ev_comm, 0));
            return FDIRW_OK;
        }
        if (c->compact) {  // N2 compacted: superpose the listed chunks, Eq.7 sums per global tile
            CUDA_TRY(superpose(c, src, out, ps, rs, 0, c->ut.nd_tiles, s));
            if (c->n_ident && copy_ident)  // identity rows (impermeable solid): C_new = C_old
                CUDA_TRY(launch_copy_chunks(src, out, ps, rs, c->ident_list, c->n_ident, g, s));
            if (!eq7) return FDIRW_OK;
            if (ps == (long)g.plane_elems) CUDA_TRY(launch_tile_mass_padded(out, c->farmask, g, c->tile_buf + 1, s));
            else CUDA_TRY(launch_tile_mass(out, c->farmask, g, c->tile_buf + 1, s));
            return far_reduce(c, s, 0, 0.0);
        }
        PHASE(halo0, s);
        PHASE(halo1, s);
        CUDA_TRY(superpose(c, src, out, ps, rs, 0, g.n_tiles, s));
        PHASE(sup, s);
        PHASE(bnd0, s);
        PHASE(bnd1, s);
        fdirw_status st = c->far && eq7 ? far_reduce(c, s, 0, 0.0) : FDIRW_OK;
        PHASE(t1, s);
        return st;
    }
    int i0, i1;
    split_tiles(g, &i0, &i1);
    CUDA_TRY(cudaEventRecord(c->ev_fork, s));
    CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
    std::string err;
    PHASE(halo0, c->comm_stream);
    if (nccl_halo(c->nccl, c->comm, src, make_halo_plan(g, c->rank, c->world), c->comm_stream, &err))
        return fail(FDIRW_E_NCCL, err);
    PHASE(halo1, c->comm_stream);
    CUDA_TRY(cudaEventRecord(c->ev_comm, c->comm_stream));
    CUDA_TRY(superpose(c, src, out, ps, rs, i0, i1, s));  // interior overlaps the exchange
    PHASE(sup, s);
    CUDA_TRY(cudaStreamWaitEvent(s, c->ev_comm, 0));
    PHASE(bnd0, s);
    if (i1 > i0) {  // both boundary bands in one launch
        CUDA_TRY(superpose(c, src, out, ps, rs, 0, g.n_tiles, s, true, -1, i0, i1));
    } else {
        CUDA_TRY(superpose(c, src, out, ps, rs, 0, g.n_tiles, s));
    }
    PHASE(bnd1, s);
    fdirw_status st = c->far ? far_reduce(c, s, 0, 0.0) : FDIRW_OK;
    PHASE(t1, s);
    return st;
}
#undef PHASE

// P2P run start (after the pack into cpad[0]): signal "packed", wait for the neighbours'
// (so nobody still reads the halo of cpad[0]), push our edge planes into their halos, signal.
static fdirw_status p2p_start(fdirw_ctx* c, cudaStream_t s)
{
    if (!c->p2p_ready) return fail(FDIRW_E_STATE, "P2P transport: call fdirw_p2p_attach first");
    const bool lo = c->peer_lo_flag != nullptr, hi = c->peer_hi_flag != nullptr;
    CUDA_TRY(p2p_signal(c->p2p_flags, c->peer_lo_flag, c->peer_hi_flag, s));
    CUDA_TRY(p2p_wait(c->p2p_flags, lo, hi, s));
    CUDA_TRY(p2p_push_planes(c->g, c->cpad[0], c->peer_lo[0], c->nzl_lo, c->peer_hi[0], s));
    CUDA_TRY(p2p_signal(c->p2p_flags, c->peer_lo_flag, c->peer_hi_flag, s));
    return FDIRW_OK;
}

static float* pad_interior(fdirw_ctx* c, int i)
{
    const Geometry& g = c->g;
    return c->cpad[i] + (size_t)g.R * g.plane_elems + (size_t)g.R * g.nxp + kPadX;
}

extern "C" fdirw_status fdirw_step(fdirw_ctx* c, const float* c_in, float* c_out, void* cuda_stream)
{
    NvtxRange nvtx("fdirw_step");
    if (!c || !c_in || !c_out) return fail(FDIRW_E_INVALID, "NULL argument");
    if (c->is_virtual) return fail(FDIRW_E_STATE, "virtual-rank context: use fdirw_step_virtual");
    if (c_in == c_out) return fail(FDIRW_E_ALIAS, "c_in == c_out");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const Geometry& g = c->g;
    CUDA_TRY(launch_pack(c_in, c->cpad[0], g, s, c->farmask));
    if (c->compact)  // targets of all-far chunks are not computed; far voxels read 0 as on every path
        CUDA_TRY(cudaMemsetAsync(c_out, 0, (size_t)g.nx * g.ny * g.nzl * 4, s));
    if (c->world > 1 && c->transport == FDIRW_TRANSPORT_P2P) {
        fdirw_status st = p2p_start(c, s);
        if (st != FDIRW_OK) return st;
    }
    return enqueue_step(c, c->cpad[0], c_out, (long)g.nx * g.ny, g.nx, s, 1);
}

// fdirw_step_host, the pipelined form (world 1, the dense closed-domain superposition): the
// slab is cut into nch plane chunks; chunk j's planes are copied from the host straight into
// the padded state (3-D strided copy on the H2D stream), the superposition of chunk j's tiles
// starts as soon as the planes it reads (its own + R on either side) have landed, and chunk j's
// result goes back to the host (D2H stream) while chunk j + 1 computes.  Only the first
// chunk's copy-in and the last chunk's copy-out stay exposed.  nch is picked so that each
// chunk's launch fills whole waves of the staged stream (2 CTAs × SMs).
static int step_host_chunks(const fdirw_ctx* c)
{
    const Geometry& g = c->g;
    if (c->world > 1 || c->far || c->ut.chunk_u || c->compact || c->prec_mode != 0 || g.nzl < 4 * g.R)
        return 1;
    // small slabs (< 8 tiles per SM): the copies are short and a chunk's launch would be a
    // fraction of a wave; one copy-in, one step, one copy-out is faster
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    if (g.n_tiles < 8 * sms) return 1;
    // chunks of at least max(8, R) planes, at most 16: the exposed head (first chunk's copy-in)
    // and tail (last chunk's copy-out) shrink with the chunk, while the chunk launches' partial
    // last waves are filled by the next chunk's launch on the other compute stream
    // (measured at cfg3: 4 / 6 / 8 chunks on one stream gave 0.83 / 0.86 / 0.88 of the
    // device-timed rate)
    return std::max(1, std::min(16, g.nzl / std::max(8, g.R)));
}

static fdirw_status step_host_pipelined(fdirw_ctx* c, const float* in, float* out, cudaStream_t s, int nch)
{
    const Geometry& g = c->g;
    if (!c->h2d_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
    if (!c->d2h_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
    if ((int)c->hx_ev.size() < 3 * nch + 1) {
        for (cudaEvent_t e : c->hx_ev) cudaEventDestroy(e);
        c->hx_ev.assign(3 * nch + 1, nullptr);
        for (auto& e : c->hx_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaEvent_t* h2d = c->hx_ev.data();
    cudaEvent_t* done = h2d + nch;
    cudaEvent_t* d2h = done + nch;
    cudaEvent_t start = c->hx_ev[3 * nch];
    const int pl = (g.nzl + nch - 1) / nch;
    const size_t plane_b = (size_t)g.nx * g.ny * 4;
    // the previous work on s (the last reads of cpad[0] and of the output staging) precedes
    // this step's copies
    CUDA_TRY(cudaEventRecord(start, s));
    CUDA_TRY(cudaStreamWaitEvent(c->h2d_stream, start, 0));
    CUDA_TRY(cudaStreamWaitEvent(c->d2h_stream, start, 0));
    for (int j = 0; j < nch; ++j) {
        const int z0 = j * pl, z1 = std::min(g.nzl, z0 + pl);
        if (z0 >= z1) { CUDA_TRY(cudaEventRecord(h2d[j], c->h2d_stream)); continue; }
        cudaMemcpy3DParms m{};
        m.srcPtr = make_cudaPitchedPtr(const_cast<float*>(in) + (size_t)z0 * g.nx * g.ny, (size_t)g.nx * 4, g.nx, g.ny);
        m.dstPtr = make_cudaPitchedPtr(c->cpad[0], (size_t)g.nxp * 4, g.nxp, g.nyp);
        m.dstPos = make_cudaPos((size_t)kPadX * 4, g.R, g.R + z0);
        m.extent = make_cudaExtent((size_t)g.nx * 4, g.ny, z1 - z0);
        m.kind = cudaMemcpyHostToDevice;
        CUDA_TRY(cudaMemcpy3DAsync(&m, c->h2d_stream));
        CUDA_TRY(cudaEventRecord(h2d[j], c->h2d_stream));
    }
    // chunks alternate between the caller's stream and a second compute stream (the context's
    // comm stream, idle at world 1) so a chunk's launch can start while the previous one drains
    CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, start, 0));
    for (int j = 0; j < nch; ++j) {
        cudaStream_t cs = (j & 1) ? c->comm_stream : s;
        const int z0 = j * pl, z1 = std::min(g.nzl, z0 + pl);
        if (z0 >= z1) { CUDA_TRY(cudaEventRecord(done[j], cs)); CUDA_TRY(cudaEventRecord(d2h[j], c->d2h_stream)); continue; }
        const int need = std::min(nch - 1, (std::min(g.nzl, z1 + g.R) - 1) / pl);  // last chunk read
        CUDA_TRY(cudaStreamWaitEvent(cs, h2d[need], 0));  // (H2D stream order covers the earlier chunks)
        CUDA_TRY(superpose(c, c->cpad[0], c->host_stage[1], (long)g.nx * g.ny, g.nx, z0 * g.tpp, z1 * g.tpp, cs));
        CUDA_TRY(cudaEventRecord(done[j], cs));
        CUDA_TRY(cudaStreamWaitEvent(c->d2h_stream, done[j], 0));
        CUDA_TRY(cudaMemcpyAsync(out + (size_t)z0 * g.nx * g.ny, c->host_stage[1] + (size_t)z0 * g.nx * g.ny,
                                 (size_t)(z1 - z0) * plane_b, cudaMemcpyDeviceToHost, c->d2h_stream));
        CUDA_TRY(cudaEventRecord(d2h[j], c->d2h_stream));
    }
    // the caller's stream covers the result (the D2H stream waited for every chunk in order)
    CUDA_TRY(cudaStreamWaitEvent(s, d2h[nch - 1], 0));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_step_host(fdirw_ctx* c, const float* c_in_host, float* c_out_host, void* cuda_stream)
{
    if (!c || !c_in_host || !c_out_host) return fail(FDIRW_E_INVALID, "NULL argument");
    if (c_in_host == c_out_host) return fail(FDIRW_E_ALIAS, "c_in == c_out");
    if (c->is_virtual) return fail(FDIRW_E_STATE, "virtual-rank context: use fdirw_step_virtual");
    CUDA_TRY(cudaSetDevice(c->device));
    const size_t bytes = (size_t)c->g.nx * c->g.ny * c->g.nzl * 4;
    for (int i = 0; i < 2; ++i)
        if (!c->host_stage[i]) {
            fdirw_status st = alloc((void**)&c->host_stage[i], bytes, "host staging");
            if (st != FDIRW_OK) return st;
        }
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    static const int force = [] {
        const char* ev = getenv("FDIRW_STEP_HOST_CHUNKS");  // A/B: 1 = the plain form
        return ev ? atoi(ev) : 0;
    }();
    const int nch = force > 0 ? (force == 1 ? 1 : std::min(force, 16)) : step_host_chunks(c);
    if (nch > 1 && step_host_chunks(c) > 1) return step_host_pipelined(c, c_in_host, c_out_host, s, nch);
    CUDA_TRY(cudaMemcpyAsync(c->host_stage[0], c_in_host, bytes, cudaMemcpyHostToDevice, s));
    fdirw_status st = fdirw_step(c, c->host_stage[0], c->host_stage[1], cuda_stream);
    if (st != FDIRW_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(c_out_host, c->host_stage[1], bytes, cudaMemcpyDeviceToHost, s));
    return FDIRW_OK;
}

// capture step(0→1); step(1→0) once; fdirw_run replays it n/2 times.  With P2P this is done
// at attach time: instantiating a graph can wait for the device, which must not happen while
// a neighbour's step spins on this context's flags.
static fdirw_status capture_graph2(fdirw_ctx* c)
{
    const Geometry& g = c->g;
    if (c->transport == FDIRW_TRANSPORT_P2P) CUDA_TRY(p2p_preload());
    const long ps = (long)g.plane_elems, rs = g.nxp;
    cudaStream_t cs = c->capture_stream;
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    fdirw_status st = enqueue_step(c, c->cpad[0], pad_interior(c, 1), ps, rs, cs, 1);
    if (st == FDIRW_OK) st = enqueue_step(c, c->cpad[1], pad_interior(c, 0), ps, rs, cs, 0);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (st != FDIRW_OK) { if (graph) cudaGraphDestroy(graph); return st; }
    if (e != cudaSuccess) return fail(FDIRW_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->graph2, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) { c->graph2 = nullptr; return fail(FDIRW_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e)); }
    CUDA_TRY(cudaGraphUpload(c->graph2, c->capture_stream));
    CUDA_TRY(cudaStreamSynchronize(c->capture_stream));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_run(fdirw_ctx* c, float* c_dev, int32_t n_steps, void* cuda_stream)
{
    NvtxRange nvtx("fdirw_run");
    if (!c || !c_dev) return fail(FDIRW_E_INVALID, "NULL argument");
    if (n_steps < 0) return fail(FDIRW_E_INVALID, "n_steps must be >= 0");
    if (c->is_virtual) return fail(FDIRW_E_STATE, "virtual-rank context: use fdirw_step_virtual");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const Geometry& g = c->g;
    if (n_steps == 0) return FDIRW_OK;
    CUDA_TRY(launch_pack(c_dev, c->cpad[0], g, s, c->farmask));
    if (c->world > 1 && c->transport == FDIRW_TRANSPORT_P2P) {
        fdirw_status st = p2p_start(c, s);
        if (st != FDIRW_OK) return st;
    }
    const long ps = (long)g.plane_elems, rs = g.nxp;
    if (n_steps >= 2 && !c->graph2) {
        fdirw_status st = capture_graph2(c);
        if (st != FDIRW_OK) return st;
    }
    for (int i = 0; i < n_steps / 2; ++i) CUDA_TRY(cudaGraphLaunch(c->graph2, s));
    int fin = 0;
    if (n_steps & 1) {
        fdirw_status st = enqueue_step(c, c->cpad[0], pad_interior(c, 1), ps, rs, s, 1);
        if (st != FDIRW_OK) return st;
        fin = 1;
    }
    CUDA_TRY(launch_unpack(c->cpad[fin], c_dev, g, s));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_profile_phases(fdirw_ctx* c, float* c_dev, int32_t n_steps, void* cuda_stream,
                                            double* ms_out)
{
    if (!c || !c_dev || !ms_out) return fail(FDIRW_E_INVALID, "NULL argument");
    if (n_steps < 1 || n_steps > 256) return fail(FDIRW_E_INVALID, "n_steps must be in [1, 256]");
    if (c->is_virtual) return fail(FDIRW_E_STATE, "virtual-rank context: use fdirw_step_virtual");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const Geometry& g = c->g;
    std::vector<PhaseEv> ev(n_steps);
    cudaError_t e = cudaSuccess;
    int made = 0;
    for (; made < n_steps && e == cudaSuccess; ++made) {
        cudaEvent_t* f[7] = {&ev[made].t0, &ev[made].halo0, &ev[made].halo1, &ev[made].sup, &ev[made].bnd0,
                             &ev[made].bnd1, &ev[made].t1};
        for (int k = 0; k < 7 && e == cudaSuccess; ++k) e = cudaEventCreate(f[k]);
    }
    auto release = [&]() {
        for (int i = 0; i < made; ++i) {
            cudaEvent_t f[7] = {ev[i].t0, ev[i].halo0, ev[i].halo1, ev[i].sup, ev[i].bnd0, ev[i].bnd1, ev[i].t1};
            for (cudaEvent_t x : f)
                if (x) cudaEventDestroy(x);
        }
    };
    fdirw_status st = FDIRW_OK;
    if (e != cudaSuccess) st = fail(FDIRW_E_CUDA, std::string("phase events: ") + cudaGetErrorString(e));
    if (st == FDIRW_OK && (e = launch_pack(c_dev, c->cpad[0], g, s, c->farmask)) != cudaSuccess)
        st = fail(FDIRW_E_CUDA, cudaGetErrorString(e));
    if (st == FDIRW_OK && c->world > 1 && c->transport == FDIRW_TRANSPORT_P2P) st = p2p_start(c, s);
    const long ps = (long)g.plane_elems, rs = g.nxp;
    int cur = 0;
    for (int i = 0; i < n_steps && st == FDIRW_OK; ++i) {
        st = enqueue_step(c, c->cpad[cur], pad_interior(c, 1 - cur), ps, rs, s, 1 - cur, &ev[i]);
        cur = 1 - cur;
    }
    if (st == FDIRW_OK && (e = launch_unpack(c->cpad[cur], c_dev, g, s)) != cudaSuccess)
        st = fail(FDIRW_E_CUDA, cudaGetErrorString(e));
    if (st == FDIRW_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess)
        st = fail(FDIRW_E_CUDA, cudaGetErrorString(e));
    if (st == FDIRW_OK && (e = cudaStreamSynchronize(c->comm_stream)) != cudaSuccess)
        st = fail(FDIRW_E_CUDA, cudaGetErrorString(e));
    double acc[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < n_steps && st == FDIRW_OK; ++i) {
        float t[5] = {0, 0, 0, 0, 0};
        const PhaseEv& p = ev[i];
        // NCCL: the interior runs on the compute stream from t0 while the exchange runs on the
        // comm stream; elsewhere it follows the halo phase
        const cudaEvent_t int0 = (c->world > 1 && c->transport == FDIRW_TRANSPORT_NCCL) ? p.t0 : p.halo1;
        e = cudaEventElapsedTime(&t[0], p.halo0, p.halo1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t[1], int0, p.sup);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t[2], p.bnd0, p.bnd1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t[3], p.bnd1, p.t1);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t[4], p.t0, p.t1);
        if (e != cudaSuccess) st = fail(FDIRW_E_CUDA, std::string("phase times: ") + cudaGetErrorString(e));
        for (int k = 0; k < 5; ++k) acc[k] += t[k];
    }
    release();
    if (st != FDIRW_OK) return st;
    for (int k = 0; k < 5; ++k) ms_out[k] = acc[k] / n_steps;
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_mass(fdirw_ctx* c, const float* c_dev, double* out_host, void* cuda_stream)
{
    if (!c || !c_dev || !out_host) return fail(FDIRW_E_INVALID, "NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const size_t n = (size_t)c->g.nx * c->g.ny * c->g.nzl;
    CUDA_TRY(launch_mass(c_dev, n, c->mass_partial, c->mass_blocks, c->mass_out, s));
    if (c->world > 1 && !c->is_virtual) {
        if (!c->comm)
            return fail(FDIRW_E_STATE, "fdirw_mass on a P2P rank without a communicator: call fdirw_comm_init "
                                       "first, or use fdirw_mass_local");
        std::string err;
        if (nccl_allreduce_sum_f64(c->nccl, c->comm, c->mass_out, s, &err)) return fail(FDIRW_E_NCCL, err);
    }
    CUDA_TRY(cudaMemcpyAsync(out_host, c->mass_out, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_comm_init(fdirw_ctx* c, const void* nccl_id)
{
    if (!c || !nccl_id) return fail(FDIRW_E_INVALID, "NULL argument");
    if (c->transport != FDIRW_TRANSPORT_P2P || c->world < 2)
        return fail(FDIRW_E_STATE, "fdirw_comm_init: a P2P context with world > 1 only (NCCL contexts own one)");
    if (c->comm) return fail(FDIRW_E_STATE, "fdirw_comm_init: the context already has a communicator");
    CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    if (!c->nccl) c->nccl = nccl_load(&err);
    if (!c->nccl) return fail(FDIRW_E_NCCL, err);
    c->comm = nccl_comm_init(c->nccl, c->world, c->rank, nccl_id, &err);
    if (!c->comm) return fail(FDIRW_E_NCCL, err);
    // connect now, outside any later stream capture
    if (nccl_allreduce_sum_f64(c->nccl, c->comm, c->mass_out, c->comm_stream, &err)) return fail(FDIRW_E_NCCL, err);
    CUDA_TRY(cudaStreamSynchronize(c->comm_stream));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_mass_local(fdirw_ctx* c, const float* c_dev, double* out_host, void* cuda_stream)
{
    if (!c || !c_dev || !out_host) return fail(FDIRW_E_INVALID, "NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const size_t n = (size_t)c->g.nx * c->g.ny * c->g.nzl;
    CUDA_TRY(launch_mass(c_dev, n, c->mass_partial, c->mass_blocks, c->mass_out, s));
    CUDA_TRY(cudaMemcpyAsync(out_host, c->mass_out, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_read_ceiling(const fdirw_ctx* c, int32_t reps, void* cuda_stream, double* gbps_out)
{
    if (!c || !gbps_out || reps < 1) return fail(FDIRW_E_INVALID, "NULL argument or reps < 1");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const Geometry& g = c->g;
    const uint64_t wt_tiles = (c->ut.chunk_u || c->compact) ? (uint64_t)c->ut.nd_tiles : (uint64_t)g.n_tiles;
    const size_t bytes = wbytes(c->fmt, (size_t)wt_tiles * (g.K - 1) * g.tile * kChunk) / 16 * 16;
    if (bytes == 0) return fail(FDIRW_E_STATE, "no weights to stream");
    int sms = 148;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    unsigned* sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    float best = 1e30f;
    cudaError_t e = cudaMalloc(&sink, 4);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    if (e == cudaSuccess) e = launch_read_stream(c->Wt, bytes, sink, sms, s);  // warm-up
    for (int r = 0; r < reps && e == cudaSuccess; ++r) {
        e = cudaEventRecord(e0, s);
        if (e == cudaSuccess) e = launch_read_stream(c->Wt, bytes, sink, sms, s);
        if (e == cudaSuccess) e = cudaEventRecord(e1, s);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e == cudaSuccess && ms < best) best = ms;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(sink);
    if (e != cudaSuccess) return fail(FDIRW_E_CUDA, std::string("read ceiling: ") + cudaGetErrorString(e));
    *gbps_out = (double)bytes / (best * 1e-3) / 1e9;
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_query(const fdirw_ctx* c, fdirw_info* info)
{
    if (!c || !info) return fail(FDIRW_E_INVALID, "NULL argument");
    const Geometry& g = c->g;
    info->n_fd = c->d.n_fd;
    info->K = g.K;
    info->z_begin = g.z0;
    info->z_end = g.z1;
    info->dt_fd = c->d.dt_fd;
    info->lambda_fast = c->d.lam_ff;
    info->lambda_fs = c->d.lam_fs;
    info->lambda_slow = c->d.lam_ss;
    const uint64_t wt_tiles = (c->ut.chunk_u || c->compact) ? (uint64_t)c->ut.nd_tiles : (uint64_t)g.n_tiles;  // N4 / N2 compact
    info->weight_bytes = wbytes(c->fmt, wt_tiles * (g.K - 1) * g.tile * kChunk) + wt_tiles * g.tile * kChunk * 8;
    info->state_bytes = (uint64_t)g.state_elems * 4 * 2;
    info->bytes_per_voxel_update = c->fmt == FDIRW_W_MX8 ? (uint64_t)((g.K - 1) * 9 + 4) / 8 + 16  // rounded
                                                         : (uint64_t)(g.K - 1) * c->b_w + 16;
    info->voxels = (uint64_t)g.nx * g.ny * g.nzl;
    info->tile_chunks = g.tile;
    info->n_tiles = g.n_tiles;
    info->kgen_sources = c->kgen_sources;
    info->kgen_windows = c->kgen_windows;
    info->kgen_steps = c->kgen_steps;
    info->kgen_kernel_ms = c->kgen_ms;
    info->chunks = (uint64_t)g.nzl * g.ny * g.nxq;
    info->uniform_chunks = (uint64_t)c->ut.n_uniform;
    info->uniform_classes = c->ut.n_u;
    return FDIRW_OK;
}

extern "C" void fdirw_destroy(fdirw_ctx* c) { free_ctx(c); }

extern "C" fdirw_status fdirw_make_plan(const fdirw_params* p, const fdirw_dist* dist, fdirw_plan* pl)
{
    static const uint8_t dummy = 0;
    fdirw_ctx* unused = nullptr;
    fdirw_status st = validate(p, &dummy, dist, &unused, false);
    if (st != FDIRW_OK) return st;
    if (!pl) return fail(FDIRW_E_INVALID, "NULL argument");
    Derived d;
    if ((st = derive(*p, &d)) != FDIRW_OK) return st;
    const int rank = dist ? dist->rank : 0, world = dist ? dist->world : 1;
    const Geometry g = make_geometry(p->nx, p->ny, p->nz, p->radius, dist ? dist->z_begin : 0,
                                     dist ? dist->z_end : p->nz,
                                     !(p->flags & FDIRW_F_DEDUP_STORAGE) && !(p->v_far > 0) && p->weights != FDIRW_W_MX8);
    const HaloPlan h = make_halo_plan(g, rank, world);
    int i0, i1;
    split_tiles(g, &i0, &i1);
    pl->z_begin = g.z0; pl->z_end = g.z1;
    pl->src_z_begin = g.sz0; pl->src_z_end = g.sz1;
    pl->mask_z_begin = g.mz0; pl->mask_z_end = g.mz1;
    pl->tile_chunks = g.tile; pl->tiles_per_plane = g.tpp; pl->n_tiles = g.n_tiles;
    pl->interior_tile_begin = world > 1 ? i0 : 0;
    pl->interior_tile_end = world > 1 ? i1 : g.n_tiles;
    pl->peer_lo = h.peer_lo; pl->peer_hi = h.peer_hi;
    pl->padded_x = g.nxp; pl->padded_y = g.nyp; pl->padded_z = g.nzp;
    pl->pad_x0 = kPadX;
    pl->halo_elems = h.count;
    pl->send_lo = h.send_lo; pl->recv_lo = h.recv_lo; pl->send_hi = h.send_hi; pl->recv_hi = h.recv_hi;
    pl->weight_bytes = (uint64_t)wbytes(p->weights, g.w_elems) + (uint64_t)g.diag_elems * 8;
    pl->state_bytes = (uint64_t)g.state_elems * 8;
    pl->n_fd = d.n_fd;
    std::vector<float> cheb;
    const int m = kgen_cheb(*p, d, &cheb);
    pl->kgen_steps = m > 0 ? kCheb_pre + m : d.n_fd;
    return FDIRW_OK;
}

extern "C" const char* fdirw_last_error(void) { return g_err.c_str(); }

#ifndef FDIRW_BUILD_ID
#define FDIRW_BUILD_ID "unknown"
#endif
extern "C" const char* fdirw_build_id(void) { return FDIRW_BUILD_ID; }

extern "C" fdirw_status fdirw_debug_stage_canary(fdirw_ctx* c, int32_t enable, uint64_t* checks, uint64_t* mismatches)
{
    if (!c || !checks || !mismatches) return fail(FDIRW_E_INVALID, "NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    if (enable && !c->canary) {
        fdirw_status st = alloc((void**)&c->canary, 16, "stage canary");
        if (st != FDIRW_OK) return st;
        CUDA_TRY(cudaMemset(c->canary, 0, 16));
        if (c->graph2) {  // the captured steps carry the old launch arguments
            cudaGraphExecDestroy(c->graph2);
            c->graph2 = nullptr;
        }
        if (c->graph_abs) {
            cudaGraphExecDestroy(c->graph_abs);
            c->graph_abs = nullptr;
        }
    }
    unsigned long long h[2] = {0, 0};
    if (c->canary) CUDA_TRY(cudaMemcpy(h, c->canary, 16, cudaMemcpyDeviceToHost));
    *checks = h[0];
    *mismatches = h[1];
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_debug_upload_weights(fdirw_ctx* c, const double* k)
{
    if (!c || !k) return fail(FDIRW_E_INVALID, "NULL argument");
    if (c->world != 1) return fail(FDIRW_E_STATE, "debug upload needs world == 1");
    if (c->ut.chunk_u || c->compact) return fail(FDIRW_E_STATE, "debug upload needs the dense layout");
    if (c->fmt == FDIRW_W_MX8) return fail(FDIRW_E_STATE, "debug upload does not write MX8 weights");
    CUDA_TRY(cudaSetDevice(c->device));
    const Geometry& g = c->g;
    const int R = g.R, L = g.L, K = g.K;
    std::vector<unsigned char> wt(g.w_elems * c->b_w, 0);
    std::vector<float2> dg(g.diag_elems, make_float2(0.f, 0.f));
    for (int sz = 0; sz < g.nz; ++sz)
        for (int sy = 0; sy < g.ny; ++sy)
            for (int sx = 0; sx < g.nx; ++sx) {
                const double* ks = k + (((size_t)sz * g.ny + sy) * g.nx + sx) * K;
                for (int o = 0; o < K; ++o) {
                    const int ox = o % L - R, oy = (o / L) % L - R, oz = o / (L * L) - R;
                    const int x = sx + ox, y = sy + oy, z = sz + oz;
                    if (x < 0 || x >= g.nx || y < 0 || y >= g.ny || z < 0 || z >= g.nz) continue;
                    const int q = y * g.nxq + (x >> 3);
                    const size_t tile = (size_t)z * g.tpp + q / g.tile;
                    const int e = q % g.tile, j = x & 7;
                    if (o == K / 2) {
                        dg[(tile * g.tile + e) * 8 + j] = fp32_pair(ks[o]);
                        continue;
                    }
                    const size_t idx = ((tile * (size_t)(K - 1) + slot_of(ox, oy, oz, R)) * g.tile + e) * 8 + j;
                    const float f = (float)ks[o];
                    if (c->fmt == FDIRW_W_FP32) {
                        memcpy(&wt[idx * 4], &f, 4);
                    } else if (c->fmt == FDIRW_W_FP16) {
                        const __half h = __float2half_rn(f);
                        memcpy(&wt[idx * 2], &h, 2);
                    } else {
                        const __nv_bfloat16 h = __float2bfloat16_rn(f);
                        memcpy(&wt[idx * 2], &h, 2);
                    }
                }
            }
    CUDA_TRY(cudaMemcpy(c->Wt, wt.data(), wt.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->diag, dg.data(), dg.size() * 8, cudaMemcpyHostToDevice));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_export_kernels(const fdirw_ctx* c, const int32_t* box, double* out)
{
    if (!c || !box || !out) return fail(FDIRW_E_INVALID, "NULL argument");
    if (box[1] < box[0] || box[3] < box[2] || box[5] < box[4]) return fail(FDIRW_E_INVALID, "bad box");
    if (c->ut.chunk_u) return fail(FDIRW_E_STATE, "export needs the dense layout (FDIRW_F_DEDUP_STORAGE compacts it)");
    CUDA_TRY(cudaSetDevice(c->device));
    const size_t n = (size_t)(box[1] - box[0]) * (box[3] - box[2]) * (box[5] - box[4]) * c->g.K;
    if (n == 0) return FDIRW_OK;
    double* d = nullptr;
    fdirw_status st = alloc((void**)&d, n * 8, "export buffer");
    if (st != FDIRW_OK) return st;
    cudaError_t e = launch_export(c->Wt, c->diag, c->g, c->fmt, box, d, nullptr, c->compact ? c->chunk_pos : nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(out, d, n * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(FDIRW_E_CUDA, std::string("export: ") + cudaGetErrorString(e));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_step_virtual(fdirw_ctx* const* ctxs, int32_t n, const float* const* c_in,
                                           float* const* c_out, void* cuda_stream)
{
    if (!ctxs || !c_in || !c_out || n < 1) return fail(FDIRW_E_INVALID, "NULL argument");
    for (int r = 0; r < n; ++r) {
        if (!ctxs[r] || !c_in[r] || !c_out[r]) return fail(FDIRW_E_INVALID, "NULL argument");
        if (ctxs[r]->world != n || ctxs[r]->rank != r) return fail(FDIRW_E_INVALID, "contexts must be ranks 0..n-1");
        if (n > 1 && !ctxs[r]->is_virtual) return fail(FDIRW_E_STATE, "not a virtual-rank context");
        if (ctxs[r]->device != ctxs[0]->device) return fail(FDIRW_E_INVALID, "virtual ranks share one device");
        if (c_in[r] == c_out[r]) return fail(FDIRW_E_ALIAS, "c_in == c_out");
    }
    CUDA_TRY(cudaSetDevice(ctxs[0]->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    for (int r = 0; r < n; ++r) CUDA_TRY(launch_pack(c_in[r], ctxs[r]->cpad[0], ctxs[r]->g, s, ctxs[r]->farmask));
    // halo planes by device copies: the planes NCCL would move (same HaloPlan as comm.cpp)
    for (int r = 0; r < n; ++r) {
        const HaloPlan h = make_halo_plan(ctxs[r]->g, r, n);
        const size_t bytes = (size_t)h.count * 4;
        if (h.peer_lo >= 0) {
            const HaloPlan hl = make_halo_plan(ctxs[h.peer_lo]->g, h.peer_lo, n);
            CUDA_TRY(cudaMemcpyAsync(ctxs[r]->cpad[0] + h.recv_lo, ctxs[h.peer_lo]->cpad[0] + hl.send_hi, bytes,
                                     cudaMemcpyDeviceToDevice, s));
        }
        if (h.peer_hi >= 0) {
            const HaloPlan hh = make_halo_plan(ctxs[h.peer_hi]->g, h.peer_hi, n);
            CUDA_TRY(cudaMemcpyAsync(ctxs[r]->cpad[0] + h.recv_hi, ctxs[h.peer_hi]->cpad[0] + hh.send_lo, bytes,
                                     cudaMemcpyDeviceToDevice, s));
        }
    }
    for (int r = 0; r < n; ++r) {
        fdirw_ctx* c = ctxs[r];
        const Geometry& g = c->g;
        int i0, i1;
        split_tiles(g, &i0, &i1);
        const long ps = (long)g.nx * g.ny, rs = g.nx;
        if (i1 > i0) {
            CUDA_TRY(superpose(c, c->cpad[0], c_out[r], ps, rs, i0, i1, s));
            CUDA_TRY(superpose(c, c->cpad[0], c_out[r], ps, rs, 0, i0, s));
            CUDA_TRY(superpose(c, c->cpad[0], c_out[r], ps, rs, i1, g.n_tiles, s));
        } else {
            CUDA_TRY(superpose(c, c->cpad[0], c_out[r], ps, rs, 0, g.n_tiles, s));
        }
    }
    if (ctxs[0]->far) CUDA_TRY(virtual_gather(ctxs, n, s, 0, 0.0));
    return FDIRW_OK;
}

// N2 on virtual ranks: every context gathers all ranks' tile sums (the NCCL all-gather's
// bytes) and runs the same Eq.7 reduction.
static cudaError_t virtual_gather(fdirw_ctx* const* ctxs, int n, cudaStream_t s, int mode, double c_far0)
{
    for (int r = 0; r < n; ++r) {
        for (int q = 0; q < n; ++q) {
            cudaError_t e = cudaMemcpyAsync(ctxs[r]->gathered + (long)q * ctxs[r]->tile_stride, ctxs[q]->tile_buf,
                                            ctxs[q]->tile_stride * 8, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = launch_far_reduce(ctxs[r]->gathered, n, ctxs[r]->tile_stride, ctxs[r]->far_state,
                                          ctxs[r]->v_far, c_far0, mode, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

extern "C" fdirw_status fdirw_far_init(fdirw_ctx* c, const float* c_dev, double c_far0, double* M0_out,
                                       void* cuda_stream)
{
    if (!c || !c_dev) return fail(FDIRW_E_INVALID, "NULL argument");
    if (!c->far) return fail(FDIRW_E_STATE, "closed-domain context (v_far = 0)");
    if (c->is_virtual) return fail(FDIRW_E_STATE, "virtual-rank context: use fdirw_far_init_virtual");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    CUDA_TRY(launch_tile_mass(c_dev, c->farmask, c->g, c->tile_buf + 1, s));
    fdirw_status st = far_reduce(c, s, 1, c_far0);
    if (st != FDIRW_OK) return st;
    double fs[2];
    CUDA_TRY(cudaMemcpyAsync(fs, c->far_state, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (M0_out) *M0_out = fs[1];
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_far_init_virtual(fdirw_ctx* const* ctxs, int32_t n, const float* const* c_dev,
                                               double c_far0, double* M0_out, void* cuda_stream)
{
    if (!ctxs || !c_dev || n < 1) return fail(FDIRW_E_INVALID, "NULL argument");
    for (int r = 0; r < n; ++r)
        if (!ctxs[r] || !ctxs[r]->far || ctxs[r]->world != n || ctxs[r]->rank != r)
            return fail(FDIRW_E_STATE, "need far-field contexts of ranks 0..n-1");
    CUDA_TRY(cudaSetDevice(ctxs[0]->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    for (int r = 0; r < n; ++r)
        CUDA_TRY(launch_tile_mass(c_dev[r], ctxs[r]->farmask, ctxs[r]->g, ctxs[r]->tile_buf + 1, s));
    CUDA_TRY(virtual_gather(ctxs, n, s, 1, c_far0));
    double fs[2];
    CUDA_TRY(cudaMemcpyAsync(fs, ctxs[0]->far_state, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (M0_out) *M0_out = fs[1];
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_set_precision_mode(fdirw_ctx* c, int32_t mode)
{
    if (!c) return fail(FDIRW_E_INVALID, "NULL argument");
    if (mode < 0 || mode > 3) return fail(FDIRW_E_INVALID, "precision mode must be 0..3");
    if (mode != 0 && c->world != 1) return fail(FDIRW_E_STATE, "precision study modes need world == 1");
    if (mode != 0 && c->ut.chunk_u) return fail(FDIRW_E_STATE, "precision study modes need the dense layout");
    if (mode == 1 && c->fmt != FDIRW_W_FP32) return fail(FDIRW_E_STATE, "mode 1 (fp32) needs FP32 weights");
    if ((mode == 2 || mode == 3) && c->fmt != FDIRW_W_FP16)
        return fail(FDIRW_E_STATE, "modes 2/3 (paper mixed / fp16) need FP16 weights");
    if (c->graph2) {  // the captured step depends on the mode
        cudaGraphExecDestroy(c->graph2);
        c->graph2 = nullptr;
    }
    if (c->graph_abs) {
        cudaGraphExecDestroy(c->graph_abs);
        c->graph_abs = nullptr;
    }
    c->prec_mode = mode;
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_absorb_run(fdirw_ctx* c, const fdirw_absorb_params* ap, float* c_dev, int32_t n,
                                         double* kinetics_host, void* cuda_stream)
{
    if (!c || !ap || !c_dev) return fail(FDIRW_E_INVALID, "NULL argument");
    if (n < 0) return fail(FDIRW_E_INVALID, "n_steps must be >= 0");
    if (c->world != 1 || !c->phase_pp) return fail(FDIRW_E_STATE, "the integrated loop needs world == 1");
    if (!(ap->D_S >= 0) || !(ap->k >= 0) || !(ap->c_S_eq > 0) || !(ap->c_L_eq > 0))
        return fail(FDIRW_E_INVALID, "need D_S >= 0, k >= 0, c_S_eq > 0, c_L_eq > 0");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const Geometry& g = c->g;
    AbsorbArgs ab{};
    const double dt = c->p.dt, dh = c->p.dh;
    if (ap->D_S > 0) {  // component (3): λ_S ≤ λ* = 0.1 (reading A5 applied to the solid)
        const double x = ap->D_S * dt / (0.1 * dh * dh);
        const double nn = std::ceil(x * (1.0 - 1e-9));
        ab.n_s = nn < 1.0 ? 1 : (int)nn;
        ab.lam_s = (float)(ap->D_S * (dt / ab.n_s) / (dh * dh));
    }
    ab.kdt = (float)(ap->k * dt);
    ab.cSeq = (float)ap->c_S_eq;
    ab.cLeq = (float)ap->c_L_eq;
    ab.n_solid = c->n_solid;
    fdirw_status st;
    if (!c->alpha) {  // (zeroed once: the grouped apply loads whole neighbour groups, whose α it uses
                      // only for interface liquid lanes — always written — so the rest is never read uninitialised)
        if ((st = alloc((void**)&c->alpha, g.state_elems * 4, "reaction scratch")) != FDIRW_OK) return st;
        CUDA_TRY(cudaMemsetAsync(c->alpha, 0, g.state_elems * 4, static_cast<cudaStream_t>(cuda_stream)));
    }
    if (!c->kin_part && (st = alloc((void**)&c->kin_part, 4 * kAbsorbMaxBlocks * 8, "kinetics")) != FDIRW_OK) return st;
    if (n > c->kin_cap) {
        cudaFree(c->kin_rec);
        c->kin_rec = nullptr;
        if ((st = alloc((void**)&c->kin_rec, (size_t)n * 4 * 8, "kinetics record")) != FDIRW_OK) return st;
        c->kin_cap = n;
    }
    if (n == 0) return FDIRW_OK;
    if (!c->abs_ctr && (st = alloc((void**)&c->abs_ctr, 4, "kinetics counter")) != FDIRW_OK) return st;
    if (!c->iface.list) CUDA_TRY(build_iface_list(c->phase_pp, g, &c->iface, s));
    // the nf path (one solid pass over the non-far groups, reading the solid values from the
    // liquid step's input, so the step skips its identity-chunk copy): Table 1's single solid pass
    // with the product kernel (the §3.3 study modes round even the identity rows' products);
    // FDIRW_ABSORB_SCALAR / FDIRW_ABSORB_SWEEP / FDIRW_ABSORB_FULL
    // keep the sweeping forms for A/B
    ab.nf_path = (ab.n_s == 1 && c->prec_mode == 0 && c->iface.nf_list && !getenv("FDIRW_ABSORB_SCALAR") &&
                  !getenv("FDIRW_ABSORB_SWEEP") && !getenv("FDIRW_ABSORB_FULL")) ? 1 : 0;
    CUDA_TRY(launch_pack(c_dev, c->cpad[0], g, s, c->farmask));
    CUDA_TRY(cudaMemsetAsync(c->abs_ctr, 0, 4, s));
    const size_t ioff = (size_t)g.R * g.plane_elems + (size_t)g.R * g.nxp + kPadX;
    // one macro step from `in`: (1) the liquid FDiRW step, (2)-(5) the tail; returns the buffer
    // holding the result (which of the two depends on the number of solid FD passes)
    auto macro = [&](float* in, cudaStream_t ss, float** res) -> fdirw_status {
        float* out = in == c->cpad[0] ? c->cpad[1] : c->cpad[0];
        fdirw_status sst = enqueue_step(c, in, out + ioff, (long)g.plane_elems, g.nxp, ss, 1, nullptr,
                                        getenv("FDIRW_ABSORB_EQ7_TWICE") != nullptr,  // (A/B)
                                        ab.nf_path == 0);
        if (sst != FDIRW_OK) return sst;
        CUDA_TRY(launch_absorb_tail(out, in, c->alpha, c->phase_pp, g, ab, c->kin_part, c->far_state, c->v_far,
                                    c->far ? 1 : 0, c->kin_rec, ss, res, c->abs_ctr, &c->iface));
        return FDIRW_OK;
    };
    const bool same = c->graph_abs && c->abs_rec_key == c->kin_rec && c->abs_key.n_s == ab.n_s &&
                      c->abs_key.lam_s == ab.lam_s && c->abs_key.kdt == ab.kdt && c->abs_key.cSeq == ab.cSeq &&
                      c->abs_key.cLeq == ab.cLeq && c->abs_key.n_solid == ab.n_solid &&
                      c->abs_key.nf_path == ab.nf_path;
    if (n >= 2 && !same) {  // capture two macro steps: they return the field to cpad[0]
        if (c->graph_abs) cudaGraphExecDestroy(c->graph_abs);
        c->graph_abs = nullptr;
        cudaStream_t cs = c->capture_stream;
        CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        float *r1 = nullptr, *r2 = nullptr;
        st = macro(c->cpad[0], cs, &r1);
        if (st == FDIRW_OK) st = macro(r1, cs, &r2);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        if (st != FDIRW_OK) { if (graph) cudaGraphDestroy(graph); return st; }
        if (e != cudaSuccess) return fail(FDIRW_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        if (r2 != c->cpad[0]) { cudaGraphDestroy(graph); return fail(FDIRW_E_STATE, "absorb: two steps must return to the first buffer"); }
        e = cudaGraphInstantiate(&c->graph_abs, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) { c->graph_abs = nullptr; return fail(FDIRW_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e)); }
        c->abs_key = ab;
        c->abs_rec_key = c->kin_rec;
    }
    for (int i = 0; i < n / 2; ++i) CUDA_TRY(cudaGraphLaunch(c->graph_abs, s));
    float* fin = c->cpad[0];
    if (n & 1) {
        float* res = nullptr;
        if ((st = macro(c->cpad[0], s, &res)) != FDIRW_OK) return st;
        fin = res;
    }
    CUDA_TRY(launch_unpack(fin, c_dev, g, s));
    if (kinetics_host) CUDA_TRY(cudaMemcpyAsync(kinetics_host, c->kin_rec, (size_t)n * 32, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_far_get(fdirw_ctx* c, double* c_far_out, void* cuda_stream)
{
    if (!c || !c_far_out) return fail(FDIRW_E_INVALID, "NULL argument");
    if (!c->far) return fail(FDIRW_E_STATE, "closed-domain context (v_far = 0)");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    CUDA_TRY(cudaMemcpyAsync(c_far_out, c->far_state, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FDIRW_OK;
}

// ---- a6 over peer memory: attach -----------------------------------------------------------
namespace {
struct P2PBlob {
    uint32_t magic;
    int32_t rank, world, nx, ny, R, nzl, device;
    cudaIpcMemHandle_t cpad[2];
    cudaIpcMemHandle_t flags;
};
static_assert(sizeof(P2PBlob) <= FDIRW_P2P_BLOB_BYTES, "blob");
constexpr uint32_t kBlobMagic = 0xFD1B2B01u;
}  // namespace

extern "C" fdirw_status fdirw_p2p_export(fdirw_ctx* c, void* blob_out)
{
    if (!c || !blob_out) return fail(FDIRW_E_INVALID, "NULL argument");
    if (c->transport != FDIRW_TRANSPORT_P2P || c->world < 2) return fail(FDIRW_E_STATE, "not a P2P context with world > 1");
    CUDA_TRY(cudaSetDevice(c->device));
    P2PBlob b{};
    b.magic = kBlobMagic;
    b.rank = c->rank; b.world = c->world; b.nx = c->g.nx; b.ny = c->g.ny; b.R = c->g.R; b.nzl = c->g.nzl;
    b.device = c->device;
    CUDA_TRY(cudaIpcGetMemHandle(&b.cpad[0], c->cpad[0]));
    CUDA_TRY(cudaIpcGetMemHandle(&b.cpad[1], c->cpad[1]));
    CUDA_TRY(cudaIpcGetMemHandle(&b.flags, c->p2p_flags));
    memset(blob_out, 0, FDIRW_P2P_BLOB_BYTES);
    memcpy(blob_out, &b, sizeof b);
    return FDIRW_OK;
}

static fdirw_status p2p_check_blob(const fdirw_ctx* c, const P2PBlob& b, int want_rank)
{
    if (b.magic != kBlobMagic) return fail(FDIRW_E_INVALID, "not an fdirw P2P blob");
    if (b.rank != want_rank || b.world != c->world) return fail(FDIRW_E_INVALID, "P2P blob from the wrong rank/world");
    if (b.nx != c->g.nx || b.ny != c->g.ny || b.R != c->g.R) return fail(FDIRW_E_INVALID, "P2P blob geometry mismatch");
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_p2p_attach(fdirw_ctx* c, const void* lo_blob, const void* hi_blob)
{
    if (!c) return fail(FDIRW_E_INVALID, "NULL argument");
    if (c->transport != FDIRW_TRANSPORT_P2P || c->world < 2) return fail(FDIRW_E_STATE, "not a P2P context with world > 1");
    if ((c->rank > 0) != (lo_blob != nullptr) || (c->rank < c->world - 1) != (hi_blob != nullptr))
        return fail(FDIRW_E_INVALID, "need lo_blob iff rank > 0 and hi_blob iff rank < world-1");
    CUDA_TRY(cudaSetDevice(c->device));
    for (int side = 0; side < 2; ++side) {
        const void* blob = side == 0 ? lo_blob : hi_blob;
        if (!blob) continue;
        P2PBlob b;
        memcpy(&b, blob, sizeof b);
        fdirw_status st = p2p_check_blob(c, b, c->rank + (side == 0 ? -1 : 1));
        if (st != FDIRW_OK) return st;
        void* q[3];
        const cudaIpcMemHandle_t hs[3] = {b.cpad[0], b.cpad[1], b.flags};
        for (int i = 0; i < 3; ++i) {
            CUDA_TRY(cudaIpcOpenMemHandle(&q[i], hs[i], cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(q[i]);
        }
        if (side == 0) {
            c->peer_lo[0] = (float*)q[0];
            c->peer_lo[1] = (float*)q[1];
            c->peer_lo_flag = (unsigned long long*)q[2] + 1;  // we are its hi neighbour
            c->nzl_lo = b.nzl;
        } else {
            c->peer_hi[0] = (float*)q[0];
            c->peer_hi[1] = (float*)q[1];
            c->peer_hi_flag = (unsigned long long*)q[2] + 0;  // we are its lo neighbour
        }
    }
    c->p2p_ready = true;
    return capture_graph2(c);
}

extern "C" fdirw_status fdirw_p2p_attach_local(fdirw_ctx* const* ctxs, int32_t n)
{
    if (!ctxs || n < 2) return fail(FDIRW_E_INVALID, "need >= 2 contexts");
    for (int r = 0; r < n; ++r) {
        fdirw_ctx* c = ctxs[r];
        if (!c || c->transport != FDIRW_TRANSPORT_P2P || c->world != n || c->rank != r)
            return fail(FDIRW_E_INVALID, "contexts must be P2P ranks 0..n-1 of one world, in order");
        if (c->g.nx != ctxs[0]->g.nx || c->g.ny != ctxs[0]->g.ny || c->g.R != ctxs[0]->g.R)
            return fail(FDIRW_E_INVALID, "geometry mismatch");
    }
    for (int r = 0; r < n; ++r) {
        fdirw_ctx* c = ctxs[r];
        if (r > 0) {
            c->peer_lo[0] = ctxs[r - 1]->cpad[0];
            c->peer_lo[1] = ctxs[r - 1]->cpad[1];
            c->peer_lo_flag = ctxs[r - 1]->p2p_flags + 1;
            c->nzl_lo = ctxs[r - 1]->g.nzl;
        }
        if (r < n - 1) {
            c->peer_hi[0] = ctxs[r + 1]->cpad[0];
            c->peer_hi[1] = ctxs[r + 1]->cpad[1];
            c->peer_hi_flag = ctxs[r + 1]->p2p_flags + 0;
        }
        c->p2p_ready = true;
    }
    for (int r = 0; r < n; ++r) {
        CUDA_TRY(cudaSetDevice(ctxs[r]->device));
        fdirw_status st = capture_graph2(ctxs[r]);
        if (st != FDIRW_OK) return st;
    }
    return FDIRW_OK;
}

extern "C" fdirw_status fdirw_p2p_check(fdirw_ctx* c, int32_t* timed_out, void* cuda_stream)
{
    if (!c || !timed_out) return fail(FDIRW_E_INVALID, "NULL argument");
    *timed_out = 0;
    if (!c->p2p_flags) return FDIRW_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    unsigned long long f[4];
    CUDA_TRY(cudaMemcpyAsync(f, c->p2p_flags, 32, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *timed_out = f[3] ? 1 : 0;
    return FDIRW_OK;
}
