// fdirw_internal.h — internal types shared by the FDiRW CUDA sources (not part of the ABI).
#pragma once
#include <vector>

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/fdirw.h"

namespace fdirw {

constexpr int kChunk = 8;     // targets per superposition thread (8 consecutive x)
constexpr int kPadX = 8;      // x padding of the padded state (≥ R_max so [x−8, x+16) is in range)
constexpr int kMaxR = 8;

// Target-slab geometry and the gather layout of the weights.
//   chunk q (within a plane) = y·nxq + x/8; tile tp = q / tile; element e = q % tile; j = x % 8
//   tile index t = (z − z0)·tpp + tp
//   Wt[t][slot][e][j] (slot = window offset o minus the centre), diag[t][e][j] fp32 pair (hi, lo) = float2 (reading A10)
//   padded state: [nzl + 2R][ny + 2R][nxp], nxp = 8·nxq + 16, x offset kPadX
struct Geometry {
    int nx, ny, nz, R, L, K;
    int z0, z1, nzl;
    int nxq, cpp, tile, tpp, n_tiles;
    int nxp, nyp, nzp;
    size_t plane_elems, state_elems;
    size_t w_elems, diag_elems;  // element counts of Wt and diag
    int mz0, mz1;                // device mask planes [mz0, mz1)
    int sz0, sz1;                // source planes whose windows reach the slab
};

// The diagonal d_s = M − Σ_{o≠0} W̃_s(o) (fp64) stored as an fp32 pair (reading A10): hi = RNE_fp32(d),
// lo = RNE_fp32(d − hi), so a stored column sums to M within ~2^-48 (one fp32 diagonal rounds d
// the same way for a whole class of identical windows: a mass bias of ~1e-8 per step).
__host__ __device__ inline float2 fp32_pair(double d)
{
    const float hi = (float)d;
    return make_float2(hi, (float)(d - (double)hi));
}

Geometry make_geometry(int nx, int ny, int nz, int R, int z0, int z1, bool balance = false);

// a6: which padded planes move where (element offsets into the padded state; −1 = no peer).
//   send padded planes [R, 2R)        → rank−1    recv padded [0, R)          ← rank−1
//   send padded planes [nzl, nzl+R)   → rank+1    recv padded [nzl+R, nzl+2R) ← rank+1
struct HaloPlan {
    long count;  // fp32 elements per message (R whole padded planes, contiguous)
    int peer_lo, peer_hi;
    long send_lo, recv_lo, send_hi, recv_hi;
};
HaloPlan make_halo_plan(const Geometry& g, int rank, int world);

struct Derived {
    int n_fd;
    double dt_fd, lam_ff, lam_fs, lam_ss;
};

// Chebyshev evaluation of x^n on the spectrum [1 − 12λ_max, 1] of an explicit-FD operator
// (fdirw_api.cu, reading A30): coefficients c_0..c_m (fp32) with tail ≤ 1e-10; returns m,
// 0 when the recurrence would not save work.  kgen and the coarse P columns run
// kCheb_pre literal substeps first.
int cheb_plan(int n, double lam_max, std::vector<float>* coef);
constexpr int kCheb_pre = 8;

// ---- kernels (kgen.cu / superpose.cu) --------------------------------------------
struct KgenArgs {
    const uint8_t* mask;  // device planes [mz0, mz1) × ny × nx
    int mz0;
    int nx, ny, nz;
    int sz0, sz1;         // source planes
    int z0, z1;           // target slab
    float lam_ff, lam_fs, lam_ss;
    double lam_d[3];      // {ff, fs, ss} in fp64 (FDIRW_F_KGEN_FP64)
    int fp64;             // FDIRW_F_KGEN_FP64: fp64 substeps in the oracle's order (reading A22)
    int symmetric;        // FDIRW_F_SYMMETRIC_RULE: write W_s(o) as target s's slot −o (reading A24)
    int n_fd;
    // Chebyshev evaluation of A^{n_fd − cheb_pre} (kgen.cu, reading A30): degree cheb_m (0 =
    // direct substeps), coefficients cheb_c[0..cheb_m] (device, fp32), face numbers 2μ = 4λ/(1 − a)
    int cheb_m, cheb_pre;  // Chebyshev degree (0 = direct) after cheb_pre direct substeps
    float cheb_scale = 1.f;  // 1 / Σ_k fp32(c_k) in fp64: an open window's result is scaled by it (A30)
    int cheb_open = 0;     // windows touching the N2 reservoir also take the recurrence (reduced-
                           // precision storage only, reading A30); else they run the literal substeps
    const float* cheb_c;
    float mu2_ff, mu2_fs, mu2_ss;
    int fmt, mass_fix;
    int columns = 0;      // FDIRW_F_KGEN_COLUMNS: the one-column-per-thread kernel at R = 5 (A/B)
    void* Wt;
    float2* diag;
    int nxq, tile, tpp, K;
    // class mode (dedup.cu): process src_list[0..n_list) (linear source indices within
    // planes [sz0, sz1)) and write class-major class_w[i][K] (storage format) + class_diag[i]
    const int* src_list;
    long n_list;
    void* class_w;
    float2* class_diag;
    double* class_mass = nullptr;  // MX8: each class kernel's own mass M (1 closed; < 1 open, N2)
};
cudaError_t launch_kgen(const KgenArgs& a, int R, cudaStream_t s);
cudaError_t launch_kgen_bal(const KgenArgs& a, int R, cudaStream_t s);    // R = 5, 8 (kgen_bal.cu)

// ---- a6 over peer memory (p2p.cu) -------------------------------------------------
cudaError_t p2p_preload();  // loads every kernel a P2P step launches (lazy loading can wait for the device)
cudaError_t p2p_wait(unsigned long long* flags, bool has_lo, bool has_hi, cudaStream_t s);
cudaError_t p2p_signal(unsigned long long* flags, unsigned long long* peer_lo_flag, unsigned long long* peer_hi_flag,
                       cudaStream_t s);
cudaError_t p2p_push_planes(const Geometry& g, const float* cpad, float* peer_lo, int nzl_lo, float* peer_hi,
                            cudaStream_t s);

// ---- window de-duplication (dedup.cu) -------------------------------------------
struct DedupArgs {
    const uint8_t* mask;
    int mz0, nx, ny, nz, R;
    int sz0, sz1, z0;
    int nxp, nyp;
    int* class_pad;  // padded-state layout, pre-filled with −1
};
struct DedupResult {
    long n_src = 0, n_class = 0;
    int* rep = nullptr;  // device [n_class]: representative source (linear index in [sz0, sz1))
    bool collision = false;
};
cudaError_t dedup_classify(const DedupArgs& a, DedupResult* res, cudaStream_t s);

struct UniformTables;
struct ExpandArgs {
    const int* class_pad;
    const void* class_w;
    const float2* class_diag;
    void* Wt;
    float2* diag;
    int nx, ny, nxq, tile, tpp, n_tiles, nxp, nyp;
    const int* list = nullptr;  // N4: compacted chunk ids (null = tile/e is the chunk)
    long n_list = 0;
    UniformTables* ut = nullptr;  // MX8 with N4 storage: the uniform tables (quantised in place)
    int nzl = 0;                  // MX8: slab planes (the diagonal pass walks every source)
    int z0 = 0, nz = 0;           // MX8: the slab's first global plane, the grid's planes
    const double* class_mass = nullptr;  // MX8: M per class (diagonal = M − Σ off-centre)
    const int* far_pos = nullptr;        // MX8 + N2 compaction: chunk_pos (≥ 0 compact, < 0 none)
};
cudaError_t launch_expand(const ExpandArgs& a, int R, int fmt, cudaStream_t s);
// N4: per-chunk uniform class tables (see superpose.cu); arrays are cudaMalloc'ed
struct UniformTables;
cudaError_t build_uniform(const ExpandArgs& a, int R, int fmt, long n_class, UniformTables* t, cudaStream_t s);

struct SuperArgs {
    const float* cpad;   // padded state, pointer to padded plane 0
    const void* Wt;
    const float2* diag;
    float* out;          // output element (z=0 of slab, y=0, x=0)
    long out_ps, out_rs; // output plane / row strides (elements)
    int nx, ny, nxq, tile, tpp, K;
    int nxp, nyp;        // padded row length, rows per padded plane
    int t_begin, t_end;  // tile range (CTA b → tile t_begin + b, plus gap_len once ≥ gap_at)
    int gap_at = 0, gap_len = 0;  // one launch over [t0, i0) ∪ [i1, t1): the slab's two boundary bands
    bool gap_last = false;        // ... followed by the gap [i0, i1) itself: every tile, boundary bands first
    // N2 (far field): + pbc·far_state[0] per target, per-tile Σ C_new into tile_sum[tile]
    const float* pbc = nullptr;
    const double* far_state = nullptr;  // {c_far, M0}
    double* tile_sum = nullptr;
    // N4 (uniform-chunk weight dedup): per chunk the uniform class u (−1: use Wt), and the
    // replicated class kernels uk8[u][slot][8]
    const int* list = nullptr;  // compacted chunk ids (orig tile·tile + e); tiles index the list
    long n_list = 0;
    // a6 over peer memory (FDIRW_TRANSPORT_P2P): targets in the first / last R slab planes are
    // also stored into the lo / hi neighbour's padded state (their next-step halo planes).
    // push_lo → the lo neighbour's padded plane (nzl_lo + R), row R, x offset kPadX;
    // push_hi → the hi neighbour's padded plane 0, row R, x offset kPadX
    float* push_lo = nullptr;
    float* push_hi = nullptr;
    int nzl = 0, pR = 0;
    bool no_bulk = false;  // FDIRW_F_NO_BULK_STREAM: weights by per-thread loads, not TMA stages
    // test support (fdirw_debug_stage_canary): the staged stream re-reads every weight a compute
    // thread takes from a stage — once after the stage's full barrier, once more just before the
    // thread's warp releases the stage — and compares both with the global copy: {checks,
    // mismatches}.  Null on every normal launch.
    unsigned long long* canary = nullptr;
};
cudaError_t launch_superpose(const SuperArgs& a, int R, int fmt, cudaStream_t s);
cudaError_t launch_read_stream(const void* p, size_t bytes, unsigned* sink, int sms, cudaStream_t s);
// identity rows (N2 compaction with D_slow = 0): out(chunk) = C_old(chunk) for the listed chunks
cudaError_t launch_copy_chunks(const float* cpad, float* out, long out_ps, long out_rs, const int* list, long n,
                               const Geometry& g, cudaStream_t s);

// N4: uniform chunks, one CTA per block of ≤ 256 chunks of one class (superpose.cu)
struct UniArgs {
    const float* cpad;
    float* out;
    long out_ps, out_rs;
    int nx, ny, nxq, tile, tpp, nxp, nyp;
    const int* list;      // uniform chunk ids (tile·tile_sz + e), grouped by class
    const int4* blocks;   // {start in list, count ≤ 256, class u, 0}
    int n_blocks;
    const float* ukf;     // [u][K−1] class kernels in slot order, decoded to fp32
    const float2* udiag;  // [u] fp32-pair diagonal (hi, lo)
    const float2* udiag_t = nullptr;  // MX8: per-target diagonal [list position][8] (replaces udiag)
};
cudaError_t launch_superpose_uniform(const UniArgs& a, int R, cudaStream_t s);
cudaError_t launch_superpose_mixed(const SuperArgs& a, const UniArgs& u, int R, int fmt, cudaStream_t s);

struct UniformTables {
    int* chunk_u = nullptr;   // [n_tiles·tile] class u or −1
    float* ukf = nullptr;
    float2* udiag = nullptr;
    int* list = nullptr;
    int4* blocks = nullptr;
    int n_blocks = 0, n_u = 0;
    long n_uniform = 0;
    int* dense_list = nullptr;  // real non-uniform chunks (chunk order), compacted into tiles
    long n_dense = 0;
    int nd_tiles = 0;
    // MX8: a target's diagonal depends on its neighbours' blocks, so uniform
    // chunks carry a per-target diagonal; chunk_map = compact index (≥ 0) or −(list pos + 2)
    float2* udiag_t = nullptr;
    int* chunk_map = nullptr;
};

// ---- N3 integrated loop + precision modes (absorb.cu) --------------------------------
// the tail sweeps launch at most this many blocks; react_apply writes 2 doubles of kinetics
// partial sums per block, so the partial buffer holds 2·kAbsorbMaxBlocks doubles
constexpr long kAbsorbMaxBlocks = 148L * 16;
struct AbsorbArgs {
    int n_s;          // solid FD substeps per macro step
    float lam_s;      // D_S·A_S/RT · (Δt/n_s) / Δh²
    float kdt;        // k·Δt (Eq.4)
    float cSeq, cLeq;
    double n_solid;   // N_S (for c̄_S)
    // 1: the liquid step skipped the identity-chunk copy (its output holds stale values at the
    // all-solid chunks); the tail's single solid pass reads the solid values from the step's
    // input and visits only the non-far groups (n_s == 1, the interface lists built)
    int nf_path = 0;
};
cudaError_t launch_phase_pad(const uint8_t* mask, const Geometry& g, uint8_t* pp, cudaStream_t s);
// the loop's interface groups (absorb.cu): groups of 4 x-voxels holding a solid voxel with a liquid
// face neighbour or a liquid voxel with a solid one — the only voxels the reaction changes.
// *list (cudaMalloc'ed, ascending group index) and *n; *tmp = n float4 of scratch
struct IfaceList {
    int* list = nullptr;
    long n = 0;
    float4* tmp = nullptr;
    int* nf_list = nullptr;  // groups holding any solid or near-liquid voxel (ascending)
    long n_nf = 0;
};
cudaError_t build_iface_list(const uint8_t* pp, const Geometry& g, IfaceList* out, cudaStream_t s);
cudaError_t launch_absorb_tail(float* cur, float* other, float* alpha, const uint8_t* pp, const Geometry& g,
                               const AbsorbArgs& ab, double* part, double* far_state, double v_far, int far,
                               double* rec, cudaStream_t s, float** result,
                               int* ctr = nullptr, const IfaceList* iface = nullptr);
struct StudyArgs {
    const float* cpad;
    float* out;           // padded layout
    const void* Wt;
    const float2* diag;
    int nx, ny, nzl, nxq, tile, tpp, nxp, nyp, R;
    const float* pbc;
    const double* far_state;
    const int* chunk_pos;  // N2 compaction: chunk → compact position or −1 (null: full layout)
};
cudaError_t launch_superpose_study(const StudyArgs& a, int mode, cudaStream_t s);

// ---- N2 far field (superpose.cu) ----------------------------------------------------
// per-tile Σ c over a dense slab field (far voxels skipped), same order as superpose's sums
cudaError_t launch_tile_mass_padded(const float* c_interior, const uint8_t* farmask, const Geometry& g,
                                    double* tile_sum, cudaStream_t s);
cudaError_t launch_tile_mass(const float* c, const uint8_t* farmask, const Geometry& g, double* tile_sum,
                             cudaStream_t s);
// padded field = 1 on in-domain non-far voxels of planes [z0−R, z1+R) (mask planes from mz0)
cudaError_t launch_ones(const uint8_t* mask, int mz0, const Geometry& g, float* cpad, cudaStream_t s);
// pbc[tile layout] = 1 − rowsum for real non-far targets, else 0
cudaError_t launch_pbc(const float* rowsum, const uint8_t* farmask, const Geometry& g, float* pbc, cudaStream_t s,
                       const int* list = nullptr, long n_list = 0, int n_list_tiles = 0, bool direct = false);
// FDIRW_F_PBC_RESERVOIR (world 1): n_fd whole-grid explicit FD substeps from 0 with the far field
// (mask 2) held at 1; faces as kgen's (harmonic λ, far cells fast); result → out (dense grid)
cudaError_t launch_reservoir_fd(const uint8_t* mask, const Geometry& g, float lff, float lfs, float lss, int n_fd,
                                float* out, float* tmp, cudaStream_t s);
// gathered = world blocks of (1 + stride−1) doubles: [count, tile sums...]; sum in global tile
// order (deterministic for any decomposition).  mode 0: c_far = (M0 − Σ)/v_far;
// mode 1 (init): M0 = Σ + c_far0·v_far, c_far = c_far0
cudaError_t launch_far_reduce(const double* gathered, int world, long stride, double* far_state, double v_far,
                              double c_far0, int mode, cudaStream_t s);

cudaError_t launch_pack(const float* c, float* cpad, const Geometry& g, cudaStream_t s,
                        const uint8_t* farmask = nullptr);
cudaError_t launch_unpack(const float* cpad, float* c, const Geometry& g, cudaStream_t s);
cudaError_t launch_mass(const float* c, size_t n, double* partial, int nblk, double* out, cudaStream_t s);
cudaError_t launch_export(const void* Wt, const float2* diag, const Geometry& g, int fmt, const int32_t* box,
                          double* out, cudaStream_t s, const int* chunk_pos = nullptr);

// ---- NCCL (comm.cpp): dlopen'ed, no link-time dependency ------------------------
struct Nccl;
Nccl* nccl_load(std::string* err);
int nccl_unique_id(Nccl*, void* out128, std::string* err);
void* nccl_comm_init(Nccl*, int world, int rank, const void* id128, std::string* err);
int nccl_halo(Nccl*, void* comm, float* cpad, const HaloPlan& h, cudaStream_t s, std::string* err);
int nccl_allreduce_sum_f64(Nccl*, void* comm, double* buf, cudaStream_t s, std::string* err);
int nccl_allgather_f64(Nccl*, void* comm, const double* send, long count, double* recv, cudaStream_t s,
                       std::string* err);
void nccl_comm_destroy(Nccl*, void* comm);

}  // namespace fdirw
