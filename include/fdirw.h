/*
 * fdirw.h — C ABI of the B200-native FDiRW hot path (arXiv 2408.11376).
 *
 * FDiRW (Finite Difference informed Random Walker) advances a strongly
 * inhomogeneous diffusion field over a LARGE step Δt by superposition of
 * pre-computed transition kernels (§3.1 Eq.8):
 *
 *     C_new(x) = Σ_s W_s(x − s) · C_old(s)                                 (a5)
 *
 * where W_s, the mass fraction moving from source voxel s to x over Δt
 * ("p_ij is the mass proportion moving from node j to node i"), is
 * obtained by an explicit finite-difference run from a single point source
 * (P:109), here inside the source's own (2R+1)^3 window (a3).  The library
 * builds all W_s on the GPU (fdirw_build_kernels), stores them in fp32, fp16
 * or bf16 (§3.3 mixed precision; accumulation always fp32), and
 * applies the step (fdirw_step / fdirw_run).  With world > 1 every rank owns a
 * z-slab of targets and exchanges R-plane halos of C over NCCL each step.
 *
 * Conventions
 *   - Grid [nz][ny][nx], x fastest.  All concentration buffers passed to the
 *     library are DEVICE pointers to dense fp32 arrays of the caller's slab
 *     [z_end − z_begin][ny][nx] (the whole grid when world == 1).
 *   - phase_host is a HOST pointer to the WHOLE grid's uint8 mask
 *     (1 = fast phase / liquid, 0 = slow phase / solid), read only
 *     during fdirw_build_kernels and copied.
 *   - Diffusivities are EFFECTIVE ones, D·A/RT (Eqs.1-3).
 *   - Window: cube of Chebyshev radius R around each source, K = (2R+1)^3.
 *     Window edges and domain edges carry no flux (closed domain; DESIGN.md
 *     readings A1-A3, A21).  Face diffusivity across phases: harmonic mean (A4).
 *   - Streams: `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 *     Every call that takes a stream only ENQUEUES work on it and returns;
 *     errors of enqueued kernels surface at the next call or synchronisation.
 *   - Errors: every entry point returns an fdirw_status; the thread-local
 *     message of the last failure is fdirw_last_error().  No C++ exception
 *     crosses the ABI.  After FDIRW_E_CUDA / FDIRW_E_NCCL the context is
 *     unusable and must be destroyed.
 *   - Ownership: the caller owns phase_host and every concentration buffer;
 *     the context owns the weights, the diagonal, the padded ping-pong state,
 *     the halo buffers, the NCCL communicator and the CUDA graph, all freed by
 *     fdirw_destroy.
 */
#ifndef FDIRW_H
#define FDIRW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fdirw_ctx fdirw_ctx; /* opaque */

typedef enum {
    FDIRW_OK = 0,
    FDIRW_E_INVALID = 1,  /* bad argument: dims < 1, R < 1 or R > 8, D_fast <= 0, D_slow < 0, dt <= 0,
                             dh <= 0, NULL pointer, bad slab split, bad weight format           */
    FDIRW_E_UNSTABLE = 2, /* explicit FD unstable: λ_max = Δt_fd·D_max/Δh² > 1/6 (given n_fd)  */
    FDIRW_E_OOM = 3,      /* device allocation failed; message names the bytes required          */
    FDIRW_E_CUDA = 4,     /* CUDA runtime error (message has the CUDA error string)              */
    FDIRW_E_NCCL = 5,     /* NCCL error, or NCCL library not loadable when world > 1              */
    FDIRW_E_ALIAS = 6,    /* c_in == c_out in fdirw_step                                          */
    FDIRW_E_STATE = 7     /* call not valid in this context state (e.g. debug upload on world>1) */
} fdirw_status;

/* Weight storage formats.  FDIRW_W_MX8 (beyond the paper's §3.3 formats): each
 * gather block (the 8 weights of 8 consecutive targets for one window offset) is 8 unsigned
 * 8-bit mantissas m plus one power-of-two scale s (8-bit exponent): w = m·s, s the smallest
 * power of two with max(block)/s <= 255, m = RNE(w/s); 1.125 bytes per weight.  The fp32
 * diagonal fix-up restores each source's mass from the decoded weights.  Accuracy is within
 * north_star's reduced-precision bar (relL2 <= 5e-3).  Supported on any slab decomposition
 * (bitwise the one-rank result), closed or open (v_far > 0: the diagonal is then the open
 * window's own mass M minus its decoded weights), without FDIRW_F_NO_MASS_FIX / _NO_DEDUP /
 * _SYMMETRIC_RULE / _KGEN_FP64, and not with the N3 precision-study modes 1-3;
 * other combinations return FDIRW_E_INVALID.  With FDIRW_F_DEDUP_STORAGE the uniform chunks
 * use their class kernel quantised as blocks of 8 equal weights (exactly what the dense
 * layout would store there) and a per-target diagonal.                                       */
typedef enum { FDIRW_W_FP32 = 0, FDIRW_W_FP16 = 1, FDIRW_W_BF16 = 2, FDIRW_W_MX8 = 3 } fdirw_weight_t;

/* fdirw_params.flags */
#define FDIRW_F_NO_MASS_FIX 1u /* diagonal = RNE_fmt(W_s(0)) instead of the fp32 mass fix-up (A10) */
#define FDIRW_F_NO_DEDUP 2u    /* run kgen on every source window instead of once per distinct window
                                  (results are bitwise identical either way)          */
#define FDIRW_F_DEDUP_STORAGE 4u /* NEXT row N4: 8-target chunks whose every source shares one window
                                  class read that class's kernel from a small L2-resident table
                                  instead of streaming their gather weights (bitwise identical
                                  results; fewer HBM bytes)                        */
#define FDIRW_F_KGEN_FP64 8u   /* kgen substeps in fp64, in the oracle's operation order (no FMA), no
                                  renormalisation: the off-centre weights equal the oracle's O5
                                  weights bit for bit (reading A22; debugging — fp64 is slower)   */
#define FDIRW_F_SYMMETRIC_RULE 16u /* exact regime only (n_fd <= R, else FDIRW_E_INVALID): P = Pᵀ,
                                  so target x's gather weights are x's own kernel reflected,
                                  W_x(−o); each rank generates only its own slab's kernels (no
                                  halo sources).  Not combined with FDIRW_F_DEDUP_STORAGE
                                  (reading A24)                                                   */
#define FDIRW_F_KGEN_DIRECT 32u /* kgen runs the n_fd explicit substeps literally.  Default:
                                  when it saves work, the same A^{n_fd}·δ_s is evaluated by a
                                  Chebyshev recurrence of degree m ≈ 160 (at n_fd = 1000, λ = 0.1)
                                  over the same stencil, truncation ‖·‖₂ ≤ 1e-10 (reading A30;
                                  fdirw_info.kgen_steps reports which)                            */
#define FDIRW_F_NO_BULK_STREAM 64u /* superposition streams each tile's weights with per-thread 128-bit
                                  loads instead of TMA bulk copies into shared-memory stages (the
                                  default for launches of >= 2 CTAs per SM).  Identical results;
                                  for A/B measurement                              */
#define FDIRW_F_KGEN_COLUMNS 128u /* R = 5, 8: kgen with one window column per thread (the round-1
                                  kernel) instead of two columns per thread over balanced z
                                  segments (kgen_bal.cu).  The same substep arithmetic; the fp64
                                  epilogue sums group cells differently.  For A/B   */
#define FDIRW_F_PBC_RESERVOIR 256u /* N2, one GPU (world == 1, else FDIRW_E_INVALID): p_BC by the
                                  reservoir's own held-Dirichlet FD (n_fd whole-grid substeps from a
                                  zero field, far field held at 1; the fine analogue of the paper's
                                  P_BC column) instead of reading A26's 1 − row sum, which goes
                                  negative where truncated windows make a row sum exceed 1
                                  (A26).  Ignored without a far field              */

/* The paper's problem statement (Table 1) + north_star's window radius / precision. */
typedef struct {
    int32_t nx, ny, nz;     /* global grid, each >= 1                                          */
    double dh;              /* voxel edge Δh > 0                                               */
    double D_fast, D_slow;  /* effective diffusivities, D_fast > 0, D_slow >= 0 (0 = impermeable) */
    double dt;              /* macro step Δt > 0                                               */
    int32_t radius;         /* window half-width R, 1 <= R <= 8                                */
    int32_t n_fd;           /* FD substeps per Δt; 0 = derive n_fd = ceil(x(1−1e-9)),
                               x = D_max·Δt/(0.1·Δh²) (λ* = 0.1 from Table 1, reading A5)     */
    int32_t weights;        /* fdirw_weight_t: storage format of W (accumulation is fp32)     */
    uint32_t flags;         /* FDIRW_F_*                                                       */
    double v_far;           /* NEXT row N2: far-field reservoir volume in voxels (V_L^far/Δh³,
                               P:93 Table 1); 0 = closed domain.  With v_far > 0 the mask may
                               hold 2 = far-field liquid: those voxels are not sources/targets
                               (their concentration is the scalar c_far), window FD
                               holds them at 0 (absorbing), each target gets p_BC(x)·c_far
                               with p_BC(x) = 1 − Σ_s W̃_s(x−s) (reading A26), and every step
                               ends with Eq.7: c_far = (M0 − Σ c)/v_far (see fdirw_far_init). */
} fdirw_params;

/* Slab decomposition (world > 1): rank r owns target planes [z_begin, z_end).
 * Slabs must tile [0, nz) in rank order and be at least R planes thick.
 * transport FDIRW_TRANSPORT_NCCL: nccl_id = 128 bytes produced by fdirw_nccl_unique_id on
 *   rank 0 and broadcast by the caller (e.g. torch.distributed); NULL = virtual ranks in
 *   one process (fdirw_step_virtual).  world == 1 needs no id.
 * transport FDIRW_TRANSPORT_P2P: the halo planes travel as peer-memory stores fused into
 *   the superposition (csrc/p2p.cu), after fdirw_p2p_attach / fdirw_p2p_attach_local; no
 *   NCCL on the step path and nccl_id is ignored.  Closed domain only (v_far == 0).  The
 *   whole-grid Σ of fdirw_mass needs a communicator: fdirw_comm_init (collective), called
 *   once every rank's build succeeded.                                                 */
#define FDIRW_TRANSPORT_NCCL 0
#define FDIRW_TRANSPORT_P2P 1
typedef struct {
    int32_t rank, world;
    int32_t z_begin, z_end;
    int32_t device;         /* CUDA device ordinal the context lives on                      */
    const void* nccl_id;    /* NULL when world == 1 (ignored with P2P, see fdirw_comm_init)  */
    int32_t transport;      /* FDIRW_TRANSPORT_NCCL (0) or FDIRW_TRANSPORT_P2P (1)           */
} fdirw_dist;

typedef struct {
    int32_t n_fd;           /* FD substeps per macro step                                      */
    int32_t K;              /* (2R+1)^3                                                        */
    int32_t z_begin, z_end; /* this context's target slab                                      */
    double dt_fd;           /* Δt / n_fd                                                        */
    double lambda_fast, lambda_fs, lambda_slow; /* face numbers Δt_fd·D/Δh² (fast-fast, cross, slow-slow) */
    uint64_t weight_bytes;  /* device bytes of the stored weights incl. the fp32-pair diagonal + padding */
    uint64_t state_bytes;   /* device bytes of the padded ping-pong concentration state         */
    uint64_t bytes_per_voxel_update; /* algorithmic: (K−1)·b_w + 8 (diag pair) + 4 (C read) + 4 (C write) */
    uint64_t voxels;        /* targets in this slab: nx·ny·(z_end − z_begin)                   */
    int32_t tile_chunks;    /* 8-voxel x-chunks per superposition tile (CTA)                   */
    int32_t n_tiles;        /* tiles in this slab                                              */
    uint64_t kgen_sources;  /* sources whose kernels the slab needs (planes [z_begin−R, z_end+R))  */
    uint64_t kgen_windows;  /* windows actually run through the FD (distinct windows with dedup)   */
    uint64_t chunks;        /* 8-target x-chunks of the slab                                        */
    uint64_t uniform_chunks;/* N4: chunks whose weights come from a shared class kernel (else 0)   */
    int32_t uniform_classes;/* N4: distinct class kernels those chunks use                          */
    int32_t kgen_steps;     /* stencil passes per kgen window: n_fd (direct substeps, also with
                               FDIRW_F_KGEN_FP64) or the Chebyshev degree m (reading A30)          */
    double kgen_kernel_ms;  /* device time of the kgen launch in fdirw_build_kernels (CUDA events) */
} fdirw_info;

/* Host-only decomposition plan of one rank (no CUDA call; usable without a GPU).
 * Offsets index the padded fp32 state [padded_z][padded_y][padded_x] whose voxel
 * (x, y, z) sits at ((z − z_begin + R)·padded_y + (y + R))·padded_x + pad_x0 + x.
 * The halo exchange of a6 moves halo_elems contiguous elements per message:
 * [send_lo, +halo_elems) → peer_lo's [recv_hi, …), [send_hi, …) → peer_hi's [recv_lo, …). */
typedef struct {
    int32_t z_begin, z_end;             /* target slab                                          */
    int32_t src_z_begin, src_z_end;     /* source planes whose windows reach the slab (kgen)    */
    int32_t mask_z_begin, mask_z_end;   /* mask planes copied to the device                     */
    int32_t tile_chunks, tiles_per_plane, n_tiles;
    int32_t interior_tile_begin, interior_tile_end; /* tiles that read no halo plane            */
    int32_t peer_lo, peer_hi;           /* neighbour ranks, −1 if none                          */
    int32_t n_fd;
    int64_t padded_x, padded_y, padded_z, pad_x0;
    int64_t halo_elems;
    int64_t send_lo, recv_lo, send_hi, recv_hi; /* element offsets, −1 if no peer            */
    uint64_t weight_bytes, state_bytes; /* device bytes the context will allocate            */
    int32_t kgen_steps;                 /* stencil passes per kgen window (= fdirw_info.kgen_steps) */
} fdirw_plan;

/* Validates exactly like fdirw_build_kernels and fills *plan.  Host only. */
fdirw_status fdirw_make_plan(const fdirw_params* params, const fdirw_dist* dist, fdirw_plan* plan);

/* Writes a fresh 128-byte ncclUniqueId to out128 (host).  Call on rank 0 only.
 * FDIRW_E_NCCL if libnccl.so.2 cannot be loaded. */
fdirw_status fdirw_nccl_unique_id(void* out128);

/* a1-a4: validate params, derive n_fd and the face numbers (host, fp64), plan
 * device memory for the slab, copy the mask planes [z_begin−2R, z_end+2R)
 * to the device, and generate every kernel W_s whose window reaches the slab
 * (sources [z_begin−R, z_end+R) ∩ [0,nz)) with the batched-window FD kernel,
 * then renormalise (fp64), quantise (RNE), fix the diagonal (an fp32 pair, A10) and write the
 * gather layout.  Enqueued on cuda_stream; the call synchronises that stream
 * before returning so the context is ready.  dist == NULL means world = 1 on
 * the current device.  On success *out owns all device memory.  */
fdirw_status fdirw_build_kernels(const fdirw_params* params, const uint8_t* phase_host,
                                 const fdirw_dist* dist, void* cuda_stream, fdirw_ctx** out);

/* a5/a6: one FDiRW step C_out = W ⊛ C_in on this rank's slab (halo exchange with
 * the z-neighbours when world > 1; every rank must call it).  c_in and c_out are
 * device fp32 [z_end−z_begin][ny][nx]; c_in is not modified; c_in == c_out →
 * FDIRW_E_ALIAS.  Asynchronous on cuda_stream. */
fdirw_status fdirw_step(fdirw_ctx* ctx, const float* c_in_dev, float* c_out_dev, void* cuda_stream);

/* a5/a6 with HOST buffers (the end-to-end call): copies c_in_host (fp32 slab, host) to the
 * device, runs fdirw_step, copies the result to c_out_host.  Everything is enqueued on
 * cuda_stream and returns before it completes: c_out_host is valid after the stream is
 * synchronised.  Page-locked (pinned) host buffers make the copies asynchronous; pageable
 * ones work but the driver stages them.  The context keeps two device staging slabs,
 * allocated on the first call.  c_in_host == c_out_host → FDIRW_E_ALIAS.
 * On one GPU with the dense closed-domain path (no far field, no N4 storage, default
 * precision mode) the slab is pipelined in plane chunks (up to 16): each chunk is copied
 * straight into the padded state, its superposition starts once the planes it reads have
 * landed (alternating between cuda_stream and an internal stream), and its result is copied
 * back while later chunks compute; the result is bitwise fdirw_step's.  The internal streams
 * are joined to cuda_stream before the call returns, so stream semantics are unchanged. */
fdirw_status fdirw_step_host(fdirw_ctx* ctx, const float* c_in_host, float* c_out_host, void* cuda_stream);

/* a7: n_steps FDiRW steps in place on c_dev (device fp32 slab), ping-ponging
 * inside the context's padded state and replayed from a CUDA graph.  n_steps
 * >= 0.  Asynchronous on cuda_stream. */
fdirw_status fdirw_run(fdirw_ctx* ctx, float* c_dev, int32_t n_steps, void* cuda_stream);

/* a7 diagnostics: Σ c over the WHOLE grid in fp64 (each rank sums its slab on
 * the device; an NCCL all-reduce combines ranks — every rank must call it).
 * Synchronises cuda_stream and writes the result to *out_host.  A virtual rank
 * (fdirw_step_virtual) returns its slab's Σ.  Errors: E_INVALID (NULL), E_STATE (a P2P
 * context at world > 1 without fdirw_comm_init), E_NCCL, E_CUDA. */
fdirw_status fdirw_mass(fdirw_ctx* ctx, const float* c_dev, double* out_host, void* cuda_stream);
/* Tracing (the per-component breakdown of Fig.7): n_steps (1..256) steps
 * on c_dev in place, enqueued eagerly (no CUDA graph) with CUDA events between the phases of
 * every step; synchronises and writes the mean device milliseconds per step of
 *   ms_out[0] halo   P2P: the neighbour-wait kernel; NCCL: the exchange on the comm stream
 *   ms_out[1] interior superposition (P2P and world 1: the single launch over every tile,
 *             boundary bands first; NCCL: the tiles that read no halo plane, overlapping [0])
 *   ms_out[2] boundary superposition (NCCL: both bands after the exchange; else 0)
 *   ms_out[3] tail   P2P: the epoch signal kernel; N2: the Eq.7 reduction; else ~0
 *   ms_out[4] the whole step.
 * Every rank must call it with the same n_steps.  E_STATE on the N3 study modes and the
 * compacted / N4 storage paths (world 1), whose steps are several launches of other kinds. */
fdirw_status fdirw_profile_phases(fdirw_ctx* ctx, float* c_dev, int32_t n_steps, void* cuda_stream, double* ms_out);
/* P2P contexts (world > 1): open the NCCL communicator fdirw_mass uses for the whole-grid Σ.
 * nccl_id: 128 bytes from fdirw_nccl_unique_id on rank 0, broadcast by the caller, not used
 * for any other communicator.  Collective: every rank calls it (blocks until all have).
 * Errors: E_INVALID (NULL), E_STATE (not a P2P context with world > 1, or already has one),
 * E_NCCL. */
fdirw_status fdirw_comm_init(fdirw_ctx* ctx, const void* nccl_id);
/* The same Σ over this rank's slab only (no communication).  Synchronous. */
fdirw_status fdirw_mass_local(fdirw_ctx* ctx, const float* c_dev, double* out_host, void* cuda_stream);

/* Measurement aid (bench.py roofline.read_ceiling): streams the context's stored
 * weights `reps` times (after one warm-up pass) with the superposition's own load
 * (128-bit, L1 no-allocate, L2 evict-first) and nothing else, timed with CUDA events on
 * cuda_stream; *gbps_out = weight bytes / best pass time (GB/s, 1e9).  The practical HBM
 * ceiling of a read-only stream on this device.  Synchronous.  Errors: E_INVALID (NULL,
 * reps < 1), E_STATE (no weights), E_CUDA. */
fdirw_status fdirw_read_ceiling(const fdirw_ctx* ctx, int32_t reps, void* cuda_stream, double* gbps_out);

/* Fills *info (host).  Never fails on a valid ctx. */
fdirw_status fdirw_query(const fdirw_ctx* ctx, fdirw_info* info);

/* N2 (v_far > 0 only): set the reservoir c_far(t0) and the conserved total
 * M0 = Σ c_dev + c_far0·v_far (Σc_{S+L}(t0) of Eq.7, fp64; all ranks must call it;
 * far-field voxels of c_dev are ignored).  *M0_out (may be NULL) receives M0.
 * Synchronises cuda_stream.  FDIRW_E_STATE on a closed-domain context. */
fdirw_status fdirw_far_init(fdirw_ctx* ctx, const float* c_dev, double c_far0, double* M0_out, void* cuda_stream);
/* N2 on virtual ranks (see fdirw_step_virtual): the same initialisation for all n contexts. */
fdirw_status fdirw_far_init_virtual(fdirw_ctx* const* ctxs, int32_t n, const float* const* c_dev, double c_far0,
                                    double* M0_out, void* cuda_stream);
/* N2: current c_far (after the last enqueued step).  Synchronises cuda_stream. */
fdirw_status fdirw_far_get(fdirw_ctx* ctx, double* c_far_out, void* cuda_stream);

/* ---- NEXT row N3: integrated absorption loop (Eqs.1-7, Fig.4) -------------
 * Table 1 quantities for components (2)-(3) of P:42. */
typedef struct {
    double D_S;     /* effective solid diffusivity D_S·A_S/RT (slow FD, solid–solid faces)   */
    double k;       /* pseudo-second-order rate constant [1/s] (Eq.4)                       */
    double c_S_eq;  /* solid equilibrium concentration (Eq.6), > 0                          */
    double c_L_eq;  /* liquid equilibrium concentration (Eq.5), > 0                         */
} fdirw_absorb_params;

/* n_steps macro steps of the integrated loop on c_dev (world == 1; build the context with
 * D_slow = 0 so the liquid FDiRW treats the solid as impermeable):
 *   (1) FDiRW liquid step (+ p_BC·c_far, Eq.8, when v_far > 0)
 *   (2) solid FD, n_s = ceil(D_S·Δt/(0.1·Δh²)) substeps
 *   (3) PSO interface reaction per solid|liquid face (Eqs.4-6, Jacobi); a liquid voxel
 *       never gives more than c − c_L_eq (reading A29)
 *   (4) Eq.7 c_far update; (5) kinetics
 * kinetics_host (may be NULL): [n_steps][4] = {Q_S, Q_L, c_far, c̄_S = Q_S/(N_S·c_S_eq)}.
 * Synchronises cuda_stream. */
fdirw_status fdirw_absorb_run(fdirw_ctx* ctx, const fdirw_absorb_params* params, float* c_dev, int32_t n_steps,
                              double* kinetics_host, void* cuda_stream);

/* §3.3 precision modes of the superposition (Figs.8-10), world == 1, dense layout:
 *   0 default: stored weights, fp32 FMA products, compensated fp32 sum (the product path)
 *   1 "FP32":  FP32 weights, fp32 products, plain fp32 running sum
 *   2 "mixed": FP16 weights, C converted to fp16, fp16 products, fp32 sum
 *   3 "FP16":  as 2 with an fp16 running sum
 * Modes 1-3 are study kernels (one thread per target), used through fdirw_run /
 * fdirw_absorb_run.  FDIRW_E_STATE if the weight format does not match. */
fdirw_status fdirw_set_precision_mode(fdirw_ctx* ctx, int32_t mode);

/* Frees everything the context owns (synchronises its device first).  NULL is a no-op. */
void fdirw_destroy(fdirw_ctx* ctx);

/* Thread-local message of the last non-OK status on this thread ("" if none). */
const char* fdirw_last_error(void);

/* The sha256 of the sources, headers, build flags and nvcc version this library was compiled
 * from (paper_2408_11376_b200/build.py); static string, never NULL. */
const char* fdirw_build_id(void);

/* ---- test support ------------------------------------------------------------
 * Replace the weights of a world == 1 context by caller-supplied per-source
 * kernels (host fp64, [nz][ny][nx][K], slot o = ((oz+R)·L+(oy+R))·L+(ox+R),
 * centre slot = the diagonal, stored as the fp32 pair hi = RNE_fp32(v), lo = RNE_fp32(v − hi)).
 * Off-centre values are converted to the
 * context's storage format with RNE; out-of-domain slots are ignored.  Used
 * to test the superposition in isolation against oracle weights.
 * Synchronous.  FDIRW_E_STATE when world > 1. */
fdirw_status fdirw_debug_upload_weights(fdirw_ctx* ctx, const double* kernels_host);

/* Read back the stored kernels of the sources in the box [x0,x1)×[y0,y1)×[z0,z1)
 * (global coordinates; box = int32[6] = x0,x1,y0,y1,z0,z1) as host fp64
 * [bz][by][bx][K], decoded from the gather layout (centre slot = diagonal).
 * Slots whose target lies outside this context's slab or the domain read 0.
 * Synchronous. */
fdirw_status fdirw_export_kernels(const fdirw_ctx* ctx, const int32_t* box, double* kernels_host);

/* Test support for the TMA-staged weight stream (compute-sanitizer racecheck does not
 * model the mbarrier complete_tx ordering of cp.async.bulk): enable != 0 makes every later
 * superposition launch of ctx re-read each weight a compute thread takes from a shared-memory
 * stage twice — after the stage's full barrier and again just before its warp releases the
 * stage to the producer — and compare both with the global copy.  Returns the 16-byte words
 * checked and the mismatches so far (a late copy or a premature refill shows as mismatches).
 * Synchronous.  Slows the step; never enable it in production. */
fdirw_status fdirw_debug_stage_canary(fdirw_ctx* ctx, int32_t enable, uint64_t* checks, uint64_t* mismatches);

/* Single-process "virtual ranks": n contexts built on ONE device with
 * dist = {r, n, slab_r, device, NULL} and flag-free params, stepped together
 * with the halo planes moved by cudaMemcpyAsync instead of NCCL.  Exercises
 * the slab, halo and interior/boundary logic of the multi-GPU path on one GPU.
 * c_in[r], c_out[r] are the ranks' slab buffers. */
fdirw_status fdirw_step_virtual(fdirw_ctx* const* ctxs, int32_t n, const float* const* c_in,
                                float* const* c_out, void* cuda_stream);

/* ---- NEXT row N1: coarse-mesh FDiRW (§3.1, Eqs.10-15) ------------------
 * The paper's own step on a coarse mesh, for the fast phase only (§3 "FDiRW solver
 * for fast diffusion in near-field liquid"), with the far-field term of NEXT row N2
 * when params->v_far > 0 (Eq.10 P_BC, Eq.7):
 *   region   Ω_L = voxels with region_host[v] == 1 (e.g. near-field liquid);
 *            region_host[v] == 2 marks far-field reservoir voxels (needs v_far > 0);
 *            any other value is outside (no flux)
 *   groups   Ω_L ∩ b×b×b blocks anchored at the origin, empty blocks dropped,
 *            numbered in block order (N = N_L/125 ⇔ b = 5)
 *   P        dense N×N; column J = group means (Eq.13) of an explicit FD run over Ω_L
 *            (faces leaving Ω_L carry no flux, face number λ = Δt_fd·D_fast/Δh²) from
 *            the group-uniform source 1 on group J, n_fd substeps; stored in
 *            params->weights format, off-diagonal RNE, fp32 diagonal fixed so that
 *            Σ_I N_I P̃_IJ = M_J = Σ_I N_I P_IJ (fp64 column mass; = N_J in a closed
 *            domain; coarse analogue of reading A10).  Faces from Ω_L into far-field
 *            voxels are Dirichlet (value 0 for the P columns).
 *   P_BC     (v_far > 0) group means of the same FD from c = 0 with the far field held
 *            at 1 (Eq.10), fp32 [N]
 *   step     C_I = Σ_{i∈I} c_i / N_I in fp32 (Eq.13, "mapping ... in FP32");
 *            C'_I = Σ_J P̃_IJ C_J (+ P_BC_I·c_far), fp32 accumulation (Eq.14);
 *            c'_i = C'_I (Eq.15); voxels outside Ω_L are copied unchanged; then (v_far > 0)
 *            Eq.7 on the device: c_far = (K0 − Σ_I N_I C'_I)/v_far, fp64.
 * params: nx, ny, nz, dh, D_fast, dt, n_fd, weights as for the fine path (D_slow and
 * radius are ignored; of the flags only FDIRW_F_KGEN_DIRECT is read: P columns by the
 * literal n_fd substeps instead of the Chebyshev evaluation, reading A30).  Single GPU.
 * Buffers are device fp32 [nz][ny][nx].
 */
typedef struct fdirw_coarse fdirw_coarse; /* opaque */

typedef struct {
    int32_t n_fd;
    int32_t block;          /* b                                                       */
    int64_t n_groups;       /* N (coarse nodes)                                        */
    int64_t n_region;       /* N_L (fine voxels in Ω_L)                                */
    uint64_t p_bytes;       /* stored P incl. fp32 diagonal                           */
    uint64_t flops_per_step;/* the paper's model N(N+1) + 2·N_L                */
    int32_t fd_passes;      /* stencil passes per P column: n_fd (literal substeps) or 8 + the
                               Chebyshev degree (reading A30; FDIRW_F_KGEN_DIRECT forces literal) */
} fdirw_coarse_info;

/* Builds groups, P (batched whole-region FD on the GPU), quantises.  Synchronous. */
fdirw_status fdirw_coarse_build(const fdirw_params* params, const uint8_t* region_host, int32_t block,
                                void* cuda_stream, fdirw_coarse** out);
/* One coarse step c_out = remap(P̃ · map(c_in)) (c_in != c_out).  Asynchronous. */
fdirw_status fdirw_coarse_step(fdirw_coarse* ctx, const float* c_in_dev, float* c_out_dev, void* cuda_stream);
/* n_steps coarse steps in place on c_dev: one map of the Ω_L voxels, n steps on the group
 * values (GEMV, and Eq.7 after each with a far field; two steps per replayed CUDA graph), one
 * remap.  Between steps the remapped field is constant over each group, so this is the operator
 * sequence of n fdirw_coarse_step calls without their intermediate map/remap pairs; it differs
 * from them only by that re-averaging's fp32 rounding (relL2 ≤ 1e-6, tested).  With the
 * environment variable FDIRW_COARSE_PER_STEP_REMAP set, each step maps and remaps (bitwise n
 * fdirw_coarse_step calls).  Asynchronous. */
fdirw_status fdirw_coarse_run(fdirw_coarse* ctx, float* c_dev, int32_t n_steps, void* cuda_stream);
fdirw_status fdirw_coarse_query(const fdirw_coarse* ctx, fdirw_coarse_info* info);
/* Host copies: P_host [N][N] fp64 decoded (diagonal = fp32 fix-up) if non-NULL;
 * group_of_host [nz][ny][nx] int32 (−1 outside Ω_L) if non-NULL.  Synchronous. */
fdirw_status fdirw_coarse_export(const fdirw_coarse* ctx, double* P_host, int32_t* group_of_host);
/* N2: starts the far-field bookkeeping (Eq.7) from the field c_dev and c_far(t0) = c_far0:
 * K0 = Σ_I N_I C_I(t0) + c_far0·v_far (C = fp32 mapping of c_dev, summed in fp64) is
 * written to *M_out if non-NULL.  Must be called before the first step of a far-field
 * context (c_far is 0 otherwise).  FDIRW_E_STATE if v_far == 0.  Synchronous. */
fdirw_status fdirw_coarse_far_init(fdirw_coarse* ctx, const float* c_dev, double c_far0, double* M_out,
                                   void* cuda_stream);
/* Current c_far (after the last enqueued step).  Synchronous on cuda_stream. */
fdirw_status fdirw_coarse_far_get(fdirw_coarse* ctx, double* c_far_out, void* cuda_stream);
/* P_BC as stored (fp32 decoded to fp64) into pbc_host [N].  FDIRW_E_STATE if v_far == 0. */
fdirw_status fdirw_coarse_export_pbc(const fdirw_coarse* ctx, double* pbc_host);
void fdirw_coarse_destroy(fdirw_coarse* ctx);

/* ---- a6 over NVLink peer memory (FDIRW_TRANSPORT_P2P) -----------------------------------
 * north_star (d)'s halo exchange without a separate collective: the CTAs computing a
 * rank's first / last R output planes store them straight into the neighbours' halo
 * planes through peer pointers; a 64-bit epoch flag per side orders the steps.
 * Bitwise equal to world == 1 for any slab decomposition (tested).
 *
 * fdirw_p2p_export: FDIRW_P2P_BLOB_BYTES bytes describing this context (geometry + CUDA IPC
 *   handles of its two state buffers and its flags); the caller all-gathers the blobs.
 * fdirw_p2p_attach: opens the neighbours' blobs (lo_blob of rank−1 or NULL on rank 0,
 *   hi_blob of rank+1 or NULL on the last rank); peer access is enabled lazily.
 *   FDIRW_E_INVALID if a blob's geometry or rank does not fit.  Synchronous.
 * fdirw_p2p_attach_local: the same for n contexts of ONE process (rank order), e.g. on
 *   one GPU for testing; each context then runs on its own stream, concurrently.
 * fdirw_p2p_check: *timed_out = 1 if a wait for a neighbour exceeded 20 s (the wait
 *   kernel then gives up instead of hanging the GPU; results are invalid).  Synchronous.
 * With P2P, fdirw_mass returns this slab's sum only (the caller reduces).             */
#define FDIRW_P2P_BLOB_BYTES 256
fdirw_status fdirw_p2p_export(fdirw_ctx* ctx, void* blob_out);
fdirw_status fdirw_p2p_attach(fdirw_ctx* ctx, const void* lo_blob, const void* hi_blob);
fdirw_status fdirw_p2p_attach_local(fdirw_ctx* const* ctxs, int32_t n);
fdirw_status fdirw_p2p_check(fdirw_ctx* ctx, int32_t* timed_out, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* FDIRW_H */
