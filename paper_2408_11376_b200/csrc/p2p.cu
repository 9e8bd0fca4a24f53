// p2p.cu — a6 over NVLink peer memory: the halo "exchange" fused into the superposition.
//
// North_star (d) asks for a z-slab halo exchange of R planes per neighbour per step.  With
// FDIRW_TRANSPORT_P2P there is no separate exchange: the boundary-tile superposition CTAs
// that produce a rank's first / last R output planes also store them straight into the
// neighbours' padded state (their halo planes for the next step) through peer pointers
// (CUDA IPC, P2P stores over NVLink/NVSwitch), tile by tile as they are computed.  Ordering
// is a per-phase epoch handshake on 64-bit flags in each rank's own memory:
//   signal:  epoch ← epoch + 1;  st.release.sys  neighbour.flag[side] ← epoch
//   wait:    spin (ld.acquire.sys) until every neighbour's flag ≥ my epoch
// A step is  interior tiles → wait → boundary tiles (+ remote stores) → signal.  The wait
// guarantees (i) the neighbours' previous-step stores into my halo are complete and
// (ii) the neighbours finished reading the halo buffer I am about to overwrite (their
// previous step, two buffers ago in the ping-pong).  The wait kernel is bounded: after
// kP2PTimeoutNs it records an error flag and returns (no GPU hang); fdirw_p2p_check reads it.
#include "fdirw_internal.h"

namespace fdirw {

constexpr unsigned long long kP2PTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// flags: [0] epoch signalled by the lo neighbour, [1] by the hi neighbour, [2] own epoch,
// [3] sticky error (wait timed out)
__global__ void p2p_wait_kernel(unsigned long long* flags, int has_lo, int has_hi)
{
    const unsigned long long e = flags[2];
    const unsigned long long t0 = globaltimer();
    for (;;) {
        const bool ok = (!has_lo || ld_acquire_sys(flags + 0) >= e) && (!has_hi || ld_acquire_sys(flags + 1) >= e);
        if (ok) return;
        if (globaltimer() - t0 > kP2PTimeoutNs) {
            flags[3] = 1;
            return;
        }
        __nanosleep(200);
    }
}

__global__ void p2p_signal_kernel(unsigned long long* flags, unsigned long long* peer_lo_flag,
                                  unsigned long long* peer_hi_flag)
{
    const unsigned long long e = flags[2] + 1;
    flags[2] = e;
    __threadfence_system();  // the previous kernels' peer stores (each fenced by its thread) come first
    if (peer_lo_flag) st_release_sys(peer_lo_flag, e);
    if (peer_hi_flag) st_release_sys(peer_hi_flag, e);
}

// Run start: our first / last R padded slab planes → the neighbours' halo planes.
__global__ void p2p_push_planes_kernel(const float4* __restrict__ lo_src, float4* lo_dst,
                                       const float4* __restrict__ hi_src, float4* hi_dst, long n4)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        if (lo_dst) lo_dst[i] = lo_src[i];
        if (hi_dst) hi_dst[i] = hi_src[i];
    }
    __threadfence_system();
}

cudaError_t preload_step_kernels();

cudaError_t p2p_preload()
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, p2p_wait_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, p2p_signal_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, p2p_push_planes_kernel);
    if (e == cudaSuccess) e = preload_step_kernels();
    return e;
}

cudaError_t p2p_wait(unsigned long long* flags, bool has_lo, bool has_hi, cudaStream_t s)
{
    p2p_wait_kernel<<<1, 1, 0, s>>>(flags, has_lo ? 1 : 0, has_hi ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t p2p_signal(unsigned long long* flags, unsigned long long* peer_lo_flag, unsigned long long* peer_hi_flag,
                       cudaStream_t s)
{
    p2p_signal_kernel<<<1, 1, 0, s>>>(flags, peer_lo_flag, peer_hi_flag);
    return cudaGetLastError();
}

// cpad: our padded buffer; peer_lo / peer_hi: the neighbours' padded buffers of the same
// parity (or null); nzl_lo: the lo neighbour's slab thickness
cudaError_t p2p_push_planes(const Geometry& g, const float* cpad, float* peer_lo, int nzl_lo, float* peer_hi,
                            cudaStream_t s)
{
    if (!peer_lo && !peer_hi) return cudaSuccess;
    const long pe = (long)g.plane_elems, n = (long)g.R * pe;  // plane_elems is a multiple of 4
    const float* lo_src = cpad + (long)g.R * pe;              // our planes [0, R)
    float* lo_dst = peer_lo ? peer_lo + (long)(nzl_lo + g.R) * pe : nullptr;  // its halo hi
    const float* hi_src = cpad + (long)g.nzl * pe;            // our planes [nzl − R, nzl)
    float* hi_dst = peer_hi;                                  // its halo lo: padded planes [0, R)
    const long n4 = n / 4;
    long blocks = (n4 + 255) / 256;
    if (blocks > 148L * 8) blocks = 148L * 8;
    p2p_push_planes_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(
        reinterpret_cast<const float4*>(lo_src), reinterpret_cast<float4*>(lo_dst),
        reinterpret_cast<const float4*>(hi_src), reinterpret_cast<float4*>(hi_dst), n4);
    return cudaGetLastError();
}

}  // namespace fdirw
