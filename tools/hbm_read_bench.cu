// hbm_read_bench.cu — practical HBM read ceiling on this B200 for a streaming kernel like
// superpose (128-bit loads, evict-first, many bytes in flight), vs the copy peak in
// MEASURED_PEAKS.json.  Design input, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_bin tools/hbm_read_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_stream(const uint4* p, unsigned long long pol)
{
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

template <int U>
__global__ void __launch_bounds__(256) rd(const uint4* __restrict__ a, size_t n16, unsigned* out)
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(a + i + u * stride, pol);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        uint4 v = ld_stream(a + i, pol);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) rd_last(const uint4* __restrict__ a, size_t n16, unsigned* out)
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(a + i + u * stride, pol);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        uint4 v = ld_stream(a + i, pol);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// chunked: each CTA streams one contiguous chunk (the superpose layout: one tile per CTA)
template <int U>
__global__ void __launch_bounds__(256) rd_chunk(const uint4* __restrict__ a, size_t chunk16, size_t nchunk, unsigned* out)
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    unsigned acc = 0;
    for (size_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const uint4* p = a + c * chunk16;
        for (size_t i = threadIdx.x; i < chunk16; i += U * blockDim.x) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = (i + u * blockDim.x < chunk16) ? ld_stream(p + i + u * blockDim.x, pol) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// superpose-like: one CTA per tile, per slot one 16-byte load per thread (4 KB per CTA);
// SLOTMAJOR = false: tile-major [tile][slot][4 KB] (the current gather layout);
// SLOTMAJOR = true: slot-major [slot][tile][4 KB] (concurrent tiles read neighbouring blocks)
template <bool SLOTMAJOR, int U>
__global__ void __launch_bounds__(256) rd_tiles(const uint4* __restrict__ a, int ntile, int nslot, unsigned* out)
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    unsigned acc = 0;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
        for (int s = 0; s < nslot; s += U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int ss = s + u < nslot ? s + u : nslot - 1;
                const size_t blk = SLOTMAJOR ? (size_t)ss * ntile + t : (size_t)t * nslot + ss;
                v[u] = ld_stream(a + blk * 256 + threadIdx.x, pol);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// TMA bulk reads (cp.async.bulk global → shared, the superposition's staged stream): one thread
// per CTA keeps S stages of B bytes in flight over its contiguous chunk; the bytes are not
// consumed (each stage is re-issued as soon as its copy completed)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32) rd_bulk(const unsigned char* __restrict__ a, size_t chunk, size_t nchunk,
                                             int S, unsigned B, unsigned* out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sm);
    unsigned char* st = sm + 128;
    if (threadIdx.x != 0) return;
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned ph[16] = {0};
    for (size_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const unsigned char* p = a + c * chunk;
        const size_t nb = chunk / B;
        for (size_t k = 0; k < nb; ++k) {
            const int s = (int)(k % S);
            if (k >= (size_t)S || c != blockIdx.x) {  // wait for the stage's previous copy
                asm volatile("{\n .reg .pred q;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}"
                             ::"r"(smem_u32(full + s)), "r"(ph[s]) : "memory");
                ph[s] ^= 1u;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(B) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                         ::"r"(smem_u32(st + (size_t)s * B)), "l"(p + k * B), "r"(B), "r"(smem_u32(full + s)), "l"(pol) : "memory");
        }
    }
    for (int s = 0; s < S; ++s)
        asm volatile("{\n .reg .pred q;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}"
                     ::"r"(smem_u32(full + s)), "r"(ph[s]) : "memory");
    if (ph[0] == 7u) out[0] = 1;
}

int main()
{
    const size_t bytes = 18905104640ull;  // cfg3's weight bytes
    uint4* a;
    unsigned* o;
    if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&o, 4);
    cudaMemset(a, 1, bytes);
    const size_t n16 = bytes / 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("%-40s %.3f ms  %.1f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
    };
    for (int bps : {4, 8, 16}) {
        const int g = 148 * bps;
        char nm[64];
        snprintf(nm, 64, "grid-stride U=4 blocks/SM=%d", bps);
        timeit(nm, [&] { rd<4><<<g, 256>>>(a, n16, o); });
        snprintf(nm, 64, "grid-stride U=8 blocks/SM=%d", bps);
        timeit(nm, [&] { rd<8><<<g, 256>>>(a, n16, o); });
    }
    // TMA bulk reads over 3456 contiguous tiles (S stages of B bytes in flight per CTA)
    {
        const size_t nchunk = 3456, chunk = (bytes / nchunk) / 65536 * 65536;
        const double gb = (double)chunk * nchunk / 1e9;
        for (int ctas : {1, 2, 3}) for (unsigned B : {16384u, 32768u, 45056u}) for (int S : {2, 3, 4}) {
            const size_t smem = 128 + (size_t)S * B;
            if (smem * ctas > 227 * 1024) continue;
            cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            const int g = 148 * ctas;
            rd_bulk<<<g, 32, smem>>>(reinterpret_cast<unsigned char*>(a), chunk, nchunk, S, B, o);
            cudaDeviceSynchronize();
            float best = 1e30f;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                rd_bulk<<<g, 32, smem>>>(reinterpret_cast<unsigned char*>(a), chunk, nchunk, S, B, o);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("TMA bulk CTAs/SM=%d B=%u S=%d  %.3f ms  %.1f GB/s\n", ctas, B, S, best, gb / (best * 1e-3));
        }
    }
    // superpose-like: 3456 tiles of 5.47 MB each, one CTA per tile
    const size_t nchunk = 3456, chunk16 = n16 / nchunk;
    timeit("chunked 3456 tiles U=4 (grid=3456)", [&] { rd_chunk<4><<<nchunk, 256>>>(a, chunk16, nchunk, o); });
    timeit("chunked 3456 tiles U=8 (grid=3456)", [&] { rd_chunk<8><<<nchunk, 256>>>(a, chunk16, nchunk, o); });
    timeit("chunked 3456 tiles U=8 (grid=592)", [&] { rd_chunk<8><<<592, 256>>>(a, chunk16, nchunk, o); });
    const int nslot = 1330;
    for (int ntile : {3456, 2960}) {
        const size_t need = (size_t)ntile * nslot * 4096;
        if (need > bytes) continue;
        const double gb = need / 1e9;
        auto t2 = [&](const char* name, auto launch) {
            launch();
            cudaDeviceSynchronize();
            float best = 1e30f;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                launch();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("%-44s tiles=%d %.3f ms  %.1f GB/s\n", name, ntile, best, gb / (best * 1e-3));
        };
        t2("tile-major  U=4 grid=ntile", [&] { rd_tiles<false, 4><<<ntile, 256>>>(a, ntile, nslot, o); });
        t2("tile-major  U=8 grid=ntile", [&] { rd_tiles<false, 8><<<ntile, 256>>>(a, ntile, nslot, o); });
        t2("slot-major  U=4 grid=ntile", [&] { rd_tiles<true, 4><<<ntile, 256>>>(a, ntile, nslot, o); });
        t2("slot-major  U=8 grid=ntile", [&] { rd_tiles<true, 8><<<ntile, 256>>>(a, ntile, nslot, o); });
        t2("tile-major  U=8 grid=592", [&] { rd_tiles<false, 8><<<592, 256>>>(a, ntile, nslot, o); });
        t2("slot-major  U=8 grid=592", [&] { rd_tiles<true, 8><<<592, 256>>>(a, ntile, nslot, o); });
    }
    // L2-resident re-read (the coarse GEMV's P̃ case): 64 MB read over and over, evict_last
    for (size_t mb : {32, 64, 96}) {
        const size_t b2 = mb << 20, n2 = b2 / 16;
        auto t3 = [&](const char* name, auto launch) {
            for (int w = 0; w < 3; ++w) launch();
            cudaDeviceSynchronize();
            float best = 1e30f;
            for (int r = 0; r < 20; ++r) {
                cudaEventRecord(e0);
                launch();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("%-40s %3zu MB %.4f ms  %.1f GB/s\n", name, mb, best, b2 / (best * 1e-3) / 1e9);
        };
        t3("L2 re-read U=8 blocks/SM=4", [&] { rd_last<8><<<148 * 4, 256>>>(a, n2, o); });
        t3("L2 re-read U=8 blocks/SM=8", [&] { rd_last<8><<<148 * 8, 256>>>(a, n2, o); });
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
