// mio_microbench.cu — per-SM throughput of the instruction mixes kgen can be built from:
// LDS.128, SHFL, LDS.128 + SHFL together, FFMA, FFMA2 (fma.rn.f32x2), FFMA + LDS.
// One CTA of NT threads per resident slot; rates in (warp-)instructions per SM clock,
// measured with clock64 inside the kernel.  Design input for kgen, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mio tools/mio_microbench.cu && /tmp/mio
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 256;
constexpr int ITERS = 4096;

__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c)
{
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(NT) bench(float* out, long long* cyc, float s)
{
    __shared__ __align__(16) float sm[NT * 8 + 64];
    const int t = threadIdx.x;
    for (int i = t; i < NT * 8 + 64; i += NT) sm[i] = (float)i * 1e-3f;
    __syncthreads();
    float4 a0 = make_float4(0, 0, 0, 0), a1 = a0;
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = s * (t + i);
    unsigned long long p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = __double_as_longlong((double)(t + i));
    int off = (t * 4) & (NT * 8 - 1);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (MODE == 0 || MODE == 2 || MODE == 5) {  // 2 LDS.128 per iteration
            const float4 x = *reinterpret_cast<const float4*>(sm + off);
            const float4 y = *reinterpret_cast<const float4*>(sm + ((off + 128) & (NT * 8 - 1)));
            a0.x += x.x; a0.y += x.y; a0.z += x.z; a0.w += x.w;
            a1.x += y.x; a1.y += y.y; a1.z += y.z; a1.w += y.w;
            off = (off + 4 * (int)(a0.x == 12345.f)) & (NT * 8 - 1);
        }
        if (MODE == 1 || MODE == 2) {  // 8 SHFL per iteration (= 2 LDS.128 of data)
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] += __shfl_xor_sync(0xffffffffu, f[i], 1 + (i & 3));
        }
        if (MODE == 3 || MODE == 5) {  // 8 independent FFMA chains x 4
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], s, 0.5f);
        }
        if (MODE == 4) {  // 8 independent FFMA2 chains x 4 (64 lane-FMAs)
            const unsigned long long ss = __double_as_longlong(0.0);
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) p[i] = fma2(p[i], ss, p[i]);
        }
    }
    long long t1 = clock64();
    float acc = a0.x + a0.y + a0.z + a0.w + a1.x + a1.y + a1.z + a1.w;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += f[i] + (float)__longlong_as_double(p[i]);
    out[blockIdx.x * NT + t] = acc;
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
static void run(const char* name, double warp_ops_per_iter_per_warp)
{
    int dev = 0, sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bench<MODE>, NT, 0);
    for (int bps : {1, 2, per}) {
        const int grid = sms * bps;
        float* out;
        long long* cyc;
        cudaMalloc(&out, (size_t)grid * NT * 4);
        cudaMalloc(&cyc, grid * 8);
        bench<MODE><<<grid, NT>>>(out, cyc, 0.999f);
        bench<MODE><<<grid, NT>>>(out, cyc, 0.999f);
        cudaDeviceSynchronize();
        long long* h = new long long[grid];
        cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double warps_per_sm = (double)bps * NT / 32;
        const double rate = warps_per_sm * ITERS * warp_ops_per_iter_per_warp / (double)mx;
        printf("%-22s blocks/SM=%2d warps/SM=%3.0f  %.3f warp-instr/clk/SM  (max cyc %lld)\n", name, bps,
               warps_per_sm, rate, mx);
        delete[] h;
        cudaFree(out);
        cudaFree(cyc);
    }
}

int main()
{
    run<0>("LDS.128 (x2)", 2);
    run<1>("SHFL (x8)", 8);
    run<2>("LDS.128x2 + SHFLx8", 10);
    run<3>("FFMA (x32)", 32);
    run<4>("FFMA2 (x32)", 32);
    run<5>("LDS.128x2 + FFMAx32", 34);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
