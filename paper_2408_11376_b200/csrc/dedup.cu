// dedup.cu — kgen work reduction by window de-duplication (a3), bit-exact.
//
// A source's kernel W_s depends only on its window: the phases of the (2R+1)³ cells
// around s and which of them lie outside the domain (the column is the FD
// solution from a point source in that local geometry).  Two sources with identical
// windows therefore have bitwise identical kernels from the same FD code.  In the
// paper's geometries most windows are homogeneous liquid (or liquid clipped by the
// same domain face), e.g. 7.08 M sources but 0.75 M distinct windows at 192³ R5.
//
//   1. rowword_kernel   2-bit codes of every window row packed in one 64-bit word (L ≤ 17);
//      hash_kernel      two 64-bit hashes of every source window's L² row words
//   2. cub radix sort   (h1, source) pairs; stable, so a class's representative is
//                       its smallest source index (deterministic)
//   3. classify         run heads → class ids (inclusive scan − 1); class map in the padded layout
//                       of the state (−1 outside the domain); every non-head member is
//                       VERIFIED byte-for-byte against its representative's window —
//                       any mismatch (a hash collision) makes the caller fall back to
//                       the direct path, so results never depend on the hash
//   4. kgen_kernel      on the representatives only, class-major output
//   5. expand_kernel    writes the gather layout Wt / diag from the class kernels,
//                       coalesced 16/32-byte stores (replaces the memset + scatter)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <vector>

#include "fdirw_internal.h"
#include "layout.cuh"
#include "mx8.cuh"

namespace fdirw {

__device__ __forceinline__ float dec_w(float v) { return v; }
__device__ __forceinline__ float dec_w(__half v) { return __half2float(v); }
__device__ __forceinline__ float dec_w(__nv_bfloat16 v) { return __bfloat162float(v); }

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ unsigned window_code(const DedupArgs& a, int gx, int gy, int gz)
{
    if (gx < 0 || gx >= a.nx || gy < 0 || gy >= a.ny || gz < 0 || gz >= a.nz) return 2u;
    const unsigned v = a.mask[((size_t)(gz - a.mz0) * a.ny + gy) * a.nx + gx];
    return v == 2u ? 3u : v;  // kgen's codes: 0 slow, 1 fast, 2 outside, 3 far field (N2)
}

// Row words: rw(x, y, z) packs the L codes of (x−R … x+R, y, z), 2 bits each (L ≤ 17),
// for y ∈ [−R, ny+R), z ∈ [sz0−R, sz1+R).  A window is then its L² row words.
struct RowWords {
    const uint64_t* w;
    int nx, nyr, R, zr0;  // nyr = ny + 2R; plane zr0 = sz0 − R
    __device__ __forceinline__ uint64_t at(int x, int y, int z) const
    {
        return w[((long)(z - zr0) * nyr + (y + R)) * nx + x];
    }
};

__global__ void rowword_kernel(const DedupArgs a, uint64_t* __restrict__ rw, int nzr)
{
    const int nyr = a.ny + 2 * a.R;
    const long n = (long)a.nx * nyr * nzr;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int x = (int)(i % a.nx), y = (int)((i / a.nx) % nyr) - a.R, z = (int)(i / ((long)a.nx * nyr)) + a.sz0 - a.R;
        uint64_t v = 0;
        for (int k = 0; k <= 2 * a.R; ++k) v |= (uint64_t)window_code(a, x - a.R + k, y, z) << (2 * k);
        rw[i] = v;
    }
}

__global__ void hash_kernel(const DedupArgs a, RowWords rw, uint64_t* __restrict__ keys, int* __restrict__ vals,
                            uint64_t* __restrict__ h2out)
{
    const long n = (long)a.nx * a.ny * (a.sz1 - a.sz0);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int sx = (int)(i % a.nx), sy = (int)((i / a.nx) % a.ny), sz = a.sz0 + (int)(i / ((long)a.nx * a.ny));
        uint64_t h1 = 0x243F6A8885A308D3ull, h2 = 0x13198A2E03707344ull;
        int k = 0;
        for (int oz = -a.R; oz <= a.R; ++oz)
            for (int oy = -a.R; oy <= a.R; ++oy, ++k) {
                const uint64_t c = rw.at(sx, sy + oy, sz + oz) + 1u;
                h1 += c * (splitmix64(2 * k) | 1ull);
                h2 += splitmix64(c ^ splitmix64(2 * k + 1));
            }
        keys[i] = h1;
        vals[i] = (int)i;
        h2out[i] = h2;
    }
}

__global__ void heads_kernel(const uint64_t* __restrict__ k, long n, int* __restrict__ head)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// class ids, representatives, class map (padded layout), and exact verification
__global__ void classify_kernel(const DedupArgs a, const uint64_t* __restrict__ h2, const int* __restrict__ vals,
                                const int* __restrict__ head, const int* __restrict__ cid, long n,
                                int* __restrict__ rep, int* __restrict__ class_pad, int* __restrict__ mismatch)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int s = vals[i];
        const int c = cid[i] - 1;  // inclusive scan of the run heads
        if (head[i]) rep[c] = s;
        const int sx = s % a.nx, sy = (s / a.nx) % a.ny, sz = a.sz0 + s / (a.nx * a.ny);
        // padded state layout covers planes [z0 − R, z1 + R) — exactly the source planes;
        // far-field voxels (N2) are not sources: class −1 → zero weights and diagonal
        class_pad[((long)(sz - a.z0 + a.R) * a.nyp + (sy + a.R)) * a.nxp + kPadX + sx] =
            window_code(a, sx, sy, sz) == 3u ? -1 : c;
    }
}

__global__ void verify_kernel(const DedupArgs a, RowWords rw, const uint64_t* __restrict__ h2,
                              const int* __restrict__ vals, const int* __restrict__ head, const int* __restrict__ cid,
                              const int* __restrict__ rep, long n, int* __restrict__ mismatch)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        if (head[i]) continue;
        const int s = vals[i], r = rep[cid[i] - 1];
        if (h2[s] != h2[r]) { atomicOr(mismatch, 1); continue; }
        const int sx = s % a.nx, sy = (s / a.nx) % a.ny, sz = a.sz0 + s / (a.nx * a.ny);
        const int rx = r % a.nx, ry = (r / a.nx) % a.ny, rz = a.sz0 + r / (a.nx * a.ny);
        bool same = true;
        for (int oz = -a.R; oz <= a.R && same; ++oz)
            for (int oy = -a.R; oy <= a.R; ++oy)
                if (rw.at(sx, sy + oy, sz + oz) != rw.at(rx, ry + oy, rz + oz)) {  // exact: all L codes of the row
                    same = false;
                    break;
                }
        if (!same) atomicOr(mismatch, 1);
    }
}

// Gather layout from class kernels: thread = 8-target chunk, loop over slots in the
// superposition's order; per (oz, oy) row the 24 class ids of source row
// (z − oz, y − oy, x−8 … x+15) are loaded once from the padded class map.
template <int R, typename WT>
__global__ void __launch_bounds__(256) expand_kernel(const ExpandArgs a)
{
    constexpr int L = 2 * R + 1, LL = L * L, K = L * L * L;
    const int tile = blockIdx.x;
    const int e = threadIdx.x;
    int zl, q;
    bool real;
    if (a.list) {  // N4: compacted non-uniform chunks
        const long idx = (long)tile * a.tile + e;
        real = idx < a.n_list;
        const int chunk = real ? a.list[idx] : 0;
        const int ot = chunk / a.tile;
        zl = ot / a.tpp;
        q = (ot % a.tpp) * a.tile + chunk % a.tile;
    } else {
        zl = tile / a.tpp;
        q = (tile % a.tpp) * a.tile + e;
        real = q < a.ny * a.nxq;
    }
    const size_t wstride = (size_t)a.tile * 8;
    WT* wt = reinterpret_cast<WT*>(a.Wt) + ((size_t)tile * (K - 1) * a.tile + e) * 8;
    const WT* cw = reinterpret_cast<const WT*>(a.class_w);
    const int y = real ? q / a.nxq : 0, x = real ? (q % a.nxq) * 8 : 0;
    const long nxp = a.nxp, plane = (long)a.nyp * nxp;
    const int* c0 = a.class_pad + (zl + R) * plane + (long)(y + R) * nxp + kPadX + x;
    {
        float2 d[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = (real && x + j < a.nx) ? c0[j] : -1;
            d[j] = c >= 0 ? a.class_diag[c] : make_float2(0.f, 0.f);
        }
        float4* dp = reinterpret_cast<float4*>(a.diag + ((size_t)tile * a.tile + e) * 8);
#pragma unroll
        for (int j = 0; j < 4; ++j) dp[j] = make_float4(d[2 * j].x, d[2 * j].y, d[2 * j + 1].x, d[2 * j + 1].y);
    }
    for (int r = -1; r < LL; ++r) {  // r = −1: the centre row first (slot order of layout.cuh)
        if (r == R * L + R) continue;
        const int oz = r < 0 ? 0 : r / L - R, oy = r < 0 ? 0 : r % L - R;
        int seg[24];
        const int* srow = c0 - (long)oz * plane - (long)oy * nxp - 8;
#pragma unroll
        for (int i = 0; i < 24; ++i) seg[i] = real ? srow[i] : -1;
#pragma unroll
        for (int ox = -R; ox <= R; ++ox) {
            if (r < 0 && ox == 0) continue;
            const int o = (oz + R) * LL + (oy + R) * L + (ox + R);
            WT v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = seg[j - ox + 8];
                v[j] = c >= 0 ? cw[(size_t)c * K + o] : WT(0.f);
            }
            WT* dst = wt + (size_t)slot_of(ox, oy, oz, R) * wstride;
            if (sizeof(WT) == 2) {
                *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
            } else {
                reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<const uint4*>(v)[0];
                reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<const uint4*>(v)[1];
            }
        }
    }
}

// N4: a chunk (8 consecutive targets of a row) is uniform when every source that reaches it
// ((x0−R … x0+7+R) × (y±R) × (z±R)) has the same window class — then all its gather weights
// are that class's kernel.  cls_out[tile·tile_sz + e] = class, or −1.
__global__ void chunk_class_kernel(const int* __restrict__ class_pad, int nx, int ny, int nxq, int tile_sz, int tpp,
                                   int n_tiles, int nxp, int nyp, int R, int* __restrict__ cls_out,
                                   int* __restrict__ used)
{
    const long n = (long)n_tiles * tile_sz;
    const long plane = (long)nyp * nxp;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int e = (int)(i % tile_sz);
        const long t = i / tile_sz;
        const int zl = (int)(t / tpp), tp = (int)(t % tpp);
        const int q = tp * tile_sz + e;
        int k = -1;
        if (q < ny * nxq) {
            const int y = q / nxq, x = (q % nxq) * 8;
            if (x + 8 <= nx) {
                const int* c0 = class_pad + (zl + R) * plane + (long)(y + R) * nxp + kPadX + x;
                k = c0[0];
                for (int oz = -R; oz <= R && k >= 0; ++oz)
                    for (int oy = -R; oy <= R && k >= 0; ++oy) {
                        const int* row = c0 + (long)oz * plane + (long)oy * nxp;
                        for (int j = -R; j < 8 + R; ++j)
                            if (row[j] != k) { k = -1; break; }
                    }
            }
        }
        cls_out[i] = k;
        if (k >= 0) used[k] = 1;
    }
}

// ukf[u][slot] = class_w[k(u)][o(slot)] decoded to fp32; udiag[u] = class_diag[k(u)]
template <typename WT>
__global__ void ukf_kernel(const WT* __restrict__ class_w, const float2* __restrict__ class_diag,
                           const int* __restrict__ used, const int* __restrict__ uid, long n_class, int R,
                           float* __restrict__ ukf, float2* __restrict__ udiag)
{
    const int L = 2 * R + 1, K = L * L * L;
    const long n = n_class * (long)(K - 1);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const long k = i / (K - 1);
        if (!used[k]) continue;
        const int s = (int)(i % (K - 1));
        // slot → offset (inverse of slot_of): centre row first, then rows ascending
        int ox, oy, oz;
        if (s < L - 1) {
            oz = 0; oy = 0; ox = s < R ? s - R : s - R + 1;
        } else {
            const int r0 = (s - (L - 1)) / L;
            const int r = r0 >= R * L + R ? r0 + 1 : r0;
            oz = r / L - R; oy = r % L - R; ox = (s - (L - 1)) % L - R;
        }
        ukf[(long)uid[k] * (K - 1) + s] = dec_w(class_w[k * K + (oz + R) * L * L + (oy + R) * L + (ox + R)]);
        if (s == 0) udiag[uid[k]] = class_diag[k];
    }
}

__global__ void chunk_uid_kernel(int* __restrict__ cls, long n, const int* __restrict__ uid)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        if (cls[i] >= 0) cls[i] = uid[cls[i]];
}

static unsigned grid_n(long n);

cudaError_t build_uniform(const ExpandArgs& a, int R, int fmt, long n_class, UniformTables* t, cudaStream_t s)
{
    const long nch = (long)a.n_tiles * a.tile;
    int *used = nullptr, *uid = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    cudaError_t e = cudaMalloc(&t->chunk_u, nch * 4);
    if (e == cudaSuccess) e = cudaMalloc(&used, (n_class + 1) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&uid, (n_class + 1) * 4);
    if (e == cudaSuccess) e = cudaMemsetAsync(used, 0, (n_class + 1) * 4, s);
    if (e == cudaSuccess) {
        chunk_class_kernel<<<grid_n(nch), 256, 0, s>>>(a.class_pad, a.nx, a.ny, a.nxq, a.tile, a.tpp, a.n_tiles,
                                                       a.nxp, a.nyp, R, t->chunk_u, used);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tb, used, uid, (int)(n_class + 1), s);
    if (e == cudaSuccess) e = cudaMalloc(&tmp, tb);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tb, used, uid, (int)(n_class + 1), s);
    int nu = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nu, uid + n_class, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    const int K = (2 * R + 1) * (2 * R + 1) * (2 * R + 1);
    const long nu1 = nu > 0 ? nu : 1;
    if (e == cudaSuccess) e = cudaMalloc(&t->ukf, nu1 * (K - 1) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&t->udiag, nu1 * 8);
    if (e == cudaSuccess && nu > 0) {
        const long n = n_class * (long)(K - 1);
        if (fmt == 0)
            ukf_kernel<float><<<grid_n(n), 256, 0, s>>>((const float*)a.class_w, a.class_diag, used, uid, n_class, R,
                                                        t->ukf, t->udiag);
        else if (fmt == 1)
            ukf_kernel<__half><<<grid_n(n), 256, 0, s>>>((const __half*)a.class_w, a.class_diag, used, uid, n_class,
                                                         R, t->ukf, t->udiag);
        else
            ukf_kernel<__nv_bfloat16><<<grid_n(n), 256, 0, s>>>((const __nv_bfloat16*)a.class_w, a.class_diag, used,
                                                                uid, n_class, R, t->ukf, t->udiag);
        e = cudaGetLastError();
        if (e == cudaSuccess) {
            chunk_uid_kernel<<<grid_n(nch), 256, 0, s>>>(t->chunk_u, nch, uid);
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) {
        // chunk lists per class and CTA blocks of ≤ 256 chunks of one class (host side: nu is small)
        std::vector<int> h(nch);
        e = cudaMemcpyAsync(h.data(), t->chunk_u, nch * 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        std::vector<std::vector<int>> per(nu > 0 ? nu : 0);
        long cnt = 0;
        for (long i = 0; i < nch; ++i)
            if (h[i] >= 0) { per[h[i]].push_back((int)i); ++cnt; }
        std::vector<int> list;
        std::vector<int4> blocks;
        list.reserve(cnt);
        for (int u = 0; u < nu; ++u) {
            for (size_t b0 = 0; b0 < per[u].size(); b0 += 256) {
                const int c = (int)std::min<size_t>(256, per[u].size() - b0);
                blocks.push_back(make_int4((int)list.size(), c, u, 0));
                list.insert(list.end(), per[u].begin() + b0, per[u].begin() + b0 + c);
            }
        }
        t->n_uniform = cnt;
        t->n_u = nu;
        t->n_blocks = (int)blocks.size();
        // the real non-uniform chunks, in chunk order, compacted into tiles of a.tile
        std::vector<int> dense;
        dense.reserve(nch - cnt);
        for (long i = 0; i < nch; ++i) {
            const long tt = i / a.tile;
            const int q = (int)(tt % a.tpp) * a.tile + (int)(i % a.tile);
            if (h[i] < 0 && q < a.ny * a.nxq) dense.push_back((int)i);
        }
        t->n_dense = (long)dense.size();
        t->nd_tiles = (int)((t->n_dense + a.tile - 1) / a.tile);
        if (e == cudaSuccess) e = cudaMalloc(&t->dense_list, std::max<size_t>(dense.size(), 1) * 4);
        if (e == cudaSuccess && !dense.empty())
            e = cudaMemcpy(t->dense_list, dense.data(), dense.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMalloc(&t->list, std::max<size_t>(list.size(), 1) * 4);
        if (e == cudaSuccess) e = cudaMalloc(&t->blocks, std::max<size_t>(blocks.size(), 1) * sizeof(int4));
        if (e == cudaSuccess && !list.empty())
            e = cudaMemcpy(t->list, list.data(), list.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess && !blocks.empty())
            e = cudaMemcpy(t->blocks, blocks.data(), blocks.size() * sizeof(int4), cudaMemcpyHostToDevice);
    }
    cudaFree(used);
    cudaFree(uid);
    cudaFree(tmp);
    return e;
}

static unsigned grid_n(long n)
{
    long b = (n + 255) / 256;
    if (b > 148L * 32) b = 148L * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

#define DCK(call)                              \
    do {                                       \
        cudaError_t e_ = (call);               \
        if (e_ != cudaSuccess) return e_;      \
    } while (0)

cudaError_t dedup_classify(const DedupArgs& a, DedupResult* res, cudaStream_t s)
{
    const long n = (long)a.nx * a.ny * (a.sz1 - a.sz0);
    res->n_src = n;
    uint64_t *keys = nullptr, *keys2 = nullptr, *h2 = nullptr, *rwb = nullptr;
    int *vals = nullptr, *vals2 = nullptr, *head = nullptr, *cid = nullptr, *mism = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0, scan_bytes = 0;
    cudaError_t e = cudaSuccess;
    auto cleanup = [&]() {
        cudaFree(keys); cudaFree(keys2); cudaFree(h2); cudaFree(vals); cudaFree(vals2);
        cudaFree(head); cudaFree(cid); cudaFree(mism); cudaFree(tmp); cudaFree(rwb);
    };
#define TRY(call)                       \
    do {                                \
        e = (call);                     \
        if (e != cudaSuccess) {         \
            cleanup();                  \
            return e;                   \
        }                               \
    } while (0)
    TRY(cudaMalloc(&keys, n * 8));
    TRY(cudaMalloc(&keys2, n * 8));
    TRY(cudaMalloc(&h2, n * 8));
    TRY(cudaMalloc(&vals, n * 4));
    TRY(cudaMalloc(&vals2, n * 4));
    TRY(cudaMalloc(&head, n * 4));
    TRY(cudaMalloc(&cid, n * 4));
    TRY(cudaMalloc(&mism, 4));
    TRY(cudaMemsetAsync(mism, 0, 4, s));
    const int nzr = a.sz1 - a.sz0 + 2 * a.R;
    const long nrw = (long)a.nx * (a.ny + 2 * a.R) * nzr;
    TRY(cudaMalloc(&rwb, nrw * 8));
    rowword_kernel<<<grid_n(nrw), 256, 0, s>>>(a, rwb, nzr);
    TRY(cudaGetLastError());
    const RowWords rw{rwb, a.nx, a.ny + 2 * a.R, a.R, a.sz0 - a.R};
    hash_kernel<<<grid_n(n), 256, 0, s>>>(a, rw, keys, vals, h2);
    TRY(cudaGetLastError());
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, 64, s));
    TRY(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, head, cid, (int)n, s));
    if (scan_bytes > tmp_bytes) tmp_bytes = scan_bytes;
    TRY(cudaMalloc(&tmp, tmp_bytes));
    TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, 64, s));
    heads_kernel<<<grid_n(n), 256, 0, s>>>(keys2, n, head);
    TRY(cudaGetLastError());
    TRY(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, head, cid, (int)n, s));  // class id + 1
    int last = 0;
    TRY(cudaMemcpyAsync(&last, cid + n - 1, 4, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    const long n_class = last;
    res->n_class = n_class;
    TRY(cudaMalloc(&res->rep, n_class * 4));
    classify_kernel<<<grid_n(n), 256, 0, s>>>(a, h2, vals2, head, cid, n, res->rep, a.class_pad, mism);
    TRY(cudaGetLastError());
    verify_kernel<<<grid_n(n), 256, 0, s>>>(a, rw, h2, vals2, head, cid, res->rep, n, mism);
    TRY(cudaGetLastError());
    int mm = 0;
    TRY(cudaMemcpyAsync(&mm, mism, 4, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    res->collision = mm != 0;
    cleanup();
    return cudaSuccess;
#undef TRY
}

// FDIRW_W_MX8 (mx8.cuh): expand_kernel's gather walk over fp32 class kernels, each
// block of 8 targets × 1 slot quantised to 8 mantissas + one scale.  Thread e writes its 8 B of
// mantissas and its scale byte per slot (consecutive e: consecutive bytes).  The diagonal comes
// after, from the decoded weights (mx8_diag_kernel).
template <int R>
__global__ void __launch_bounds__(256) expand_mx8_kernel(const ExpandArgs a)
{
    constexpr int L = 2 * R + 1, LL = L * L, K = L * L * L;
    const int tile = blockIdx.x;
    const int e = threadIdx.x;
    int zl, q;
    bool real;
    if (a.list) {  // N4: compacted non-uniform chunks
        const long idx = (long)tile * a.tile + e;
        real = idx < a.n_list;
        const int chunk = real ? a.list[idx] : 0;
        const int ot = chunk / a.tile;
        zl = ot / a.tpp;
        q = (ot % a.tpp) * a.tile + chunk % a.tile;
    } else {
        zl = tile / a.tpp;
        q = (tile % a.tpp) * a.tile + e;
        real = q < a.ny * a.nxq;
    }
    unsigned char* wq = reinterpret_cast<unsigned char*>(a.Wt);
    const float* cw = reinterpret_cast<const float*>(a.class_w);
    const int y = real ? q / a.nxq : 0, x = real ? (q % a.nxq) * 8 : 0;
    const long nxp = a.nxp, plane = (long)a.nyp * nxp;
    const int* c0 = a.class_pad + (zl + R) * plane + (long)(y + R) * nxp + kPadX + x;
    for (int r = -1; r < LL; ++r) {  // r = −1: the centre row first (slot order of layout.cuh)
        if (r == R * L + R) continue;
        const int oz = r < 0 ? 0 : r / L - R, oy = r < 0 ? 0 : r % L - R;
        int seg[24];
        const int* srow = c0 - (long)oz * plane - (long)oy * nxp - 8;
#pragma unroll
        for (int i = 0; i < 24; ++i) seg[i] = real ? srow[i] : -1;
#pragma unroll
        for (int ox = -R; ox <= R; ++ox) {
            if (r < 0 && ox == 0) continue;
            const int o = (oz + R) * LL + (oy + R) * L + (ox + R);
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = seg[j - ox + 8];
                v[j] = c >= 0 ? cw[(size_t)c * K + o] : 0.f;
            }
            uint2 m;
            uint32_t E;
            mx8_quant(v, &m, &E);
            size_t mo, so;
            mx8_addr(tile, slot_of(ox, oy, oz, R), e, 0, L, K, a.tile, &mo, &so);
            *reinterpret_cast<uint2*>(wq + mo) = m;
            wq[so] = (unsigned char)E;
        }
    }
}

// diag[target s] = fp32_pair(1 − Σ_{o≠0} decoded W_s(o)) in fp64 (kgen's mass fix, reading A10), the
// source's weights read back from the gather blocks at targets s + o (one thread per source,
// x fastest: neighbouring threads read neighbouring bytes).  Sources outside the domain
// (class −1) and dummy targets keep 0.  One rank (the whole grid is the slab).
template <int R, int TT>  // TT: the tile width when it is 256 (shifts instead of divisions), else 0
__global__ void __launch_bounds__(256) mx8_diag_kernel(const ExpandArgs a, int nzl, const int* __restrict__ cmap,
                                                       const int* __restrict__ chunk_u, const float* __restrict__ ukq,
                                                       float2* __restrict__ udiag_t)
{
    constexpr int L = 2 * R + 1, K = L * L * L;
    const long n = (long)a.nx * a.ny * nzl;
    const unsigned char* wq = reinterpret_cast<const unsigned char*>(a.Wt);
    const long nxp = a.nxp, plane = (long)a.nyp * nxp;
    const int T_ = TT ? TT : a.tile;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const int sx = (int)(i % a.nx), sy = (int)((i / a.nx) % a.ny), sz = (int)(i / ((long)a.nx * a.ny));
        const int cls = a.class_pad[(sz + R) * plane + (long)(sy + R) * nxp + kPadX + sx];
        const int q0 = sy * a.nxq + (sx >> 3);
        const size_t ch0 = ((size_t)sz * a.tpp + q0 / T_) * T_ + q0 % T_;
        float2* dp = a.diag + ch0 * 8 + (sx & 7);
        if (cmap) {  // N4 storage: compact dense position, or the uniform list position
            const int m = cmap[ch0];
            dp = m >= 0 ? a.diag + (size_t)m * 8 + (sx & 7) : udiag_t + (size_t)(-m - 2) * 8 + (sx & 7);
        } else if (a.far_pos) {  // N2 compaction: all-far / identity chunks store no diagonal
            const int m = a.far_pos[ch0];
            if (m < 0) continue;
            dp = a.diag + (size_t)m * 8 + (sx & 7);
        }
        if (cls < 0) {
            *dp = make_float2(0.f, 0.f);
            continue;
        }
        double off = 0.0;
        for (int oz = -R; oz <= R; ++oz) {
            const int z = sz + oz;
            if (z + a.z0 < 0 || z + a.z0 >= a.nz) continue;  // outside the grid
            const bool off_slab = z < 0 || z >= nzl;  // another rank's target (world > 1)
            for (int oy = -R; oy <= R; ++oy) {
                const int y = sy + oy;
                if (y < 0 || y >= a.ny) continue;
#pragma unroll
                for (int ox = -R; ox <= R; ++ox) {
                    const int x = sx + ox;
                    if ((ox == 0 && oy == 0 && oz == 0) || x < 0 || x >= a.nx) continue;
                    const int sl = slot_of(ox, oy, oz, R);
                    if (off_slab) {
                        // that rank stores this block; quantise it here from the class kernels
                        // exactly as its expand_mx8_kernel does (the block's 8 sources
                        // x0 + j − ox lie in this source's own row; identical windows have
                        // bitwise identical kernels, so every rank decides the same codes)
                        const int x0 = x & ~7;
                        const int* crow = a.class_pad + (sz + R) * plane + (long)(sy + R) * nxp + kPadX;
                        const float* cw = reinterpret_cast<const float*>(a.class_w);
                        const int o = (oz + R) * L * L + (oy + R) * L + (ox + R);
                        float v[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int c = crow[x0 + j - ox];
                            v[j] = c >= 0 ? cw[(size_t)c * K + o] : 0.f;
                        }
                        uint2 m;
                        uint32_t E;
                        mx8_quant(v, &m, &E);
                        const int jj = x & 7;
                        off += (double)mx8_decode(((jj < 4 ? m.x : m.y) >> (8 * (jj & 3))) & 0xffu, E);
                        continue;
                    }
                    const int q = y * a.nxq + (x >> 3);
                    size_t tl = (size_t)z * a.tpp + q / T_;
                    int e = q % T_;
                    if (a.far_pos) {  // N2 compaction: no weights stored (all 0) for m < 0
                        const int m = a.far_pos[tl * T_ + e];
                        if (m < 0) continue;
                        tl = (size_t)(m / T_);
                        e = m % T_;
                    } else if (cmap) {
                        const int m = cmap[tl * T_ + e];
                        if (m < 0) {  // uniform chunk: its class kernel, quantised as 8 equal weights
                            off += (double)ukq[(size_t)chunk_u[tl * T_ + e] * (K - 1) + sl];
                            continue;
                        }
                        tl = (size_t)(m / T_);
                        e = m % T_;
                    }
                    size_t mo, so;
                    mx8_addr(tl, sl, e, x & 7, L, K, T_, &mo, &so);
                    off += (double)mx8_decode(__ldg(wq + mo), __ldg(wq + so));
                }
            }
        }
        *dp = fp32_pair((a.class_mass ? a.class_mass[cls] : 1.0) - off);
    }
}

// MX8 + N4 storage: a uniform chunk's block for slot o is 8 equal weights W_u(o), so its
// stored value is W_u(o) quantised alone (m ∈ [128, 255]); ukf is rewritten in place.
__global__ void mx8_uniform_quant_kernel(float* __restrict__ ukf, long n)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = ukf[i];
        uint2 m;
        uint32_t E;
        mx8_quant(v, &m, &E);
        ukf[i] = mx8_decode(m.x & 0xffu, E);
    }
}

__global__ void mx8_chunk_map_kernel(const int* __restrict__ dense, long n_dense, const int* __restrict__ ulist,
                                     long n_uni, int* __restrict__ cmap)
{
    const long n = n_dense + n_uni;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        if (i < n_dense) cmap[dense[i]] = (int)i;
        else cmap[ulist[i - n_dense]] = -(int)(i - n_dense) - 2;
    }
}

template <int R>
static cudaError_t launch_expand_r(const ExpandArgs& a, int fmt, cudaStream_t s)
{
    if (fmt == FDIRW_W_MX8) {
        const int K = (2 * R + 1) * (2 * R + 1) * (2 * R + 1);
        UniformTables* ut = a.ut;
        cudaError_t e = cudaSuccess;
        if (ut) {
            const long nch = (long)a.nzl * a.tpp * a.tile;
            e = cudaMalloc(&ut->chunk_map, nch * 4);
            if (e == cudaSuccess) e = cudaMalloc(&ut->udiag_t, (size_t)std::max<long>(ut->n_uniform, 1) * 8 * 8);
            if (e == cudaSuccess) e = cudaMemsetAsync(ut->chunk_map, 0xff, nch * 4, s);
            if (e == cudaSuccess) e = cudaMemsetAsync(ut->udiag_t, 0, (size_t)std::max<long>(ut->n_uniform, 1) * 64, s);
            if (e == cudaSuccess && ut->n_u > 0) {
                const long n = (long)ut->n_u * (K - 1);
                mx8_uniform_quant_kernel<<<grid_n(n), 256, 0, s>>>(ut->ukf, n);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess && ut->n_dense + ut->n_uniform > 0) {
                mx8_chunk_map_kernel<<<grid_n(ut->n_dense + ut->n_uniform), 256, 0, s>>>(
                    ut->dense_list, ut->n_dense, ut->list, ut->n_uniform, ut->chunk_map);
                e = cudaGetLastError();
            }
            if (e != cudaSuccess) return e;
        }
        if (a.n_tiles > 0) {
            expand_mx8_kernel<R><<<a.n_tiles, a.tile, 0, s>>>(a);
            e = cudaMemsetAsync(a.diag, 0, (size_t)a.n_tiles * a.tile * 8 * 8, s);
            if (e != cudaSuccess) return e;
        }
        if (a.tile == 256)
            mx8_diag_kernel<R, 256><<<148 * 8, 256, 0, s>>>(a, a.nzl, ut ? ut->chunk_map : nullptr,
                                                            ut ? ut->chunk_u : nullptr, ut ? ut->ukf : nullptr,
                                                            ut ? ut->udiag_t : nullptr);
        else
            mx8_diag_kernel<R, 0><<<148 * 8, 256, 0, s>>>(a, a.nzl, ut ? ut->chunk_map : nullptr,
                                                          ut ? ut->chunk_u : nullptr, ut ? ut->ukf : nullptr,
                                                          ut ? ut->udiag_t : nullptr);
        return cudaGetLastError();
    }
    if (a.n_tiles <= 0) return cudaSuccess;
    if (fmt == 0) expand_kernel<R, float><<<a.n_tiles, a.tile, 0, s>>>(a);
    else if (fmt == 1) expand_kernel<R, __half><<<a.n_tiles, a.tile, 0, s>>>(a);
    else expand_kernel<R, __nv_bfloat16><<<a.n_tiles, a.tile, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_expand(const ExpandArgs& a, int R, int fmt, cudaStream_t s)
{
    switch (R) {
        case 1: return launch_expand_r<1>(a, fmt, s);
        case 2: return launch_expand_r<2>(a, fmt, s);
        case 3: return launch_expand_r<3>(a, fmt, s);
        case 4: return launch_expand_r<4>(a, fmt, s);
        case 5: return launch_expand_r<5>(a, fmt, s);
        case 6: return launch_expand_r<6>(a, fmt, s);
        case 7: return launch_expand_r<7>(a, fmt, s);
        case 8: return launch_expand_r<8>(a, fmt, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fdirw
