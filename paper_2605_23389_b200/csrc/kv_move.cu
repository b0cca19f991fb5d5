// Device-to-device KV page moves on the SMs (C2 admit / C3 evict of a (prefetch,
// decode) pair; reference aligned_boundary cluster_sim.hpp:517, :551 price them
// as NVLink transfers).  One CTA per (page, layer) slice gathers the slice from
// the source pool and scatters it into the destination pool (both layer-major in
// page groups, include/asv.h) with 16-byte loads / stores; for the partial last
// page only the s % 16 valid token rows of every 4 KiB (K|V, head) block move,
// so the bytes moved are exactly s * kv_bytes_per_token (cluster_sim.hpp:239-241).
// Across two GPUs the kernel runs on the destination (decode) GPU and pulls over
// NVLink through peer pointers: one launch per request instead of one copy-engine
// call per page.
#include <cuda_runtime.h>
#include <stdint.h>

#include "asv_internal.h"

namespace asv {
namespace {

struct MoveParams {
    const char* src;
    char* dst;
    int64_t slice;           // bytes of one layer of one page
    int64_t src_gp, dst_gp;  // pages per layer-major group of each pool
    int32_t layers;
    int32_t npg;             // pages in this launch
    int32_t last_rows;       // valid rows of this launch's last page (16: whole page)
    int32_t dst_pages[kMoveChunk];
    int32_t src_pages[kMoveChunk];
};

__device__ __forceinline__ int64_t slot_of(int64_t p, int64_t gp, int64_t layers) {
    return p + (p / gp) * gp * (layers - 1);
}

__global__ void __launch_bounds__(256) kv_move_kernel(const __grid_constant__ MoveParams p) {
    const int j = blockIdx.x, l = blockIdx.y;
    const int64_t so = (slot_of(p.src_pages[j], p.src_gp, p.layers) + static_cast<int64_t>(l) * p.src_gp) * p.slice;
    const int64_t dof = (slot_of(p.dst_pages[j], p.dst_gp, p.layers) + static_cast<int64_t>(l) * p.dst_gp) * p.slice;
    const int4* s = reinterpret_cast<const int4*>(p.src + so);
    int4* d = reinterpret_cast<int4*>(p.dst + dof);
    const int rows = j == p.npg - 1 ? p.last_rows : 16;
    if (rows == 16) {
        const int64_t n = p.slice / 16;
        int64_t i = threadIdx.x;
        for (; i + 3 * 256 < n; i += 4 * 256) {  // four 16-byte loads in flight per thread
            const int4 a = s[i], b = s[i + 256], c = s[i + 512], e = s[i + 768];
            d[i] = a;
            d[i + 256] = b;
            d[i + 512] = c;
            d[i + 768] = e;
        }
        for (; i < n; i += 256) d[i] = s[i];
    } else {
        // 4 KiB blocks of 16 rows x 256 B: rows [0, rows) = the first rows * 16 int4 of each block
        const int per = rows * 16;
        const int64_t n = (p.slice / 4096) * per;
        for (int64_t i = threadIdx.x; i < n; i += 256) {
            const int64_t b = i / per, w = i - b * per;
            d[b * 256 + w] = s[b * 256 + w];
        }
    }
}

}  // namespace

cudaError_t kv_move_launch(const void* src_pool, int64_t src_gp, void* dst_pool, int64_t dst_gp, int64_t slice,
                           int32_t layers, const int32_t* src_pages, const int32_t* dst_pages, int64_t tokens,
                           cudaStream_t st) {
    const int64_t npg = (tokens + 15) / 16;
    for (int64_t j0 = 0; j0 < npg; j0 += kMoveChunk) {
        MoveParams p;
        p.src = static_cast<const char*>(src_pool);
        p.dst = static_cast<char*>(dst_pool);
        p.slice = slice;
        p.src_gp = src_gp;
        p.dst_gp = dst_gp;
        p.layers = layers;
        const int64_t n = npg - j0 < kMoveChunk ? npg - j0 : kMoveChunk;
        p.npg = static_cast<int32_t>(n);
        const bool last = j0 + n == npg;
        p.last_rows = last && tokens % 16 != 0 ? static_cast<int32_t>(tokens % 16) : 16;
        for (int64_t j = 0; j < n; ++j) {
            p.dst_pages[j] = dst_pages[j0 + j];
            p.src_pages[j] = src_pages[j0 + j];
        }
        kv_move_kernel<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>(layers)), 256, 0, st>>>(p);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t kv_move_preload() {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, kv_move_kernel);
}

}  // namespace asv
