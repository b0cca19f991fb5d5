// HBM read-bandwidth probe (tools only): the ceiling a streaming-read kernel reaches on
// this B200, to put the decode kernel's achieved GB/s in context beside the driver's
// copy-based peak (MEASURED_PEAKS.json: read+write of a torch copy).
//   ldg:  grid-stride 16-byte loads, 8 in flight per thread, XOR-reduced (no DCE)
//   bulk: per warp a ring of `stages` 4 KiB cp.async.bulk loads (the decode kernel's
//         producer pattern: 4 KiB blocks, mbarrier complete_tx), no compute
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) ldg_kernel(const int4* __restrict__ p, int64_t n, int* out) {
    int acc = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    for (; i < n; i += stride) {
        const int4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x7fffffff) *out = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int S>
__global__ void __launch_bounds__(128) bulk_kernel(const char* __restrict__ p, int64_t nblocks, int* out) {
    extern __shared__ __align__(128) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* ring = smem + warp * (S * 4096 + 128);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * 4096);
    if (lane == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t w = static_cast<int64_t>(blockIdx.x) * 4 + warp, nw = static_cast<int64_t>(gridDim.x) * 4;
    int64_t b = w;
    int acc = 0, issued = 0, consumed = 0;
    auto issue = [&](int slot) {
        if (lane == 0) {
            const uint32_t bar = smem_u32(bars + slot);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(bar) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                             smem_u32(ring + slot * 4096)),
                         "l"(p + b * 4096), "r"(bar)
                         : "memory");
        }
        b += nw;
        ++issued;
    };
    for (int s = 0; s < S && b < nblocks; ++s) issue(s);
    while (consumed < issued) {
        const int slot = consumed % S;
        const uint32_t ph = (consumed / S) & 1;
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(bars + slot)), "r"(ph) : "memory");
        }
        acc ^= reinterpret_cast<const int*>(ring + slot * 4096)[lane];
        __syncwarp();
        ++consumed;
        if (b < nblocks) issue(slot);
    }
    if (acc == 0x7fffffff) *out = acc;
}

extern "C" int probe_ldg(const void* p, int64_t bytes, int* out, int blocks, void* st) {
    ldg_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(st)>>>(static_cast<const int4*>(p), bytes / 16, out);
    return static_cast<int>(cudaGetLastError());
}

extern "C" int probe_bulk(const void* p, int64_t bytes, int* out, int ctas_per_sm, int stages, void* st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 4 * (stages * 4096 + 128);
    cudaError_t e = cudaSuccess;
    switch (stages) {
#define CASE(S)                                                                                          \
    case S:                                                                                              \
        cudaFuncSetAttribute(bulk_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);         \
        bulk_kernel<S><<<sms * ctas_per_sm, 128, smem, static_cast<cudaStream_t>(st)>>>(                 \
            static_cast<const char*>(p), bytes / 4096, out);                                             \
        break;
        CASE(2) CASE(4) CASE(6) CASE(8) CASE(12)
#undef CASE
        default: return -1;
    }
    e = cudaGetLastError();
    return static_cast<int>(e);
}
