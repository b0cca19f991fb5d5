// Decode-step linear layers on the 5th-generation tensor cores (tcgen05) — the
// GEMM half of a decode iteration that the reference prices as the MLP term of
// iteration_latency (cost_model.hpp:60-63, 130-131).
//
// Decode GEMMs have a tiny M (the batch) and are weight-streaming bound, so the
// kernel swaps A and B: the weight rows are the MMA M dimension (128 per tile)
// and the batch is the MMA N dimension (padded to a multiple of 16, <= 256):
//     D[n_out rows][batch] (TMEM, fp32) = W[n_out][K] · X[batch][K]^T
// One CTA per (128-row tile, K split); warp 0 lane 0 streams W and X tiles with
// TMA (2-D tensor maps, 128-byte swizzle) into a multi-stage mbarrier ring,
// warp 1 lane 0 issues tcgen05.mma (kind::f16, bf16 in, fp32 accumulate in
// TMEM) and frees each stage with tcgen05.commit; all four warps then read the
// accumulator with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31 = output
// rows).  The K splits of one tile are one thread-block cluster: partials meet
// in distributed shared memory, each CTA reduces a slice of the batch columns
// and runs the fused epilogue on it:
//   STORE     y[b][n]  = acc
//   RESIDUAL  y[b][n] += acc                         (o_proj / down_proj + residual)
//   SILU_MUL  y[b][j]  = silu(acc_gate) * acc_up       (gate/up rows interleaved per tile)
//   QKV_ROPE  q/k/v heads with rotary embedding on q and k (one head per tile)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <utility>
#include <vector>

#include "../../include/asv.h"
#include "asv_internal.h"
#include "tc_ptx.cuh"

namespace asv {
namespace {

constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 100 * 1024;  // ring <= ~100 KiB: two CTAs per SM keep more of W in flight
constexpr int kMaxSplits = 8;            // K splits of a tile = one portable thread-block cluster
constexpr int kResCols = 64;             // epilogue inputs staged in smem during the main loop: <= 64 columns
constexpr int kResBytes = kResCols * 128 * 2;  // residual rows of this CTA's columns (bf16), or positions
// smem the schedule reserves per epilogue for its staged inputs (STORE, RESIDUAL, SILU_MUL, QKV_ROPE)
constexpr int kStageMargin[4] = {0, 2048, 0, 1024};

struct LinearParams {
    int32_t n_out, k, batch, bn;     // bn: batch padded to a multiple of 16 (MMA N)
    int32_t kb_per_split, splits, stages;
    int32_t epi;
    __nv_bfloat16* y;
    int32_t y_ld;
    // QKV_ROPE
    const int32_t* positions;        // [batch] position of the new token
    float rope_log2_theta;           // log2(theta)
    __nv_bfloat16 *q, *kk, *v;       // [batch][heads][128]
    int32_t n_q_heads, n_kv_heads;
    // fused RMSNorm (asv.h): producer writes ss_out, consumer scales by rsqrt(sum(ss_in) / dim + eps)
    float* ss_out;
    const float* ss_in;
    int32_t ss_parts, ss_ld;
    float ss_inv_dim, ss_eps;
    // next linear's first ring stages -> L2 (0 tiles: off)
    int32_t next_tiles, next_splits, next_kb_per_split, next_kbs, next_pre, next_first;
    unsigned long long* trace;       // optional [grid][kTrSlots] %globaltimer stamps (asv_linear_trace)
    int32_t staged_bytes;            // smem bytes of the staged inputs
    int32_t stage_in;                // 1: the idle warps stage the epilogue's inputs (residual rows /
                                     // positions of this CTA's columns) in smem during the main loop
};

// timeline probe (asv_linear_trace, measurement only): per CTA of a launch
//   0 entry  1 producer: activations' dependency satisfied  2 producer: last weight load issued
//   3 MMA: first stage landed  4 accumulator complete  5 cluster reduce entered  6 exit  7 SM id
constexpr int kTrSlots = 8, kTrLaunches = 64, kTrCtas = 1024;
__device__ __forceinline__ void trace_stamp(const LinearParams& p, int slot) {
    if (p.trace == nullptr) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[static_cast<int64_t>(blockIdx.x) * kTrSlots + slot] = t;
}

using namespace tc;

// ------------------------------------------------------------------ kernel
// smem: [stages][A 16 KiB][B bn*128 B] (1024-aligned) | full[stages] empty[stages] done | tmem base
template <int EPI>
__global__ void __launch_bounds__(128, 2)
    linear_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                  const __grid_constant__ CUtensorMap tm_next, const LinearParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = kABytes + p.bn * 128;
    const int nst = p.stages;
    // the epilogue reuses the ring for the [bn][128] fp32 accumulator tile: barriers after both
    const int ring = nst * stage_bytes > p.bn * 512 ? nst * stage_bytes : p.bn * 512;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages + 1);
    float* rs = reinterpret_cast<float*>(tmem_slot + 4);  // fused RMSNorm: 1/rms per batch column of this CTA
    // epilogue inputs staged during the main loop (stage_in): residual rows [column][128] bf16 or positions
    uint8_t* staged = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rs + 256) + 15) & ~uintptr_t(15));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0 && p.trace != nullptr) {
        trace_stamp(p, 0);
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[static_cast<int64_t>(blockIdx.x) * kTrSlots + 7] = smid;
    }
    const int tile = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
    const int kb0 = split * p.kb_per_split;
    const int kb1 = min(kb0 + p.kb_per_split, p.k / kBK);
    const uint32_t ncols = p.bn <= 32 ? 32 : p.bn <= 64 ? 64 : p.bn <= 128 ? 128 : 256;

    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kMaxStages), done = smem_u32(bars + 2 * kMaxStages);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_w)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_x)) : "memory");
    }
    if (warp == 1) {  // TMEM accumulator: 128 lanes x ncols fp32
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // the next kernel may start its own prologue / weight prefetch now (it waits for
    // this grid's completion before touching what this grid writes)
    grid_dep_launch();

    if (warp == 0 && lane == 0) {
        // ---- TMA producer: W tiles (streamed once: evict-first), X tiles (reused by every tile: evict-last)
        // The weights never depend on the previous kernel: the first ring's worth
        // of W is requested BEFORE griddepcontrol.wait (with PDL this overlaps the
        // producing kernel's tail); the activations X only after it.
        const uint64_t pw = policy_evict_first(), px = policy_evict_last();
        const int pre = min(nst, kb1 - kb0);
        for (int i = 0; i < pre; ++i) {
            mbar_expect_tx(full0 + 8 * i, static_cast<uint32_t>(stage_bytes));
            tma_load_2d(smem_u32(smem + i * stage_bytes), &tm_w, (kb0 + i) * kBK, tile * kBM, full0 + 8 * i, pw);
        }
        grid_dep_wait();
        trace_stamp(p, 1);
        for (int i = 0; i < pre; ++i) {
            tma_load_2d(smem_u32(smem + i * stage_bytes) + kABytes, &tm_x, (kb0 + i) * kBK, 0, full0 + 8 * i, px);
        }
        int s = pre == nst ? 0 : pre;
        uint32_t ph = pre == nst ? 1 : 0;
        for (int kb = kb0 + pre; kb < kb1; ++kb) {
            mbar_wait(empty0 + 8 * s, ph ^ 1);
            const uint32_t a = smem_u32(smem + s * stage_bytes);
            mbar_expect_tx(full0 + 8 * s, static_cast<uint32_t>(stage_bytes));
            tma_load_2d(a, &tm_w, kb * kBK, tile * kBM, full0 + 8 * s, pw);
            tma_load_2d(a + kABytes, &tm_x, kb * kBK, 0, full0 + 8 * s, px);
            if (++s == nst) {
                s = 0;
                ph ^= 1;
            }
        }
        trace_stamp(p, 2);
        // every weight load of this CTA is issued: keep HBM busy through the tail and the next launch's
        // prologue by pulling a share of the next linear's first ring stages into L2
        if (p.next_tiles > 0) {
            const int total = p.next_tiles * p.next_splits * p.next_pre;
            for (int i = blockIdx.x; i < total; i += gridDim.x) {
                const int j = i / p.next_pre, st = i - j * p.next_pre;
                const int nt = j / p.next_splits, ns = j - nt * p.next_splits;
                const int kb = ns * p.next_kb_per_split + p.next_first + st;  // after the next CTA's ring
                if (p.next_first + st < p.next_kb_per_split && kb < p.next_kbs)
                    tma_prefetch_l2(&tm_next, kb * kBK, nt * kBM);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: one thread drives the tensor core for the whole CTA
        const uint32_t idesc = umma_idesc(static_cast<uint32_t>(p.bn));
        int s = 0;
        uint32_t ph = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(full0 + 8 * s, ph);
            if (kb == kb0) trace_stamp(p, 3);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + s * stage_bytes);
            const uint64_t ad = umma_desc_sw128(a), bd = umma_desc_sw128(a + kABytes);
#pragma unroll
            for (int kk = 0; kk < kBK / kUmmaK; ++kk) {
                // +32 bytes of K per step inside the 128-byte swizzle row: +2 in the >>4 address field
                umma_f16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            }
            umma_commit(empty0 + 8 * s);  // stage reusable once these MMAs have read it
            if (++s == nst) {
                s = 0;
                ph ^= 1;
            }
        }
        umma_commit(done);  // accumulator complete
    } else if (warp >= 2 && (p.ss_in != nullptr || p.stage_in != 0)) {
        grid_dep_wait();
        const int per_c = (p.batch + p.splits - 1) / p.splits;
        const int c0 = split * per_c, c1 = min(c0 + per_c, p.batch);
        if (p.stage_in != 0) {
            // the epilogue's other inputs (written by the previous kernel) come to smem now, so the
            // reduce after the last MMA has no global-memory round trip on its critical path
            const int t = static_cast<int>(threadIdx.x) - 64;
            if constexpr (EPI == ASV_EPI_RESIDUAL) {
                uint4* dst = reinterpret_cast<uint4*>(staged);
                for (int i = t; i < (c1 - c0) * 16; i += 64) {
                    const int c = i >> 4, j = i & 15;
                    dst[i] = __ldcg(reinterpret_cast<const uint4*>(p.y + static_cast<int64_t>(c0 + c) * p.y_ld +
                                                                   tile * kBM) + j);
                }
            } else if constexpr (EPI == ASV_EPI_QKV_ROPE) {
                int32_t* dst = reinterpret_cast<int32_t*>(staged);
                for (int c = c0 + t; c < c1; c += 64) dst[c - c0] = __ldcg(p.positions + c);
            }
        }
        // fused RMSNorm: the two idle warps turn the producer's partial sums of squares into
        // 1/rms for this CTA's batch columns while the main loop runs (8 independent partial
        // sums per column, combined in a fixed order: deterministic)
        for (int c = c0 + static_cast<int>(threadIdx.x) - 64; p.ss_in != nullptr && c < c1; c += 64) {
            float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            int i = 0;
            for (; i + 8 <= p.ss_parts; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc8[j] += p.ss_in[static_cast<int64_t>(i + j) * p.ss_ld + c];
            }
            for (; i < p.ss_parts; ++i) acc8[0] += p.ss_in[static_cast<int64_t>(i) * p.ss_ld + c];
            const float ssum = ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
            rs[c - c0] = rsqrtf(ssum * p.ss_inv_dim + p.ss_eps);
        }
    }
    __syncwarp();

    // ---- epilogue 1: TMEM -> this CTA's smem as [bn][128] fp32 (the ring is free:
    // every stage was consumed by an MMA that has completed)
    mbar_wait(done, 0);
    if (threadIdx.x == 0) trace_stamp(p, 4);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    float* part = reinterpret_cast<float*>(smem);
    for (int c0 = 0; c0 < p.bn; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + static_cast<uint32_t>(c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) part[(c0 + i) * kBM + threadIdx.x] = v[i];
    }
    tc_fence_before();
    __syncthreads();  // (also publishes the fused-RMSNorm scales rs[] to every thread)
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
    }
    // ---- epilogue 2: the K splits of this tile form one thread-block cluster; after a
    // cluster barrier every CTA reduces a slice of the batch columns straight out of
    // the other CTAs' shared memory (DSMEM) and applies the fused epilogue to it.
    // Thread t handles row pair (r, r + 64), r = t & 63, so the SiLU gate/up and
    // RoPE rotate-half partners are in one thread's registers.
    if (p.splits > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    grid_dep_wait();  // outputs / residual / positions may belong to the previous kernel
    if (threadIdx.x == 0) trace_stamp(p, 5);
    const int per = (p.batch + p.splits - 1) / p.splits;
    const int cb = split * per, ce = min(cb + per, p.batch);
    const int r = threadIdx.x & 63;
    const uint32_t part_s = smem_u32(part);
    for (int c = cb + (threadIdx.x >> 6); c < ce; c += 2) {
        float lo = 0.f, hi = 0.f;
        const uint32_t off_lo = part_s + static_cast<uint32_t>((c * kBM + r) * 4);
        if (p.splits > 1) {
            // every split's partial in flight at once, then summed in split order (deterministic)
            float x0[kMaxSplits], x1[kMaxSplits];
#pragma unroll
            for (int s2 = 0; s2 < kMaxSplits; ++s2) {
                if (s2 < p.splits) {
                    uint32_t ra;
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(off_lo), "r"(s2));
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x0[s2]) : "r"(ra));
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x1[s2]) : "r"(ra + 64 * 4));
                }
            }
#pragma unroll
            for (int s2 = 0; s2 < kMaxSplits; ++s2) {
                if (s2 < p.splits) {
                    lo += x0[s2];
                    hi += x1[s2];
                }
            }
        } else {
            lo = part[c * kBM + r];
            hi = part[c * kBM + r + 64];
        }
        const int b = c;
        if (p.ss_in != nullptr) {
            lo *= rs[c - cb];
            hi *= rs[c - cb];
        }
        if constexpr (EPI == ASV_EPI_STORE || EPI == ASV_EPI_RESIDUAL) {
            __nv_bfloat16* dst = p.y + static_cast<int64_t>(b) * p.y_ld + tile * kBM + r;
            if constexpr (EPI == ASV_EPI_RESIDUAL) {
                if (p.stage_in != 0) {
                    const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(staged) + (c - cb) * kBM + r;
                    lo += __bfloat162float(res[0]);
                    hi += __bfloat162float(res[64]);
                } else {
                    lo += __bfloat162float(dst[0]);
                    hi += __bfloat162float(dst[64]);
                }
            }
            const __nv_bfloat16 blo = __float2bfloat16(lo), bhi = __float2bfloat16(hi);
            dst[0] = blo;
            dst[64] = bhi;
            if (p.ss_out != nullptr) {  // the next linear's fused RMSNorm: sum of squares of the stored row
                const float fl = __bfloat162float(blo), fh = __bfloat162float(bhi);
                float sq = fl * fl + fh * fh;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
                if ((threadIdx.x & 31) == 0)
                    p.ss_out[static_cast<int64_t>(tile * 2 + ((threadIdx.x >> 5) & 1)) * p.ss_ld + b] = sq;
            }
        } else if constexpr (EPI == ASV_EPI_SILU_MUL) {
            // tile rows [0,64) gate, [64,128) the matching up rows of outputs 64*tile + r
            p.y[static_cast<int64_t>(b) * p.y_ld + tile * 64 + r] = __float2bfloat16(silu(lo) * hi);
        } else if constexpr (EPI == ASV_EPI_QKV_ROPE) {
            // one head per tile: [q heads | k heads | v heads]; rotate-half RoPE on q and k
            const int head = tile;
            const bool is_q = head < p.n_q_heads, is_k = !is_q && head < p.n_q_heads + p.n_kv_heads;
            __nv_bfloat16* dst = is_q ? p.q : is_k ? p.kk : p.v;
            const int h = is_q ? head : is_k ? head - p.n_q_heads : head - p.n_q_heads - p.n_kv_heads;
            const int nh = is_q ? p.n_q_heads : p.n_kv_heads;
            if (is_q || is_k) {
                const float inv_freq = exp2f(-p.rope_log2_theta * (2.f * r / 128.f));  // theta^(-2r/128)
                float sn, cs;
                const int32_t pos = p.stage_in != 0 ? reinterpret_cast<const int32_t*>(staged)[c - cb] : p.positions[b];
                sincosf(static_cast<float>(pos) * inv_freq, &sn, &cs);
                const float a0 = lo * cs - hi * sn, a1 = hi * cs + lo * sn;
                lo = a0;
                hi = a1;
            }
            __nv_bfloat16* o = dst + (static_cast<int64_t>(b) * nh + h) * 128;
            o[r] = __float2bfloat16(lo);
            o[r + 64] = __float2bfloat16(hi);
        }
    }
    if (p.splits > 1) {  // no CTA may exit while a peer still reads its shared memory
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) trace_stamp(p, 6);
}

// ------------------------------------------------------------------ host side
unsigned long long* g_trace = nullptr;  // [kTrLaunches][kTrCtas][kTrSlots] (asv_linear_trace)
int g_trace_seq = 0, g_trace_skipped = 0;
std::mutex g_trace_mu;
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<EncodeFn>(p);
        }
    });
    return fn;
}

// 2-D bf16 row-major [rows][cols] map with a {64, box_rows} box and 128-byte swizzle
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeFn fn = encode_fn();
    if (fn == nullptr) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// smem of one CTA: the ring (the epilogue reuses it for the [bn][128] fp32 accumulator tile),
// barriers, TMEM slot, 1/rms scales and the staged epilogue inputs (LinearParams::stage_in)
int smem_for(int bn, int stages, int staged) {
    const int ring = stages * (kABytes + bn * 128);
    return (ring > bn * 512 ? ring : bn * 512) + 1024 + (2 * kMaxStages + 1) * 8 + 16 + 256 * 4 + 16 + staged;
}

template <int EPI>
cudaError_t configure_epi() {
    static cudaError_t once = cudaFuncSetAttribute(linear_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   227 * 1024);  // the sm_100 per-CTA maximum
    return once;
}
template <int EPI>
cudaError_t launch_epi(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& tn, const LinearParams& p,
                       int grid, bool pdl, cudaStream_t st) {
    const cudaError_t ce = configure_epi<EPI>();
    if (ce != cudaSuccess) return ce;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem_for(p.bn, p.stages, p.stage_in != 0 ? p.staged_bytes : 0);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (p.splits > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;  // the K splits of a tile form a cluster
        attr[n].val.clusterDim.x = p.splits;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, linear_kernel<EPI>, tw, tx, tn, p);
}

}  // namespace

// Round-1 schedule (ASV_LINEAR_PLAN=0, A/B only): the largest power-of-two split with
// tiles x splits <= 2 CTAs per SM and a fixed ~100 KiB ring.
int linear_splits_r1(int n_out, int k, int sms) {
    const int tiles = n_out / kBM, kbs = k / kBK;
    int sp = 1;
    while (sp * 2 <= kMaxSplits && sp * 2 <= kbs / 2 && tiles * sp * 2 <= 2 * sms) sp *= 2;
    const int per = (kbs + sp - 1) / sp;
    return (kbs + per - 1) / per;
}
int stages_r1(int bn) {
    const int st = kSmemBudget / (kABytes + bn * 128);
    return st < 2 ? 2 : st > kMaxStages ? kMaxStages : st;
}

// Schedule of one decode linear layer: K splits per tile (= cluster size) and ring stages.
// A weight-streaming GEMM runs at the rate its bytes in flight allow (Little's law; measured on
// B200: ~16 MB in flight -> 6.0 TB/s, ~23 MB -> 6.9 TB/s, profiles/linear_trace_r02g.txt), so the
// schedule maximises the grid's ring bytes in flight, CTAs x min(stages, K blocks per split) x
// stage bytes (saturating at kFlyCap), over every (splits, stages) that runs in ONE wave: CTAs per
// SM from shared memory and TMEM columns, and clusters filling at most kClusterFill of the slots
// (GPC placement: a 3-CTA cluster schedule at 97% of the slots ran as two waves).  Near-ties go to
// more, smaller CTAs.  Measured against every (splits, stages) of the 7B projections at batch
// 4/16/64 (tools/linear_schedule_sweep.py, profiles/linear_sched_sweep_r02.jsonl): within 1.6% of
// the best forced schedule in total, 3.8% faster than round 1's fixed ~100 KiB ring / power-of-two
// split.  (cudaOccupancyMaxActiveClusters reports ~1 CTA per SM for this kernel whatever its
// shared memory, so the model is explicit.)  Cached per shape.
struct LinPlan {
    int splits, stages;
};
LinPlan g_force{0, 0};
std::mutex g_force_mu;
constexpr double kFlyCap = 24e6, kFlyTie = 1.03, kClusterFill = 0.9;
// tuning experiments only: ASV_LINEAR_FLYCAP_MB / ASV_LINEAR_FILL override the two model constants
double fly_cap() {
    static const double v = [] {
        const char* e = getenv("ASV_LINEAR_FLYCAP_MB");
        return e != nullptr ? atof(e) * 1e6 : kFlyCap;
    }();
    return v;
}
double cluster_fill() {
    static const double v = [] {
        const char* e = getenv("ASV_LINEAR_FILL");
        return e != nullptr ? atof(e) : kClusterFill;
    }();
    return v;
}

template <int EPI>
LinPlan linear_plan(int n_out, int k, int bn, int sms) {
    static std::mutex mu;
    static std::vector<std::pair<uint64_t, LinPlan>> cache;
    const uint64_t key = (static_cast<uint64_t>(n_out) << 40) ^ (static_cast<uint64_t>(k) << 16) ^
                         (static_cast<uint64_t>(bn) << 4) ^ static_cast<uint64_t>(sms & 15);
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : cache)
        if (e.first == key) return e.second;
    static const int mode = [] {
        const char* e = getenv("ASV_LINEAR_PLAN");
        return e != nullptr ? atoi(e) : 1;
    }();
    static const int verbose = [] {
        const char* e = getenv("ASV_LINEAR_PLAN_LOG");
        return e != nullptr ? atoi(e) : 0;
    }();
    const int tiles = n_out / kBM, kbs = k / kBK, stage_bytes = kABytes + bn * 128;
    const int ncols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
    LinPlan best{linear_splits_r1(n_out, k, sms), stages_r1(bn)};
    if (mode != 0) {
        double best_fly = -1.0;
        int best_ctas = 0;
        for (int sp = 1; sp <= kMaxSplits; ++sp) {
            const int per = (kbs + sp - 1) / sp;
            if ((sp > 1 && per < 2) || (kbs + per - 1) / per != sp) continue;
            for (int st = 2; st <= kMaxStages; ++st) {
                const int smem = smem_for(bn, st, kStageMargin[EPI]);
                if (smem > 227 * 1024) break;
                const int by_smem = (228 * 1024) / (smem + 1024), by_tmem = 512 / ncols;
                const int slots = (by_smem < by_tmem ? by_smem : by_tmem) * sms;
                const int ctas = tiles * sp;
                if (ctas > (sp > 1 ? static_cast<int>(slots * cluster_fill()) : slots)) continue;
                double fly = static_cast<double>(ctas) * (st < per ? st : per) * stage_bytes;
                if (fly > fly_cap()) fly = fly_cap();
                if (verbose > 1)
                    fprintf(stderr, "  cand splits %d stages %d: %d CTAs, %d slots, %.1f MB in flight\n", sp, st, ctas,
                            slots, fly / 1e6);
                if (best_fly < 0.0 || fly > best_fly * kFlyTie || (fly * kFlyTie >= best_fly && ctas > best_ctas)) {
                    best_fly = fly;
                    best_ctas = ctas;
                    best = LinPlan{sp, st};
                }
            }
        }
    }
    cache.emplace_back(key, best);
    if (verbose > 0)
        fprintf(stderr, "asv_linear plan: n_out %d k %d bn %d epi %d -> splits %d stages %d (%d CTAs)\n", n_out, k, bn,
                EPI, best.splits, best.stages, tiles * best.splits);
    return best;
}

cudaError_t linear_preload() {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, linear_kernel<ASV_EPI_STORE>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, linear_kernel<ASV_EPI_RESIDUAL>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, linear_kernel<ASV_EPI_SILU_MUL>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, linear_kernel<ASV_EPI_QKV_ROPE>);
    return e;
}

static int linear_run(const asv_linear_args* a, cudaStream_t st) {
    if (a == nullptr || a->w == nullptr || a->x == nullptr) return fail(ASV_ERR_INVALID, "linear: null pointer");
    if (a->n_out <= 0 || a->n_out % kBM != 0) return fail(ASV_ERR_INVALID, "linear: n_out must be a multiple of 128");
    if (a->k <= 0 || a->k % kBK != 0) return fail(ASV_ERR_INVALID, "linear: k must be a multiple of 64");
    if (a->batch < 1 || a->batch > 256) return fail(ASV_ERR_INVALID, "linear: batch must be in [1, 256]");
    const int bn = ((a->batch + 15) / 16) * 16;
    if (a->x_rows < bn) return fail(ASV_ERR_INVALID, "linear: x must have >= batch rounded up to 16 rows");
    if (a->epilogue == ASV_EPI_QKV_ROPE) {
        if (a->positions == nullptr || a->q == nullptr || a->k_out == nullptr || a->v_out == nullptr ||
            a->n_out != 128 * (a->n_q_heads + 2 * a->n_kv_heads))
            return fail(ASV_ERR_INVALID, "linear: bad QKV/RoPE arguments");
    } else if (a->y == nullptr) {
        return fail(ASV_ERR_INVALID, "linear: null y");
    }
    if (a->ss_out != nullptr && (a->epilogue != ASV_EPI_RESIDUAL || a->ss_ld < a->batch))
        return fail(ASV_ERR_INVALID, "linear: ss_out needs the RESIDUAL epilogue and ss_ld >= batch");
    if (a->ss_in != nullptr && (a->ss_parts < 1 || a->ss_ld < a->batch || a->ss_dim < 1))
        return fail(ASV_ERR_INVALID, "linear: bad fused-RMSNorm arguments (ss_parts, ss_ld, ss_dim)");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = a->n_out / kBM, kbs = a->k / kBK;
    LinPlan plan{1, 2};
    switch (a->epilogue) {
        case ASV_EPI_STORE: plan = linear_plan<ASV_EPI_STORE>(a->n_out, a->k, bn, sms); break;
        case ASV_EPI_RESIDUAL: plan = linear_plan<ASV_EPI_RESIDUAL>(a->n_out, a->k, bn, sms); break;
        case ASV_EPI_SILU_MUL: plan = linear_plan<ASV_EPI_SILU_MUL>(a->n_out, a->k, bn, sms); break;
        case ASV_EPI_QKV_ROPE: plan = linear_plan<ASV_EPI_QKV_ROPE>(a->n_out, a->k, bn, sms); break;
        default: return fail(ASV_ERR_INVALID, "linear: unknown epilogue");
    }
    {
        std::lock_guard<std::mutex> lk(g_force_mu);
        if (g_force.splits > 0) {  // asv_linear_set_schedule (measurement only); no empty split
            const int kbs_ = a->k / kBK, want = g_force.splits < kbs_ ? g_force.splits : kbs_;
            const int per = (kbs_ + want - 1) / want;
            plan.splits = (kbs_ + per - 1) / per;
            plan.stages = g_force.stages > 1 ? (g_force.stages > kMaxStages ? kMaxStages : g_force.stages) : plan.stages;
        }
    }
    int splits = plan.splits;
    if (const char* e = getenv("ASV_LINEAR_SPLITS")) {  // tuning experiments only
        const int kbs_ = a->k / kBK, want = atoi(e);
        if (want >= 1 && want <= kMaxSplits && want <= kbs_) {
            const int per = (kbs_ + want - 1) / want;
            splits = (kbs_ + per - 1) / per;
        }
    }
    CUtensorMap tw, tx;
    if (!make_map(&tw, a->w, static_cast<uint64_t>(a->n_out), static_cast<uint64_t>(a->k), kBM) ||
        !make_map(&tx, a->x, static_cast<uint64_t>(a->x_rows), static_cast<uint64_t>(a->k), static_cast<uint32_t>(bn)))
        return fail(ASV_ERR_CUDA, "linear: cuTensorMapEncodeTiled failed");
    LinearParams p{};
    p.n_out = a->n_out;
    p.k = a->k;
    p.batch = a->batch;
    p.bn = bn;
    p.splits = splits;
    p.stages = plan.stages;
    p.kb_per_split = (kbs + splits - 1) / splits;
    p.epi = a->epilogue;
    p.y = static_cast<__nv_bfloat16*>(a->y);
    p.y_ld = a->y_ld;
    p.positions = a->positions;
    p.rope_log2_theta = log2f(a->rope_theta > 0.f ? a->rope_theta : 10000.f);
    p.q = static_cast<__nv_bfloat16*>(a->q);
    p.kk = static_cast<__nv_bfloat16*>(a->k_out);
    p.v = static_cast<__nv_bfloat16*>(a->v_out);
    p.n_q_heads = a->n_q_heads;
    p.n_kv_heads = a->n_kv_heads;
    p.ss_out = a->ss_out;
    p.ss_in = a->ss_in;
    p.ss_parts = a->ss_parts;
    p.ss_ld = a->ss_ld;
    p.ss_inv_dim = a->ss_dim > 0 ? 1.f / static_cast<float>(a->ss_dim) : 0.f;
    p.ss_eps = a->ss_eps;
    {
        const int per = (a->batch + splits - 1) / splits;
        if (a->epilogue == ASV_EPI_RESIDUAL) {
            p.staged_bytes = per * kBM * 2;
            p.stage_in = per <= kResCols && (reinterpret_cast<uintptr_t>(a->y) & 15) == 0 && a->y_ld % 8 == 0;
        } else if (a->epilogue == ASV_EPI_QKV_ROPE) {
            p.staged_bytes = (per * 4 + 15) / 16 * 16;
            p.stage_in = p.staged_bytes <= kResBytes;
        }
        // never at the cost of the second CTA per SM (228 KiB per SM, 1 KiB reserved per CTA)
        // never beyond the room the schedule left for them (it may cost a co-resident CTA)
        if (p.staged_bytes > kStageMargin[a->epilogue]) p.stage_in = 0;
        static const bool no_stage = getenv("ASV_LINEAR_NO_STAGE") != nullptr;  // A/B only
        if (no_stage) p.stage_in = 0;
    }
    // the next linear's weights: ASV_LINEAR_NEXT_PF=N prefetches the first N ring stages of every
    // next-launch CTA into L2 from this launch's tail.  Off by default: measured on B200 (r02, C2 full
    // step 565.8 tok/s off vs 559-568 with N = 2..8; 7B GEMM stack -2 to -4%), the boundary is not an
    // idle-HBM gap that L2 prefetch can fill
    CUtensorMap tn = tw;
    static const int next_pf = [] {
        const char* e = getenv("ASV_LINEAR_NEXT_PF");
        return e != nullptr ? atoi(e) : 0;
    }();
    if (a->next_w != nullptr && next_pf != 0 && a->next_n_out > 0 && a->next_n_out % kBM == 0 && a->next_k > 0 &&
        a->next_k % kBK == 0 && make_map(&tn, a->next_w, static_cast<uint64_t>(a->next_n_out),
                                         static_cast<uint64_t>(a->next_k), kBM)) {
        LinPlan np{1, 2};  // the next launch's schedule: its ring covers its first np.stages K blocks
        switch (a->next_epilogue) {
            case ASV_EPI_RESIDUAL: np = linear_plan<ASV_EPI_RESIDUAL>(a->next_n_out, a->next_k, bn, sms); break;
            case ASV_EPI_SILU_MUL: np = linear_plan<ASV_EPI_SILU_MUL>(a->next_n_out, a->next_k, bn, sms); break;
            case ASV_EPI_QKV_ROPE: np = linear_plan<ASV_EPI_QKV_ROPE>(a->next_n_out, a->next_k, bn, sms); break;
            default: np = linear_plan<ASV_EPI_STORE>(a->next_n_out, a->next_k, bn, sms); break;
        }
        const int nsp = np.splits;
        p.next_tiles = a->next_n_out / kBM;
        p.next_splits = nsp;
        p.next_kbs = a->next_k / kBK;
        p.next_kb_per_split = (p.next_kbs + nsp - 1) / nsp;
        p.next_first = next_pf > 0 ? np.stages : 0;  // ASV_LINEAR_NEXT_PF < 0: the ring's own stages (A/B)
        p.next_pre = next_pf > 0 ? next_pf : -next_pf;
    }
    const int grid = tiles * splits;
    {
        std::lock_guard<std::mutex> lk(g_trace_mu);
        static const int skip = [] {  // ASV_LINEAR_TRACE_SKIP=n: record from the n-th armed launch on
            const char* e = getenv("ASV_LINEAR_TRACE_SKIP");
            return e != nullptr ? atoi(e) : 0;
        }();
        if (g_trace != nullptr && grid <= kTrCtas && g_trace_seq < kTrLaunches && g_trace_skipped++ >= skip)
            p.trace = g_trace + static_cast<int64_t>(g_trace_seq++) * kTrCtas * kTrSlots;
    }
    cudaError_t e;
    switch (a->epilogue) {
        case ASV_EPI_STORE: e = launch_epi<ASV_EPI_STORE>(tw, tx, tn, p, grid, a->pdl != 0, st); break;
        case ASV_EPI_RESIDUAL: e = launch_epi<ASV_EPI_RESIDUAL>(tw, tx, tn, p, grid, a->pdl != 0, st); break;
        case ASV_EPI_SILU_MUL: e = launch_epi<ASV_EPI_SILU_MUL>(tw, tx, tn, p, grid, a->pdl != 0, st); break;
        case ASV_EPI_QKV_ROPE: e = launch_epi<ASV_EPI_QKV_ROPE>(tw, tx, tn, p, grid, a->pdl != 0, st); break;
        default: return fail(ASV_ERR_INVALID, "linear: unknown epilogue");
    }
    if (e != cudaSuccess) return cuda_fail(e, "linear launch");
    return ASV_OK;
}

// ------------------------------------------------------------------ RMSNorm
// out[b][:] = h[b][:] * rsqrt(mean(h^2) + eps) * gamma, rows [batch, rows_out) zeroed
// (they are the MMA-N padding of the next linear layer's activation tile)
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* __restrict__ h,
                                                      const __nv_bfloat16* __restrict__ gamma,
                                                      __nv_bfloat16* __restrict__ out, int dim, int batch, float eps) {
    // one row per CTA, one pass: every thread keeps its <= 4 x 8 values in registers
    constexpr int kVec = 4;
    grid_dep_wait();  // h is the previous kernel's output (no-op without PDL)
    grid_dep_launch();
    const int b = blockIdx.x;
    __nv_bfloat16* o = out + static_cast<int64_t>(b) * dim;
    if (b >= batch) {
        for (int i = threadIdx.x * 8; i < dim; i += blockDim.x * 8) *reinterpret_cast<uint4*>(o + i) = make_uint4(0, 0, 0, 0);
        return;
    }
    const __nv_bfloat16* x = h + static_cast<int64_t>(b) * dim;
    uint4 u[kVec], g[kVec];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
        const int i = (threadIdx.x + j * blockDim.x) * 8;
        if (i < dim) {
            u[j] = *reinterpret_cast<const uint4*>(x + i);
            g[j] = __ldg(reinterpret_cast<const uint4*>(gamma + i));
            const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&u[j]);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float f = __bfloat162float(e[t]);
                ss += f * f;
            }
        }
    }
    __shared__ float red[32];
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / dim + eps);
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
        const int i = (threadIdx.x + j * blockDim.x) * 8;
        if (i < dim) {
            const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&u[j]);
            const __nv_bfloat16* ge = reinterpret_cast<const __nv_bfloat16*>(&g[j]);
            uint4 r;
            __nv_bfloat16* re = reinterpret_cast<__nv_bfloat16*>(&r);
#pragma unroll
            for (int t = 0; t < 8; ++t) re[t] = __float2bfloat16(__bfloat162float(e[t]) * inv * __bfloat162float(ge[t]));
            *reinterpret_cast<uint4*>(o + i) = r;
        }
    }
}

cudaError_t rmsnorm_launch(const void* h, const void* gamma, void* out, int dim, int batch, int rows_out, float eps,
                           bool pdl, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(rows_out);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, rmsnorm_kernel, static_cast<const __nv_bfloat16*>(h),
                              static_cast<const __nv_bfloat16*>(gamma), static_cast<__nv_bfloat16*>(out), dim, batch,
                              eps);
}

// synthetic weights / activations: splitmix64(seed + i) -> U[-1, 1) * scale + offset, bf16
__global__ void fill_random_kernel(__nv_bfloat16* p, int64_t n, uint64_t seed, float scale, float offset) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + static_cast<uint64_t>(i) * 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f) * 2.f - 1.f;
        p[i] = __float2bfloat16(u * scale + offset);
    }
}

cudaError_t fill_random_bf16(void* p, int64_t n, uint64_t seed, float scale, float offset, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    fill_random_kernel<<<148 * 8, 256, 0, st>>>(static_cast<__nv_bfloat16*>(p), n, seed, scale, offset);
    return cudaGetLastError();
}

cudaError_t rmsnorm_preload() {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, rmsnorm_kernel);
}

}  // namespace asv

// ------------------------------------------------------------------ C ABI
extern "C" {

int asv_linear(const asv_linear_args* args, void* stream) {
    return asv::linear_run(args, static_cast<cudaStream_t>(stream));
}

int asv_linear_schedule(int32_t n_out, int32_t k, int32_t batch, int32_t epilogue, int32_t sms, int32_t* splits,
                        int32_t* stages, int32_t* smem_bytes) {
    if (n_out <= 0 || n_out % asv::kBM != 0 || k <= 0 || k % asv::kBK != 0 || batch < 1 || batch > 256 || sms < 1)
        return asv::fail(ASV_ERR_INVALID, "linear_schedule: bad shape");
    const int bn = (batch + 15) / 16 * 16;
    asv::LinPlan pl{1, 2};
    switch (epilogue) {
        case ASV_EPI_STORE: pl = asv::linear_plan<ASV_EPI_STORE>(n_out, k, bn, sms); break;
        case ASV_EPI_RESIDUAL: pl = asv::linear_plan<ASV_EPI_RESIDUAL>(n_out, k, bn, sms); break;
        case ASV_EPI_SILU_MUL: pl = asv::linear_plan<ASV_EPI_SILU_MUL>(n_out, k, bn, sms); break;
        case ASV_EPI_QKV_ROPE: pl = asv::linear_plan<ASV_EPI_QKV_ROPE>(n_out, k, bn, sms); break;
        default: return asv::fail(ASV_ERR_INVALID, "linear_schedule: unknown epilogue");
    }
    if (splits != nullptr) *splits = pl.splits;
    if (stages != nullptr) *stages = pl.stages;
    if (smem_bytes != nullptr) *smem_bytes = asv::smem_for(bn, pl.stages, asv::kStageMargin[epilogue]);
    return ASV_OK;
}

int asv_linear_set_schedule(int32_t splits, int32_t stages) {
    if (splits < 0 || splits > asv::kMaxSplits || stages < 0) return asv::fail(ASV_ERR_INVALID, "linear_set_schedule");
    std::lock_guard<std::mutex> lk(asv::g_force_mu);
    asv::g_force = asv::LinPlan{splits, stages};
    return ASV_OK;
}

int asv_linear_trace(int32_t enable, uint64_t* out, int64_t cap, int64_t* n) {
    std::lock_guard<std::mutex> lk(asv::g_trace_mu);
    const size_t words = static_cast<size_t>(asv::kTrLaunches) * asv::kTrCtas * asv::kTrSlots;
    if (out != nullptr) {
        if (asv::g_trace == nullptr) return asv::fail(ASV_ERR_INVALID, "linear_trace: not enabled");
        const size_t m = static_cast<size_t>(asv::g_trace_seq) * asv::kTrCtas * asv::kTrSlots;
        if (static_cast<int64_t>(m) > cap) return asv::fail(ASV_ERR_INVALID, "linear_trace: out too small");
        cudaError_t e = cudaDeviceSynchronize();
        if (e == cudaSuccess) e = cudaMemcpy(out, asv::g_trace, m * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return asv::cuda_fail(e, "linear_trace copy");
        if (n != nullptr) *n = static_cast<int64_t>(m);
    }
    if (enable != 0) {  // (re)arm: the next kTrLaunches launches record
        if (asv::g_trace == nullptr) {
            const cudaError_t e = cudaMalloc(&asv::g_trace, words * 8);
            if (e != cudaSuccess) return asv::cuda_fail(e, "linear_trace");
        }
        cudaMemset(asv::g_trace, 0, words * 8);
        asv::g_trace_seq = 0;
        asv::g_trace_skipped = 0;
    } else if (out == nullptr && asv::g_trace != nullptr) {
        cudaFree(asv::g_trace);
        asv::g_trace = nullptr;
        asv::g_trace_seq = 0;
    }
    return ASV_OK;
}

int asv_rmsnorm(const void* h, const void* gamma, void* out, int32_t dim, int32_t batch, int32_t rows_out, float eps,
                int32_t pdl, void* stream) {
    if (h == nullptr || gamma == nullptr || out == nullptr || dim <= 0 || dim % 8 != 0 || dim > 256 * 8 * 4 ||
        batch < 1 || rows_out < batch)
        return asv::fail(ASV_ERR_INVALID, "rmsnorm: bad arguments");
    cudaError_t e =
        asv::rmsnorm_launch(h, gamma, out, dim, batch, rows_out, eps, pdl != 0, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return asv::cuda_fail(e, "rmsnorm launch");
    return ASV_OK;
}

}  // extern "C"
