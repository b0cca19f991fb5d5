// Persistent stream-K chain of decode linear layers on tcgen05 (SURVEY §8(f)
// rank 1: the MLP / projection term of iteration_latency, cost_model.hpp:60-63,
// 130-131).
//
// One launch runs up to four DEPENDENT GEMMs of a decode step — per layer
// O-proj (+residual) -> gate/up (+SiLU) -> down (+residual) -> next layer's QKV
// (+RoPE) — on a grid of exactly 2 CTAs per SM.  Why (measured): with
// one launch per GEMM every kernel boundary drains the HBM pipe (ramp, tail,
// epilogue), and tile counts that are not multiples of the SM count leave SMs
// idle (gate/up: 172 tiles on 148 SMs; O / down: 32 tiles x 8 K splits); the
// O projection reached 45% of the HBM peak.
//
// Work split (stream-K): a GEMM is tiles x kbs units (128 weight rows x 64 K);
// CTA c of G runs the contiguous unit range [c U / G, (c+1) U / G), so every CTA
// streams the same number of weight bytes in every phase.  A tile cut between
// CTAs is finished by its OWNER, the CTA holding the tile's first K block (for
// that CTA it is the last segment of the phase, so the other pieces — the first
// segment of the next CTAs — are normally ready): contributors store their fp32
// partial (one per CTA and phase) and bump the tile's arrival counter; the owner
// adds them in CTA order (deterministic), applies the fused epilogue and bumps
// the phase's done counter.  The producer of the next phase streams its first
// ring of weights (which depend on nothing) and waits for the done counter only
// before the activations, so the weight stream never stops at a GEMM boundary.
//
// Warp roles (256 threads): 0-3 epilogue (TMEM lanes 32w..32w+31), 4 TMA
// producer, 5 MMA issuer (+ TMEM owner), 6-7 fused-RMSNorm scales.  The
// accumulator is double-buffered in TMEM (two segments in flight) when
// 2 x 2 CTAs x columns fit the 512 TMEM columns (batch <= 128), else single.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <string>

#include "../../include/asv.h"
#include "asv_internal.h"
#include "tc_ptx.cuh"

struct asv_linear_chain_ws {
    int device;
    int sms;
    uint32_t* done;    // [kMaxPhases] monotonically increasing tile counters
    uint32_t* arrive;  // [kMaxPhases][kMaxTiles] contributor arrivals per tile, reset by the owner
    float* part;       // [2 * sms][128][256] contributor partials (row-major: row, batch column)
    float* pre;        // [2 * sms][128][256] owner's pre-reduced contributor sum
    uint32_t base[4];  // host: done[] value at the end of the previous launch
    unsigned long long* trace;  // optional timeline of the last launch (asv_linear_chain_ws_trace)
    int32_t trace_grid;         // grid of the last traced launch
    // cluster split-K chain (default kernel): per-phase CTA counters + exit counter, reset by the
    // last CTA of every launch (graph-safe); the launch grid that proved co-resident
    uint32_t* done2;            // [kMaxPhases + 1]
    int32_t grid2;              // CTAs (clusters x 8); 0 = not yet determined
    int32_t coop2;              // 1: cooperative launch (co-residency guaranteed by the driver)
    int32_t logged2;
};

namespace asv {
namespace {

using namespace tc;

constexpr int kMaxPhases = 4;
constexpr int kMaxTiles = 1024;          // n_out <= 131072 per phase
constexpr int kStagesMax = 8;
constexpr int kRingBudget = 92 * 1024;   // + 10 KiB epilogue / scale buffers: two CTAs per SM
constexpr int kThreads = 256;
constexpr int kProducerWarp = 4, kMmaWarp = 5, kHelperWarp0 = 6;
constexpr int kChunk = 16;               // accumulator columns per epilogue round
// timeline probe (asv_linear_chain_ws_trace): per CTA and phase, %globaltimer at
//   0 producer: activations' dependency satisfied   1 producer: last unit issued
//   2 epilogue: first segment accumulated            3 epilogue: last segment accumulated
//   4 epilogue: contributors' partials complete      5 epilogue: phase finished (done / arrive bumped)
constexpr int kTraceSlots = 6;

struct alignas(64) ChainMaps {
    CUtensorMap w[kMaxPhases];
    CUtensorMap x[kMaxPhases];
};

struct ChainPhase {
    int32_t tiles, kbs;  // kbs = k / 64 = units per tile
    int64_t units;
    int32_t epi;
    __nv_bfloat16* y;
    int32_t y_ld;
    const int32_t* positions;
    float rope_log2_theta;
    __nv_bfloat16 *q, *kk, *v;
    int32_t n_q_heads, n_kv_heads;
    float* ss_out;
    const float* ss_in;
    int32_t ss_parts, ss_ld;
    float ss_inv_dim, ss_eps;
    uint32_t done_target;  // done[phase] once every tile of this phase is finished in this launch
};

struct ChainParams {
    int32_t nphases, batch, bn, stages, nslots, ncols;
    uint32_t* done;
    uint32_t* arrive;
    float* part;
    float* pre;
    unsigned long long* trace;  // optional [grid][kMaxPhases][kTraceSlots] %globaltimer stamps
    ChainPhase ph[kMaxPhases];
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// spin until *p >= target (wrap-aware); a protocol bug traps instead of hanging the GPU
__device__ __forceinline__ void wait_count(const uint32_t* p, uint32_t target) {
    uint32_t n = 0;
    while (static_cast<int32_t>(ld_acquire(p) - target) < 0) {
        __nanosleep(40);
        if (++n > (1u << 27)) __trap();
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void stamp(const ChainParams& p, int c, int q, int k) {
    if (p.trace == nullptr) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(static_cast<int64_t>(c) * kMaxPhases + q) * kTraceSlots + k] = t;
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void helper_bar() { asm volatile("bar.sync 2, 64;" ::: "memory"); }

__device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t unit_begin(int64_t units, int c, int grid) {
    return units * c / grid;
}
// the CTA whose unit range holds unit u (every range is non-empty: grid <= units)
__device__ __forceinline__ int cta_of(int64_t u, int64_t units, int grid) {
    return static_cast<int>(((u + 1) * grid - 1) / units);
}

// One 16-column round of the owner's fused epilogue: chunk = [16][128] fp32 (column-major by
// batch column).  Thread t owns the row pair (r, r + 64), r = t & 63, of columns half*8..half*8+7,
// so SiLU gate/up and RoPE rotate-half partners are in one thread (same layout as decode_gemm.cu).
__device__ __forceinline__ void epilogue_round(const ChainPhase& P, int tile, int c0, int batch, const float* chunk,
                                               const float* rs) {
    const int r = threadIdx.x & 63, half = threadIdx.x >> 6;
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
        const int cc = half * 8 + j, b = c0 + cc;
        if (b >= batch) break;  // warp-uniform (half and j are)
        float lo = chunk[cc * kBM + r], hi = chunk[cc * kBM + r + 64];
        if (P.ss_in != nullptr) {
            lo *= rs[b];
            hi *= rs[b];
        }
        if (P.epi == ASV_EPI_STORE || P.epi == ASV_EPI_RESIDUAL) {
            __nv_bfloat16* dst = P.y + static_cast<int64_t>(b) * P.y_ld + tile * kBM + r;
            if (P.epi == ASV_EPI_RESIDUAL) {
                lo += __bfloat162float(__ldcg(dst));
                hi += __bfloat162float(__ldcg(dst + 64));
            }
            const __nv_bfloat16 blo = __float2bfloat16(lo), bhi = __float2bfloat16(hi);
            dst[0] = blo;
            dst[64] = bhi;
            if (P.ss_out != nullptr) {  // next linear's fused RMSNorm: sum of squares of the stored row
                const float fl = __bfloat162float(blo), fh = __bfloat162float(bhi);
                float sq = fl * fl + fh * fh;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
                if ((threadIdx.x & 31) == 0)
                    P.ss_out[static_cast<int64_t>(tile * 2 + ((threadIdx.x >> 5) & 1)) * P.ss_ld + b] = sq;
            }
        } else if (P.epi == ASV_EPI_SILU_MUL) {
            P.y[static_cast<int64_t>(b) * P.y_ld + tile * 64 + r] = __float2bfloat16(silu(lo) * hi);
        } else {  // ASV_EPI_QKV_ROPE: one head per tile, [q heads | k heads | v heads]
            const int head = tile;
            const bool is_q = head < P.n_q_heads, is_k = !is_q && head < P.n_q_heads + P.n_kv_heads;
            __nv_bfloat16* dst = is_q ? P.q : is_k ? P.kk : P.v;
            const int h = is_q ? head : is_k ? head - P.n_q_heads : head - P.n_q_heads - P.n_kv_heads;
            const int nh = is_q ? P.n_q_heads : P.n_kv_heads;
            if (is_q || is_k) {
                const float inv_freq = exp2f(-P.rope_log2_theta * (2.f * r / 128.f));
                float sn, cs;
                sincosf(static_cast<float>(__ldcg(P.positions + b)) * inv_freq, &sn, &cs);
                const float a0 = lo * cs - hi * sn, a1 = hi * cs + lo * sn;
                lo = a0;
                hi = a1;
            }
            __nv_bfloat16* o = dst + (static_cast<int64_t>(b) * nh + h) * 128;
            o[r] = __float2bfloat16(lo);
            o[r + 64] = __float2bfloat16(hi);
        }
    }
}

// smem: ring [stages][W 16 KiB | X bn*128 B] | chunk [16][128] fp32 | rs [2][256] fp32 |
//       full[8] empty[8] tfull[2] tempty[2] rsfull[2] | tmem base
__global__ void __launch_bounds__(kThreads, 2)
    linear_chain_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ ChainParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = kABytes + p.bn * 128;
    const int nst = p.stages;
    float* chunk = reinterpret_cast<float*>(smem + nst * stage_bytes);
    float* rsbuf = chunk + kChunk * kBM;
    uint64_t* bars = reinterpret_cast<uint64_t*>(rsbuf + 512);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStagesMax + 6);
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * kStagesMax, tfull0 = empty0 + 8 * kStagesMax,
                   tempty0 = tfull0 + 16, rsfull0 = tempty0 + 16;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull0 + 8 * i, 1);
            mbar_init(tempty0 + 8 * i, 4);   // the four epilogue warps
            mbar_init(rsfull0 + 8 * i, 2);   // the two scale warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int q = 0; q < p.nphases; ++q) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[q])) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.x[q])) : "memory");
        }
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(static_cast<uint32_t>(p.nslots * p.ncols))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_launch();  // the next kernel may run its prologue; it waits for our completion before our outputs

    if (warp == kProducerWarp) {
        if (lane == 0) {
            // ---- TMA producer: one ring across every phase and segment
            const uint64_t pw = policy_evict_first(), px = policy_evict_last();
            int s = 0;
            uint32_t ph = 0;
            for (int q = 0; q < p.nphases; ++q) {
                const ChainPhase& P = p.ph[q];
                const int64_t u0 = unit_begin(P.units, c, G), u1 = unit_begin(P.units, c + 1, G);
                const int pre = static_cast<int>(i64min(nst, u1 - u0));
                const int s_pre = s;
                // weights never depend on an earlier phase or kernel: the first ring of them goes now
                for (int i = 0; i < pre; ++i) {
                    const int64_t u = u0 + i;
                    mbar_wait(empty0 + 8 * s, ph ^ 1);
                    mbar_expect_tx(full0 + 8 * s, static_cast<uint32_t>(stage_bytes));
                    tma_load_2d(smem_u32(smem + s * stage_bytes), &maps.w[q], static_cast<int32_t>(u % P.kbs) * kBK,
                                static_cast<int32_t>(u / P.kbs) * kBM, full0 + 8 * s, pw);
                    if (++s == nst) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                // the activations are the previous phase's (or kernel's) output
                if (q == 0) {
                    grid_dep_wait();
                } else {
                    wait_count(p.done + (q - 1), p.ph[q - 1].done_target);
                }
                stamp(p, c, q, 0);
                fence_proxy_async();
                for (int i = 0, st = s_pre; i < pre; ++i) {
                    tma_load_2d(smem_u32(smem + st * stage_bytes) + kABytes, &maps.x[q],
                                static_cast<int32_t>((u0 + i) % P.kbs) * kBK, 0, full0 + 8 * st, px);
                    if (++st == nst) st = 0;
                }
                for (int64_t u = u0 + pre; u < u1; ++u) {
                    mbar_wait(empty0 + 8 * s, ph ^ 1);
                    const uint32_t a = smem_u32(smem + s * stage_bytes);
                    const int32_t kx = static_cast<int32_t>(u % P.kbs) * kBK;
                    mbar_expect_tx(full0 + 8 * s, static_cast<uint32_t>(stage_bytes));
                    tma_load_2d(a, &maps.w[q], kx, static_cast<int32_t>(u / P.kbs) * kBM, full0 + 8 * s, pw);
                    tma_load_2d(a + kABytes, &maps.x[q], kx, 0, full0 + 8 * s, px);
                    if (++s == nst) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                stamp(p, c, q, 1);
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            // ---- MMA issuer: per segment (the units of one tile in this CTA's range) one accumulator
            const uint32_t idesc = umma_idesc(static_cast<uint32_t>(p.bn));
            int s = 0, seg = 0;
            uint32_t ph = 0;
            for (int q = 0; q < p.nphases; ++q) {
                const ChainPhase& P = p.ph[q];
                const int64_t u0 = unit_begin(P.units, c, G), u1 = unit_begin(P.units, c + 1, G);
                for (int64_t u = u0; u < u1; ++seg) {
                    const int64_t seg0 = u, seg1 = i64min(u1, (u / P.kbs + 1) * P.kbs);
                    const int slot = p.nslots == 2 ? (seg & 1) : 0;
                    const int use = p.nslots == 2 ? (seg >> 1) : seg;
                    mbar_wait(tempty0 + 8 * slot, static_cast<uint32_t>(use & 1) ^ 1u);
                    tc_fence_after();
                    const uint32_t dacc = tmem + static_cast<uint32_t>(slot * p.ncols);
                    for (; u < seg1; ++u) {
                        mbar_wait(full0 + 8 * s, ph);
                        tc_fence_after();
                        const uint32_t a = smem_u32(smem + s * stage_bytes);
                        const uint64_t ad = umma_desc_sw128(a), bd = umma_desc_sw128(a + kABytes);
#pragma unroll
                        for (int kk = 0; kk < kBK / kUmmaK; ++kk) {
                            umma_f16(dacc, ad + 2 * kk, bd + 2 * kk, idesc, (u > seg0 || kk > 0) ? 1u : 0u);
                        }
                        umma_commit(empty0 + 8 * s);
                        if (++s == nst) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                    umma_commit(tfull0 + 8 * slot);  // segment accumulator complete
                }
            }
        }
    } else if (warp >= kHelperWarp0) {
        // ---- fused RMSNorm: 1/rms of every batch column of a phase whose input is the raw residual
        // stream, from the producing phase's partial sums of squares (fixed order: deterministic)
        const int t = static_cast<int>(threadIdx.x) - kHelperWarp0 * 32;
        for (int q = 0; q < p.nphases; ++q) {
            const ChainPhase& P = p.ph[q];
            if (q == 0) {
                grid_dep_wait();
            } else {
                if (t == 0) wait_count(p.done + (q - 1), p.ph[q - 1].done_target);
                helper_bar();
            }
            if (P.ss_in != nullptr) {
                for (int b = t; b < p.batch; b += 64) {
                    float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                    int i = 0;
                    for (; i + 8 <= P.ss_parts; i += 8) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc8[j] += __ldcg(P.ss_in + static_cast<int64_t>(i + j) * P.ss_ld + b);
                    }
                    for (; i < P.ss_parts; ++i) acc8[0] += __ldcg(P.ss_in + static_cast<int64_t>(i) * P.ss_ld + b);
                    const float ssum =
                        ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
                    rsbuf[(q & 1) * 256 + b] = rsqrtf(ssum * P.ss_inv_dim + P.ss_eps);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(rsfull0 + 8 * (q & 1));
        }
    } else {
        // ---- epilogue warps 0-3: thread = accumulator row (TMEM lane)
        grid_dep_wait();  // residual / outputs may belong to the previous kernel
        const int row = threadIdx.x;
        const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
        int seg = 0;
        for (int q = 0; q < p.nphases; ++q) {
            const ChainPhase& P = p.ph[q];
            const int64_t u0 = unit_begin(P.units, c, G), u1 = unit_begin(P.units, c + 1, G);
            for (int64_t u = u0; u < u1; ++seg) {
                const int64_t t = u / P.kbs, tile0 = t * P.kbs, seg1 = i64min(u1, tile0 + P.kbs);
                const bool owner = u == tile0;
                const int slot = p.nslots == 2 ? (seg & 1) : 0;
                const int use = p.nslots == 2 ? (seg >> 1) : seg;
                const int ncol = (p.batch + kChunk - 1) / kChunk * kChunk;
                uint32_t* arrive = p.arrive + q * kMaxTiles + t;
                const int last = owner ? cta_of(tile0 + P.kbs - 1, P.units, G) : c;  // contributors c+1..last
                float* pre = p.pre + static_cast<int64_t>(c) * kBM * 256 + row * 256;
                if (owner && last > c) {
                    // while the MMA still runs this segment: sum the contributors' partials (their first
                    // segments, ready early) in CTA order, 128-bit loads, two pieces in flight
                    if (threadIdx.x == 0) {
                        wait_count(arrive, static_cast<uint32_t>(last - c));
                        stamp(p, c, q, 4);
                    }
                    epi_bar();
                    for (int c0 = 0; c0 < ncol; c0 += kChunk) {
                        float4 acc[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
                        for (int pc = c + 1; pc <= last; ++pc) {
                            const float4* src = reinterpret_cast<const float4*>(
                                p.part + (static_cast<int64_t>(pc) * kBM + row) * 256 + c0);
                            float4 x[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) x[k] = __ldcg(src + k);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                acc[k].x += x[k].x;
                                acc[k].y += x[k].y;
                                acc[k].z += x[k].z;
                                acc[k].w += x[k].w;
                            }
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k) reinterpret_cast<float4*>(pre + c0)[k] = acc[k];
                    }
                }
                mbar_wait(tfull0 + 8 * slot, static_cast<uint32_t>(use & 1));
                tc_fence_after();
                if (threadIdx.x == 0) stamp(p, c, q, u == u0 ? 2 : 3);
                const uint32_t taddr = tmem + static_cast<uint32_t>(slot * p.ncols) + lane_off;
                if (!owner) {
                    // contributor: this CTA's first segment of the phase -> fp32 partial, then arrive
                    float4* dst = reinterpret_cast<float4*>(p.part + (static_cast<int64_t>(c) * kBM + row) * 256);
                    for (int c0 = 0; c0 < ncol; c0 += kChunk) {
                        float v[kChunk];
                        tmem_ld16(taddr + static_cast<uint32_t>(c0), v);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            dst[c0 / 4 + k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty0 + 8 * slot);
                    __threadfence();
                    epi_bar();
                    if (threadIdx.x == 0) {
                        red_release_add(arrive, 1u);
                        stamp(p, c, q, 5);
                    }
                } else {
                    // the residual rows / positions this epilogue reads were written by earlier phases
                    if (threadIdx.x == 0 && q > 0) wait_count(p.done + (q - 1), p.ph[q - 1].done_target);
                    if (P.ss_in != nullptr) mbar_wait(rsfull0 + 8 * (q & 1), static_cast<uint32_t>((q >> 1) & 1));
                    epi_bar();
                    const float* rs = rsbuf + (q & 1) * 256;
                    for (int c0 = 0; c0 < ncol; c0 += kChunk) {
                        float v[kChunk];
                        tmem_ld16(taddr + static_cast<uint32_t>(c0), v);
                        if (c0 + kChunk >= ncol) {  // accumulator fully read: the MMA may reuse the slot
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(tempty0 + 8 * slot);
                        }
                        if (last > c) {  // own piece + the contributors' sum (this thread wrote it)
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float4 x = reinterpret_cast<const float4*>(pre + c0)[k];
                                v[4 * k] += x.x;
                                v[4 * k + 1] += x.y;
                                v[4 * k + 2] += x.z;
                                v[4 * k + 3] += x.w;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < kChunk; ++i) chunk[i * kBM + row] = v[i];
                        epi_bar();
                        epilogue_round(P, static_cast<int>(t), c0, p.batch, chunk, rs);
                        epi_bar();
                    }
                    if (threadIdx.x == 0 && last > c) *arrive = 0u;  // next use: the next launch
                    fence_proxy_async();  // outputs are read by the next phase's TMA loads
                    __threadfence();
                    epi_bar();
                    if (threadIdx.x == 0) {
                        red_release_add(p.done + q, 1u);
                        stamp(p, c, q, 5);
                    }
                }
                u = seg1;
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(static_cast<uint32_t>(p.nslots * p.ncols))
                     : "memory");
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn chain_encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<EncodeFn>(ptr);
        }
    });
    return fn;
}

bool chain_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeFn fn = chain_encode_fn();
    if (fn == nullptr) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int chain_stages(int bn) {
    const int st = kRingBudget / (kABytes + bn * 128);
    return st < 2 ? 2 : st > kStagesMax ? kStagesMax : st;
}
int chain_smem(int bn) {
    return 1024 + chain_stages(bn) * (kABytes + bn * 128) + kChunk * kBM * 4 + 512 * 4 + (2 * kStagesMax + 6) * 8 + 16;
}


// ============================================================================
// Cluster split-K chain (the default asv_linear_chain kernel).
//
// The stream-K kernel above reduces tiles cut between CTAs through global memory, and that
// reduction sits on every phase boundary while the weight ring keeps the memory system saturated
// (measured 0.6x the per-GEMM path, profiles/chain_trace_r02g.txt).  This kernel keeps the
// per-GEMM kernel's reduction — the 8 K splits of a tile are one thread-block cluster and reduce
// through distributed shared memory — and makes only the phase handoff global:
//   * persistent grid of G clusters x 8 CTAs (co-resident: cooperative launch), cluster c takes
//     tiles c, c + G, ... of every phase; CTA rank r streams K blocks [r*per, (r+1)*per) of each;
//   * warp 4 (TMA producer) streams one ring across tiles and phases: the weights of phase q are
//     issued as soon as ring slots free up, the activations of phase q only once every CTA has
//     finished phase q-1 (per-phase counter, release/acquire) — the ring runs ahead across the
//     boundary by at most its own size;
//   * warp 5 issues tcgen05.mma into a double-buffered TMEM accumulator (the next tile's MMAs
//     overlap the previous tile's epilogue);
//   * warps 0-3 (epilogue): 16 accumulator columns at a time go to a double-buffered smem chunk,
//     one cluster-scope mbarrier round (remote arrives) publishes it, and every CTA reduces 2 of the
//     16 columns from all 8 CTAs' chunks (DSMEM) and applies the fused epilogue (same math and
//     summation order as decode_gemm.cu: results are bit-identical to the per-GEMM launches);
//   * warps 6-7: fused-RMSNorm scales of a phase from the previous phase's partial sums.
// ============================================================================
constexpr int kS2 = 8;            // K splits per tile = cluster size
constexpr int kChunk2 = 16;       // accumulator columns per cluster reduction round
constexpr int kRing2Budget = 92 * 1024;

struct Chain2Params {
    int32_t nphases, batch, bn, stages, nslots, ncols;
    uint32_t* done;               // [kMaxPhases] CTAs finished per phase, [kMaxPhases] = exit counter
    unsigned long long* trace;    // optional [grid][kMaxPhases][kTraceSlots]
    ChainPhase ph[kMaxPhases];
};

__device__ __forceinline__ void stamp2(const Chain2Params& p, int q, int k) {
    if (p.trace == nullptr) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(static_cast<int64_t>(blockIdx.x) * kMaxPhases + q) * kTraceSlots + k] = t;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// the activations of phase q may be read once every CTA finished phase q-1 (q = 0: the previous kernel)
__device__ __forceinline__ bool dep_ready2(const Chain2Params& p, int q) {
    return q == 0 || static_cast<int32_t>(ld_acquire(p.done + (q - 1)) - gridDim.x) >= 0;
}
__device__ __forceinline__ void dep_wait2(const Chain2Params& p, int q) {
    if (q == 0) {
        grid_dep_wait();
    } else {
        wait_count(p.done + (q - 1), gridDim.x);
    }
}

// one (batch column, row pair) of a phase's fused epilogue: same math as decode_gemm.cu
__device__ __forceinline__ void epilogue2(const ChainPhase& P, int tile, int b, int r, float lo, float hi,
                                          float scale, bool do_ss) {
    lo *= scale;
    hi *= scale;
    if (P.epi == ASV_EPI_STORE || P.epi == ASV_EPI_RESIDUAL) {
        __nv_bfloat16* dst = P.y + static_cast<int64_t>(b) * P.y_ld + tile * kBM + r;
        if (P.epi == ASV_EPI_RESIDUAL) {
            lo += __bfloat162float(__ldcg(dst));
            hi += __bfloat162float(__ldcg(dst + 64));
        }
        const __nv_bfloat16 blo = __float2bfloat16(lo), bhi = __float2bfloat16(hi);
        dst[0] = blo;
        dst[64] = bhi;
        if (do_ss) {  // next linear's fused RMSNorm: sum of squares of the stored row (warp-uniform branch)
            const float fl = __bfloat162float(blo), fh = __bfloat162float(bhi);
            float sq = fl * fl + fh * fh;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
            if ((threadIdx.x & 31) == 0)
                P.ss_out[static_cast<int64_t>(tile * 2 + ((threadIdx.x >> 5) & 1)) * P.ss_ld + b] = sq;
        }
    } else if (P.epi == ASV_EPI_SILU_MUL) {
        P.y[static_cast<int64_t>(b) * P.y_ld + tile * 64 + r] = __float2bfloat16(silu(lo) * hi);
    } else {  // ASV_EPI_QKV_ROPE
        const int head = tile;
        const bool is_q = head < P.n_q_heads, is_k = !is_q && head < P.n_q_heads + P.n_kv_heads;
        __nv_bfloat16* dst = is_q ? P.q : is_k ? P.kk : P.v;
        const int h = is_q ? head : is_k ? head - P.n_q_heads : head - P.n_q_heads - P.n_kv_heads;
        const int nh = is_q ? P.n_q_heads : P.n_kv_heads;
        if (is_q || is_k) {
            const float inv_freq = exp2f(-P.rope_log2_theta * (2.f * r / 128.f));
            float sn, cs;
            sincosf(static_cast<float>(__ldcg(P.positions + b)) * inv_freq, &sn, &cs);
            const float a0 = lo * cs - hi * sn, a1 = hi * cs + lo * sn;
            lo = a0;
            hi = a1;
        }
        __nv_bfloat16* o = dst + (static_cast<int64_t>(b) * nh + h) * 128;
        o[r] = __float2bfloat16(lo);
        o[r + 64] = __float2bfloat16(hi);
    }
}

// smem: ring [stages][W 16 KiB | X bn*128 B] | chunk [2][16][128] fp32 | rs [2][256] fp32 |
//       full[8] empty[8] tfull[2] tempty[2] rsfull[2] cready[2] | tmem base
__global__ void __launch_bounds__(kThreads, 2)
    linear_chain2_kernel(const __grid_constant__ ChainMaps maps, const __grid_constant__ Chain2Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = kABytes + p.bn * 128;
    const int nst = p.stages;
    float* chunk = reinterpret_cast<float*>(smem + nst * stage_bytes);
    float* rsbuf = chunk + 2 * kChunk2 * kBM;
    uint64_t* bars = reinterpret_cast<uint64_t*>(rsbuf + 512);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStagesMax + 12);
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * kStagesMax, tfull0 = empty0 + 8 * kStagesMax,
                   tempty0 = tfull0 + 32, rsfull0 = tempty0 + 32, cready0 = rsfull0 + 16;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x / kS2, cid = blockIdx.x / kS2;
    const int rank = static_cast<int>(cluster_rank());

    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(tfull0 + 8 * i, 1);
            mbar_init(tempty0 + 8 * i, 4);    // the four epilogue warps
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(rsfull0 + 8 * i, 2);    // the two scale warps
            mbar_init(cready0 + 8 * i, kS2);  // one remote arrive per cluster CTA and chunk
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int q = 0; q < p.nphases; ++q) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[q])) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.x[q])) : "memory");
        }
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(static_cast<uint32_t>(p.nslots * p.ncols))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync_all();  // every CTA's chunk barriers exist before any remote arrive
    const uint32_t tmem = *tmem_slot;
    // (no early griddepcontrol.launch_dependents: the next kernel's CTAs must not take SM room
    // before every CTA of this grid is resident — the phase handoff waits on all of them)

    if (warp == kProducerWarp) {
        if (lane == 0) {
            const uint64_t pw = policy_evict_first(), px = policy_evict_last();
            int s = 0;
            uint32_t ph = 0;
            int pend_slot[kStagesMax], pend_kb[kStagesMax];
            bool prev_grid_done = false;  // the counters belong to this launch only after griddepcontrol.wait
            for (int q = 0; q < p.nphases; ++q) {
                const ChainPhase& P = p.ph[q];
                const int per = (P.kbs + kS2 - 1) / kS2;
                const int kb0 = rank * per, kb1 = min(kb0 + per, P.kbs);
                bool dep = false;
                int npend = 0;
                if (q > 0 && !prev_grid_done) {  // (a CTA without phase-0 tiles has not waited yet)
                    grid_dep_wait();
                    prev_grid_done = true;
                }
                auto flush = [&]() {
                    dep_wait2(p, q);
                    prev_grid_done = true;
                    fence_proxy_async();
                    stamp2(p, q, 0);
                    for (int i = 0; i < npend; ++i)
                        tma_load_2d(smem_u32(smem + pend_slot[i] * stage_bytes) + kABytes, &maps.x[q],
                                    pend_kb[i] * kBK, 0, full0 + 8 * pend_slot[i], px);
                    npend = 0;
                    dep = true;
                };
                for (int t = cid; t < P.tiles; t += G) {
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(empty0 + 8 * s, ph ^ 1);
                        if (q > 0 && !dep && dep_ready2(p, q)) flush();
                        const uint32_t a = smem_u32(smem + s * stage_bytes);
                        mbar_expect_tx(full0 + 8 * s, static_cast<uint32_t>(stage_bytes));
                        tma_load_2d(a, &maps.w[q], kb * kBK, t * kBM, full0 + 8 * s, pw);
                        if (dep) {
                            tma_load_2d(a + kABytes, &maps.x[q], kb * kBK, 0, full0 + 8 * s, px);
                        } else {
                            pend_slot[npend] = s;
                            pend_kb[npend] = kb;
                            if (++npend == nst) flush();  // the ring holds nothing but weights: wait
                        }
                        if (++s == nst) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
                if (!dep && npend > 0) flush();
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            const uint32_t idesc = umma_idesc(static_cast<uint32_t>(p.bn));
            int s = 0, seg = 0;
            uint32_t ph = 0;
            for (int q = 0; q < p.nphases; ++q) {
                const ChainPhase& P = p.ph[q];
                const int per = (P.kbs + kS2 - 1) / kS2;
                const int kb0 = rank * per, kb1 = min(kb0 + per, P.kbs);
                for (int t = cid; t < P.tiles; t += G, ++seg) {
                    const int slot = seg % p.nslots;
                    const int use = seg / p.nslots;
                    mbar_wait(tempty0 + 8 * slot, static_cast<uint32_t>(use & 1) ^ 1u);
                    tc_fence_after();
                    const uint32_t dacc = tmem + static_cast<uint32_t>(slot * p.ncols);
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(full0 + 8 * s, ph);
                        tc_fence_after();
                        const uint32_t a = smem_u32(smem + s * stage_bytes);
                        const uint64_t ad = umma_desc_sw128(a), bd = umma_desc_sw128(a + kABytes);
#pragma unroll
                        for (int kk = 0; kk < kBK / kUmmaK; ++kk)
                            umma_f16(dacc, ad + 2 * kk, bd + 2 * kk, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
                        umma_commit(empty0 + 8 * s);
                        if (++s == nst) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                    umma_commit(tfull0 + 8 * slot);  // (an empty split commits at once: its epilogue reads zeros)
                }
            }
        }
    } else if (warp >= kHelperWarp0) {
        const int t = static_cast<int>(threadIdx.x) - kHelperWarp0 * 32;
        grid_dep_wait();  // the phase counters belong to this launch only after the previous grid is done
        for (int q = 0; q < p.nphases; ++q) {
            const ChainPhase& P = p.ph[q];
            if (P.ss_in == nullptr) continue;
            if (t == 0) dep_wait2(p, q);
            helper_bar();
            for (int b = t; b < p.batch; b += 64) {
                float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                int i = 0;
                for (; i + 8 <= P.ss_parts; i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc8[j] += __ldcg(P.ss_in + static_cast<int64_t>(i + j) * P.ss_ld + b);
                }
                for (; i < P.ss_parts; ++i) acc8[0] += __ldcg(P.ss_in + static_cast<int64_t>(i) * P.ss_ld + b);
                const float ssum =
                    ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
                rsbuf[(q & 1) * 256 + b] = rsqrtf(ssum * P.ss_inv_dim + P.ss_eps);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(rsfull0 + 8 * (q & 1));
        }
    } else {
        // ---- epilogue warps 0-3: thread = accumulator row (TMEM lane)
        grid_dep_wait();  // residual / positions / outputs may belong to the previous kernel
        const int row = threadIdx.x;
        const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
        const int ncol = (p.batch + kChunk2 - 1) / kChunk2 * kChunk2;
        const int r = threadIdx.x & 63, half = threadIdx.x >> 6;
        uint32_t peer_chunk[kS2];
#pragma unroll
        for (int j = 0; j < kS2; ++j) peer_chunk[j] = mapa_u32(smem_u32(chunk), static_cast<uint32_t>(j));
        uint32_t cc = 0;  // chunk rounds so far (double-buffered chunk, parity of cready)
        int seg = 0;
        int rs_uses[2] = {0, 0};
        for (int q = 0; q < p.nphases; ++q) {
            const ChainPhase& P = p.ph[q];
            const int per = (P.kbs + kS2 - 1) / kS2;
            const bool empty_split = rank * per >= P.kbs;
            if (q > 0) {
                // the residual rows / positions this phase reads were written by earlier phases
                if (threadIdx.x == 0) wait_count(p.done + (q - 1), gridDim.x);
                epi_bar();
            }
            const float* rs = nullptr;
            if (P.ss_in != nullptr) {
                mbar_wait(rsfull0 + 8 * (q & 1), static_cast<uint32_t>(rs_uses[q & 1]++ & 1));
                rs = rsbuf + (q & 1) * 256;
            }
            const bool do_ss = P.ss_out != nullptr;
            for (int t = cid; t < P.tiles; t += G, ++seg) {
                const int slot = seg % p.nslots;
                const int use = seg / p.nslots;
                mbar_wait(tfull0 + 8 * slot, static_cast<uint32_t>(use & 1));
                tc_fence_after();
                if (threadIdx.x == 0) stamp2(p, q, t == cid ? 1 : 2);
                const uint32_t taddr = tmem + static_cast<uint32_t>(slot * p.ncols) + lane_off;
                for (int c0 = 0; c0 < ncol; c0 += kChunk2, ++cc) {
                    float v[kChunk2];
                    if (!empty_split) {
                        tmem_ld16(taddr + static_cast<uint32_t>(c0), v);
                    } else {
#pragma unroll
                        for (int i = 0; i < kChunk2; ++i) v[i] = 0.f;
                    }
                    if (c0 + kChunk2 >= ncol) {  // accumulator fully read: the MMA may reuse the slot
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(tempty0 + 8 * slot);
                    }
                    float* buf = chunk + (cc & 1) * kChunk2 * kBM;
#pragma unroll
                    for (int i = 0; i < kChunk2; ++i) buf[i * kBM + row] = v[i];
                    epi_bar();
                    if (threadIdx.x == 0) {
#pragma unroll
                        for (int j = 0; j < kS2; ++j) mbar_arrive_remote(mapa_u32(cready0 + 8 * (cc & 1), j));
                    }
                    mbar_wait_cluster(cready0 + 8 * (cc & 1), (cc >> 1) & 1);
                    // this CTA's 2 of the 16 columns, summed over the 8 splits in split order
                    const int cl = 2 * rank + half, b = c0 + cl;
                    if (b < p.batch) {
                        const uint32_t off = static_cast<uint32_t>(((cc & 1) * kChunk2 * kBM + cl * kBM + r) * 4);
                        float x0[kS2], x1[kS2];
#pragma unroll
                        for (int j = 0; j < kS2; ++j) {
                            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x0[j]) : "r"(peer_chunk[j] + off));
                            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x1[j]) : "r"(peer_chunk[j] + off + 256));
                        }
                        float lo = 0.f, hi = 0.f;
#pragma unroll
                        for (int j = 0; j < kS2; ++j) {
                            lo += x0[j];
                            hi += x1[j];
                        }
                        epilogue2(P, t, b, r, lo, hi, rs != nullptr ? rs[b] : 1.f, do_ss);
                    }
                }
                if (threadIdx.x == 0 && t + G >= P.tiles) stamp2(p, q, 3);
            }
            // this CTA's part of phase q is written: publish it (TMA readers: async proxy)
            fence_proxy_async();
            __threadfence();
            epi_bar();
            if (threadIdx.x == 0) {
                red_release_add(p.done + q, 1u);
                stamp2(p, q, 4);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync_all();  // no CTA leaves while a peer may still read its chunk buffers
    grid_dep_launch();   // every CTA of this grid is past its last handoff wait
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(static_cast<uint32_t>(p.nslots * p.ncols))
                     : "memory");
    }
    if (threadIdx.x == 0) {
        // the last CTA out resets the counters for the next launch (which reads them only after its
        // griddepcontrol.wait, i.e. after this grid completed): graph replays see the same state
        __threadfence();
        const uint32_t prev = atomicAdd(p.done + kMaxPhases, 1u);
        if (prev == gridDim.x - 1) {
            for (int q = 0; q < kMaxPhases; ++q) p.done[q] = 0u;
            p.done[kMaxPhases] = 0u;
            __threadfence();
        }
    }
}


// Co-residency probe for the persistent chain: the same launch shape (cluster of 8, 256 threads,
// the chain's shared memory and TMEM columns) with every CTA counting itself in and spinning until
// all are in or ~20 ms pass.  The driver's cooperative limit for this kernel is ~1 CTA per SM
// (15 clusters), far below what actually co-resides, so the grid is measured instead.
__global__ void __launch_bounds__(kThreads, 2) chain2_probe_kernel(uint32_t* counter, uint32_t* ok, uint32_t ncols) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    smem_raw[threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(counter, 1u);
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        bool all = false;
        do {
            all = ld_acquire(counter) >= gridDim.x;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        } while (!all && t - t0 < 20000000ull);
        if (!all) atomicExch(ok, 0u);
    }
    __syncthreads();
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(ncols) : "memory");
    }
}

int chain2_stages(int bn) {
    const int st = kRing2Budget / (kABytes + bn * 128);
    return st < 2 ? 2 : st > kStagesMax ? kStagesMax : st;
}
int chain2_smem(int bn) {
    return 1024 + chain2_stages(bn) * (kABytes + bn * 128) + 2 * kChunk2 * kBM * 4 + 512 * 4 +
           (2 * kStagesMax + 12) * 8 + 16;
}


// Launch of the cluster split-K chain.  Every CTA must be co-resident (the phase handoff waits on
// all of them): the grid is the largest cluster count (<= 2 CTAs per SM) that the co-residency probe
// saw resident together on this device, measured once per workspace with the largest shared memory
// any batch uses; the spin waits trap (kernel error, not a hang) if that ever fails to hold.
int chain2_grid(asv_linear_chain_ws* ws, cudaStream_t st) {
    if (ws->grid2 > 0) return ws->grid2;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return -1;  // the probe synchronises: run one chain launch before capturing a graph
    uint32_t* dev = nullptr;
    if (cudaMalloc(&dev, 8) != cudaSuccess) return 0;
    cudaFuncSetAttribute(chain2_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chain2_smem(16));
    int grid = 0;
    for (int g = (2 * ws->sms) / kS2 * kS2; g >= kS2; g -= kS2) {
        const uint32_t init[2] = {0u, 1u};
        cudaMemcpy(dev, init, 8, cudaMemcpyHostToDevice);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = chain2_smem(16);  // the largest: 5 stages at bn 16
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kS2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const bool log = getenv("ASV_LINEAR_PLAN_LOG") != nullptr;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, chain2_probe_kernel, dev, dev + 1, 64u);
        if (le != cudaSuccess) {
            if (log) fprintf(stderr, "  chain probe grid %d: launch %s\n", g, cudaGetErrorString(le));
            cudaGetLastError();
            continue;
        }
        uint32_t res[2] = {0u, 0u};
        cudaError_t ce = cudaMemcpyAsync(res, dev, 8, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (log) fprintf(stderr, "  chain probe grid %d: %s counter %u ok %u\n", g, cudaGetErrorString(ce), res[0], res[1]);
        if (ce != cudaSuccess) break;
        if (res[1] == 1u && res[0] == static_cast<uint32_t>(g)) {
            grid = g;
            break;
        }
    }
    cudaFree(dev);
    ws->grid2 = grid;
    if (getenv("ASV_LINEAR_PLAN_LOG") != nullptr)
        fprintf(stderr, "asv_linear_chain: co-resident grid %d CTAs (%d clusters of %d)\n", grid, grid / kS2, kS2);
    return grid;
}

int chain2_launch(const ChainParams& p1, const ChainMaps& maps, bool pdl, asv_linear_chain_ws* ws, cudaStream_t st) {
    Chain2Params p{};
    p.nphases = p1.nphases;
    p.batch = p1.batch;
    p.bn = p1.bn;
    p.stages = chain2_stages(p1.bn);
    p.ncols = p1.ncols;
    // TMEM accumulator slots: as many as 2 CTAs per SM can hold (<= 4): the MMA runs up to
    // nslots - 1 tiles ahead of the epilogue
    {
        static const int want = [] {
            const char* e = getenv("ASV_CHAIN_SLOTS");
            return e != nullptr ? atoi(e) : 4;
        }();
        int ns = 256 / p1.ncols;
        if (ns > want) ns = want;
        if (ns > 4) ns = 4;
        p.nslots = ns < 1 ? 1 : ns;
    }
    p.done = ws->done2;
    p.trace = ws->trace;
    for (int q = 0; q < p1.nphases; ++q) p.ph[q] = p1.ph[q];
    static bool configured = false;
    if (!configured) {
        const cudaError_t e = cudaFuncSetAttribute(linear_chain2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   227 * 1024);
        if (e != cudaSuccess) return cuda_fail(e, "linear_chain: smem attribute");
        configured = true;
    }
    const int grid = chain2_grid(ws, st);
    if (grid < 0)
        return fail(ASV_ERR_INVALID, "linear_chain: the first launch on a workspace measures the co-resident grid "
                                     "and cannot be stream-captured");
    if (grid == 0) return fail(ASV_ERR_CUDA, "linear_chain: no co-resident cluster grid");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = chain2_smem(p.bn);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = kS2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    ws->trace_grid = grid;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, linear_chain2_kernel, maps, p);
    if (e != cudaSuccess) return cuda_fail(e, "linear_chain launch");
    return ASV_OK;
}

int chain_run(const asv_linear_args* ph, int n, asv_linear_chain_ws* ws, cudaStream_t st) {
    if (ph == nullptr || ws == nullptr || n < 1 || n > kMaxPhases)
        return fail(ASV_ERR_INVALID, "linear_chain: need 1-4 phases and a workspace");
    const int batch = ph[0].batch;
    if (batch < 1 || batch > 256) return fail(ASV_ERR_INVALID, "linear_chain: batch must be in [1, 256]");
    const int bn = (batch + 15) / 16 * 16;
    ChainMaps maps;
    ChainParams p{};
    p.nphases = n;
    p.batch = batch;
    p.bn = bn;
    p.stages = chain_stages(bn);
    p.ncols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
    p.nslots = p.ncols <= 128 ? 2 : 1;  // 2 CTAs/SM x slots x columns <= 512 TMEM columns
    p.done = ws->done;
    p.arrive = ws->arrive;
    p.part = ws->part;
    p.pre = ws->pre;
    p.trace = ws->trace;
    int64_t min_units = INT64_MAX;
    for (int q = 0; q < n; ++q) {
        const asv_linear_args& a = ph[q];
        if (a.w == nullptr || a.x == nullptr) return fail(ASV_ERR_INVALID, "linear_chain: null pointer");
        if (a.batch != batch) return fail(ASV_ERR_INVALID, "linear_chain: every phase must have the same batch");
        if (a.n_out <= 0 || a.n_out % kBM != 0 || a.n_out / kBM > kMaxTiles)
            return fail(ASV_ERR_INVALID, "linear_chain: n_out must be a multiple of 128 (<= 131072)");
        if (a.k <= 0 || a.k % kBK != 0) return fail(ASV_ERR_INVALID, "linear_chain: k must be a multiple of 64");
        if (a.x_rows < bn) return fail(ASV_ERR_INVALID, "linear_chain: x must have >= batch rounded up to 16 rows");
        if (a.epilogue == ASV_EPI_QKV_ROPE) {
            if (a.positions == nullptr || a.q == nullptr || a.k_out == nullptr || a.v_out == nullptr ||
                a.n_out != 128 * (a.n_q_heads + 2 * a.n_kv_heads))
                return fail(ASV_ERR_INVALID, "linear_chain: bad QKV/RoPE arguments");
        } else if (a.epilogue < ASV_EPI_STORE || a.epilogue > ASV_EPI_SILU_MUL || a.y == nullptr) {
            return fail(ASV_ERR_INVALID, "linear_chain: bad epilogue or null y");
        }
        if (a.ss_out != nullptr && (a.epilogue != ASV_EPI_RESIDUAL || a.ss_ld < batch))
            return fail(ASV_ERR_INVALID, "linear_chain: ss_out needs the RESIDUAL epilogue and ss_ld >= batch");
        if (a.ss_in != nullptr && (a.ss_parts < 1 || a.ss_ld < batch || a.ss_dim < 1))
            return fail(ASV_ERR_INVALID, "linear_chain: bad fused-RMSNorm arguments");
        if (!chain_map(&maps.w[q], a.w, static_cast<uint64_t>(a.n_out), static_cast<uint64_t>(a.k), kBM) ||
            !chain_map(&maps.x[q], a.x, static_cast<uint64_t>(a.x_rows), static_cast<uint64_t>(a.k),
                       static_cast<uint32_t>(bn)))
            return fail(ASV_ERR_CUDA, "linear_chain: cuTensorMapEncodeTiled failed");
        ChainPhase& P = p.ph[q];
        P.tiles = a.n_out / kBM;
        P.kbs = a.k / kBK;
        P.units = static_cast<int64_t>(P.tiles) * P.kbs;
        P.epi = a.epilogue;
        P.y = static_cast<__nv_bfloat16*>(a.y);
        P.y_ld = a.y_ld;
        P.positions = a.positions;
        P.rope_log2_theta = log2f(a.rope_theta > 0.f ? a.rope_theta : 10000.f);
        P.q = static_cast<__nv_bfloat16*>(a.q);
        P.kk = static_cast<__nv_bfloat16*>(a.k_out);
        P.v = static_cast<__nv_bfloat16*>(a.v_out);
        P.n_q_heads = a.n_q_heads;
        P.n_kv_heads = a.n_kv_heads;
        P.ss_out = a.ss_out;
        P.ss_in = a.ss_in;
        P.ss_parts = a.ss_parts;
        P.ss_ld = a.ss_ld;
        P.ss_inv_dim = a.ss_dim > 0 ? 1.f / static_cast<float>(a.ss_dim) : 0.f;
        P.ss_eps = a.ss_eps;
        if (P.units < min_units) min_units = P.units;
    }
    static const bool streamk = [] {  // ASV_CHAIN_KIND=streamk: the stream-K kernel (A/B only)
        const char* e = getenv("ASV_CHAIN_KIND");
        return e != nullptr && std::string(e) == "streamk";
    }();
    if (!streamk && bn <= 128) return chain2_launch(p, maps, ph[0].pdl != 0, ws, st);
    // every CTA gets a non-empty unit range in every phase (the owner protocol counts on it)
    const int grid = static_cast<int>(2 * ws->sms < min_units ? 2 * ws->sms : min_units);
    for (int q = 0; q < n; ++q) {
        p.ph[q].done_target = ws->base[q] + static_cast<uint32_t>(p.ph[q].tiles);
    }
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(linear_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             chain_smem(256));
        if (e != cudaSuccess) return cuda_fail(e, "linear_chain: smem attribute");
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = chain_smem(bn);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ph[0].pdl ? 1 : 0;
    ws->trace_grid = grid;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, linear_chain_kernel, maps, p);
    if (e != cudaSuccess) return cuda_fail(e, "linear_chain launch");
    for (int q = 0; q < n; ++q) ws->base[q] = p.ph[q].done_target;
    return ASV_OK;
}

}  // namespace

cudaError_t linear_chain_preload() {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, linear_chain_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, linear_chain2_kernel);
    return e;
}

}  // namespace asv

// ------------------------------------------------------------------ C ABI
extern "C" {

int asv_linear_chain_ws_create(int32_t device, asv_linear_chain_ws** out) {
    if (out == nullptr) return asv::fail(ASV_ERR_INVALID, "linear_chain_ws_create: null out");
    *out = nullptr;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return asv::cuda_fail(e, "linear_chain_ws_create: device");
    auto* ws = new asv_linear_chain_ws{};
    ws->device = device;
    cudaDeviceGetAttribute(&ws->sms, cudaDevAttrMultiProcessorCount, device);
    const size_t part = static_cast<size_t>(2 * ws->sms) * 256 * 128 * sizeof(float);
    e = cudaMalloc(&ws->done, asv::kMaxPhases * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&ws->arrive, asv::kMaxPhases * asv::kMaxTiles * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&ws->part, part);
    if (e == cudaSuccess) e = cudaMalloc(&ws->pre, part);
    if (e == cudaSuccess) e = cudaMalloc(&ws->done2, (asv::kMaxPhases + 1) * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(ws->done2, 0, (asv::kMaxPhases + 1) * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(ws->done, 0, asv::kMaxPhases * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(ws->arrive, 0, asv::kMaxPhases * asv::kMaxTiles * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        asv_linear_chain_ws_destroy(ws);
        return asv::cuda_fail(e, "linear_chain_ws_create");
    }
    *out = ws;
    return ASV_OK;
}

void asv_linear_chain_ws_destroy(asv_linear_chain_ws* ws) {
    if (ws == nullptr) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ws->device);
    if (ws->done) cudaFree(ws->done);
    if (ws->arrive) cudaFree(ws->arrive);
    if (ws->part) cudaFree(ws->part);
    if (ws->pre) cudaFree(ws->pre);
    if (ws->done2) cudaFree(ws->done2);
    if (ws->trace) cudaFree(ws->trace);
    cudaSetDevice(prev);
    delete ws;
}

int asv_linear_chain_ws_trace(asv_linear_chain_ws* ws, int32_t enable, uint64_t* out, int64_t cap, int64_t* n) {
    if (ws == nullptr) return asv::fail(ASV_ERR_INVALID, "linear_chain_ws_trace: null workspace");
    const size_t words = static_cast<size_t>(2 * ws->sms) * asv::kMaxPhases * asv::kTraceSlots;
    if (enable != 0 && ws->trace == nullptr) {
        const cudaError_t e = cudaMalloc(&ws->trace, words * 8);
        if (e != cudaSuccess) return asv::cuda_fail(e, "linear_chain_ws_trace");
        cudaMemset(ws->trace, 0, words * 8);
    }
    if (enable == 0 && ws->trace != nullptr) {
        cudaFree(ws->trace);
        ws->trace = nullptr;
    }
    if (n != nullptr) *n = 0;
    if (out != nullptr && ws->trace != nullptr) {
        const size_t m = static_cast<size_t>(ws->trace_grid) * asv::kMaxPhases * asv::kTraceSlots;
        if (static_cast<int64_t>(m) > cap) return asv::fail(ASV_ERR_INVALID, "linear_chain_ws_trace: out too small");
        const cudaError_t e = cudaMemcpy(out, ws->trace, m * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return asv::cuda_fail(e, "linear_chain_ws_trace copy");
        if (n != nullptr) *n = static_cast<int64_t>(m);
    }
    return ASV_OK;
}

int asv_linear_chain(const asv_linear_args* phases, int32_t n, asv_linear_chain_ws* ws, void* stream) {
    return asv::chain_run(phases, n, ws, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
