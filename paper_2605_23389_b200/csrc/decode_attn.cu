// Paged split-KV decode attention for sm_100a (K1 + fused split merge K2 + fused
// KV append K3).  Replaces the *priced* attention term of
// prefixsim::iteration_latency (reference cost_model.hpp:112-135), computing
// PAPER Eq. 2: O = softmax(q K^T / sqrt(d)) V over exactly
// s = prefix_len tokens per (request, head) — the `lens` vector the reference
// builds in SchedulerState::running order (cluster_sim.hpp:476-479).
//
// Design:
//  * persistent kernel; every WARP is an independent worker that both produces
//    (one elected lane issues 1-D bulk TMA, cp.async.bulk + mbarrier, into a
//    private S-stage shared-memory ring) and consumes its pages;
//  * work items (request, kv head, <=32-page split) are grabbed dynamically from
//    a global counter in longest-first order (host plan), with a two-item
//    lookahead: the next item's descriptor + page indices are loaded while the
//    current one streams, so the TMA ring never waits on index loads;
//  * pages are stored XOR-swizzled in HBM (chunk c of row t at c ^ (t&7)), so the
//    bulk copy lands them bank-conflict-free with no tensor map;
//  * MHA (group 1): CUDA-core math with the sm_100 mixed-precision
//    fma.rn.f32.bf16 (one FHFMA per MAC, no converts), warp-shuffle softmax;
//  * GQA (group 2..8): mma.sync.m16n8k16 bf16 on the query group (rows = heads),
//    S fragment reused in registers as the PV A operand;
//  * split requests publish (o, m, l) partials; a small PDL-chained merge kernel
//    (K2) combines them (log-sum-exp), so the streaming kernel carries no
//    fences, semaphores or grid barriers and finished CTAs free their SM for the
//    next layer's prefetch;
//  * the owner of a request's last split appends the step's K/V row at position
//    seq_len (prefix_len += 1, cluster_sim.hpp:443-447);
//  * programmatic dependent launch: the KV prefetch of layer l+1 overlaps layer
//    l's tail; q, outputs and the append wait on griddepcontrol.wait;
//  * KV element type bf16 (default) or fp16 (template flag F16): q, KV, the
//    appended row and the output share it; the same FHFMA / HMMA instructions
//    exist in both types, P is rounded to the KV type before P.V.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "asv_internal.h"

namespace asv {
namespace {

constexpr int kD = 128;
constexpr int kPage = 16;
constexpr int kRowBytes = kD * 2;               // 256
constexpr int kBlockBytes = kPage * kRowBytes;  // 4096: one (page, layer, K|V, head) block
constexpr int kStageBytes = 2 * kBlockBytes;    // K + V
constexpr int kDefaultL2Prefetch = 0;           // L2 bulk prefetch beyond the TMA ring: measured slower on B200, off
constexpr int kWarpExtra = 768;                 // per warp: mbarriers | descriptor ring | P scratch
constexpr float kLog2e = 1.4426950408889634f;

struct Params {
    const uint16_t* q;          // bf16 or fp16 bits (F16)
    const char* pool;
    char* pool_w;
    int64_t page_bytes;
    int64_t layer_off;
    int64_t v_off;
    int32_t group_pages;        // layer-major page groups (asv_internal.h pool_slot)
    int32_t group_skip;
    int32_t usable_pages;       // valid page ids: [0, usable_pages)
    const int32_t* gdesc;       // [G][kDescWords]
    const int32_t* split_base;  // [b+1]
    int32_t num_items;
    int32_t n_kv;
    int32_t n_q;
    int32_t total_warps;
    const uint16_t* k_new;
    const uint16_t* v_new;
    uint16_t* out;
    float* lse;
    float* part_o;    // [slots * n_q][128]
    float2* part_ml;  // [slots * n_q]
    uint32_t* work;   // [3]: grab counter, arrived warps, exited warps (this launch parity)
    const int32_t* merge_reqs;  // requests split more than once
    int32_t merge_rows;         // merge_reqs count * n_q
    float scale_log2;
    // deferred merge of the PREVIOUS launch (same plan, other workspace parity): its split rows are
    // merged by this launch's warps right after the dependency wait (prev_rows = 0: none)
    const float* prev_part_o;
    const float2* prev_part_ml;
    uint16_t* prev_out;
    float* prev_lse;
    int32_t prev_rows;
    int32_t l2_prefetch;          // pages beyond the TMA ring prefetched into L2 (0: off)
    unsigned long long* warp_ts;  // optional [total_warps][2] %globaltimer start/end (bubble probe, I1)
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
// Bulk prefetch of a block into L2 (no shared memory, no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
// d = a.{lo|hi} * b.{lo|hi} + c   (bf16 x bf16 or fp16 x fp16 -> fp32, sm_100 FHFMA)
template <bool F16, int AH, int BH>
__device__ __forceinline__ float fma_kv(uint32_t a, uint32_t b, float c) {
    if constexpr (F16) {
        asm("{\n .reg .b16 a0, a1, b0, b1;\n mov.b32 {a0, a1}, %1;\n mov.b32 {b0, b1}, %2;\n"
            " fma.rn.f32.f16 %0, a%3, b%4, %0;\n}\n"
            : "+f"(c)
            : "r"(a), "r"(b), "n"(AH), "n"(BH));
    } else {
        asm("{\n .reg .b16 a0, a1, b0, b1;\n mov.b32 {a0, a1}, %1;\n mov.b32 {b0, b1}, %2;\n"
            " fma.rn.f32.bf16 %0, a%3, b%4, %0;\n}\n"
            : "+f"(c)
            : "r"(a), "r"(b), "n"(AH), "n"(BH));
    }
    return c;
}
template <bool F16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    if constexpr (F16) {
        __half2 v = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&v);
    } else {
        __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&v);
    }
}
// x rounded to the KV type: its bits, and (in *f) its value
template <bool F16>
__device__ __forceinline__ uint16_t round_kv(float x, float* f) {
    if constexpr (F16) {
        const __half h = __float2half_rn(x);
        *f = __half2float(h);
        return __half_as_ushort(h);
    } else {
        const __nv_bfloat16 h = __float2bfloat16_rn(x);
        *f = __bfloat162float(h);
        return __bfloat16_as_ushort(h);
    }
}

__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}
// m16n8k16 with a full A fragment (a0..a3) and B fragment (b0, b1), fp32 accumulate
template <bool F16>
__device__ __forceinline__ void mma_m16(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
    if constexpr (F16) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7},"
            " {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7},"
            " {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
}
// transpose of an 8x8 16-bit matrix held one b32 (two elements) per lane
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
// zero the 16-bit halves of a packed pair {token k (lo), token k+1 (hi)} past `valid`
__device__ __forceinline__ uint32_t mask_tokens(uint32_t b, int k, int valid) {
    if (k >= valid) return 0u;
    if (k + 1 >= valid) return b & 0x0000ffffu;
    return b;
}
// swizzled byte offset of (row t, 16-byte chunk c) inside a 4 KiB block
__device__ __forceinline__ uint32_t swz(int t, int c) {
    return static_cast<uint32_t>(t * kRowBytes + ((c ^ (t & 7)) << 4));
}

// ------------------------------------------------------- work items
// Host plan descriptor per global split g (asv_attn_plan_build):
//   [0] request  [1] partial slot  [2] page_begin  [3] page_end  [4] seq_len
//   [5] nsplit   [6] append page (physical id, -1: none)  [7] 0
//   [8 .. 8+32) physical page ids of pages page_begin .. page_end-1
struct Desc {
    int r, slot, pb, pe, seq, nsplit, append_phys, head;
};

// lane 0 reserves `n` consecutive item ids; the raw result stays in lane 0's
// register until broadcast, so the atomic's latency overlaps useful work.
__device__ __forceinline__ uint32_t grab_raw(const Params& p, int lane, uint32_t n) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(p.work, n);
    return k;
}
__device__ __forceinline__ uint32_t bcast(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

// Issue the (independent) loads of item k's descriptor; lane j also fetches the
// physical id of the item's j-th page.  Nothing here is consumed until the item
// becomes current, so the latency hides behind the previous item.
__device__ __forceinline__ void load_desc(const Params& p, uint32_t k, int lane, Desc& d, int& phys) {
    if (k >= static_cast<uint32_t>(p.num_items)) {
        d.pb = d.pe = 0;
        phys = 0;
        return;
    }
    const int g = static_cast<int>(k) / p.n_kv;
    d.head = static_cast<int>(k) - g * p.n_kv;
    const int32_t* gd = p.gdesc + static_cast<int64_t>(g) * kDescWords;
    const int4 a = __ldg(reinterpret_cast<const int4*>(gd));
    const int4 b = __ldg(reinterpret_cast<const int4*>(gd) + 1);
    phys = __ldg(gd + 8 + lane);
    // a page id outside the pool would make the fused KV append write outside it: fail loudly
    if ((lane < a.w - a.z && static_cast<uint32_t>(phys) >= static_cast<uint32_t>(p.usable_pages)) ||
        b.z >= p.usable_pages) {
        __trap();
    }
    phys += (phys / p.group_pages) * p.group_skip;  // page id -> slice index in the grouped pool
    d.r = a.x;
    d.slot = a.y;
    d.pb = a.z;
    d.pe = a.w;
    d.seq = b.x;
    d.nsplit = b.y;
    d.append_phys = b.z < 0 ? b.z : b.z + (b.z / p.group_pages) * p.group_skip;
}

// ------------------------------------------------------------- epilogues
template <bool F16>
__device__ __forceinline__ void write_final_row(const Params& p, int r, int qh, int lane, const float* o,
                                                float m, float l) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint2 w;
    w.x = pack2<F16>(o[0] * inv, o[1] * inv);
    w.y = pack2<F16>(o[2] * inv, o[3] * inv);
    *reinterpret_cast<uint2*>(p.out + (static_cast<int64_t>(r) * p.n_q + qh) * kD + lane * 4) = w;
    if (p.lse != nullptr && lane == 0) {
        p.lse[static_cast<int64_t>(r) * p.n_q + qh] = l > 0.f ? (m + __log2f(l)) / kLog2e : -INFINITY;
    }
}

// Deferred split merge, one warp per (request, query head) row of the previous launch: lane l owns
// dims 4l..4l+3; online (max, sum) over 8-split batches of coalesced 512-byte loads.
template <bool F16>
__device__ __forceinline__ void merge_prev_row(const Params& p, int row, int lane) {
    const int r = __ldg(p.merge_reqs + row / p.n_q);
    const int qh = row % p.n_q;
    const int s0 = __ldg(p.split_base + r);
    const int ns = __ldg(p.split_base + r + 1) - s0;
    const float2* ml = p.prev_part_ml + static_cast<int64_t>(s0) * p.n_q + qh;
    const float4* po = reinterpret_cast<const float4*>(p.prev_part_o + (static_cast<int64_t>(s0) * p.n_q + qh) * kD) + lane;
    const int64_t ostride = static_cast<int64_t>(p.n_q) * (kD / 4);
    float M = -INFINITY, L = 0.f;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int base = 0; base < ns; base += 8) {
        float4 v[8];
        float2 w[8];
        float bm = -INFINITY;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (base + j < ns) {
                v[j] = __ldcg(po + (base + j) * ostride);
                w[j] = __ldcg(ml + static_cast<int64_t>(base + j) * p.n_q);
            } else {
                v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                w[j] = make_float2(-INFINITY, 0.f);
            }
            bm = fmaxf(bm, w[j].x);
        }
        const float mn = fmaxf(M, bm);
        if (mn == -INFINITY) continue;
        const float a = exp2f(M - mn);
        L *= a;
        o[0] *= a;
        o[1] *= a;
        o[2] *= a;
        o[3] *= a;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float e = (w[j].x == -INFINITY) ? 0.f : exp2f(w[j].x - mn);
            L += e * w[j].y;
            o[0] += e * v[j].x;
            o[1] += e * v[j].y;
            o[2] += e * v[j].z;
            o[3] += e * v[j].w;
        }
        M = mn;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    uint2 wv;
    wv.x = pack2<F16>(o[0] * inv, o[1] * inv);
    wv.y = pack2<F16>(o[2] * inv, o[3] * inv);
    *reinterpret_cast<uint2*>(p.prev_out + (static_cast<int64_t>(r) * p.n_q + qh) * kD + lane * 4) = wv;
    if (p.prev_lse != nullptr && lane == 0) {
        p.prev_lse[static_cast<int64_t>(r) * p.n_q + qh] = L > 0.f ? (M + __log2f(L)) / kLog2e : -INFINITY;
    }
}

// KV append (K3): lanes 0-15 write the K row, 16-31 the V row (16 B each, swizzled).
__device__ __forceinline__ void append_row(const Params& p, const Desc& d, int lane) {
    if (p.k_new == nullptr || d.append_phys < 0) return;
    const int t = d.seq % kPage;
    const int c = lane & 15;
    const bool is_v = lane >= 16;
    const uint16_t* src = (is_v ? p.v_new : p.k_new) + (static_cast<int64_t>(d.r) * p.n_kv + d.head) * kD + c * 8;
    char* dst = p.pool_w + static_cast<int64_t>(d.append_phys) * p.page_bytes + p.layer_off +
                (is_v ? p.v_off : 0) + static_cast<int64_t>(d.head) * kBlockBytes + swz(t, c);
    *reinterpret_cast<uint4*>(dst) = __ldg(reinterpret_cast<const uint4*>(src));
}

// ------------------------------------------------------------- q staging
// MHA: lane (t = lane & 15, half = lane >> 4) keeps the 64 q dims of its half.
template <int GROUP>
struct QRegs;

template <>
struct QRegs<1> {
    uint32_t v[32];
    __device__ __forceinline__ void load(const Params& p, const Desc& d, int lane) {
        const uint4* src = reinterpret_cast<const uint4*>(
            p.q + (static_cast<int64_t>(d.r) * p.n_q + d.head) * kD + (lane >> 4) * 64);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 x = __ldg(src + j);
            v[4 * j + 0] = x.x;
            v[4 * j + 1] = x.y;
            v[4 * j + 2] = x.z;
            v[4 * j + 3] = x.w;
        }
    }
};

// GQA: B fragments of Q^T (k = 16 dims per step, n = the GROUP heads padded to 8):
// lane holds Q[head = lane/4][dims 16ks + 2(lane%4) .. +1] and the same +8.
template <int GROUP>
struct QRegs {
    uint32_t v[16];
    __device__ __forceinline__ void load(const Params& p, const Desc& d, int lane) {
        const int head = lane >> 2, kc = (lane & 3) * 2;
        const bool hv = head < GROUP;
        const uint16_t* src = p.q + (static_cast<int64_t>(d.r) * p.n_q + d.head * GROUP + (hv ? head : 0)) * kD;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            v[2 * ks] = hv ? __ldg(reinterpret_cast<const uint32_t*>(src + ks * 16 + kc)) : 0u;
            v[2 * ks + 1] = hv ? __ldg(reinterpret_cast<const uint32_t*>(src + ks * 16 + 8 + kc)) : 0u;
        }
    }
};

// ------------------------------------------------------- per-item state
template <int GROUP, bool F16>
struct Acc;

template <bool F16>
struct Acc<1, F16> {
    float m, l, o[4];
    __device__ __forceinline__ void reset() {
        m = -INFINITY;
        l = 0.f;
        o[0] = o[1] = o[2] = o[3] = 0.f;
    }
    // one 16-token page: scores, online softmax, P.V
    __device__ __forceinline__ void page(const QRegs<1>& q, uint32_t ks, uint32_t vs, uint32_t sp,
                                         uint16_t* scratch, int valid, float scale, int lane) {
        const int t = lane & 15;
        const int half = lane >> 4;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 kv = lds128(ks + swz(t, half * 8 + j));
            a0 = fma_kv<F16, 0, 0>(kv.x, q.v[4 * j + 0], a0);
            a1 = fma_kv<F16, 1, 1>(kv.x, q.v[4 * j + 0], a1);
            a2 = fma_kv<F16, 0, 0>(kv.y, q.v[4 * j + 1], a2);
            a3 = fma_kv<F16, 1, 1>(kv.y, q.v[4 * j + 1], a3);
            a0 = fma_kv<F16, 0, 0>(kv.z, q.v[4 * j + 2], a0);
            a1 = fma_kv<F16, 1, 1>(kv.z, q.v[4 * j + 2], a1);
            a2 = fma_kv<F16, 0, 0>(kv.w, q.v[4 * j + 3], a2);
            a3 = fma_kv<F16, 1, 1>(kv.w, q.v[4 * j + 3], a3);
        }
        float s = (a0 + a1) + (a2 + a3);
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        s = (t < valid) ? s * scale : -INFINITY;
        float mx = s;
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        const float m_new = fmaxf(m, mx);
        if (m_new > m) {  // warp-uniform: the running max moved
            const float alpha = exp2f(m - m_new);
            l *= alpha;
            o[0] *= alpha;
            o[1] *= alpha;
            o[2] *= alpha;
            o[3] *= alpha;
        }
        m = m_new;
        // P rounded to the KV type for the PV product (FA2/FA3 convention); l sums
        // the rounded weights so O / l stays an exact convex combination of V rows.
        float pf;
        const uint16_t pb = round_kv<F16>(exp2f(s - m_new), &pf);
        l += (half == 0) ? pf : 0.f;
        if (half == 0) scratch[t] = pb;
        __syncwarp();
        const uint4 p0 = lds128(sp);
        const uint4 p1 = lds128(sp + 16);
        const uint32_t pw[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
        const int cidx = lane >> 1;
        const uint32_t coff = (lane & 1) * 8;
        if (valid == kPage) {
#pragma unroll
            for (int tt = 0; tt < kPage; tt += 2) {
                const uint2 v0 = lds64(vs + swz(tt, cidx) + coff);
                const uint2 v1 = lds64(vs + swz(tt + 1, cidx) + coff);
                const uint32_t pp = pw[tt >> 1];
                o[0] = fma_kv<F16, 0, 0>(v0.x, pp, o[0]);
                o[1] = fma_kv<F16, 1, 0>(v0.x, pp, o[1]);
                o[2] = fma_kv<F16, 0, 0>(v0.y, pp, o[2]);
                o[3] = fma_kv<F16, 1, 0>(v0.y, pp, o[3]);
                o[0] = fma_kv<F16, 0, 1>(v1.x, pp, o[0]);
                o[1] = fma_kv<F16, 1, 1>(v1.x, pp, o[1]);
                o[2] = fma_kv<F16, 0, 1>(v1.y, pp, o[2]);
                o[3] = fma_kv<F16, 1, 1>(v1.y, pp, o[3]);
            }
        } else {
            // partial last page: rows >= valid may hold stale data (0 * NaN = NaN)
#pragma unroll
            for (int tt = 0; tt < kPage; tt += 2) {
                uint2 v0 = lds64(vs + swz(tt, cidx) + coff);
                uint2 v1 = lds64(vs + swz(tt + 1, cidx) + coff);
                if (tt >= valid) v0 = make_uint2(0u, 0u);
                if (tt + 1 >= valid) v1 = make_uint2(0u, 0u);
                const uint32_t pp = pw[tt >> 1];
                o[0] = fma_kv<F16, 0, 0>(v0.x, pp, o[0]);
                o[1] = fma_kv<F16, 1, 0>(v0.x, pp, o[1]);
                o[2] = fma_kv<F16, 0, 0>(v0.y, pp, o[2]);
                o[3] = fma_kv<F16, 1, 0>(v0.y, pp, o[3]);
                o[0] = fma_kv<F16, 0, 1>(v1.x, pp, o[0]);
                o[1] = fma_kv<F16, 1, 1>(v1.x, pp, o[1]);
                o[2] = fma_kv<F16, 0, 1>(v1.y, pp, o[2]);
                o[3] = fma_kv<F16, 1, 1>(v1.y, pp, o[3]);
            }
        }
    }
    // returns true when a partial was published for the merge kernel
    __device__ __forceinline__ bool finish(const Params& p, const Desc& d, int lane) {
        float lt = l;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, off);
        if (d.nsplit == 1) {
            write_final_row<F16>(p, d.r, d.head, lane, o, m, lt);
            return false;
        }
        const int64_t slot = static_cast<int64_t>(d.slot) * p.n_q + d.head;
        __stcg(reinterpret_cast<float4*>(p.part_o + slot * kD) + lane, make_float4(o[0], o[1], o[2], o[3]));
        if (lane == 0) __stcg(p.part_ml + slot, make_float2(m, lt));
        return true;
    }
};

// GQA: tokens are the MMA M dimension.  S^T[16 tok x 8 heads] = K[16 x 128] Q^T
// (8 HMMA: all 16 M rows are real tokens), then O^T[128 d x 8 heads] += V^T P^T
// (8 HMMA, A = V^T via ldmatrix.trans).  A lane owns query heads 2(lane%4),
// 2(lane%4)+1 in both the S and the O fragments, so the online-softmax state is
// per lane and the rescale needs no data movement; P^T crosses lanes once per
// page through a 256-byte shared-memory transpose.
template <int GROUP, bool F16>
struct Acc {
    float m[2], l[2];  // heads h0 = 2(lane%4), h0+1
    float o[8][4];     // O^T fragments: d = 16mt + lane/4 (+8), heads h0, h0+1
    __device__ __forceinline__ void reset() {
        m[0] = m[1] = -INFINITY;
        l[0] = l[1] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    }
    __device__ __forceinline__ void page(const QRegs<GROUP>& q, uint32_t ks, uint32_t vs, uint32_t sp,
                                         uint16_t* pt, int valid, float scale, int lane) {
        const int tA = lane >> 2, tB = tA + 8;     // this lane's token rows
        const int hc = (lane & 3) * 2;             // this lane's head pair
        // ---- S^T = K Q^T (two accumulators: 4-deep HMMA chains)
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
        const int arow = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
            uint32_t a0, a1, a2, a3, c0, c1, c2, c3;
            ldsm_x4(ks + swz(arow, 2 * kk + (lane >> 4)), a0, a1, a2, a3);
            ldsm_x4(ks + swz(arow, 2 * kk + 2 + (lane >> 4)), c0, c1, c2, c3);
            mma_m16<F16>(sa, a0, a1, a2, a3, q.v[2 * kk], q.v[2 * kk + 1]);
            mma_m16<F16>(sb, c0, c1, c2, c3, q.v[2 * kk + 2], q.v[2 * kk + 3]);
        }
        // lane: s[0] = (tA, h0), s[1] = (tA, h1), s[2] = (tB, h0), s[3] = (tB, h1)
        float sv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int tok = (e < 2) ? tA : tB;
            sv[e] = (tok < valid) ? (sa[e] + sb[e]) * scale : -INFINITY;
        }
        float mx0 = fmaxf(sv[0], sv[2]), mx1 = fmaxf(sv[1], sv[3]);
#pragma unroll
        for (int off = 4; off <= 16; off <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);
        if (__any_sync(0xffffffffu, (mn0 > m[0]) || (mn1 > m[1]))) {
            const float al0 = exp2f(m[0] - mn0), al1 = exp2f(m[1] - mn1);
            l[0] *= al0;
            l[1] *= al1;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                o[i][0] *= al0;
                o[i][1] *= al1;
                o[i][2] *= al0;
                o[i][3] *= al1;
            }
        }
        m[0] = mn0;
        m[1] = mn1;
        float f0, f1, f2, f3;
        const uint16_t p0 = round_kv<F16>(exp2f(sv[0] - mn0), &f0);
        const uint16_t p1 = round_kv<F16>(exp2f(sv[1] - mn1), &f1);
        const uint16_t p2 = round_kv<F16>(exp2f(sv[2] - mn0), &f2);
        const uint16_t p3 = round_kv<F16>(exp2f(sv[3] - mn1), &f3);
        l[0] += f0 + f2;
        l[1] += f1 + f3;
        // ---- P^T -> B fragments (k = tokens, n = heads): the S^T accumulator fragment of
        // tokens 0-7 / 8-15 (row = token lane/4, cols = heads 2(lane%4)..+1) transposed in
        // registers (movmatrix) is exactly the m16n8k16 B fragment (k = tokens 2(lane%4)..+1,
        // n = head lane/4) — no shared-memory round trip, no warp barrier
        const uint32_t pb0 = movmatrix_t(static_cast<uint32_t>(p0) | (static_cast<uint32_t>(p1) << 16));
        const uint32_t pb1 = movmatrix_t(static_cast<uint32_t>(p2) | (static_cast<uint32_t>(p3) << 16));
        // ---- O^T += V^T P^T over 8 d-tiles of 16
        const int vrow = (lane & 7) + (lane >> 4) * 8;
        if (valid == kPage) {
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vs + swz(vrow, 2 * mt + ((lane >> 3) & 1)), a0, a1, a2, a3);
                mma_m16<F16>(o[mt], a0, a1, a2, a3, pb0, pb1);
            }
        } else {
            // stale rows >= valid: P is 0 there but 0 * NaN = NaN, so mask V too
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vs + swz(vrow, 2 * mt + ((lane >> 3) & 1)), a0, a1, a2, a3);
                a0 = mask_tokens(a0, hc, valid);
                a1 = mask_tokens(a1, hc, valid);
                a2 = mask_tokens(a2, hc + 8, valid);
                a3 = mask_tokens(a3, hc + 8, valid);
                mma_m16<F16>(o[mt], a0, a1, a2, a3, pb0, pb1);
            }
        }
    }
    __device__ __forceinline__ bool finish(const Params& p, const Desc& d, int lane) {
        float lt0 = l[0], lt1 = l[1];
#pragma unroll
        for (int off = 4; off <= 16; off <<= 1) {
            lt0 += __shfl_xor_sync(0xffffffffu, lt0, off);
            lt1 += __shfl_xor_sync(0xffffffffu, lt1, off);
        }
        const int hc = (lane & 3) * 2, dr = lane >> 2;
        const bool nsplit1 = d.nsplit == 1;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int h = hc + e;
            if (h >= GROUP) continue;
            const int qh = d.head * GROUP + h;
            const float lt = e ? lt1 : lt0, mm = e ? m[1] : m[0];
            if (nsplit1) {
                const float inv = lt > 0.f ? 1.f / lt : 0.f;
                uint16_t* dst = p.out + (static_cast<int64_t>(d.r) * p.n_q + qh) * kD;
                float unused;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    dst[16 * mt + dr] = round_kv<F16>(o[mt][e] * inv, &unused);
                    dst[16 * mt + dr + 8] = round_kv<F16>(o[mt][2 + e] * inv, &unused);
                }
                if (p.lse != nullptr && dr == 0) {
                    p.lse[static_cast<int64_t>(d.r) * p.n_q + qh] = lt > 0.f ? (mm + __log2f(lt)) / kLog2e : -INFINITY;
                }
            } else {
                const int64_t slot = static_cast<int64_t>(d.slot) * p.n_q + qh;
                float* dst = p.part_o + slot * kD;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    __stcg(dst + 16 * mt + dr, o[mt][e]);
                    __stcg(dst + 16 * mt + dr + 8, o[mt][2 + e]);
                }
                if (dr == 0) __stcg(p.part_ml + slot, make_float2(mm, lt));
            }
        }
        return !nsplit1;
    }
};

// ============================================================ the kernel
template <int NW, int S, int GROUP, bool F16>
__global__ void __launch_bounds__(NW * 32, (NW == 2 ? 4 : 2))
decode_attn_kernel(const Params p) {
    constexpr int kRing = S + 1;  // descriptor ring must cover the TMA lookahead
    static_assert(S <= 8, "mbarrier area holds 8 stages");
    extern __shared__ __align__(1024) char smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // per warp: S stages (8 KiB) | S mbarriers (64 B) | desc ring (<= 288 B) | P scratch (256 B @ +512)
    constexpr int kWarpBytes = S * kStageBytes + kWarpExtra;
    char* wbase = smem_raw + warp * kWarpBytes;
    const uint32_t stage0 = smem_u32(wbase);
    const uint32_t bar0 = smem_u32(wbase + S * kStageBytes);
    uint16_t* scratch = reinterpret_cast<uint16_t*>(wbase + S * kStageBytes + 512);
    const uint32_t sp = smem_u32(scratch);
    Desc* ring = reinterpret_cast<Desc*>(wbase + S * kStageBytes + 64);

    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint64_t pol = evict_first_policy();
    unsigned long long ts_begin = 0;
    if (p.warp_ts != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_begin));

    // ---- producer state: current item (descriptor + lane-distributed page ids),
    // next item (loads in flight), and the id after that (atomic in flight)
    Desc cur, nxt;
    int cur_phys, nxt_phys;
    const uint32_t k0 = bcast(grab_raw(p, lane, 3u));
    uint32_t k1 = k0 + 1u;
    uint32_t k2_raw = k0 + 2u;  // valid on every lane here; later only on lane 0
    load_desc(p, k0, lane, cur, cur_phys);
    load_desc(p, k1, lane, nxt, nxt_phys);
    int ppage = cur.pb;
    bool have_cur = k0 < static_cast<uint32_t>(p.num_items);
    int pushed = 0;
    if (have_cur && lane == 0) ring[0] = cur;
    if (have_cur) pushed = 1;
    __syncwarp();

    auto advance_producer = [&]() {
        cur = nxt;
        cur_phys = nxt_phys;
        have_cur = k1 < static_cast<uint32_t>(p.num_items);
        if (have_cur) {
            k1 = bcast(k2_raw);
            ppage = cur.pb;
            if (lane == 0) ring[pushed % kRing] = cur;
            ++pushed;
            load_desc(p, k1, lane, nxt, nxt_phys);
            if (k1 < static_cast<uint32_t>(p.num_items)) k2_raw = grab_raw(p, lane, 1u);
        }
    };
    auto issue = [&](int slot) {
        const int phys = __shfl_sync(0xffffffffu, cur_phys, ppage - cur.pb);
        // L2 prefetch of the page `l2_prefetch` positions further along this
        // warp's stream (current item, else the looked-ahead next item)
        if (p.l2_prefetch > 0) {
            const int ahead = ppage + p.l2_prefetch;
            int pf = -1, pf_head = cur.head;
            if (ahead < cur.pe) {
                pf = __shfl_sync(0xffffffffu, cur_phys, ahead - cur.pb);
            } else if (k1 < static_cast<uint32_t>(p.num_items) && ahead - cur.pe < nxt.pe - nxt.pb) {
                pf = __shfl_sync(0xffffffffu, nxt_phys, ahead - cur.pe);
                pf_head = nxt.head;
            }
            if (pf >= 0 && lane == 0) {
                const char* blk = p.pool + static_cast<int64_t>(pf) * p.page_bytes + p.layer_off +
                                  static_cast<int64_t>(pf_head) * kBlockBytes;
                bulk_prefetch_l2(blk, kBlockBytes);
                bulk_prefetch_l2(blk + p.v_off, kBlockBytes);
            }
        }
        if (lane == 0) {
            const char* kblk = p.pool + static_cast<int64_t>(phys) * p.page_bytes + p.layer_off +
                               static_cast<int64_t>(cur.head) * kBlockBytes;
            const uint32_t bar = bar0 + 8 * slot;
            const uint32_t dst = stage0 + slot * kStageBytes;
            mbar_expect_tx(bar, kStageBytes);
            bulk_g2s(dst, kblk, kBlockBytes, bar, pol);
            bulk_g2s(dst + kBlockBytes, kblk + p.v_off, kBlockBytes, bar, pol);
        }
        if (++ppage >= cur.pe) advance_producer();
    };

    // prologue: fill the ring (KV does not depend on the previous layer)
    int issued = 0;
    for (; issued < S && have_cur; ++issued) issue(issued);

    // everything below reads q / writes outputs: wait for the previous grid
    grid_dep_wait();
    grid_dep_launch();

    // the previous launch deferred its split merge: its rows are this launch's first work (its
    // partials are complete: the dependency wait covered that grid); the KV ring keeps filling
    if (p.prev_rows > 0) {
        for (;;) {
            uint32_t row = 0;
            if (lane == 0) row = atomicAdd(p.work + 2, 1u);
            row = bcast(row);
            if (row >= static_cast<uint32_t>(p.prev_rows)) break;
            merge_prev_row<F16>(p, static_cast<int>(row), lane);
        }
    }

    QRegs<GROUP> q, qn;
    Acc<GROUP, F16> acc;
    int consumed = 0;   // pages
    int citem = 0;      // items started by the consumer
    bool qn_ready = false;
    Desc cd;            // consumer's current item
    int cpage = 0;

    while (citem < pushed) {
        // ---- start the next item (the producer pushed it >= 1 page ago or just now)
        __syncwarp();
        cd = ring[citem % kRing];
        ++citem;
        if (qn_ready) {
            q = qn;
            qn_ready = false;
        } else {
            q.load(p, cd, lane);
        }
        acc.reset();
        append_row(p, cd, lane);
        for (cpage = cd.pb; cpage < cd.pe; ++cpage) {
            const int slot = consumed % S;
            mbar_wait(bar0 + 8 * slot, (consumed / S) & 1);
            const uint32_t ks = stage0 + slot * kStageBytes;
            acc.page(q, ks, ks + kBlockBytes, sp, scratch, min(kPage, cd.seq - cpage * kPage), p.scale_log2, lane);
            __syncwarp();
            ++consumed;
            if (have_cur) {
                issue(slot);
                ++issued;
                __syncwarp();  // lane 0 may just have pushed the next item's descriptor into the ring
            }
            if (!qn_ready && citem < pushed) {  // prefetch the next item's q
                qn.load(p, ring[citem % kRing], lane);
                qn_ready = true;
            }
        }
        acc.finish(p, cd, lane);  // final row (single split) or a partial for the merge kernel
    }

    if (p.warp_ts != nullptr && lane == 0) {
        unsigned long long ts_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_end));
        const int64_t w = static_cast<int64_t>(blockIdx.x) * NW + warp;
        p.warp_ts[2 * w] = ts_begin;
        p.warp_ts[2 * w + 1] = ts_end;
    }
    // last warp out re-arms the work counters of this launch parity
    if (lane == 0) {
        const uint32_t done = atomicAdd(p.work + 1, 1u);
        if (done == static_cast<uint32_t>(p.total_warps) - 1u) {
            p.work[0] = 0u;
            p.work[1] = 0u;
            p.work[2] = 0u;
        }
    }
}

// ============================================================ split merge (K2)
// One warp per (request, query head) of every split request.  Chained with
// programmatic dependent launch: its CTAs become resident while the streaming
// kernel runs, let the NEXT layer's streaming kernel launch at once (so its KV
// prefetch overlaps this merge), and park on griddepcontrol.wait until the
// streaming grid has completed (which also publishes its partial stores) — no
// fences or semaphores anywhere on the streaming path.
constexpr int kMergeWarps = 4;

// One CTA per (request, query head) row: the 8 warps take every 8th split and
// keep an online (max, sum, o[4 dims per lane]) state over 8-split batches of
// coalesced loads, then the 8 states are combined through shared memory.
template <bool F16>
__global__ void __launch_bounds__(kMergeWarps * 32, 6)
merge_splits_kernel(const Params p, const int32_t* __restrict__ merge_reqs, int32_t rows) {
    grid_dep_launch();
    grid_dep_wait();
    __shared__ float s_o[kMergeWarps][kD];
    __shared__ float s_m[kMergeWarps], s_l[kMergeWarps];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {
        const int r = __ldg(merge_reqs + row / p.n_q);
        const int qh = row % p.n_q;
        const int s0 = __ldg(p.split_base + r);
        const int ns = __ldg(p.split_base + r + 1) - s0;
        const float2* ml = p.part_ml + static_cast<int64_t>(s0) * p.n_q + qh;
        const float4* po = reinterpret_cast<const float4*>(p.part_o + (static_cast<int64_t>(s0) * p.n_q + qh) * kD) + lane;
        const int64_t mstride = p.n_q, ostride = static_cast<int64_t>(p.n_q) * (kD / 4);
        float M = -INFINITY, L = 0.f;
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        for (int base = warp; base < ns; base += 8 * kMergeWarps) {
            float4 v[8];
            float2 w[8];
            float bm = -INFINITY;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int sidx = base + j * kMergeWarps;
                if (sidx < ns) {
                    v[j] = __ldcg(po + sidx * ostride);
                    w[j] = __ldcg(ml + sidx * mstride);
                } else {
                    v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                    w[j] = make_float2(-INFINITY, 0.f);
                }
                bm = fmaxf(bm, w[j].x);
            }
            const float mn = fmaxf(M, bm);
            if (mn == -INFINITY) continue;
            const float a = exp2f(M - mn);
            L *= a;
            o[0] *= a;
            o[1] *= a;
            o[2] *= a;
            o[3] *= a;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float e = (w[j].x == -INFINITY) ? 0.f : exp2f(w[j].x - mn);
                L += e * w[j].y;
                o[0] += e * v[j].x;
                o[1] += e * v[j].y;
                o[2] += e * v[j].z;
                o[3] += e * v[j].w;
            }
            M = mn;
        }
        *reinterpret_cast<float4*>(&s_o[warp][4 * lane]) = make_float4(o[0], o[1], o[2], o[3]);
        if (lane == 0) {
            s_m[warp] = M;
            s_l[warp] = L;
        }
        __syncthreads();
        if (warp == 0) {
            float Mt = -INFINITY;
#pragma unroll
            for (int w = 0; w < kMergeWarps; ++w) Mt = fmaxf(Mt, s_m[w]);
            float ot[4] = {0.f, 0.f, 0.f, 0.f};
            float Lt = 0.f;
#pragma unroll
            for (int w = 0; w < kMergeWarps; ++w) {
                const float e = (s_m[w] == -INFINITY) ? 0.f : exp2f(s_m[w] - Mt);
                const float4 x = *reinterpret_cast<const float4*>(&s_o[w][4 * lane]);
                ot[0] += e * x.x;
                ot[1] += e * x.y;
                ot[2] += e * x.z;
                ot[3] += e * x.w;
                Lt += e * s_l[w];
            }
            write_final_row<F16>(p, r, qh, lane, ot, Mt, Lt);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------- launcher
// (warps per CTA, TMA stages per warp) variants; the default is chosen per group
// from B200 measurements, ASV_ATTN_VARIANT=<NW>x<S> overrides it (tuning only).
template <int NW, int S, int GROUP, bool F16>
struct Launch {
    static constexpr int kSmem = NW * (S * kStageBytes + kWarpExtra);
    static cudaError_t configure() {
        return cudaFuncSetAttribute(decode_attn_kernel<NW, S, GROUP, F16>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    }
    static cudaError_t occupancy(int* blocks) {
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, decode_attn_kernel<NW, S, GROUP, F16>, NW * 32,
                                                             kSmem);
    }
    static cudaError_t run(const Params& p, int grid, bool pdl, cudaStream_t st) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(NW * 32);
        cfg.dynamicSmemBytes = kSmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        return cudaLaunchKernelEx(&cfg, decode_attn_kernel<NW, S, GROUP, F16>, p);
    }
};

template <int NW, int S, int GROUP, bool F16>
cudaError_t dispatch_variant(bool query, int* blocks, const Params* p, int grid, bool pdl, cudaStream_t st) {
    using L = Launch<NW, S, GROUP, F16>;
    static bool configured = false;  // attribute set is idempotent; a race is harmless
    if (!configured) {
        cudaError_t e = L::configure();
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (query) return L::occupancy(blocks);
    return L::run(*p, grid, pdl, st);
}

struct Variant {
    int nw, stages;
};

Variant default_variant(int group) {
    (void)group;
    return Variant{4, 3};
}

Variant selected_variant(int group) {
    static const char* env = getenv("ASV_ATTN_VARIANT");
    if (env != nullptr) {
        int nw = 0, st = 0;
        if (sscanf(env, "%dx%d", &nw, &st) == 2) return Variant{nw, st};
    }
    return default_variant(group);
}

// fp16 KV: the default (4 warps x 3 stages) variant only
template <int GROUP, bool F16>
cudaError_t dispatch_group(bool query, int* blocks, const Params* p, int grid, bool pdl, cudaStream_t st) {
    const Variant v = selected_variant(GROUP);
    if (v.nw == 4 && v.stages == 3) return dispatch_variant<4, 3, GROUP, F16>(query, blocks, p, grid, pdl, st);
    if constexpr (!F16 && (GROUP == 1 || GROUP == 5 || GROUP == 4)) {
        if (v.nw == 4 && v.stages == 4) return dispatch_variant<4, 4, GROUP, F16>(query, blocks, p, grid, pdl, st);
        if (v.nw == 2 && v.stages == 6) return dispatch_variant<2, 6, GROUP, F16>(query, blocks, p, grid, pdl, st);
        if (v.nw == 4 && v.stages == 2) return dispatch_variant<4, 2, GROUP, F16>(query, blocks, p, grid, pdl, st);
        if (v.nw == 2 && v.stages == 4) return dispatch_variant<2, 4, GROUP, F16>(query, blocks, p, grid, pdl, st);
    }
    return dispatch_variant<4, 3, GROUP, F16>(query, blocks, p, grid, pdl, st);
}

bool variant_available(int group, bool f16, Variant v) {
    if (v.nw == 4 && v.stages == 3) return true;
    if (f16 || (group != 1 && group != 4 && group != 5)) return false;
    return (v.nw == 4 && (v.stages == 4 || v.stages == 2)) || (v.nw == 2 && (v.stages == 6 || v.stages == 4));
}

template <bool F16>
cudaError_t dispatch_t(int group, bool query, int* blocks, const Params* p, int grid, bool pdl, cudaStream_t st) {
    switch (group) {
        case 1: return dispatch_group<1, F16>(query, blocks, p, grid, pdl, st);
        case 2: return dispatch_group<2, F16>(query, blocks, p, grid, pdl, st);
        case 4: return dispatch_group<4, F16>(query, blocks, p, grid, pdl, st);
        case 5: return dispatch_group<5, F16>(query, blocks, p, grid, pdl, st);
        case 8: return dispatch_group<8, F16>(query, blocks, p, grid, pdl, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t dispatch(int group, bool f16, bool query, int* blocks, const Params* p, int grid, bool pdl,
                     cudaStream_t st) {
    return f16 ? dispatch_t<true>(group, query, blocks, p, grid, pdl, st)
               : dispatch_t<false>(group, query, blocks, p, grid, pdl, st);
}

}  // namespace

int attn_warps_per_cta(int group, bool f16) {
    const Variant v = selected_variant(group);
    return variant_available(group, f16, v) ? v.nw : 4;
}

__global__ void sm_copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16);
__global__ void warp_span_reduce_kernel(unsigned long long* __restrict__ ts, int32_t workers,
                                        unsigned long long* __restrict__ out);

cudaError_t attn_occupancy(int group, int* blocks_per_sm) {
    // both KV types: same shared memory and occupancy; loading both keeps lazy module
    // loading off the launch path
    int other = 0;
    cudaError_t e = dispatch(group, true, true, &other, nullptr, 0, false, nullptr);
    if (e != cudaSuccess) return e;
    e = dispatch(group, false, true, blocks_per_sm, nullptr, 0, false, nullptr);
    if (e != cudaSuccess) return e;
    // Load every kernel of the path now (lazy module loading would load them at
    // their first launch, which blocks on device-wide progress: a first launch
    // queued behind a stream-memory-op wait then deadlocks; measured).
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, merge_splits_kernel<false>);
    if (e != cudaSuccess) return e;
    e = cudaFuncGetAttributes(&fa, merge_splits_kernel<true>);
    if (e != cudaSuccess) return e;
    e = cudaFuncGetAttributes(&fa, warp_span_reduce_kernel);
    if (e != cudaSuccess) return e;
    return cudaFuncGetAttributes(&fa, sm_copy_kernel);
}

cudaError_t merge_launch(const Params& p, const int32_t* merge_reqs, int32_t n_merge, int sms, bool pdl, bool f16,
                         cudaStream_t st) {
    const int32_t rows = n_merge * p.n_q;
    if (rows <= 0) return cudaSuccess;
    const int blocks = min(rows, 6 * sms);  // one CTA per row, grid-strided beyond 6 CTAs/SM
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kMergeWarps * 32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return f16 ? cudaLaunchKernelEx(&cfg, merge_splits_kernel<true>, p, merge_reqs, rows)
               : cudaLaunchKernelEx(&cfg, merge_splits_kernel<false>, p, merge_reqs, rows);
}

// 16-byte SM copy between any two device-accessible buffers, used where a
// small transfer must not queue behind multi-GB copy-engine work: the plan
// upload from mapped pinned host memory (asv_plan_upload) and the e2e result
// read-back into mapped pinned host memory.  Grid-strided, all loads in flight
// at once (one PCIe round trip for a typical 10-100 KB buffer).
__global__ void sm_copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        dst[i] = src[i];
    }
}

cudaError_t sm_copy(const int32_t* src, int32_t* dst, int64_t n_int32, cudaStream_t st) {
    const int64_t n16 = (n_int32 + 3) / 4;
    if (n16 <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256;
    int64_t blocks = (n16 + threads - 1) / threads;
    if (blocks > sms) blocks = sms;
    sm_copy_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(reinterpret_cast<const int4*>(src),
                                                                      reinterpret_cast<int4*>(dst), n16);
    return cudaGetLastError();
}

// Measured bubble: one CTA per attention launch reduces the launch's
// per-warp (start, end) %globaltimer pairs to (first start, last end, summed busy
// time of the warps that ran).  idle = (last end - first start) * warps - busy.
__global__ void warp_span_reduce_kernel(unsigned long long* __restrict__ ts, int32_t workers,
                                        unsigned long long* __restrict__ out) {
    unsigned long long* t = ts + static_cast<int64_t>(blockIdx.x) * workers * 2;
    unsigned long long lo = ~0ull, hi = 0, busy = 0;
    for (int w = threadIdx.x; w < workers; w += blockDim.x) {
        const unsigned long long a = t[2 * w], b = t[2 * w + 1];
        t[2 * w] = t[2 * w + 1] = 0;  // consumed: a warp that does not run next time is skipped, not stale
        if (b <= a) continue;
        lo = min(lo, a);
        hi = max(hi, b);
        busy += b - a;
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        busy += __shfl_xor_sync(0xffffffffu, busy, o);
    }
    __shared__ unsigned long long s_lo[8], s_hi[8], s_busy[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_lo[warp] = lo;
        s_hi[warp] = hi;
        s_busy[warp] = busy;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            lo = min(lo, s_lo[w]);
            hi = max(hi, s_hi[w]);
            busy += s_busy[w];
        }
        out[3 * blockIdx.x] = lo;
        out[3 * blockIdx.x + 1] = hi;
        out[3 * blockIdx.x + 2] = busy;
    }
}

cudaError_t warp_span_reduce(uint64_t* ts, int32_t workers, int32_t launches, uint64_t* out, cudaStream_t st) {
    if (launches <= 0) return cudaSuccess;
    warp_span_reduce_kernel<<<launches, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(ts), workers,
                                                      reinterpret_cast<unsigned long long*>(out));
    return cudaGetLastError();
}

// L2-warm mode (asv_attn_args.l2_warm_items): one thread per (item, page) of the first `items` work
// items in the order the persistent warps take them (longest first) and the first `pages` pages of
// each, two 4 KiB bulk L2 prefetches (K, V block).  Lets a side stream pull the first wave of a later
// attention launch into L2 while other kernels leave HBM idle (measurement experiment).
__global__ void attn_l2_warm_kernel(const Params p, int items, int pages) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = i / pages, j = i - item * pages;
    if (item >= items || item >= p.num_items) return;
    const int g = item / p.n_kv, head = item - g * p.n_kv;
    const int32_t* gd = p.gdesc + static_cast<int64_t>(g) * kDescWords;
    const int pb = __ldg(gd + 2), pe = __ldg(gd + 3);
    if (pb + j >= pe) return;
    int phys = __ldg(gd + 8 + j);
    if (static_cast<uint32_t>(phys) >= static_cast<uint32_t>(p.usable_pages)) return;
    phys += (phys / p.group_pages) * p.group_skip;
    const char* blk = p.pool + static_cast<int64_t>(phys) * p.page_bytes + p.layer_off +
                      static_cast<int64_t>(head) * kBlockBytes;
    bulk_prefetch_l2(blk, kBlockBytes);
    bulk_prefetch_l2(blk + p.v_off, kBlockBytes);
}

cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t st) {
    Params p;
    p.q = static_cast<const uint16_t*>(a.q);
    p.pool = static_cast<const char*>(a.pool);
    p.pool_w = static_cast<char*>(a.pool);
    p.page_bytes = a.page_bytes;
    p.layer_off = a.layer_off;
    p.v_off = a.v_off;
    p.group_pages = a.group_pages;
    p.group_skip = a.group_skip;
    p.usable_pages = a.usable_pages;
    p.gdesc = a.gdesc;
    p.split_base = a.split_base;
    p.num_items = a.num_items;
    p.n_kv = a.n_kv;
    p.n_q = a.n_q;
    p.total_warps = a.grid * attn_warps_per_cta(a.group, a.f16);
    p.k_new = static_cast<const uint16_t*>(a.k_new);
    p.v_new = static_cast<const uint16_t*>(a.v_new);
    p.out = static_cast<uint16_t*>(a.out);
    p.lse = a.lse;
    p.part_o = a.part_o;
    p.part_ml = reinterpret_cast<float2*>(a.part_ml);
    p.work = a.work;
    p.merge_reqs = a.merge_reqs;
    p.merge_rows = a.n_merge * a.n_q;
    p.scale_log2 = a.sm_scale * kLog2e;
    p.warp_ts = a.warp_ts;
    p.prev_part_o = a.prev_part_o;
    p.prev_part_ml = reinterpret_cast<const float2*>(a.prev_part_ml);
    p.prev_out = static_cast<uint16_t*>(a.prev_out);
    p.prev_lse = a.prev_lse;
    p.prev_rows = a.prev_out != nullptr ? a.n_merge * a.n_q : 0;
    {
        static const int pf = [] {
            const char* e = getenv("ASV_L2_PREFETCH");
            return e != nullptr ? atoi(e) : kDefaultL2Prefetch;
        }();
        p.l2_prefetch = pf;
    }
    if (p.num_items <= 0) return cudaSuccess;
    if (a.warm_items > 0) {
        const int pages = a.warm_pages > 0 ? a.warm_pages : 1;
        const int64_t n = static_cast<int64_t>(a.warm_items < p.num_items ? a.warm_items : p.num_items) * pages;
        attn_l2_warm_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p, a.warm_items, pages);
        return cudaGetLastError();
    }
    cudaError_t e = dispatch(a.group, a.f16, false, nullptr, &p, a.grid, a.pdl, st);
    if (e != cudaSuccess) return e;
    if (a.defer_merge) return cudaSuccess;  // the next launch merges these partials
    return merge_launch(p, a.merge_reqs, a.n_merge, a.sms, a.pdl, a.f16, st);
}

}  // namespace asv
