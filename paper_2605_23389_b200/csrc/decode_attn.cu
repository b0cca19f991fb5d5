// Paged split-KV decode attention for sm_100a (K1 + fused split merge K2 + fused
// KV append K3).  Replaces the *priced* attention term of
// prefixsim::iteration_latency (reference cost_model.hpp:112-135), computing
// PAPER Eq. 2: O = softmax(q K^T / sqrt(d)) V over exactly
// s = prefix_len tokens per (request, head) — the `lens` vector the reference
// builds in SchedulerState::running order (cluster_sim.hpp:476-479).
//
// Design:
//  * persistent kernel, every WARP is an independent worker with its own
//    S-stage shared-memory ring fed by 1-D bulk TMA (cp.async.bulk + mbarrier);
//    warps walk a static round-robin over equal-sized (request, kv head, split)
//    work items built by the host plan, so every warp streams a near-equal KV
//    span (length-aligned batches make the items near-identical);
//  * pages are stored XOR-swizzled in HBM (chunk c of row t at c ^ (t&7)), so the
//    bulk copy lands them bank-conflict-free with no tensor map;
//  * MHA (group 1): CUDA-core math with the sm_100 mixed-precision
//    fma.rn.f32.bf16 (one FHFMA per MAC, no bf16->fp32 converts), warp-shuffle
//    online softmax;
//  * GQA (group 2..8): mma.sync.m16n8k16 bf16 on the query group (rows = heads),
//    FA2-style register reuse of the S fragment as the PV A operand;
//  * split partials merge in-kernel: the last-arriving warp per (request, kv head)
//    (semaphore) combines the log-sum-exp partials and writes the output;
//  * the warp that owns a request's last split appends the step's K/V row at
//    position seq_len (prefix_len += 1, cluster_sim.hpp:443-447).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "asv_internal.h"

namespace asv {
namespace {

constexpr int kD = 128;
constexpr int kPage = 16;
constexpr int kRowBytes = kD * 2;                 // 256
constexpr int kBlockBytes = kPage * kRowBytes;    // 4096: one (page, layer, K|V, head) block
constexpr int kStageBytes = 2 * kBlockBytes;      // K + V
constexpr float kLog2e = 1.4426950408889634f;

struct Params {
    const __nv_bfloat16* q;
    const char* pool;          // bytes
    char* pool_w;              // same, writable (append)
    int64_t page_bytes;        // one page, all layers
    int64_t layer_off;         // byte offset of the layer slice inside a page
    int64_t v_off;             // K block -> V block, bytes (n_kv * 4096)
    const int32_t* seq_lens;
    const int32_t* page_indptr;
    const int32_t* page_indices;
    const int32_t* split_indptr;
    const int2* item_tab;      // per global split: {request, split}
    int32_t num_items;
    int32_t n_kv;
    int32_t n_q;
    const __nv_bfloat16* k_new;
    const __nv_bfloat16* v_new;
    __nv_bfloat16* out;
    float* lse;
    float* part_o;             // [G * n_q][128]
    float2* part_ml;           // [G * n_q] (m in log2 units, l)
    int32_t* sem;              // [b * n_kv]
    float scale_log2;          // sm_scale * log2(e)
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
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
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
// d = a.lo * b.lo + c  /  a.hi * b.hi + c   (bf16 x bf16 -> fp32, sm_100 FHFMA)
template <int AH, int BH>
__device__ __forceinline__ float fma_bf(uint32_t a, uint32_t b, float c) {
    asm("{\n .reg .b16 a0, a1, b0, b1;\n mov.b32 {a0, a1}, %1;\n mov.b32 {b0, b1}, %2;\n"
        " fma.rn.f32.bf16 %0, a%3, b%4, %0;\n}\n"
        : "+f"(c)
        : "r"(a), "r"(b), "n"(AH), "n"(BH));
    return c;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

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
__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7},"
        " {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// zero the bf16 halves of a packed pair {token k (lo), token k+1 (hi)} past `valid`
__device__ __forceinline__ uint32_t mask_tokens(uint32_t b, int k, int valid) {
    if (k >= valid) return 0u;
    if (k + 1 >= valid) return b & 0x0000ffffu;
    return b;
}

// swizzled byte offset of (row t, 16-byte chunk c) inside a 4 KiB block
__device__ __forceinline__ uint32_t swz(int t, int c) {
    return static_cast<uint32_t>(t * kRowBytes + ((c ^ (t & 7)) << 4));
}

// ------------------------------------------------------- work-item decoding
struct Item {
    int r, head, split, nsplit, g;
    int pb, pe;          // page range [pb, pe) within the request's page list
    int seq;             // tokens attended
    int idx_base;        // page_indptr[r]
};

__device__ __forceinline__ Item decode_item(const Params& p, int k) {
    Item it;
    it.g = k / p.n_kv;
    it.head = k - it.g * p.n_kv;
    const int2 rs = __ldg(p.item_tab + it.g);
    it.r = rs.x;
    it.split = rs.y;
    const int s0 = __ldg(p.split_indptr + it.r);
    it.nsplit = __ldg(p.split_indptr + it.r + 1) - s0;
    it.seq = __ldg(p.seq_lens + it.r);
    it.idx_base = __ldg(p.page_indptr + it.r);
    const int npages = (it.seq + kPage - 1) / kPage;
    const int chunk = (npages + it.nsplit - 1) / it.nsplit;
    it.pb = it.split * chunk;
    it.pe = min(npages, it.pb + chunk);
    if (it.pe < it.pb) it.pe = it.pb;
    return it;
}

// Warp-local cursor over the flattened (item, page) stream of one warp.
struct Cursor {
    int k;      // current item id (>= num_items => done)
    int page;   // absolute page index inside the item range
    Item it;
};

__device__ __forceinline__ void cursor_seek(const Params& p, Cursor& c, int stride) {
    // advance to the first item (from c.k) that has at least one page
    while (c.k < p.num_items) {
        c.it = decode_item(p, c.k);
        if (c.it.pe > c.it.pb) {
            c.page = c.it.pb;
            return;
        }
        c.k += stride;
    }
}

__device__ __forceinline__ void cursor_next(const Params& p, Cursor& c, int stride) {
    if (++c.page >= c.it.pe) {
        c.k += stride;
        cursor_seek(p, c, stride);
    }
}

// ------------------------------------------------------------- epilogues
// Finish one (request, q head) row: o (unnormalised, 4 dims per lane for MHA
// layout), m (log2 units) and l.  Either writes the output directly
// (single split) or publishes a partial and lets the last arrival merge.
struct RowOut {
    float o[4];   // dims 4*lane .. 4*lane+3
};

__device__ __forceinline__ void write_final_row(const Params& p, int r, int qh, int lane, const float* o,
                                                float m, float l) {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint2 w;
    w.x = pack_bf16(o[0] * inv, o[1] * inv);
    w.y = pack_bf16(o[2] * inv, o[3] * inv);
    *reinterpret_cast<uint2*>(p.out + (static_cast<int64_t>(r) * p.n_q + qh) * kD + lane * 4) = w;
    if (p.lse != nullptr && lane == 0) {
        p.lse[static_cast<int64_t>(r) * p.n_q + qh] = l > 0.f ? (m + __log2f(l)) / kLog2e : -INFINITY;
    }
}

// Merge all split partials of (r, qh); every lane owns dims 4*lane..+3.
__device__ __forceinline__ void merge_row(const Params& p, int r, int qh, int lane) {
    const int s0 = __ldg(p.split_indptr + r);
    const int ns = __ldg(p.split_indptr + r + 1) - s0;
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) {
        const float2 ml = __ldcg(p.part_ml + static_cast<int64_t>(s0 + s) * p.n_q + qh);
        M = fmaxf(M, ml.x);
    }
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    float L = 0.f;
    for (int s = 0; s < ns; ++s) {
        const int64_t slot = static_cast<int64_t>(s0 + s) * p.n_q + qh;
        const float2 ml = __ldcg(p.part_ml + slot);
        const float w = (ml.x == -INFINITY) ? 0.f : exp2f(ml.x - M);
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p.part_o + slot * kD) + lane);
        o[0] += w * v.x;
        o[1] += w * v.y;
        o[2] += w * v.z;
        o[3] += w * v.w;
        L += w * ml.y;
    }
    write_final_row(p, r, qh, lane, o, M, L);
}

// Publish one row partial; returns via the caller's semaphore logic.
__device__ __forceinline__ void store_partial_row(const Params& p, int g, int qh, int lane, const float* o,
                                                  float m, float l) {
    const int64_t slot = static_cast<int64_t>(g) * p.n_q + qh;
    __stcg(reinterpret_cast<float4*>(p.part_o + slot * kD) + lane, make_float4(o[0], o[1], o[2], o[3]));
    if (lane == 0) __stcg(p.part_ml + slot, make_float2(m, l));
}

// After all rows of an item are published: bump the (r, kv head) semaphore and
// return true on the last arrival (which then merges).
__device__ __forceinline__ bool arrive_last(const Params& p, const Item& it, int lane) {
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) {
        int32_t* s = p.sem + static_cast<int64_t>(it.r) * p.n_kv + it.head;
        const int prev = atomicAdd(s, 1);
        last = (prev == it.nsplit - 1);
        if (last) *s = 0;  // re-arm for the next launch (stream-ordered)
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) __threadfence();
    return last != 0;
}

// KV append (K3): the owner of the last split writes token row `seq` of
// (layer, head).  Lanes 0-15: K row, 16-31: V row; 16 bytes each, swizzled.
__device__ __forceinline__ void append_row(const Params& p, const Item& it, int lane) {
    if (p.k_new == nullptr || it.split != it.nsplit - 1) return;
    const int pos = it.seq;
    const int pidx = pos / kPage;
    const int npl = __ldg(p.page_indptr + it.r + 1) - it.idx_base;
    if (pidx >= npl) return;  // host did not provision the append page
    const int t = pos % kPage;
    const int64_t phys = __ldg(p.page_indices + it.idx_base + pidx);
    const int c = lane & 15;
    const bool is_v = lane >= 16;
    const __nv_bfloat16* src = (is_v ? p.v_new : p.k_new) +
                               (static_cast<int64_t>(it.r) * p.n_kv + it.head) * kD + c * 8;
    char* dst = p.pool_w + phys * p.page_bytes + p.layer_off + (is_v ? p.v_off : 0) +
                static_cast<int64_t>(it.head) * kBlockBytes + swz(t, c);
    *reinterpret_cast<uint4*>(dst) = __ldg(reinterpret_cast<const uint4*>(src));
}

// ============================================================ the kernel
template <int NW, int S, int GROUP>
__global__ void __launch_bounds__(NW * 32)
decode_attn_kernel(const Params p) {
    extern __shared__ __align__(1024) char smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // per-warp region: S stages (8 KiB each) + S mbarriers + scratch
    constexpr int kWarpBytes = S * kStageBytes + 128;
    char* wbase = smem_raw + warp * kWarpBytes;
    const uint32_t stage0 = smem_u32(wbase);
    const uint32_t bar0 = smem_u32(wbase + S * kStageBytes);
    char* scratch = wbase + S * kStageBytes + 64;  // 64 bytes

    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    const int stride = gridDim.x * NW;            // total persistent warps
    const int wid = blockIdx.x * NW + warp;       // this warp's worker id
    const uint64_t pol = evict_first_policy();

    // producer cursor (only lane 0 issues, but all lanes track it uniformly)
    Cursor pc;
    pc.k = wid;
    cursor_seek(p, pc, stride);

    auto issue = [&](int slot) {
        if (lane == 0) {
            const int64_t phys = __ldg(p.page_indices + pc.it.idx_base + pc.page);
            const char* kblk = p.pool + phys * p.page_bytes + p.layer_off +
                               static_cast<int64_t>(pc.it.head) * kBlockBytes;
            const uint32_t bar = bar0 + 8 * slot;
            const uint32_t dst = stage0 + slot * kStageBytes;
            mbar_expect_tx(bar, kStageBytes);
            bulk_g2s(dst, kblk, kBlockBytes, bar, pol);
            bulk_g2s(dst + kBlockBytes, kblk + p.v_off, kBlockBytes, bar, pol);
        }
        cursor_next(p, pc, stride);
    };

    // prologue: fill the ring
    int issued = 0;
#pragma unroll 1
    for (; issued < S && pc.k < p.num_items; ++issued) issue(issued);

    Cursor cc;  // consumer cursor
    cc.k = wid;
    cursor_seek(p, cc, stride);
    int consumed = 0;

    if constexpr (GROUP == 1) {
        // ---------------------------------------------------------- MHA / FHFMA
        const int t = lane & 15;      // token row for QK
        const int half = lane >> 4;   // which 64-dim half of the row
        uint32_t qreg[32];            // this lane's 64 q dims (bf16x2)
        float m = -INFINITY, l = 0.f;
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        int cur_k = -1;
#pragma unroll 1
        while (cc.k < p.num_items) {
            const Item& it = cc.it;
            if (cc.k != cur_k) {
                // new item: load q, reset state, append the step's KV row
                cur_k = cc.k;
                const uint4* qs = reinterpret_cast<const uint4*>(
                    p.q + (static_cast<int64_t>(it.r) * p.n_q + it.head) * kD + half * 64);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint4 v = __ldg(qs + j);
                    qreg[4 * j + 0] = v.x;
                    qreg[4 * j + 1] = v.y;
                    qreg[4 * j + 2] = v.z;
                    qreg[4 * j + 3] = v.w;
                }
                m = -INFINITY;
                l = 0.f;
                o[0] = o[1] = o[2] = o[3] = 0.f;
                append_row(p, it, lane);
            }
            const int slot = consumed % S;
            const uint32_t phase = (consumed / S) & 1;
            mbar_wait(bar0 + 8 * slot, phase);
            const uint32_t ks = stage0 + slot * kStageBytes;
            const uint32_t vs = ks + kBlockBytes;
            const int valid = min(kPage, it.seq - cc.page * kPage);

            // ---- scores: lane (t, half) dots its 64 dims, then combine halves
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint4 kv = lds128(ks + swz(t, half * 8 + j));
                a0 = fma_bf<0, 0>(kv.x, qreg[4 * j + 0], a0);
                a1 = fma_bf<1, 1>(kv.x, qreg[4 * j + 0], a1);
                a2 = fma_bf<0, 0>(kv.y, qreg[4 * j + 1], a2);
                a3 = fma_bf<1, 1>(kv.y, qreg[4 * j + 1], a3);
                a0 = fma_bf<0, 0>(kv.z, qreg[4 * j + 2], a0);
                a1 = fma_bf<1, 1>(kv.z, qreg[4 * j + 2], a1);
                a2 = fma_bf<0, 0>(kv.w, qreg[4 * j + 3], a2);
                a3 = fma_bf<1, 1>(kv.w, qreg[4 * j + 3], a3);
            }
            float s = (a0 + a1) + (a2 + a3);
            s += __shfl_xor_sync(0xffffffffu, s, 16);
            s = (t < valid) ? s * p.scale_log2 : -INFINITY;
            // ---- online softmax (warp-uniform running max)
            float mx = s;
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            const float m_new = fmaxf(m, mx);
            const float alpha = exp2f(m - m_new);  // m=-inf -> 0
            m = m_new;
            const float pf = exp2f(s - m_new);     // masked rows -> 0
            // P is rounded to bf16 for the PV product (FA2/FA3 convention); l sums
            // the rounded weights so O/l stays an exact convex combination.
            const __nv_bfloat16 pb = __float2bfloat16_rn(pf);
            l = l * alpha + ((half == 0) ? __bfloat162float(pb) : 0.f);
            o[0] *= alpha;
            o[1] *= alpha;
            o[2] *= alpha;
            o[3] *= alpha;
            if (half == 0) reinterpret_cast<__nv_bfloat16*>(scratch)[t] = pb;
            __syncwarp();
            const uint32_t sp = smem_u32(scratch);
            const uint4 p0 = lds128(sp);
            const uint4 p1 = lds128(sp + 16);
            const uint32_t pw[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
            // ---- PV: lane owns dims 4*lane .. 4*lane+3
            const int cidx = lane >> 1;           // 16-byte chunk holding the dims
            const uint32_t coff = (lane & 1) * 8; // 8-byte half inside the chunk
            if (valid == kPage) {
#pragma unroll
                for (int tt = 0; tt < kPage; tt += 2) {
                    const uint2 v0 = lds64(vs + swz(tt, cidx) + coff);
                    const uint2 v1 = lds64(vs + swz(tt + 1, cidx) + coff);
                    const uint32_t pp = pw[tt >> 1];
                    o[0] = fma_bf<0, 0>(v0.x, pp, o[0]);
                    o[1] = fma_bf<1, 0>(v0.x, pp, o[1]);
                    o[2] = fma_bf<0, 0>(v0.y, pp, o[2]);
                    o[3] = fma_bf<1, 0>(v0.y, pp, o[3]);
                    o[0] = fma_bf<0, 1>(v1.x, pp, o[0]);
                    o[1] = fma_bf<1, 1>(v1.x, pp, o[1]);
                    o[2] = fma_bf<0, 1>(v1.y, pp, o[2]);
                    o[3] = fma_bf<1, 1>(v1.y, pp, o[3]);
                }
            } else {
                // partial last page: never touch rows >= valid (may be stale)
#pragma unroll
                for (int tt = 0; tt < kPage; tt += 2) {
                    uint2 v0 = lds64(vs + swz(tt, cidx) + coff);
                    uint2 v1 = lds64(vs + swz(tt + 1, cidx) + coff);
                    if (tt >= valid) v0 = make_uint2(0u, 0u);
                    if (tt + 1 >= valid) v1 = make_uint2(0u, 0u);
                    const uint32_t pp = pw[tt >> 1];
                    o[0] = fma_bf<0, 0>(v0.x, pp, o[0]);
                    o[1] = fma_bf<1, 0>(v0.x, pp, o[1]);
                    o[2] = fma_bf<0, 0>(v0.y, pp, o[2]);
                    o[3] = fma_bf<1, 0>(v0.y, pp, o[3]);
                    o[0] = fma_bf<0, 1>(v1.x, pp, o[0]);
                    o[1] = fma_bf<1, 1>(v1.x, pp, o[1]);
                    o[2] = fma_bf<0, 1>(v1.y, pp, o[2]);
                    o[3] = fma_bf<1, 1>(v1.y, pp, o[3]);
                }
            }
            __syncwarp();
            ++consumed;
            // refill the slot we just drained
            if (pc.k < p.num_items) {
                fence_proxy_async();
                issue(slot);
                ++issued;
            }
            const bool item_end = (cc.page + 1 >= it.pe);
            if (item_end) {
                // finalize the (request, head) row of this item
                float lt = l;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, off);
                if (it.nsplit == 1) {
                    write_final_row(p, it.r, it.head, lane, o, m, lt);
                } else {
                    store_partial_row(p, it.g, it.head, lane, o, m, lt);
                    if (arrive_last(p, it, lane)) merge_row(p, it.r, it.head, lane);
                }
            }
            cursor_next(p, cc, stride);
        }
    } else {
        // -------------------------------------------------- GQA / mma.sync
        // rows of the m16 tile = the GROUP query heads of this kv head (padded)
        const int qrow = lane >> 2;          // A/C fragment row owned (0..7)
        const int qcol = (lane & 3) * 2;     // fragment column pair
        uint32_t qa[8][2];                   // A fragments (rows 0-7) for 8 k-steps
        float oacc[16][2];                   // C rows 0-7, 16 n-tiles of 8 dims
        float m = -INFINITY, l = 0.f;
        int cur_k = -1;
#pragma unroll 1
        while (cc.k < p.num_items) {
            const Item& it = cc.it;
            if (cc.k != cur_k) {
                cur_k = cc.k;
                const int qh = it.head * GROUP + qrow;
                const bool rv = qrow < GROUP;
                const __nv_bfloat16* qsrc = p.q + (static_cast<int64_t>(it.r) * p.n_q + qh) * kD;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    qa[ks][0] = rv ? __ldg(reinterpret_cast<const uint32_t*>(qsrc + ks * 16 + qcol)) : 0u;
                    qa[ks][1] = rv ? __ldg(reinterpret_cast<const uint32_t*>(qsrc + ks * 16 + 8 + qcol)) : 0u;
                }
#pragma unroll
                for (int nt = 0; nt < 16; ++nt) oacc[nt][0] = oacc[nt][1] = 0.f;
                m = -INFINITY;
                l = 0.f;
                append_row(p, it, lane);
            }
            const int slot = consumed % S;
            const uint32_t phase = (consumed / S) & 1;
            mbar_wait(bar0 + 8 * slot, phase);
            const uint32_t ks_base = stage0 + slot * kStageBytes;
            const uint32_t vs_base = ks_base + kBlockBytes;
            const int valid = min(kPage, it.seq - cc.page * kPage);

            // ---- S = Q K^T : two n-tiles of 8 tokens, 8 k-steps of 16 dims
            float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int trow = nt * 8 + (lane & 7);
#pragma unroll
                for (int kk = 0; kk < 8; kk += 2) {
                    // matrices: chunks 2kk, 2kk+1, 2kk+2, 2kk+3 of rows trow
                    const int chunk = 2 * kk + (lane >> 3);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(ks_base + swz(trow, chunk), b0, b1, b2, b3);
                    mma_bf16(sacc[nt], qa[kk][0], 0u, qa[kk][1], 0u, b0, b1);
                    mma_bf16(sacc[nt], qa[kk + 1][0], 0u, qa[kk + 1][1], 0u, b2, b3);
                }
            }
            // lane holds S[row=qrow][tokens nt*8 + qcol, +1] in sacc[nt][0..1]
            float sv[4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int tok = nt * 8 + qcol + e;
                    sv[nt * 2 + e] = (tok < valid) ? sacc[nt][e] * p.scale_log2 : -INFINITY;
                }
            }
            float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m, mx);
            const float alpha = exp2f(m - m_new);
            m = m_new;
            uint32_t pa[2];
            float psum = 0.f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const float e0 = exp2f(sv[nt * 2] - m_new);
                const float e1 = exp2f(sv[nt * 2 + 1] - m_new);
                pa[nt] = pack_bf16(e0, e1);
                psum += bf16_lo(pa[nt]) + bf16_hi(pa[nt]);
            }
            l = l * alpha + psum;
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) {
                oacc[nt][0] *= alpha;
                oacc[nt][1] *= alpha;
            }
            // ---- O += P V : A = P (k = 16 tokens), B = V tile via ldmatrix.trans
            // rows >= valid of V must not leak NaN/Inf: P is 0 there, but 0*Inf = NaN,
            // so for partial pages re-zero the stale rows' contribution by masking B.
#pragma unroll
            for (int dn = 0; dn < 16; dn += 2) {
                // matrices: (tokens 0-7, dims 8dn..), (tokens 8-15, dims 8dn..),
                //           (tokens 0-7, dims 8dn+8..), (tokens 8-15, dims 8dn+8..)
                const int trow = (lane & 7) + ((lane >> 3) & 1) * 8;
                const int chunk = dn + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vs_base + swz(trow, chunk), b0, b1, b2, b3);
                if (valid < kPage) {
                    // lane holds B[k = tokens qcol, qcol+1 (b0,b2) / +8 (b1,b3)][n]
                    b0 = mask_tokens(b0, qcol, valid);
                    b2 = mask_tokens(b2, qcol, valid);
                    b1 = mask_tokens(b1, qcol + 8, valid);
                    b3 = mask_tokens(b3, qcol + 8, valid);
                }
                float c0[4] = {oacc[dn][0], oacc[dn][1], 0.f, 0.f};
                float c1[4] = {oacc[dn + 1][0], oacc[dn + 1][1], 0.f, 0.f};
                mma_bf16(c0, pa[0], 0u, pa[1], 0u, b0, b1);
                mma_bf16(c1, pa[0], 0u, pa[1], 0u, b2, b3);
                oacc[dn][0] = c0[0];
                oacc[dn][1] = c0[1];
                oacc[dn + 1][0] = c1[0];
                oacc[dn + 1][1] = c1[1];
            }
            __syncwarp();
            ++consumed;
            if (pc.k < p.num_items) {
                fence_proxy_async();
                issue(slot);
                ++issued;
            }
            const bool item_end = (cc.page + 1 >= it.pe);
            if (item_end) {
                float lt = l;
                lt += __shfl_xor_sync(0xffffffffu, lt, 1);
                lt += __shfl_xor_sync(0xffffffffu, lt, 2);
                // lane holds O[row qrow][dims 8nt + qcol, +1]; stage through the
                // (drained) scratch-free path: write rows directly.
                const bool rv = qrow < GROUP;
                const int qh = it.head * GROUP + qrow;
                if (it.nsplit == 1) {
                    if (rv) {
                        const float inv = lt > 0.f ? 1.f / lt : 0.f;
                        __nv_bfloat16* dst = p.out + (static_cast<int64_t>(it.r) * p.n_q + qh) * kD;
#pragma unroll
                        for (int nt = 0; nt < 16; ++nt) {
                            *reinterpret_cast<uint32_t*>(dst + nt * 8 + qcol) =
                                pack_bf16(oacc[nt][0] * inv, oacc[nt][1] * inv);
                        }
                        if (p.lse != nullptr && (lane & 3) == 0) {
                            p.lse[static_cast<int64_t>(it.r) * p.n_q + qh] =
                                lt > 0.f ? (m + __log2f(lt)) / kLog2e : -INFINITY;
                        }
                    }
                } else {
                    if (rv) {
                        const int64_t slotp = static_cast<int64_t>(it.g) * p.n_q + qh;
                        float* dst = p.part_o + slotp * kD;
#pragma unroll
                        for (int nt = 0; nt < 16; ++nt) {
                            __stcg(reinterpret_cast<float2*>(dst + nt * 8 + qcol),
                                   make_float2(oacc[nt][0], oacc[nt][1]));
                        }
                        if ((lane & 3) == 0) __stcg(p.part_ml + slotp, make_float2(m, lt));
                    }
                    if (arrive_last(p, it, lane)) {
                        for (int gh = 0; gh < GROUP; ++gh) merge_row(p, it.r, it.head * GROUP + gh, lane);
                    }
                }
            }
            cursor_next(p, cc, stride);
        }
    }
}

// ------------------------------------------------------------- launcher
template <int NW, int S, int GROUP>
struct Launch {
    static constexpr int kSmem = NW * (S * kStageBytes + 128);
    static cudaError_t configure() {
        return cudaFuncSetAttribute(decode_attn_kernel<NW, S, GROUP>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    }
    static cudaError_t occupancy(int* blocks) {
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, decode_attn_kernel<NW, S, GROUP>,
                                                             NW * 32, kSmem);
    }
    static cudaError_t run(const Params& p, int grid, cudaStream_t st) {
        decode_attn_kernel<NW, S, GROUP><<<grid, NW * 32, kSmem, st>>>(p);
        return cudaGetLastError();
    }
};

constexpr int kNW = 4;
constexpr int kStages = 3;

template <int GROUP>
cudaError_t dispatch_group(bool query, int* blocks, const Params* p, int grid, cudaStream_t st) {
    using L = Launch<kNW, kStages, GROUP>;
    static bool configured = false;  // attribute set is idempotent; racing is harmless
    if (!configured) {
        cudaError_t e = L::configure();
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (query) return L::occupancy(blocks);
    return L::run(*p, grid, st);
}

cudaError_t dispatch(int group, bool query, int* blocks, const Params* p, int grid, cudaStream_t st) {
    switch (group) {
        case 1: return dispatch_group<1>(query, blocks, p, grid, st);
        case 2: return dispatch_group<2>(query, blocks, p, grid, st);
        case 4: return dispatch_group<4>(query, blocks, p, grid, st);
        case 5: return dispatch_group<5>(query, blocks, p, grid, st);
        case 8: return dispatch_group<8>(query, blocks, p, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

int attn_warps_per_cta() { return kNW; }

cudaError_t attn_occupancy(int group, int* blocks_per_sm) {
    return dispatch(group, true, blocks_per_sm, nullptr, 0, nullptr);
}

cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t st) {
    Params p;
    p.q = static_cast<const __nv_bfloat16*>(a.q);
    p.pool = static_cast<const char*>(a.pool);
    p.pool_w = static_cast<char*>(a.pool);
    p.page_bytes = a.page_bytes;
    p.layer_off = a.layer_off;
    p.v_off = a.v_off;
    p.seq_lens = a.seq_lens;
    p.page_indptr = a.page_indptr;
    p.page_indices = a.page_indices;
    p.split_indptr = a.split_indptr;
    p.item_tab = reinterpret_cast<const int2*>(a.item_tab);
    p.num_items = a.num_items;
    p.n_kv = a.n_kv;
    p.n_q = a.n_q;
    p.k_new = static_cast<const __nv_bfloat16*>(a.k_new);
    p.v_new = static_cast<const __nv_bfloat16*>(a.v_new);
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.lse = a.lse;
    p.part_o = a.part_o;
    p.part_ml = reinterpret_cast<float2*>(a.part_ml);
    p.sem = a.sem;
    p.scale_log2 = a.sm_scale * kLog2e;
    if (p.num_items <= 0) return cudaSuccess;
    return dispatch(a.group, false, nullptr, &p, a.grid, st);
}

}  // namespace asv
