// KV page moves between the pinned host pool (page-major pages) and layer-major
// device page pools (include/asv.h): C1 host -> prefetch GPU, C2/C3 prefetch
// <-> decode GPU.  Replace the PRICED transfers of the reference
// (transfer_time, cluster_sim.hpp:60-66; start_async_transfer / sync_transfer
// :220-232) with copy-engine work.  A request with s tokens moves floor(s/16)
// whole pages (one 2-D copy each: L slices at its page group's < 2 GiB layer
// pitch) and the s%16 valid rows of its last page (one 3-D copy: rows x blocks
// x layers) — exactly s * kv_bytes_per_token bytes (cluster_sim.hpp:239-241).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "../../include/asv.h"
#include "asv_internal.h"

namespace asv {
namespace {

constexpr int64_t kBlock = 4096;

struct Geo {
    int64_t slice;  // one layer of one page
    int64_t bps;    // 4 KiB blocks per slice
    int64_t layers;
    int64_t page_bytes;
};

int geo(const asv_attn_shape* s, Geo* g) {
    const int64_t pb = asv_page_bytes(s);
    if (pb <= 0) return fail(ASV_ERR_INVALID, asv_last_error());
    g->bps = 2 * static_cast<int64_t>(s->num_kv_heads);
    g->slice = g->bps * kBlock;
    g->layers = s->num_layers;
    g->page_bytes = pb;
    return ASV_OK;
}

cudaPitchedPtr pitched(const void* base, int64_t rows_per_layer) {
    return make_cudaPitchedPtr(const_cast<void*>(base), kBlock, kBlock, static_cast<size_t>(rows_per_layer));
}

// A layer-major pool in page groups (asv_internal.h): page p's layer-0 slice,
// the layer pitch of its group, and its group's base (3-D views of a group).
struct PoolView {
    char* base;
    int64_t group_pages, layers, slice;
    PoolView(const void* b, int64_t pool_pages, const Geo& g)
        : base(static_cast<char*>(const_cast<void*>(b))),
          group_pages(pool_group_pages(g.slice, pool_pages)),
          layers(g.layers),
          slice(g.slice) {}
    char* page0(int32_t p) const { return base + pool_slot(p, group_pages, layers) * slice; }
    size_t pitch() const { return static_cast<size_t>(group_pages * slice); }
    char* group_base(int32_t p) const { return base + (p / group_pages) * group_pages * layers * slice; }
    int64_t in_group(int32_t p) const { return p % group_pages; }
};

int check_pages(const int32_t* pages, int64_t n, int64_t pool_pages, const Geo& g) {
    const int64_t usable = pool_usable_pages(g.slice, pool_pages);
    for (int64_t j = 0; j < n; ++j) {
        if (pages[j] < 0 || pages[j] >= usable) {
            return fail(ASV_ERR_INVALID, "kv copy: page id " + std::to_string(pages[j]) + " outside the usable pool (" +
                                             std::to_string(usable) + " pages)");
        }
    }
    return ASV_OK;
}

// host <-> device, `to_device` selects the direction
int host_device(const asv_attn_shape* shape, void* pool, int64_t pool_pages, const int32_t* pages, int64_t tokens,
                void* const* host_pages, bool to_device, cudaStream_t st, int64_t* bytes_out) {
    Geo g;
    if (int rc = geo(shape, &g)) return rc;
    if (pool == nullptr || pages == nullptr || host_pages == nullptr || tokens < 0 || pool_pages < 1)
        return fail(ASV_ERR_INVALID, "bad kv copy arguments");
    const int64_t full = tokens / 16, rows = tokens % 16;
    if (int rc = check_pages(pages, (tokens + 15) / 16, pool_pages, g)) return rc;
    const PoolView pv(pool, pool_pages, g);
    const size_t dpitch = pv.pitch();
    const cudaMemcpyKind kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    int64_t moved = 0;
    for (int64_t j = 0; j < full; ++j) {
        char* d = pv.page0(pages[j]);
        char* h = static_cast<char*>(host_pages[j]);
        cudaError_t e = to_device ? cudaMemcpy2DAsync(d, dpitch, h, g.slice, g.slice, g.layers, kind, st)
                                  : cudaMemcpy2DAsync(h, g.slice, d, dpitch, g.slice, g.layers, kind, st);
        if (e != cudaSuccess) return cuda_fail(e, "kv page copy");
        moved += g.page_bytes;
    }
    if (rows > 0) {
        cudaMemcpy3DParms m = {};
        const cudaPitchedPtr dev = pitched(pv.group_base(pages[full]), pv.group_pages * g.bps);
        const cudaPitchedPtr host = pitched(host_pages[full], g.bps);
        const cudaPos dpos = make_cudaPos(0, static_cast<size_t>(pv.in_group(pages[full]) * g.bps), 0);
        m.srcPtr = to_device ? host : dev;
        m.dstPtr = to_device ? dev : host;
        m.srcPos = to_device ? make_cudaPos(0, 0, 0) : dpos;
        m.dstPos = to_device ? dpos : make_cudaPos(0, 0, 0);
        m.extent = make_cudaExtent(static_cast<size_t>(rows) * 256, static_cast<size_t>(g.bps),
                                   static_cast<size_t>(g.layers));
        m.kind = kind;
        cudaError_t e = cudaMemcpy3DAsync(&m, st);
        if (e != cudaSuccess) return cuda_fail(e, "kv partial page copy");
        moved += rows * 256 * g.bps * g.layers;
    }
    if (bytes_out) *bytes_out = moved;
    return ASV_OK;
}

}  // namespace
}  // namespace asv

using namespace asv;

extern "C" {

int asv_kv_copy_h2d(const asv_attn_shape* shape, void* pool, int64_t pool_pages, const int32_t* pages,
                    int64_t tokens, const void* const* host_pages, void* stream, int64_t* bytes_out) {
    return host_device(shape, pool, pool_pages, pages, tokens, const_cast<void* const*>(host_pages), true,
                       static_cast<cudaStream_t>(stream), bytes_out);
}

int asv_kv_copy_d2h(const asv_attn_shape* shape, const void* pool, int64_t pool_pages, const int32_t* pages,
                    int64_t tokens, void* const* host_pages, void* stream, int64_t* bytes_out) {
    return host_device(shape, const_cast<void*>(pool), pool_pages, pages, tokens, host_pages, false,
                       static_cast<cudaStream_t>(stream), bytes_out);
}

int asv_kv_copy_d2d(const asv_attn_shape* shape, void* dst_pool, int64_t dst_pool_pages, int32_t dst_device,
                    const int32_t* dst_pages, const void* src_pool, int64_t src_pool_pages, int32_t src_device,
                    const int32_t* src_pages, int64_t tokens, void* stream, int64_t* bytes_out) {
    Geo g;
    if (int rc = geo(shape, &g)) return rc;
    if (dst_pool == nullptr || src_pool == nullptr || dst_pages == nullptr || src_pages == nullptr || tokens < 0 ||
        dst_pool_pages < 1 || src_pool_pages < 1)
        return fail(ASV_ERR_INVALID, "bad kv copy arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t full = tokens / 16, rows = tokens % 16;
    const int64_t npg = (tokens + 15) / 16;
    if (int rc = check_pages(dst_pages, npg, dst_pool_pages, g)) return rc;
    if (int rc = check_pages(src_pages, npg, src_pool_pages, g)) return rc;
    const PoolView dv(dst_pool, dst_pool_pages, g), sv(src_pool, src_pool_pages, g);
    // SM gather/scatter kernel (kv_move.cu): one launch per request; across a pair it pulls over
    // NVLink through peer pointers.  ASV_D2D_COPY_ENGINE=1 selects per-page copy-engine copies.
    static const bool copy_engine = [] {
        const char* e = getenv("ASV_D2D_COPY_ENGINE");
        return e != nullptr && atoi(e) != 0;
    }();
    if (!copy_engine) {
        if (tokens > 0) {
            cudaError_t e = kv_move_launch(src_pool, sv.group_pages, dst_pool, dv.group_pages, g.slice,
                                           static_cast<int32_t>(g.layers), src_pages, dst_pages, tokens, st);
            if (e != cudaSuccess) return cuda_fail(e, "kv page move");
        }
        if (bytes_out) *bytes_out = tokens * g.bps * 256 * g.layers;
        return ASV_OK;
    }
    const size_t dp = dv.pitch(), sp = sv.pitch();
    int64_t moved = 0;
    for (int64_t j = 0; j < full; ++j) {
        cudaError_t e = cudaMemcpy2DAsync(dv.page0(dst_pages[j]), dp, sv.page0(src_pages[j]), sp, g.slice, g.layers,
                                          cudaMemcpyDefault, st);
        if (e != cudaSuccess) return cuda_fail(e, "kv peer page copy");
        moved += g.page_bytes;
    }
    if (rows > 0) {
        const cudaExtent ext = make_cudaExtent(static_cast<size_t>(rows) * 256, static_cast<size_t>(g.bps),
                                               static_cast<size_t>(g.layers));
        const cudaPitchedPtr d = pitched(dv.group_base(dst_pages[full]), dv.group_pages * g.bps);
        const cudaPitchedPtr s = pitched(sv.group_base(src_pages[full]), sv.group_pages * g.bps);
        const cudaPos dpos = make_cudaPos(0, static_cast<size_t>(dv.in_group(dst_pages[full]) * g.bps), 0);
        const cudaPos spos = make_cudaPos(0, static_cast<size_t>(sv.in_group(src_pages[full]) * g.bps), 0);
        cudaError_t e;
        if (dst_device != src_device) {
            cudaMemcpy3DPeerParms m = {};
            m.dstPtr = d;
            m.dstPos = dpos;
            m.dstDevice = dst_device;
            m.srcPtr = s;
            m.srcPos = spos;
            m.srcDevice = src_device;
            m.extent = ext;
            e = cudaMemcpy3DPeerAsync(&m, st);
        } else {
            cudaMemcpy3DParms m = {};
            m.dstPtr = d;
            m.dstPos = dpos;
            m.srcPtr = s;
            m.srcPos = spos;
            m.extent = ext;
            m.kind = cudaMemcpyDeviceToDevice;
            e = cudaMemcpy3DAsync(&m, st);
        }
        if (e != cudaSuccess) return cuda_fail(e, "kv peer partial page copy");
        moved += rows * 256 * g.bps * g.layers;
    }
    if (bytes_out) *bytes_out = moved;
    return ASV_OK;
}

}  // extern "C"
