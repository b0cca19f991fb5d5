/*
 * asv.h — C ABI of the B200-native AlignedServe decode-iteration hot path.
 *
 * The reference (`/root/reference/proj`, header-only C++20 `prefixsim`) never
 * executes the decode iteration: it PRICES it.  Each entry point below is the
 * executed replacement of one priced/modeled function on that path; the C++
 * API the reference's callers see (namespace `prefixsim`, same headers, same
 * signatures) is kept verbatim in paper_2605_23389_b200/include/prefixsim/ and
 * sits on top of this ABI (see INTEGRATION.md for the binding).
 *
 * Conventions: plain pointers and sizes, no C++ or torch types; every entry
 * returns 0 on success or an ASV_ERR_* code; the message of the last failure
 * on the calling thread is available from asv_last_error().  CUDA streams are
 * passed as `void*` (cudaStream_t).  The ABI never allocates on the hot path:
 * device buffers (KV page pool, plan, workspace, outputs) belong to the caller.
 */
#ifndef ASV_H_
#define ASV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes; the C++ wrapper rethrows the reference's exception types */
#define ASV_OK 0
#define ASV_ERR_INVALID 1 /* std::invalid_argument (e.g. "empty batch", cost_model.hpp:114) */
#define ASV_ERR_RUNTIME 2 /* std::runtime_error ("unschedulable: zero-capacity HBM", scheduler.hpp:155) */
#define ASV_ERR_LOGIC 3   /* std::logic_error (engine invariants, cluster_sim.hpp:641-697) */
#define ASV_ERR_CUDA 4    /* CUDA runtime failure (no counterpart: the reference has no GPU) */

const char* asv_last_error(void);
int asv_abi_version(void);
/* sizeof() of a boundary struct by name ("asv_attn_shape", "asv_attn_plan", "asv_attn_args",
 * "asv_linear_args", "asv_engine_opts", "asv_engine_stats"); -1 for an unknown name.  Lets a
 * binding (ctypes / cgo / N-API) check its struct mirrors against the compiled library. */
int64_t asv_struct_size(const char* name);

/* ------------------------------------------------------------------------ */
/* Paged KV layout.  A page holds 16 tokens (= ClusterConfig::block_size,     */
/* cluster_sim.hpp:45) of every layer, K and V, every kv head.                */
/*  * device pool (HBM), LAYER-MAJOR in page groups: group g holds pages      */
/*    [g*G, (g+1)*G) as [num_layers][G][2 (K,V)][num_kv_heads][16][128], with  */
/*    G = asv_pool_group_pages() chosen so the layer pitch G * slice stays     */
/*    below 2 GiB (the copy engines' full-rate 2-D pitch; measured).  A pool  */
/*    that fits one group is plain [num_layers][pool_pages][...], so one      */
/*    layer's slices of all pages are dense per decode launch.  Page ids must  */
/*    be < asv_pool_usable_pages() (= groups * G, at most groups-1 fewer).     */
/*  * host pool / transfer format, PAGE-MAJOR: one page is                      */
/*      [num_layers][2][num_kv_heads][16][128] contiguous (asv_page_bytes).    */
/* Every (page, layer, K|V, head) block is 4 KiB, bf16, and XOR-swizzled: the  */
/* 16-byte chunk c of token row t is stored at chunk position c ^ (t & 7), so */
/* a 1-D bulk TMA of the block lands bank-conflict-free in shared memory for  */
/* both the FFMA (MHA) and ldmatrix/mma (GQA) consumers.  KV moves are strided */
/* byte copies (one 2-D copy per page, a 3-D copy for the valid rows of a     */
/* partial last page): bytes moved = s * kv_bytes_per_token                    */
/* (cost_model.hpp:34-36, cluster_sim.hpp:239-241).                            */
/* ------------------------------------------------------------------------ */
typedef struct asv_attn_shape {
    int32_t num_q_heads;  /* n_h */
    int32_t num_kv_heads; /* n_kv; n_h % n_kv == 0, group n_h/n_kv <= 8 */
    int32_t head_dim;     /* must be 128 */
    int32_t page_size;    /* must be 16 */
    int32_t num_layers;   /* L (layers resident per page) */
} asv_attn_shape;

/* bytes of one page (all layers, K and V) */
int64_t asv_page_bytes(const asv_attn_shape* shape);
/* byte offset of element (layer, kv, head, token, dim) inside one PAGE-MAJOR (host) page */
int64_t asv_page_offset(const asv_attn_shape* shape, int32_t layer, int32_t kv, int32_t head,
                        int32_t token, int32_t dim);
/* byte offset of element (page, layer, kv, head, token, dim) in a LAYER-MAJOR device pool */
int64_t asv_pool_offset(const asv_attn_shape* shape, int64_t pool_pages, int64_t page, int32_t layer,
                        int32_t kv, int32_t head, int32_t token, int32_t dim);
/* pages per layer-major group G of a pool of `pool_pages` pages (-1 on bad arguments) */
int64_t asv_pool_group_pages(const asv_attn_shape* shape, int64_t pool_pages);
/* page ids valid in such a pool: [0, groups * G) */
int64_t asv_pool_usable_pages(const asv_attn_shape* shape, int64_t pool_pages);

/* ------------------------------------------------------------------------ */
/* Split-KV work plan (host side, K4 in SURVEY §2).  Built once per decode    */
/* iteration from the batch in `SchedulerState::running` order                */
/* (scheduler.hpp:59; cluster_sim.hpp:476-478) and uploaded as ONE int32      */
/* buffer; reused by every layer of that iteration.                          */
/* ------------------------------------------------------------------------ */
typedef struct asv_attn_plan {
    int32_t batch;          /* b */
    int32_t total_splits;   /* G: sum over requests of their split counts */
    int32_t num_items;      /* G * num_kv_heads warp work items */
    int32_t num_pages;      /* P = page_indptr[batch] */
    int32_t num_workers;    /* persistent warps the plan was balanced for */
    int32_t off_desc;       /* int32 offset of the G split descriptors (40 words each,
                               sorted longest first: the dynamic schedule is LPT) */
    int32_t off_split_base; /* int32 offset of split_base[b+1] (partial slots per request) */
    int32_t off_merge;      /* int32 offset of the requests split more than once */
    int32_t n_merge;        /* their count (rows of the merge kernel = n_merge * n_h) */
    int32_t total_int32;    /* size of the plan buffer in int32 */
    int32_t max_item_pages; /* largest work item, pages (<= 32) */
    int32_t append_missing; /* requests whose page list does not cover position seq_len: a launch
                               with k_new / v_new set is rejected (ASV_ERR_INVALID) instead of
                               silently dropping their appended row */
} asv_attn_plan;

/* Persistent warp count of the decode-attention kernel on `device` (SMs x resident warps). */
int asv_attn_num_workers(const asv_attn_shape* shape, int device, int32_t* workers_out);

/* Fill `plan_buf` (host, capacity `plan_cap` int32) for a batch.
 *   seq_lens[b]        tokens attended per request (= prefix_len, >= 1)
 *   page_indptr[b+1]   CSR over page_indices; request i owns
 *                      page_indices[page_indptr[i] .. page_indptr[i+1]) which must cover
 *                      ceil((seq_lens[i]+1)/16) pages when a KV append is requested
 *   page_indices[P]    physical page ids in the device pool
 * The split count per request is chosen so every warp streams a near-equal KV span. */
int asv_attn_plan_build(const asv_attn_shape* shape, int32_t batch, const int32_t* seq_lens,
                        const int32_t* page_indptr, const int32_t* page_indices,
                        int32_t num_workers, int32_t* plan_buf, int64_t plan_cap,
                        asv_attn_plan* plan_out);

/* Upload a plan buffer from MAPPED pinned host memory (cudaHostAllocMapped) into
 * device memory with SM loads over PCIe (one small kernel on `stream`), not with
 * a copy-engine memcpy: a plan upload issued on the compute stream must never
 * queue behind multi-GB KV prefetches on the shared host-to-device copy engine
 * (measured: a cudaMemcpyAsync plan upload serialised every decode iteration
 * behind the batch prefetch in flight).  `host_plan` must be readable for
 * n_int32 rounded up to a multiple of 4.  The next kernel on `stream` must not
 * be launched with programmatic dependent launch. */
int asv_plan_upload(const int32_t* host_plan, int32_t* plan_dev, int64_t n_int32, void* stream);

/* Workspace: the dynamic-schedule counters + split partials. */
size_t asv_attn_workspace_bytes(const asv_attn_shape* shape, int32_t max_batch,
                                int32_t max_total_splits);
int asv_attn_workspace_init(void* workspace, size_t bytes, void* stream);

typedef struct asv_attn_args {
    const void* q;          /* [b][n_h][128] bf16 (fp16 with kv_dtype = ASV_KV_F16), this layer */
    void* kv_pool;          /* device page pool base (layer-major layout above) */
    int64_t pool_pages;     /* pages in the pool: the layer stride of the layer-major pool */
    int32_t layer;          /* layer slice of every page to attend over */
    const int32_t* plan_dev;/* device copy of the plan buffer */
    const asv_attn_plan* plan;
    const void* k_new;      /* [b][n_kv][128] bf16 appended at position seq_len (nullable) */
    const void* v_new;      /* [b][n_kv][128] bf16 (nullable together with k_new) */
    void* out;              /* [b][n_h][128] bf16 */
    float* lse;             /* [b][n_h] natural-log sum-exp (nullable) */
    void* workspace;
    size_t workspace_bytes;
    float sm_scale;         /* 1/sqrt(128) for the paper's Eq. 2 */
    uint32_t launch_index;  /* consecutive launches on one workspace must alternate parity */
    int32_t pdl;            /* 1: programmatic dependent launch (overlap with the previous kernel) */
    uint64_t* warp_timestamps; /* optional [workers][2] device-accessible buffer (device or mapped host):
                                  %globaltimer at each persistent warp's start and end — the measured
                                  intra-iteration bubble */
    int32_t kv_dtype;       /* ASV_KV_BF16 (0, default) or ASV_KV_F16: the element type of the KV pool,
                               q, k_new / v_new and out (the layout is the same 16-bit one) */
    /* Deferred split merge (consecutive launches on one workspace with the SAME plan, e.g. the L layers
     * of an attention-only decode step): defer_merge = 1 leaves this launch's split-request partials in
     * the workspace half of its launch_index parity and launches no merge kernel; the next launch, with
     * prev_out (and optionally prev_lse) set to where those rows go, merges them with its own warps
     * right after its dependency wait — one grid boundary per layer instead of two.  The last launch
     * of a chain keeps defer_merge = 0. */
    int32_t defer_merge;
    void* prev_out;
    float* prev_lse;
    /* Measurement experiment: l2_warm_items > 0 turns the call into an L2 prefetch of the first
     * l2_warm_pages pages (K and V blocks of the launch's layer) of the first l2_warm_items work items,
     * in the order the kernel's warps take them — no attention, no merge, no output. */
    int32_t l2_warm_items, l2_warm_pages;
} asv_attn_args;

#define ASV_KV_BF16 0
#define ASV_KV_F16 1

/* K1+K2+K3: paged split-KV decode attention with fused KV append (K1+K3), then the
 * log-sum-exp merge of split requests (K2), chained with programmatic dependent
 * launch when pdl = 1.  Replaces the attention term of iteration_latency
 * (cost_model.hpp:112-135). */
int asv_decode_attention(const asv_attn_shape* shape, const asv_attn_args* args, void* stream);

/* ------------------------------------------------------------------------ */
/* KV page moves (copy engines).  Replace the PRICED transfers of the          */
/* reference (transfer_time cluster_sim.hpp:60-66; start_async_transfer /     */
/* sync_transfer :220-232).  A request with `tokens` tokens owns               */
/* ceil(tokens/16) pages; exactly tokens * kv_bytes_per_token bytes move:     */
/* whole pages as 2-D copies, the valid rows of a partial last page as a 3-D   */
/* copy.  host_pages[j] = page j of the request in the host (page-major)       */
/* format.  Asynchronous on `stream`; *bytes_out = bytes moved.                */
/* ------------------------------------------------------------------------ */
/* C1: pinned host pool -> device pool (batch_prefetch / stray_prefetch, PCIe) */
int asv_kv_copy_h2d(const asv_attn_shape* shape, void* pool, int64_t pool_pages, const int32_t* pages,
                    int64_t tokens, const void* const* host_pages, void* stream, int64_t* bytes_out);
/* device pool -> pinned host pool (spill / flush / FCFS swap-out, PCIe) */
int asv_kv_copy_d2h(const asv_attn_shape* shape, const void* pool, int64_t pool_pages, const int32_t* pages,
                    int64_t tokens, void* const* host_pages, void* stream, int64_t* bytes_out);
/* C2/C3: device pool -> device pool, across a (prefetch, decode) pair over NVLink
 * (admit / evict) or within one device */
int asv_kv_copy_d2d(const asv_attn_shape* shape, void* dst_pool, int64_t dst_pool_pages, int32_t dst_device,
                    const int32_t* dst_pages, const void* src_pool, int64_t src_pool_pages, int32_t src_device,
                    const int32_t* src_pages, int64_t tokens, void* stream, int64_t* bytes_out);

/* ------------------------------------------------------------------------ */
/* Host-side decision path (reference API underneath, C ABI on top).          */
/* ------------------------------------------------------------------------ */

/* Run one experiment config (reference JSON format, proj/configs/<name>.json,
 * io.hpp:184-254) through the B200-native engine in VIRTUAL-CLOCK mode (the
 * reference cost model advances time, so decisions are bit-exact) and return
 * the schema-1 JSONL log (io.hpp:279-323).  `*out` is malloc'ed; free it with
 * asv_free().  `policy_override` may be NULL. */
int asv_run_config_jsonl(const char* config_json, const char* policy_override, char** out,
                         int64_t* out_len);
void asv_free(void* p);

/* Same, for data-parallel shard `shard_index` of `shard_count` (request i of the
 * trace belongs to shard i % shard_count) — what each rank of a multi-GPU run
 * decides; no cross-shard communication exists on the decision path. */
int asv_run_config_jsonl_shard(const char* config_json, const char* policy_override, int32_t shard_index,
                               int32_t shard_count, char** out, int64_t* out_len);

/* ------------------------------------------------------------------------ */
/* Decode-step linear layers on tcgen05 (the GEMM half of */
/* a decode iteration, priced by the reference as the MLP term of             */
/* iteration_latency, cost_model.hpp:60-63, 130-131).                         */
/*   y[b][n] = epilogue( sum_k x[b][k] * w[n][k] ),  b < batch <= 256         */
/* bf16 in/out, fp32 accumulate (TMEM).  Weights are the MMA M dimension      */
/* (swap-AB: decode batches are far below the 128-row MMA tile).              */
/* ------------------------------------------------------------------------ */
#define ASV_EPI_STORE 0      /* y[b][n] = acc */
#define ASV_EPI_RESIDUAL 1   /* y[b][n] += acc (residual stream updated in place) */
#define ASV_EPI_SILU_MUL 2   /* w rows of tile t: [0,64) gate, [64,128) up of outputs 64t..64t+63;
                                y[b][64t + j] = silu(gate) * up */
#define ASV_EPI_QKV_ROPE 3   /* w rows: n_q_heads q heads, n_kv_heads k heads, n_kv_heads v heads
                                (128 rows each); rotate-half RoPE (theta) at positions[b] on q, k */
typedef struct asv_linear_args {
    const void* w;           /* [n_out][k] bf16 row-major; n_out % 128 == 0, k % 64 == 0 */
    int32_t n_out, k;
    const void* x;           /* [x_rows][k] bf16; x_rows >= batch rounded up to 16 (extra rows: any
                                finite values, they only feed unused accumulator columns) */
    int32_t x_rows, batch;
    void* y;                 /* [batch][y_ld] bf16 (STORE / RESIDUAL / SILU_MUL) */
    int32_t y_ld;
    int32_t epilogue;        /* ASV_EPI_* */
    const int32_t* positions;/* QKV_ROPE: [batch] token positions (= prefix_len) */
    float rope_theta;        /* QKV_ROPE: 10000 for Llama-2 */
    void* q;                 /* QKV_ROPE: [batch][n_q_heads][128] */
    void* k_out;             /* QKV_ROPE: [batch][n_kv_heads][128] */
    void* v_out;             /* QKV_ROPE: [batch][n_kv_heads][128] */
    int32_t n_q_heads, n_kv_heads;
    int32_t pdl;             /* 1: programmatic dependent launch — W streams into the ring while the
                                previous kernel on the stream finishes; X, y wait for it */
    /* Fused RMSNorm (optional; both sides zero/null = off).  A RESIDUAL linear with ss_out writes,
     * per 128-row tile and half tile, the sum of squares of each updated (bf16) y row:
     * ss_out[(tile * 2 + half) * ss_ld + b].  The next linear takes x = that raw residual stream
     * (the norm weight gamma folded into its w columns) with ss_in = those ss_parts partial sums and
     * scales output column b by rsqrt(sum(ss_in[.][b]) / ss_dim + ss_eps) — RMSNorm(h) W^T without a
     * norm kernel; fixed summation order (deterministic). */
    float* ss_out;
    const float* ss_in;
    int32_t ss_parts, ss_ld, ss_dim;
    float ss_eps;
    /* Optional: the weights of the NEXT linear on the stream ([next_n_out][next_k], same batch).  With
     * ASV_LINEAR_NEXT_PF=N set, a CTA that has issued its last weight load prefetches into L2
     * (cp.async.bulk.prefetch.tensor) a share of the N stages each CTA of the next launch streams right
     * AFTER its ring (which it requests itself at entry), so the next launch's refills after its
     * dependency wait hit L2.  No effect on results. */
    const void* next_w;
    int32_t next_n_out, next_k;
    int32_t next_epilogue;   /* the next linear's ASV_EPI_* (its schedule decides which stages come after
                                its ring) */
} asv_linear_args;

/* One launch: one CTA per (128-row tile, K split); the K splits of a tile are one
 * thread-block cluster and reduce through distributed shared memory, so no
 * workspace is needed.  Stream-ordered; no host synchronisation. */
int asv_linear(const asv_linear_args* args, void* stream);

/* Persistent CHAIN of up to 4 dependent linear layers in ONE launch (decode_chain.cu; measured
 * slower than one asv_linear per GEMM, DESIGN §4 — an experiment, opt-in in the engine):
 * phase i+1 may read what phase i writes (x, residual stream, fused-RMSNorm sums) — e.g. per
 * decoder layer O-proj+residual -> gate/up+SiLU -> down+residual -> next layer's QKV+RoPE.  Default
 * kernel (batch <= 128): 8-CTA clusters take whole tiles, the K splits of a tile reduce through
 * distributed shared memory (results bit-identical to asv_linear), phases hand off through per-phase
 * counters; otherwise (or ASV_CHAIN_KIND=streamk) every phase's (tile, 64-K block) units are split
 * evenly over a grid of 2 CTAs per SM and tiles cut between CTAs are reduced (fixed CTA order:
 * deterministic) by the CTA holding their first K block.  The weight stream runs ahead across phase
 * boundaries in both.  Same per-phase semantics and
 * weight layouts as asv_linear (all phases share `batch`; `pdl` is taken from phases[0]).
 * The workspace holds the cross-CTA counters and partials of one device; launches that share a
 * workspace must be stream-ordered (one compute stream). */
typedef struct asv_linear_chain_ws asv_linear_chain_ws;
int asv_linear_chain_ws_create(int32_t device, asv_linear_chain_ws** out);
void asv_linear_chain_ws_destroy(asv_linear_chain_ws* ws);
int asv_linear_chain(const asv_linear_args* phases, int32_t n, asv_linear_chain_ws* ws, void* stream);
/* (The default chain kernel keeps 8-CTA clusters co-resident; the first launch on a workspace measures
 * how many are with a probe kernel (synchronous), so it must not be stream-captured.  ASV_CHAIN_KIND=
 * streamk selects the stream-K kernel.) */
/* Measurement only: enable (1) / disable (0) a per-CTA, per-phase %globaltimer timeline of the chain
 * launches on `ws`; with `out` (capacity `cap` words) copies the last launch's [grid][4][6] stamps
 * (decode_chain.cu kTraceSlots) and sets *n.  Synchronous. */
int asv_linear_chain_ws_trace(asv_linear_chain_ws* ws, int32_t enable, uint64_t* out, int64_t cap, int64_t* n);
/* The schedule asv_linear picks for a shape (host-only, no GPU needed): K splits (= cluster size),
 * ring stages and the CTA's dynamic shared memory, on a device with `sms` SMs (decode_gemm.cu
 * linear_plan: bytes in flight maximised within one wave). */
int asv_linear_schedule(int32_t n_out, int32_t k, int32_t batch, int32_t epilogue, int32_t sms, int32_t* splits,
                        int32_t* stages, int32_t* smem_bytes);
/* Measurement only: force every following asv_linear launch to `splits` K splits (cluster size,
 * 1-8) and `stages` ring stages (2-8; 0 keeps the schedule's); splits = 0 restores the automatic
 * schedule (decode_gemm.cu linear_plan).  Results are identical up to fp32 summation order. */
int asv_linear_set_schedule(int32_t splits, int32_t stages);
/* Measurement only: per-CTA %globaltimer timeline of asv_linear launches (decode_gemm.cu kTrSlots:
 * entry, dependency satisfied, last weight load issued, first stage landed, accumulator complete,
 * cluster reduce entered, exit, SM id).  enable=1 arms the probe for the next 64 launches (grid <= 1024);
 * `out` (capacity `cap` words) receives [launches][1024][8] stamps of the armed launches and *n the word
 * count; enable=0 with out=NULL frees the probe.  Synchronous (device-wide). */
int asv_linear_trace(int32_t enable, uint64_t* out, int64_t cap, int64_t* n);
/* out[b][:] = h[b][:] * rsqrt(mean(h[b]^2) + eps) * gamma; rows [batch, rows_out) of out zeroed */
int asv_rmsnorm(const void* h, const void* gamma, void* out, int32_t dim, int32_t batch, int32_t rows_out,
                float eps, int32_t pdl, void* stream);

/* ------------------------------------------------------------------------ */
/* Decode engine on the GPU: the reference engine's decisions (virtual clock, */
/* bit-exact) executed for real — KV moves as copies, every iteration as      */
/* page-table build + L decode-attention launches — with measured times.      */
/* Replaces Simulation::run's priced path (cluster_sim.hpp:131-160, 437-569). */
/* ------------------------------------------------------------------------ */
typedef struct asv_engine_opts {
    int32_t decode_device;      /* CUDA device of the decode GPU */
    int32_t prefetch_device;    /* partner holding the candidate buffers; == decode_device: single GPU */
    int32_t num_q_heads;        /* attention shape; num_kv_heads*128*2*2*num_layers must equal */
    int32_t num_kv_heads;       /* the config model's kv_bytes_per_token (bytes moved == reference) */
    int32_t num_layers;
    int32_t execute_transfers;  /* 1: real KV moves from/to the pinned host pool (e2e); 0: KV resident */
    int64_t host_pool_bytes;    /* pinned host arena; request KV pages alias into it (synthetic data) */
    int64_t exec_begin;         /* first iteration executed on the GPU (earlier: decisions only) */
    int64_t exec_end;           /* one past the last executed iteration (-1: all) */
    int64_t timed_begin;        /* first iteration of the timed window (>= exec_begin) */
    int32_t shard_index;        /* data-parallel shard of the trace: requests i with */
    int32_t shard_count;        /* i % shard_count == shard_index (1: whole trace) */
    int32_t pdl;                /* programmatic dependent launch between layer kernels */
    int32_t run_ahead;          /* max iterations the host may run ahead of the GPU (ring depth) */
    int64_t copy_begin;         /* first iteration whose boundary KV moves are executed (<= exec_begin:
                                   lets prefetches issued before the executed span reach steady state) */
    int32_t pair_mode;          /* 1: separate candidate-buffer pool even when prefetch_device ==
                                   decode_device (exercises the admit/evict copy path on one GPU) */
    int32_t full_step;          /* 1: every iteration runs the whole decoder layer stack (RMSNorm,
                                   QKV+RoPE, attention, O + residual, RMSNorm, gate/up SiLU, down +
                                   residual) with synthetic weights, not attention alone */
    int32_t intermediate_size;  /* MLP width for full_step (0: 11008 for hidden 4096, 13824 for 5120,
                                   else 8/3 hidden rounded up to 128) */
    int32_t execute_prefill_offload; /* 1 (with execute_transfers): every prefill_offload transfer
                                   (cluster_sim.hpp:285-299) is a real D2H copy of the request's
                                   s x kv_bytes_per_token bytes from the prefill GPU (= the prefetch
                                   device) into its host-pool pages, on its own PCIe stream; a later
                                   host->GPU fetch of the request waits for it (pool_insert happens
                                   at transfer completion).  Prefill compute itself stays virtual. */
    int32_t probe_bubble;       /* 1: per-warp %globaltimer start/end of EVERY attention launch of every
                                   timed iteration -> measured intra-iteration bubble per iteration
                                   (reference bubble_from_per_request cost_model.hpp:149-155,
                                   IterationRecord.bubble_ms cluster_sim.hpp:489).  Off: no probe. */
    double* bubble_out;         /* optional [bubble_out_cap]: measured bubble (ms, idle time per warp summed
                                   over the iteration's launches) of each timed iteration, in order */
    int64_t bubble_out_cap;
    /* Content-check test mode (1): every KV row and query is a pure function of (global request id,
     * token position, layer, K|V|Q, head) — 128 values int8/128 (queries int8/8) from splitmix64, see
     * oracle/attn_oracle.c asv_oracle_content_row — the host pool is per request (not aliased) and
     * filled with the prompt rows, every iteration uploads its queries and appended rows, the device
     * pools start poisoned (NaN), and every iteration's attention output of every layer is captured.
     * Requires execute_transfers, exec_begin = copy_begin = 0, exec_end = -1, no full_step, no
     * prefill offload; batches <= 1024 rows. */
    int32_t content_check;
    const char* capture_path;   /* binary file, one record per executed iteration:
                                   int64 seq; int32 b, L, n_q, head; int64 ids[b] (global request ids,
                                   running order); int32 lens[b] (each request's seq_len decoded from the
                                   split descriptors of the UPLOADED plan = tokens the kernel attends);
                                   content_check: bf16 out[L][b][n_q][128] when head == -1 (every
                                   capture_every-th iteration, by seq) else out[L][b][128] of query head
                                   `head`; without content_check head == -2 and no outputs follow */
    int64_t capture_every;
    /* Decision clock.  0 (default): the reference's virtual clock (calibrated cost model), so batch
     * composition, order and bytes moved are bit-exact with the reference (SURVEY §7 hard part 1).
     * 1: wall clock — every executed iteration's duration is its MEASURED GPU time (CUDA events around
     * its launches); the orchestrator waits for it before the next boundary, so arrivals, starvation
     * clocks, batch gating and transfer completions are decided against measured time (the serving
     * mode; logs then differ from the reference by design).  KV-move durations stay modelled
     * (transfer_time); the data plane still orders every real copy. */
    int32_t wall_clock;
} asv_engine_opts;

/* transfer kinds for the per-kind byte counters */
#define ASV_XFER_PREFILL_OFFLOAD 0
#define ASV_XFER_BATCH_PREFETCH 1
#define ASV_XFER_STRAY_PREFETCH 2
#define ASV_XFER_ADMIT 3
#define ASV_XFER_EVICT 4
#define ASV_XFER_SPILL 5
#define ASV_XFER_FLUSH 6
#define ASV_XFER_KINDS 7

typedef struct asv_engine_stats {
    int64_t iterations_total;     /* decode iterations of the whole run (log) */
    int64_t iterations_timed;     /* iterations inside the timed window */
    int64_t tokens_timed;         /* sum of batch sizes inside the window */
    double window_ms;             /* GPU time of the window (CUDA events, compute stream) */
    double attn_ms;               /* sum of attention-kernel time inside the window */
    int64_t attn_bytes;           /* algorithmic K/V + q + out + index bytes inside the window */
    int64_t attn_launches;        /* kernel launches inside the window */
    int64_t h2d_bytes;            /* physical bytes moved over the executed span */
    int64_t d2h_bytes;
    int64_t p2p_bytes;
    double h2d_busy_ms;           /* copy-engine busy time of those moves (events) */
    double p2p_busy_ms;
    int64_t logical_bytes[ASV_XFER_KINDS]; /* whole run, == sum of the reference's TransferRecord.bytes */
    int64_t logical_count[ASV_XFER_KINDS];
    double virtual_decode_tok_s;  /* decode_throughput of the virtual-clock log */
    double host_decide_ms;        /* host time spent in the decision path (engine + planning) */
    int64_t max_batch;
    int64_t pages_decode;         /* physical page pools */
    int64_t pages_prefetch;
    double bubble_ms_timed;       /* sum of per-iteration bubble (virtual) inside the window */
    int64_t kernel_launches_timed;/* our kernels launched inside the window (attention + merge) */
    double virtual_window_ms;     /* reference-clock duration of the same window */
    int64_t h2d_bytes_window;     /* the physical moves above restricted to the timed window */
    int64_t d2h_bytes_window;
    int64_t p2p_bytes_window;
    double measured_idle_frac;    /* probe_bubble: 1 - sum(warp busy) / (warps x launch span) over every
                                     attention launch of the timed iterations (per-warp %globaltimer) */
    double measured_bubble_ms;    /* probe_bubble: sum over timed iterations of the idle time per warp,
                                     summed over the iteration's launches */
    double pcie_union_ms;         /* union of the PCIe copy-group intervals (both directions) inside the
                                     window: time the host link had work (with a separate prefetch GPU: the union
                                     of its timed PCIe copy groups, from the first one) */
    double host_wait_ms;          /* host time blocked on the GPU (run-ahead ring, page reclaim) */
    int64_t hazard_waits;         /* copy-stream waits on a page's last iteration (page reuse) */
    int64_t result_d2h_bytes_window; /* e2e: each iteration's attention output [b][n_h][128] bf16 read back
                                        to pinned host memory (SM stores, no copy-engine queue) */
    int64_t weight_bytes;         /* full_step: decoder weight bytes streamed inside the window */
    int64_t offload_bytes;        /* prefill_offload D2H bytes executed (== logical prefill_offload bytes
                                     of the executed span) */
    int64_t offload_bytes_window; /* the same restricted to the timed window */
    /* probe_bubble: distribution of the measured per-iteration bubble over the timed iterations */
    int64_t bubble_iterations;
    double bubble_p50_ms, bubble_p90_ms, bubble_p99_ms, bubble_max_ms;
    int64_t content_inplace_bytes;        /* content mode: merged-FCFS prompts written in place (not a
                                             reference transfer, not in h2d_bytes) */
    int64_t content_iterations_captured;  /* records written to capture_path */
} asv_engine_stats;

int asv_engine_run(const char* config_json, const char* policy_override, const asv_engine_opts* opts,
                   asv_engine_stats* stats);
/* asv_engine_run plus the run's artefacts, replacing `prefixsim run --config X`
 * (reference tools/prefixsim_main.cpp:66-111, write_run_artifacts :31-49):
 *   out_dir (nullable): writes log.jsonl (schema 1, byte-identical to the reference's log of the same
 *     config/shard: the decisions are the reference's), summary.json, ttft_cdf.csv, sched_cdf.csv
 *     (io.hpp summary_to_json / cdf_to_csv) and gpu_stats.json (the measured B200 numbers);
 *   log_out (nullable): the schema-1 JSONL log, malloc'ed (release with asv_free), length in *log_len. */
int asv_engine_run_ex(const char* config_json, const char* policy_override, const asv_engine_opts* opts,
                      asv_engine_stats* stats, const char* out_dir, char** log_out, int64_t* log_len);

/* Density-first search on a pool snapshot (batch_gen.hpp:126-210).
 * residents: n x {id, prefix_len, kv_blocks} in insertion order (all inserted at t=0).
 * Writes the batch member ids in page-table order; returns count via *n_out (0 = no batch). */
int asv_dfs_batch(const int64_t* residents, int64_t n, int64_t b_max, int64_t k_min,
                  int64_t* ids_out, int64_t* n_out, int64_t* total_blocks_out);

#ifdef __cplusplus
}
#endif
#endif /* ASV_H_ */
