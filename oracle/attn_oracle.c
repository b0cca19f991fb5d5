/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for paged decode attention.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the
 * CPU baseline; the product path (paper_2605_23389_b200/) never calls it.
 *
 * What it restates: the reference has NO numeric attention (
 * cost_model.hpp:13-27 only counts ops/bytes), so this follows PAPER Eq. 2
 * (PAPER.md:149-153), softmax(q K^T / sqrt(d_k)) V, over exactly
 * s = prefix_len tokens per request (cluster_sim.hpp:476-479 passes prefix_len
 * in running order), with the cost model's shape convention
 * (cost_model.hpp:16-26: h = n_heads * d per layer) and the 16-token block rule
 * (request.hpp:53-55).  Parity status: UNPINNED by the reference (no golden
 * attention vectors exist there); pinned instead by known-answer tests
 * (tests/test_oracle.py) and an independent numpy restatement.
 *
 * Numerics: bf16 (or IEEE fp16, kv_dtype 1) inputs widened to fp32 exactly; dot products in fp32, the
 * softmax normaliser and the weighted V sum accumulated in double.
 * Layout and swizzle: include/asv.h (device pool LAYER-MAJOR in page groups of
 * G pages, each group [L][G][2][n_kv][16][128], G the largest equal split with
 * G * slice < 2 GiB; one group = [L][pool_pages][...] for every test-sized pool).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* IEEE binary16 -> fp32, exact (subnormals, inf, nan) */
static inline float f16_to_f32(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const int exp = (h >> 10) & 0x1f;
    uint32_t mant = h & 0x3ffu, u;
    if (exp == 0x1f) {
        u = sign | 0x7f800000u | (mant << 13);
    } else if (exp != 0) {
        u = sign | ((uint32_t)(exp - 15 + 127) << 23) | (mant << 13);
    } else if (mant == 0) {
        u = sign;
    } else {  /* subnormal: normalise */
        int e = -14;
        while (!(mant & 0x400u)) {
            mant <<= 1;
            --e;
        }
        u = sign | ((uint32_t)(e + 127) << 23) | ((mant & 0x3ffu) << 13);
    }
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static inline float kv_to_f32(uint16_t h, int f16) { return f16 ? f16_to_f32(h) : bf16_to_f32(h); }

/* byte offset of (token t, dim d) inside one 4 KiB (page, layer, K|V, head) block */
static inline int64_t swz_off(int t, int d) {
    int c = d / 8;
    return (int64_t)t * 256 + (int64_t)((c ^ (t & 7)) << 4) + (int64_t)(d % 8) * 2;
}

typedef struct {
    int n_q, n_kv, L, layer, batch;
    const uint16_t* q;
    const uint8_t* pool;
    int64_t pool_pages;
    const int32_t* seq_lens;
    const int32_t* indptr;
    const int32_t* indices;
    float sm_scale;
    int f16;             /* element type: 0 bf16, 1 fp16 */
    float* out;
    float* lse;
    int next;            /* work counter (guarded by mu) */
    pthread_mutex_t mu;
} job_t;

static void one_row(const job_t* j, int r, int h) {
    const int D = 128;
    const int g = j->n_q / j->n_kv;
    const int kvh = h / g;
    const int s = j->seq_lens[r];
    const uint16_t* qv = j->q + ((int64_t)r * j->n_q + h) * D;
    float qf[128];
    for (int d = 0; d < D; ++d) qf[d] = kv_to_f32(qv[d], j->f16);
    float* scores = (float*)malloc(sizeof(float) * (size_t)(s > 0 ? s : 1));
    /* block (page, layer, kv, head) of the grouped layer-major pool */
    const int64_t slice = (int64_t)2 * j->n_kv * 4096;
    const int64_t gmax = (((int64_t)1 << 31) - 1) / slice;
    const int64_t gp = j->pool_pages / ((j->pool_pages + gmax - 1) / gmax);
#define BLOCK(page, kv) \
    ((((page) / gp) * gp * j->L + (int64_t)j->layer * gp + (page) % gp) * slice + ((int64_t)(kv) * j->n_kv + kvh) * 4096)
    float mx = -INFINITY;
    for (int t = 0; t < s; ++t) {
        const int64_t page = j->indices[j->indptr[r] + t / 16];
        const uint8_t* base = j->pool + BLOCK(page, 0);
        float acc = 0.f;
        for (int d = 0; d < D; ++d) {
            uint16_t kb;
            memcpy(&kb, base + swz_off(t % 16, d), 2);
            acc += qf[d] * kv_to_f32(kb, j->f16);
        }
        scores[t] = acc * j->sm_scale;
        if (scores[t] > mx) mx = scores[t];
    }
    double l = 0.0;
    double o[128];
    for (int d = 0; d < D; ++d) o[d] = 0.0;
    for (int t = 0; t < s; ++t) {
        const double p = exp((double)scores[t] - (double)mx);
        l += p;
        const int64_t page = j->indices[j->indptr[r] + t / 16];
        const uint8_t* base = j->pool + BLOCK(page, 1);
        for (int d = 0; d < D; ++d) {
            uint16_t vb;
            memcpy(&vb, base + swz_off(t % 16, d), 2);
            o[d] += p * (double)kv_to_f32(vb, j->f16);
        }
    }
    float* dst = j->out + ((int64_t)r * j->n_q + h) * D;
    for (int d = 0; d < D; ++d) dst[d] = s > 0 ? (float)(o[d] / l) : 0.f;
    if (j->lse) j->lse[(int64_t)r * j->n_q + h] = s > 0 ? (float)((double)mx + log(l)) : -INFINITY;
    free(scores);
#undef BLOCK
}

static void* worker(void* arg) {
    job_t* j = (job_t*)arg;
    const int rows = j->batch * j->n_q;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int k = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (k >= rows) break;
        one_row(j, k / j->n_q, k % j->n_q);
    }
    return NULL;
}

/* out: [batch][n_q][128] fp32; lse: [batch][n_q] natural log (nullable).
 * kv_dtype: 0 bf16, 1 fp16 (q and the pool).  Returns 0 on success. */
int asv_oracle_decode_attention_dt(int n_q, int n_kv, int num_layers, int layer, const uint16_t* q,
                                   const uint8_t* pool, int64_t pool_pages, const int32_t* seq_lens,
                                   const int32_t* indptr, const int32_t* indices, int batch,
                                   float sm_scale, float* out, float* lse, int threads, int kv_dtype) {
    if (n_kv <= 0 || n_q % n_kv != 0 || batch < 1 || (kv_dtype != 0 && kv_dtype != 1)) return 1;
    job_t j;
    j.n_q = n_q;
    j.n_kv = n_kv;
    j.L = num_layers;
    j.layer = layer;
    j.batch = batch;
    j.q = q;
    j.pool = pool;
    j.pool_pages = pool_pages;
    j.seq_lens = seq_lens;
    j.indptr = indptr;
    j.indices = indices;
    j.sm_scale = sm_scale;
    j.f16 = kv_dtype;
    j.out = out;
    j.lse = lse;
    j.next = 0;
    pthread_mutex_init(&j.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tids[256];
    for (int i = 0; i < threads; ++i) pthread_create(&tids[i], NULL, worker, &j);
    for (int i = 0; i < threads; ++i) pthread_join(tids[i], NULL);
    pthread_mutex_destroy(&j.mu);
    return 0;
}

int asv_oracle_decode_attention(int n_q, int n_kv, int num_layers, int layer, const uint16_t* q,
                                const uint8_t* pool, int64_t pool_pages, const int32_t* seq_lens,
                                const int32_t* indptr, const int32_t* indices, int batch,
                                float sm_scale, float* out, float* lse, int threads) {
    return asv_oracle_decode_attention_dt(n_q, n_kv, num_layers, layer, q, pool, pool_pages, seq_lens, indptr,
                                          indices, batch, sm_scale, out, lse, threads, 0);
}

/* Write (token t of layer/kv/head) row into a page buffer using the swizzle —
 * used by tests to build inputs and to check the fused append. */
void asv_oracle_put_row(uint8_t* page, int n_kv, int layer, int kv, int head, int t,
                        const uint16_t* row128) {
    const int64_t blk = (((int64_t)layer * 2 + kv) * n_kv + head) * 4096;
    for (int d = 0; d < 128; ++d) memcpy(page + blk + swz_off(t, d), &row128[d], 2);
}

void asv_oracle_get_row(const uint8_t* page, int n_kv, int layer, int kv, int head, int t,
                        uint16_t* row128) {
    const int64_t blk = (((int64_t)layer * 2 + kv) * n_kv + head) * 4096;
    for (int d = 0; d < 128; ++d) memcpy(&row128[d], page + blk + swz_off(t, d), 2);
}
