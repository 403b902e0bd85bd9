/*
 * TEST INFRASTRUCTURE ONLY - the checker, never the product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.
 *
 * CPU restatement of the per-decode-step data path the B200 kernels execute:
 *   - GQA decode attention over paged KV (one new token attends to every
 *     cached token of its request, query head j reads KV head j / (Hq/Hkv)):
 *     PAPER.md:238-244 (decode + GQA), PAPER.md:367 (16-token paged blocks),
 *     PAPER.md:750 (per-request, layer-aware table).  The reference package
 *     (/root/reference/pkg/src/kvsim) contains no attention arithmetic - it
 *     prices it as per_layer_compute (core.py:257-261) - and the paper's
 *     implementation lives in un-vendored vLLM v0.6.6 PagedAttention.  This
 *     attention oracle is therefore pinned against an independent float64
 *     dense softmax(QK^T)V and against golden outputs of vLLM's
 *     PagedAttention v2 kernel (0.22, same kernel family) recorded on a B200
 *     (tests/golden/vllm_attention.npz, tests/test_oracle.py) - not against
 *     kvsim outputs, which do not exist: "parity unpinned by the reference".
 *   - the new-token append (RequestState.record_generated_token,
 *     core.py:95-102; engine.py:389-392): the row lands at token index
 *     `pos` of the slab, i.e. block pos/16, slot pos%16.
 *
 * Arithmetic: bf16 inputs widened exactly to float, dot products and softmax
 * accumulated in double, result rounded to float.  Layout identical to the
 * device: block = bf16 [Hkv][2][16][128].
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HEAD_DIM 128
#define BLOCK_TOKENS 16

static inline float bf16_to_f32(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return f;
}

typedef struct {
  const uint16_t* q;
  const uint16_t* pool;
  const int32_t* block_tables;
  int32_t max_blocks;
  const int32_t* seq_lens;
  float* out;
  int32_t batch, hq, hkv;
  float scale;
  int next;             /* shared work counter over (b, h) pairs */
  pthread_mutex_t mu;
} attn_job;

static void attend_one(const attn_job* j, int b, int h) {
  const int group = j->hq / j->hkv;
  const int kvh = h / group;
  const size_t block_elems = (size_t)j->hkv * 2 * BLOCK_TOKENS * HEAD_DIM;
  const int seq = j->seq_lens[b];
  float* o = j->out + ((size_t)b * j->hq + h) * HEAD_DIM;
  if (seq <= 0) {
    memset(o, 0, sizeof(float) * HEAD_DIM);
    return;
  }
  double qv[HEAD_DIM];
  for (int d = 0; d < HEAD_DIM; ++d) qv[d] = bf16_to_f32(j->q[((size_t)b * j->hq + h) * HEAD_DIM + d]);
  double* scores = (double*)malloc(sizeof(double) * (size_t)seq);
  double mx = -INFINITY;
  for (int t = 0; t < seq; ++t) {
    const int blk = j->block_tables[(size_t)b * j->max_blocks + t / BLOCK_TOKENS];
    const uint16_t* krow = j->pool + (size_t)blk * block_elems +
                           (((size_t)kvh * 2 + 0) * BLOCK_TOKENS + t % BLOCK_TOKENS) * HEAD_DIM;
    double s = 0.0;
    for (int d = 0; d < HEAD_DIM; ++d) s += qv[d] * bf16_to_f32(krow[d]);
    s *= j->scale;
    scores[t] = s;
    if (s > mx) mx = s;
  }
  double acc[HEAD_DIM];
  for (int d = 0; d < HEAD_DIM; ++d) acc[d] = 0.0;
  double denom = 0.0;
  for (int t = 0; t < seq; ++t) {
    const double p = exp(scores[t] - mx);
    denom += p;
    const int blk = j->block_tables[(size_t)b * j->max_blocks + t / BLOCK_TOKENS];
    const uint16_t* vrow = j->pool + (size_t)blk * block_elems +
                           (((size_t)kvh * 2 + 1) * BLOCK_TOKENS + t % BLOCK_TOKENS) * HEAD_DIM;
    for (int d = 0; d < HEAD_DIM; ++d) acc[d] += p * bf16_to_f32(vrow[d]);
  }
  for (int d = 0; d < HEAD_DIM; ++d) o[d] = (float)(acc[d] / denom);
  free(scores);
}

static void* attn_worker(void* arg) {
  attn_job* j = (attn_job*)arg;
  const int total = j->batch * j->hq;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int idx = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (idx >= total) break;
    attend_one(j, idx / j->hq, idx % j->hq);
  }
  return NULL;
}

/* out[b][hq][d] (float32).  Tokens >= seq_lens[b] are ignored.  `threads`
 * host threads share the (request, head) pairs. */
void oracle_decode_attention(const uint16_t* q, const uint16_t* pool, const int32_t* block_tables,
                             int32_t max_blocks, const int32_t* seq_lens, float* out,
                             int32_t batch, int32_t hq, int32_t hkv, float scale, int32_t threads) {
  attn_job j = {q, pool, block_tables, max_blocks, seq_lens, out, batch, hq, hkv, scale, 0,
                PTHREAD_MUTEX_INITIALIZER};
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tids[256];
  for (int i = 1; i < threads; ++i) pthread_create(&tids[i], NULL, attn_worker, &j);
  attn_worker(&j);
  for (int i = 1; i < threads; ++i) pthread_join(tids[i], NULL);
}

/* Append of one layer: rows k_new/v_new [B][Hkv][128] at token positions[b]
 * of the slab addressed through block_tables (pool blocks). */
void oracle_kv_append(const uint16_t* k_new, const uint16_t* v_new, uint16_t* pool,
                      const int32_t* block_tables, int32_t max_blocks, const int32_t* positions,
                      int32_t batch, int32_t hkv) {
  const size_t block_elems = (size_t)hkv * 2 * BLOCK_TOKENS * HEAD_DIM;
  for (int b = 0; b < batch; ++b) {
    const int pos = positions[b];
    if (pos < 0) continue;
    const int blk = block_tables[(size_t)b * max_blocks + pos / BLOCK_TOKENS];
    if (blk < 0) continue;
    for (int h = 0; h < hkv; ++h) {
      for (int kv = 0; kv < 2; ++kv) {
        const uint16_t* src = (kv ? v_new : k_new) + ((size_t)b * hkv + h) * HEAD_DIM;
        uint16_t* dst = pool + (size_t)blk * block_elems +
                        (((size_t)h * 2 + kv) * BLOCK_TOKENS + pos % BLOCK_TOKENS) * HEAD_DIM;
        memcpy(dst, src, sizeof(uint16_t) * HEAD_DIM);
      }
    }
  }
}

