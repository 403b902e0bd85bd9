/*
 * orbitflow_b200.h - C ABI of the B200 (sm_100a) per-decode-step KV data path.
 *
 * This is the drop-in boundary underneath the kvsim host API
 * (/root/reference/pkg/src/kvsim).  The reference only *prices* a decode step;
 * every entry point below *does* the corresponding work on the GPU.  Each
 * declaration cites the reference interface whose semantics it realises.
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch types.  Device pointers are
 *     CUDA device (or UVA-mapped host) addresses, `stream` is a cudaStream_t
 *     passed as void* (NULL = legacy default stream).
 *   - Every function returns 0 on success, a cudaError_t value (>0) for a CUDA
 *     failure, or -1 for an argument error; ofb_last_error() returns the
 *     thread-local message.  There is no CPU fallback: a missing GPU is an
 *     error (reference error convention: ValueError / RuntimeError classes,
 *     kvsim/latency.py:78-79, kvsim/engine.py:53-58).
 *   - KV layout (pool blocks, staging slots and host slabs alike): one paged
 *     block of 16 tokens (kvsim DEFAULT_BLOCK_SIZE, core.py:24) for all KV heads
 *     of one layer is  bf16 [Hkv][2 (K,V)][16][128]  = Hkv * 8 KiB.
 *     A (request, layer) slab is a run of such blocks; in host memory it is
 *     contiguous, in HBM it is addressed through a block table.
 *   - head_dim must be 128; q-group Hq/Hkv must be <= 16.
 */
#ifndef ORBITFLOW_B200_H_
#define ORBITFLOW_B200_H_

#include <stdint.h>

#if defined(__GNUC__)
#define OFB_API __attribute__((visibility("default")))
#else
#define OFB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ----------------------------------------------------------- */
OFB_API const char* ofb_version(void);
OFB_API const char* ofb_last_error(void);
/* K1 work decomposition for later launches: 0 = persistent stream-K, 1 = fixed
 * splits + last-CTA combine, 2 = auto (default: cluster for latency-bound
 * launches, split otherwise), 3 = cluster splits combined through distributed
 * shared memory.  Returns the previous variant. */
OFB_API int ofb_set_attention_kernel(int32_t variant);
/* Which decomposition a launch of this shape would use now: 0 stream-K, 1 split,
 * 3 cluster. */
OFB_API int ofb_attention_variant_for(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len);
/* Split plan of the (default) split K1, host arithmetic only: blocks per split
 * and splits per (request, KV head) on a GPU with `num_sms` SMs and
 * `ctas_per_sm` resident K1 CTAs (ofb_device_info); the launch uses the same
 * function with the live device's values. */
/* Cluster plan of the cluster K1 (host arithmetic): CTAs per cluster, clusters
 * per (request, KV head), blocks per CTA and TMA ring depth, given
 * cluster_slots[k] = clusters of 2^k CTAs the GPU places at once (k = 0..4,
 * ofb_attention_cluster_slots).  Returns 1 when the shape is not a one-wave
 * cluster shape (the cluster kernel refuses it; auto never picks it). */
OFB_API int ofb_attention_cluster_plan(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len,
                                       const int32_t* cluster_slots, int32_t* cluster,
                                       int32_t* clusters_per_pair, int32_t* blocks_per_cta,
                                       int32_t* stages);
/* cluster_slots[k] (k = 0..4) of this GPU for the cluster K1 (initialises the device). */
OFB_API int ofb_attention_cluster_slots(int32_t* cluster_slots);
OFB_API int ofb_attention_split_plan(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                     int32_t max_seq_len, int32_t num_sms, int32_t ctas_per_sm,
                                     int32_t* blocks_per_split, int32_t* splits);
/* Host arithmetic: the K1 plan of an attention-only in-step launch (every layer
 * of a step without fetches but the first) - the split kernel, whose consumers
 * wait for the previous layer only before their global writes, on the balanced
 * plan (one narrow CTA per SM less one per (request, KV head) pair; *narrow = 1)
 * where it measured best, else on the cost-model plan (profiles/r02_k1_instep.md). */
OFB_API int ofb_attention_instep_plan(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                      int32_t max_seq_len, int32_t num_sms, int32_t ctas_per_sm,
                                      int32_t* blocks_per_split, int32_t* splits, int32_t* narrow);
/* Diagnostics: stream-K K1 launches write 6 globaltimer stamps per CTA (entry,
 * past the dependency wait, first tile ready, last tile consumed, exit, SM id)
 * into `device_buffer` (uint64 [448][6]); NULL switches tracing off. */
OFB_API int ofb_k1_trace(void* device_buffer);
/* Same for any K1 variant with an explicit capacity in CTAs: the split kernel
 * writes 8 stamps per CTA (entry, prologue done, first tile ready, ring drained,
 * partial written, ticket taken, exit, SM id) at index
 * (request * Hkv + kv head) * splits + split; CTAs past `ctas` are not traced. */
OFB_API int ofb_k1_trace_sized(void* device_buffer, int32_t ctas);
/* SM count and resident attention CTAs per SM on the current device. */
OFB_API int ofb_device_info(int32_t* num_sms, int32_t* attn_ctas_per_sm);

/* ---- pinned host pool -------------------------------------------------- */
/* Page-locked, device-mapped host memory (cudaHostAlloc Mapped|Portable).
 * Backs the host-resident KV slabs: offloaded layers (x[r][l] = 0,
 * kvsim/core.py:110-122) and evicted/removable layers (kvsim/engine.py:126-204).
 * Returns NULL on failure. */
OFB_API void* ofb_host_alloc(int64_t bytes);
OFB_API int ofb_host_free(void* ptr);

/* ---- K1: paged GQA flash-decode attention (one layer) ------------------ */
/* Bytes of scratch ofb_decode_attention needs; zero it once before first use
 * (the kernel re-arms its counters itself). */
OFB_API int64_t ofb_attention_workspace_bytes(int32_t batch, int32_t num_q_heads,
                                      int32_t num_kv_heads, int32_t max_seq_len);

/* out[b][hq][:] = softmax(scale * q[b][hq] . K_b^T) V_b over the first
 * seq_lens[b] tokens of request b's paged KV, with K/V of kv head hq/(Hq/Hkv).
 * Realises the compute the reference prices as per_layer_compute
 * (kvsim/core.py:257-261) inside batch_decode_latency_fast
 * (kvsim/latency.py:252-274).
 *   q, out        bf16 [batch][Hq][128]
 *   kv_pool       block pool base, pool_blocks blocks of Hkv*8 KiB
 *   block_tables  int32 [batch][max_blocks] pool block ids
 *   seq_lens      int32 [batch] tokens per request (device)
 *   max_seq_len   host-side upper bound of seq_lens (grid sizing) */
OFB_API int ofb_decode_attention(const void* q, void* out, const void* kv_pool, int64_t pool_blocks,
                         const int32_t* block_tables, int32_t max_blocks,
                         const int32_t* seq_lens, void* workspace, int64_t workspace_bytes,
                         int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                         int32_t head_dim, int32_t max_seq_len, float scale, void* stream);

/* ---- K3: new-token KV append ------------------------------------------- */
/* For every layer l < num_layers, request b, kv head h: write k_new/v_new
 * [l][b][h][:] at token positions[b] (skip if < 0) into
 *   - the pool block block_tables[l][b][positions[b]/16] (skip if < 0), and
 *   - the mapped host slab host_slabs[l][b] (skip if 0 or host_slabs NULL).
 * Realises RequestState.record_generated_token / sync_blocks
 * (kvsim/core.py:95-102) as called per step at kvsim/engine.py:389-392, and
 * the paper's "fresh KV written to its host slot" for offloaded layers
 * (PAPER.md:489). */
OFB_API int ofb_kv_append(const void* k_new, const void* v_new, void* kv_pool,
                  const int32_t* block_tables, int32_t max_blocks, const int32_t* positions,
                  const uint64_t* host_slabs, int32_t num_layers, int32_t batch,
                  int32_t num_kv_heads, int32_t head_dim, void* stream);

/* ---- K5: prefill KV written straight to its planned location ----------- */
/* Scatter a request's prompt K/V (bf16 [L][tokens][Hkv][128] each, token-major
 * as a prefill produces it) into the paged layout of L slabs whose base
 * addresses are dst[L] (device array): an HBM extent for a resident layer, the
 * mapped pinned host slab for an offloaded one - no staging, no second copy.
 * Realises what the reference leaves free (kvsim/engine.py:495-503:
 * prefill is only priced) and the paper's direct host write. */
OFB_API int ofb_kv_prefill(const void* k, const void* v, const uint64_t* dst, int32_t num_layers,
                           int32_t tokens, int32_t num_kv_heads, int32_t head_dim, void* stream);

/* ---- K2 + K3 + K1: one decode step of the whole layer stack ------------ */
typedef struct ofb_runtime ofb_runtime;

typedef struct ofb_step_desc {
  int32_t num_layers, batch, num_q_heads, num_kv_heads, head_dim;
  float scale;
  /* device tensors */
  const void* q;              /* bf16 [L][B][Hq][128] */
  void* out;                  /* bf16 [L][B][Hq][128] */
  const void* k_new;          /* bf16 [L][B][Hkv][128] */
  const void* v_new;          /* bf16 [L][B][Hkv][128] */
  void* kv_pool;
  int64_t pool_blocks;
  const int32_t* block_tables; /* int32 [L][B][max_blocks]: resident slab or staging slot */
  int32_t max_blocks;
  const int32_t* seq_lens;    /* int32 [B], after this step's append */
  const int32_t* positions;   /* int32 [B], index of the appended token (<0: no append) */
  const uint64_t* host_slabs_dev; /* [L][B] mapped host slab bases, 0 = GPU-resident */
  void* workspace;
  int64_t workspace_bytes;
  int32_t max_seq_len;
  /* host-side transfer plan */
  const uint64_t* host_slabs;  /* [L][B] same values, host copy: x[r][l]=0 <=> != 0 */
  const uint64_t* staging_dst; /* [L][B] device address of the staging slot for (l, b) */
  const int64_t* fetch_bytes;  /* [B] bytes fetched per offloaded (b, l) slab */
  int32_t staging_slots;       /* 1 = reference single-slot launch rule, 2 = double buffer */
  int32_t record_timing;       /* 1 = record per-layer / per-copy CUDA events */
  /* Cross-step prefetch (NULL = off): [B] bytes each request will fetch per
   * offloaded slab in the NEXT step.  After this step the runtime already
   * enqueues, per request, the next step's first staging_slots fetches (same
   * slabs, same slots), each gated on this step's last attention that used
   * its slot, so the copy engines stay busy while the host turns the step
   * around.  The next step adopts them if its transfer plan matches (and
   * counts them in its timing record), else they are fenced and re-issued. */
  const int64_t* next_fetch_bytes;
  /* 0: one append of every resident row at step start (the token's K/V of all
   * layers is known up front).  1: the append of layer l runs right before its
   * attention, inside ofb_runtime_step_layers - a decoder whose k_new/v_new of
   * layer l are produced by work the caller interleaves after layer l-1.  2: as
   * 1, but the producer of k_new/v_new already wrote the resident rows into the
   * pool (ofb_oproj_desc.kv_pool): only rows with a host slab are appended
   * (host slab + staging), and a layer without fetches launches no append. */
  int32_t append_per_layer;
} ofb_step_desc;

typedef struct ofb_step_timing {
  int32_t layers;           /* attention launches timed */
  float attn_ms_total;      /* sum of per-layer attention kernel durations */
  float attn_ms_max;
  int32_t copies;           /* H2D slab fetches timed */
  float copy_ms_sum;        /* sum of per-copy durations */
  double copy_bytes;        /* bytes fetched */
  float copy_span_ms;       /* first copy start -> last copy end */
  float step_ms;            /* step start -> last attention end */
  int32_t copy_streams;     /* copy streams used */
  float mig_ms;             /* last ofb_runtime_migrate span (0 if none timed) */
  double mig_h2d_bytes, mig_d2h_bytes;
  /* accumulated over every timed step since the last ofb_runtime_timing_reset */
  int32_t acc_steps, acc_attn_launches;
  double acc_attn_ms, acc_copy_bytes, acc_step_ms;
} ofb_step_timing;

OFB_API ofb_runtime* ofb_runtime_create(int32_t max_copy_streams);
OFB_API int ofb_runtime_destroy(ofb_runtime* rt);

/* Enqueue one full decode step on `stream` (the compute stream) plus the
 * runtime's copy streams, asynchronously:
 *   1. append (K3) for every layer (resident -> pool, offloaded -> host slab),
 *   2. per request, one copy stream fetches its offloaded slabs in layer order
 *      into its staging slot(s) (K2), honouring the reference launch rule
 *      (kvsim/latency.py:159-169): with staging_slots = 1 the
 *      fetch of offloaded layer l' starts only after the attention of that
 *      request's previous offloaded layer released the slot,
 *   3. per layer, attention (K1) waits only for the fetches whose destination
 *      is that layer - the stall of kvsim/latency.py:185-187, now physical.
 * Replaces the pricing call batch_decode_latency_fast at
 * kvsim/engine.py:715-734 with the execution it prices. */
OFB_API int ofb_runtime_decode_step(ofb_runtime* rt, const ofb_step_desc* desc, void* stream);

/* The same step split in three so a caller can interleave per-layer work of
 * its own on `stream` (e.g. a tensor-parallel o-projection + all-reduce after
 * each layer's attention): begin (step-start append, copy streams armed),
 * layers(count) (fetches + staging append + attention of the next `count`
 * layers), end.  The host arrays of `desc` must stay valid until end. */
OFB_API int ofb_runtime_step_begin(ofb_runtime* rt, const ofb_step_desc* desc, void* stream);
OFB_API int ofb_runtime_step_layers(ofb_runtime* rt, int32_t count);
OFB_API int ofb_runtime_step_end(ofb_runtime* rt);
/* Abandon a step begun with ofb_runtime_step_begin after a caller-side failure:
 * waits for the work already enqueued, drops any cross-step prefetch and leaves
 * the runtime ready for the next step.  Never fails on an idle runtime. */
OFB_API int ofb_runtime_step_abort(ofb_runtime* rt);
/* Make `stream` wait for every cross-step prefetch still in flight and drop
 * it (call before reusing staging or host slabs, e.g. after a plan change or a
 * released request). */
OFB_API int ofb_runtime_prefetch_fence(ofb_runtime* rt, void* stream);
/* Steps that adopted the previous step's prefetch / prefetches dropped on a plan mismatch. */
OFB_API int ofb_runtime_prefetch_stats(ofb_runtime* rt, int64_t* adopted, int64_t* dropped);

/* K4: plan-change reconfiguration.  Enqueue n whole-slab moves
 * (kind 0 = host->device restore, 1 = device->host eviction, 2 = device->device)
 * on the migration streams after all work already on `stream`.  `stream` (and
 * the next decode step) then waits for the restores; evictions overlap the next
 * step and only fetches of a slab still being evicted wait for them.  Realises
 * apply_plan (kvsim/engine.py:213-248), BlockTable.evict_for_space
 * (kvsim/engine.py:184-204) and reconfiguration_delta (kvsim/latency.py:277-297). */
OFB_API int ofb_runtime_migrate(ofb_runtime* rt, int32_t n, const uint64_t* dst, const uint64_t* src,
                        const int64_t* bytes, const int32_t* kinds, int32_t record_timing,
                        void* stream);

/* 1 while the last migration batch's evictions (D2H) are still in flight, else 0;
 * with wait != 0 it first blocks until they land.  Evicted HBM extents may be
 * reused only after this returns 0.  Restores (H2D) are always complete before
 * later work on the compute stream. */
OFB_API int ofb_runtime_migration_pending(ofb_runtime* rt, int32_t wait);

/* Timing of the last timed decode step / migration plus totals over all timed
 * steps (synchronises on their events; steps are timed into a 4-deep ring, so
 * the host can keep enqueuing without waiting). */
OFB_API int ofb_runtime_timing(ofb_runtime* rt, ofb_step_timing* out);
OFB_API int ofb_runtime_timing_reset(ofb_runtime* rt);
/* Per copy stream over the same timed steps: bytes fetched and busy time (sum of
 * that stream's copy spans); `streams` returns how many streams carried copies. */
OFB_API int ofb_runtime_stream_stats(ofb_runtime* rt, int32_t max_streams, double* bytes,
                                     double* busy_ms, int32_t* streams);

/* ---- K6 / C1: o-projection + all-reduce over peer memory (TP) ----------- */
/* after each layer's attention a KV-head-sharded rank holds
 * attn[B, Hq/N * 128] for its own heads; the decoder needs
 * hidden[B, H] = sum over ranks of attn_r @ W_o[rows of r]^T.  The reference
 * has no multi-GPU path; the paper runs NCCL after the projection
 * (PAPER.md:727-729).  One kernel does both: tcgen05 tensor cores compute this
 * rank's partial tile by tile (TMA-staged W_o rows, accumulator in TMEM) and
 * each finished tile is pushed straight into every peer's inbox over
 * NVLink (P2P stores into IPC-mapped symmetric buffers) and flagged; the last
 * CTA of a tile sums the world's copies of it in rank order, so every rank
 * ends with a bit-identical hidden state and the exchange overlaps the math
 * tile by tile.  world = 1 is the projection alone. */

/* Symmetric (IPC-shareable) device buffer: cudaMalloc'd, zeroed. */
OFB_API int ofb_symm_alloc(int64_t bytes, void** ptr);
OFB_API int ofb_symm_free(void* ptr);
/* CUDA IPC: 64-byte handle of a symm buffer; open a peer's handle (P2P enabled). */
OFB_API int ofb_ipc_get_handle(void* ptr, void* handle64);
OFB_API int ofb_ipc_open_handle(const void* handle64, void** ptr);
OFB_API int ofb_ipc_close_handle(void* ptr);

/* Bytes of each rank's symmetric buffer (inbox [2][world][hidden/128][max_batch][128]
 * bf16 + flags) and of its private workspace (split-K partials + tile tickets;
 * zero it once). */
OFB_API int64_t ofb_oproj_symm_bytes(int32_t world, int32_t max_batch, int32_t hidden);
OFB_API int64_t ofb_oproj_workspace_bytes(int32_t max_batch, int32_t k, int32_t hidden);

typedef struct ofb_oproj_desc {
  const void* x;       /* bf16 [layers][batch][k]: this rank's attention output, heads flattened */
  const void* w;       /* bf16 [layers][hidden][k]: W_o rows of this rank's heads (Linear layout) */
  void* out;           /* bf16 [batch][hidden]: the all-reduced result (same bits on every rank) */
  int32_t layers, layer, batch, k, hidden;
  void* workspace;
  int64_t workspace_bytes;
  int32_t world, rank, max_batch;   /* world <= 8; batch <= max_batch <= 256 */
  void* symm[8];       /* symm[r] = rank r's symmetric buffer as mapped here; symm[rank] local */
  uint32_t epoch;      /* > 0, +1 per call, identical on every rank */
  int32_t* status;     /* device int32: set to 1 if a peer's tile never arrived (timeout) */
  int64_t timeout_ns;  /* spin limit per tile wait (0 = 5 s) */
  int32_t w_layout;    /* 0: w is [layers][hidden][k] (Linear); 1: packed
                          [layers][hidden/128][k/64][128][64] - every TMA box a
                          contiguous 16 KiB (weights are static: pack once) */
  const void* residual; /* NULL, or bf16 [batch][hidden] added to the reduced sum before
                          the single rounding (the decoder's x += o_proj(attn)); may
                          alias `out`, identical on every rank */
  int32_t out_parts;    /* 0/1: `out` is [batch][hidden].  n in 2..4 (world 1 only): the
                          hidden columns are cut into n consecutive ranges of
                          part_cols[i] (multiples of 128) written to separate bf16
                          [batch][part_cols[i]] tensors part_out[i] - e.g. one launch for
                          the q / k / v projections straight into their own buffers */
  int32_t part_cols[4];
  void* part_out[4];
  /* Fused RMSNorm across two launches (the whole-decoder step; NULL = off):
   * ss_out: fp32 [hidden/128][max_batch] - per hidden tile, the sum over its 128
   *   columns of the final output^2 (after the residual add) of every batch row;
   * ss_in (world 1): fp32 [ss_tiles][max_batch] from a previous launch's ss_out (or
   *   ofb_row_sumsq): every output row b is scaled by rsqrt(sum_t ss_in[t][b] /
   *   (128 ss_tiles) + eps) - RMSNorm(x) . W^T with the norm weight folded into w. */
  float* ss_out;
  const float* ss_in;
  int32_t ss_tiles;
  float eps;
  /* swiglu = 1 (world 1, no residual / parts): w rows interleaved per 64 (gate rows
   * 64t..64t+63, then up rows 64t..64t+63, per 128-row tile); out is bf16
   * [batch][hidden/2] = silu(gate) * up of the rounded projections. */
  int32_t swiglu;
  /* x_layers: 0 = x holds `layers` layers and layer `layer` is read; 1 = x is one
   * bf16 [batch][k] input for every layer (the decoder's residual stream). */
  int32_t x_layers;
  /* K3 folded into a q/k/v projection (world 1, out_parts): parts kv_part and
   * kv_part + 1 are k and v of part_cols/128 local KV heads; each batch row's
   * token is also written to the paged pool at slot kv_positions[b] of block
   * kv_tables[b][pos/16] (bytes kv_block_bytes per block, layout of
   * ofb_kv_append), for rows whose kv_host_slabs[b] is 0 (NULL: all rows);
   * rows with a host slab are left to the runtime's append. NULL kv_pool = off. */
  void* kv_pool;
  const int32_t* kv_tables;     /* [batch][kv_max_blocks] of this layer */
  const int32_t* kv_positions;  /* [batch], < 0 = skip */
  const uint64_t* kv_host_slabs;
  int32_t kv_max_blocks;
  int32_t kv_part;
  int64_t kv_block_bytes;
} ofb_oproj_desc;

OFB_API int ofb_oproj_allreduce(const ofb_oproj_desc* desc, void* stream);

/* ---- decoder glue of the whole-decoder TP step (cfg4; not a north-star piece) */
/* out[r] = x[r] / sqrt(mean(x[r]^2) + eps) * weight, bf16 [rows][hidden], hidden % 8 == 0. */
OFB_API int ofb_rmsnorm(const void* x, const void* weight, void* out, int32_t rows, int32_t hidden,
                        float eps, void* stream);
/* act[b][i] = silu(gate_up[b][i]) * gate_up[b][inter + i], bf16, inter % 8 == 0. */
OFB_API int ofb_silu_mul(const void* gate_up, void* act, int32_t batch, int32_t inter, void* stream);
/* ss_out[t][b] = sum over columns 128t..128t+127 of x[b][c]^2 (fp32, row stride
 * ld_batch >= rows): the ss_in of the first fused-RMSNorm projection of a step. */
OFB_API int ofb_row_sumsq(const void* x, float* ss_out, int32_t rows, int32_t hidden, int32_t ld_batch,
                          void* stream);
/* Diagnostics: K6 launches write globaltimer stamps per CTA (entry, prologue done,
 * accumulator ready, cluster synced, output start, exit) into `device_buffer`
 * (uint64 [grid][8]); NULL switches tracing off. */
OFB_API int ofb_k6_trace(void* device_buffer);

/* ---- native exact placement solver (host code, no GPU needed) ---------- */
/* Bit-exact restatement of kvsim solve / solve_capacity_only
 * (kvsim/planner.py:437-560), multithreaded.  Balances follow the reference's
 * two seeds: `live_balance` / `parked_balance` = snapshot.get(id,
 * deposit_balance) (first-step pre-rejection, planner.py:470-483) and
 * `forecast_live` / `forecast_parked` = the forecast's seed
 * (planner.py:160-163). */
typedef struct ofb_plan_problem {
  int32_t num_layers, batch, num_paused, block_size;
  double compute_base_ms, compute_per_token_ms, bandwidth_blocks_per_ms;
  int64_t gpu_block_budget;
  double tbt_ms, violation_cap;
  int32_t window_min, window_max, current_step;
  int32_t mode;                   /* 0 = solve, 1 = solve_capacity_only */
  int32_t threads;
  const int64_t* total_tokens;    /* [batch] */
  const int64_t* blocks;          /* [batch] blocks per layer */
  const double* live_balance;     /* [batch] */
  const double* parked_balance;   /* [num_paused] */
  const double* forecast_live;    /* [batch] */
  const double* forecast_parked;  /* [num_paused] */
  int32_t* strides_out;           /* [batch] chosen stride, -1 = resident */
  int32_t device_enumerate;       /* 1: enumerate + sort the candidate space on the GPU
                                     (same order, same plan; needs a CUDA device) */
} ofb_plan_problem;

typedef struct ofb_plan_result {
  int32_t status;         /* 0 plan, 1 no placement fits the budget, 2 cap unsatisfiable */
  int32_t decode_window, expiry_step;
  int64_t candidates_feasible, candidates_priced, candidates_ranked;
  int32_t enumeration_windows;   /* device_enumerate: sorted windows materialised (bounded
                                    memory: the list is served in runs of whole keys) */
} ofb_plan_result;

OFB_API int ofb_plan_solve(const ofb_plan_problem* problem, ofb_plan_result* result);
OFB_API const char* ofb_plan_last_error(void);

/* Host-link probe: best-of-reps pinned cudaMemcpyAsync in each direction. */
OFB_API int ofb_link_probe(void* host, void* dev, int64_t bytes, int32_t reps, double* h2d_gbs,
                   double* d2h_gbs);

#ifdef __cplusplus
}
#endif

#endif /* ORBITFLOW_B200_H_ */
