// Native step runtime + C ABI (include/orbitflow_b200.h).
//
// K2 (offloaded-layer streaming) and K4 (plan-change migration) live here as
// copy-engine work ordered by CUDA events; K1/K3 launches are issued on the
// caller's compute stream.  One ofb_runtime_decode_step call enqueues a whole
// step (1 append + L attention launches + every slab fetch) without blocking
// the host, so the reference's Alg.-1 schedule (kvsim/latency.py:141-209) is
// enforced by the GPU itself rather than simulated.  A step also enqueues the
// next step's first fetches (cross-step prefetch), adopted by that step if its
// transfer plan is unchanged, so the copy engines never wait for the host.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/orbitflow_b200.h"
#include "common.cuh"

namespace ofb {
size_t attention_workspace_bytes(int batch, int hq, int hkv, int max_seq_len);
cudaError_t launch_decode_attention(const CUtensorMap& map, const void* q, void* out,
                                    const int32_t* block_tables, int max_blocks,
                                    const int32_t* seq_lens, void* workspace,
                                    size_t workspace_bytes, int batch, int hq, int hkv,
                                    int max_seq_len, float scale, cudaStream_t stream,
                                    int kv_ready = 0, bool standalone = false);
cudaError_t launch_kv_append(const void* k_new, const void* v_new, void* pool,
                             const int32_t* block_tables, int max_blocks,
                             const int32_t* positions, const uint64_t* host_slabs,
                             int num_layers, int batch, int hkv, int mode,
                             cudaStream_t stream, bool pdl = false);
int attention_occupancy();
int set_attention_variant(int variant);
int attention_variant_for(int batch, int hq, int hkv, int max_seq_len);
int attention_cluster_slots(int* slots);
int attention_cluster_plan(int batch, int hkv, int max_seq_len, const int* slots, int* C, int* P,
                           int* bps, int* stages);
int attention_split_plan(int batch, int hq, int hkv, int max_seq_len, int num_sms, int occupancy,
                         int* blocks_per_split, int* splits);
int attention_instep_plan(int batch, int hq, int hkv, int max_seq_len, int num_sms, int occupancy,
                          int* blocks_per_split, int* splits, int* narrow);
void set_k1_trace_buffer(void* buf, int ctas);
cudaError_t launch_kv_prefill(const void* k, const void* v, const uint64_t* dst, int num_layers,
                              int tokens, int hkv, cudaStream_t stream);
}  // namespace ofb

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code == 0 ? -1 : code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return static_cast<int>(e);
}

#define OFB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int load_encoder() {
  if (g_encode) return 0;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  OFB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || fn == nullptr)
    return fail(-1, "cuTensorMapEncodeTiled not available from the driver");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return 0;
}

// Tensor-map cache: the pool is described as a 2-D bf16 tensor of 128-wide
// rows (one token row of one head, K or V); one box = 32 rows (K tile + V tile
// of one (block, head)) x 64 columns, 128-byte swizzled.
struct MapCache {
  std::mutex mu;
  struct Entry {
    void* pool;
    int64_t blocks;
    int hkv;
    alignas(64) CUtensorMap map;
  };
  std::vector<Entry> entries;
};
MapCache g_maps;

int get_kv_map(void* pool, int64_t pool_blocks, int hkv, CUtensorMap* out) {
  std::lock_guard<std::mutex> lock(g_maps.mu);
  for (auto& e : g_maps.entries) {
    if (e.pool == pool && e.blocks == pool_blocks && e.hkv == hkv) {
      *out = e.map;
      return 0;
    }
  }
  int rc = load_encoder();
  if (rc) return rc;
  MapCache::Entry e;
  e.pool = pool;
  e.blocks = pool_blocks;
  e.hkv = hkv;
  const uint64_t rows = static_cast<uint64_t>(pool_blocks) * hkv * ofb::kTileRows;
  if (rows >= (1ull << 32)) return fail(-1, "kv pool too large for one tensor map");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ofb::kHeadDim), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ofb::kRowBytes)};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(ofb::kTileRows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(&e.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(-1, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  if (g_maps.entries.size() > 64) g_maps.entries.erase(g_maps.entries.begin());
  g_maps.entries.push_back(e);
  *out = e.map;
  return 0;
}

}  // namespace

// Helpers shared with the other translation units (oproj_allreduce.cu).
namespace ofb {
int report_error(int code, const char* msg) { return fail(code, msg); }
int report_cuda(cudaError_t e, const char* what) { return cuda_fail(e, what); }

// bf16 tensor map with 128-byte swizzle and zero fill out of bounds.
int encode_bf16_map(CUtensorMap* map, void* base, int rank, const uint64_t* dims,
                    const uint64_t* byte_strides, const uint32_t* box) {
  int rc = load_encoder();
  if (rc) return rc;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base,
                        reinterpret_cast<const cuuint64_t*>(dims),
                        reinterpret_cast<const cuuint64_t*>(byte_strides),
                        reinterpret_cast<const cuuint32_t*>(box), estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(-1, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return 0;
}
}  // namespace ofb

// ------------------------------------------------------------------ runtime

struct CopyTiming {
  cudaEvent_t start, stop;
  double bytes;
  int stream;
};

// Timing events of one step.  Steps are timed into a ring of records so the
// host never has to wait on step N to enqueue step N+1; a record is harvested
// (its events read and accumulated) when it is reused or on ofb_runtime_timing.
struct StepRecord {
  bool pending = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t start = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> attn;
  std::vector<CopyTiming> copies;
  int streams = 0;
};

struct StepValues {
  int32_t layers = 0, copies = 0, streams = 0;
  float attn_total = 0, attn_max = 0, copy_sum = 0, copy_span = 0, step = 0;
  double copy_bytes = 0;
};

constexpr int kTimingRing = 4;

// Next step's first fetches per request, enqueued at the end of a step.
struct PrefetchEntry {
  int b, layer, stream;
  uint64_t dst, src;
  int64_t bytes;
  cudaEvent_t done, t0, t1;   // t0/t1: timing, handed to the adopting step's record
};

constexpr int kPrefetchGens = kTimingRing + 1;   // timing events outlive the record that reads them

struct PrefetchRec {
  bool valid = false;
  std::vector<PrefetchEntry> entries;
  std::vector<cudaEvent_t> pool;               // timing-disabled, owned here
  std::vector<cudaEvent_t> tpool[kPrefetchGens];  // timing-enabled, per generation
  int gen = 0;
};

struct StepState {
  bool active = false;
  ofb_step_desc d{};
  cudaStream_t cs = nullptr;
  CUtensorMap map;
  StepRecord* rec = nullptr;
  std::vector<std::vector<int>> offl;
  std::vector<size_t> next;
  std::vector<cudaEvent_t> attn_done, fetch_done;
  std::vector<char> adopted;        // [L*B]: fetch already issued by the previous step's prefetch
  std::vector<char> waited_d2h;
  int nstreams = 0;
  bool any_fetch = false;
  int next_layer = 0;
};

struct ofb_runtime {
  StepState step;
  int device = 0;
  int max_streams = 16;
  std::vector<cudaStream_t> copy;
  cudaStream_t mig_h2d = nullptr, mig_d2h = nullptr;
  std::vector<cudaEvent_t> sync_events;  // timing-disabled, reused every step
  size_t next_sync = 0;
  StepRecord ring[kTimingRing];
  int ring_pos = 0;
  StepValues last;
  int32_t acc_steps = 0, acc_launches = 0;
  double acc_attn_ms = 0, acc_copy_bytes = 0, acc_step_ms = 0;
  // per copy stream, accumulated like the above: bytes and busy time (sum of copy spans)
  std::vector<double> acc_stream_bytes, acc_stream_ms;
  int streams_used = 0;
  // migration
  cudaEvent_t mig_done_h2d = nullptr, mig_done_d2h = nullptr;
  cudaEvent_t mig_t0 = nullptr, mig_t1 = nullptr, mig_t2 = nullptr;
  bool mig_timed = false;
  double mig_h2d_bytes = 0, mig_d2h_bytes = 0;
  // host ranges still being written by the last eviction batch (D2H); fetches
  // reading them wait for mig_done_d2h, everything else overlaps it
  std::vector<std::pair<uint64_t, uint64_t>> pending_d2h;
  PrefetchRec pf;
  int64_t pf_adopted = 0, pf_dropped = 0;
};

namespace {

int next_sync_event(ofb_runtime* rt, cudaEvent_t* ev) {
  if (rt->next_sync == rt->sync_events.size()) {
    cudaEvent_t e;
    OFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    rt->sync_events.push_back(e);
  }
  *ev = rt->sync_events[rt->next_sync++];
  return 0;
}

int next_timing_event(StepRecord* rec, cudaEvent_t* ev) {
  if (rec->next == rec->pool.size()) {
    cudaEvent_t e;
    OFB_CUDA(cudaEventCreate(&e));
    rec->pool.push_back(e);
  }
  *ev = rec->pool[rec->next++];
  return 0;
}

// Read a finished record's events into rt->last and the accumulators.
int harvest(ofb_runtime* rt, StepRecord* rec) {
  if (!rec->pending) return 0;
  rec->pending = false;
  StepValues v;
  v.streams = rec->streams;
  float ms = 0;
  for (auto& p : rec->attn) {
    OFB_CUDA(cudaEventSynchronize(p.second));
    OFB_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
    v.attn_total += ms;
    v.attn_max = std::max(v.attn_max, ms);
  }
  v.layers = static_cast<int32_t>(rec->attn.size());
  if (!rec->attn.empty()) {
    OFB_CUDA(cudaEventElapsedTime(&ms, rec->start, rec->attn.back().second));
    v.step = ms;
  }
  float first = 1e30f, lastc = 0.f;
  for (auto& c : rec->copies) {
    OFB_CUDA(cudaEventSynchronize(c.stop));
    OFB_CUDA(cudaEventElapsedTime(&ms, c.start, c.stop));
    v.copy_sum += ms;
    v.copy_bytes += c.bytes;
    if (static_cast<int>(rt->acc_stream_bytes.size()) <= c.stream) {
      rt->acc_stream_bytes.resize(c.stream + 1, 0.0);
      rt->acc_stream_ms.resize(c.stream + 1, 0.0);
    }
    rt->acc_stream_bytes[c.stream] += c.bytes;
    rt->acc_stream_ms[c.stream] += ms;
    float a = 0, b = 0;
    OFB_CUDA(cudaEventElapsedTime(&a, rec->start, c.start));
    OFB_CUDA(cudaEventElapsedTime(&b, rec->start, c.stop));
    first = std::min(first, std::max(a, 0.f));   // adopted prefetches began before the step
    lastc = std::max(lastc, b);
  }
  v.copies = static_cast<int32_t>(rec->copies.size());
  v.copy_span = rec->copies.empty() ? 0.f : lastc - first;
  rt->last = v;
  rt->acc_steps += 1;
  rt->acc_launches += v.layers;
  rt->acc_attn_ms += v.attn_total;
  rt->acc_copy_bytes += v.copy_bytes;
  rt->acc_step_ms += v.step;
  return 0;
}

int harvest_all(ofb_runtime* rt) {
  // oldest first: the record after ring_pos was written longest ago
  for (int i = 0; i < kTimingRing; ++i) {
    int rc = harvest(rt, &rt->ring[(rt->ring_pos + i) % kTimingRing]);
    if (rc) return rc;
  }
  return 0;
}

// Every stream in `waiters` waits for all in-flight prefetches; the record is dropped.
int prefetch_fence(ofb_runtime* rt, const std::vector<cudaStream_t>& waiters) {
  if (!rt->pf.valid) return 0;
  for (auto& e : rt->pf.entries)
    for (cudaStream_t w : waiters) OFB_CUDA(cudaStreamWaitEvent(w, e.done, 0));
  rt->pf.valid = false;
  rt->pf.entries.clear();
  return 0;
}

int ensure_streams(ofb_runtime* rt, int n) {
  while (static_cast<int>(rt->copy.size()) < n) {
    cudaStream_t s;
    OFB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rt->copy.push_back(s);
  }
  return 0;
}

}  // namespace

extern "C" {

const char* ofb_version(void) { return "orbitflow-b200 0.1 sm_100a"; }

const char* ofb_last_error(void) { return g_err.c_str(); }

int ofb_set_attention_kernel(int32_t variant) {
  if (variant < 0 || variant > 4)
    return fail(-1, "variant must be 0 (stream-K), 1 (split), 2 (auto), 3 (cluster) or 4 (split2)");
  return ofb::set_attention_variant(variant);
}

int ofb_attention_variant_for(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len) {
  return ofb::attention_variant_for(batch, num_kv_heads, num_kv_heads, max_seq_len);
}

int ofb_attention_cluster_plan(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len,
                               const int32_t* cluster_slots, int32_t* cluster,
                               int32_t* clusters_per_pair, int32_t* blocks_per_cta,
                               int32_t* stages) {
  if (!cluster_slots || !cluster || !clusters_per_pair || !blocks_per_cta || !stages ||
      max_seq_len < 0)
    return ofb::report_error(-1, "ofb_attention_cluster_plan: bad arguments");
  if (ofb::attention_cluster_plan(batch, num_kv_heads, max_seq_len, cluster_slots, cluster,
                                  clusters_per_pair, blocks_per_cta, stages) != 0)
    return ofb::report_error(1, "ofb_attention_cluster_plan: not a one-wave cluster shape");
  return 0;
}

int ofb_attention_cluster_slots(int32_t* slots) {
  if (!slots) return ofb::report_error(-1, "ofb_attention_cluster_slots: null pointer");
  if (ofb::attention_cluster_slots(slots) != 0)
    return ofb::report_error(1, "ofb_attention_cluster_slots: no device");
  return 0;
}

int ofb_attention_split_plan(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                             int32_t max_seq_len, int32_t num_sms, int32_t ctas_per_sm,
                             int32_t* blocks_per_split, int32_t* splits) {
  if (ofb::attention_split_plan(batch, num_q_heads, num_kv_heads, max_seq_len, num_sms, ctas_per_sm,
                                blocks_per_split, splits) != 0)
    return ofb::report_error(-1, "ofb_attention_split_plan: bad arguments");
  return 0;
}

int ofb_attention_instep_plan(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                              int32_t max_seq_len, int32_t num_sms, int32_t ctas_per_sm,
                              int32_t* blocks_per_split, int32_t* splits, int32_t* narrow) {
  if (ofb::attention_instep_plan(batch, num_q_heads, num_kv_heads, max_seq_len, num_sms, ctas_per_sm,
                                 blocks_per_split, splits, narrow) != 0)
    return ofb::report_error(-1, "ofb_attention_instep_plan: bad arguments");
  return 0;
}

int ofb_k1_trace(void* device_buffer) {
  ofb::set_k1_trace_buffer(device_buffer, 448);
  return 0;
}

int ofb_k1_trace_sized(void* device_buffer, int32_t ctas) {
  if (ctas < 1) return fail(-1, "ofb_k1_trace_sized: capacity must be >= 1 CTA");
  ofb::set_k1_trace_buffer(device_buffer, ctas);
  return 0;
}

int ofb_device_info(int32_t* num_sms, int32_t* attn_ctas_per_sm) {
  int dev = 0;
  OFB_CUDA(cudaGetDevice(&dev));
  int sms = 0;
  OFB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (num_sms) *num_sms = sms;
  if (attn_ctas_per_sm) *attn_ctas_per_sm = ofb::attention_occupancy();
  return 0;
}

void* ofb_host_alloc(int64_t bytes) {
  if (bytes <= 0) {
    g_err = "ofb_host_alloc: bytes must be > 0";
    return nullptr;
  }
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, static_cast<size_t>(bytes),
                                cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaHostAlloc");
    return nullptr;
  }
  return p;
}

int ofb_host_free(void* ptr) {
  if (ptr) OFB_CUDA(cudaFreeHost(ptr));
  return 0;
}

int64_t ofb_attention_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                      int32_t max_seq_len) {
  return static_cast<int64_t>(
      ofb::attention_workspace_bytes(batch, num_q_heads, num_kv_heads, max_seq_len));
}

static int check_shapes(int32_t batch, int32_t hq, int32_t hkv, int32_t head_dim) {
  if (head_dim != ofb::kHeadDim) return fail(-1, "head_dim must be 128");
  if (batch < 0 || hq <= 0 || hkv <= 0) return fail(-1, "batch/heads must be positive");
  if (hq % hkv != 0 || hq / hkv > 16) return fail(-1, "Hq must be a multiple of Hkv with group <= 16");
  return 0;
}

int ofb_decode_attention(const void* q, void* out, const void* kv_pool, int64_t pool_blocks,
                         const int32_t* block_tables, int32_t max_blocks,
                         const int32_t* seq_lens, void* workspace, int64_t workspace_bytes,
                         int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                         int32_t head_dim, int32_t max_seq_len, float scale, void* stream) {
  int rc = check_shapes(batch, num_q_heads, num_kv_heads, head_dim);
  if (rc) return rc;
  if (batch == 0) return 0;
  if (!q || !out || !kv_pool || !block_tables || !seq_lens || !workspace)
    return fail(-1, "ofb_decode_attention: null pointer");
  if (max_seq_len > max_blocks * ofb::kBlockTokens)
    return fail(-1, "max_seq_len exceeds the block-table width");
  CUtensorMap map;
  rc = get_kv_map(const_cast<void*>(kv_pool), pool_blocks, num_kv_heads, &map);
  if (rc) return rc;
  cudaError_t e = ofb::launch_decode_attention(
      map, q, out, block_tables, max_blocks, seq_lens, workspace,
      static_cast<size_t>(workspace_bytes), batch, num_q_heads, num_kv_heads, max_seq_len, scale,
      static_cast<cudaStream_t>(stream), /*kv_ready*/ 0, /*standalone*/ true);
  if (e != cudaSuccess) return cuda_fail(e, "paged_gqa_decode_kernel launch");
  return 0;
}

int ofb_kv_append(const void* k_new, const void* v_new, void* kv_pool,
                  const int32_t* block_tables, int32_t max_blocks, const int32_t* positions,
                  const uint64_t* host_slabs, int32_t num_layers, int32_t batch,
                  int32_t num_kv_heads, int32_t head_dim, void* stream) {
  if (head_dim != ofb::kHeadDim) return fail(-1, "head_dim must be 128");
  if (num_kv_heads <= 0 || num_kv_heads * 32 > 1024 * 64) return fail(-1, "bad num_kv_heads");
  if (!k_new || !v_new || !positions) return fail(-1, "ofb_kv_append: null pointer");
  if (block_tables && !kv_pool) return fail(-1, "ofb_kv_append: block tables need a pool");
  cudaError_t e = ofb::launch_kv_append(k_new, v_new, kv_pool, block_tables, max_blocks,
                                        positions, host_slabs, num_layers, batch, num_kv_heads,
                                        /*kAppendAll*/ 1, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "kv_append_kernel launch");
  return 0;
}

int ofb_kv_prefill(const void* k, const void* v, const uint64_t* dst, int32_t num_layers,
                   int32_t tokens, int32_t num_kv_heads, int32_t head_dim, void* stream) {
  if (head_dim != ofb::kHeadDim) return fail(-1, "head_dim must be 128");
  if (!k || !v || !dst) return fail(-1, "ofb_kv_prefill: null pointer");
  if (num_layers < 0 || tokens < 0 || num_kv_heads <= 0) return fail(-1, "ofb_kv_prefill: bad sizes");
  cudaError_t e = ofb::launch_kv_prefill(k, v, dst, num_layers, tokens, num_kv_heads,
                                         static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "kv_prefill_kernel launch");
  return 0;
}

ofb_runtime* ofb_runtime_create(int32_t max_copy_streams) {
  ofb_runtime* rt = new ofb_runtime();
  if (cudaGetDevice(&rt->device) != cudaSuccess) {
    g_err = "ofb_runtime_create: no CUDA device";
    delete rt;
    return nullptr;
  }
  rt->max_streams = std::max(1, std::min<int>(max_copy_streams, 64));
  bool ok = cudaStreamCreateWithFlags(&rt->mig_h2d, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&rt->mig_d2h, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&rt->mig_done_h2d, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&rt->mig_done_d2h, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreate(&rt->mig_t0) == cudaSuccess &&
            cudaEventCreate(&rt->mig_t1) == cudaSuccess &&
            cudaEventCreate(&rt->mig_t2) == cudaSuccess;
  if (!ok) {
    g_err = "ofb_runtime_create: stream/event creation failed";
    delete rt;
    return nullptr;
  }
  return rt;
}

int ofb_runtime_destroy(ofb_runtime* rt) {
  if (!rt) return 0;
  cudaDeviceSynchronize();
  for (auto s : rt->copy) cudaStreamDestroy(s);
  if (rt->mig_h2d) cudaStreamDestroy(rt->mig_h2d);
  if (rt->mig_d2h) cudaStreamDestroy(rt->mig_d2h);
  for (auto e : rt->sync_events) cudaEventDestroy(e);
  for (auto e : rt->pf.pool) cudaEventDestroy(e);
  for (auto& v : rt->pf.tpool)
    for (auto e : v) cudaEventDestroy(e);
  for (auto& rec : rt->ring)
    for (auto e : rec.pool) cudaEventDestroy(e);
  for (cudaEvent_t e : {rt->mig_done_h2d, rt->mig_done_d2h, rt->mig_t0, rt->mig_t1, rt->mig_t2})
    if (e) cudaEventDestroy(e);
  delete rt;
  return 0;
}

namespace {

// One decode step in progress: begin() validates and issues the step-start
// work, layers() enqueues fetches + compute for the next layers, end() checks
// that every fetch was issued.  Splitting lets a caller interleave per-layer
// work of its own (e.g. the TP o-projection + all-reduce) on the same stream.
int step_begin(ofb_runtime* rt, const ofb_step_desc* d, cudaStream_t cs) {
  StepState& st = rt->step;
  if (st.active) return fail(-1, "a decode step is already in progress");
  int rc = check_shapes(d->batch, d->num_q_heads, d->num_kv_heads, d->head_dim);
  if (rc) return rc;
  const int L = d->num_layers, B = d->batch;
  if (L <= 0) return fail(-1, "num_layers must be > 0");
  if (B <= 0) return fail(-1, "batch must be > 0");
  if (d->staging_slots < 1 || d->staging_slots > 8) return fail(-1, "staging_slots must be 1..8");
  if (!d->host_slabs || !d->staging_dst || !d->fetch_bytes)
    return fail(-1, "host transfer plan arrays are required");
  rc = get_kv_map(d->kv_pool, d->pool_blocks, d->num_kv_heads, &st.map);
  if (rc) return rc;
  st.d = *d;
  st.cs = cs;
  st.next_layer = 0;

  rt->next_sync = 0;
  st.rec = nullptr;
  if (d->record_timing) {
    st.rec = &rt->ring[rt->ring_pos];
    rt->ring_pos = (rt->ring_pos + 1) % kTimingRing;
    rc = harvest(rt, st.rec);  // step N-4: long finished in steady state
    if (rc) return rc;
    st.rec->next = 0;
    st.rec->attn.clear();
    st.rec->copies.clear();
    st.rec->pending = true;
  }
  StepRecord* rec = st.rec;

  // Per-request offload lists (layer order) -> this step's fetch schedule.
  st.offl.assign(B, {});
  st.any_fetch = false;
  for (int l = 0; l < L; ++l)
    for (int b = 0; b < B; ++b)
      if (d->host_slabs[(size_t)l * B + b] != 0) {
        st.offl[b].push_back(l);
        st.any_fetch = true;
      }
  st.nstreams = st.any_fetch ? std::min(B, rt->max_streams) : 0;
  rc = ensure_streams(rt, st.nstreams);
  if (rc) return rc;
  rt->streams_used = st.nstreams;
  if (rec) rec->streams = st.nstreams;

  // Adopt the previous step's prefetch if it fetched exactly this step's first
  // fetches per request (same slab, slot, size, stream); otherwise fence it.
  st.adopted.assign((size_t)L * B, 0);
  if (rt->pf.valid) {
    bool ok = st.nstreams > 0;
    for (auto& e : rt->pf.entries) {
      if (!ok) break;
      if (e.b >= B) { ok = false; break; }
      const auto& ol = st.offl[e.b];
      size_t k = 0;
      while (k < ol.size() && ol[k] != e.layer) ++k;
      const size_t idx = (size_t)e.layer * B + e.b;
      ok = k < ol.size() && k < (size_t)d->staging_slots && e.stream == e.b % st.nstreams &&
           e.dst == d->staging_dst[idx] && e.src == d->host_slabs[idx] && e.bytes == d->fetch_bytes[e.b];
    }
    if (ok) {
      size_t expected = 0;
      for (int b = 0; b < B; ++b) expected += std::min<size_t>(st.offl[b].size(), (size_t)d->staging_slots);
      ok = expected == rt->pf.entries.size();
    }
    if (ok) {
      for (auto& e : rt->pf.entries) {
        st.adopted[(size_t)e.layer * B + e.b] = 1;
        if (rec) rec->copies.push_back({e.t0, e.t1, static_cast<double>(e.bytes), e.stream});
      }
      rt->pf_adopted += 1;
      // the record stays valid until step_layers has consumed its events
    } else {
      std::vector<cudaStream_t> waiters(rt->copy.begin(), rt->copy.begin() + st.nstreams);
      waiters.push_back(cs);
      rc = prefetch_fence(rt, waiters);
      if (rc) return rc;
      rt->pf_dropped += 1;
    }
  }

  // Step start: the append of every resident row.  Copy streams start after
  // it (staging from the previous step released).  Offloaded rows get their
  // token after their fetch lands (step_layers), so a fetch moves exactly the
  // b_r blocks the reference's blocks_to_fetch counts.
  if (!rt->pending_d2h.empty() && cudaEventQuery(rt->mig_done_d2h) == cudaSuccess)
    rt->pending_d2h.clear();
  st.waited_d2h.assign(st.nstreams, 0);
  if (rec) {
    rc = next_timing_event(rec, &rec->start);
    if (rc) return rc;
    OFB_CUDA(cudaEventRecord(rec->start, cs));
  }
  if (!d->append_per_layer) {
    cudaError_t e = ofb::launch_kv_append(d->k_new, d->v_new, d->kv_pool, d->block_tables,
                                          d->max_blocks, d->positions, d->host_slabs_dev, L, B,
                                          d->num_kv_heads, /*kAppendResident*/ 0, cs);
    if (e != cudaSuccess) return cuda_fail(e, "kv_append_kernel launch");
  }
  cudaEvent_t ev_start;
  rc = next_sync_event(rt, &ev_start);
  if (rc) return rc;
  OFB_CUDA(cudaEventRecord(ev_start, cs));
  for (int s = 0; s < st.nstreams; ++s) OFB_CUDA(cudaStreamWaitEvent(rt->copy[s], ev_start, 0));
  st.attn_done.assign(L, nullptr);
  st.fetch_done.assign((size_t)L * B, nullptr);
  st.next.assign(B, 0);
  st.active = true;
  return 0;
}

int step_layers(ofb_runtime* rt, int count) {
  StepState& st = rt->step;
  if (!st.active) return fail(-1, "no decode step in progress");
  const ofb_step_desc* d = &st.d;
  const int L = d->num_layers, B = d->batch;
  const int S = d->staging_slots;
  const size_t q_layer = (size_t)B * d->num_q_heads * ofb::kHeadDim * 2;
  const size_t bt_layer = (size_t)B * d->max_blocks;
  cudaStream_t cs = st.cs;
  StepRecord* rec = st.rec;
  int rc = 0;
  cudaError_t e;
  const int stop = std::min(L, st.next_layer + std::max(count, 0));
  for (int l = st.next_layer; l < stop; ++l) {
    // Fetches whose staging slot is (or will be, in stream order) free.
    for (int b = 0; b < B; ++b) {
      while (st.next[b] < st.offl[b].size()) {
        const size_t k = st.next[b];
        const int dst_layer = st.offl[b][k];
        cudaStream_t s = rt->copy[b % st.nstreams];
        if (k >= (size_t)S) {
          const int prev = st.offl[b][k - S];
          if (prev >= l) break;  // that layer's attention is not enqueued yet
          OFB_CUDA(cudaStreamWaitEvent(s, st.attn_done[prev], 0));
        }
        const size_t idx = (size_t)dst_layer * B + b;
        if (st.adopted[idx]) {   // already in flight since the previous step
          for (auto& e : rt->pf.entries)
            if (e.b == b && e.layer == dst_layer) st.fetch_done[idx] = e.done;
          ++st.next[b];
          continue;
        }
        if (!rt->pending_d2h.empty() && !st.waited_d2h[b % st.nstreams]) {
          const uint64_t lo = d->host_slabs[idx], hi = lo + (uint64_t)d->fetch_bytes[b];
          for (auto& iv : rt->pending_d2h)
            if (lo < iv.second && iv.first < hi) {  // this slab is still being evicted
              OFB_CUDA(cudaStreamWaitEvent(s, rt->mig_done_d2h, 0));
              st.waited_d2h[b % st.nstreams] = 1;
              break;
            }
        }
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        if (rec) {
          if ((rc = next_timing_event(rec, &t0)) || (rc = next_timing_event(rec, &t1))) return rc;
          OFB_CUDA(cudaEventRecord(t0, s));
        }
        OFB_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(d->staging_dst[idx]),
                                 reinterpret_cast<const void*>(d->host_slabs[idx]),
                                 static_cast<size_t>(d->fetch_bytes[b]), cudaMemcpyHostToDevice, s));
        if (rec) {
          OFB_CUDA(cudaEventRecord(t1, s));
          rec->copies.push_back({t0, t1, static_cast<double>(d->fetch_bytes[b]), b % st.nstreams});
        }
        cudaEvent_t done;
        if ((rc = next_sync_event(rt, &done))) return rc;
        OFB_CUDA(cudaEventRecord(done, s));
        st.fetch_done[idx] = done;
        ++st.next[b];
      }
    }
    // Layer l: stall until its own fetches landed (latency.py:185-187), write
    // the new token into the staged slabs (and their host slabs), then attend.
    bool layer_fetches = false;
    for (int b = 0; b < B; ++b) {
      cudaEvent_t f = st.fetch_done[(size_t)l * B + b];
      if (f) {
        OFB_CUDA(cudaStreamWaitEvent(cs, f, 0));
        layer_fetches = true;
      }
    }
    if (layer_fetches || d->append_per_layer == 1) {
      const size_t kv_layer = (size_t)B * d->num_kv_heads * ofb::kHeadDim * 2;
      e = ofb::launch_kv_append(static_cast<const uint8_t*>(d->k_new) + l * kv_layer,
                                static_cast<const uint8_t*>(d->v_new) + l * kv_layer, d->kv_pool,
                                d->block_tables + l * bt_layer, d->max_blocks, d->positions,
                                d->host_slabs_dev + (size_t)l * B, 1, B, d->num_kv_heads,
                                d->append_per_layer == 1 ? /*kAppendAll*/ 1 : /*kAppendOffloaded*/ 2, cs,
                                /*pdl*/ d->append_per_layer && !layer_fetches);
      if (e != cudaSuccess) return cuda_fail(e, "kv_append_kernel launch");
    }
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (rec) {
      if ((rc = next_timing_event(rec, &t0)) || (rc = next_timing_event(rec, &t1))) return rc;
      OFB_CUDA(cudaEventRecord(t0, cs));
    }
    // KV of a layer with no fetch this step was complete before the previous
    // layer's K1 passed its dependency wait (step-start append), so K1 may stream
    // it before its own wait; q / outputs / workspace still wait.
    // (2: the whole-decoder step with K3 folded into the q/k/v projection - all of
    // the layer's KV but the blocks receiving this step's token predates it)
    // (the first layer of an ordinary step follows the step-start append: the same)
    const int kv_ready = (l > 0 && !layer_fetches && !d->append_per_layer) ? 1
                         : (!layer_fetches && (d->append_per_layer == 2 || (l == 0 && !d->append_per_layer))) ? 2
                                                                                                            : 0;
    e = ofb::launch_decode_attention(
        st.map, static_cast<const uint8_t*>(d->q) + l * q_layer,
        static_cast<uint8_t*>(d->out) + l * q_layer, d->block_tables + l * bt_layer, d->max_blocks,
        d->seq_lens, d->workspace, static_cast<size_t>(d->workspace_bytes), B, d->num_q_heads,
        d->num_kv_heads, d->max_seq_len, d->scale, cs, kv_ready);
    if (e != cudaSuccess) return cuda_fail(e, "paged_gqa_decode_kernel launch");
    if (rec) {
      OFB_CUDA(cudaEventRecord(t1, cs));
      rec->attn.push_back({t0, t1});
    }
    if (st.any_fetch) {
      cudaEvent_t done;
      if ((rc = next_sync_event(rt, &done))) return rc;
      OFB_CUDA(cudaEventRecord(done, cs));
      st.attn_done[l] = done;
    }
  }
  st.next_layer = stop;
  return 0;
}

int step_end(ofb_runtime* rt) {
  StepState& st = rt->step;
  if (!st.active) return fail(-1, "no decode step in progress");
  st.active = false;
  if (st.next_layer != st.d.num_layers) return fail(-1, "decode step ended before its last layer");
  for (int b = 0; b < st.d.batch; ++b)
    if (st.next[b] != st.offl[b].size()) return fail(-1, "internal: fetch schedule did not drain");
  // the adopted prefetch (if any) is consumed: its events were waited on above
  rt->pf.valid = false;
  rt->pf.entries.clear();
  const ofb_step_desc* d = &st.d;
  if (!d->next_fetch_bytes || !st.any_fetch) return 0;
  // Cross-step prefetch: the next step's first S fetches of every request, each
  // gated on the last attention of this step that read its staging slot (which
  // also orders it after this step's append into that host slab).
  const int B = d->batch, S = d->staging_slots;
  size_t n = 0;
  for (int b = 0; b < B; ++b) n += std::min<size_t>(st.offl[b].size(), (size_t)S);
  while (rt->pf.pool.size() < n) {
    cudaEvent_t e;
    OFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    rt->pf.pool.push_back(e);
  }
  auto& tp = rt->pf.tpool[rt->pf.gen];
  rt->pf.gen = (rt->pf.gen + 1) % kPrefetchGens;
  while (tp.size() < 2 * n) {
    cudaEvent_t e;
    OFB_CUDA(cudaEventCreate(&e));
    tp.push_back(e);
  }
  size_t used = 0;
  for (int b = 0; b < B; ++b) {
    const auto& ol = st.offl[b];
    const size_t K = ol.size();
    cudaStream_t s = rt->copy[b % st.nstreams];
    for (size_t k = 0; k < K && k < (size_t)S; ++k) {
      size_t j_last = k;
      while (j_last + S < K) j_last += S;   // last fetch of this step into slot k % S
      OFB_CUDA(cudaStreamWaitEvent(s, st.attn_done[ol[j_last]], 0));
      const size_t idx = (size_t)ol[k] * B + b;
      PrefetchEntry e{b, ol[k], b % st.nstreams, d->staging_dst[idx], d->host_slabs[idx],
                      d->next_fetch_bytes[b], rt->pf.pool[used], tp[2 * used], tp[2 * used + 1]};
      ++used;
      OFB_CUDA(cudaEventRecord(e.t0, s));
      OFB_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(e.dst), reinterpret_cast<const void*>(e.src),
                               static_cast<size_t>(e.bytes), cudaMemcpyHostToDevice, s));
      OFB_CUDA(cudaEventRecord(e.t1, s));
      OFB_CUDA(cudaEventRecord(e.done, s));
      rt->pf.entries.push_back(e);
    }
  }
  rt->pf.valid = !rt->pf.entries.empty();
  return 0;
}

}  // namespace

int ofb_runtime_decode_step(ofb_runtime* rt, const ofb_step_desc* d, void* stream_) {
  if (!rt || !d) return fail(-1, "ofb_runtime_decode_step: null argument");
  if (d->batch == 0) return 0;
  int rc = step_begin(rt, d, static_cast<cudaStream_t>(stream_));
  if (rc) return rc;
  rc = step_layers(rt, d->num_layers);
  if (rc) {
    rt->step.active = false;
    return rc;
  }
  return step_end(rt);
}

int ofb_runtime_step_begin(ofb_runtime* rt, const ofb_step_desc* d, void* stream_) {
  if (!rt || !d) return fail(-1, "ofb_runtime_step_begin: null argument");
  return step_begin(rt, d, static_cast<cudaStream_t>(stream_));
}

int ofb_runtime_step_layers(ofb_runtime* rt, int32_t count) {
  if (!rt) return fail(-1, "ofb_runtime_step_layers: null runtime");
  int rc = step_layers(rt, count);
  if (rc) rt->step.active = false;
  return rc;
}

int ofb_runtime_step_end(ofb_runtime* rt) {
  if (!rt) return fail(-1, "ofb_runtime_step_end: null runtime");
  return step_end(rt);
}

int ofb_runtime_step_abort(ofb_runtime* rt) {
  if (!rt) return fail(-1, "ofb_runtime_step_abort: null runtime");
  StepState& st = rt->step;
  const bool was_active = st.active;
  st.active = false;
  if (!was_active && !rt->pf.valid) return 0;
  if (st.cs) OFB_CUDA(cudaStreamSynchronize(st.cs));
  for (auto s : rt->copy) OFB_CUDA(cudaStreamSynchronize(s));
  rt->pf.valid = false;
  rt->pf.entries.clear();
  if (st.rec) st.rec->pending = false;
  return 0;
}

int ofb_runtime_prefetch_stats(ofb_runtime* rt, int64_t* adopted, int64_t* dropped) {
  if (!rt) return fail(-1, "ofb_runtime_prefetch_stats: null runtime");
  if (adopted) *adopted = rt->pf_adopted;
  if (dropped) *dropped = rt->pf_dropped;
  return 0;
}

int ofb_runtime_prefetch_fence(ofb_runtime* rt, void* stream) {
  if (!rt) return fail(-1, "ofb_runtime_prefetch_fence: null runtime");
  if (rt->step.active) return fail(-1, "ofb_runtime_prefetch_fence: a decode step is in progress");
  std::vector<cudaStream_t> waiters(rt->copy.begin(), rt->copy.end());
  waiters.push_back(static_cast<cudaStream_t>(stream));
  return prefetch_fence(rt, waiters);
}

int ofb_runtime_migrate(ofb_runtime* rt, int32_t n, const uint64_t* dst, const uint64_t* src,
                        const int64_t* bytes, const int32_t* kinds, int32_t record_timing,
                        void* stream_) {
  if (!rt) return fail(-1, "ofb_runtime_migrate: null runtime");
  if (n <= 0) return 0;
  if (!dst || !src || !bytes || !kinds) return fail(-1, "ofb_runtime_migrate: null array");
  cudaStream_t cs = static_cast<cudaStream_t>(stream_);
  cudaEvent_t ev;
  rt->next_sync = 0;
  int rc = next_sync_event(rt, &ev);
  if (rc) return rc;
  OFB_CUDA(cudaEventRecord(ev, cs));
  OFB_CUDA(cudaStreamWaitEvent(rt->mig_h2d, ev, 0));
  OFB_CUDA(cudaStreamWaitEvent(rt->mig_d2h, ev, 0));
  // a restore may read a host slab the previous eviction batch is still writing
  OFB_CUDA(cudaStreamWaitEvent(rt->mig_h2d, rt->mig_done_d2h, 0));
  rt->pending_d2h.clear();
  rt->mig_timed = record_timing != 0;
  if (rt->mig_timed) OFB_CUDA(cudaEventRecord(rt->mig_t0, cs));
  rt->mig_h2d_bytes = rt->mig_d2h_bytes = 0;
  for (int i = 0; i < n; ++i) {
    cudaMemcpyKind kind;
    cudaStream_t s;
    switch (kinds[i]) {
      case 0: kind = cudaMemcpyHostToDevice; s = rt->mig_h2d; rt->mig_h2d_bytes += bytes[i]; break;
      case 1:
        kind = cudaMemcpyDeviceToHost;
        s = rt->mig_d2h;
        rt->mig_d2h_bytes += bytes[i];
        if (bytes[i] > 0) rt->pending_d2h.emplace_back(dst[i], dst[i] + (uint64_t)bytes[i]);
        break;
      case 2: kind = cudaMemcpyDeviceToDevice; s = rt->mig_h2d; break;
      default: return fail(-1, "ofb_runtime_migrate: bad kind");
    }
    if (bytes[i] <= 0) continue;
    OFB_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst[i]), reinterpret_cast<const void*>(src[i]),
                             static_cast<size_t>(bytes[i]), kind, s));
  }
  OFB_CUDA(cudaEventRecord(rt->mig_done_h2d, rt->mig_h2d));
  OFB_CUDA(cudaEventRecord(rt->mig_done_d2h, rt->mig_d2h));
  if (rt->mig_timed) {
    OFB_CUDA(cudaEventRecord(rt->mig_t1, rt->mig_h2d));
    OFB_CUDA(cudaEventRecord(rt->mig_t2, rt->mig_d2h));
  }
  // Later compute (and, via its start event, the next step's fetches) waits for
  // the restores only.  Evictions (D2H) overlap the next step's H2D fetches on
  // the full-duplex link; only fetches of a slab still being written wait (see
  // ofb_runtime_decode_step), and the caller recycles evicted HBM extents only
  // once ofb_runtime_migration_pending() reports the batch done.
  OFB_CUDA(cudaStreamWaitEvent(cs, rt->mig_done_h2d, 0));
  return 0;
}

int ofb_runtime_migration_pending(ofb_runtime* rt, int32_t wait) {
  if (!rt) return fail(-1, "ofb_runtime_migration_pending: null runtime");
  if (rt->pending_d2h.empty()) return 0;
  if (wait) OFB_CUDA(cudaEventSynchronize(rt->mig_done_d2h));
  cudaError_t q = cudaEventQuery(rt->mig_done_d2h);
  if (q == cudaErrorNotReady) return 1;
  if (q != cudaSuccess) return cuda_fail(q, "cudaEventQuery(mig_done_d2h)");
  rt->pending_d2h.clear();
  return 0;
}

int ofb_runtime_timing(ofb_runtime* rt, ofb_step_timing* out) {
  if (!rt || !out) return fail(-1, "ofb_runtime_timing: null argument");
  std::memset(out, 0, sizeof(*out));
  int rc = harvest_all(rt);
  if (rc) return rc;
  const StepValues& v = rt->last;
  out->copy_streams = v.streams;
  out->layers = v.layers;
  out->attn_ms_total = v.attn_total;
  out->attn_ms_max = v.attn_max;
  out->copies = v.copies;
  out->copy_ms_sum = v.copy_sum;
  out->copy_bytes = v.copy_bytes;
  out->copy_span_ms = v.copy_span;
  out->step_ms = v.step;
  out->acc_steps = rt->acc_steps;
  out->acc_attn_launches = rt->acc_launches;
  out->acc_attn_ms = rt->acc_attn_ms;
  out->acc_copy_bytes = rt->acc_copy_bytes;
  out->acc_step_ms = rt->acc_step_ms;
  if (rt->mig_timed) {
    float a = 0, b = 0;
    OFB_CUDA(cudaEventSynchronize(rt->mig_t1));
    OFB_CUDA(cudaEventSynchronize(rt->mig_t2));
    OFB_CUDA(cudaEventElapsedTime(&a, rt->mig_t0, rt->mig_t1));
    OFB_CUDA(cudaEventElapsedTime(&b, rt->mig_t0, rt->mig_t2));
    out->mig_ms = std::max(a, b);
    out->mig_h2d_bytes = rt->mig_h2d_bytes;
    out->mig_d2h_bytes = rt->mig_d2h_bytes;
  }
  return 0;
}

int ofb_runtime_stream_stats(ofb_runtime* rt, int32_t max_streams, double* bytes, double* busy_ms,
                             int32_t* streams) {
  if (!rt) return fail(-1, "ofb_runtime_stream_stats: null runtime");
  int rc = harvest_all(rt);
  if (rc) return rc;
  const int n = static_cast<int>(rt->acc_stream_bytes.size());
  if (streams) *streams = n;
  for (int i = 0; i < n && i < max_streams; ++i) {
    if (bytes) bytes[i] = rt->acc_stream_bytes[i];
    if (busy_ms) busy_ms[i] = rt->acc_stream_ms[i];
  }
  return 0;
}

int ofb_runtime_timing_reset(ofb_runtime* rt) {
  if (!rt) return fail(-1, "ofb_runtime_timing_reset: null runtime");
  int rc = harvest_all(rt);
  if (rc) return rc;
  rt->acc_steps = rt->acc_launches = 0;
  rt->acc_attn_ms = rt->acc_copy_bytes = rt->acc_step_ms = 0;
  rt->acc_stream_bytes.clear();
  rt->acc_stream_ms.clear();
  return 0;
}

int ofb_link_probe(void* host, void* dev, int64_t bytes, int32_t reps, double* h2d_gbs,
                   double* d2h_gbs) {
  if (!host || !dev || bytes <= 0 || reps <= 0) return fail(-1, "ofb_link_probe: bad arguments");
  cudaStream_t s;
  cudaEvent_t a, b;
  OFB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  OFB_CUDA(cudaEventCreate(&a));
  OFB_CUDA(cudaEventCreate(&b));
  double best[2] = {0, 0};
  for (int dir = 0; dir < 2; ++dir) {
    for (int i = 0; i < reps; ++i) {
      OFB_CUDA(cudaEventRecord(a, s));
      if (dir == 0)
        OFB_CUDA(cudaMemcpyAsync(dev, host, (size_t)bytes, cudaMemcpyHostToDevice, s));
      else
        OFB_CUDA(cudaMemcpyAsync(host, dev, (size_t)bytes, cudaMemcpyDeviceToHost, s));
      OFB_CUDA(cudaEventRecord(b, s));
      OFB_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      OFB_CUDA(cudaEventElapsedTime(&ms, a, b));
      best[dir] = std::max(best[dir], (double)bytes / (ms * 1e-3) / 1e9);
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  if (h2d_gbs) *h2d_gbs = best[0];
  if (d2h_gbs) *d2h_gbs = best[1];
  return 0;
}

}  // extern "C"
