// K1, cluster variant: paged GQA decode attention for LATENCY-bound launches
// (few (request, KV head) pairs and short-to-medium contexts: cfg3's B=1 steps,
// the 70B TP8 shard at small batch).  Same math and tile routine as the split
// kernel (attn_tile.cuh); what changes is where the splits meet.
//
// The split kernel combines a pair's splits through global memory: every CTA
// writes (O, lse) partials, fences, takes an atomic ticket, and the last one
// reads all partials back from L2 - three dependent L2 round trips after the
// last tile.  Here the splits of a pair form a thread-block CLUSTER (C <= 16
// CTAs): after the 4-warp merge each CTA leaves its normalised O[g][128] and
// lse[g] in its own shared memory, one cluster barrier publishes them, and CTA
// c combines head-dim slice c of all C CTAs by DSMEM loads (one ~0.1 us
// round trip) and writes its slice of the output.  Pairs too long for one
// cluster get P clusters; each CTA then writes its combined slice as a partial
// and the last of the P CTAs owning that slice (a per-slice ticket, no cluster
// wide wait) combines P partials instead of P x C.
//
// Work: grid (C*P, Hkv, B), cluster (C,1,1); CTA `split` streams blocks
// [split*bps, split*bps + bps) of its request's table with TMA into a ring
// deep enough to hold the whole split when it fits (no ring recycling at the
// shapes this variant serves), 4 consumer warps run attend_tile.
// Reference cost this realises: per_layer_compute, kvsim/core.py:257-261.
#include <cooperative_groups.h>

#include <cstdlib>

#include "attn_tile.cuh"

namespace cg = cooperative_groups;

namespace ofb {

unsigned long long* k1_trace_buffer();
int k1_trace_capacity();

namespace {

constexpr int kCWarps = 4;                       // consumer warps
constexpr int kCThreads = (kCWarps + 1) * 32;    // + producer warp
constexpr int kCMaxStages = 24;
constexpr int kCMinStages = 5;                   // the 4-warp merge scratch overlays the ring
static_assert(kCMinStages > 4, "the consumer loop wraps the ring at most once per step");
constexpr int kCMaxCluster = 16;
constexpr int kCMaxBps = 256;
constexpr size_t kCCounterBytes = 65536;         // shared counter region (split kernel layout)
static_assert(sizeof(MergeSlots<kCWarps>) + sizeof(MergeWeights<kCWarps>) <=
                  size_t(kCMinStages) * kHeadBlockBytes,
              "the merge scratch overlays the shallowest ring");

struct ClusterArgs {
  const __nv_bfloat16* q;       // [B][Hq][128]
  __nv_bfloat16* out;           // [B][Hq][128]
  const int32_t* block_tables;  // [B][max_blocks]
  const int32_t* seq_lens;      // [B]
  float* ws_o;                  // [B*Hkv][P][g][128]  (P > 1 only)
  float* ws_lse;                // [B*Hkv][C][P][g]
  int32_t* counters;            // [B*Hkv][C], zero at rest
  int max_blocks, hq, hkv, group;
  int bps, stages, clusters;    // blocks per split, ring depth, P
  float scale_log2;
  int kv_ready;
  unsigned long long* trace;    // ofb_k1_trace_sized: 8 stamps per CTA, or null
  int trace_ctas;
};

// trace slots per CTA (12): entry, prologue, first tile ready, ring drained,
// CTA merge done, cluster barrier passed, DSMEM gather done, slice written,
// ticket taken, exit, -, SM id
__device__ __forceinline__ unsigned long long cl_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Shared memory tail after the ring (the ring itself is 1024-aligned).
struct ClusterTail {
  float res_o[kMaxGroup][kHeadDim];          // this CTA's normalised O (cluster-visible)
  float res_lse[kMaxGroup];                  // and its lse (log2 domain)
  int32_t blk_ids[kCMaxBps];
  int flag;
};

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

size_t cluster_smem_bytes(int stages) {
  return 1024 + (size_t)stages * kHeadBlockBytes + 2 * (size_t)stages * sizeof(uint64_t) +
         sizeof(ClusterTail) + 16;
}

// C (CTAs per cluster) is a template parameter: the slice / item index math
// becomes shifts and the shuffle reductions unroll.
template <int C>
__global__ void __launch_bounds__(kCThreads, 2)
paged_gqa_decode_cluster_kernel(const __grid_constant__ CUtensorMap kv_map, const ClusterArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank());
  const int split = blockIdx.x;
  const int pc = split / C;                  // cluster index within the pair
  const int kvh = blockIdx.y;
  const int req = blockIdx.z;
  const int pair = req * a.hkv + kvh;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const bool early = a.kv_ready != 0;
  if (!early) pdl_wait();
  pdl_trigger();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)a.stages * kHeadBlockBytes);
  uint64_t* empty = full + a.stages;
  ClusterTail* tl = reinterpret_cast<ClusterTail*>(ring + (size_t)a.stages * kHeadBlockBytes +
                                                   ((2 * a.stages * sizeof(uint64_t) + 15) & ~15u));
  unsigned long long* tr = nullptr;
  if (a.trace) {
    const int cta = pair * gridDim.x + split;
    if (cta < a.trace_ctas) tr = a.trace + (size_t)cta * 12;
  }
  if (tr && tid == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tr[0] = cl_gtimer();
    tr[11] = smid;
  }

  const int b_begin = split * a.bps;
  {
    const int span = min(a.bps, a.max_blocks - b_begin);
    const int32_t* bt = a.block_tables + (size_t)req * a.max_blocks + b_begin;
    for (int i = tid; i < span; i += kCThreads) tl->blk_ids[i] = bt[i];
  }
  const int seq = a.seq_lens[req];
  const int nblk = (seq + kBlockTokens - 1) / kBlockTokens;
  const int n = max(0, min(a.bps, nblk - b_begin));
  const int g = a.group;
  const int qh0 = kvh * g;

  // ring barriers initialised in parallel (thread s: stage s), not by one thread
  if (tid == 0) prefetch_tma_desc(&kv_map);
  if (tid < a.stages) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tr && tid == 0) tr[1] = cl_gtimer();

  WarpAttnState st;
  st.reset();
  if (warp == kCWarps) {
    // producer: the whole warp, converged; the elected lane issues
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < n; ++i) {
      if (i >= a.stages) mbar_wait(&empty[s], ph ^ 1u);
      if (elect_one()) {
        const int row = (tl->blk_ids[i] * a.hkv + kvh) * kTileRows;
        uint8_t* dst = ring + (size_t)s * kHeadBlockBytes;
        mbar_arrive_expect_tx(&full[s], kHeadBlockBytes);
        tma_load_2d(dst, &kv_map, &full[s], 0, row);
        tma_load_2d(dst + kHeadBlockBytes / 2, &kv_map, &full[s], 64, row);
      }
      __syncwarp();
      if (++s == a.stages) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else {
    if (early) pdl_wait();
    uint32_t qa[8][4];
    load_q_frag(qa, a.q + ((size_t)req * a.hq + qh0) * kHeadDim, g, lane);
    // stage / phase advance incrementally (stages >= kCMinStages > kCWarps: at most
    // one wrap per step) - no division by the runtime ring depth per tile
    int s = warp;
    uint32_t ph = 0;
    for (int i = warp; i < n; i += kCWarps) {
      mbar_wait(&full[s], ph);
      if (tr && i == 0 && lane == 0) tr[2] = cl_gtimer();
      const int valid = min(kBlockTokens, seq - (b_begin + i) * kBlockTokens);
      attend_tile(st, qa, ring + (size_t)s * kHeadBlockBytes, valid, a.scale_log2, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      s += kCWarps;
      if (s >= a.stages) {
        s -= a.stages;
        ph ^= 1u;
      }
    }
  }
  __syncthreads();   // ring drained
  if (tr && tid == 0) tr[3] = cl_gtimer();

  // ---- 4-warp merge into this CTA's cluster-visible result
  MergeSlots<kCWarps>* ms = reinterpret_cast<MergeSlots<kCWarps>*>(ring);
  MergeWeights<kCWarps>* mwt =
      reinterpret_cast<MergeWeights<kCWarps>*>(ring + sizeof(MergeSlots<kCWarps>));
  if (warp < kCWarps) publish_state<kCWarps>(ms, st, warp, lane, g);
  __syncthreads();
  merge_weights<kCWarps>(ms, mwt, g, tid);
  __syncthreads();
  for (int it = tid; it < g * (kHeadDim / 4); it += kCThreads) {
    const int row = it / (kHeadDim / 4);
    const int q4 = it - row * (kHeadDim / 4);
    *reinterpret_cast<float4*>(&tl->res_o[row][q4 * 4]) = merged_quad<kCWarps>(ms, mwt, row, q4);
  }
  if (tid < g) tl->res_lse[tid] = mwt->lse[tid];
  if (early) pdl_wait();        // the producer warp writes outputs / workspace below
  if (tr && tid == 0) tr[4] = cl_gtimer();
  cluster_arrive_release();     // publish res_o / res_lse to the cluster
  cluster_wait_acquire();
  if (tr && tid == 0) tr[5] = cl_gtimer();

  // ---- cluster combine of head-dim slice `crank` (W = 128 / C dims): one
  // group of C consecutive lanes per (row, 4 dims) item, lane s reading CTA s's
  // lse and float4 by DSMEM (a single round trip), weights / sums by shuffles.
  constexpr int W = kHeadDim / C;
  constexpr int Q = W / 4;      // float4 per row slice; Q * C == 32
  const bool single = a.clusters == 1;
  for (int base = 0; base < g * 32; base += kCThreads) {
    if (base + warp * 32 >= g * 32) break;        // warp-uniform
    const int t = base + tid;
    const int s = t % C;
    const int item = t / C;
    const int row = item / Q, qd = item - row * Q;
    const int d0 = crank * W + qd * 4;
    const float lse = dsmem_ld_f32(dsmem_map(&tl->res_lse[row], s));
    const float4 v = dsmem_ld_f4(dsmem_map(&tl->res_o[row][d0], s));
    float M = lse;
#pragma unroll
    for (int off = 1; off < C; off <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    const float w = M > -INFINITY ? fast_exp2(lse - M) : 0.f;
    float S = w;
    float4 acc = make_float4(w * v.x, w * v.y, w * v.z, w * v.w);
#pragma unroll
    for (int off = 1; off < C; off <<= 1) {
      S += __shfl_xor_sync(0xffffffffu, S, off);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
    }
    if (s == 0) {
      const float inv = S > 0.f ? 1.f / S : 0.f;
      acc = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      const size_t qrow = (size_t)req * a.hq + qh0 + row;
      if (single) {
        __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.out + qrow * kHeadDim + d0);
        dst[0] = __floats2bfloat162_rn(acc.x, acc.y);
        dst[1] = __floats2bfloat162_rn(acc.z, acc.w);
      } else {
        *reinterpret_cast<float4*>(a.ws_o + (((size_t)pair * a.clusters + pc) * g + row) * kHeadDim +
                                   d0) = acc;
        if (qd == 0)
          a.ws_lse[(((size_t)pair * C + crank) * a.clusters + pc) * g + row] =
              S > 0.f ? M + __log2f(S) : -INFINITY;
      }
    }
  }
  __syncthreads();
  if (tr && tid == 0) tr[6] = cl_gtimer();
  cluster_arrive_relaxed();     // every remote read of this CTA is done (exit guard)

  if (!single) {
    // ---- last of the P CTAs owning slice `crank` combines the P partials
    __syncthreads();
    if (tr && tid == 0) tr[7] = cl_gtimer();
    if (tid == 0) {
      const int ticket = ticket_acq_rel(&a.counters[pair * kCMaxCluster + crank]);
      tl->flag = (ticket == a.clusters - 1);
    }
    __syncthreads();
    if (tr && tid == 0) tr[8] = cl_gtimer();
    if (tl->flag) {
      // One L2 round trip: every item loads its P lse values and P partial
      // float4s together, then weighs them in registers.
      const int P = a.clusters;
      const float* lp = a.ws_lse + ((size_t)pair * C + crank) * P * g;
      for (int item = tid; item < g * Q; item += kCThreads) {
        const int row = item / Q, qd = item - row * Q;
        const int d0 = crank * W + qd * 4;
        // the lse values first (one round trip), partials in rounds of 8 loads
        float lv[kCMaxCluster];
#pragma unroll
        for (int p = 0; p < kCMaxCluster; ++p) lv[p] = p < P ? __ldcg(lp + p * g + row) : -INFINITY;
        float M = -INFINITY;
#pragma unroll
        for (int p = 0; p < kCMaxCluster; ++p) M = fmaxf(M, lv[p]);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float S = 0.f;
#pragma unroll
        for (int p0 = 0; p0 < kCMaxCluster; p0 += 8) {
          if (p0 >= P) break;
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p0 + u < P)
              v[u] = __ldcg(reinterpret_cast<const float4*>(
                  a.ws_o + (((size_t)pair * P + p0 + u) * g + row) * kHeadDim + d0));
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (p0 + u < P) {
              const float w = M > -INFINITY ? fast_exp2(lv[p0 + u] - M) : 0.f;
              S += w;
              acc.x += w * v[u].x;
              acc.y += w * v[u].y;
              acc.z += w * v[u].z;
              acc.w += w * v[u].w;
            }
          }
        }
        const float inv = S > 0.f ? 1.f / S : 0.f;
        const size_t qrow = (size_t)req * a.hq + qh0 + row;
        __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.out + qrow * kHeadDim + d0);
        dst[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
        dst[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
      }
      if (tid == 0) a.counters[pair * kCMaxCluster + crank] = 0;   // re-arm
    }
  }
  cluster_wait_acquire();       // no CTA leaves while a peer may still read its smem
  if (tr && tid == 0) tr[9] = cl_gtimer();
}

using ClusterKernel = void (*)(const CUtensorMap, const ClusterArgs);
constexpr ClusterKernel kClusterKernels[5] = {
    paged_gqa_decode_cluster_kernel<1>, paged_gqa_decode_cluster_kernel<2>,
    paged_gqa_decode_cluster_kernel<4>, paged_gqa_decode_cluster_kernel<8>,
    paged_gqa_decode_cluster_kernel<16>};

int g_cluster_init = 0;
// g_cluster_slots[k]: clusters of 2^k CTAs the GPU holds at once with one CTA
// per SM (the deepest ring), i.e. what one wave can place.
int g_cluster_slots[5] = {0, 0, 0, 0, 0};

cudaError_t cluster_init_once() {
  if (g_cluster_init) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  for (int k = 0; k < 5; ++k) {
    e = cudaFuncSetAttribute(kClusterKernels[k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)cluster_smem_bytes(kCMaxStages));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kClusterKernels[k], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  g_cluster_slots[0] = sms;
  for (int k = 1; k < 5; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1 << k, 1, 1);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = cluster_smem_bytes(kCMaxStages);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1 << k;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kClusterKernels[k], &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    g_cluster_slots[k] = n;
  }
  g_cluster_init = 1;
  return cudaSuccess;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

}  // namespace

// Cluster plan for a launch: C CTAs per cluster, P clusters per (request, KV
// head), bps blocks per CTA, ring depth.  The whole grid must fit one wave
// (pairs * P clusters of C <= slots[log2 C]) so no CTA waits for another's SM;
// the largest C that leaves every pair at least one cluster wins (fewer global
// partials), and P is capped so a CTA keeps at least OFB_K1_CLUSTER_MIN_BPS
// (default 4) blocks.
int attention_cluster_plan(int batch, int hkv, int max_seq_len, const int* slots, int* C_out,
                           int* P_out, int* bps_out, int* stages_out) {
  const int nblk = (max_seq_len + kBlockTokens - 1) / kBlockTokens;
  const long pairs = (long)batch * hkv;
  if (pairs < 1 || !slots) return -1;
  int cap = env_int("OFB_K1_CLUSTER", kCMaxCluster);     // tuning experiments only
  const int min_bps = env_int("OFB_K1_CLUSTER_MIN_BPS", 4) < 1 ? 1 : env_int("OFB_K1_CLUSTER_MIN_BPS", 4);
  const long want = nblk > 0 ? (nblk + min_bps - 1) / min_bps : 1;   // CTAs per pair at min_bps
  int C = 0, P = 0;
  for (int k = 4; k >= 0; --k) {
    const int c = 1 << k;
    if (c > cap || slots[k] < 1) continue;
    long p = slots[k] / pairs;
    if (p < 1) continue;
    if (c > want && k > 0) continue;          // more CTAs than blocks worth splitting
    const long pmax = (want + c - 1) / c;
    if (p > pmax) p = pmax;
    if (p > kCMaxCluster) p = kCMaxCluster;
    C = c;
    P = (int)p;
    break;
  }
  if (C == 0) return -1;                      // not one wave: not a cluster-kernel shape
  const int bps = nblk > 0 ? (nblk + C * P - 1) / (C * P) : 1;
  if (bps > kCMaxBps) return -1;
  *C_out = C;
  *P_out = P;
  *bps_out = bps;
  *stages_out = bps < kCMinStages ? kCMinStages : (bps > kCMaxStages ? kCMaxStages : bps);
  return 0;
}

int attention_cluster_slots(int* slots) {
  if (cluster_init_once() != cudaSuccess) return -1;
  for (int k = 0; k < 5; ++k) slots[k] = g_cluster_slots[k];
  return 0;
}

size_t attention_cluster_workspace_bytes(int batch, int hq, int hkv, int max_seq_len) {
  (void)max_seq_len;
  // P <= 16 partial rows per (pair, row) and C*P <= 256 lse entries
  return kCCounterBytes + (((size_t)batch * hq * 256 * sizeof(float) + 255) & ~size_t(255)) +
         (size_t)batch * hq * kCMaxCluster * kHeadDim * sizeof(float);
}

cudaError_t launch_decode_attention_cluster(const CUtensorMap& map, const void* q, void* out,
                                            const int32_t* block_tables, int max_blocks,
                                            const int32_t* seq_lens, void* workspace,
                                            size_t workspace_bytes, int batch, int hq, int hkv,
                                            int max_seq_len, float scale, cudaStream_t stream,
                                            bool kv_ready) {
  if (batch <= 0) return cudaSuccess;
  if (hkv <= 0 || hq % hkv != 0 || hq / hkv > kMaxGroup) return cudaErrorInvalidValue;
  if ((size_t)batch * hkv * kCMaxCluster * sizeof(int32_t) > kCCounterBytes)
    return cudaErrorInvalidValue;
  cudaError_t e = cluster_init_once();
  if (e != cudaSuccess) return e;
  int C, P, bps, stages;
  if (attention_cluster_plan(batch, hkv, max_seq_len, g_cluster_slots, &C, &P, &bps, &stages) != 0)
    return cudaErrorInvalidValue;
  const int g = hq / hkv;
  const size_t lse_bytes = ((size_t)batch * hkv * C * P * g * sizeof(float) + 255) & ~size_t(255);
  const size_t need = kCCounterBytes + lse_bytes + (size_t)batch * hkv * P * g * kHeadDim * 4;
  if (workspace_bytes < need) return cudaErrorInvalidValue;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  ClusterArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.block_tables = block_tables;
  a.seq_lens = seq_lens;
  a.counters = reinterpret_cast<int32_t*>(ws);
  a.ws_lse = reinterpret_cast<float*>(ws + kCCounterBytes);
  a.ws_o = reinterpret_cast<float*>(ws + kCCounterBytes + lse_bytes);
  a.max_blocks = max_blocks;
  a.hq = hq;
  a.hkv = hkv;
  a.group = g;
  a.bps = bps;
  a.stages = stages;
  a.clusters = P;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.kv_ready = kv_ready ? 1 : 0;
  a.trace = k1_trace_buffer();
  a.trace_ctas = a.trace ? k1_trace_capacity() : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * P, hkv, batch);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = cluster_smem_bytes(stages);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  int k = 0;
  while ((1 << k) < C) ++k;
  return cudaLaunchKernelEx(&cfg, kClusterKernels[k], map, a);
}

}  // namespace ofb
