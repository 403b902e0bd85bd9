// K1, persistent stream-K decomposition (variant 0; selectable, not the
// default: the split kernel - and the cluster kernel on latency-bound shapes -
// measured faster on every shape of profiles/r01_k1_sweep.md and
// profiles/r02_k1_variants.md).
//
// Same arithmetic as decode_attention.cu (attn_tile.cuh), different work
// split: all (request, kv head, block) tiles of the layer are flattened into
// one index space W (pair-major, pair = request * Hkv + head), and CTA c of a
// grid sized to 148 SMs x resident CTAs processes the contiguous range
// [c*W/G, (c+1)*W/G).  Every CTA therefore streams the same number of 8 KiB
// tiles (no tail wave, no per-split ramp), and the TMA producer keeps the ring
// full across pair boundaries while the consumers merge a finished pair.
// Only the first and last pair of a CTA's range can be shared with neighbour
// CTAs; those write (O, lse) partials to per-CTA slots and the last CTA of the
// pair to arrive (atomic ticket) combines them.  Pairs wholly inside one CTA
// are written directly.
//
// Launched with programmatic dependent launch: everything before the
// griddepcontrol.wait touches launch inputs only; with kv_ready (a layer with
// no fetch this step, whose KV the host knows complete) the TMA producer also
// starts streaming KV before the wait, so this layer's CTAs fill the SMs the
// previous kernel's early finishers free.  ofb_k1_trace records per-CTA
// timelines (tools/k1_trace.py).
#include <cstddef>

#include "attn_tile.cuh"

namespace ofb {

constexpr int kSConsumers = 4;
constexpr int kSThreads = (kSConsumers + 1) * 32;
constexpr int kSStages = 8;
constexpr int kSMaxBatch = 1024;
constexpr int kSMaxGrid = 448;   // >= 148 SMs x 2 resident CTAs
constexpr size_t kSRing = size_t(kSStages) * kHeadBlockBytes;
constexpr size_t kSCounterBytes = 65536;

using SMerge = MergeSlots<kSConsumers>;
static_assert(offsetof(SMerge, m) >= kMaxGroup * kSMaxGrid * sizeof(float) + kSMaxGrid * sizeof(int),
              "combine weights + segment offsets must fit before SMerge::m");

constexpr size_t kSSmemBytes = 1024 + kSRing + sizeof(SMerge) + 2 * kSStages * sizeof(uint64_t) +
                               (kSMaxBatch + 1) * sizeof(int) + 64;

struct StreamArgs {
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  const int32_t* block_tables;
  const int32_t* seq_lens;
  float* ws_o;        // [G][2][16][128]
  float* ws_lse;      // [G][2][16]
  int32_t* counters;  // [B * Hkv], zero at rest
  int max_blocks, batch, hq, hkv, group, grid;
  float scale_log2;
  int kv_ready;       // 1: KV is complete before the PDL wait - the producer may stream early
  unsigned long long* trace;  // diagnostics (ofb_k1_trace): per CTA globaltimer stamps, or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// trace slots per CTA: entry, past pdl_wait, first tile ready, last tile
// consumed, exit, SM id
constexpr int kTraceSlots = 6;

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

struct Space {
  const int* rp;  // rp[r] = blocks of requests < r (one head)
  int batch, hkv;
  long long W;
  int grid;

  __device__ long long start_of(int c) const { return (long long)c * W / grid; }
  __device__ long long pair_begin(int p) const {
    const int r = p / hkv, h = p - r * hkv;
    return (long long)rp[r] * hkv + (long long)h * (rp[r + 1] - rp[r]);
  }
  // pair containing global tile x (requests with zero blocks are skipped)
  __device__ int pair_of(long long x) const {
    int lo = 0, hi = batch - 1;  // last r with rp[r]*hkv <= x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((long long)rp[mid] * hkv <= x) lo = mid; else hi = mid - 1;
    }
    int r = lo;
    while (r + 1 < batch && rp[r + 1] == rp[r]) ++r;  // defensive: skip empty requests
    const int nb = rp[r + 1] - rp[r];
    const int h = (int)((x - (long long)rp[r] * hkv) / nb);
    return r * hkv + h;
  }
  __device__ int cta_of(long long x) const {
    int c = (int)(x * grid / W);
    if (c + 1 < grid && start_of(c + 1) <= x) ++c;
    return c;
  }
};

__global__ void __launch_bounds__(kSThreads, 2)
paged_gqa_decode_stream_kernel(const __grid_constant__ CUtensorMap kv_map, const StreamArgs a) {
  const int cta = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = a.group;
  unsigned long long* tr = (a.trace && tid == 0) ? a.trace + (size_t)cta * kTraceSlots : nullptr;
  if (tr) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tr[0] = gtimer();
    tr[5] = smid;
  }

  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  SMerge* ms = reinterpret_cast<SMerge*>(ring + kSRing);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ms) + sizeof(SMerge));
  uint64_t* empty = full + kSStages;
  int* rp = reinterpret_cast<int*>(empty + kSStages);
  int* flag = rp + kSMaxBatch + 1;

  // prefix of blocks per request (one head), warp 0
  if (warp == 0) {
    int carry = 0;
    for (int base = 0; base < a.batch; base += 32) {
      const int r = base + lane;
      int nb = r < a.batch ? (a.seq_lens[r] + kBlockTokens - 1) / kBlockTokens : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, nb, off);
        if (lane >= off) nb += v;
      }
      if (r < a.batch) rp[r + 1] = carry + nb;
      carry += __shfl_sync(0xffffffffu, nb, 31);
    }
    if (lane == 0) rp[0] = 0;
  }
  // ring barriers initialised in parallel (thread s: stage s), not by one thread
  if (tid == 0) prefetch_tma_desc(&kv_map);
  if (tid < kSStages) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // Everything above touched only launch inputs; the previous kernel on the
  // stream (an append into this layer's slabs, an o-projection producing q,
  // the previous layer's K1 sharing this workspace) must be complete past here.
  // With kv_ready the host guarantees this layer's KV was complete before the
  // previous kernel started, so the producer streams it while that kernel
  // drains (only the ring fills: consumers still wait for q).
  if (!(a.kv_ready && warp == kSConsumers)) pdl_wait();
  pdl_trigger();
  if (tr) tr[1] = gtimer();

  // Effective grid: the host sized it for max_seq_len; with shorter actual
  // sequences keep >= 1 tile per CTA so no CTA range is empty (ticket counts
  // below assume every CTA of a pair's span touches it).
  const long long W = (long long)rp[a.batch] * a.hkv;
  const int grid_eff = (int)(W < a.grid ? (W > 0 ? W : 1) : a.grid);
  Space sp{rp, a.batch, a.hkv, W, grid_eff};

  // empty requests: defined (zero) output, pairs spread over CTAs
  for (int p = cta; p < a.batch * a.hkv; p += a.grid) {
    const int r = p / a.hkv;
    if (rp[r + 1] == rp[r] && tid < kSConsumers * 32) {
      const int h = p - r * a.hkv;
      for (int i = tid; i < g * kHeadDim; i += kSConsumers * 32)
        a.out[((size_t)r * a.hq + h * g) * kHeadDim + i] = __float2bfloat16(0.f);
    }
  }
  if (sp.W == 0 || cta >= grid_eff) return;
  const long long begin = sp.start_of(cta), end = sp.start_of(cta + 1);
  const int n = (int)(end - begin);
  if (n <= 0) return;

  if (warp == kSConsumers) {
    // ------------------------------------------------------------ producer
    // Block ids are looked up 32 at a time, one batch ahead of the TMA issue,
    // so the ring never drains while a lookup is in flight.
    auto lookup = [&](int i) -> int {
      if (i >= n) return 0;
      const long long x = begin + i;
      const int p = sp.pair_of(x);
      const int r = p / a.hkv, h = p - r * a.hkv;
      const int lb = (int)(x - sp.pair_begin(p));
      const int blk = __ldg(&a.block_tables[(size_t)r * a.max_blocks + lb]);
      return (blk * a.hkv + h) * kTileRows;
    };
    int row_cur = lookup(lane);
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int row_next = lookup(i0 + 32 + lane);
      const int cnt = min(32, n - i0);
      for (int j = 0; j < cnt; ++j) {
        const int rj = __shfl_sync(0xffffffffu, row_cur, j);
        const int e = i0 + j, st = e % kSStages;
        if (e >= kSStages) mbar_wait(&empty[st], ((e / kSStages) - 1) & 1);
        if (elect_one()) {   // converged warp, elected lane issues
          uint8_t* dst = ring + (size_t)st * kHeadBlockBytes;
          mbar_arrive_expect_tx(&full[st], kHeadBlockBytes);
          tma_load_2d(dst, &kv_map, &full[st], 0, rj);
          tma_load_2d(dst + kHeadBlockBytes / 2, &kv_map, &full[st], 64, rj);
        }
        __syncwarp();
      }
      row_cur = row_next;
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int first_pair = sp.pair_of(begin);
  long long x = begin;
  while (x < end) {
    const int p = sp.pair_of(x);
    const long long pb = sp.pair_begin(p);
    const int r = p / a.hkv, h = p - r * a.hkv;
    const int nb = rp[r + 1] - rp[r];
    const long long pe = pb + nb;
    const long long seg_end = pe < end ? pe : end;
    const int seq = a.seq_lens[r];
    const size_t qrow0 = (size_t)r * a.hq + (size_t)h * g;

    uint32_t qa[8][4];
    load_q_frag(qa, a.q + qrow0 * kHeadDim, g, lane);
    WarpAttnState st;
    st.reset();
    const int e_lo = (int)(x - begin), e_hi = (int)(seg_end - begin);
    // ring entries are dealt round-robin by CTA-local entry index
    int e = e_lo + ((warp - e_lo % kSConsumers) + kSConsumers) % kSConsumers;
    for (; e < e_hi; e += kSConsumers) {
      const int s = e % kSStages;
      mbar_wait(&full[s], (e / kSStages) & 1);
      if (tr) {
        if (e == 0) tr[2] = gtimer();
        if (e + kSConsumers >= n) tr[3] = gtimer();
      }
      const int lb = (int)(begin + e - pb);
      const int valid = min(kBlockTokens, seq - lb * kBlockTokens);
      attend_tile(st, qa, ring + (size_t)s * kHeadBlockBytes, valid, a.scale_log2, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    publish_state(ms, st, warp, lane, g);
    consumer_bar();

    const bool whole = (pb >= begin) && (pe <= end);
    const int slot = (p == first_pair) ? 0 : 1;
    for (int idx = tid; idx < g * kHeadDim; idx += kSConsumers * 32) {
      const int row = idx / kHeadDim, d = idx - row * kHeadDim;
      float lse;
      const float v = merged_value(ms, row, d, &lse);
      if (whole) {
        a.out[(qrow0 + row) * kHeadDim + d] = __float2bfloat16(v);
      } else {
        a.ws_o[(((size_t)cta * 2 + slot) * kMaxGroup + row) * kHeadDim + d] = v;
        if (d == 0) a.ws_lse[((size_t)cta * 2 + slot) * kMaxGroup + row] = lse;
      }
    }
    if (!whole) {
      // last of the pair's CTAs to arrive combines its partials
      const int c_lo = sp.cta_of(pb), c_hi = sp.cta_of(pe - 1);
      consumer_bar();        // every partial write of the CTA happens-before thread 0's
      if (tid == 0) {        // gpu-scope fence + ticket (cumulative release)
        __threadfence();
        const int ticket = atomicAdd(&a.counters[p], 1);
        *flag = (ticket == c_hi - c_lo);
      }
      consumer_bar();
      if (*flag) {
        __threadfence();
        const int nseg = c_hi - c_lo + 1;
        // smem: weights [16][kSMaxGrid] in ms->o, per-segment partial offsets
        // after them, 1/sum per row in ms->l[0]
        float* wts = reinterpret_cast<float*>(ms);
        int* seg_off = reinterpret_cast<int*>(wts + kMaxGroup * kSMaxGrid);
        for (int k = tid; k < nseg; k += kSConsumers * 32) {
          const int c = c_lo + k;
          const int sl = (sp.pair_of(sp.start_of(c)) == p) ? 0 : 1;
          seg_off[k] = (c * 2 + sl) * kMaxGroup;   // row base of this segment's partial
        }
        consumer_bar();
        for (int row = warp; row < g; row += kSConsumers) {
          float M = -INFINITY;
          for (int k = lane; k < nseg; k += 32) {
            const float v = __ldcg(&a.ws_lse[seg_off[k] + row]);
            wts[row * kSMaxGrid + k] = v;
            M = fmaxf(M, v);
          }
#pragma unroll
          for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
          float S = 0.f;
          for (int k = lane; k < nseg; k += 32) {
            const float w = fast_exp2(wts[row * kSMaxGrid + k] - M);
            wts[row * kSMaxGrid + k] = w;
            S += w;
          }
#pragma unroll
          for (int off = 16; off; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
          if (lane == 0) ms->l[0][row] = 1.f / S;
        }
        consumer_bar();
        // thread = head-dim column; all g rows per segment in flight at once
        const int d = tid;
        float acc[kMaxGroup];
#pragma unroll
        for (int row = 0; row < kMaxGroup; ++row) acc[row] = 0.f;
        // 4 segments x g rows of loads in flight before any FMA (latency-bound tail)
        for (int k0 = 0; k0 < nseg; k0 += 4) {
          float v[4][kMaxGroup];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = k0 + u < nseg ? k0 + u : nseg - 1;
            const float* src = a.ws_o + (size_t)seg_off[k] * kHeadDim + d;
#pragma unroll
            for (int row = 0; row < kMaxGroup; ++row) v[u][row] = row < g ? __ldcg(src + row * kHeadDim) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (k0 + u >= nseg) break;
#pragma unroll
            for (int row = 0; row < kMaxGroup; ++row)
              if (row < g) acc[row] += wts[row * kSMaxGrid + k0 + u] * v[u][row];
          }
        }
#pragma unroll
        for (int row = 0; row < kMaxGroup; ++row)
          if (row < g) a.out[(qrow0 + row) * kHeadDim + d] = __float2bfloat16(acc[row] * ms->l[0][row]);
        if (tid == 0) a.counters[p] = 0;  // re-arm
      }
    }
    consumer_bar();  // merge scratch is reused by the next pair
    x = seg_end;
  }
  if (tr) tr[4] = gtimer();
}

// ------------------------------------------------------------------ host side

static unsigned long long* g_k1_trace = nullptr;
static int g_k1_trace_ctas = 448;
unsigned long long* k1_trace_buffer() { return g_k1_trace; }
int k1_trace_capacity() { return g_k1_trace_ctas; }
void set_k1_trace_buffer(void* buf, int ctas) {
  g_k1_trace = static_cast<unsigned long long*>(buf);
  g_k1_trace_ctas = ctas > 0 ? ctas : 448;
}

static int g_stream_occ = 0, g_stream_sms = 0;

static cudaError_t stream_init_once() {
  if (g_stream_occ > 0) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&g_stream_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(paged_gqa_decode_stream_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSSmemBytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, paged_gqa_decode_stream_kernel,
                                                    kSThreads, kSSmemBytes);
  if (e != cudaSuccess) return e;
  g_stream_occ = occ > 0 ? occ : 1;
  return cudaSuccess;
}

static int stream_grid(int batch, int hkv, int max_seq_len) {
  const long long nblk = (max_seq_len + kBlockTokens - 1) / kBlockTokens;
  const long long W = (long long)batch * hkv * nblk;
  long long G = (long long)g_stream_sms * g_stream_occ;
  const long long by_work = (W + 3) / 4;  // at least ~4 tiles per CTA
  if (G > by_work) G = by_work;
  if (G > kSMaxGrid) G = kSMaxGrid;
  return (int)(G < 1 ? 1 : G);
}

// Stream-K pays a combine over every CTA a pair spans; with few (request, kv
// head) pairs relative to the grid (e.g. one long request) fixed splits win.
bool stream_preferred(int batch, int hkv, int max_seq_len) {
  if (stream_init_once() != cudaSuccess) return false;
  if (batch > kSMaxBatch) return false;
  const int G = stream_grid(batch, hkv, max_seq_len);
  return (long long)batch * hkv * 32 >= G;
}

size_t attention_stream_workspace_bytes(int batch, int hq, int hkv, int max_seq_len) {
  (void)batch; (void)hq; (void)hkv; (void)max_seq_len;
  return kSCounterBytes + (size_t)kSMaxGrid * 2 * kMaxGroup * sizeof(float) +
         (size_t)kSMaxGrid * 2 * kMaxGroup * kHeadDim * sizeof(float);
}

cudaError_t launch_decode_attention_stream(const CUtensorMap& map, const void* q, void* out,
                                           const int32_t* block_tables, int max_blocks,
                                           const int32_t* seq_lens, void* workspace,
                                           size_t workspace_bytes, int batch, int hq, int hkv,
                                           int max_seq_len, float scale, cudaStream_t stream,
                                           bool kv_ready) {
  if (batch <= 0) return cudaSuccess;
  if (batch > kSMaxBatch || hkv <= 0 || hq % hkv != 0 || hq / hkv > kMaxGroup)
    return cudaErrorInvalidValue;
  if ((size_t)batch * hkv * sizeof(int32_t) > kSCounterBytes) return cudaErrorInvalidValue;
  cudaError_t e = stream_init_once();
  if (e != cudaSuccess) return e;
  if (workspace_bytes < attention_stream_workspace_bytes(batch, hq, hkv, max_seq_len))
    return cudaErrorInvalidValue;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  StreamArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.block_tables = block_tables;
  a.seq_lens = seq_lens;
  a.counters = reinterpret_cast<int32_t*>(ws);
  a.ws_lse = reinterpret_cast<float*>(ws + kSCounterBytes);
  a.ws_o = reinterpret_cast<float*>(ws + kSCounterBytes +
                                    (size_t)kSMaxGrid * 2 * kMaxGroup * sizeof(float));
  a.trace = k1_trace_buffer();
  a.kv_ready = kv_ready ? 1 : 0;
  a.max_blocks = max_blocks;
  a.batch = batch;
  a.hq = hq;
  a.hkv = hkv;
  a.group = hq / hkv;
  a.grid = stream_grid(batch, hkv, max_seq_len);
  a.scale_log2 = scale * 1.4426950408889634f;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(kSThreads);
  cfg.dynamicSmemBytes = kSSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, paged_gqa_decode_stream_kernel, map, a);
}

}  // namespace ofb
