// K1: paged GQA flash-decoding attention for one layer of a decode step.
//
// Realises what the reference only prices: per_layer_compute
// (/root/reference/pkg/src/kvsim/core.py:257-261) is the stand-in cost of this
// kernel; the paper's arithmetic is GQA decode over
// 16-token paged blocks in a per-request, layer-aware table
// (PAPER.md:750).
//
// Work decomposition: one CTA per (split, kv head, request).  A split is a
// contiguous run of `blocks_per_split` paged blocks of that request's table.
//   * warp 4 (producer): one elected lane streams the split's (block, head)
//     K+V tiles (8 KiB each) into an 8-stage shared-memory ring with TMA
//     (cp.async.bulk.tensor, 128B swizzle -> conflict-free ldmatrix).
//   * warps 0-3 (consumers): warp w takes ring entries w, w+4, ...; each does
//     S = Q.K^T and O += P.V for 16 tokens as mma.m16n8k16 tiles (the GQA
//     group, <=16 query heads, is the M dimension; tokens / head dims are N),
//     with an online softmax in registers (quad shuffles for row max).
//   * the 4 warp states merge through shared memory; multi-split requests
//     write (O, lse) partials and the last CTA of a (request, kv head) to
//     arrive (atomic ticket) combines them - no second launch.
#include "attn_tile.cuh"
#include <cstdlib>
#include <cstring>

namespace ofb {

// Two instantiations: narrow (4 consumer warps, 8-stage ring, two CTAs per SM)
// for bandwidth-bound launches, wide (8 consumer warps, 16 stages, one CTA per
// SM) for launches whose whole grid is one wave: there a CTA's own tile rate
// bounds the launch, and a second warp per scheduler hides the tile latency.
constexpr int kConsumerWarps = 4;
constexpr int kAttnThreads = (kConsumerWarps + 1) * 32;
constexpr int kStages = 8;
constexpr int kWideWarps = 8;
constexpr int kWideStages = 24;
constexpr int kMaxSplits = 256;
constexpr int kMaxBlocksPerSplit = 256;         // cost-model plans (both instantiations)
// the narrow instantiation's block-table run holds 512 entries so the balanced
// in-step plan (narrow only) reaches past 256 blocks per split; the wide one
// stays at 256: one more KiB would push its smem past the 196 KB carve-out and
// halve L1 (latency-bound launches measured 0.3-0.45 us slower)
constexpr int kMaxBlocksPerSplitNarrow = 512;
template <int kW>
constexpr int blk_cap() { return kW == kWideWarps ? kMaxBlocksPerSplit : kMaxBlocksPerSplitNarrow; }
// Split tickets live in a fixed region at the start of the workspace, sized for
// the largest (request x kv head) grid, so partials of a previous launch with
// a different batch can never alias a counter.
constexpr size_t kCounterRegionBytes = 65536;      // 16384 (request, kv head) pairs

struct AttnArgs {
  const __nv_bfloat16* q;       // [B][Hq][128]
  __nv_bfloat16* out;           // [B][Hq][128]
  const int32_t* block_tables;  // [B][max_blocks]
  const int32_t* seq_lens;      // [B]
  float* ws_o;                  // [B][Hq][max_splits][128]
  float* ws_lse;                // [B][Hq][max_splits]   (log2 domain)
  int32_t* counters;            // [B][Hkv], zero at rest
  int max_blocks;
  int hq, hkv, group;
  int blocks_per_split, max_splits;
  float scale_log2;
  int kv_ready;                 // 1: KV complete before the PDL wait (see the stream kernel);
                                // 2: all but each request's last block (the one receiving
                                //    this step's token, written by the predecessor)
  int defer_combine;            // 1: multi-split pairs stop after their partials (attn_combine_kernel)
  unsigned long long* trace;    // diagnostics (ofb_k1_trace): kSplitTraceSlots stamps per CTA
  int trace_ctas;               // capacity of `trace` in CTAs
};

// split-kernel trace slots per CTA: entry, prologue done (table + seq_lens +
// barriers), first tile ready, ring drained, partial written, ticket taken,
// exit, SM id
constexpr int kSplitTraceSlots = 8;

__device__ __forceinline__ unsigned long long split_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr size_t kRingBytes = size_t(kStages) * kHeadBlockBytes;
static_assert(sizeof(MergeSlots<kConsumerWarps>) + sizeof(MergeWeights<kConsumerWarps>) <= kRingBytes,
              "merge scratch must fit in the ring");
static_assert(kMaxGroup * kMaxSplits * sizeof(float) + kMaxGroup * 2 * sizeof(float) <= kRingBytes,
              "combine scratch must fit in the ring");

static_assert(sizeof(MergeSlots<kWideWarps>) + sizeof(MergeWeights<kWideWarps>) <=
                  size_t(kWideStages) * kHeadBlockBytes,
              "wide merge scratch must fit in the wide ring");

template <int kW, int kS>
constexpr size_t attn_smem_bytes() {
  return 1024 + size_t(kS) * kHeadBlockBytes + 2 * kS * sizeof(uint64_t) +
         blk_cap<kW>() * sizeof(int32_t) + 16;
}

constexpr size_t kAttnSmemBytes = 1024 /*align slack*/ + kRingBytes +
                                  2 * kStages * sizeof(uint64_t) +
                                  kMaxBlocksPerSplitNarrow * sizeof(int32_t) + 16;

// acc += sum_u w[s + u*parts] * src[(s + u*parts) rows]: N float4 partial loads
// in flight, then the FMAs in split order.
template <int N>
__device__ __forceinline__ void combine_round(float4& acc, const float4* __restrict__ src,
                                              const float* w, int s, int parts) {
  constexpr int kQuads = kHeadDim / 4;
  float4 v[N];
#pragma unroll
  for (int u = 0; u < N; ++u) v[u] = __ldcg(src + (size_t)(s + u * parts) * kQuads);
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const float wu = w[s + u * parts];
    acc.x += wu * v[u].x;
    acc.y += wu * v[u].y;
    acc.z += wu * v[u].z;
    acc.w += wu * v[u].w;
  }
}

template <int kW, int kS>
__device__ __forceinline__ void paged_gqa_decode_body(const CUtensorMap& kv_map, const AttnArgs& a) {
  constexpr int kThr = (kW + 1) * 32;
  constexpr size_t kRing = size_t(kS) * kHeadBlockBytes;
  const int split = blockIdx.x;
  const int kvh = blockIdx.y;
  const int req = blockIdx.z;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  unsigned long long* tr = nullptr;
  if (a.trace) {
    const int cta = (req * a.hkv + kvh) * gridDim.x + split;
    if (cta < a.trace_ctas) tr = a.trace + (size_t)cta * kSplitTraceSlots;
  }
  if (tr && tid == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tr[0] = split_gtimer();
    tr[7] = smid;
  }

  // see decode_attention_stream.cu: the predecessor must be complete before q,
  // outputs or workspace are touched; with kv_ready (host-guaranteed) the
  // launch inputs and this layer's KV may be read - and the producer stream it -
  // while the predecessor drains
  const bool early = a.kv_ready != 0;
  // kv_ready 3 (= 1 with a late wait): q and this layer's KV are launch inputs,
  // so the consumers run the whole split before waiting; only the global
  // writes (partials / out / ticket, which the predecessor's combine may still
  // read) follow the predecessor's completion
  const bool late = a.kv_ready == 3;
  if (!early) pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned, derived by an offset so the compiler keeps the shared space
  // (shared loads / stores instead of generic ones)
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kRing);
  uint64_t* empty = full + kS;
  int32_t* blk_ids = reinterpret_cast<int32_t*>(empty + kS);
  int* flag = blk_ids + blk_cap<kW>();
  // The split's table run is loaded speculatively (bounded by the row, not by
  // the sequence length) so it does not wait for the seq_lens round trip.
  const int b_begin = split * a.blocks_per_split;
  {
    const int span = min(a.blocks_per_split, a.max_blocks - b_begin);
    const int32_t* bt = a.block_tables + (size_t)req * a.max_blocks + b_begin;
    for (int i = tid; i < span; i += kThr) blk_ids[i] = bt[i];
  }
  const int seq = a.seq_lens[req];
  const int nblk = (seq + kBlockTokens - 1) / kBlockTokens;
  const int nsplit = (nblk + a.blocks_per_split - 1) / a.blocks_per_split;
  const int g = a.group;
  const int qh0 = kvh * g;

  if (nblk == 0) {  // empty request: defined output
    if (early) pdl_wait();
    if (split == 0) {
      for (int i = tid; i < g * kHeadDim; i += kThr)
        a.out[((size_t)req * a.hq + qh0) * kHeadDim + i] = __float2bfloat16(0.f);
    }
    if (tr && tid == 0) tr[6] = split_gtimer();
    return;
  }
  if (split >= nsplit) {
    if (tr && tid == 0) tr[6] = split_gtimer();
    return;
  }
  const int n = min(a.blocks_per_split, nblk - b_begin);

  // ring barriers initialised in parallel (thread s: stage s), not by one thread
  if (tid == 0) prefetch_tma_desc(&kv_map);
  if (tid < kS) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tr && tid == 0) tr[1] = split_gtimer();

  const float NEG_INF = -INFINITY;
  // per-lane softmax state (rows r0 and r0+8 of the padded 16-row group)
  float o[16][4];
  float m_run[2] = {NEG_INF, NEG_INF};
  float l_run[2] = {0.f, 0.f};
  const int r0 = lane >> 2;
  const int c0 = (lane & 3) * 2;

  if (warp == kW) {
    // ---------------------------------------------------------- producer
    // (the whole warp, converged; the elected lane issues)
    const int last_blk = (seq - 1) / kBlockTokens;   // block of this step's token
    for (int i = 0; i < n; ++i) {
      const int st = i % kS;
      if (i >= kS) mbar_wait(&empty[st], ((i / kS) - 1) & 1);
      if (a.kv_ready == 2 && b_begin + i == last_blk) pdl_wait();   // the token's K/V is the predecessor's
      if (elect_one()) {
        const int row = (blk_ids[i] * a.hkv + kvh) * kTileRows;
        uint8_t* dst = ring + (size_t)st * kHeadBlockBytes;
        mbar_arrive_expect_tx(&full[st], kHeadBlockBytes);
        tma_load_2d(dst, &kv_map, &full[st], 0, row);
        tma_load_2d(dst + kHeadBlockBytes / 2, &kv_map, &full[st], 64, row);
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------- consumers
    if (early && !late) pdl_wait();
    // Q as the A operand (rows = query heads of this group, zero padded).
    uint32_t qa[8][4];
    {
      const __nv_bfloat16* qb = a.q + ((size_t)req * a.hq + qh0) * kHeadDim;
      const bool v0 = r0 < g, v1 = (r0 + 8) < g;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int col = kk * 16 + c0;
        qa[kk][0] = v0 ? *reinterpret_cast<const uint32_t*>(qb + r0 * kHeadDim + col) : 0u;
        qa[kk][1] = v1 ? *reinterpret_cast<const uint32_t*>(qb + (r0 + 8) * kHeadDim + col) : 0u;
        qa[kk][2] = v0 ? *reinterpret_cast<const uint32_t*>(qb + r0 * kHeadDim + col + 8) : 0u;
        qa[kk][3] = v1 ? *reinterpret_cast<const uint32_t*>(qb + (r0 + 8) * kHeadDim + col + 8) : 0u;
      }
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;

    const int mi = lane >> 3;  // ldmatrix sub-matrix this lane addresses
    const int mr = lane & 7;
    for (int i = warp; i < n; i += kW) {
      const int st = i % kS;
      mbar_wait(&full[st], (i / kS) & 1);
      if (tr && i == 0 && lane == 0) tr[2] = split_gtimer();
      const uint32_t base = smem_u32(ring + (size_t)st * kHeadBlockBytes);
      const int tok0 = (b_begin + i) * kBlockTokens;
      const bool partial = tok0 + kBlockTokens > seq;
      if (partial) {
        // Slots past the sequence end hold whatever the block held before
        // (possibly NaN bit patterns): P is 0 there, but 0 * NaN poisons the
        // P.V tile, so clear those V rows (tile rows 16+valid..31, both halves).
        const int valid = seq - tok0;
        uint8_t* tile = ring + (size_t)st * kHeadBlockBytes;
        for (int c = lane; c < (kBlockTokens - valid) * 16; c += 32) {
          const int row = kBlockTokens + valid + (c >> 4);
          *reinterpret_cast<uint4*>(tile + ((c >> 3) & 1) * (kHeadBlockBytes / 2) + row * 128 +
                                    (c & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }

      // S = Q K^T over 16 tokens: s[j] covers tokens 8j..8j+7.
      float s[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(tile_addr(base, j * 8 + mr, kp * 4 + mi), b0, b1, b2, b3);
          mma_bf16_16816(s[j], qa[2 * kp], b0, b1);
          mma_bf16_16816(s[j], qa[2 * kp + 1], b2, b3);
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = s[j][e] * a.scale_log2;
          if (partial && (tok0 + j * 8 + c0 + (e & 1)) >= seq) v = NEG_INF;
          s[j][e] = v;
        }
      }
      float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
      float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m_run[0], mx0);
      const float mn1 = fmaxf(m_run[1], mx1);
      const float corr0 = fast_exp2(m_run[0] - mn0);
      const float corr1 = fast_exp2(m_run[1] - mn1);
      m_run[0] = mn0;
      m_run[1] = mn1;
      float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        s[j][0] = fast_exp2(s[j][0] - mn0);
        s[j][1] = fast_exp2(s[j][1] - mn0);
        s[j][2] = fast_exp2(s[j][2] - mn1);
        s[j][3] = fast_exp2(s[j][3] - mn1);
        rs0 += s[j][0] + s[j][1];
        rs1 += s[j][2] + s[j][3];
      }
      l_run[0] = l_run[0] * corr0 + rs0;
      l_run[1] = l_run[1] * corr1 + rs1;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        o[nt][0] *= corr0;
        o[nt][1] *= corr0;
        o[nt][2] *= corr1;
        o[nt][3] *= corr1;
      }
      // P (accumulator layout == A-operand layout for k16)
      uint32_t pa[4];
      pa[0] = pack_bf16(s[0][0], s[0][1]);
      pa[1] = pack_bf16(s[0][2], s[0][3]);
      pa[2] = pack_bf16(s[1][0], s[1][1]);
      pa[3] = pack_bf16(s[1][2], s[1][3]);
      // O += P V : V rows live at tile rows 16..31.
#pragma unroll
      for (int np = 0; np < 8; ++np) {
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(tile_addr(base, 16 + (mi & 1) * 8 + mr, 2 * np + (mi >> 1)), v0, v1, v2, v3);
        mma_bf16_16816(o[2 * np], pa, v0, v1);
        mma_bf16_16816(o[2 * np + 1], pa, v2, v3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 1);
    l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 2);
    l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 1);
    l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 2);
  }
  __syncthreads();  // ring drained: every issued TMA was consumed
  if (tr && tid == 0) tr[3] = split_gtimer();

  // -------------------------------------------------------- merge 4 warps
  MergeSlots<kW>* ms = reinterpret_cast<MergeSlots<kW>*>(ring);
  MergeWeights<kW>* mwt = reinterpret_cast<MergeWeights<kW>*>(
      ring + sizeof(MergeSlots<kW>));
  if (warp < kW) {   // only the g real query rows (the mma pads the group to 16)
    if (r0 < g) {
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
        *reinterpret_cast<float2*>(&ms->o[warp][r0][nt * 8 + c0]) = make_float2(o[nt][0], o[nt][1]);
      if ((lane & 3) == 0) {
        ms->m[warp][r0] = m_run[0];
        ms->l[warp][r0] = l_run[0];
      }
    }
    if (r0 + 8 < g) {
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
        *reinterpret_cast<float2*>(&ms->o[warp][r0 + 8][nt * 8 + c0]) = make_float2(o[nt][2], o[nt][3]);
      if ((lane & 3) == 0) {
        ms->m[warp][r0 + 8] = m_run[1];
        ms->l[warp][r0 + 8] = l_run[1];
      }
    }
  }
  __syncthreads();
  merge_weights<kW>(ms, mwt, g, tid);
  __syncthreads();
  if (late) pdl_wait();

  const bool single = (nsplit == 1);
  constexpr int kQ = kHeadDim / 4;
  for (int it = tid; it < g * kQ; it += kThr) {
    const int row = it / kQ;
    const int q4 = it - row * kQ;
    const float4 v = merged_quad<kW>(ms, mwt, row, q4);
    const size_t qrow = (size_t)req * a.hq + qh0 + row;
    if (single) {
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.out + qrow * kHeadDim + q4 * 4);
      dst[0] = __floats2bfloat162_rn(v.x, v.y);
      dst[1] = __floats2bfloat162_rn(v.z, v.w);
    } else {
      *reinterpret_cast<float4*>(a.ws_o + (qrow * a.max_splits + split) * kHeadDim + q4 * 4) = v;
      if (q4 == 0) a.ws_lse[qrow * a.max_splits + split] = mwt->lse[row];
    }
  }
  if (tr && tid == 0) tr[4] = split_gtimer();
  if (single || a.defer_combine) {
    if (tr && tid == 0) tr[6] = split_gtimer();
    return;
  }
  if (early) pdl_wait();   // the producer warp joins the combine below

  // ------------------------------------------- last CTA combines the splits
  __syncthreads();        // every partial write of the CTA happens-before thread 0's
  if (tid == 0) {         // acq_rel ticket (cumulative release, acquire for the winner)
    const int ticket = ticket_acq_rel(&a.counters[req * a.hkv + kvh]);
    *flag = (ticket == nsplit - 1);
  }
  __syncthreads();
  if (tr && tid == 0) tr[5] = split_gtimer();
  if (!*flag) {
    if (tr && tid == 0) tr[6] = split_gtimer();
    return;
  }

  float* wts = reinterpret_cast<float*>(ring);        // [16][nsplit]
  float* inv = wts + kMaxGroup * kMaxSplits;          // [16]
  for (int row = warp; row < g; row += kThr / 32) {
    const size_t qrow = (size_t)req * a.hq + qh0 + row;
    float M = NEG_INF;
    for (int s2 = lane; s2 < nsplit; s2 += 32) {
      const float v = __ldcg(&a.ws_lse[qrow * a.max_splits + s2]);
      wts[row * kMaxSplits + s2] = v;
      M = fmaxf(M, v);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float S = 0.f;
    for (int s2 = lane; s2 < nsplit; s2 += 32) {
      const float w = fast_exp2(wts[row * kMaxSplits + s2] - M);
      wts[row * kMaxSplits + s2] = w;
      S += w;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
    if (lane == 0) inv[row] = 1.f / S;
  }
  __syncthreads();
  // The combine reads g x nsplit partial rows of 512 B from L2 with one CTA, so
  // it is bound by loads in flight: a thread owns 4 dims of one row (a warp a
  // whole coalesced row), keeps 16 float4 loads in flight, and when the group is
  // small the splits are dealt round-robin to `parts` thread groups whose sums
  // meet in smem.
  constexpr int kQuads = kHeadDim / 4;
  const int items = g * kQuads;
  const int parts = items >= kThr ? 1 : kThr / items;
  float4* red = reinterpret_cast<float4*>(inv + kMaxGroup);   // [parts][items]
  for (int it = tid; it < items * parts; it += kThr) {
    const int item = it % items;
    const int part = it / items;
    const int row = item / kQuads;
    const int q4 = item - row * kQuads;
    const size_t qrow = (size_t)req * a.hq + qh0 + row;
    const float4* src = reinterpret_cast<const float4*>(a.ws_o + qrow * a.max_splits * kHeadDim) + q4;
    const float* w = wts + row * kMaxSplits;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int s2 = part;
    // rounds of 16, then 8, loads in flight (FMAs in split order after each
    // round), then at most 7 single loads
    for (; s2 + 15 * parts < nsplit; s2 += 16 * parts) combine_round<16>(acc, src, w, s2, parts);
    for (; s2 + 7 * parts < nsplit; s2 += 8 * parts) combine_round<8>(acc, src, w, s2, parts);
    for (; s2 < nsplit; s2 += parts) combine_round<1>(acc, src, w, s2, parts);
    if (parts == 1) {
      const float r = inv[row];
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.out + qrow * kHeadDim + q4 * 4);
      dst[0] = __floats2bfloat162_rn(acc.x * r, acc.y * r);
      dst[1] = __floats2bfloat162_rn(acc.z * r, acc.w * r);
    } else {
      red[part * items + item] = acc;
    }
  }
  if (parts > 1) {
    __syncthreads();
    for (int item = tid; item < items; item += kThr) {
      float4 acc = red[item];
      for (int p = 1; p < parts; ++p) {
        const float4 v = red[p * items + item];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      const int row = item / kQuads;
      const int q4 = item - row * kQuads;
      const float r = inv[row];
      const size_t qrow = (size_t)req * a.hq + qh0 + row;
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.out + qrow * kHeadDim + q4 * 4);
      dst[0] = __floats2bfloat162_rn(acc.x * r, acc.y * r);
      dst[1] = __floats2bfloat162_rn(acc.z * r, acc.w * r);
    }
  }
  if (tid == 0) a.counters[req * a.hkv + kvh] = 0;  // re-arm for the next launch
  if (tr && tid == 0) tr[6] = split_gtimer();
}

// Deferred combine (variant "split2"): a second, programmatically launched
// kernel merges the splits of every (request, KV head, query row) - one CTA each,
// the splits dealt to 4 thread groups (one row's 32 dim-quads per group) that
// stream lse + partial with an online rescale and meet in smem.  Replaces the
// split kernel's ticket (~0.9 us) and its one-CTA-per-pair serial combine.
__global__ void __launch_bounds__(128) attn_combine_kernel(const AttnArgs a) {
  // release the next kernel at once (the next layer's K1 may stream its KV
  // while this waits; it cannot touch q / out / the workspace before its own
  // wait, which follows this kernel's completion), then wait for every partial
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int seq = a.seq_lens[req];
  const int nblk = (seq + kBlockTokens - 1) / kBlockTokens;
  const int nsplit = (nblk + a.blocks_per_split - 1) / a.blocks_per_split;
  if (nsplit <= 1) return;               // written directly by the split kernel
  const int q4 = threadIdx.x & 31, part = threadIdx.x >> 5;
  const size_t qrow = (size_t)req * a.hq + kvh * a.group + row;
  const float4* src = reinterpret_cast<const float4*>(a.ws_o + qrow * a.max_splits * kHeadDim) + q4;
  const float* lse = a.ws_lse + qrow * a.max_splits;
  const float NEG_INF = -INFINITY;
  float M = NEG_INF, S = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s0 = part; s0 < nsplit; s0 += 4 * 16) {
    float lv[16];
    float4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int s2 = s0 + 4 * u;
      const bool ok = s2 < nsplit;
      lv[u] = ok ? __ldcg(lse + s2) : NEG_INF;
      v[u] = ok ? __ldcg(src + (size_t)s2 * (kHeadDim / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float mr = lv[0];
#pragma unroll
    for (int u = 1; u < 16; ++u) mr = fmaxf(mr, lv[u]);
    const float Mn = fmaxf(M, mr);
    const float sc = M > NEG_INF ? fast_exp2(M - Mn) : 0.f;
    S *= sc;
    acc = make_float4(acc.x * sc, acc.y * sc, acc.z * sc, acc.w * sc);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const float w = lv[u] > NEG_INF ? fast_exp2(lv[u] - Mn) : 0.f;
      S += w;
      acc.x += w * v[u].x;
      acc.y += w * v[u].y;
      acc.z += w * v[u].z;
      acc.w += w * v[u].w;
    }
    M = Mn;
  }
  __shared__ float sm_m[4][32], sm_s[4][32];
  __shared__ float4 sm_o[4][32];
  sm_m[part][q4] = M;
  sm_s[part][q4] = S;
  sm_o[part][q4] = acc;
  __syncthreads();
  if (part != 0) return;
  float Mt = NEG_INF;
#pragma unroll
  for (int p = 0; p < 4; ++p) Mt = fmaxf(Mt, sm_m[p][q4]);
  float St = 0.f;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 4; ++p) {           // part order: deterministic
    const float w = sm_m[p][q4] > NEG_INF ? fast_exp2(sm_m[p][q4] - Mt) : 0.f;
    St += w * sm_s[p][q4];
    o.x += w * sm_o[p][q4].x;
    o.y += w * sm_o[p][q4].y;
    o.z += w * sm_o[p][q4].z;
    o.w += w * sm_o[p][q4].w;
  }
  const float r = St > 0.f ? 1.f / St : 0.f;
  __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.out + qrow * kHeadDim + q4 * 4);
  dst[0] = __floats2bfloat162_rn(o.x * r, o.y * r);
  dst[1] = __floats2bfloat162_rn(o.z * r, o.w * r);
}

// The two instantiations, each with its own launch bounds (narrow: two CTAs per SM).
__global__ void __launch_bounds__(160, 2)
paged_gqa_decode_kernel(const __grid_constant__ CUtensorMap kv_map, const AttnArgs a) {
  paged_gqa_decode_body<kConsumerWarps, kStages>(kv_map, a);
}

__global__ void __launch_bounds__(288, 1)
paged_gqa_decode_wide_kernel(const __grid_constant__ CUtensorMap kv_map, const AttnArgs a) {
  paged_gqa_decode_body<kWideWarps, kWideStages>(kv_map, a);
}
static_assert((kConsumerWarps + 1) * 32 == 160 && (kWideWarps + 1) * 32 == 288,
              "launch bounds follow the warp counts");

// ------------------------------------------------------------------ host side

int encode_kv_map(CUtensorMap* map, void* pool, int64_t pool_blocks, int hkv);  // runtime.cu

struct AttnPlan {
  int blocks_per_split;
  int max_splits;
};

static int g_attn_occupancy = 0;
static int g_num_sms = 0;

static cudaError_t attn_init_once() {
  if (g_attn_occupancy > 0) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(paged_gqa_decode_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAttnSmemBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(paged_gqa_decode_wide_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)attn_smem_bytes<kWideWarps, kWideStages>());
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, paged_gqa_decode_kernel,
                                                    kAttnThreads, kAttnSmemBytes);
  if (e != cudaSuccess) return e;
  g_attn_occupancy = occ > 0 ? occ : 1;
  return cudaSuccess;
}

// Pick the split length for the widest request (cost model below); grids are
// sized against 148 SMs x resident CTAs per SM.
static AttnPlan plan_splits(int batch, int hq, int hkv, int max_seq_len, int num_sms, int occupancy) {
  const int nblk = (max_seq_len + kBlockTokens - 1) / kBlockTokens;
  AttnPlan p{1, 1};
  if (nblk <= 0) return p;
  const long pairs = (long)batch * hkv;
  int lo = (nblk + kMaxSplits - 1) / kMaxSplits;
  lo = lo < 1 ? 1 : lo;
  int hi = nblk < kMaxBlocksPerSplit ? nblk : kMaxBlocksPerSplit;
  if (lo > hi) lo = hi;
  // Cost model over power-of-two split lengths (profiles/r01_k1_bps_sweep.jsonl,
  // tools/k1_bps_sweep.py: on all 21 swept shapes its pick is within 2% of the
  // measured best):
  //   stream  = max(bytes / min(HBM, resident CTAs x per-CTA rate),
  //                 waves x split bytes / per-CTA rate)
  //   combine = splits x passes x per-split cost   (one CTA reads g x splits
  //             partial rows; passes = its 160 threads over g x 32 float4s)
  // A CTA streams ~40 GB/s alone, HBM reads top out near 6.5 TB/s, and a split
  // row pass costs ~50 ns in the combine (fitted to the sweep with the 16-deep
  // combine); power-of-two lengths also measured faster than their neighbours
  // (aligned 128 KiB runs of the table).
  constexpr double kCtaGBs = 40.0, kHbmGBs = 6500.0, kCombineUs = 0.05;
  const int group = hq / hkv;
  const long passes = (group * (kHeadDim / 4) + kAttnThreads - 1) / kAttnThreads;
  const long slots = (long)num_sms * occupancy;
  double best = 1e30;
  int bps = hi;
  for (int cand = 8; cand <= 256; cand *= 2) {
    int b = cand > nblk ? nblk : cand;
    if (b < lo) continue;
    const long ns = (nblk + b - 1) / b;
    const long ctas = pairs * ns;
    const double conc = (double)(ctas < slots ? ctas : slots);
    const double kb = (double)kHeadBlockBytes / 1e3;   // per block, in KB -> us at GB/s
    const double rate = conc * kCtaGBs < kHbmGBs ? conc * kCtaGBs : kHbmGBs;
    double t = (double)pairs * nblk * kb / rate;
    const double tw = (double)((ctas + slots - 1) / slots) * b * kb / kCtaGBs;
    t = t > tw ? t : tw;
    if (ns > 1) t += (double)ns * passes * kCombineUs;
    if (t < best - 1e-9) {
      best = t;
      bps = b;
    }
    if (cand >= nblk) break;
  }
  bps = bps < lo ? lo : (bps > hi ? hi : bps);
  p.blocks_per_split = bps;
  if (const char* f = std::getenv("OFB_K1_BPS")) {   // tuning experiments only
    const int v = std::atoi(f);
    if (v >= lo && v <= hi) p.blocks_per_split = v;
  }
  p.max_splits = (nblk + p.blocks_per_split - 1) / p.blocks_per_split;
  return p;
}

size_t attention_stream_workspace_bytes(int batch, int hq, int hkv, int max_seq_len);
unsigned long long* k1_trace_buffer();
int k1_trace_capacity();
cudaError_t launch_decode_attention_stream(const CUtensorMap& map, const void* q, void* out,
                                           const int32_t* block_tables, int max_blocks,
                                           const int32_t* seq_lens, void* workspace,
                                           size_t workspace_bytes, int batch, int hq, int hkv,
                                           int max_seq_len, float scale, cudaStream_t stream,
                                           bool kv_ready);

// K1 work decomposition: 0 = persistent stream-K, 1 = fixed splits + last-CTA
// combine, 3 = cluster splits with a DSMEM combine (decode_attention_cluster.cu),
// 2 = auto (default; OFB_K1=stream|split|cluster pins one).
static int g_k1_variant = -1;

static int k1_variant() {
  if (g_k1_variant < 0) {
    const char* v = std::getenv("OFB_K1");
    g_k1_variant = !v ? 2
                   : std::strcmp(v, "split") == 0   ? 1
                   : std::strcmp(v, "stream") == 0  ? 0
                   : std::strcmp(v, "cluster") == 0 ? 3
                   : std::strcmp(v, "split2") == 0  ? 4
                                                    : 2;
  }
  return g_k1_variant;
}

size_t attention_cluster_workspace_bytes(int batch, int hq, int hkv, int max_seq_len);
cudaError_t launch_decode_attention_cluster(const CUtensorMap& map, const void* q, void* out,
                                            const int32_t* block_tables, int max_blocks,
                                            const int32_t* seq_lens, void* workspace,
                                            size_t workspace_bytes, int batch, int hq, int hkv,
                                            int max_seq_len, float scale, cudaStream_t stream,
                                            bool kv_ready);

// Auto: the cluster kernel for latency-bound launches (the whole launch fits one
// wave of one-CTA-per-SM clusters and moves little data), the split kernel
// otherwise (with its plan it beat stream-K on every shape of
// profiles/r01_k1_sweep.md); stream-K stays selectable (variant 0).
int attention_cluster_slots(int* slots);
int attention_cluster_plan(int batch, int hkv, int max_seq_len, const int* slots, int* C, int* P,
                           int* bps, int* stages);

// Choice between the split kernel (global ticket + combine) and the cluster
// kernel (DSMEM combine) for launches whose consumers wait for the predecessor
// first (kv_ready 0 / 2: fetch layers, the whole-decoder step; attention-only
// in-step launches follow the late-wait policy in launch_decode_attention), from
// the all-resident step probe before the late wait
// (tools/small_step_probe.py, profiles/r02_k1_issue_loops.md): the cluster kernel
// wins with one cluster of <= 4 CTAs per (request, KV head) (8B / 70B at B 4-16,
// up to 8K) or one cluster with <= 20 blocks per CTA, and with >= 5 clusters per
// pair (the 70B TP8 shard at B = 1, 8K-32K); 2-4 clusters per pair lose 0.3-0.7 us.
static bool cluster_pick(int C, int P, int bps) {
  return (P == 1 && (C <= 4 || bps <= 20)) || (P >= 5 && bps <= 40);
}

bool cluster_preferred(int batch, int hq, int hkv, int max_seq_len) {
  (void)hq;
  int slots[5], C, P, bps, stages;
  if (attention_cluster_slots(slots) != 0) return false;
  if (attention_cluster_plan(batch, hkv, max_seq_len, slots, &C, &P, &bps, &stages) != 0)
    return false;
  return cluster_pick(C, P, bps);
}

// Standalone launches with <= 8 blocks per CTA of a picked cluster plan (1K
// contexts): the cluster kernel beat split2 there (4.9-5.4 vs 5.9-6.4 us).
static bool cluster_short(int batch, int hkv, int max_seq_len) {
  int slots[5], C, P, bps, stages;
  if (attention_cluster_slots(slots) != 0) return false;
  if (attention_cluster_plan(batch, hkv, max_seq_len, slots, &C, &P, &bps, &stages) != 0)
    return false;
  return cluster_pick(C, P, bps) && bps <= 8;
}

// Auto.  A standalone launch (the public entry point, which waits for its
// predecessor before streaming) with a one-wave, multi-split grid over <= 16
// pairs uses split2 (the separate combine kernel), unless a short cluster plan
// applies (profiles/r02_k1_split2.md, r02_k1_issue_loops.md).  Inside a step one
// kernel per layer is kept (split / cluster): the later layers stream their KV
// before the PDL wait, and a combine kernel between two layers cost 0.5 us per
// layer there (the next cluster K1 places its clusters around it).
static int pick_variant(int batch, int hq, int hkv, int max_seq_len, bool standalone = false) {
  const int v = k1_variant();
  if (v != 2) return v;
  if (standalone && attn_init_once() == cudaSuccess && hkv > 0 && hq % hkv == 0) {
    if (cluster_short(batch, hkv, max_seq_len)) return 3;
    const AttnPlan p = plan_splits(batch, hq, hkv, max_seq_len, g_num_sms, g_attn_occupancy);
    const long ctas = (long)p.max_splits * hkv * batch;
    // <= 16 (request, KV head) pairs: beyond that the last-CTA combine spreads over
    // enough CTAs and the extra launch costs more than it saves (8B B=4: 0.3 us)
    if (p.max_splits > 1 && (long)batch * hkv <= 16 && ctas <= (long)g_num_sms * g_attn_occupancy) return 4;
  }
  return cluster_preferred(batch, hq, hkv, max_seq_len) ? 3 : 1;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = std::getenv("OFB_PDL");
    on = (v && std::strcmp(v, "0") == 0) ? 0 : 1;
  }
  return on == 1;
}

// Host arithmetic only (no device): the split plan a launch would use on a GPU
// with `num_sms` SMs and `occupancy` resident K1 CTAs per SM.
int attention_split_plan(int batch, int hq, int hkv, int max_seq_len, int num_sms, int occupancy,
                         int* blocks_per_split, int* splits) {
  if (batch < 1 || hkv < 1 || hq % hkv != 0 || hq / hkv > kMaxGroup || max_seq_len < 0 ||
      num_sms < 1 || occupancy < 1 || !blocks_per_split || !splits)
    return -1;
  const AttnPlan p = plan_splits(batch, hq, hkv, max_seq_len, num_sms, occupancy);
  *blocks_per_split = p.blocks_per_split;
  *splits = p.max_splits;
  return 0;
}

int attention_variant_for(int batch, int hq, int hkv, int max_seq_len) {
  return pick_variant(batch, hq, hkv, max_seq_len, /*standalone*/ true);
}

int set_attention_variant(int variant) {
  const int prev = k1_variant();
  if (variant >= 0 && variant <= 4) g_k1_variant = variant;
  return prev;
}

static size_t split_workspace_bytes(int batch, int hq, int hkv, int max_seq_len);

size_t attention_workspace_bytes(int batch, int hq, int hkv, int max_seq_len) {
  const size_t a = split_workspace_bytes(batch, hq, hkv, max_seq_len);
  const size_t b = attention_stream_workspace_bytes(batch, hq, hkv, max_seq_len);
  const size_t c = attention_cluster_workspace_bytes(batch, hq, hkv, max_seq_len);
  const size_t ab = a > b ? a : b;
  return ab > c ? ab : c;
}

static size_t split_workspace_bytes(int batch, int hq, int hkv, int max_seq_len) {
  const int nblk = (max_seq_len + kBlockTokens - 1) / kBlockTokens;
  int splits = nblk < 1 ? 1 : nblk;
  if (splits > kMaxSplits) splits = kMaxSplits;
  const size_t counters = kCounterRegionBytes;
  const size_t lse = ((size_t)batch * hq * splits * sizeof(float) + 255) & ~size_t(255);
  const size_t o = (size_t)batch * hq * splits * kHeadDim * sizeof(float);
  return counters + lse + o;
}

// Balanced in-step plan: one narrow CTA per SM less one SM per (request, KV
// head) pair (that pair's combining CTA), so every SM holds one CTA of this
// layer and the next layer's CTAs fit beside it.  {0, 0} when the split length
// would exceed the kernel's limits.
static AttnPlan balanced_plan(int batch, int hkv, int max_seq_len, int num_sms) {
  AttnPlan p{0, 0};
  const int nblk = (max_seq_len + kBlockTokens - 1) / kBlockTokens;
  if (nblk <= 0) return p;
  const long pairs = (long)batch * hkv;
  long ns = ((long)num_sms - pairs) / pairs;
  ns = ns < 1 ? 1 : ns;
  const int bps = (int)((nblk + ns - 1) / ns);
  if (bps > kMaxBlocksPerSplitNarrow || (nblk + bps - 1) / bps > kMaxSplits) return p;
  p.blocks_per_split = bps;
  p.max_splits = (nblk + bps - 1) / bps;
  return p;
}

// Where the balanced plan beat the cost-model plan in a step (k1_instep_sweep:
// 8B and 70B TP8-shard heads, B 1-16, 1K-64K): enough blocks per CTA, or few
// splits per pair; never with many splits per pair (the combine grows with them).
static bool balanced_preferred(const AttnPlan& p, int group) {
  const int ns = p.max_splits, bps = p.blocks_per_split;
  if (ns > 80) return false;
  return bps >= 30 || ns <= 8 || (group <= 4 && bps >= 16);
}

cudaError_t launch_decode_attention(const CUtensorMap& map, const void* q, void* out,
                                    const int32_t* block_tables, int max_blocks,
                                    const int32_t* seq_lens, void* workspace,
                                    size_t workspace_bytes, int batch, int hq, int hkv,
                                    int max_seq_len, float scale, cudaStream_t stream,
                                    int kv_ready, bool standalone) {
  if (batch <= 0) return cudaSuccess;
  // In-step attention-only launches (kv_ready 1: q and KV are launch inputs, the
  // split kernel's consumers wait for the previous layer only before their global
  // writes, so consecutive layers overlap): the split kernel, on the balanced
  // narrow plan (one CTA per SM less one per (request, KV head) pair, so the next
  // layer's CTAs co-reside) where it measured best, else on the cost-model plan
  // (tools/k1_instep_sweep.py, profiles/r02_k1_instep.md: with the late wait the
  // split kernel beat the cluster kernel in a step on every swept shape but one
  // 1K case).  OFB_K1_INSTEP=split|bal|cluster pins one (tuning only; read at
  // every launch).
  int instep = 0;   // 0 auto, 1 split (cost-model plan), 2 balanced narrow, 3 cluster
  AttnPlan bal{0, 0};
  if (kv_ready == 1 && hkv > 0 && hq % hkv == 0) {
    if (const char* f = std::getenv("OFB_K1_INSTEP")) {
      instep = std::strcmp(f, "split") == 0 ? 1 : std::strcmp(f, "bal") == 0 ? 2
               : std::strcmp(f, "cluster") == 0 ? 3 : 0;
    }
    if (attn_init_once() == cudaSuccess) bal = balanced_plan(batch, hkv, max_seq_len, g_num_sms);
    if (instep == 0 && k1_variant() == 2)
      instep = (bal.max_splits > 0 && balanced_preferred(bal, hq / hkv)) ? 2 : 1;
  }
  int variant = pick_variant(batch, hq, hkv, max_seq_len, standalone);
  if (instep == 3) {
    int slots[5], C, P, bps, stages;
    if (attention_cluster_slots(slots) == 0 &&
        attention_cluster_plan(batch, hkv, max_seq_len, slots, &C, &P, &bps, &stages) == 0)
      variant = 3;
  } else if (instep == 1 || instep == 2) {
    variant = 1;
  }
  if (variant == 3)
    return launch_decode_attention_cluster(map, q, out, block_tables, max_blocks, seq_lens,
                                           workspace, workspace_bytes, batch, hq, hkv,
                                           max_seq_len, scale, stream, kv_ready == 1);
  if (variant == 0)
    return launch_decode_attention_stream(map, q, out, block_tables, max_blocks, seq_lens,
                                          workspace, workspace_bytes, batch, hq, hkv, max_seq_len,
                                          scale, stream, kv_ready == 1);
  if (hkv <= 0 || hq % hkv != 0 || hq / hkv > kMaxGroup) return cudaErrorInvalidValue;
  if ((size_t)batch * hkv * sizeof(int32_t) > kCounterRegionBytes) return cudaErrorInvalidValue;
  cudaError_t e = attn_init_once();
  if (e != cudaSuccess) return e;
  if (workspace_bytes < split_workspace_bytes(batch, hq, hkv, max_seq_len))
    return cudaErrorInvalidValue;
  AttnPlan plan = plan_splits(batch, hq, hkv, max_seq_len, g_num_sms, g_attn_occupancy);
  const int nblk = (max_seq_len + kBlockTokens - 1) / kBlockTokens;
  const bool force_narrow = instep == 2 && bal.max_splits > 0;
  if (force_narrow) plan = bal;
  int ws_splits = nblk < 1 ? 1 : nblk;
  if (ws_splits > kMaxSplits) ws_splits = kMaxSplits;

  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const size_t counters = kCounterRegionBytes;
  const size_t lse = ((size_t)batch * hq * ws_splits * sizeof(float) + 255) & ~size_t(255);

  AttnArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.block_tables = block_tables;
  a.seq_lens = seq_lens;
  a.counters = reinterpret_cast<int32_t*>(ws);
  a.ws_lse = reinterpret_cast<float*>(ws + counters);
  a.ws_o = reinterpret_cast<float*>(ws + counters + lse);
  a.max_blocks = max_blocks;
  a.hq = hq;
  a.hkv = hkv;
  a.group = hq / hkv;
  a.blocks_per_split = plan.blocks_per_split;
  a.max_splits = ws_splits;
  a.scale_log2 = scale * 1.4426950408889634f;
  static const int late_env = std::getenv("OFB_K1_LATE") ? std::atoi(std::getenv("OFB_K1_LATE")) : 1;
  a.kv_ready = (kv_ready == 1 && late_env) ? 3 : kv_ready;
  a.defer_combine = (variant == 4 && plan.max_splits > 1) ? 1 : 0;
  a.trace = k1_trace_buffer();
  a.trace_ctas = a.trace ? k1_trace_capacity() : 0;
  dim3 grid(plan.max_splits, hkv, batch);
  // one wave at one CTA per SM: the wide instantiation (OFB_K1_WIDE=0|1 pins it)
  const long ctas = (long)plan.max_splits * hkv * batch;
  static const int wide_env = std::getenv("OFB_K1_WIDE") ? std::atoi(std::getenv("OFB_K1_WIDE")) : -1;
  const bool wide = force_narrow ? false : wide_env >= 0 ? wide_env == 1 : ctas <= g_num_sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(wide ? (kWideWarps + 1) * 32 : kAttnThreads);
  cfg.dynamicSmemBytes = wide ? attn_smem_bytes<kWideWarps, kWideStages>() : kAttnSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  e = wide ? cudaLaunchKernelEx(&cfg, paged_gqa_decode_wide_kernel, map, a)
           : cudaLaunchKernelEx(&cfg, paged_gqa_decode_kernel, map, a);
  if (e != cudaSuccess || !a.defer_combine) return e;
  cudaLaunchConfig_t cc = cfg;
  cc.gridDim = dim3(a.group, hkv, batch);
  cc.blockDim = dim3(128);
  cc.dynamicSmemBytes = 0;
  return cudaLaunchKernelEx(&cc, attn_combine_kernel, a);
}

// Host arithmetic only (no device): the plan an attention-only in-step launch
// (kv_ready 1) takes under the auto policy - always the split kernel, on the
// balanced narrow plan where balanced_preferred holds (*narrow = 1), else on the
// cost-model plan (*narrow = 1 unless that grid is one wave of wide CTAs).
int attention_instep_plan(int batch, int hq, int hkv, int max_seq_len, int num_sms, int occupancy,
                          int* blocks_per_split, int* splits, int* narrow) {
  if (batch < 1 || hkv < 1 || hq % hkv != 0 || hq / hkv > kMaxGroup || max_seq_len < 0 ||
      num_sms < 1 || occupancy < 1 || !blocks_per_split || !splits || !narrow)
    return -1;
  const AttnPlan bal = balanced_plan(batch, hkv, max_seq_len, num_sms);
  if (bal.max_splits > 0 && balanced_preferred(bal, hq / hkv)) {
    *blocks_per_split = bal.blocks_per_split;
    *splits = bal.max_splits;
    *narrow = 1;
    return 0;
  }
  const AttnPlan p = plan_splits(batch, hq, hkv, max_seq_len, num_sms, occupancy);
  *blocks_per_split = p.blocks_per_split;
  *splits = p.max_splits;
  *narrow = (long)p.max_splits * hkv * batch <= num_sms ? 0 : 1;
  return 0;
}

int attention_occupancy() {
  attn_init_once();
  return g_attn_occupancy;
}

}  // namespace ofb
