// Per-warp building blocks of K1 shared by both work decompositions:
// Q fragments, one 16-token (block, head) tile of online-softmax attention on
// mma.sync m16n8k16 tiles, and the warp-state hand-off through shared memory.
//
// Tile in shared memory (written by TMA, 128B swizzle): two halves of
// [32 rows][64 bf16]; rows 0-15 = K of the block's 16 tokens, rows 16-31 = V.
#pragma once

#include "common.cuh"

namespace ofb {

constexpr int kMaxGroup = 16;

__device__ __forceinline__ uint32_t tile_addr(uint32_t base, int row, int chunk) {
  // `chunk` = 16 B column unit (0..15) of the logical 256 B row.
  return base + ((chunk >> 3) << 12) + (row << 7) + ((((chunk & 7) ^ (row & 7))) << 4);
}

// Per-lane online-softmax state of one consumer warp: rows r0 and r0+8 of the
// zero-padded 16-row query group, O accumulators of 16 n-tiles of head dims.
struct WarpAttnState {
  float o[16][4];
  float m[2];
  float l[2];

  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.f;
  }
};

// Q as the mma A operand: rows = the g query heads of one KV head (padded to 16).
__device__ __forceinline__ void load_q_frag(uint32_t (&qa)[8][4], const __nv_bfloat16* qb, int g,
                                            int lane) {
  const int r0 = lane >> 2, c0 = (lane & 3) * 2;
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

// One 16-token tile: S = Q K^T, online softmax update, O += P V.
// `valid` = tokens of this block inside the sequence (1..16).
__device__ __forceinline__ void attend_tile(WarpAttnState& st, const uint32_t (&qa)[8][4],
                                            uint8_t* tile, int valid, float scale_log2,
                                            int lane) {
  const uint32_t base = smem_u32(tile);
  const int mi = lane >> 3, mr = lane & 7;
  const int c0 = (lane & 3) * 2;
  if (valid < kBlockTokens) {
    // Slots past the sequence end hold stale bits (possibly NaN): P is 0 there
    // but 0 * NaN poisons the P.V tile, so clear those V rows first.
    for (int c = lane; c < (kBlockTokens - valid) * 16; c += 32) {
      const int row = kBlockTokens + valid + (c >> 4);
      *reinterpret_cast<uint4*>(tile + ((c >> 3) & 1) * (kHeadBlockBytes / 2) + row * 128 +
                                (c & 7) * 16) = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
  }
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
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float v = s[j][e] * scale_log2;
      if (j * 8 + c0 + (e & 1) >= valid) v = -INFINITY;
      s[j][e] = v;
    }
  float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
  float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  const float mn0 = fmaxf(st.m[0], mx0), mn1 = fmaxf(st.m[1], mx1);
  const float corr0 = fast_exp2(st.m[0] - mn0), corr1 = fast_exp2(st.m[1] - mn1);
  st.m[0] = mn0;
  st.m[1] = mn1;
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
  st.l[0] = st.l[0] * corr0 + rs0;
  st.l[1] = st.l[1] * corr1 + rs1;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    st.o[nt][0] *= corr0;
    st.o[nt][1] *= corr0;
    st.o[nt][2] *= corr1;
    st.o[nt][3] *= corr1;
  }
  uint32_t pa[4];  // accumulator layout == A-operand layout for k16
  pa[0] = pack_bf16(s[0][0], s[0][1]);
  pa[1] = pack_bf16(s[0][2], s[0][3]);
  pa[2] = pack_bf16(s[1][0], s[1][1]);
  pa[3] = pack_bf16(s[1][2], s[1][3]);
#pragma unroll
  for (int np = 0; np < 8; ++np) {
    uint32_t v0, v1, v2, v3;
    ldsm_x4_t(tile_addr(base, 16 + (mi & 1) * 8 + mr, 2 * np + (mi >> 1)), v0, v1, v2, v3);
    mma_bf16_16816(st.o[2 * np], pa, v0, v1);
    mma_bf16_16816(st.o[2 * np + 1], pa, v2, v3);
  }
}

// Warp-state exchange buffer for merging the consumer warps of one CTA.  Row
// stride 136 floats: a warp's float2 stores of 4 rows x 8 dims fill the 32
// banks exactly (two wavefronts per 8 rows, no conflicts).
constexpr int kMergeStride = kHeadDim + 8;
template <int kWarps>
struct MergeSlots {
  float o[kWarps][kMaxGroup][kMergeStride];
  float m[kWarps][kMaxGroup];
  float l[kWarps][kMaxGroup];
};

// Only the g real query rows are published (the mma pads the group to 16 rows):
// at g = 4 that is a quarter of the stores.
template <int kWarps>
__device__ __forceinline__ void publish_state(MergeSlots<kWarps>* ms, WarpAttnState& st, int warp,
                                              int lane, int g) {
  float l0 = st.l[0], l1 = st.l[1];
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const int r0 = lane >> 2, c0 = (lane & 3) * 2;
  if (r0 < g) {
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
      *reinterpret_cast<float2*>(&ms->o[warp][r0][nt * 8 + c0]) = make_float2(st.o[nt][0], st.o[nt][1]);
    if ((lane & 3) == 0) {
      ms->m[warp][r0] = st.m[0];
      ms->l[warp][r0] = l0;
    }
  }
  if (r0 + 8 < g) {
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
      *reinterpret_cast<float2*>(&ms->o[warp][r0 + 8][nt * 8 + c0]) = make_float2(st.o[nt][2], st.o[nt][3]);
    if ((lane & 3) == 0) {
      ms->m[warp][r0 + 8] = st.m[1];
      ms->l[warp][r0 + 8] = l1;
    }
  }
}

// Merged (row, d) value of the CTA's warps: returns O / L and sets *lse_out.
template <int kWarps>
__device__ __forceinline__ float merged_value(const MergeSlots<kWarps>* ms, int row, int d,
                                              float* lse_out) {
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) M = fmaxf(M, ms->m[w][row]);
  float acc = 0.f, L = 0.f;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const float mw = ms->m[w][row];
    if (mw != -INFINITY) {
      const float sc = fast_exp2(mw - M);
      acc += sc * ms->o[w][row][d];
      L += sc * ms->l[w][row];
    }
  }
  *lse_out = M + __log2f(L);
  return acc / L;
}

// Two-phase merge of the CTA's warp states, used by the split and cluster
// kernels: per-row weights once (g threads), then every (row, 4 dims) output
// is a kWarps-term weighted sum of float4 smem loads - no per-element max /
// exp2 / divide, which left the old per-element merge latency-bound (~2 us
// with one 5-warp CTA per SM, tools/k1_split_trace.py).
template <int kWarps>
struct MergeWeights {
  float w[kWarps][kMaxGroup];   // exp2(m_w - M) / L, 0 for a warp that saw no token
  float lse[kMaxGroup];         // M + log2(L) (log2 domain), -inf for an empty row
};

template <int kWarps>
__device__ __forceinline__ void merge_weights(const MergeSlots<kWarps>* ms, MergeWeights<kWarps>* mw,
                                              int g, int tid) {
  if (tid < g) {
    const int row = tid;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, ms->m[w][row]);
    float sc[kWarps];
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float mw_ = ms->m[w][row];
      sc[w] = mw_ > -INFINITY ? fast_exp2(mw_ - M) : 0.f;
      L += sc[w] * ms->l[w][row];
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mw->w[w][row] = sc[w] * inv;
    mw->lse[row] = L > 0.f ? M + __log2f(L) : -INFINITY;
  }
}

// Normalised merged O of `row`, head dims 4q .. 4q+3.
template <int kWarps>
__device__ __forceinline__ float4 merged_quad(const MergeSlots<kWarps>* ms,
                                              const MergeWeights<kWarps>* mw, int row, int q) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const float wt = mw->w[w][row];
    const float4 v = *reinterpret_cast<const float4*>(&ms->o[w][row][q * 4]);
    acc.x += wt * v.x;
    acc.y += wt * v.y;
    acc.z += wt * v.z;
    acc.w += wt * v.w;
  }
  return acc;
}

}  // namespace ofb
