// K5: prefill KV written straight to its planned
// location.
//
// In the reference, prefill placement is free and decided by the immediate
// batch-change re-plan (engine.py:495-503 prices only prefill time).
// Here the prompt's K/V, produced token-major by a prefill ([L][P][Hkv][128]
// per K and V), is scattered into the paged layout at its planned location
// in one launch per request: resident layers into their HBM extent, offloaded
// layers straight into their pinned host slab through the mapped address
// (PAPER.md:489 - no HBM staging and no second copy).
//
// One warp per (layer, block, kv head): lanes 0-15 move K rows, 16-31 V rows,
// 16 B per lane per row -> 16 rows x 256 B = 4 KiB each, coalesced.
#include "common.cuh"

namespace ofb {

struct PrefillArgs {
  const uint4* k;              // [L][P][Hkv][128] bf16
  const uint4* v;
  const uint64_t* dst;         // [L] slab base address (HBM extent or mapped host slab)
  int num_layers, tokens, hkv;
};

__global__ void __launch_bounds__(256) kv_prefill_kernel(const PrefillArgs a) {
  const int warps = blockDim.x >> 5;
  const int w = blockIdx.x * warps + (threadIdx.x >> 5);
  const int nblk = (a.tokens + kBlockTokens - 1) / kBlockTokens;
  const int per_layer = nblk * a.hkv;
  if (w >= per_layer * a.num_layers) return;
  const int layer = w / per_layer;
  const int rem = w - layer * per_layer;
  const int blk = rem / a.hkv, h = rem - blk * a.hkv;
  const int lane = threadIdx.x & 31;
  const int kv = lane >> 4, part = lane & 15;
  const uint4* src = kv ? a.v : a.k;
  uint8_t* base = reinterpret_cast<uint8_t*>(a.dst[layer]);
  const size_t block_bytes = (size_t)a.hkv * kHeadBlockBytes;
  uint8_t* tile = base + blk * block_bytes + (size_t)(h * 2 + kv) * kBlockTokens * kRowBytes;
  const int t0 = blk * kBlockTokens;
#pragma unroll 4
  for (int t = 0; t < kBlockTokens; ++t) {
    const int tok = t0 + t;
    if (tok >= a.tokens) break;   // the tail of the last block is never read (masked)
    const uint4 val = src[(((size_t)layer * a.tokens + tok) * a.hkv + h) * (kHeadDim / 8) + part];
    *reinterpret_cast<uint4*>(tile + (size_t)t * kRowBytes + part * 16) = val;
  }
}

cudaError_t launch_kv_prefill(const void* k, const void* v, const uint64_t* dst, int num_layers,
                              int tokens, int hkv, cudaStream_t stream) {
  if (num_layers <= 0 || tokens <= 0) return cudaSuccess;
  PrefillArgs a;
  a.k = static_cast<const uint4*>(k);
  a.v = static_cast<const uint4*>(v);
  a.dst = dst;
  a.num_layers = num_layers;
  a.tokens = tokens;
  a.hkv = hkv;
  const long long warps = (long long)num_layers * ((tokens + kBlockTokens - 1) / kBlockTokens) * hkv;
  const int per_cta = 8;
  kv_prefill_kernel<<<(unsigned)((warps + per_cta - 1) / per_cta), per_cta * 32, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace ofb
