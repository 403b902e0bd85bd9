// K3: new-token KV append for a decode step.
//
// Realises RequestState.record_generated_token / sync_blocks
// (/root/reference/pkg/src/kvsim/core.py:95-102), called once per decoding
// request per step at /root/reference/pkg/src/kvsim/engine.py:389-392: the
// token count grows by one and a new 16-token block is claimed at block
// boundaries (core.py:27-36).  Physically, each (layer, request, kv head)
// writes one K row and one V row (256 B each) at slot `pos % 16` of the block
// that holds token `pos`:
//   * through the layer's block table (resident HBM slab or, for an
//     offloaded layer, the staging slot that was just filled), and
//   * for offloaded layers, also straight into the pinned host slab through
//     its mapped address (fresh KV goes to its host slot).
// One warp per (request, kv head): lanes 0-15 move the K row, 16-31 the V
// row, 16 B each (fully coalesced 128-bit stores).
#include "common.cuh"

namespace ofb {

// Which (layer, request) rows an append launch touches.  A row is "offloaded"
// when it has a host slab (host_slabs[l][b] != 0).
enum AppendMode : int {
  kAppendResident = 0,   // resident rows only (pool write)
  kAppendAll = 1,        // every row: host slab (if any) + pool/staging via table
  kAppendOffloaded = 2,  // offloaded rows only: host slab + staging via table
};

struct AppendArgs {
  const uint4* k_new;            // [L][B][Hkv][128] bf16
  const uint4* v_new;
  uint8_t* pool;                 // HBM block pool base (nullable when no tables)
  const int32_t* block_tables;   // [L][B][max_blocks], -1 = no device copy
  const int32_t* positions;      // [B]  token index written this step (<0: skip)
  const uint64_t* host_slabs;    // [L][B] mapped host slab base, 0 = none (nullable)
  int max_blocks;
  int batch;
  int hkv;
  int mode;                      // kAppendResident / kAppendAll / kAppendOffloaded
};

__global__ void __launch_bounds__(256) kv_append_kernel(const AppendArgs a) {
  // k_new / v_new may be the previous kernel's output, and it may read the pool.
  // No early launch_dependents: the next K1 (cluster variant) would place its
  // clusters around these CTAs and lose its one-wave fit (measured +0.5 us/layer).
  pdl_wait();
  const int layer = blockIdx.y;
  const int pair = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (pair >= a.batch * a.hkv) return;
  const int req = pair / a.hkv;
  const int h = pair - req * a.hkv;
  const int lane = threadIdx.x & 31;
  const int pos = a.positions[req];
  if (pos < 0) return;
  const int kv = lane >> 4;
  const int part = lane & 15;

  const size_t lb = (size_t)layer * a.batch + req;
  const uint4 val = (kv ? a.v_new : a.k_new)[(lb * a.hkv + h) * (kHeadDim / 8) + part];
  const int blk_local = pos / kBlockTokens;
  const int slot = pos - blk_local * kBlockTokens;
  const size_t block_bytes = (size_t)a.hkv * kHeadBlockBytes;
  const size_t in_block = ((size_t)(h * 2 + kv) * kBlockTokens + slot) * kRowBytes + part * 16;

  const uint64_t host = a.host_slabs != nullptr ? a.host_slabs[lb] : 0;
  if (host != 0 ? a.mode == kAppendResident : a.mode == kAppendOffloaded) return;
  if (host != 0)
    *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(host) + blk_local * block_bytes + in_block) = val;
  if (a.block_tables != nullptr) {
    const int blk = a.block_tables[lb * a.max_blocks + blk_local];
    if (blk >= 0) *reinterpret_cast<uint4*>(a.pool + blk * block_bytes + in_block) = val;
  }
}

cudaError_t launch_kv_append(const void* k_new, const void* v_new, void* pool,
                             const int32_t* block_tables, int max_blocks,
                             const int32_t* positions, const uint64_t* host_slabs,
                             int num_layers, int batch, int hkv, int mode,
                             cudaStream_t stream, bool pdl) {
  if (batch <= 0 || num_layers <= 0) return cudaSuccess;
  AppendArgs a;
  a.k_new = static_cast<const uint4*>(k_new);
  a.v_new = static_cast<const uint4*>(v_new);
  a.pool = static_cast<uint8_t*>(pool);
  a.block_tables = block_tables;
  a.positions = positions;
  a.host_slabs = host_slabs;
  a.max_blocks = max_blocks;
  a.batch = batch;
  a.hkv = hkv;
  a.mode = mode;
  const int warps_per_cta = 8;
  dim3 grid((batch * hkv + warps_per_cta - 1) / warps_per_cta, num_layers);
  // `pdl`: programmatic launch (unless OFB_PDL=0) - the launch latency overlaps
  // the predecessor's tail and the kernel itself waits for it before touching
  // memory.  Used between the whole-decoder step's kernels (q/k/v projection ->
  // append -> K1); the step-start append follows a timing event and stays a
  // plain launch (programmatic there measured 16 us slower per step).
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(warps_per_cta * 32);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kv_append_kernel, a);
}

}  // namespace ofb
