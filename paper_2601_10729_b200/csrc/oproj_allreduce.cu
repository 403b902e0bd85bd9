// K6 / C1: tensor-parallel o-projection fused with its all-reduce over peer
// memory (PAPER.md:727-729 runs NCCL after the projection).
//
// hidden[B, H] = sum_r attn_r[B, K] @ W_r[H, K]^T, K = (Hq/N)*128 per rank.
// At decode B is 16-64, so the GEMM is a weight stream (16 MiB of W_o per
// layer at 70B/TP8) - HBM bound at 2*B flop per W byte.  It runs "swap AB" on
// the 5th-gen tensor cores: UMMA M = 128 rows of W (one hidden tile per CTA),
// N = the batch padded to 32, K streamed in 64-element (128 B) chunks by TMA
// with 128-byte swizzle into a mbarrier ring; one elected thread issues
// tcgen05.mma (kind::f16, bf16 in, fp32 accumulate in TMEM) and commits each
// stage back to the producer.  The epilogue reads TMEM with tcgen05.ld.
//
// Split-K spreads the hidden tiles over every SM: the CTAs of one tile form a
// thread-block cluster, the non-leaders ship their fp32 partial into the
// leader's shared memory (DSMEM) - a reduction region of its own, so they need
// not wait for the leader's MMAs - and one cluster barrier later the leader sums
// in split order.  It then
// pushes the bf16 tile into every peer's inbox slot for this rank (P2P stores
// over NVLink into IPC-mapped symmetric buffers), raises the tile's flag on
// each peer (st.release.sys), waits for every rank's flag on its own copy of
// the tile (ld.acquire.sys) and sums the world's partials in rank order - a
// one-shot all-reduce overlapped with the GEMM tile by tile.  Every rank sums
// the same bf16 values in the same order, so all ranks hold identical bits.
//
// Reuse of an inbox slot two calls later is safe with two parities: a peer
// can only write epoch e+2 after finishing e+1, which needs this rank's e+1
// pushes, which come after this rank finished reading epoch e (stream order).
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/orbitflow_b200.h"
#include "common.cuh"

namespace ofb {
int report_error(int code, const char* msg);
int report_cuda(cudaError_t e, const char* what);
int encode_bf16_map(CUtensorMap* map, void* base, int rank, const uint64_t* dims,
                    const uint64_t* byte_strides, const uint32_t* box);

namespace {

constexpr int kTileM = 128;        // hidden rows per CTA = UMMA M = TMEM lanes
constexpr int kChunkK = 64;        // K elements per pipeline stage (one 128 B swizzle atom)
constexpr int kThreads = 128;      // 4 warps: TMA producer, MMA issuer, TMEM owner, all epilogue
constexpr int kMaxPeers = 8;
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 200 * 1024;   // one CTA per SM, deepest ring

struct OprojArgs {
  int layer, batch, npad, k, hidden, tiles, splits, chunks, stages;
  int world, rank, max_batch;
  uint32_t epoch;
  long long timeout_ns;
  __nv_bfloat16* out;       // [batch][hidden]
  int* status;
  char* symm[kMaxPeers];
  long long flags_off;
  unsigned long long* trace;   // diagnostics (ofb_k6_trace): per CTA stamps, or null
  const __nv_bfloat16* residual;   // added before the final rounding, or null (may alias out)
  int parts;                       // > 1: column ranges written to separate tensors (world 1)
  float* ss_out;                   // fp32 [tiles][max_batch]: sum over the tile's columns of out^2, or null
  const float* ss_in;              // fp32 [ss_tiles][max_batch]: a producer's ss_out (fused RMSNorm), or null
  int ss_tiles;
  float eps;
  int swiglu;                      // 1: rows interleaved gate 64 / up 64; out [batch][hidden/2] = silu(g) * u
  int x_layer;                     // x's layer coordinate (0 when one x serves every layer)
  uint8_t* kv_pool;                // K3 folded in (see ofb_oproj_desc), or null
  const int32_t* kv_tables;
  const int32_t* kv_positions;
  const uint64_t* kv_host;
  int kv_max_blocks, kv_part;
  long long kv_block_bytes;
  int part_lo[5];                  // first column of range i (part_lo[parts] = hidden)
  __nv_bfloat16* part_out[4];
  int rs;                          // split-K reduce-scatter: every CTA of a tile finalises a row slice
};

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t addr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols)
               : "memory");
}

// Shared-memory matrix descriptor: K-major operand, 128-byte swizzle, rows of
// 128 B, 8-row groups 1024 B apart (SBO); LBO is unused for swizzled K-major.
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;               // LBO (ignored)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;       // SBO
  d |= static_cast<uint64_t>(1) << 46;               // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;               // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// One 64-element K chunk: four K=16 MMAs (+32 B along the swizzle atom each) in
// one asm block, so the single issuing thread spends a handful of instructions
// per chunk (at decode shapes the whole W tile often lands at once and the MMA
// issue is what remains after the last byte)
__device__ __forceinline__ void umma_chunk(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, t;\nsetp.ne.b32 p, %4, 0;\nsetp.eq.b32 t, 0, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, t;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %3, t;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %10, %3, t;\n}\n"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate),
        "l"(adesc + 2), "l"(bdesc + 2), "l"(adesc + 4), "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

// 32 lanes x 32 columns of fp32: thread i of the warp gets its lane's 32 columns.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)),
        "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ---------------------------------------------------------------- system-scope flags
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float sumsq_bf16x8(uint4 u) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    s += f.x * f.x + f.y * f.y;
  }
  return s;
}

__device__ __forceinline__ void add_bf16x8(float* acc, uint4 u) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    acc[2 * i] += f.x;
    acc[2 * i + 1] += f.y;
  }
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t map_to_cta(uint32_t saddr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(cta));
  return r;
}

// Grid = tiles x splits, cluster = (splits, 1, 1): the CTAs of a cluster share
// one hidden tile and split its K range; non-leaders ship their fp32 partial
// into the leader's shared memory (DSMEM) and the leader sums in split order.
__global__ void __launch_bounds__(kThreads, 1)
oproj_allreduce_kernel(const __grid_constant__ CUtensorMap wmap,
                       const __grid_constant__ CUtensorMap xmap,
                       const __grid_constant__ OprojArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned for the 128-byte swizzle; derived from smem_raw by an
  // offset so the compiler keeps the shared address space (STS, not ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], acc_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / a.splits, split = blockIdx.x % a.splits;   // split = rank in cluster
  unsigned long long* tr = (a.trace && threadIdx.x == 0) ? a.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tr) tr[0] = globaltimer();
  const int c0 = split * a.chunks / a.splits;
  const int nchunks = (split + 1) * a.chunks / a.splits - c0;
  const int stage_w = kTileM * kChunkK * 2;          // 16 KiB of W rows
  const int stage_bytes = stage_w + a.npad * kChunkK * 2;
  const uint32_t tcols = a.npad <= 32 ? 32u : a.npad <= 64 ? 64u : a.npad <= 128 ? 128u : 256u;
  const int pre = nchunks < a.stages ? nchunks : a.stages;

  if (threadIdx.x == 0) {
    prefetch_tma_desc(&wmap);
    prefetch_tma_desc(&xmap);
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&acc_bar, 1);
    fence_mbar_init();
    // W_o does not depend on the previous kernel (attention), so the first
    // ring's worth of weight tiles is requested first thing - before the TMEM
    // allocation and the CTA barrier, and before the programmatic-dependent-
    // launch wait; x (the attention output) after it.
    for (int i = 0; i < pre; ++i) {
      mbar_arrive_expect_tx(&full_bar[i], stage_bytes);
      tma_load_4d(smem + i * stage_bytes, &wmap, &full_bar[i], 0, 0, c0 + i, a.layer * a.tiles + tile);
    }
  }
  __syncwarp();   // warp 0 re-converges after its lane-0 setup
  if (warp == 2) tmem_alloc(&tmem_base_sh, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  // "every CTA of the cluster has started" is only needed before the first DSMEM
  // access: arrive now, wait right before the partials are shipped (by then every
  // peer has long arrived, so the barrier is off the critical path)
  if (a.splits > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (tr) tr[1] = globaltimer();

  if (warp == 0) {
    // TMA producer (the whole warp, converged; one elected lane issues): the
    // first stages' W loads are in flight (above)
    pdl_wait();
    if (elect_one())
      for (int i = 0; i < pre; ++i)
        tma_load_3d(smem + i * stage_bytes + stage_w, &xmap, &full_bar[i], (c0 + i) * kChunkK, 0, a.x_layer);
    __syncwarp();
    // refills: chunk i >= pre = stages reuses stage i % stages once its MMAs read it
    int s = 0;
    uint32_t ph = 0;
    for (int i = pre; i < nchunks; ++i) {
      mbar_wait(&empty_bar[s], ph);
      if (elect_one()) {
        uint8_t* sw = smem + s * stage_bytes;
        mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
        tma_load_4d(sw, &wmap, &full_bar[s], 0, 0, c0 + i, a.layer * a.tiles + tile);
        tma_load_3d(sw + stage_w, &xmap, &full_bar[s], (c0 + i) * kChunkK, 0, a.x_layer);
      }
      __syncwarp();
      if (++s == a.stages) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else if (warp == 1) {
    // MMA issuer (the whole warp, converged; one elected lane issues):
    // D[128 x npad] (TMEM) += W_tile[128 x 64] . X[npad x 64]^T per stage
    const uint32_t idesc = umma_idesc_bf16(kTileM, a.npad);
    // descriptors advance by the stage size (address field = byte address >> 4;
    // shared addresses < 256 KiB never carry out of it); no per-chunk division
    const uint64_t ad0 = sw128_kmajor_desc(smem_u32(smem)), bd0 = sw128_kmajor_desc(smem_u32(smem + stage_w));
    const uint64_t dstep = static_cast<uint64_t>(stage_bytes >> 4);
    uint64_t ad = ad0, bd = bd0;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunks; ++i) {
      mbar_wait(&full_bar[s], ph);
      tc_fence_after();
      if (elect_one()) {
        umma_chunk(tmem, ad, bd, idesc, i > 0 ? 1u : 0u);
        umma_commit(&empty_bar[s]);            // frees the stage once these MMAs have read it
      }
      __syncwarp();
      if (++s == a.stages) {
        s = 0;
        ph ^= 1u;
        ad = ad0;
        bd = bd0;
      } else {
        ad += dstep;
        bd += dstep;
      }
    }
    if (elect_one()) umma_commit(&acc_bar);
    __syncwarp();
  }
  __syncwarp();

  // ---- epilogue (row m = warp*32 + lane of the tile)
  // Fused RMSNorm of the input rows (ss_in): the producer of x left, per hidden
  // tile, the sum of squares of each row; summed here in tile order while the
  // MMAs still run.  out[b] = (x[b] . W'^T) * rsqrt(mean(x[b]^2) + eps), the
  // norm weight having been folded into W' (pack time).
  __shared__ float rsc[256];
  __shared__ long long kvoff[256];   // K3 folded in: pool byte offset of each row's slot, or -1
  // the k / v part this tile belongs to (one KV head's 128 dims), if K3 is folded in
  int kvsel = -1;
  if (a.kv_pool) {
    for (int r = 0; r < a.parts; ++r)
      if (tile * kTileM >= a.part_lo[r] && tile * kTileM < a.part_lo[r + 1]) kvsel = r - a.kv_part;
    if (kvsel != 0 && kvsel != 1) kvsel = -1;
  }
  // Per-row prologue of the leader, done by warps 2-3 while the MMAs run: warps 0
  // and 1 are the TMA producer and the MMA issuer and reach the epilogue only
  // after their loops (the producer after its last refill), so work dealt to
  // them by row would sit on the epilogue's critical path.  The x loads already
  // wait for the predecessor, so the early PDL wait costs nothing.
  //  - K3 fold: every row's pool slot (two dependent loads per row);
  //  - fused RMSNorm (ss_in): 1/rms of every row from the producer's per-32-column
  //    sums of squares, several lanes per row combined in a fixed shuffle order;
  //  - the residual tile of the first 32 batch rows, staged in smem (16-byte loads).
  __shared__ __align__(16) __nv_bfloat16 res_s[32 * kTileM];
  // (with the reduce-scatter every CTA of the tile finalises rows, so every one
  // needs the per-row inputs; otherwise only the leader)
  const bool fin = split == 0 || a.rs;
  const bool res_pre = a.world == 1 && a.residual && fin;
  const bool pro = fin && (kvsel >= 0 || a.ss_in || res_pre);
  if (pro && warp >= 2) {
    pdl_wait();
    const int pt = threadIdx.x - 64;           // 0..63
    if (kvsel >= 0) {
      const int head = (tile * kTileM - a.part_lo[a.kv_part + kvsel]) / kTileM;
      for (int b = pt; b < a.batch; b += 64) {
        long long off = -1;
        const int pos = a.kv_positions[b];
        if (pos >= 0 && (!a.kv_host || a.kv_host[b] == 0)) {
          const int blk = a.kv_tables[static_cast<size_t>(b) * a.kv_max_blocks + pos / kBlockTokens];
          if (blk >= 0)
            off = static_cast<long long>(blk) * a.kv_block_bytes +
                  static_cast<long long>((head * 2 + kvsel) * kBlockTokens + pos % kBlockTokens) * kRowBytes;
        }
        kvoff[b] = off;
      }
    }
    if (a.ss_in) {
      int lpr = 1;                              // lanes per row: a power of two <= 32
      while (lpr < 32 && lpr * 2 * a.batch <= 64) lpr *= 2;
      const int part = pt & (lpr - 1);
      for (int b0 = 0; b0 < a.batch; b0 += 64 / lpr) {
        const int b = b0 + pt / lpr;            // uniform trip count: every lane shuffles
        float sum = 0.f;
        if (b < a.batch)
          for (int t = part; t < a.ss_tiles; t += lpr)
            sum += __ldcg(a.ss_in + static_cast<size_t>(t) * a.max_batch + b);
        for (int off = lpr >> 1; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        if (b < a.batch && part == 0) rsc[b] = rsqrtf(sum / static_cast<float>(a.ss_tiles * kTileM) + a.eps);
      }
    }
    if (res_pre) {
      const int rows = a.batch < 32 ? a.batch : 32;
      for (int i = pt; i < rows * (kTileM / 8); i += 64) {
        const int b = i >> 4, q = i & 15;
        *reinterpret_cast<uint4*>(res_s + b * kTileM + q * 8) = *reinterpret_cast<const uint4*>(
            a.residual + static_cast<size_t>(b) * a.hidden + tile * kTileM + q * 8);
      }
    }
  }
  if (pro && a.splits == 1) __syncthreads();   // publish (else the cluster barrier below does)
  mbar_wait(&acc_bar, 0);
  if (tr) tr[2] = globaltimer();
  tc_fence_after();
  pdl_wait();                       // every thread: the predecessor's writes are visible
  pdl_trigger();                    // the next kernel may start its own prologue (releasing it
                                    // right after the prologue measured slower in the decoder step)
  const int m = warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  // leader smem: red [splits-1][npad][128] fp32 after the ring (its own region, so
  // non-leaders may write it while the leader's MMAs still run), stg [npad][128]
  // bf16 in the ring (idle once the leader's own MMAs completed)
  float* red = reinterpret_cast<float*>(smem + static_cast<size_t>(a.stages) * stage_bytes);
  __nv_bfloat16* stg = reinterpret_cast<__nv_bfloat16*>(smem);
  if (a.splits > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (a.rs) {
    // ---- reduce-scatter (world 1, splits in {2, 4, 8}): CTA r of the cluster owns
    // tile rows [r*128/S, (r+1)*128/S); every row's fp32 partial goes to its owner
    // (owner's red: [S-1 sources][npad][slice], a warp's rows one contiguous run),
    // so each CTA takes in (S-1)/S of a tile partial instead of the leader taking
    // in S-1 of them, and every CTA finalises and stores its own slice.
    const int S = a.splits, sl = kTileM / S;
    const int own = m / sl;                       // owner of this thread's row
    const int my_lo = split * sl;
    // (tcgen05.ld is warp-wide and .aligned: every lane loads, converged; a warp's
    // rows can span two owners, so only the stores are predicated)
    const bool ship = own != split;
    const int slot_me = split < own ? split : split - 1;
    const uint32_t dst =
        ship ? map_to_cta(smem_u32(red + static_cast<size_t>(slot_me) * a.npad * sl + (m - own * sl)), own) : 0u;
    for (int c = 0; c < a.npad / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(trow + c * 32, v);
      if (ship) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          asm volatile("st.shared::cluster.f32 [%0], %1;"
                       ::"r"(dst + ((c * 32 + j) * sl) * 4), "f"(__uint_as_float(v[j]))
                       : "memory");
      }
      __syncwarp();
    }
    tc_fence_before();
    cluster_sync_all();                           // every slice's partials have landed
    tc_fence_after();
    if (tr) tr[3] = globaltimer();
    // the owning rows: sources summed in split order (own partial in its place)
    __nv_bfloat16* stg2 = stg;                    // [npad][sl] bf16 in the (idle) ring
    if (warp * 32 < my_lo + sl && warp * 32 + 32 > my_lo) {   // warp-uniform
      const int i = m - my_lo;
      for (int c = 0; c < a.npad / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        if (own == split) {
        // sources in split order, own partial in its place: a compact loop (straight-
        // line code run once per launch costs instruction fetches, not ALU time)
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
        for (int src = 0; src < S; ++src) {
          if (src == split) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] += __uint_as_float(v[j]);
          } else {
            const float* rp = red + (static_cast<size_t>(src < split ? src : src - 1) * a.npad + c * 32) * sl + i;
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] += rp[j * sl];
          }
        }
        if (a.ss_in) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j < a.batch) acc[j] *= rsc[c * 32 + j];
        }
        if (a.residual) {
          const __nv_bfloat16* rb = c == 0 ? res_s + m : a.residual + static_cast<size_t>(c * 32) * a.hidden + tile * kTileM + m;
          const int rstride = c == 0 ? kTileM : a.hidden;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j < a.batch) acc[j] += __bfloat162float(rb[static_cast<size_t>(j) * rstride]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) stg2[(c * 32 + j) * sl + i] = __float2bfloat16_rn(acc[j]);
        }
        __syncwarp();
      }
    }
    if (tr) tr[4] = globaltimer();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, tcols);
    if (tr) tr[6] = globaltimer();   // the slice stores start
    // this CTA's slice of the tile: 16-byte vectors per batch row
    __nv_bfloat16* dst_base = a.out;
    int dst_stride = a.hidden, col0 = tile * kTileM;
    for (int r = 0; r < a.parts; ++r)
      if (col0 >= a.part_lo[r] && col0 < a.part_lo[r + 1]) {
        dst_base = a.part_out[r];
        dst_stride = a.part_lo[r + 1] - a.part_lo[r];
        col0 -= a.part_lo[r];
      }
    const int vpr = sl / 8;                       // vectors per batch row
    for (int q = threadIdx.x; q < a.batch * vpr; q += kThreads) {
      const int b = q / vpr, o = q - b * vpr;
      const uint4 val = *reinterpret_cast<const uint4*>(stg2 + b * sl + o * 8);
      *reinterpret_cast<uint4*>(dst_base + static_cast<size_t>(b) * dst_stride + col0 + my_lo + o * 8) = val;
      if (kvsel >= 0 && kvoff[b] >= 0)
        *reinterpret_cast<uint4*>(a.kv_pool + kvoff[b] + (my_lo + o * 8) * 2) = val;
    }
    if (tr) tr[5] = globaltimer();
    return;
  }
  if (a.splits > 1 && split != 0) {
    // ship this split's fp32 partial into the leader's smem: element (n, m) at
    // n * 128 + m, so a warp's 32 rows are one contiguous 128-byte DSMEM store
    const uint32_t dst = map_to_cta(smem_u32(red + static_cast<size_t>(split - 1) * a.npad * kTileM), 0);
    for (int c = 0; c < a.npad / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(trow + c * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        asm volatile("st.shared::cluster.f32 [%0], %1;"
                     ::"r"(dst + ((c * 32 + j) * kTileM + m) * 4), "f"(__uint_as_float(v[j]))
                     : "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, tcols);
    // one cluster barrier: the partials are visible in the leader past it, and the
    // leader (whose smem they target) cannot have exited before it
    cluster_sync_all();
    if (tr) tr[5] = globaltimer();
    return;
  }
  if (a.splits > 1) {
    cluster_sync_all();               // every non-leader's partial has landed
    if (tr) tr[3] = globaltimer();
  }
  for (int c = 0; c < a.npad / 32; ++c) {
    uint32_t v[32];
    tmem_ld32(trow + c * 32, v);
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = __uint_as_float(v[j]);
    for (int s = 1; s < a.splits; ++s) {       // split order: deterministic
      const float* src = red + (static_cast<size_t>(s - 1) * a.npad + c * 32) * kTileM + m;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] += src[j * kTileM];
    }
    if (a.ss_in) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c * 32 + j < a.batch) acc[j] *= rsc[c * 32 + j];
    }
    if (a.world == 1 && a.residual) {   // x += o_proj(attn): one rounding of x + sum
      if (c == 0) {                    // staged by the prologue (rows < min(batch, 32))
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < a.batch) acc[j] += __bfloat162float(res_s[j * kTileM + m]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int b = c * 32 + j;
          if (b < a.batch)
            acc[j] += __bfloat162float(a.residual[static_cast<size_t>(b) * a.hidden + tile * kTileM + m]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[(c * 32 + j) * kTileM + m] = __float2bfloat16_rn(acc[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, tcols);

  const int nvec = a.batch * (kTileM / 8);     // 16-byte vectors of the [batch][128] tile
  const uint4* s4 = reinterpret_cast<const uint4*>(stg);
  if (tr) tr[4] = globaltimer();
  if (a.world == 1 && a.ss_out) {
    // per batch row, the sum of squares of this tile's final (rounded) values: one
    // warp per row, fixed order - the next projection's fused RMSNorm
    for (int b = warp; b < a.batch; b += kThreads / 32) {
      const uint2 u = reinterpret_cast<const uint2*>(stg + static_cast<size_t>(b) * kTileM)[lane];
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      float s = f0.x * f0.x + f0.y * f0.y + f1.x * f1.x + f1.y * f1.y;
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) a.ss_out[static_cast<size_t>(tile) * a.max_batch + b] = s;
    }
  }
  if (a.world == 1 && a.swiglu) {
    // SwiGLU: tile rows 0-63 are gate columns 64*tile.., rows 64-127 the matching
    // up columns; act[b][64*tile + i] = silu(gate) * up from the bf16-rounded values
    const int inter = a.hidden / 2;
    for (int i = threadIdx.x; i < a.batch * 8; i += kThreads) {
      const int b = i >> 3, q = i & 7;
      const uint4 gv = s4[b * 16 + q], uv = s4[b * 16 + 8 + q];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
      const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
      float o[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 g = __bfloat1622float2(g2[e]), u = __bfloat1622float2(u2[e]);
        o[2 * e] = g.x / (1.f + __expf(-g.x)) * u.x;
        o[2 * e + 1] = g.y / (1.f + __expf(-g.y)) * u.y;
      }
      uint4 pk;
      pk.x = pack_bf16(o[0], o[1]);
      pk.y = pack_bf16(o[2], o[3]);
      pk.z = pack_bf16(o[4], o[5]);
      pk.w = pack_bf16(o[6], o[7]);
      *reinterpret_cast<uint4*>(a.out + static_cast<size_t>(b) * inter + tile * 64 + q * 8) = pk;
    }
    if (tr) tr[5] = globaltimer();
    return;
  }
  if (a.world == 1) {
    // the column range (tensor) this tile belongs to: one lookup per CTA
    __nv_bfloat16* dst_base = a.out;
    int dst_stride = a.hidden, col0 = tile * kTileM;
    for (int r = 0; r < a.parts; ++r)
      if (col0 >= a.part_lo[r] && col0 < a.part_lo[r + 1]) {
        dst_base = a.part_out[r];
        dst_stride = a.part_lo[r + 1] - a.part_lo[r];
        col0 -= a.part_lo[r];
      }
    // K3 folded in: a k or v tile is one KV head's 128 dims; its rows also go to
    // the token's slot in the paged pool (resident rows; host-slab rows are the
    // runtime append's, which also fills their staged copy)
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      const int b = i >> 4, o = i & 15;
      *reinterpret_cast<uint4*>(dst_base + static_cast<size_t>(b) * dst_stride + col0 + o * 8) = s4[i];
      if (kvsel >= 0 && kvoff[b] >= 0)
        *reinterpret_cast<uint4*>(a.kv_pool + kvoff[b] + o * 16) = s4[i];
    }
    if (tr) tr[5] = globaltimer();
    return;
  }

  // ---- one-shot all-reduce of this tile over peer memory
  const int p = static_cast<int>(a.epoch & 1u);
  const size_t slot = static_cast<size_t>(a.max_batch) * kTileM;          // elements per (src, tile)
  const size_t src_stride = static_cast<size_t>(a.tiles) * slot;
  const size_t mine = (static_cast<size_t>(p) * a.world + a.rank) * src_stride + tile * slot;
  for (int r = 0; r < a.world; ++r) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.symm[r]) + mine);
    for (int i = threadIdx.x; i < nvec; i += kThreads) dst[i] = s4[i];
  }
  __threadfence_system();
  __syncthreads();
  const size_t flag_idx = (static_cast<size_t>(p) * a.world + a.rank) * a.tiles + tile;
  if (threadIdx.x < a.world)
    st_release_sys(reinterpret_cast<unsigned int*>(a.symm[threadIdx.x] + a.flags_off) + flag_idx, a.epoch);
  if (threadIdx.x < a.world) {
    const unsigned int* f = reinterpret_cast<const unsigned int*>(a.symm[a.rank] + a.flags_off) +
                            (static_cast<size_t>(p) * a.world + threadIdx.x) * a.tiles + tile;
    const long long t0 = globaltimer();
    while (static_cast<int>(ld_acquire_sys(f) - a.epoch) < 0) {
      if (globaltimer() - t0 > a.timeout_ns) {
        atomicExch(a.status, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  const __nv_bfloat16* inbox = reinterpret_cast<const __nv_bfloat16*>(a.symm[a.rank]) +
                               static_cast<size_t>(p) * a.world * src_stride + tile * slot;
  constexpr int kUnroll = 4;   // vectors per thread whose loads are all issued before any store
  // warp-uniform trip count (the ss_out shuffles need every lane)
  for (int i0 = threadIdx.x; i0 - lane < nvec; i0 += kThreads * kUnroll) {
    float acc[kUnroll][8];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
    for (int r = 0; r < a.world; ++r) {         // rank order: identical sums on every rank
      const uint4* src = reinterpret_cast<const uint4*>(inbox + r * src_stride);
      uint4 t[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = i0 + u * kThreads;
        t[u] = i < nvec ? __ldcg(src + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) add_bf16x8(acc[u], t[u]);
    }
    if (a.residual) {                  // every rank adds the same residual after the sum
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = i0 + u * kThreads;
        if (i < nvec) {
          const int b = i >> 4, q = i & 15;
          add_bf16x8(acc[u], *reinterpret_cast<const uint4*>(
                                 a.residual + static_cast<size_t>(b) * a.hidden + tile * kTileM + q * 8));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int i = i0 + u * kThreads;
      uint4 o;
      o.x = pack_bf16(acc[u][0], acc[u][1]);
      o.y = pack_bf16(acc[u][2], acc[u][3]);
      o.z = pack_bf16(acc[u][4], acc[u][5]);
      o.w = pack_bf16(acc[u][6], acc[u][7]);
      const int b = i >> 4, q = i & 15;
      if (i < nvec)
        *reinterpret_cast<uint4*>(a.out + static_cast<size_t>(b) * a.hidden + tile * kTileM + q * 8) = o;
      if (a.ss_out) {
        // the 16 vectors of row b sit in 16 consecutive lanes: reduce them in a
        // fixed order (identical on every rank, like the sum itself)
        float s = i < nvec ? sumsq_bf16x8(o) : 0.f;
#pragma unroll
        for (int off = 8; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (i < nvec && q == 0) a.ss_out[static_cast<size_t>(tile) * a.max_batch + b] = s;
      }
    }
  }
}

int padded_batch(int batch) { return (batch + 31) / 32 * 32; }

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

size_t red_bytes(int splits, int npad) {
  return static_cast<size_t>(splits - 1) * npad * kTileM * 4;
}

int ring_stages(int npad, int splits) {
  const int stage_bytes = kTileM * kChunkK * 2 + npad * kChunkK * 2;
  const long avail = static_cast<long>(kSmemBudget) - static_cast<long>(red_bytes(splits, npad));
  return std::max(2, std::min<int>(kMaxStages, static_cast<int>(avail / stage_bytes)));
}

// CTAs per hidden tile (= cluster size): enough to cover the SMs, at most 8
// (portable clusters), at most one K chunk each, and the leader's reduction
// buffers must fit beside a ring of at least 2 stages.  8 splits are what the
// narrow q/k/v projection needs (10 tiles at 70B TP8: 80 CTAs, 9.8 us vs 11.6 us
// at 4 splits; synccheck / racecheck / memcheck clean, profiles/sanitizer/).
int choose_splits(int tiles, int chunks, int npad) {
  int s = num_sms() / tiles;
  if (const char* f = std::getenv("OFB_K6_SPLITS")) s = std::atoi(f);   // tuning experiments
  int cap = 8;   // portable cluster size; the leader gathers splits-1 fp32 partials
  if (const char* f = std::getenv("OFB_K6_SPLIT_CAP")) cap = std::atoi(f);   // tuning experiments
  s = std::max(1, std::min(s, std::min(std::min(cap, 8), chunks)));
  // more than 4 splits only when every CTA still streams >= 4 K chunks: compute-
  // sanitizer synccheck reports a divergent warp at the prologue barrier for 8-CTA
  // clusters of 2-chunk splits (results correct; not understood - not used)
  if (s > 4 && chunks / s < 4) s = 4;
  // the reduction buffers + a 2-stage ring must fit; the bf16 staging reuses the ring
  const int stage_bytes = kTileM * kChunkK * 2 + npad * kChunkK * 2;
  while (s > 1 && red_bytes(s, npad) + 2 * static_cast<size_t>(stage_bytes) > static_cast<size_t>(kSmemBudget))
    --s;
  return s;
}

size_t inbox_bytes(int world, int max_batch, int hidden) {
  return static_cast<size_t>(2) * world * static_cast<size_t>(hidden) * max_batch * 2;
}

size_t flags_bytes(int world, int hidden) {
  return static_cast<size_t>(2) * world * (hidden / kTileM) * 4;
}

struct MapKey {
  const void* x;
  const void* w;
  int layers, batch, k, hidden, npad, w_layout, x_layers;
  CUtensorMap xmap, wmap;
};
unsigned long long* g_k6_trace = nullptr;
std::mutex g_map_mu;
std::vector<MapKey> g_map_cache;

int get_maps(const ofb_oproj_desc* d, int npad, CUtensorMap* xmap, CUtensorMap* wmap) {
  std::lock_guard<std::mutex> lock(g_map_mu);
  for (auto& e : g_map_cache)
    if (e.x == d->x && e.w == d->w && e.layers == d->layers && e.batch == d->batch &&
        e.k == d->k && e.hidden == d->hidden && e.npad == npad && e.w_layout == d->w_layout &&
        e.x_layers == d->x_layers) {
      *xmap = e.xmap;
      *wmap = e.wmap;
      return 0;
    }
  MapKey e{d->x, d->w, d->layers, d->batch, d->k, d->hidden, npad, d->w_layout, d->x_layers, {}, {}};
  const uint64_t row = static_cast<uint64_t>(d->k) * 2;
  {  // X: [layers][batch][k]; box 64 x npad x 1 (rows past the batch read as zero)
    uint64_t dims[3] = {static_cast<uint64_t>(d->k), static_cast<uint64_t>(d->batch),
                        static_cast<uint64_t>(d->x_layers == 1 ? 1 : d->layers)};
    uint64_t strides[2] = {row, row * d->batch};
    uint32_t box[3] = {static_cast<uint32_t>(kChunkK), static_cast<uint32_t>(npad), 1};
    int rc = encode_bf16_map(&e.xmap, const_cast<void*>(d->x), 3, dims, strides, box);
    if (rc) return rc;
  }
  {  // W as 4-D (element in chunk, row in tile, K chunk, layer*tiles + tile); box 64 x 128 x 1 x 1.
    // Linear layout [layers][hidden][k]: a box is 128 rows x 128 B, rows k*2 B apart.
    // Packed layout [layers][hidden/128][k/64][128][64]: a box is 16 KiB contiguous.
    const uint64_t chunks = static_cast<uint64_t>(d->k) / kChunkK;
    const uint64_t tiles = static_cast<uint64_t>(d->hidden) / kTileM;
    uint64_t dims[4] = {static_cast<uint64_t>(kChunkK), static_cast<uint64_t>(kTileM), chunks,
                        tiles * static_cast<uint64_t>(d->layers)};
    uint64_t strides[3];
    if (d->w_layout == 1) {
      strides[0] = kChunkK * 2;                         // row in tile
      strides[1] = kChunkK * 2 * kTileM;                // next K chunk: 16 KiB
      strides[2] = strides[1] * chunks;                 // next tile
    } else {
      strides[0] = row;                                 // row in tile
      strides[1] = kChunkK * 2;                         // next K chunk: 128 B along the row
      strides[2] = row * kTileM;                        // next tile: 128 rows
    }
    uint32_t box[4] = {static_cast<uint32_t>(kChunkK), static_cast<uint32_t>(kTileM), 1, 1};
    int rc = encode_bf16_map(&e.wmap, const_cast<void*>(d->w), 4, dims, strides, box);
    if (rc) return rc;
  }
  if (g_map_cache.size() > 256) g_map_cache.erase(g_map_cache.begin());
  g_map_cache.push_back(e);
  *xmap = e.xmap;
  *wmap = e.wmap;
  return 0;
}

// Clusters of this launch's shape the GPU holds at once (cached per device,
// cluster size and dynamic smem).
int oproj_coresident_clusters(const cudaLaunchConfig_t* launch, const cudaLaunchAttribute* cluster_attr,
                              int* out) {
  static std::mutex mu;
  static std::vector<std::array<long long, 4>> cache;   // dev, splits, smem, clusters
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return report_cuda(e, "cudaGetDevice");
  const long long key_splits = cluster_attr->val.clusterDim.x;
  const long long key_smem = static_cast<long long>(launch->dynamicSmemBytes);
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& c : cache)
    if (c[0] == dev && c[1] == key_splits && c[2] == key_smem) {
      *out = static_cast<int>(c[3]);
      return 0;
    }
  cudaLaunchConfig_t cfg = *launch;
  cudaLaunchAttribute attr = *cluster_attr;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  e = cudaOccupancyMaxActiveClusters(&n, oproj_allreduce_kernel, &cfg);
  if (e != cudaSuccess) return report_cuda(e, "cudaOccupancyMaxActiveClusters(oproj_allreduce_kernel)");
  cache.push_back({dev, key_splits, key_smem, n});
  *out = n;
  return 0;
}

}  // namespace
}  // namespace ofb

extern "C" {

int ofb_symm_alloc(int64_t bytes, void** ptr) {
  if (!ptr || bytes <= 0) return ofb::report_error(-1, "ofb_symm_alloc: bad arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, static_cast<size_t>(bytes));
  if (e != cudaSuccess) return ofb::report_cuda(e, "cudaMalloc (symmetric buffer)");
  e = cudaMemset(p, 0, static_cast<size_t>(bytes));
  if (e != cudaSuccess) return ofb::report_cuda(e, "cudaMemset (symmetric buffer)");
  *ptr = p;
  return 0;
}

int ofb_symm_free(void* ptr) {
  if (ptr) {
    cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) return ofb::report_cuda(e, "cudaFree (symmetric buffer)");
  }
  return 0;
}

int ofb_ipc_get_handle(void* ptr, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
  if (!ptr || !handle64) return ofb::report_error(-1, "ofb_ipc_get_handle: null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return ofb::report_cuda(e, "cudaIpcGetMemHandle");
  memcpy(handle64, &h, sizeof(h));
  return 0;
}

int ofb_ipc_open_handle(const void* handle64, void** ptr) {
  if (!handle64 || !ptr) return ofb::report_error(-1, "ofb_ipc_open_handle: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return ofb::report_cuda(e, "cudaIpcOpenMemHandle");
  return 0;
}

int ofb_ipc_close_handle(void* ptr) {
  if (ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) return ofb::report_cuda(e, "cudaIpcCloseMemHandle");
  }
  return 0;
}

int ofb_k6_trace(void* device_buffer) {
  ofb::g_k6_trace = static_cast<unsigned long long*>(device_buffer);
  return 0;
}

int64_t ofb_oproj_symm_bytes(int32_t world, int32_t max_batch, int32_t hidden) {
  if (world < 1 || world > ofb::kMaxPeers || max_batch < 1 || hidden < ofb::kTileM) return -1;
  const size_t inbox = (ofb::inbox_bytes(world, max_batch, hidden) + 255) / 256 * 256;
  return static_cast<int64_t>(inbox + ofb::flags_bytes(world, hidden));
}

int64_t ofb_oproj_workspace_bytes(int32_t max_batch, int32_t k, int32_t hidden) {
  if (max_batch < 1 || k < ofb::kChunkK || hidden < ofb::kTileM) return -1;
  return 256;   // reserved: split-K partials are reduced on chip (cluster DSMEM)
}

int ofb_oproj_allreduce(const ofb_oproj_desc* d, void* stream) {
  using namespace ofb;
  if (!d) return report_error(-1, "ofb_oproj_allreduce: null descriptor");
  if (!d->x || !d->w || (!d->out && d->out_parts <= 1))
    return report_error(-1, "ofb_oproj_allreduce: null tensor");
  if (d->batch < 1 || d->batch > d->max_batch || d->max_batch > 256)
    return report_error(-1, "ofb_oproj_allreduce: need 1 <= batch <= max_batch <= 256");
  if (d->k < kChunkK || d->k % kChunkK) return report_error(-1, "ofb_oproj_allreduce: k must be a multiple of 64");
  if (d->hidden < kTileM || d->hidden % kTileM)
    return report_error(-1, "ofb_oproj_allreduce: hidden must be a multiple of 128");
  if (d->layer < 0 || d->layer >= d->layers) return report_error(-1, "ofb_oproj_allreduce: layer out of range");
  if (d->w_layout != 0 && d->w_layout != 1) return report_error(-1, "ofb_oproj_allreduce: w_layout must be 0 or 1");
  if (d->world < 1 || d->world > kMaxPeers || d->rank < 0 || d->rank >= d->world)
    return report_error(-1, "ofb_oproj_allreduce: bad world / rank");
  if (d->world > 1) {
    if (d->epoch == 0) return report_error(-1, "ofb_oproj_allreduce: epoch must be > 0");
    if (!d->status) return report_error(-1, "ofb_oproj_allreduce: status pointer required");
    for (int r = 0; r < d->world; ++r)
      if (!d->symm[r]) return report_error(-1, "ofb_oproj_allreduce: missing peer buffer");
  }
  {  // the decoder-layer epilogues (validated before any driver call)
    const int parts = d->out_parts > 1 ? d->out_parts : 0;
    if (d->ss_in && (d->world != 1 || d->ss_tiles < 1 || !(d->eps >= 0.f)))
      return report_error(-1, "ofb_oproj_allreduce: ss_in needs world 1, ss_tiles >= 1 and eps >= 0");
    if (d->swiglu && (d->world != 1 || d->residual || parts || d->ss_out || !d->out))
      return report_error(-1, "ofb_oproj_allreduce: swiglu needs world 1, an out tensor, no residual / parts / ss_out");
    if (d->ss_out && parts) return report_error(-1, "ofb_oproj_allreduce: ss_out excludes out_parts");
    if (d->x_layers != 0 && d->x_layers != 1)
      return report_error(-1, "ofb_oproj_allreduce: x_layers must be 0 or 1");
    if (d->kv_pool && (d->world != 1 || parts < 2 || d->kv_part < 0 || d->kv_part + 1 >= parts ||
                       !d->kv_tables || !d->kv_positions || d->kv_max_blocks < 1 || d->kv_block_bytes <= 0 ||
                       d->part_cols[d->kv_part] != d->part_cols[d->kv_part + 1]))
      return report_error(-1, "ofb_oproj_allreduce: kv_pool needs world 1, k / v parts of equal width, "
                              "tables, positions and a block size");
  }
  const int npad = padded_batch(d->batch);
  const int tiles = d->hidden / kTileM;
  const int chunks = d->k / kChunkK;
  const int splits = choose_splits(tiles, chunks, npad);
  CUtensorMap xmap, wmap;
  int rc = get_maps(d, npad, &xmap, &wmap);
  if (rc) return rc;

  OprojArgs a{};
  a.layer = d->layer;
  a.batch = d->batch;
  a.npad = npad;
  a.k = d->k;
  a.hidden = d->hidden;
  a.tiles = tiles;
  a.splits = splits;
  a.chunks = chunks;
  const int stage_bytes = kTileM * kChunkK * 2 + npad * kChunkK * 2;
  a.stages = ring_stages(npad, splits);
  {
    // When a CTA's whole K range fits the ring, every stage is requested at once
    // and lands at the end together, leaving all MMAs after the last byte; a ring of
    // 3/4 of the chunks staggers the arrivals (70B TP8 o-proj, 8 chunks per CTA:
    // 6.25 -> 6.01 us at 6 stages; profiles/r02_k6_experiments.md)
    const int per_cta = (chunks + splits - 1) / splits;
    if (per_cta >= 8 && per_cta <= a.stages) a.stages = per_cta * 3 / 4;
  }
  a.world = d->world;
  a.rank = d->rank;
  a.max_batch = d->max_batch;
  a.epoch = d->epoch;
  a.timeout_ns = d->timeout_ns > 0 ? d->timeout_ns : 5000000000LL;
  a.out = static_cast<__nv_bfloat16*>(d->out);
  a.status = d->status;
  for (int r = 0; r < d->world; ++r) a.symm[r] = static_cast<char*>(d->symm[r]);
  a.trace = g_k6_trace;
  a.residual = static_cast<const __nv_bfloat16*>(d->residual);
  a.parts = d->out_parts > 1 ? d->out_parts : 0;
  if (a.parts) {
    if (d->world != 1 || d->residual || a.parts > 4)
      return report_error(-1, "ofb_oproj_allreduce: out_parts needs world 1, no residual, <= 4 parts");
    int lo = 0;
    for (int r = 0; r < a.parts; ++r) {
      if (!d->part_out[r] || d->part_cols[r] <= 0 || d->part_cols[r] % kTileM)
        return report_error(-1, "ofb_oproj_allreduce: part_cols must be positive multiples of 128");
      a.part_lo[r] = lo;
      a.part_out[r] = static_cast<__nv_bfloat16*>(d->part_out[r]);
      lo += d->part_cols[r];
    }
    a.part_lo[a.parts] = lo;
    if (lo != d->hidden) return report_error(-1, "ofb_oproj_allreduce: part_cols must sum to hidden");
  }
  a.flags_off = static_cast<long long>((inbox_bytes(d->world, d->max_batch, d->hidden) + 255) / 256 * 256);
  a.ss_out = d->ss_out;
  a.ss_in = d->ss_in;
  a.ss_tiles = d->ss_tiles;
  a.eps = d->eps;
  a.swiglu = d->swiglu;
  a.x_layer = d->x_layers == 1 ? 0 : d->layer;
  a.kv_pool = static_cast<uint8_t*>(d->kv_pool);
  a.kv_tables = d->kv_tables;
  a.kv_positions = d->kv_positions;
  a.kv_host = d->kv_host_slabs;
  a.kv_max_blocks = d->kv_max_blocks;
  a.kv_part = d->kv_part;
  a.kv_block_bytes = d->kv_block_bytes;
  {
    static const int rs_env = std::getenv("OFB_K6_RS") ? std::atoi(std::getenv("OFB_K6_RS")) : 1;
    // measured (profiles/r02_k6_experiments.md): wins at 8 splits (q/k/v 9.70 -> 8.94 us),
    // ties at 2, loses at 4 - kept for 8-CTA clusters only
    a.rs = (rs_env && d->world == 1 && !d->swiglu && !d->ss_out && splits == 8) ? 1 : 0;
  }




  const size_t smem = static_cast<size_t>(a.stages) * stage_bytes + red_bytes(splits, npad) + 1024;
  {  // the dynamic-smem opt-in is per device: set it once for each device used
    static std::mutex mu;
    static std::vector<int> configured;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return report_cuda(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(configured.begin(), configured.end(), dev) == configured.end()) {
      e = cudaFuncSetAttribute(oproj_allreduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kSmemBudget + 2048));
      if (e != cudaSuccess) return report_cuda(e, "cudaFuncSetAttribute(oproj_allreduce_kernel)");
      configured.push_back(dev);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles * splits);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  if (d->world > 1) {
    // Forward progress of the exchange: a tile's CTA spins until every rank's
    // copy of that tile has landed, so all tiles of every rank must be resident
    // at once (any CTA still waiting for an SM could be the one a spinning peer
    // needs).  Refuse a grid larger than what the GPU co-schedules.
    int coresident = 0;
    rc = oproj_coresident_clusters(&cfg, attr, &coresident);
    if (rc) return rc;
    if (tiles > coresident)
      return report_error(-1, ("ofb_oproj_allreduce: " + std::to_string(tiles) + " clusters of " +
                               std::to_string(splits) + " CTAs exceed the " +
                               std::to_string(coresident) +
                               " this GPU co-schedules; the peer-flag wait needs the whole grid "
                               "resident (use hidden <= 128 x that many tiles, or world 1)")
                                  .c_str());
  }
  // W_o prefetch overlaps the attention kernel's tail (the x loads wait)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, oproj_allreduce_kernel, wmap, xmap, a);
  if (e != cudaSuccess) return report_cuda(e, "oproj_allreduce_kernel launch");
  return 0;
}

}  // extern "C"
