// Decoder glue around the data path for the whole-decoder TP step (SURVEY.md
// 8(d) cfg4): RMSNorm of the residual stream and the SwiGLU activation.  Not
// among the four north-star pieces.  With K6 (c1="k6") both are folded into the
// projections (the residual add, the RMSNorm's row sums of squares and 1/rms row
// scale, and SwiGLU all live in K6's epilogues), so only ofb_row_sumsq runs, once
// per step for the embeddings; rmsnorm / silu_mul serve the cuBLAS + NCCL arm.
//
//   rmsnorm:    a[b] = x[b] / sqrt(mean(x[b]^2) + eps) * w        (one CTA per row)
//   silu_mul:   act[b, i] = silu(gu[b, i]) * gu[b, inter + i]      (grid-stride)
//   row_sumsq:  ss[t][b] = sum of x[b][128t .. 128t+127]^2          (one CTA per tile)
#include "common.cuh"

#include "../../include/orbitflow_b200.h"

namespace ofb {
int report_error(int code, const char* msg);
int report_cuda(cudaError_t e, const char* what);

namespace {

constexpr int kNormThreads = 512;

__device__ __forceinline__ void unpack8(uint4 u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}

// One CTA per row; each thread holds up to kPer 8-element vectors in registers.
template <int kPer>
__global__ void __launch_bounds__(kNormThreads)
rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
               __nv_bfloat16* __restrict__ out, int hidden, float eps) {
  pdl_wait();      // x is the previous kernel's output
  pdl_trigger();   // the next projection may start streaming its weights
  const int row = blockIdx.x;
  const int nvec = hidden / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(row) * hidden);
  float v[kPer][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nvec) {
      unpack8(xr[i], v[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[k][e] * v[k][e];
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  __shared__ float part[kNormThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += part[i];
  const float r = rsqrtf(tot / hidden + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* orow = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * hidden);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < nvec) {
      float g[8];
      unpack8(wr[i], g);
      uint4 o;
      o.x = pack_bf16(v[k][0] * r * g[0], v[k][1] * r * g[1]);
      o.y = pack_bf16(v[k][2] * r * g[2], v[k][3] * r * g[3]);
      o.z = pack_bf16(v[k][4] * r * g[4], v[k][5] * r * g[5]);
      o.w = pack_bf16(v[k][6] * r * g[6], v[k][7] * r * g[7]);
      orow[i] = o;
    }
  }
}

__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act,
                                int batch, int inter) {
  pdl_wait();
  pdl_trigger();
  const int nvec = inter / 8;
  const size_t total = static_cast<size_t>(batch) * nvec;
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t b = t / nvec, i = t - b * nvec;
    const uint4* row = reinterpret_cast<const uint4*>(gu + b * 2 * inter);
    float g[8], u[8];
    unpack8(row[i], g);
    unpack8(row[nvec + i], u);
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = g[e] / (1.f + __expf(-g[e])) * u[e];
    uint4 p;
    p.x = pack_bf16(o[0], o[1]);
    p.y = pack_bf16(o[2], o[3]);
    p.z = pack_bf16(o[4], o[5]);
    p.w = pack_bf16(o[6], o[7]);
    reinterpret_cast<uint4*>(act + b * inter)[i] = p;
  }
}

// ss[t][b] = sum of x[b][128t .. 128t+127]^2: one CTA per 128-column tile, one
// warp per row (4 columns per lane, a fixed shuffle order).
__global__ void row_sumsq_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ ss, int rows,
                                 int hidden, int ld_batch) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = warp; b < rows; b += blockDim.x >> 5) {
    const uint2 u = *reinterpret_cast<const uint2*>(x + static_cast<size_t>(b) * hidden + t * 128 + lane * 4);
    const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    float s = f0.x * f0.x + f0.y * f0.y + f1.x * f1.x + f1.y * f1.y;
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) ss[static_cast<size_t>(t) * ld_batch + b] = s;
  }
}

// Launch with programmatic stream serialization (unless OFB_PDL=0): the glue
// kernels wait for their predecessor before reading anything and release their
// dependent at once, so the next K6 requests its weight ring while they run.
template <typename... Params, typename... Args>
cudaError_t launch_pdl(void (*kernel)(Params...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace
}  // namespace ofb

extern "C" {

int ofb_rmsnorm(const void* x, const void* weight, void* out, int32_t rows, int32_t hidden, float eps,
                void* stream) {
  using namespace ofb;
  if (!x || !weight || !out || rows < 0) return report_error(-1, "ofb_rmsnorm: bad arguments");
  if (hidden <= 0 || hidden % 8 || hidden > 8 * kNormThreads * 4)
    return report_error(-1, "ofb_rmsnorm: hidden must be a multiple of 8 and <= 16384");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  const int per = (hidden / 8 + kNormThreads - 1) / kNormThreads;
  const auto* xp = static_cast<const __nv_bfloat16*>(x);
  const auto* wp = static_cast<const __nv_bfloat16*>(weight);
  auto* op = static_cast<__nv_bfloat16*>(out);
  const cudaError_t e = per <= 1   ? launch_pdl(rmsnorm_kernel<1>, rows, kNormThreads, s, xp, wp, op, hidden, eps)
                       : per <= 2 ? launch_pdl(rmsnorm_kernel<2>, rows, kNormThreads, s, xp, wp, op, hidden, eps)
                                  : launch_pdl(rmsnorm_kernel<4>, rows, kNormThreads, s, xp, wp, op, hidden, eps);
  return e == cudaSuccess ? 0 : report_cuda(e, "rmsnorm_kernel launch");
}

int ofb_row_sumsq(const void* x, float* ss_out, int32_t rows, int32_t hidden, int32_t ld_batch,
                  void* stream) {
  using namespace ofb;
  if (!x || !ss_out || rows < 0 || ld_batch < rows || hidden <= 0 || hidden % 128)
    return report_error(-1, "ofb_row_sumsq: bad arguments (hidden % 128, ld_batch >= rows)");
  if (rows == 0) return 0;
  const cudaError_t e = launch_pdl(row_sumsq_kernel, hidden / 128, 256, static_cast<cudaStream_t>(stream),
                                   static_cast<const __nv_bfloat16*>(x), ss_out, rows, hidden, ld_batch);
  return e == cudaSuccess ? 0 : report_cuda(e, "row_sumsq_kernel launch");
}

int ofb_silu_mul(const void* gate_up, void* act, int32_t batch, int32_t inter, void* stream) {
  using namespace ofb;
  if (!gate_up || !act || batch < 0 || inter <= 0 || inter % 8)
    return report_error(-1, "ofb_silu_mul: bad arguments (inter must be a multiple of 8)");
  if (batch == 0) return 0;
  const size_t total = static_cast<size_t>(batch) * (inter / 8);
  int blocks = static_cast<int>((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  const cudaError_t e = launch_pdl(silu_mul_kernel, blocks, 256, static_cast<cudaStream_t>(stream),
                                   static_cast<const __nv_bfloat16*>(gate_up),
                                   static_cast<__nv_bfloat16*>(act), batch, inter);
  return e == cudaSuccess ? 0 : report_cuda(e, "silu_mul_kernel launch");
}

}  // extern "C"
