// HBM read floor for small weight-streaming launches: G CTAs each pull a
// contiguous share of S bytes with 1-D TMA bulk copies (chunk bytes, D stages
// in flight) and discard it.  Graph-replayed chain of launches over rotating
// buffers (> L2), so the per-launch time is what a K6-sized kernel that does
// nothing but stream its operand can reach.  Standalone diagnostic:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_floor read_floor.cu
//   ./read_floor            -> one JSON line per (S, G, chunk, D)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32, 1) read_kernel(const uint8_t* base, long long bytes, int chunk, int depth,
                                                     unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[16];
  const long long lo = bytes * blockIdx.x / gridDim.x / 16 * 16;
  const long long hi = bytes * (blockIdx.x + 1) / gridDim.x / 16 * 16;
  const int n = static_cast<int>((hi - lo + chunk - 1) / chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < depth; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int i) {
    const int s = i % depth;
    const long long off = lo + static_cast<long long>(i) * chunk;
    const uint32_t len = static_cast<uint32_t>((chunk < hi - off ? (long long)chunk : hi - off));
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(su32(&bar[s])), "r"(len) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(smem + s * chunk)), "l"(base + off), "r"(len), "r"(su32(&bar[s])) : "memory");
  };
  for (int i = 0; i < (n < depth ? n : depth); ++i) issue(i);
  for (int i = 0; i < n; ++i) {
    const int s = i % depth;
    const uint32_t par = (i / depth) & 1;
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n"
        ::"r"(su32(&bar[s])), "r"(par) : "memory");
    if (i + depth < n) issue(i + depth);
  }
  if (smem[0] == 0xFF && smem[1] == 0xFE) atomicAdd(sink, 1ull);
}

__global__ void empty_kernel() {}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long sizes[] = {8552448LL, 17367040LL, 34209792LL, 67895296LL, 135266304LL};
  const int nbuf = 12;
  const long long maxs = 135266304LL;
  std::vector<uint8_t*> bufs(nbuf);
  for (auto& b : bufs) {
    cudaMalloc(&b, maxs);
    cudaMemset(b, 1, maxs);
  }
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_graph = [&](auto launch, int iters) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < iters; ++i) launch(i);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    std::vector<float> ts;
    for (int r = 0; r < 7; ++r) {
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1000.f / iters);
    }
    std::sort(ts.begin(), ts.end());
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ts[ts.size() / 2];
  };
  printf("{\"empty_kernel_us\": %.3f}\n", time_graph([&](int) { empty_kernel<<<sms, 32, 0, st>>>(); }, 64));
  const int grids[] = {64, 128, 148, 296};
  const int chunks[] = {8192, 16384, 32768};
  const int depths[] = {2, 4, 6, 8, 12};
  for (long long s : sizes)
    for (int g : grids)
      for (int ch : chunks)
        for (int d : depths) {
          if (static_cast<long long>(ch) * d > 196 * 1024) continue;
          if (g == 296 && static_cast<long long>(ch) * d > 96 * 1024) continue;
          const size_t smem = static_cast<size_t>(ch) * d;
          float us = time_graph(
              [&](int i) { read_kernel<<<g, 32, smem, st>>>(bufs[i % nbuf], s, ch, d, sink); }, 48);
          cudaError_t e = cudaGetLastError();
          printf("{\"bytes\": %lld, \"grid\": %d, \"chunk\": %d, \"depth\": %d, \"us\": %.3f, \"gbs\": %.1f%s}\n", s, g,
                 ch, d, us, s / (us * 1e-6) / 1e9, e == cudaSuccess ? "" : ", \"error\": true");
          fflush(stdout);
        }
  return 0;
}
