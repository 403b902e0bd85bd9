// Latency of the split-K fix-up chain that K1 and K6 end with: every CTA of a
// group publishes a 16 KiB fp32 partial, takes the group's ticket, and the last
// to arrive reads the group's partials back.  Per-phase globaltimer stamps,
// several ticket / read-back variants:
//   ticket 0: atom.add.acq_rel.gpu after a CTA barrier (common.cuh ticket_acq_rel)
//   ticket 1: __threadfence() by every writer, then atom.add.relaxed.gpu
//   ticket 2: fence.acq_rel.gpu by thread 0 only, then atom.add.relaxed.gpu
//   read 0: per-thread __ldcg, contributor by contributor (what K6 v2 did)
//   read 1: per-thread __ldcg, every contributor's loads issued before any add
//   read 2: cp.async.bulk of each contributor's partial into shared memory
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fixup_probe fixup_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

__device__ __forceinline__ long long gt() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int kElems = 4096;   // 16 KiB fp32 partial (batch 32 x 128 rows)
constexpr int kMaxGroup = 8;

__global__ void __launch_bounds__(128, 1) fixup_kernel(float* ws, int* tickets, float* out, int group, int tmode,
                                                       int rmode, long long* stamps) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int last_sh;
  const int g = blockIdx.x, grp = g / group, first = grp * group;
  const int n = min(group, gridDim.x - first);
  long long* st = stamps + g * 8;
  if (threadIdx.x == 0) {
    st[0] = gt();
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = g * 0.5f + j;
  float* mine = ws + static_cast<size_t>(g) * kElems;
#pragma unroll
  for (int j = 0; j < 32; ++j) __stcg(mine + j * 128 + threadIdx.x, v[j]);
  if (tmode == 1) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    st[1] = gt();
    int old;
    if (tmode == 0) {
      asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(tickets + grp) : "memory");
    } else {
      if (tmode == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("atom.add.relaxed.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(tickets + grp) : "memory");
      if (old == n - 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    last_sh = old == n - 1;
    if (last_sh) tickets[grp] = 0;
    st[2] = gt();
  }
  __syncthreads();
  if (!last_sh) {
    if (threadIdx.x == 0) st[3] = st[4] = gt();
    return;
  }
  float acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.f;
  if (rmode == 0) {
    for (int c = 0; c < n; ++c) {
      const float* src = ws + static_cast<size_t>(first + c) * kElems;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] += __ldcg(src + j * 128 + threadIdx.x);
    }
  } else if (rmode == 1) {
    for (int j0 = 0; j0 < 32; j0 += 8) {
      float t[kMaxGroup][8];
#pragma unroll
      for (int c = 0; c < kMaxGroup; ++c)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          t[c][j] = c < n ? __ldcg(ws + static_cast<size_t>(first + c) * kElems + (j0 + j) * 128 + threadIdx.x) : 0.f;
#pragma unroll
      for (int c = 0; c < kMaxGroup; ++c)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j0 + j] += t[c][j];
    }
  } else {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                   "r"(n * kElems * 4) : "memory");
      for (int c = 0; c < n; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + c * kElems)), "l"(ws + static_cast<size_t>(first + c) * kElems), "r"(kElems * 4),
                     "r"(su32(&bar)) : "memory");
    }
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], 0;\n@!P bra W_%=;\n}\n"
        ::"r"(su32(&bar)) : "memory");
    for (int c = 0; c < n; ++c)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] += sm[c * kElems + j * 128 + threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) st[3] = gt();
#pragma unroll
  for (int j = 0; j < 32; ++j) out[static_cast<size_t>(grp) * kElems + j * 128 + threadIdx.x] = acc[j];
  __syncthreads();
  if (threadIdx.x == 0) st[4] = gt();
}

int main() {
  const int grid = 148;
  float *ws, *out;
  int* tickets;
  long long* stamps;
  cudaMalloc(&ws, sizeof(float) * kElems * grid);
  cudaMalloc(&out, sizeof(float) * kElems * grid);
  cudaMalloc(&tickets, 4 * grid);
  cudaMemset(tickets, 0, 4 * grid);
  cudaMalloc(&stamps, 8 * 8 * grid);
  cudaFuncSetAttribute(fixup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxGroup * kElems * 4);
  std::vector<long long> h(8 * grid);
  for (int group : {2, 3, 8})
    for (int tmode = 0; tmode < 3; ++tmode)
      for (int rmode = 0; rmode < 3; ++rmode) {
        std::vector<double> ph[4];
        for (int rep = 0; rep < 20; ++rep) {
          cudaMemset(stamps, 0, 8 * 8 * grid);
          fixup_kernel<<<grid, 128, kMaxGroup * kElems * 4>>>(ws, tickets, out, group, tmode, rmode, stamps);
          cudaDeviceSynchronize();
          if (rep < 5) continue;
          cudaMemcpy(h.data(), stamps, 8 * 8 * grid, cudaMemcpyDeviceToHost);
          for (int g = 0; g < grid; ++g) {
            const long long* s = &h[g * 8];
            ph[0].push_back((s[1] - s[0]) / 1e3);   // partial store + barrier
            ph[1].push_back((s[2] - s[1]) / 1e3);   // ticket
            if (s[3] != s[4]) {
              ph[2].push_back((s[3] - s[2]) / 1e3);   // read-back + sum (finalizers)
              ph[3].push_back((s[4] - s[3]) / 1e3);   // output store
            }
          }
        }
        printf("{\"group\": %d, \"ticket\": %d, \"read\": %d", group, tmode, rmode);
        const char* names[4] = {"store_us", "ticket_us", "readback_us", "out_us"};
        for (int p = 0; p < 4; ++p) {
          auto& x = ph[p];
          std::sort(x.begin(), x.end());
          printf(", \"%s\": [%.3f, %.3f, %.3f]", names[p], x.empty() ? 0 : x[x.size() / 10],
                 x.empty() ? 0 : x[x.size() / 2], x.empty() ? 0 : x[x.size() * 9 / 10]);
        }
        printf("}\n");
        fflush(stdout);
      }
  printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
