// GPU enumeration for the native exact planner ("a
// GPU-vectorized port of _feasible_candidates").
//
// kvsim's solve ranks the product space of per-request distance choices
// (planner.py:310-341): a candidate survives the Eq.-1 capacity filter when
// resident blocks + the heaviest layer's offloaded demand fit the budget, and
// candidates are then priced in lower-bound order, ties in enumeration order
// (planner.py:344-414).  On the host that enumeration dominates beyond B = 7
// (B = 8, L = 32: 47 M feasible of 214 M; 4 s of the 4.6 s solve).  Here one
// thread tests one candidate (integer arithmetic, identical to the host DFS's
// final condition), survivors are compacted with warp-aggregated atomics as a
// 64-bit composite (lower-bound key << 32 | enumeration index), and one stable
// radix sort puts them in exactly the host's order.  planner.cpp then pulls
// the sorted list in chunks and prices/ranks it unchanged.
#include <cub/device/device_radix_sort.cuh>

#include <cstdint>
#include <string>

namespace ofb {

namespace {

constexpr int kMaxC = 32;
constexpr int kMaxL = 128;
constexpr int kMaxB = 12;

struct EnumArgs {
  int B, C, L;
  int64_t budget;
  double compL, bw;
  unsigned long long total;
  int count[kMaxC];
  long long blocks[kMaxB];
};

__global__ void enumerate_kernel(const __grid_constant__ EnumArgs a, const uint8_t* __restrict__ mask,
                                 unsigned long long* __restrict__ out,
                                 unsigned long long* __restrict__ n_out) {
  __shared__ uint8_t smask[kMaxC * kMaxL];
  for (int i = threadIdx.x; i < a.C * a.L; i += blockDim.x) smask[i] = mask[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < a.total;
       base += stride) {
    const unsigned long long idx = base + threadIdx.x;
    bool keep = false;
    unsigned long long word = 0;
    if (idx < a.total) {
      int pick[kMaxB];
      unsigned long long v = idx;
      for (int r = a.B - 1; r >= 0; --r) {   // request 0 most significant (planner.cpp decode)
        pick[r] = (int)(v % (unsigned)a.C);
        v /= (unsigned)a.C;
      }
      long long res = 0, fetch = 0;
      for (int r = 0; r < a.B; ++r) {
        res += a.blocks[r] * (a.L - a.count[pick[r]]);
        fetch += a.blocks[r] * a.count[pick[r]];
      }
      if (res <= a.budget) {
        long long worst = 0;
        for (int l = 0; l < a.L; ++l) {
          long long d = 0;
          for (int r = 0; r < a.B; ++r) d += smask[pick[r] * a.L + l] ? a.blocks[r] : 0;
          worst = d > worst ? d : worst;
        }
        if (res + worst <= a.budget) {
          const unsigned long long key =
              ((double)fetch / a.bw <= a.compL) ? 0ull : (unsigned long long)fetch + 1ull;
          word = (key << 32) | idx;
          keep = true;
        }
      }
    }
    // warp-aggregated compaction (order is restored by the sort)
    const unsigned ballot = __ballot_sync(0xffffffffu, keep);
    if (ballot) {
      unsigned long long slot = 0;
      if (lane == 0) slot = atomicAdd(n_out, (unsigned long long)__popc(ballot));
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (keep) out[slot + __popc(ballot & ((1u << lane) - 1u))] = word;
    }
  }
}

struct Handle {
  unsigned long long* keys = nullptr;   // sorted composite keys
  long long n = 0;
};

}  // namespace

// Feasible candidates of the product space, sorted by (lower-bound key,
// enumeration index); returns 0 and a handle, or an error code with *err set.
int plan_gpu_enumerate(int B, int C, int L, const int* count, const uint8_t* mask,
                       const int64_t* blocks, int64_t budget, double compL, double bw,
                       void** handle, int64_t* n_feasible, std::string* err) {
  *handle = nullptr;
  *n_feasible = 0;
  if (B > kMaxB || C > kMaxC || L > kMaxL) {
    *err = "planner enumeration: shape beyond the GPU kernel's limits";
    return -1;
  }
  unsigned long long total = 1;
  for (int r = 0; r < B; ++r) total *= (unsigned long long)C;
  if (total > 0xffffffffull) {
    *err = "planner enumeration: candidate space exceeds 2^32";
    return -1;
  }
  EnumArgs a{};
  a.B = B;
  a.C = C;
  a.L = L;
  a.budget = budget;
  a.compL = compL;
  a.bw = bw;
  a.total = total;
  for (int c = 0; c < C; ++c) a.count[c] = count[c];
  for (int r = 0; r < B; ++r) a.blocks[r] = blocks[r];
  // every key must fit 32 bits above the index
  long long max_fetch = 0;
  for (int r = 0; r < B; ++r) max_fetch += blocks[r] * L;
  if (max_fetch + 1 >= (1ll << 31)) {
    *err = "planner enumeration: fetch volume too large for the 64-bit key";
    return -1;
  }
  auto cuda = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess) *err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaSuccess;
  };
  cudaStream_t s = nullptr;
  uint8_t* d_mask = nullptr;
  unsigned long long *d_out = nullptr, *d_sorted = nullptr, *d_n = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  unsigned long long n = 0;
  bool ok = cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate") &&
            cuda(cudaMallocAsync(&d_mask, (size_t)C * L, s), "cudaMallocAsync") &&
            cuda(cudaMallocAsync(&d_n, sizeof(unsigned long long), s), "cudaMallocAsync") &&
            cuda(cudaMemcpyAsync(d_mask, mask, (size_t)C * L, cudaMemcpyHostToDevice, s), "H2D") &&
            cuda(cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), s), "memset");
  // one pass into a buffer sized for the whole space (8 B per candidate, <= 2 GiB
  // at the 2^28 cap planner.cpp enforces)
  if (ok) ok = cuda(cudaMallocAsync(&d_out, (size_t)total * 8, s), "cudaMallocAsync(out)");
  if (ok) {
    enumerate_kernel<<<148 * 8, 256, 0, s>>>(a, d_mask, d_out, d_n);
    ok = cuda(cudaGetLastError(), "enumerate_kernel") &&
         cuda(cudaMemcpyAsync(&n, d_n, sizeof(n), cudaMemcpyDeviceToHost, s), "D2H") &&
         cuda(cudaStreamSynchronize(s), "sync");
  }
  if (ok && n > 0) {
    int end_bit = 32;
    while (end_bit < 64 && ((unsigned long long)(max_fetch + 1) >> (end_bit - 32))) ++end_bit;
    ok = cuda(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_out, d_sorted, (int)n, 0,
                                             end_bit, s), "cub sizing") &&
         cuda(cudaMalloc(&d_sorted, (size_t)n * 8), "cudaMalloc(sorted)") &&
         cuda(cudaMallocAsync(&d_tmp, tmp_bytes, s), "cudaMallocAsync(tmp)") &&
         cuda(cub::DeviceRadixSort::SortKeys(d_tmp, tmp_bytes, d_out, d_sorted, (int)n, 0,
                                             end_bit, s), "cub SortKeys") &&
         cuda(cudaStreamSynchronize(s), "sync");
  }
  if (d_tmp) cudaFreeAsync(d_tmp, s);
  if (d_out) cudaFreeAsync(d_out, s);
  if (d_mask) cudaFreeAsync(d_mask, s);
  if (d_n) cudaFreeAsync(d_n, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (!ok) {
    if (d_sorted) cudaFree(d_sorted);
    return -1;
  }
  Handle* h = new Handle();
  h->keys = d_sorted;
  h->n = (long long)n;
  *handle = h;
  *n_feasible = (int64_t)n;
  return 0;
}

// Copy sorted composite keys [from, from + count) to the host.
int plan_gpu_fetch(void* handle, int64_t from, int64_t count, uint64_t* dst, std::string* err) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || from < 0 || from + count > h->n) {
    *err = "plan_gpu_fetch: range out of bounds";
    return -1;
  }
  cudaError_t e = cudaMemcpy(dst, h->keys + from, (size_t)count * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    *err = std::string("plan_gpu_fetch: ") + cudaGetErrorString(e);
    return -1;
  }
  return 0;
}

void plan_gpu_free(void* handle) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return;
  if (h->keys) cudaFree(h->keys);
  delete h;
}

}  // namespace ofb
