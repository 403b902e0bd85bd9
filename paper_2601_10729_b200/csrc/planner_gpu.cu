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
// 64-bit composite (lower-bound key << index bits | enumeration index), and
// one radix sort puts them in exactly the host's order.  A histogram pass over
// the keys first bounds memory: the list is materialised in windows of whole
// keys (or index ranges of one oversized key), so B = 9-10 at L = 32 (2.4 G /
// 26 G candidates) enumerate without holding every survivor.  planner.cpp
// pulls the sorted list in chunks and prices/ranks it unchanged.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace ofb {

namespace {

constexpr int kMaxC = 32;
constexpr int kMaxL = 128;
constexpr int kMaxB = 12;
constexpr int kIdxBitsMax = 36;                 // B = 10 at C = 11 is 2^34.6
constexpr long long kMaxKeyBins = 1ll << 26;    // lower-bound keys (fetch volume + 1)
constexpr long long kDefaultWindow = 1ll << 26; // candidates materialised at once (512 MiB)

struct EnumArgs {
  int B, C, L;
  int lo_reqs;                 // the last lo_reqs requests decode from the low 32-bit part
  unsigned lo_span;            // C^lo_reqs
  int idx_bits;
  int64_t budget;
  double compL, bw;
  unsigned long long idx_begin, idx_end;   // enumeration range of this pass
  long long key_lo, key_hi;                // materialise pass: keep keys in [key_lo, key_hi]
  unsigned long long out_cap;              // materialise pass: output capacity (overflow is counted, not written)
  int count[kMaxC];
  long long blocks[kMaxB];
};

// Capacity filter of one candidate (the host DFS's final condition) and its
// lower-bound key: 0 when compute-bound, else fetch volume + 1.
__device__ __forceinline__ bool feasible(const EnumArgs& a, const uint8_t* smask,
                                         unsigned long long idx, long long* key) {
  int pick[kMaxB];
  // request 0 most significant (planner.cpp decode); two 32-bit halves so no
  // 64-bit division runs per request
  unsigned hi = (unsigned)(idx / a.lo_span);
  unsigned lo = (unsigned)(idx - (unsigned long long)hi * a.lo_span);
  for (int r = a.B - 1; r >= a.B - a.lo_reqs; --r) {
    pick[r] = (int)(lo % (unsigned)a.C);
    lo /= (unsigned)a.C;
  }
  for (int r = a.B - a.lo_reqs - 1; r >= 0; --r) {
    pick[r] = (int)(hi % (unsigned)a.C);
    hi /= (unsigned)a.C;
  }
  long long res = 0, fetch = 0;
  for (int r = 0; r < a.B; ++r) {
    res += a.blocks[r] * (a.L - a.count[pick[r]]);
    fetch += a.blocks[r] * a.count[pick[r]];
  }
  if (res > a.budget) return false;
  long long worst = 0;
  for (int l = 0; l < a.L; ++l) {
    long long d = 0;
    for (int r = 0; r < a.B; ++r) d += smask[pick[r] * a.L + l] ? a.blocks[r] : 0;
    worst = d > worst ? d : worst;
  }
  if (res + worst > a.budget) return false;
  *key = ((double)fetch / a.bw <= a.compL) ? 0 : fetch + 1;
  return true;
}

// Pass 1: feasible candidates per lower-bound key (same-key lanes of a warp
// aggregate first: the compute-bound key 0 is the hot bin).
__global__ void histogram_kernel(const __grid_constant__ EnumArgs a, const uint8_t* __restrict__ mask,
                                 unsigned long long* __restrict__ hist) {
  __shared__ uint8_t smask[kMaxC * kMaxL];
  for (int i = threadIdx.x; i < a.C * a.L; i += blockDim.x) smask[i] = mask[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = a.idx_begin + (unsigned long long)blockIdx.x * blockDim.x;
       base < a.idx_end; base += stride) {
    const unsigned long long idx = base + threadIdx.x;
    long long key = -1;
    if (idx < a.idx_end && !feasible(a, smask, idx, &key)) key = -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && lane == (unsigned)(__ffs(peers) - 1))
      atomicAdd(&hist[key], (unsigned long long)__popc(peers));
  }
}

// Pass 2: feasible candidates of [idx_begin, idx_end) with key in [key_lo,
// key_hi], compacted with warp-aggregated atomics as (key << idx_bits | idx);
// one radix sort restores exactly the host's (key, enumeration index) order.
__global__ void materialise_kernel(const __grid_constant__ EnumArgs a, const uint8_t* __restrict__ mask,
                                   unsigned long long* __restrict__ out,
                                   unsigned long long* __restrict__ n_out) {
  __shared__ uint8_t smask[kMaxC * kMaxL];
  for (int i = threadIdx.x; i < a.C * a.L; i += blockDim.x) smask[i] = mask[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = a.idx_begin + (unsigned long long)blockIdx.x * blockDim.x;
       base < a.idx_end; base += stride) {
    const unsigned long long idx = base + threadIdx.x;
    long long key = -1;
    const bool keep = idx < a.idx_end && feasible(a, smask, idx, &key) && key >= a.key_lo &&
                      key <= a.key_hi;
    const unsigned ballot = __ballot_sync(0xffffffffu, keep);
    if (ballot) {
      unsigned long long slot = 0;
      if (lane == 0) slot = atomicAdd(n_out, (unsigned long long)__popc(ballot));
      slot = __shfl_sync(0xffffffffu, slot, 0);
      const unsigned long long at = slot + __popc(ballot & ((1u << lane) - 1u));
      if (keep && at < a.out_cap) out[at] = ((unsigned long long)key << a.idx_bits) | idx;
    }
  }
}

struct Handle {
  EnumArgs args{};
  cudaStream_t stream = nullptr;
  uint8_t* d_mask = nullptr;
  std::vector<unsigned long long> hist;   // feasible per key (host copy)
  long long window_cap = kDefaultWindow;
  long long n = 0;                        // feasible in all
  int end_bit = 64;
  // the materialised window: sorted candidates [wstart, wstart + wn) of the list
  unsigned long long* keys = nullptr;
  unsigned long long* sorted = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  long long wstart = 0, wn = 0;
  // cursor of the next window: whole keys from next_key on, or (bucket mode) the
  // index range [bucket_pos, ...) of one key whose bucket exceeds the window
  long long next_key = 0;
  bool bucket_mode = false;
  unsigned long long bucket_pos = 0;
  unsigned long long total = 0;
  int windows = 0;
};

// Private stream-ordered pool that keeps its memory between solves (the
// engine re-plans every few steps; fresh cudaMalloc/cudaFree of the window
// buffers cost more than a small solve).
cudaMemPool_t plan_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      pools[dev] = nullptr;
      return nullptr;
    }
    unsigned long long keep = 2ull << 30;   // keep up to one window's buffers cached
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return pools[dev];
}

template <typename T>
cudaError_t pool_alloc(T** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = plan_pool();
  if (!pool) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, s);
}

bool cuda_ok(cudaError_t e, const char* what, std::string* err) {
  if (e != cudaSuccess) *err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaSuccess;
}

// Materialise the next window after the current one.
bool advance(Handle* h, std::string* err) {
  EnumArgs a = h->args;
  h->wstart += h->wn;
  h->wn = 0;
  const long long nkeys = (long long)h->hist.size();
  if (!h->bucket_mode) {
    while (h->next_key < nkeys && h->hist[h->next_key] == 0) ++h->next_key;
    if (h->next_key >= nkeys) {
      *err = "plan_gpu_fetch: past the end of the candidate list";
      return false;
    }
    if ((long long)h->hist[h->next_key] > h->window_cap) {
      h->bucket_mode = true;
      h->bucket_pos = 0;
    }
  }
  if (h->bucket_mode) {   // one key, an index range of at most window_cap candidates
    a.key_lo = a.key_hi = h->next_key;
    a.idx_begin = h->bucket_pos;
    a.idx_end = h->bucket_pos + (unsigned long long)h->window_cap;
    if (a.idx_end > h->total) a.idx_end = h->total;
    h->bucket_pos = a.idx_end;
    if (h->bucket_pos >= h->total) {
      h->bucket_mode = false;
      ++h->next_key;
    }
  } else {                // whole keys while they fit the window
    long long k = h->next_key, sum = 0;
    while (k < nkeys && sum + (long long)h->hist[k] <= h->window_cap) sum += (long long)h->hist[k++];
    a.key_lo = h->next_key;
    a.key_hi = k - 1;
    a.idx_begin = 0;
    a.idx_end = h->total;
    h->next_key = k;
  }
  a.out_cap = (unsigned long long)h->window_cap;
  unsigned long long got = 0;
  unsigned long long* d_n = nullptr;
  cudaStream_t s = h->stream;
  bool ok = cuda_ok(pool_alloc(&d_n, sizeof(unsigned long long), s), "pool alloc", err) &&
            cuda_ok(cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), s), "memset", err);
  if (ok) {
    materialise_kernel<<<148 * 8, 256, 0, s>>>(a, h->d_mask, h->keys, d_n);
    ok = cuda_ok(cudaGetLastError(), "materialise_kernel", err) &&
         cuda_ok(cudaMemcpyAsync(&got, d_n, sizeof(got), cudaMemcpyDeviceToHost, s), "D2H", err) &&
         cuda_ok(cudaStreamSynchronize(s), "sync", err);
  }
  if (d_n) cudaFreeAsync(d_n, s);
  if (!ok) return false;
  if (got > (unsigned long long)h->window_cap) {
    *err = "plan_gpu_fetch: window overflow";
    return false;
  }
  if (got > 0) {
    size_t need = 0;
    ok = cuda_ok(cub::DeviceRadixSort::SortKeys(nullptr, need, h->keys, h->sorted, (int)got, 0,
                                                h->end_bit, s), "cub sizing", err);
    if (ok && need > h->tmp_bytes) {
      if (h->tmp) cudaFreeAsync(h->tmp, s);
      h->tmp = nullptr;
      h->tmp_bytes = 0;
      ok = cuda_ok(pool_alloc(&h->tmp, need, s), "pool alloc(tmp)", err);
      if (ok) h->tmp_bytes = need;
    }
    ok = ok && cuda_ok(cub::DeviceRadixSort::SortKeys(h->tmp, h->tmp_bytes, h->keys, h->sorted,
                                                      (int)got, 0, h->end_bit, s), "cub SortKeys", err) &&
         cuda_ok(cudaStreamSynchronize(s), "sync", err);
    if (!ok) return false;
  }
  h->wn = (long long)got;
  ++h->windows;
  return true;
}

void destroy(Handle* h) {
  if (!h) return;
  cudaStream_t s = h->stream;
  if (h->keys) cudaFreeAsync(h->keys, s);
  if (h->sorted) cudaFreeAsync(h->sorted, s);
  if (h->tmp) cudaFreeAsync(h->tmp, s);
  if (h->d_mask) cudaFreeAsync(h->d_mask, s);
  if (s) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  delete h;
}

}  // namespace

// Feasible candidates of the product space, in (lower-bound key, enumeration
// index) order, served in windows: one histogram pass counts the feasible
// candidates per key, then each window materialises and sorts a run of whole
// keys (or an index range of one oversized key) of at most `window` candidates,
// so memory stays bounded for spaces up to 2^36 (B = 10 at L = 32).
// Returns 0 and a handle, or an error code with *err set.
int plan_gpu_enumerate(int B, int C, int L, const int* count, const uint8_t* mask,
                       const int64_t* blocks, int64_t budget, double compL, double bw,
                       void** handle, int64_t* n_feasible, std::string* err) {
  *handle = nullptr;
  *n_feasible = 0;
  if (B > kMaxB || C > kMaxC || L > kMaxL || C < 1) {
    *err = "planner enumeration: shape beyond the GPU kernel's limits";
    return -1;
  }
  unsigned long long total = 1;
  for (int r = 0; r < B; ++r) {
    total *= (unsigned long long)C;
    if (total > (1ull << kIdxBitsMax)) {
      *err = "planner enumeration: candidate space exceeds 2^36";
      return -1;
    }
  }
  long long max_fetch = 0;
  for (int r = 0; r < B; ++r) max_fetch += blocks[r] * L;
  if (max_fetch + 2 > kMaxKeyBins) {
    *err = "planner enumeration: fetch volume beyond the key histogram";
    return -1;
  }
  Handle* h = new Handle();
  EnumArgs& a = h->args;
  a.B = B;
  a.C = C;
  a.L = L;
  a.lo_reqs = 0;
  a.lo_span = 1;
  // the low part covers the last requests up to 2^16 (so the split decode is
  // exercised at every batch, not only past 2^32)
  while (a.lo_reqs < B && (unsigned long long)a.lo_span * C <= (1ull << 16)) {
    a.lo_span *= (unsigned)C;
    ++a.lo_reqs;
  }
  a.idx_bits = 1;
  while (a.idx_bits < 64 && (1ull << a.idx_bits) < total) ++a.idx_bits;
  a.budget = budget;
  a.compL = compL;
  a.bw = bw;
  a.idx_begin = 0;
  a.idx_end = total;
  for (int c = 0; c < C; ++c) a.count[c] = count[c];
  for (int r = 0; r < B; ++r) a.blocks[r] = blocks[r];
  h->total = total;
  int key_bits = 1;
  while ((1ll << key_bits) <= max_fetch + 1) ++key_bits;
  h->end_bit = a.idx_bits + key_bits;
  if (h->end_bit > 64) {
    *err = "planner enumeration: (key, index) does not fit 64 bits";
    destroy(h);
    return -1;
  }
  if (const char* w = std::getenv("OFB_PLAN_WINDOW")) {   // tests: force small windows
    const long long v = std::atoll(w);
    if (v > 0 && v <= (1ll << 30)) h->window_cap = v;
  }
  const size_t nbins = (size_t)max_fetch + 2;
  unsigned long long* d_hist = nullptr;
  cudaStream_t& s = h->stream;
  bool ok = cuda_ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate", err) &&
            cuda_ok(pool_alloc(&h->d_mask, (size_t)C * L, s), "pool alloc(mask)", err) &&
            cuda_ok(pool_alloc(&d_hist, nbins * 8, s), "pool alloc(hist)", err) &&
            cuda_ok(cudaMemcpyAsync(h->d_mask, mask, (size_t)C * L, cudaMemcpyHostToDevice, s), "H2D", err) &&
            cuda_ok(cudaMemsetAsync(d_hist, 0, nbins * 8, s), "memset", err);
  if (ok) {
    histogram_kernel<<<148 * 8, 256, 0, s>>>(a, h->d_mask, d_hist);
    h->hist.resize(nbins);
    ok = cuda_ok(cudaGetLastError(), "histogram_kernel", err) &&
         cuda_ok(cudaMemcpyAsync(h->hist.data(), d_hist, nbins * 8, cudaMemcpyDeviceToHost, s), "D2H", err) &&
         cuda_ok(cudaStreamSynchronize(s), "sync", err);
  }
  if (d_hist) cudaFreeAsync(d_hist, s);
  if (ok) {
    for (unsigned long long c : h->hist) h->n += (long long)c;
    const long long cap = h->n < h->window_cap ? h->n : h->window_cap;
    if (cap > 0)
      ok = cuda_ok(pool_alloc(&h->keys, (size_t)cap * 8, s), "pool alloc(window)", err) &&
           cuda_ok(pool_alloc(&h->sorted, (size_t)cap * 8, s), "pool alloc(sorted)", err);
    if (cap < h->window_cap) h->window_cap = cap > 0 ? cap : 1;
  }
  if (ok && h->n > 0) ok = advance(h, err);   // the first window up front
  if (!ok) {
    destroy(h);
    return -1;
  }
  *handle = h;
  *n_feasible = (int64_t)h->n;
  return 0;
}

// Enumeration indices of sorted candidates [from, from + count); the ranker
// pulls in order, so a request past the current window materialises the next.
int plan_gpu_fetch(void* handle, int64_t from, int64_t count, uint64_t* dst, std::string* err) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || from < 0 || count < 0 || from + count > h->n) {
    *err = "plan_gpu_fetch: range out of bounds";
    return -1;
  }
  const uint64_t mask = (h->args.idx_bits >= 64) ? ~0ull : ((1ull << h->args.idx_bits) - 1);
  while (count > 0) {
    if (from < h->wstart) {
      *err = "plan_gpu_fetch: candidates are served in order (window already released)";
      return -1;
    }
    while (from >= h->wstart + h->wn)
      if (!advance(h, err)) return -1;
    const int64_t take = std::min<int64_t>(count, h->wstart + h->wn - from);
    // on the handle's non-blocking stream: a re-plan never waits for decode
    // steps queued on the legacy default stream
    cudaError_t e = cudaMemcpyAsync(dst, h->sorted + (from - h->wstart), (size_t)take * 8,
                                    cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
      *err = std::string("plan_gpu_fetch: ") + cudaGetErrorString(e);
      return -1;
    }
    for (int64_t i = 0; i < take; ++i) dst[i] &= mask;
    dst += take;
    from += take;
    count -= take;
  }
  return 0;
}

int plan_gpu_windows(void* handle) {
  Handle* h = static_cast<Handle*>(handle);
  return h ? h->windows : 0;
}

void plan_gpu_free(void* handle) { destroy(static_cast<Handle*>(handle)); }

}  // namespace ofb
