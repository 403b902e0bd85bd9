// Native exact placement solver (host code).
//
// Restates kvsim's ranked exhaustive solve (/root/reference/pkg/src/kvsim/
// planner.py:234-560) so that it returns the *same* plan bit-for-bit, only
// faster (C++, multithreaded):
//   * candidates = product of enumerate_distances(L) over the batch, Eq. 1
//     capacity filter at current sizes (planner.py:310-341);
//   * latency of a candidate = the batched float evaluator's arithmetic in its
//     exact operation order (planner.py:234-299: equal-share completion times
//     as a cumulative sum divided by the bandwidth once, survivors credited
//     base + (window - t_k) * bw / survivors, clamped at zero);
//   * rank key (round-half-even(latency / 1e-9), fetched blocks, stride keys
//     lexicographically) (planner.py:394-395), candidates priced lazily in
//     lower-bound order max(L * comp, fetch / bw) (planner.py:344-414);
//   * first-step pre-rejection, window_min forecast, window_max forecast and
//     greedy window extension (planner.py:136-208, :417-498), the forecast
//     using the scalar schedule (latency.py:141-209) and CPython's
//     compensated float sum() for sum(stalls).
// Build with -ffp-contract=off: no FMA may change a rounding.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <cstdlib>
#include <thread>
#include <vector>

#include "../../include/orbitflow_b200.h"

namespace ofb {
int plan_gpu_enumerate(int B, int C, int L, const int* count, const uint8_t* mask,
                       const int64_t* blocks, int64_t budget, double compL, double bw,
                       void** handle, int64_t* n_feasible, std::string* err);
int plan_gpu_fetch(void* handle, int64_t from, int64_t count, uint64_t* dst, std::string* err);
void plan_gpu_free(void* handle);
int plan_gpu_windows(void* handle);
}  // namespace ofb

namespace {

thread_local std::string g_plan_err;

constexpr double kRankEps = 1e-9;
constexpr double kSlackEps = 1e-9;
constexpr double kCapEps = 1e-9;

struct Options {
  int L = 0, C = 0, depth = 1;
  std::vector<int> stride;     // -1 = resident
  std::vector<int> count;      // offloaded layers
  std::vector<int> key;        // sort key
  std::vector<uint8_t> mask;   // [C][L], 1 = offloaded
  std::vector<int> dests;      // [C][depth], 1-based layers ascending, 0-padded

  explicit Options(int layers) : L(layers) {
    // RESIDENT, widest stride per distinct count L//k (k=2..L) ascending, stride 1
    std::vector<int> counts;
    for (int k = 2; k <= L; ++k) counts.push_back(L / k);
    std::sort(counts.begin(), counts.end());
    counts.erase(std::unique(counts.begin(), counts.end()), counts.end());
    stride.push_back(-1);
    for (int c : counts) stride.push_back(L / c);
    stride.push_back(1);
    C = (int)stride.size();
    for (int s : stride) {
      count.push_back(s < 0 ? 0 : L / s);
      key.push_back(s < 0 ? L + 1 : s);
    }
    depth = std::max(1, *std::max_element(count.begin(), count.end()));
    mask.assign((size_t)C * L, 0);
    dests.assign((size_t)C * depth, 0);
    for (int c = 0; c < C; ++c) {
      if (stride[c] < 0) continue;
      int j = 0;
      for (int l = stride[c]; l <= L; l += stride[c]) {
        mask[(size_t)c * L + l - 1] = 1;
        dests[(size_t)c * depth + j++] = l;
      }
    }
  }
};

// CPython >= 3.12 sum() over floats: Neumaier-compensated (Python/bltinmodule.c).
struct PySum {
  double f = 0.0, c = 0.0;
  bool started = false;
  void add(double x) {
    if (!started) {
      f = 0.0 + x;
      started = true;
      return;
    }
    const double t = f + x;
    if (std::fabs(f) >= std::fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  double result() const {
    double r = started ? f : 0.0;
    if (c != 0.0 && std::isfinite(c)) r += c;
    return r;
  }
};

// ---------------------------------------------------------------- evaluators

// Batched-evaluator arithmetic for one candidate (planner.py:234-299).
double vector_latency(const Options& op, const int* pick, const double* sizes, int B, double comp,
                      double bw) {
  const int L = op.L;
  double rem[64], sa[64], t[64];
  int dest[64], ptr[64], order[64];
  uint8_t active[64];
  for (int r = 0; r < B; ++r) {
    rem[r] = 0.0;
    dest[r] = 0;
    ptr[r] = 0;
  }
  double stall_tot = 0.0;
  for (int layer = 1; layer <= L; ++layer) {
    bool pending = false, inflight = false;
    for (int r = 0; r < B; ++r) {
      pending |= ptr[r] < op.count[pick[r]];
      inflight |= rem[r] > 0.0;
    }
    if (!pending && !inflight) break;
    for (int r = 0; r < B; ++r) {
      const int c = pick[r];
      const int nd = op.dests[(size_t)c * op.depth + std::min(ptr[r], op.depth - 1)];
      if (rem[r] <= 0.0 && ptr[r] < op.count[c] &&
          (nd == layer || op.mask[(size_t)c * L + layer - 1] == 0)) {
        rem[r] = sizes[r];
        dest[r] = nd;
        ptr[r] += 1;
      }
    }
    int nact = 0;
    for (int r = 0; r < B; ++r) {
      active[r] = rem[r] > 0.0;
      if (active[r]) order[nact++] = r;
    }
    if (nact == 0) continue;
    // stable ascending by remaining (inactive sort last as +inf in the original)
    std::stable_sort(order, order + nact, [&](int x, int y) { return rem[x] < rem[y]; });
    double acc = 0.0, prev = 0.0;
    for (int j = 0; j < nact; ++j) {
      sa[j] = rem[order[j]];
      acc = acc + (sa[j] - prev) * (double)(nact - j);
      t[j] = acc / bw;
      prev = sa[j];
    }
    double stall = 0.0;
    for (int j = 0; j < nact; ++j)
      if (dest[order[j]] == layer && t[j] > stall) stall = t[j];
    const double window = stall + comp;
    const double limit = window + kSlackEps * (1.0 + window);
    int k = 0;
    for (int j = 0; j < nact; ++j)
      if (t[j] <= limit) ++k;
    const double base = k > 0 ? sa[k - 1] : 0.0;
    const double t_k = k > 0 ? t[k - 1] : 0.0;
    const int surv = nact - k;
    const double served = surv > 0 ? base + (window - t_k) * bw / (double)std::max(surv, 1) : 0.0;
    for (int j = 0; j < nact; ++j) {
      const int r = order[j];
      if (t[j] <= limit) {
        rem[r] = 0.0;
      } else {
        rem[r] = rem[r] - served;
        if (rem[r] <= 0.0) rem[r] = 0.0;
      }
    }
    for (int r = 0; r < B; ++r)
      if (!(rem[r] > 0.0)) dest[r] = 0;
    stall_tot += stall;
  }
  return comp * (double)L + stall_tot;
}

// Scalar schedule (latency.py:141-209), float flavour; returns sum(stalls)
// with CPython's summation.
double scalar_stall_sum(const int* sizes, const uint8_t* offl, int B, int L, double comp,
                        double bw) {
  struct F {
    bool on = false;
    int dest = 0;
    double rem = 0, fin = 0;
  };
  F f[64];
  int nxt[64];
  for (int r = 0; r < B; ++r) nxt[r] = 0;
  int order[64];
  PySum total;
  for (int layer = 1; layer <= L; ++layer) {
    for (int r = 0; r < B; ++r) {
      if (f[r].on) continue;
      int d = -1;
      for (int l = nxt[r]; l < L; ++l)
        if (offl[(size_t)r * L + l]) {
          d = l + 1;
          break;
        }
      if (d < 0) continue;
      if (d == layer || !offl[(size_t)r * L + layer - 1]) {
        f[r].on = true;
        f[r].dest = d;
        f[r].rem = (double)sizes[r];
        nxt[r] = d;
      }
    }
    int m = 0;
    for (int r = 0; r < B; ++r)
      if (f[r].on) order[m++] = r;
    double stall = 0.0;
    if (m > 0) {
      std::sort(order, order + m, [&](int x, int y) {
        if (f[x].rem != f[y].rem) return f[x].rem < f[y].rem;
        if (f[x].dest != f[y].dest) return f[x].dest < f[y].dest;
        return x < y;
      });
      double tt = 0.0, prev = 0.0;
      for (int j = 0; j < m; ++j) {
        F& s = f[order[j]];
        tt = tt + (s.rem - prev) * (double)(m - j) / bw;
        s.fin = tt;
        prev = s.rem;
      }
      bool blocked = false;
      for (int j = 0; j < m; ++j) {
        const F& s = f[order[j]];
        if (s.dest == layer && (!blocked || s.fin > stall)) {
          stall = s.fin;
          blocked = true;
        }
      }
      const double window = stall + comp;
      const double limit = window + kSlackEps * (1.0 + window);
      int k = 0;
      for (int j = 0; j < m; ++j)
        if (f[order[j]].fin <= limit) ++k;
      if (k < m) {
        const double base = k > 0 ? f[order[k - 1]].rem : 0.0;
        const double t_k = k > 0 ? f[order[k - 1]].fin : 0.0;
        const double served = base + (window - t_k) * bw / (double)(m - k);
        for (int j = 0; j < m; ++j)
          if (f[order[j]].fin > limit) f[order[j]].rem = f[order[j]].rem - served;
      }
      for (int j = 0; j < m; ++j)
        if (f[order[j]].fin <= limit) f[order[j]].on = false;
    }
    total.add(stall);
  }
  return total.result();
}

struct Problem {
  const ofb_plan_problem* p;
  Options op;
  std::vector<double> sizes_d;
  double comp = 0;
  explicit Problem(const ofb_plan_problem* pp) : p(pp), op(pp->num_layers) {
    int64_t tokens = 0;
    for (int r = 0; r < pp->batch; ++r) {
      sizes_d.push_back((double)pp->blocks[r]);
      tokens += pp->total_tokens[r];
    }
    comp = pp->compute_base_ms + pp->compute_per_token_ms * (double)tokens;
  }
};

// forecast_violations (planner.py:136-208) for a stride assignment.
int forecast(const Problem& P, const int* pick, int horizon, const double* live_seed,
             const double* parked_seed, int num_paused, std::vector<int>* fails_out) {
  const ofb_plan_problem* p = P.p;
  const int B = p->batch, L = p->num_layers;
  std::vector<uint8_t> offl((size_t)B * L);
  std::vector<int> resident_count(B);
  for (int r = 0; r < B; ++r) {
    int res = 0;
    for (int l = 0; l < L; ++l) {
      offl[(size_t)r * L + l] = P.op.mask[(size_t)pick[r] * L + l];
      res += !offl[(size_t)r * L + l];
    }
    resident_count[r] = res;
  }
  std::vector<double> live(live_seed, live_seed + B), parked(parked_seed, parked_seed + num_paused);
  std::vector<int> sizes(B);
  fails_out->clear();
  for (int step = 1; step <= horizon; ++step) {
    int64_t tok_sum = 0;
    for (int r = 0; r < B; ++r) {
      const int64_t tok = p->total_tokens[r] + step - 1;
      sizes[r] = (int)((tok + p->block_size - 1) / p->block_size);
      tok_sum += tok;
    }
    int64_t resident = 0, buffer = 0;
    for (int r = 0; r < B; ++r) resident += (int64_t)sizes[r] * resident_count[r];
    for (int l = 0; l < L; ++l) {
      int64_t demand = 0;
      for (int r = 0; r < B; ++r)
        if (offl[(size_t)r * L + l]) demand += sizes[r];
      buffer = std::max(buffer, demand);
    }
    if (resident + buffer > p->gpu_block_budget) return step;  // truncated_at
    const double comp = p->compute_base_ms + p->compute_per_token_ms * (double)tok_sum;
    const double latency =
        comp * (double)L +
        scalar_stall_sum(sizes.data(), offl.data(), B, L, comp, p->bandwidth_blocks_per_ms);
    const bool late = latency > p->tbt_ms;
    int fails = 0;
    for (int r = 0; r < B; ++r) {
      const double bal = live[r] + 1.0 - latency / p->tbt_ms;
      if (late && bal < 0.0) ++fails;
      live[r] = std::max(bal, 0.0);
    }
    for (int j = 0; j < num_paused; ++j) {
      const double bal = parked[j] - latency / p->tbt_ms;
      if (bal < 0.0) ++fails;
      parked[j] = std::max(bal, 0.0);
    }
    fails_out->push_back(fails);
  }
  return 0;
}

// ------------------------------------------------------------------ ranking

struct Cand {
  int64_t idx;    // mixed-radix choice tuple, request 0 most significant
  int64_t fetch;
};

struct Ranked {
  double rkey;    // round-half-even(lat / 1e-9)
  int64_t fetch;
  int64_t idx;
  double lat;
};

void decode(int64_t idx, int C, int B, int* pick) {
  for (int r = B - 1; r >= 0; --r) {
    pick[r] = (int)(idx % C);
    idx /= C;
  }
}

// true if a ranks strictly before b: (rkey, fetch, stride keys lexicographic)
bool rank_less(const Options& op, int B, const Ranked& a, const Ranked& b) {
  if (a.rkey != b.rkey) return a.rkey < b.rkey;
  if (a.fetch != b.fetch) return a.fetch < b.fetch;
  int pa[64], pb[64];
  decode(a.idx, op.C, B, pa);
  decode(b.idx, op.C, B, pb);
  for (int r = 0; r < B; ++r) {
    const int ka = op.key[pa[r]], kb = op.key[pb[r]];
    if (ka != kb) return ka < kb;
  }
  return false;
}

template <typename Fn>
void parallel_for(int64_t n, int threads, Fn fn) {
  if (threads <= 1 || n < 4096) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> ts;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    ts.emplace_back([=, &fn] { fn(lo, hi); });
  }
  for (auto& th : ts) th.join();
}

struct Ranker {
  const Problem& P;
  int B, threads;
  std::vector<Cand> cands;        // capacity-feasible, in lower-bound order (a prefix
                                  // when the list lives on the GPU, pulled in chunks)
  std::vector<double> lb;
  int64_t total = 0;              // feasible candidates in all
  void* gpu = nullptr;            // device-sorted candidate list (build_gpu)
  ~Ranker() { ofb::plan_gpu_free(gpu); }
  size_t priced = 0;
  std::vector<Ranked> heap;       // min-heap of priced, unreleased candidates
  int64_t n_priced = 0;

  Ranker(const Problem& pr, int th) : P(pr), B(pr.p->batch), threads(th) {}

  // Capacity-feasible candidates in lower-bound order (planner.py:310-341, :365-372).
  // Depth-first over requests in enumeration order: resident blocks and every
  // layer's offloaded demand only grow as requests are added, so a partial
  // assignment already over budget prunes its whole subtree.  Subtrees of the
  // first requests' choices run in parallel; concatenating them in root order
  // keeps enumeration order.  The lower bound max(L*comp, fetch/bw) is then a
  // stable counting sort on the integer fetch volume.
  bool build() {
    const Options& op = P.op;
    const int C = op.C, L = op.L;
    const int64_t budget = P.p->gpu_block_budget;
    const int split = std::min(B, C >= 8 ? 2 : 3);
    int64_t roots = 1;
    for (int r = 0; r < split; ++r) roots *= C;
    std::vector<std::vector<Cand>> part(roots);
    std::atomic<int64_t> next_root{0};
    auto worker = [&] {
      std::vector<int64_t> demand((size_t)(B + 1) * L);
      std::vector<int64_t> res(B + 1), fet(B + 1);
      int pick[64];
      while (true) {
        const int64_t root = next_root.fetch_add(1);
        if (root >= roots) break;
        std::vector<Cand>& out = part[root];
        // decode the root prefix
        int64_t rr = root;
        for (int r = split - 1; r >= 0; --r) {
          pick[r] = (int)(rr % C);
          rr /= C;
        }
        std::fill(demand.begin(), demand.begin() + L, 0);
        res[0] = fet[0] = 0;
        bool ok = true;
        for (int r = 0; r < split && ok; ++r) {
          const int c = pick[r];
          const int64_t sz = P.p->blocks[r];
          res[r + 1] = res[r] + sz * (L - op.count[c]);
          fet[r + 1] = fet[r] + sz * op.count[c];
          int64_t worst = 0;
          for (int l = 0; l < L; ++l) {
            const int64_t v = demand[(size_t)r * L + l] + (op.mask[(size_t)c * L + l] ? sz : 0);
            demand[(size_t)(r + 1) * L + l] = v;
            worst = std::max(worst, v);
          }
          ok = res[r + 1] + worst <= budget;
        }
        if (!ok) continue;
        if (split == B) {
          out.push_back({root, fet[B]});
          continue;
        }
        // iterative DFS below the root
        int depth = split;
        pick[depth] = -1;
        while (depth >= split) {
          const int c = ++pick[depth];
          if (c >= C) {
            --depth;
            continue;
          }
          const int64_t sz = P.p->blocks[depth];
          const int64_t rs = res[depth] + sz * (L - op.count[c]);
          if (rs > budget) continue;
          const int64_t* dprev = &demand[(size_t)depth * L];
          int64_t* dnext = &demand[(size_t)(depth + 1) * L];
          const uint8_t* m = &op.mask[(size_t)c * L];
          int64_t worst = 0;
          for (int l = 0; l < L; ++l) {
            const int64_t v = dprev[l] + (m[l] ? sz : 0);
            dnext[l] = v;
            worst = std::max(worst, v);
          }
          if (rs + worst > budget) continue;
          res[depth + 1] = rs;
          fet[depth + 1] = fet[depth] + sz * op.count[c];
          if (depth + 1 == B) {
            int64_t idx = 0;
            for (int r = 0; r < B; ++r) idx = idx * C + pick[r];
            out.push_back({idx, fet[B]});
          } else {
            ++depth;
            pick[depth] = -1;
          }
        }
      }
    };
    // Threads only pay off on large spaces: spawning them costs ~30 us each, which
    // made a B <= 3 solve (<= 36k candidates, microseconds of work) take 0.5 ms -
    // the serving loop's largest host cost when it re-plans every step.
    double space = 1.0;
    for (int r = 0; r < B; ++r) space *= C;
    const int workers = space < 65536.0 ? 1 : std::min<int64_t>(threads, roots);
    std::vector<std::thread> ts;
    for (int t = 1; t < workers; ++t) ts.emplace_back(worker);
    worker();
    for (auto& th : ts) th.join();
    size_t n = 0;
    for (auto& v : part) n += v.size();
    if (n == 0) return false;
    // stable counting sort by lower bound: fetch/bw <= L*comp all tie at L*comp
    const double compL = P.comp * (double)L;
    const double bw = P.p->bandwidth_blocks_per_ms;
    int64_t max_f = 0;
    for (auto& v : part)
      for (auto& c : v) max_f = std::max(max_f, c.fetch);
    auto key = [&](int64_t f) -> int64_t { return ((double)f / bw <= compL) ? 0 : f + 1; };
    std::vector<int64_t> count((size_t)max_f + 2, 0);
    for (auto& v : part)
      for (auto& c : v) ++count[(size_t)key(c.fetch)];
    int64_t run = 0;
    for (auto& x : count) {
      const int64_t k = x;
      x = run;
      run += k;
    }
    cands.resize(n);
    for (auto& v : part) {
      for (auto& c : v) cands[(size_t)count[(size_t)key(c.fetch)]++] = c;
      std::vector<Cand>().swap(v);
    }
    lb.resize(n);
    for (size_t i = 0; i < n; ++i) lb[i] = std::max(compL, (double)cands[i].fetch / bw);
    total = (int64_t)n;
    return true;
  }

  // Same list, enumerated and sorted on the GPU (planner_gpu.cu); the host keeps
  // only the prefix the ranking has reached.
  bool build_gpu() {
    const Options& op = P.op;
    const double compL = P.comp * (double)op.L;
    std::string err;
    if (ofb::plan_gpu_enumerate(B, op.C, op.L, op.count.data(), op.mask.data(), P.p->blocks,
                                P.p->gpu_block_budget, compL, P.p->bandwidth_blocks_per_ms,
                                &gpu, &total, &err) != 0)
      throw std::runtime_error(err);
    if (total == 0) return false;
    pull();
    return true;
  }

  static constexpr int64_t kPull = 1 << 20;

  void pull() {   // next chunk of the GPU-sorted list
    const int64_t from = (int64_t)cands.size();
    const int64_t n = std::min(kPull, total - from);
    if (n <= 0) return;
    std::vector<uint64_t> keys((size_t)n);
    std::string err;
    if (ofb::plan_gpu_fetch(gpu, from, n, keys.data(), &err) != 0) throw std::runtime_error(err);
    const Options& op = P.op;
    const double compL = P.comp * (double)op.L, bw = P.p->bandwidth_blocks_per_ms;
    int pick[64];
    for (uint64_t k : keys) {
      const int64_t idx = (int64_t)k;   // plan_gpu_fetch returns enumeration indices
      decode(idx, op.C, B, pick);
      int64_t fetch = 0;
      for (int r = 0; r < B; ++r) fetch += P.p->blocks[r] * op.count[pick[r]];
      cands.push_back({idx, fetch});
      lb.push_back(std::max(compL, (double)fetch / bw));
    }
  }

  void price_chunk() {
    const size_t lo = priced, hi = std::min(cands.size(), priced + 65536);
    std::vector<Ranked> out(hi - lo);
    const Options& op = P.op;
    const double bw = P.p->bandwidth_blocks_per_ms;
    parallel_for((int64_t)(hi - lo), threads, [&](int64_t a, int64_t b) {
      int pick[64];
      for (int64_t i = a; i < b; ++i) {
        const Cand& c = cands[lo + i];
        decode(c.idx, op.C, B, pick);
        const double lat = vector_latency(op, pick, P.sizes_d.data(), B, P.comp, bw);
        out[i] = {std::nearbyint(lat / kRankEps), c.fetch, c.idx, lat};
      }
    });
    priced = hi;
    n_priced += (int64_t)out.size();
    auto greater = [&](const Ranked& a, const Ranked& b) { return rank_less(op, B, b, a); };
    for (auto& r : out) {
      heap.push_back(r);
      std::push_heap(heap.begin(), heap.end(), greater);
    }
  }

  // Optional pricing cutoff: once it returns true for the next unpriced lower
  // bound, every unpriced candidate is known to be rejected downstream.
  std::function<bool(double)> hopeless;

  // next candidate in exact rank order (planner.py:398-414), or false
  bool next(Ranked* out) {
    auto greater = [&](const Ranked& a, const Ranked& b) { return rank_less(P.op, B, b, a); };
    while (true) {
      if (priced >= cands.size() && (int64_t)cands.size() < total) pull();
      bool drained = priced >= cands.size();
      if (!drained && hopeless && hopeless(lb[priced])) {
        cands.resize(priced);  // nothing past here can pass: stop pricing
        total = (int64_t)priced;
        drained = true;
      }
      if (!heap.empty() && (drained || heap.front().lat + kRankEps < lb[priced])) {
        std::pop_heap(heap.begin(), heap.end(), greater);
        *out = heap.back();
        heap.pop_back();
        return true;
      }
      if (drained) return false;
      price_chunk();
    }
  }
};

int window_extend(const ofb_plan_problem* p, const std::vector<int>& fails) {
  int window = p->window_min;
  while (window < p->window_max && window < (int)fails.size()) {
    int64_t s = 0;
    for (int i = 0; i <= window; ++i) s += fails[i];
    if (!((double)s <= p->violation_cap * (double)(window + 1) + kCapEps)) break;
    ++window;
  }
  return window;
}

}  // namespace

extern "C" {

const char* ofb_plan_last_error(void) { return g_plan_err.c_str(); }

static int solve_ranked(const ofb_plan_problem* p, const Problem& P, Ranker& rk, ofb_plan_result* out) {
  int pick[64];
  std::vector<int> fails;
  const int B = p->batch;
  if (p->mode == 1) {  // solve_capacity_only (planner.py:527-560)
    Ranked best;
    rk.next(&best);
    decode(best.idx, P.op.C, B, pick);
    const int trunc = forecast(P, pick, p->window_max, p->forecast_live, nullptr, 0, &fails);
    (void)trunc;
    const int horizon = (int)fails.size();
    out->decode_window = std::max(1, std::min(horizon, p->window_max));
  } else {
    const double tbt = p->tbt_ms, cap = p->violation_cap;
    // First-step failures grow with latency and latency >= its lower bound
    // (pure compute, and the bus time fetch/bw), so when the next unpriced
    // bound already fails the pre-rejection, all remaining candidates would.
    auto first_fails = [&](double lat) {
      int f = 0;
      if (lat > tbt)
        for (int r = 0; r < B; ++r)
          if (p->live_balance[r] + 1.0 - lat / tbt < 0.0) ++f;
      for (int j = 0; j < p->num_paused; ++j)
        if (p->parked_balance[j] - lat / tbt < 0.0) ++f;
      return f;
    };
    // The stall model's completion slack (kSlackEps per layer, scaled by the
    // window) can put a modelled latency below its bound by ~L*1e-9*(1+bound):
    // test the bound minus that absolute margin so the cutoff never fires early.
    const double slack_margin = (double)P.op.L * kSlackEps;
    rk.hopeless = [&](double bound) {
      const double lo = bound * (1.0 - 1e-12) - slack_margin * (1.0 + bound);
      return (double)first_fails(lo) > cap + kCapEps;
    };
    while (true) {
      Ranked cand;
      if (!rk.next(&cand)) {
        out->status = 2;  // violation cap unsatisfiable for every placement
        out->candidates_priced = rk.n_priced;
        return 0;
      }
      out->candidates_ranked += 1;
      if ((double)first_fails(cand.lat) > cap + kCapEps) continue;
      decode(cand.idx, P.op.C, B, pick);
      forecast(P, pick, p->window_min, p->forecast_live, p->forecast_parked, p->num_paused, &fails);
      if ((int)fails.size() < p->window_min) continue;
      int64_t s = 0;
      for (int v : fails) s += v;
      if ((double)s > cap * (double)p->window_min + kCapEps) continue;
      forecast(P, pick, p->window_max, p->forecast_live, p->forecast_parked, p->num_paused, &fails);
      out->decode_window = window_extend(p, fails);
      break;
    }
  }
  out->expiry_step = p->current_step + out->decode_window;
  for (int r = 0; r < B; ++r) p->strides_out[r] = P.op.stride[pick[r]];
  out->candidates_priced = rk.n_priced;
  out->status = 0;
  return 0;
}


int ofb_plan_solve(const ofb_plan_problem* p, ofb_plan_result* out) {
  if (!p || !out) {
    g_plan_err = "null argument";
    return -1;
  }
  std::memset(out, 0, sizeof(*out));
  if (p->batch < 1 || p->batch > 12 || p->num_layers < 1 || p->num_paused < 0 ||
      p->num_paused > 64) {
    g_plan_err = "batch must be 1..12 and num_layers >= 1";
    return -1;
  }
  Problem P(p);
  int64_t space = 1;
  for (int r = 0; r < p->batch; ++r) space *= P.op.C;
  // host DFS: 2^28 (its list lives in host memory); GPU enumeration: 2^36,
  // served in bounded windows
  int host_log2 = 28;
  if (const char* v = std::getenv("OFB_PLAN_HOST_SPACE_LOG2")) {   // tests: oracle runs past 2^28
    const int x = std::atoi(v);
    if (x > 0 && x <= 36) host_log2 = x;
  }
  if (space > ((int64_t)1 << (p->device_enumerate ? 36 : host_log2))) {
    g_plan_err = "candidate space too large for exhaustive search";
    return -1;
  }
  const int threads = std::max(1, p->threads);
  Ranker rk(P, threads);
  bool any = false;
  try {
    any = p->device_enumerate ? rk.build_gpu() : rk.build();
  } catch (const std::exception& e) {
    g_plan_err = e.what();
    return -1;
  }
  if (!any) {
    out->enumeration_windows = rk.gpu ? ofb::plan_gpu_windows(rk.gpu) : 0;
    out->status = 1;  // no placement fits the GPU block budget
    return 0;
  }
  out->candidates_feasible = rk.total;
  try {
    const int rc = solve_ranked(p, P, rk, out);
    out->enumeration_windows = rk.gpu ? ofb::plan_gpu_windows(rk.gpu) : 0;
    return rc;
  } catch (const std::exception& e) {   // a GPU chunk pull failed
    g_plan_err = e.what();
    return -1;
  }
}

}  // extern "C"
