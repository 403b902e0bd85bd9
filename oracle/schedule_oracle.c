/*
 * TEST INFRASTRUCTURE ONLY - the checker, never the product path.
 *
 * Plain-C restatement of the reference's per-step transfer schedule and its
 * integer accounting, for parity checks of the host mirror
 * (paper_2601_10729_b200/latency.py) and of the fetch volumes the copy
 * streams actually move:
 *   - oracle_stall_schedule: float flavour of _simulate_stalls
 *     (/root/reference/pkg/src/kvsim/latency.py:141-209): launch rule
 *     (:159-169), equal-share completion order by (remaining, dest, request)
 *     (:172-184), blocking max (:185-187), window progress with the
 *     1e-9*(1+window) completion slack (:36, :189-204);
 *     total = comp*L + sum(stalls) (latency.py:264-266), with sum() being
 *     CPython's compensated float sum (see pysum_t).
 *   - oracle_blocks_to_fetch      latency.py:99-105
 *   - oracle_prefetch_buffer      latency.py:108-119 (Eq. 1)
 *   - oracle_reconfiguration_delta latency.py:277-297
 * Same IEEE-754 double operation order as the reference; build with
 * -ffp-contract=off so no FMA fusion changes a rounding.
 * Pinned by tests/test_oracle.py against golden vectors generated from the
 * reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define SLACK_EPS 1e-9

/* CPython >= 3.12 builtin sum() over floats: Neumaier-compensated running sum
 * (Python/bltinmodule.c builtin_sum_impl).  sum(stalls) in the reference
 * (latency.py:266, planner.py:192) therefore rounds differently from a plain
 * left fold; restated here so totals match to the bit.  The first term enters
 * exactly (0 + s1 == s1), compensation starts with the second. */
typedef struct {
  double f, c;
  int started;
} pysum_t;

static void pysum_add(pysum_t* s, double x) {
  if (!s->started) {
    s->f = 0.0 + x;
    s->started = 1;
    return;
  }
  const double t = s->f + x;
  if (fabs(s->f) >= fabs(x))
    s->c += (s->f - t) + x;
  else
    s->c += (x - t) + s->f;
  s->f = t;
}

static double pysum_result(const pysum_t* s) {
  double f = s->started ? s->f : 0.0;
  if (s->c != 0.0 && isfinite(s->c)) f += s->c;
  return f;
}

typedef struct {
  int active;
  int dest;
  double rem;
  double finish;
} stream_t;

/* sizes[r]: blocks per layer; offloaded[r*L + l] (l 0-based) = 1 if layer l+1
 * is host-resident.  stalls_out[L] optional.  Returns total latency (ms). */
double oracle_stall_schedule(int32_t n, const int64_t* sizes, const uint8_t* offloaded,
                             int32_t L, double comp, double bw, double* stalls_out) {
  stream_t* st = (stream_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(stream_t));
  int* next = (int*)calloc((size_t)(n > 0 ? n : 1), sizeof(int));
  int* order = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  pysum_t stall_sum = {0.0, 0.0, 0};
  for (int layer = 1; layer <= L; ++layer) {
    /* launch rule at the boundary of `layer` */
    for (int r = 0; r < n; ++r) {
      if (st[r].active) continue;
      int dest = -1;
      for (int l = next[r]; l < L; ++l)
        if (offloaded[(size_t)r * L + l]) { dest = l + 1; break; }
      if (dest < 0) continue;
      if (dest == layer || !offloaded[(size_t)r * L + (layer - 1)]) {
        st[r].active = 1;
        st[r].dest = dest;
        st[r].rem = (double)sizes[r];
        next[r] = dest; /* next search starts after dest (0-based index dest) */
      }
    }
    int m = 0;
    for (int r = 0; r < n; ++r)
      if (st[r].active) order[m++] = r;
    double stall = 0.0;
    if (m > 0) {
      /* insertion sort by (rem, dest, request) */
      for (int i = 1; i < m; ++i) {
        int v = order[i], j = i - 1;
        while (j >= 0) {
          const stream_t* a = &st[order[j]];
          const stream_t* b = &st[v];
          int greater = a->rem > b->rem || (a->rem == b->rem && (a->dest > b->dest ||
                        (a->dest == b->dest && order[j] > v)));
          if (!greater) break;
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = v;
      }
      double t = 0.0, prev = 0.0;
      for (int j = 0; j < m; ++j) {
        stream_t* s = &st[order[j]];
        t = t + (s->rem - prev) * (double)(m - j) / bw;
        s->finish = t;
        prev = s->rem;
      }
      int blocked = 0;
      for (int j = 0; j < m; ++j) {
        const stream_t* s = &st[order[j]];
        if (s->dest == layer) {
          if (!blocked || s->finish > stall) stall = s->finish;
          blocked = 1;
        }
      }
      const double window = stall + comp;
      const double slack = SLACK_EPS * (1.0 + window);
      int k = 0;
      for (int j = 0; j < m; ++j)
        if (st[order[j]].finish <= window + slack) ++k;
      if (k < m) {
        const double base = k > 0 ? st[order[k - 1]].rem : 0.0;
        const double t_k = k > 0 ? st[order[k - 1]].finish : 0.0;
        const double served = base + (window - t_k) * bw / (double)(m - k);
        for (int j = 0; j < m; ++j) {
          stream_t* s = &st[order[j]];
          if (s->finish > window + slack) s->rem = s->rem - served;
        }
      }
      for (int j = 0; j < m; ++j) {
        stream_t* s = &st[order[j]];
        if (s->finish <= window + slack) s->active = 0;
      }
    }
    if (stalls_out) stalls_out[layer - 1] = stall;
    pysum_add(&stall_sum, stall);
  }
  free(st);
  free(next);
  free(order);
  return comp * (double)L + pysum_result(&stall_sum);
}

int64_t oracle_blocks_to_fetch(int32_t n, const int64_t* sizes, const uint8_t* offloaded, int32_t L) {
  int64_t total = 0;
  for (int r = 0; r < n; ++r)
    for (int l = 0; l < L; ++l)
      if (offloaded[(size_t)r * L + l]) total += sizes[r];
  return total;
}

int64_t oracle_prefetch_buffer(int32_t n, const int64_t* sizes, const uint8_t* offloaded, int32_t L) {
  int64_t worst = 0;
  for (int l = 0; l < L; ++l) {
    int64_t demand = 0;
    for (int r = 0; r < n; ++r)
      if (offloaded[(size_t)r * L + l]) demand += sizes[r];
    if (demand > worst) worst = demand;
  }
  return worst;
}

/* old/new: resident masks (1 = GPU).  out[0] = host->gpu blocks, out[1] = gpu->host. */
void oracle_reconfiguration_delta(int32_t n, const int64_t* sizes, const uint8_t* old_res,
                                  const uint8_t* new_res, int32_t L, int64_t* out) {
  out[0] = out[1] = 0;
  for (int r = 0; r < n; ++r)
    for (int l = 0; l < L; ++l) {
      const uint8_t a = old_res[(size_t)r * L + l], b = new_res[(size_t)r * L + l];
      if (a == 0 && b == 1) out[0] += sizes[r];
      else if (a == 1 && b == 0) out[1] += sizes[r];
    }
}
