/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the Eager K-truss hot path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj),
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the CHECKER. It is never linked or loaded by the product library
 * (paper_2009_07929_b200/), which fails loudly without its CUDA extension.
 *
 * Parity of this restatement is pinned in tests/test_oracle.py against
 *   (1) the reference's own known-answer vectors (test_support.cpp,
 *       test_truss.cpp, test_graph_io.cpp; committed as tests/golden/kat.json), and
 *   (2) the unmodified reference library compiled from its sources into
 *       oracle/_ref/libktruss_ref.so (oracle/Makefile), on the seeded corpus.
 *
 * Each function cites the reference lines it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- support (support.cpp) ------------------------------------------------ */

/* intersect_tails, support.cpp:64-91: two-pointer merge of the pivot row tail
 * col[pivot+1..] and the predecessor's row col[row_ptr[pred]..]; both stop at
 * the first zero. Each match bumps both matching slots. */
uint32_t orc_intersect_tails(const uint32_t* row_ptr, const uint32_t* col, uint32_t pivot_slot,
                             uint32_t predecessor, uint32_t* S) {
  uint32_t a = pivot_slot + 1;
  uint32_t b = row_ptr[predecessor];
  uint32_t found = 0;
  while (col[a] != 0 && col[b] != 0) {
    if (col[a] == col[b]) {
#pragma omp atomic
      S[a] += 1;
#pragma omp atomic
      S[b] += 1;
      ++found;
      ++a;
      ++b;
    } else if (col[b] > col[a]) {
      ++a;
    } else {
      ++b;
    }
  }
  return found;
}

/* compute_supports, Fine branch, support.cpp:115-127: one task per slot,
 * sentinel / pruned slots skipped, pivot add of the local count. S must be
 * zero on entry (support.hpp:48-51). Returns the triangle total. */
uint64_t orc_compute_supports(const uint32_t* row_ptr, uint32_t n, const uint32_t* col,
                              uint64_t slots, uint32_t* S, int threads) {
  (void)n;
  uint64_t triangles = 0;
  const int64_t count = (int64_t)slots;
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads) reduction(+ : triangles)
  for (int64_t slot = 0; slot < count; ++slot) {
    const uint32_t pred = col[slot];
    if (pred != 0) {
      const uint32_t found = orc_intersect_tails(row_ptr, col, (uint32_t)slot, pred, S);
      if (found != 0) {
#pragma omp atomic
        S[slot] += found;
      }
      triangles += found;
    }
  }
  return triangles;
}

/* check_16bit, support.cpp:53-60: first slot whose count exceeds 65535, or
 * UINT64_MAX if none. */
uint64_t orc_first_overflow_16(const uint32_t* S, uint64_t slots) {
  for (uint64_t s = 0; s < slots; ++s)
    if (S[s] > 0xFFFFu) return s;
  return UINT64_MAX;
}

/* ---- prune + fixpoint (truss.cpp) ----------------------------------------- */

/* prune_edges, truss.cpp:9-37: per-row stable compaction of the slots whose
 * support is >= k-2, zero-filling the vacated tail. Returns removed count. */
uint64_t orc_prune_edges(const uint32_t* row_ptr, uint32_t n, uint32_t* col, const uint32_t* S,
                         uint32_t k, int threads) {
  const uint32_t threshold = k - 2;
  uint64_t removed = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads) reduction(+ : removed)
  for (int64_t v = 1; v <= (int64_t)n; ++v) {
    uint32_t read = row_ptr[v];
    uint32_t write = read;
    for (; col[read] != 0; ++read)
      if (S[read] >= threshold) col[write++] = col[read];
    removed += read - write;
    for (; write < read; ++write) col[write] = 0;
  }
  return removed;
}

/* detail::run_fixpoint, truss.cpp:41-53: {reset; compute; prune} until a
 * round removes nothing. Returns the iteration count; hist gets up to cap
 * removal counts. */
uint32_t orc_run_fixpoint(const uint32_t* row_ptr, uint32_t n, uint32_t* col, uint64_t slots,
                          uint32_t* S, uint32_t k, int threads, uint64_t* hist, uint32_t cap) {
  uint32_t it = 0;
  for (;;) {
    memset(S, 0, slots * sizeof(uint32_t)); /* reset_supports, support.cpp:134-136 */
    orc_compute_supports(row_ptr, n, col, slots, S, threads);
    const uint64_t removed = orc_prune_edges(row_ptr, n, col, S, k, threads);
    if (it < cap) hist[it] = removed;
    ++it;
    if (removed == 0) break;
  }
  return it;
}

uint64_t orc_count_live(const uint32_t* row_ptr, uint32_t n, const uint32_t* col) {
  /* count_live_edges, csr.cpp:108-114 */
  uint64_t live = 0;
  for (uint32_t v = 1; v <= n; ++v)
    for (uint32_t s = row_ptr[v]; col[s] != 0; ++s) ++live;
  return live;
}

/* kmax_search, truss.cpp:73-103: one support pass bounds k by max(S)+2, then
 * binary search over [3, bound], every probe from the pristine graph.
 * Returns k_max (0 if the graph has no live edge -- the reference throws). */
uint32_t orc_kmax(const uint32_t* row_ptr, uint32_t n, const uint32_t* col, uint64_t slots,
                  int threads) {
  if (orc_count_live(row_ptr, n, col) == 0) return 0;
  uint32_t* S = (uint32_t*)calloc(slots, sizeof(uint32_t));
  uint32_t* work = (uint32_t*)malloc(slots * sizeof(uint32_t));
  uint64_t hist[1];
  orc_compute_supports(row_ptr, n, col, slots, S, threads);
  uint32_t max_support = 0;
  for (uint64_t s = 0; s < slots; ++s)
    if (S[s] > max_support) max_support = S[s];
  uint32_t lo = 2;
  if (max_support > 0) {
    lo = 3;
    uint32_t hi = max_support + 2;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo + 1) / 2;
      memcpy(work, col, slots * sizeof(uint32_t));
      orc_run_fixpoint(row_ptr, n, work, slots, S, mid, threads, hist, 0);
      if (orc_count_live(row_ptr, n, work) == 0)
        hi = mid - 1;
      else
        lo = mid;
    }
  }
  free(S);
  free(work);
  return lo;
}

/* ---- closed-form work of one support round ----------------- */

/* L = sum_v [ d+(v)(d+(v)-1)/2 + d+(v) d-(v) ] over live degrees: the list
 * elements a full two-pointer merge touches in one compute_supports pass.
 * Also returns the live edge count and the max live out-degree. */
void orc_round_work(const uint32_t* row_ptr, uint32_t n, const uint32_t* col, uint64_t* L_out,
                    uint64_t* live_out, uint32_t* max_out_deg) {
  uint32_t* din = (uint32_t*)calloc((size_t)n + 2, sizeof(uint32_t));
  uint64_t live = 0;
  uint32_t maxd = 0;
  for (uint32_t v = 1; v <= n; ++v) {
    uint32_t d = 0;
    for (uint32_t s = row_ptr[v]; col[s] != 0; ++s) {
      ++din[col[s]];
      ++d;
    }
    live += d;
    if (d > maxd) maxd = d;
  }
  uint64_t L = 0;
  for (uint32_t v = 1; v <= n; ++v) {
    uint64_t d = 0;
    for (uint32_t s = row_ptr[v]; col[s] != 0; ++s) ++d;
    L += d * (d ? d - 1 : 0) / 2 + d * (uint64_t)din[v];
  }
  free(din);
  *L_out = L;
  *live_out = live;
  *max_out_deg = maxd;
}

/* ---- brute-force oracle (oracle.cpp) -------------------------------------- */

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* edge_supports, oracle.cpp:44-56: support(u,v) = |N(u) ∩ N(v)| over full
 * symmetric sorted adjacency sets. edges are m (u,v) pairs, u<v. */
void orc_brute_supports(uint32_t n, const uint32_t* edges, uint64_t m, uint32_t* out) {
  uint64_t* deg = (uint64_t*)calloc((size_t)n + 2, sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    ++deg[edges[2 * i] + 1];
    ++deg[edges[2 * i + 1] + 1];
  }
  for (uint32_t v = 1; v <= n + 1; ++v) deg[v] += deg[v - 1];
  uint32_t* adj = (uint32_t*)malloc((2 * m + 1) * sizeof(uint32_t));
  uint64_t* cur = (uint64_t*)malloc(((size_t)n + 2) * sizeof(uint64_t));
  memcpy(cur, deg, ((size_t)n + 2) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = edges[2 * i], v = edges[2 * i + 1];
    adj[cur[u]++] = v;
    adj[cur[v]++] = u;
  }
  for (uint32_t v = 0; v <= n; ++v) qsort(adj + deg[v], deg[v + 1] - deg[v], 4, cmp_u32);
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = edges[2 * i], v = edges[2 * i + 1];
    uint64_t a = deg[u], ae = deg[u + 1], b = deg[v], be = deg[v + 1];
    uint32_t c = 0;
    while (a < ae && b < be) {
      if (adj[a] == adj[b]) {
        ++c;
        ++a;
        ++b;
      } else if (adj[a] < adj[b]) {
        ++a;
      } else {
        ++b;
      }
    }
    out[i] = c;
  }
  free(deg);
  free(adj);
  free(cur);
}

/* ---- mt19937_64 + seeded G(n,p) (oracle.cpp:89-109) ----------------------- */

typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* The raw pairs random_graph feeds to canonicalize (oracle.cpp:95-103):
 * first attempt with at least one edge. Returns the pair count written to
 * out (capacity n(n-1)/2 pairs), or 0 if every attempt drew nothing. */
uint64_t orc_random_graph_raw(uint32_t n, double p, uint64_t seed, uint64_t* out) {
  for (uint64_t attempt = 0; attempt < 64; ++attempt) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed + attempt * 0x9E3779B97F4A7C15ULL);
    uint64_t m = 0;
    for (uint32_t u = 1; u <= n; ++u)
      for (uint32_t v = u + 1; v <= n; ++v) {
        const double unit = (double)(orc_mt64_next(&g) >> 11) * 0x1.0p-53;
        if (unit < p) {
          out[2 * m] = u;
          out[2 * m + 1] = v;
          ++m;
        }
      }
    if (m) return m;
  }
  return 0;
}

/* ---- multi-GPU task partition (mirror of the device planner) -------------- */

/* The engine's support tasks (paper_2009_07929_b200/csrc/ktg_kernels.cuh,
 * k_plan_count / k_plan_write / k_support_chunked): the slot space is cut
 * into `chunk`-slot chunks; off-diagonal tasks (q, q') for the last row of
 * chunk q whose live part reaches chunk q' > q come first (q ascending, then
 * q'), then the diagonal tasks (q, q). Off-diagonal task t belongs to rank
 * t % world; diagonal tasks are split into work-balanced contiguous chunk
 * ranges (orc_task_cost below). A task processes the pivots of chunk q against the part of their a12 tails
 * lying in chunk q'. Diagonal tasks run from the last chunk to the first
 * (densest rows of the degree order first). This restatement computes one
 * rank's partial supports
 * with the reference's merge (support.cpp:64-91) restricted to that tail
 * part. Returns the partial triangle count. S must be zero on entry. */
static uint32_t row_of_slot(const uint32_t* row_ptr, uint32_t n, uint64_t s) {
  uint32_t lo = 0, hi = n + 2;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= s) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

static uint64_t merge_range(const uint32_t* row_ptr, const uint32_t* col, uint64_t pivot, uint64_t t_lo,
                            uint64_t t_hi, uint32_t* S) {
  /* tail slots [t_lo, t_hi) of the pivot's row (stops at a zero) vs row col[pivot] */
  uint64_t a = t_lo, b = row_ptr[col[pivot]];
  uint32_t found = 0;
  while (a < t_hi && col[a] != 0 && col[b] != 0) {
    if (col[a] == col[b]) {
      ++S[a];
      ++S[b];
      ++found;
      ++a;
      ++b;
    } else if (col[b] > col[a]) {
      ++a;
    } else {
      ++b;
    }
  }
  S[pivot] += found;
  return found;
}

/* Work estimate of diagonal task q (the multi-GPU split, mirror of the
 * engine's k_task_cost): over the chunk's live pivots s, the tail inside the
 * chunk + 1 + the live out-degree of col[s]. A chunk goes to rank
 * min(world-1, prefix(q) * world / total): contiguous, work-balanced ranges
 * (SURVEY.md §8(e)). */
uint64_t orc_task_cost(const uint32_t* row_ptr, uint32_t n, const uint32_t* col, uint64_t slots, uint32_t chunk,
                       uint64_t q) {
  (void)n;
  const uint64_t p0 = q * chunk, p1 = (q + 1) * chunk < slots ? (q + 1) * chunk : slots;
  uint64_t c = 0, z = p1; /* next zero inside the chunk, scanning backwards */
  for (uint64_t s = p1; s-- > p0;) {
    if (col[s] == 0) {
      z = s;
      continue;
    }
    uint64_t d = 0;
    const uint32_t v = col[s];
    while (col[row_ptr[v] + d] != 0) ++d; /* live out-degree of v */
    c += (z - s - 1) + 1 + d;
  }
  return c;
}

uint64_t orc_support_tasks(const uint32_t* row_ptr, uint32_t n, const uint32_t* col, uint64_t slots,
                           uint32_t chunk, uint32_t rank, uint32_t world, uint32_t* S) {
  const uint64_t Q = (slots + chunk - 1) / chunk;
  uint64_t t = 0, tri = 0;
  /* off-diagonal tasks */
  for (uint64_t q = 0; q < Q; ++q) {
    const uint64_t e = ((q + 1) * chunk < slots ? (q + 1) * chunk : slots);
    const uint32_t i = row_of_slot(row_ptr, n, e - 1);
    if (i < 1) continue;
    uint64_t le = row_ptr[i];
    while (col[le] != 0) ++le; /* live end */
    if (le <= e) continue;
    const uint64_t last = (le - 1) / chunk;
    for (uint64_t q2 = q + 1; q2 <= last; ++q2, ++t) {
      if (t % world != rank) continue;
      const uint64_t p_lo = row_ptr[i] > q * chunk ? row_ptr[i] : q * chunk;
      const uint64_t a0 = q2 * chunk, a1 = (q2 + 1) * chunk < slots ? (q2 + 1) * chunk : slots;
      for (uint64_t s = p_lo; s < e; ++s) tri += merge_range(row_ptr, col, s, a0, a1, S);
    }
  }
  /* diagonal tasks: this rank's work-balanced range (orc_task_cost) */
  uint64_t* pre = (uint64_t*)malloc((Q + 1) * sizeof(uint64_t));
  if (!pre) return 0;
  pre[0] = 0;
  for (uint64_t q = 0; q < Q; ++q) pre[q + 1] = pre[q] + orc_task_cost(row_ptr, n, col, slots, chunk, q);
  const uint64_t T = pre[Q];
  for (uint64_t q = 0; q < Q; ++q) {
    uint64_t owner = 0;
    if (T) {
      owner = pre[q] * world / T;
      if (owner > world - 1) owner = world - 1;
    }
    if (owner != rank) continue;
    const uint64_t p0 = q * chunk, p1 = (q + 1) * chunk < slots ? (q + 1) * chunk : slots;
    for (uint64_t s = p0; s < p1; ++s)
      if (col[s] != 0) tri += merge_range(row_ptr, col, s, s + 1, p1, S);
  }
  free(pre);
  return tri;
}
