// Host-side graph preparation for the K-truss engine (harness, not the hot path).
//
// * Synthetic generators exactly as SURVEY.md §8(d) specifies them (R-MAT with
//   Graph500 a/b/c, Fisher-Yates vertex permutation; Erdős–Rényi by uniform
//   endpoint draws), on std::mt19937_64.
// * canonicalize + build_csr restated for large inputs (parallel counting sort
//   instead of a global comparison sort) with output byte-identical to the
//   reference: canonicalize  /root/reference/proj/src/edge_list.cpp:62-103,
//   build_csr     /root/reference/proj/src/csr.cpp:10-32. Identity with the
//   reference is checked in tests/test_graph_host.py against
//   oracle/_ref/libktruss_ref.so.
// * Closed-form work statistics used for the roofline.
//
// Plain C ABI; see include/ktg_graph.h.
#include "../../include/ktg_graph.h"

#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <random>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct Csr {
  std::uint32_t n = 0;
  std::vector<std::uint32_t> row_ptr;
  std::vector<std::uint32_t> col;
  std::vector<std::uint64_t> original_ids;  // [0] unused
};

struct Raw {
  std::vector<std::uint32_t> pairs;  // 2*m labels
};

// Builds the zero-terminated CSR from relabeled, oriented (u<v) pairs in 1..n.
// Duplicates allowed on input; output rows are sorted and deduplicated, which
// is exactly canonicalize's sort+unique followed by build_csr's scatter.
int build_from_oriented(std::uint32_t n, std::vector<std::uint32_t>& us, std::vector<std::uint32_t>& vs,
                        Csr& out) {
  const std::size_t m = us.size();
  std::vector<std::uint64_t> off(static_cast<std::size_t>(n) + 2, 0);
  {
    std::vector<std::atomic<std::uint32_t>> cnt(static_cast<std::size_t>(n) + 2);
#pragma omp parallel for schedule(static)
    for (std::int64_t v = 0; v < static_cast<std::int64_t>(n) + 2; ++v) cnt[v].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i)
      cnt[us[i]].fetch_add(1, std::memory_order_relaxed);
    for (std::uint32_t v = 1; v <= n; ++v) off[v + 1] = off[v] + cnt[v].load(std::memory_order_relaxed);
  }
  std::vector<std::uint32_t> bucket(m);
  {
    std::vector<std::atomic<std::uint64_t>> cur(static_cast<std::size_t>(n) + 2);
#pragma omp parallel for schedule(static)
    for (std::int64_t v = 0; v < static_cast<std::int64_t>(n) + 2; ++v)
      cur[v].store(off[v], std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i)
      bucket[cur[us[i]].fetch_add(1, std::memory_order_relaxed)] = vs[i];
  }
  std::vector<std::uint32_t>().swap(us);
  std::vector<std::uint32_t>().swap(vs);
  // per-row sort + unique; keep the unique count
  std::vector<std::uint32_t> deg(static_cast<std::size_t>(n) + 2, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (std::int64_t v = 1; v <= static_cast<std::int64_t>(n); ++v) {
    std::uint32_t* b = bucket.data() + off[v];
    std::uint32_t* e = bucket.data() + off[v + 1];
    std::sort(b, e);
    deg[v] = static_cast<std::uint32_t>(std::unique(b, e) - b);
  }
  std::uint64_t slots = 0;
  for (std::uint32_t v = 1; v <= n; ++v) slots += deg[v] + 1ull;
  if (slots > std::numeric_limits<std::uint32_t>::max()) {
    g_err = "graph exceeds 2^32-1 CSR slots";  // csr.cpp:15-17
    return KTGG_ERR_INVALID_INPUT;
  }
  out.n = n;
  out.row_ptr.assign(static_cast<std::size_t>(n) + 2, 0);
  for (std::uint32_t v = 1; v <= n; ++v) out.row_ptr[v + 1] = out.row_ptr[v] + deg[v] + 1;
  out.col.assign(slots, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (std::int64_t v = 1; v <= static_cast<std::int64_t>(n); ++v)
    std::memcpy(out.col.data() + out.row_ptr[v], bucket.data() + off[v], deg[v] * sizeof(std::uint32_t));
  return KTGG_OK;
}

// canonicalize (edge_list.cpp:62-103) + build_csr for labels given as T.
template <typename T>
int canonical_csr(const T* raw, std::uint64_t m, Csr& out) {
  // Collect labels of non-self-loop pairs (self-loops dropped first, :63-71).
  T max_label = 0;
  std::uint64_t kept = 0;
#pragma omp parallel for reduction(max : max_label) reduction(+ : kept)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
    const T a = raw[2 * i], b = raw[2 * i + 1];
    if (a == b) continue;
    ++kept;
    max_label = std::max(max_label, std::max(a, b));
  }
  if (kept == 0) {
    g_err = "no edges survive canonicalization";
    return KTGG_ERR_EMPTY_GRAPH;
  }
  std::vector<std::uint32_t> us(kept), vs(kept);
  std::uint32_t n = 0;
  const bool dense = static_cast<std::uint64_t>(max_label) < (std::uint64_t{1} << 32) - 1 &&
                     static_cast<std::uint64_t>(max_label) <= 64 * kept + 1024;
  // Compact the kept pairs in order (prefix over per-thread counts).
  std::vector<std::uint64_t> pos(m + 1, 0);
  {
    const int nt = omp_get_max_threads();
    std::vector<std::uint64_t> part(static_cast<std::size_t>(nt) + 1, 0);
#pragma omp parallel num_threads(nt)
    {
      const int t = omp_get_thread_num();
      const std::uint64_t lo = m * t / nt, hi = m * (t + 1) / nt;
      std::uint64_t c = 0;
      for (std::uint64_t i = lo; i < hi; ++i) c += raw[2 * i] != raw[2 * i + 1];
      part[t + 1] = c;
#pragma omp barrier
#pragma omp single
      for (int q = 1; q <= nt; ++q) part[q] += part[q - 1];
      c = part[t];
      for (std::uint64_t i = lo; i < hi; ++i) {
        pos[i] = c;
        c += raw[2 * i] != raw[2 * i + 1];
      }
    }
  }
  if (dense) {
    // Rank = 1 + number of present labels below; equals lower_bound+1 (:81-84).
    const std::size_t N = static_cast<std::size_t>(max_label) + 1;
    std::vector<std::uint32_t> rank(N, 0);
#pragma omp parallel for
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
      const T a = raw[2 * i], b = raw[2 * i + 1];
      if (a == b) continue;
      rank[a] = 1;  // benign race: every writer stores 1
      rank[b] = 1;
    }
    std::uint32_t c = 0;
    out.original_ids.assign(1, 0);
    for (std::size_t x = 0; x < N; ++x) {
      if (rank[x]) {
        rank[x] = ++c;
        out.original_ids.push_back(x);
      }
    }
    n = c;
#pragma omp parallel for
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
      const T a = raw[2 * i], b = raw[2 * i + 1];
      if (a == b) continue;
      const std::uint32_t u = rank[a], v = rank[b];
      us[pos[i]] = std::min(u, v);
      vs[pos[i]] = std::max(u, v);
    }
  } else {
    std::vector<T> labels;
    labels.reserve(2 * kept);
    for (std::uint64_t i = 0; i < m; ++i) {
      if (raw[2 * i] == raw[2 * i + 1]) continue;
      labels.push_back(raw[2 * i]);
      labels.push_back(raw[2 * i + 1]);
    }
    std::sort(labels.begin(), labels.end());
    labels.erase(std::unique(labels.begin(), labels.end()), labels.end());
    if (labels.size() > std::numeric_limits<std::uint32_t>::max() - 1ull) {
      g_err = "vertex count exceeds 32-bit id space";
      return KTGG_ERR_INVALID_INPUT;
    }
    n = static_cast<std::uint32_t>(labels.size());
    out.original_ids.assign(1, 0);
    out.original_ids.insert(out.original_ids.end(), labels.begin(), labels.end());
    auto relabel = [&](T x) {
      return static_cast<std::uint32_t>(std::lower_bound(labels.begin(), labels.end(), x) - labels.begin()) + 1;
    };
#pragma omp parallel for
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
      const T a = raw[2 * i], b = raw[2 * i + 1];
      if (a == b) continue;
      const std::uint32_t u = relabel(a), v = relabel(b);
      us[pos[i]] = std::min(u, v);
      vs[pos[i]] = std::max(u, v);
    }
  }
  std::vector<std::uint64_t>().swap(pos);
  return build_from_oriented(n, us, vs, out);
}

inline double unit53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

// validate_csr (csr.cpp:34-80), same checks in the same order, same messages.
// Returns an empty string when valid.
std::string validate(std::uint32_t n, const std::uint32_t* rp, std::uint64_t rp_len, const std::uint32_t* col,
                     std::uint64_t slots) {
  if (n == 0) return "csr has no vertices";
  if (rp_len != n + 2ull) return "row_ptr must have num_vertices + 2 entries";
  if (rp[0] != 0 || rp[1] != 0) return "phantom vertex 0 must own no slots";
  if (slots > 0xFFFFFFFFull) return "slot count exceeds 32-bit offsets";
  if (rp[n + 1] != slots) return "row_ptr end does not match slot count";
  for (std::uint32_t v = 1; v <= n; ++v) {
    const std::uint32_t b = rp[v], e = rp[v + 1];
    if (b >= e) return "row " + std::to_string(v) + " owns no sentinel slot";
    if (col[e - 1] != 0) return "row " + std::to_string(v) + " does not end in a zero slot";
    std::uint32_t prev = v;
    bool zero_tail = false;
    for (std::uint32_t s = b; s < e; ++s) {
      const std::uint32_t w = col[s];
      if (w == 0) {
        zero_tail = true;
        continue;
      }
      if (zero_tail) return "row " + std::to_string(v) + " has a nonzero after a zero slot";
      if (w <= prev) return "row " + std::to_string(v) + " entries are not strictly ascending above the vertex";
      if (w > n) return "row " + std::to_string(v) + " references vertex beyond n";
      prev = w;
    }
  }
  return "";
}

constexpr char kMagic[8] = {'Z', 'T', 'C', 'S', 'R', '1', '\0', '\0'};

}  // namespace

extern "C" {

const char* ktgg_last_error(void) { return g_err.c_str(); }

int ktgg_rmat_raw(std::uint32_t scale, std::uint32_t edgefactor, std::uint64_t seed, double a, double b,
                  double c, ktgg_raw** out) {
  if (scale == 0 || scale > 31 || edgefactor == 0) {
    g_err = "rmat: scale must be in 1..31 and edgefactor >= 1";
    return KTGG_ERR_INVALID_PARAMETER;
  }
  try {
    const std::uint64_t N = std::uint64_t{1} << scale;
    const std::uint64_t m = N * edgefactor;
    auto* r = new Raw;
    r->pairs.resize(2 * m);
    const double ab = a + b, abc = a + b + c;
    std::mt19937_64 g(seed);
    std::uint32_t* p = r->pairs.data();
    for (std::uint64_t e = 0; e < m; ++e) {
      std::uint32_t u = 0, v = 0;
      for (std::uint32_t level = 0; level < scale; ++level) {
        const double x = unit53(g);
        std::uint32_t bu, bv;
        if (x < a) {
          bu = 0; bv = 0;
        } else if (x < ab) {
          bu = 0; bv = 1;
        } else if (x < abc) {
          bu = 1; bv = 0;
        } else {
          bu = 1; bv = 1;
        }
        u = (u << 1) | bu;
        v = (v << 1) | bv;
      }
      p[2 * e] = u;
      p[2 * e + 1] = v;
    }
    // Graph500-style relabel by an explicit Fisher-Yates permutation.
    std::vector<std::uint32_t> perm(N);
    for (std::uint64_t i = 0; i < N; ++i) perm[i] = static_cast<std::uint32_t>(i);
    std::mt19937_64 g2(seed ^ 0xABCDEFull);
    for (std::uint64_t i = N - 1; i >= 1; --i) {
      const std::uint64_t j = g2() % (i + 1);
      std::swap(perm[i], perm[j]);
    }
#pragma omp parallel for
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(2 * m); ++i) p[i] = perm[p[i]];
    *out = reinterpret_cast<ktgg_raw*>(r);
    return KTGG_OK;
  } catch (const std::bad_alloc&) {
    g_err = "rmat: out of host memory";
    return KTGG_ERR_OOM;
  }
}

int ktgg_er_raw(std::uint32_t log_n, std::uint64_t m, std::uint64_t seed, ktgg_raw** out) {
  if (log_n == 0 || log_n > 31) {
    g_err = "er: log_n must be in 1..31";
    return KTGG_ERR_INVALID_PARAMETER;
  }
  try {
    const std::uint64_t N = std::uint64_t{1} << log_n;
    auto* r = new Raw;
    r->pairs.resize(2 * m);
    std::mt19937_64 g(seed);
    for (std::uint64_t e = 0; e < 2 * m; ++e) r->pairs[e] = static_cast<std::uint32_t>(g() % N);
    *out = reinterpret_cast<ktgg_raw*>(r);
    return KTGG_OK;
  } catch (const std::bad_alloc&) {
    g_err = "er: out of host memory";
    return KTGG_ERR_OOM;
  }
}

std::uint64_t ktgg_raw_count(const ktgg_raw* r) { return reinterpret_cast<const Raw*>(r)->pairs.size() / 2; }
const std::uint32_t* ktgg_raw_pairs(const ktgg_raw* r) { return reinterpret_cast<const Raw*>(r)->pairs.data(); }
void ktgg_raw_free(ktgg_raw* r) { delete reinterpret_cast<Raw*>(r); }

int ktgg_csr_from_raw(const ktgg_raw* r, ktgg_csr** out) {
  const Raw* raw = reinterpret_cast<const Raw*>(r);
  return ktgg_csr_from_pairs_u32(raw->pairs.data(), raw->pairs.size() / 2, out);
}

int ktgg_csr_from_pairs_u32(const std::uint32_t* pairs, std::uint64_t m, ktgg_csr** out) {
  try {
    auto* c = new Csr;
    const int rc = canonical_csr<std::uint32_t>(pairs, m, *c);
    if (rc != KTGG_OK) {
      delete c;
      return rc;
    }
    *out = reinterpret_cast<ktgg_csr*>(c);
    return KTGG_OK;
  } catch (const std::bad_alloc&) {
    g_err = "canonicalize: out of host memory";
    return KTGG_ERR_OOM;
  }
}

int ktgg_csr_from_pairs_u64(const std::uint64_t* pairs, std::uint64_t m, ktgg_csr** out) {
  try {
    auto* c = new Csr;
    const int rc = canonical_csr<std::uint64_t>(pairs, m, *c);
    if (rc != KTGG_OK) {
      delete c;
      return rc;
    }
    *out = reinterpret_cast<ktgg_csr*>(c);
    return KTGG_OK;
  } catch (const std::bad_alloc&) {
    g_err = "canonicalize: out of host memory";
    return KTGG_ERR_OOM;
  }
}

std::uint32_t ktgg_csr_n(const ktgg_csr* c) { return reinterpret_cast<const Csr*>(c)->n; }
std::uint64_t ktgg_csr_slots(const ktgg_csr* c) { return reinterpret_cast<const Csr*>(c)->col.size(); }
void ktgg_csr_copy(const ktgg_csr* c, std::uint32_t* row_ptr, std::uint32_t* col, std::uint64_t* original_ids) {
  const Csr* g = reinterpret_cast<const Csr*>(c);
  if (row_ptr) std::memcpy(row_ptr, g->row_ptr.data(), g->row_ptr.size() * 4);
  if (col) std::memcpy(col, g->col.data(), g->col.size() * 4);
  if (original_ids) std::memcpy(original_ids, g->original_ids.data(), g->original_ids.size() * 8);
}
void ktgg_csr_free(ktgg_csr* c) { delete reinterpret_cast<Csr*>(c); }

// ZTCSR1 cache (csr_cache.hpp:11-21, csr_cache.cpp:71-111): little-endian
// magic | u32 n | u64 slots | row_ptr (n+2) x u32 | col_idx slots x u32.
int ktgg_write_csr_cache(const char* path, const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                         std::uint64_t slots) {
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_err = "cache write failed";
    return KTGG_ERR_IO;
  }
  bool ok = std::fwrite(kMagic, 1, 8, f) == 8;
  ok = ok && std::fwrite(&n, 4, 1, f) == 1;  // x86/ARM hosts are little-endian
  ok = ok && std::fwrite(&slots, 8, 1, f) == 1;
  ok = ok && std::fwrite(row_ptr, 4, n + std::size_t{2}, f) == n + std::size_t{2};
  ok = ok && std::fwrite(col, 4, slots, f) == slots;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    g_err = "cache write failed";
    return KTGG_ERR_IO;
  }
  return KTGG_OK;
}

int ktgg_read_csr_cache(const char* path, ktgg_csr** out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    g_err = std::string("cannot open ") + path;
    return KTGG_ERR_IO;
  }
  auto corrupt = [&](const std::string& m) {
    std::fclose(f);
    g_err = m;
    return KTGG_ERR_CORRUPT_CACHE;
  };
  char magic[8];
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0) return corrupt("bad cache magic");
  std::uint32_t n = 0;
  std::uint64_t slots = 0;
  if (std::fread(&n, 4, 1, f) != 1 || std::fread(&slots, 8, 1, f) != 1) return corrupt("truncated cache header");
  if (n == 0 || slots < n || slots > 0xFFFFFFFFull) return corrupt("implausible cache dimensions");
  Csr* c = nullptr;
  try {
    c = new Csr;
    c->n = n;
    c->row_ptr.resize(n + std::size_t{2});
    if (std::fread(c->row_ptr.data(), 4, c->row_ptr.size(), f) != c->row_ptr.size()) {
      delete c;
      return corrupt("truncated cache payload");
    }
    if (c->row_ptr[n + 1] != slots) {
      delete c;
      return corrupt("row_ptr end does not match slot count");
    }
    c->col.resize(slots);
    if (std::fread(c->col.data(), 4, slots, f) != slots) {
      delete c;
      return corrupt("truncated cache payload");
    }
    if (std::fgetc(f) != EOF) {
      delete c;
      return corrupt("trailing bytes after cache payload");
    }
  } catch (const std::bad_alloc&) {
    delete c;
    std::fclose(f);
    g_err = "cache read: out of host memory";
    return KTGG_ERR_OOM;
  }
  std::fclose(f);
  const std::string bad = validate(n, c->row_ptr.data(), c->row_ptr.size(), c->col.data(), slots);
  if (!bad.empty()) {
    delete c;
    g_err = "cache violates csr invariants: " + bad;
    return KTGG_ERR_CORRUPT_CACHE;
  }
  c->original_ids.assign(n + std::size_t{1}, 0);
  for (std::uint32_t v = 1; v <= n; ++v) c->original_ids[v] = v;
  *out = reinterpret_cast<ktgg_csr*>(c);
  return KTGG_OK;
}

// validate_csr restated; 0 if valid, else KTGG_ERR_INVALID_INPUT + message.
int ktgg_validate_csr(const std::uint32_t* row_ptr, std::uint64_t rp_len, std::uint32_t n, const std::uint32_t* col,
                      std::uint64_t slots) {
  const std::string bad = validate(n, row_ptr, rp_len, col, slots);
  if (bad.empty()) return KTGG_OK;
  g_err = bad;
  return KTGG_ERR_INVALID_INPUT;
}

// Closed-form merge work of one compute_supports pass over the live graph
// (SURVEY.md §8(d)): L = sum_v d+(d+-1)/2 + d+ d-. Split into its two terms.
void ktgg_round_work(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                     ktgg_work* w) {
  std::vector<std::uint32_t> dout(static_cast<std::size_t>(n) + 2, 0);
  std::vector<std::atomic<std::uint32_t>> din(static_cast<std::size_t>(n) + 2);
#pragma omp parallel for
  for (std::int64_t v = 0; v < static_cast<std::int64_t>(n) + 2; ++v) din[v].store(0, std::memory_order_relaxed);
  std::uint64_t live = 0;
  std::uint32_t maxd = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : live) reduction(max : maxd)
  for (std::int64_t v = 1; v <= static_cast<std::int64_t>(n); ++v) {
    std::uint32_t d = 0;
    for (std::uint32_t s = row_ptr[v]; col[s] != 0; ++s, ++d) din[col[s]].fetch_add(1, std::memory_order_relaxed);
    dout[v] = d;
    live += d;
    maxd = std::max(maxd, d);
  }
  std::uint64_t tail = 0, cross = 0, sq = 0;
#pragma omp parallel for reduction(+ : tail, cross, sq)
  for (std::int64_t v = 1; v <= static_cast<std::int64_t>(n); ++v) {
    const std::uint64_t d = dout[v];
    tail += d * (d ? d - 1 : 0) / 2;
    cross += d * din[v].load(std::memory_order_relaxed);
    sq += d * d;
  }
  w->live_edges = live;
  w->max_out_degree = maxd;
  w->tail_elements = tail;
  w->cross_elements = cross;
  w->L = tail + cross;
  w->sum_dout_sq = sq;
}

}  // extern "C"
