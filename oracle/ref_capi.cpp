// TEST INFRASTRUCTURE ONLY -- a C shim over the UNMODIFIED reference library
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libktruss_ref.so). It lets the Python tests and bench.py's
// reference/cpu_baseline legs call the reference's own code through ctypes.
// Nothing on the product path links or loads this file.
//
// Every entry point wraps one reference function:
//   ref_compute_supports -> ktruss::compute_supports  (support.hpp:52-54)
//   ref_prune_edges      -> ktruss::prune_edges       (truss.hpp:38-39)
//   ref_run_fixpoint     -> ktruss::detail::run_fixpoint (truss.hpp:62-63)
//   ref_ktruss           -> ktruss::ktruss            (truss.hpp:44-45)
//   ref_kmax_search      -> ktruss::kmax_search       (truss.hpp:56)
//   ref_canonicalize_csr -> ktruss::canonicalize + build_csr (edge_list.hpp:53, csr.hpp:27)
//   ref_random_graph_csr -> ktruss::oracle::random_graph + build_csr (oracle.hpp:38)
//   ref_oracle_*         -> ktruss::oracle::{edge_supports,ktruss_edges,kmax,triangle_count}
//   ref_rmat_csr / ref_er_csr -> the SURVEY §8(d) synthetic generators (restated
//                           here, independent of the product's graph_host.cpp),
//                           then either the reference canonicalize + build_csr
//                           (fast=0) or a parallel restatement of canonicalize
//                           feeding the reference build_csr (fast=1; pinned
//                           byte-equal to fast=0 by tests/test_oracle.py and the
//                           s20/s24 digests in tests/golden/large_ref.json).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <fstream>
#include <parallel/algorithm>
#include <random>
#include <sstream>

#include "ktruss/bench.hpp"
#include "ktruss/csr_cache.hpp"
#include "ktruss/csr.hpp"
#include "ktruss/edge_list.hpp"
#include "ktruss/errors.hpp"
#include "ktruss/oracle.hpp"
#include "ktruss/support.hpp"
#include "ktruss/truss.hpp"

using namespace ktruss;

namespace {

thread_local std::string g_err;
thread_local std::uint64_t g_err_slot = 0;

// 0 ok, 1 InvalidParameterError, 2 SupportOverflowError, 3 InvalidInputError,
// 4 EmptyGraphError, 5 other ktruss::Error, 6 other std::exception
int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const InvalidParameterError*>(&e)) return 1;
  if (auto* o = dynamic_cast<const SupportOverflowError*>(&e)) {
    g_err_slot = o->slot;
    return 2;
  }
  if (dynamic_cast<const InvalidInputError*>(&e)) return 3;
  if (dynamic_cast<const EmptyGraphError*>(&e)) return 4;
  if (dynamic_cast<const Error*>(&e)) return 5;
  return 6;
}

ZeroTerminatedCsr make_csr(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                           std::uint64_t slots) {
  ZeroTerminatedCsr g;
  g.num_vertices = n;
  g.row_ptr.assign(row_ptr, row_ptr + (n + std::size_t{2}));
  g.col_idx.assign(col, col + slots);
  return g;
}

Strategy strat(int s) { return s == 0 ? Strategy::Serial : s == 1 ? Strategy::Coarse : Strategy::Fine; }

struct CsrOut {
  ZeroTerminatedCsr csr;
};

void fill_edges(const std::vector<SupportedEdge>& edges, std::uint32_t* u, std::uint32_t* v,
                std::uint32_t* s) {
  for (std::size_t i = 0; i < edges.size(); ++i) {
    u[i] = edges[i].u;
    v[i] = edges[i].v;
    s[i] = edges[i].support;
  }
}

struct TrussOut {
  TrussResult result;
  std::uint32_t k_max = 0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
std::uint64_t ref_last_error_slot() { return g_err_slot; }

int ref_compute_supports(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                         std::uint64_t slots, std::uint32_t* supports, std::uint64_t s_len,
                         int strategy, int threads, int width16, std::uint64_t* triangles) {
  try {
    const ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
    SupportArray s;
    s.counts.assign(supports, supports + s_len);
    *triangles = compute_supports(g, s, strat(strategy), threads,
                                  width16 ? SupportWidth::Bits16 : SupportWidth::Bits32);
    std::memcpy(supports, s.counts.data(), s_len * 4);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_prune_edges(const std::uint32_t* row_ptr, std::uint32_t n, std::uint32_t* col,
                    std::uint64_t slots, const std::uint32_t* supports, std::uint64_t s_len,
                    std::uint32_t k, int threads, std::uint64_t* removed) {
  try {
    ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
    SupportArray s;
    s.counts.assign(supports, supports + s_len);
    *removed = prune_edges(g, s, k, threads);
    std::memcpy(col, g.col_idx.data(), slots * 4);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Runs detail::run_fixpoint on (col, supports) in place. *elapsed_ms brackets
// the run_fixpoint call only, exactly like run_bench (bench.cpp:33-40).
int ref_run_fixpoint(const std::uint32_t* row_ptr, std::uint32_t n, std::uint32_t* col,
                     std::uint64_t slots, std::uint32_t* supports, std::uint32_t k, int strategy,
                     int threads, int width16, std::uint64_t* hist, std::uint32_t hist_cap,
                     std::uint32_t* iterations, double* elapsed_ms) {
  try {
    ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
    SupportArray s;
    s.counts.assign(supports, supports + slots);
    TrussOptions opt;
    opt.strategy = strat(strategy);
    opt.threads = threads;
    opt.width = width16 ? SupportWidth::Bits16 : SupportWidth::Bits32;
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<std::uint64_t> h = detail::run_fixpoint(g, s, k, opt);
    const auto t1 = std::chrono::steady_clock::now();
    if (elapsed_ms) *elapsed_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    *iterations = static_cast<std::uint32_t>(h.size());
    for (std::size_t i = 0; i < h.size() && i < hist_cap; ++i) hist[i] = h[i];
    std::memcpy(col, g.col_idx.data(), slots * 4);
    std::memcpy(supports, s.counts.data(), slots * 4);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// ktruss / kmax_search return an opaque TrussOut; read it with ref_truss_*.
int ref_ktruss(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
               std::uint64_t slots, std::uint32_t k, int strategy, int threads, void** out) {
  try {
    const ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
    auto* t = new TrussOut;
    TrussOptions opt;
    opt.strategy = strat(strategy);
    opt.threads = threads;
    t->result = ktruss::ktruss(g, k, opt);
    *out = t;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_kmax_search(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                    std::uint64_t slots, int strategy, int threads, void** out) {
  try {
    const ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
    auto* t = new TrussOut;
    TrussOptions opt;
    opt.strategy = strat(strategy);
    opt.threads = threads;
    KmaxResult r = kmax_search(g, opt);
    t->k_max = r.k_max;
    t->result = std::move(r.truss);
    *out = t;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

std::uint32_t ref_truss_kmax(void* h) { return static_cast<TrussOut*>(h)->k_max; }
std::uint32_t ref_truss_k(void* h) { return static_cast<TrussOut*>(h)->result.k; }
std::uint64_t ref_truss_num_edges(void* h) { return static_cast<TrussOut*>(h)->result.edges.size(); }
std::uint32_t ref_truss_iterations(void* h) { return static_cast<TrussOut*>(h)->result.iterations; }
void ref_truss_removed(void* h, std::uint64_t* out) {
  const auto& r = static_cast<TrussOut*>(h)->result.removed_per_iteration;
  for (std::size_t i = 0; i < r.size(); ++i) out[i] = r[i];
}
void ref_truss_edges(void* h, std::uint32_t* u, std::uint32_t* v, std::uint32_t* s) {
  fill_edges(static_cast<TrussOut*>(h)->result.edges, u, v, s);
}
void ref_truss_free(void* h) { delete static_cast<TrussOut*>(h); }

// canonicalize(raw) + build_csr; raw is m pairs of u64 labels.
int ref_canonicalize_csr(const std::uint64_t* raw, std::uint64_t m, void** out) {
  try {
    std::vector<RawEdge> edges(m);
    for (std::uint64_t i = 0; i < m; ++i) edges[i] = {raw[2 * i], raw[2 * i + 1]};
    auto* c = new CsrOut;
    c->csr = build_csr(canonicalize(edges));
    *out = c;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_random_graph_csr(std::uint32_t n, double p, std::uint64_t seed, void** out) {
  try {
    auto* c = new CsrOut;
    c->csr = build_csr(oracle::random_graph(n, p, seed));
    *out = c;
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

std::uint32_t ref_csr_n(void* h) { return static_cast<CsrOut*>(h)->csr.num_vertices; }
std::uint64_t ref_csr_slots(void* h) { return static_cast<CsrOut*>(h)->csr.col_idx.size(); }
void ref_csr_copy(void* h, std::uint32_t* row_ptr, std::uint32_t* col) {
  const auto& g = static_cast<CsrOut*>(h)->csr;
  std::memcpy(row_ptr, g.row_ptr.data(), g.row_ptr.size() * 4);
  std::memcpy(col, g.col_idx.data(), g.col_idx.size() * 4);
}
void ref_csr_free(void* h) { delete static_cast<CsrOut*>(h); }

int ref_validate_csr(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                     std::uint64_t slots) {
  try {
    validate_csr(make_csr(row_ptr, n, col, slots));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Brute-force oracle (oracle.cpp) over the live edges of a CSR.
namespace {
EdgeList edges_of(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                  std::uint64_t slots) {
  const ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
  EdgeList el;
  el.num_vertices = n;
  el.edges = extract_edges(g);
  el.original_ids.resize(n + std::size_t{1});
  for (std::uint32_t v = 1; v <= n; ++v) el.original_ids[v] = v;
  return el;
}
}  // namespace

std::uint32_t ref_oracle_kmax(const std::uint32_t* row_ptr, std::uint32_t n,
                              const std::uint32_t* col, std::uint64_t slots) {
  return oracle::kmax(edges_of(row_ptr, n, col, slots));
}

std::uint64_t ref_oracle_triangle_count(const std::uint32_t* row_ptr, std::uint32_t n,
                                        const std::uint32_t* col, std::uint64_t slots) {
  return oracle::triangle_count(edges_of(row_ptr, n, col, slots));
}

// Survivors of oracle::ktruss_edges at k with their oracle supports, in
// lexicographic order (acceptance.cpp:47-54). Returns the edge count; the
// arrays must hold m entries.
std::uint64_t ref_oracle_truss(const std::uint32_t* row_ptr, std::uint32_t n,
                               const std::uint32_t* col, std::uint64_t slots, std::uint32_t k,
                               std::uint32_t* u, std::uint32_t* v, std::uint32_t* s) {
  const EdgeList el = edges_of(row_ptr, n, col, slots);
  const std::vector<Edge> survivors = oracle::ktruss_edges(el, k);
  const auto sup = oracle::edge_supports(el.num_vertices, survivors);
  for (std::size_t i = 0; i < survivors.size(); ++i) {
    u[i] = survivors[i].u;
    v[i] = survivors[i].v;
    s[i] = sup.at(survivors[i]);
  }
  return survivors.size();
}

// write_csr_cache / read_csr_cache (csr_cache.cpp:71-111) to / from a file.
int ref_write_csr_cache(const char* path, const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                        std::uint64_t slots) {
  try {
    std::ofstream out(path, std::ios::binary);
    write_csr_cache(make_csr(row_ptr, n, col, slots), out);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_read_csr_cache(const char* path, void** out) {
  try {
    std::ifstream in(path, std::ios::binary);
    auto* c = new CsrOut;
    try {
      c->csr = read_csr_cache(in);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
    return 0;
  } catch (const CorruptCacheError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

double ref_millions_of_edges_per_second(std::uint64_t edges, double ms) {
  return millions_of_edges_per_second(edges, ms);
}

int ref_hardware_threads() { return hardware_threads(); }

}  // extern "C"

// ---- synthetic inputs -------------------------------------
namespace {

double u01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

// R-MAT raw pairs, Graph500 quadrant draw per level, then the explicit
// Fisher-Yates relabel driven by mt19937_64(seed ^ 0xABCDEF).
std::vector<RawEdge> rmat_raw(std::uint32_t scale, std::uint32_t ef, std::uint64_t seed, double a, double b,
                              double c) {
  const std::uint64_t N = std::uint64_t{1} << scale, m = N * ef;
  std::vector<RawEdge> raw(m);
  std::mt19937_64 g(seed);
  for (auto& e : raw) {
    std::uint64_t u = 0, v = 0;
    for (std::uint32_t l = 0; l < scale; ++l) {
      const double x = u01(g);
      const std::uint64_t bu = x < a + b ? 0 : 1;
      const std::uint64_t bv = (x < a || (x >= a + b && x < a + b + c)) ? 0 : 1;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    e = {u, v};
  }
  std::vector<std::uint64_t> perm(N);
  for (std::uint64_t i = 0; i < N; ++i) perm[i] = i;
  std::mt19937_64 g2(seed ^ 0xABCDEFull);
  for (std::uint64_t i = N - 1; i >= 1; --i) std::swap(perm[i], perm[g2() % (i + 1)]);
#pragma omp parallel for schedule(static)
  for (std::uint64_t i = 0; i < m; ++i) raw[i] = {perm[raw[i].first], perm[raw[i].second]};
  return raw;
}

// Parallel restatement of canonicalize (edge_list.cpp:62-103) for labels
// below `bound`: dense rank of the labels seen in non-loop pairs (= sorted
// unique + lower_bound + 1), orient u<v, sort, unique. Same EdgeList.
EdgeList canonicalize_fast(const std::vector<RawEdge>& raw, std::uint64_t bound) {
  std::vector<std::uint32_t> seen(bound, 0);
#pragma omp parallel for schedule(static)
  for (std::uint64_t i = 0; i < raw.size(); ++i) {
    if (raw[i].first == raw[i].second) continue;
    __atomic_store_n(&seen[raw[i].first], 1u, __ATOMIC_RELAXED);
    __atomic_store_n(&seen[raw[i].second], 1u, __ATOMIC_RELAXED);
  }
  EdgeList el;
  el.original_ids.push_back(0);
  std::uint32_t n = 0;
  for (std::uint64_t l = 0; l < bound; ++l) {
    if (seen[l]) {
      seen[l] = ++n;
      el.original_ids.push_back(l);
    }
  }
  if (n == 0) throw EmptyGraphError("no edges survive canonicalization");
  el.num_vertices = n;
  std::vector<std::uint64_t> keys(raw.size());
#pragma omp parallel for schedule(static)
  for (std::uint64_t i = 0; i < raw.size(); ++i) {
    const auto [x, y] = raw[i];
    const std::uint64_t u = seen[x], v = seen[y];
    keys[i] = x == y ? ~std::uint64_t{0} : (u < v ? (u << 32 | v) : (v << 32 | u));
  }
  __gnu_parallel::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  if (!keys.empty() && keys.back() == ~std::uint64_t{0}) keys.pop_back();
  el.edges.resize(keys.size());
#pragma omp parallel for schedule(static)
  for (std::uint64_t i = 0; i < keys.size(); ++i)
    el.edges[i] = {static_cast<std::uint32_t>(keys[i] >> 32), static_cast<std::uint32_t>(keys[i])};
  return el;
}

CsrOut* csr_of(std::vector<RawEdge>& raw, std::uint64_t bound, int fast) {
  auto* c = new CsrOut;
  try {
    c->csr = build_csr(fast ? canonicalize_fast(raw, bound) : canonicalize(raw));
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

}  // namespace

extern "C" {

// R-MAT(scale, ef, seed; a,b,c) plus `n_extra` extra label pairs (planted
// cliques), canonicalized and built into the reference CSR.
int ref_rmat_csr(std::uint32_t scale, std::uint32_t ef, std::uint64_t seed, double a, double b, double c,
                 const std::uint64_t* extra, std::uint64_t n_extra, int fast, void** out) {
  try {
    std::vector<RawEdge> raw = rmat_raw(scale, ef, seed, a, b, c);
    const std::uint64_t base = raw.size();
    raw.resize(base + n_extra);
    for (std::uint64_t i = 0; i < n_extra; ++i) raw[base + i] = {extra[2 * i], extra[2 * i + 1]};
    *out = csr_of(raw, std::uint64_t{1} << scale, fast);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Erdos-Renyi: m draws of (g() % 2^log_n, g() % 2^log_n) from mt19937_64(seed).
int ref_er_csr(std::uint32_t log_n, std::uint64_t m, std::uint64_t seed, int fast, void** out) {
  try {
    const std::uint64_t N = std::uint64_t{1} << log_n;
    std::vector<RawEdge> raw(m);
    std::mt19937_64 g(seed);
    for (auto& e : raw) {
      const std::uint64_t x = g() % N;
      e = {x, g() % N};
    }
    *out = csr_of(raw, N, fast);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Fine branch of compute_supports (support.cpp:115-127) restricted to the
// 256-slot chunks c (the omp dynamic,256 grain) with c % stride == phase, each
// slot through the reference's own intersect_tails. A bounded sample of one
// support pass for bench.py's cpu_baseline; supports accumulate into S.
// *elapsed_ms brackets the task loop only.
int ref_fine_sample(const std::uint32_t* row_ptr, std::uint32_t n, const std::uint32_t* col,
                    std::uint64_t slots, std::uint32_t* supports, std::uint32_t stride, std::uint32_t phase,
                    int threads, std::uint64_t* triangles, double* elapsed_ms) {
  try {
    if (threads < 1 || stride < 1) throw InvalidParameterError("thread count must be >= 1");
    const ZeroTerminatedCsr g = make_csr(row_ptr, n, col, slots);
    SupportArray s;
    s.counts.assign(supports, supports + slots);
    const std::uint64_t chunks = (slots + 255) / 256;
    std::uint64_t tri = 0;
    const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(+ : tri)
    for (std::uint64_t c = phase; c < chunks; c += stride) {
      const std::uint64_t end = std::min<std::uint64_t>(slots, (c + 1) * 256);
      for (std::uint64_t slot = c * 256; slot < end; ++slot) {
        const std::uint32_t pred = g.col_idx[slot];
        if (pred == 0) continue;
        const std::uint32_t found = intersect_tails(g, static_cast<std::uint32_t>(slot), pred, s);
        if (found != 0) std::atomic_ref<std::uint32_t>(s.counts[slot]).fetch_add(found, std::memory_order_relaxed);
        tri += found;
      }
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (elapsed_ms) *elapsed_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    *triangles = tri;
    std::memcpy(supports, s.counts.data(), slots * 4);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

}  // extern "C"
