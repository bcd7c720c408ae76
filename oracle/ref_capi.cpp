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
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <fstream>
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
