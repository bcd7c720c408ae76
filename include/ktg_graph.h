/*
 * ktg_graph.h -- host-side graph preparation for the B200 K-truss engine.
 *
 * Not the hot path: this is the input side of the boundary (synthetic
 * generators of SURVEY.md §8(d), and canonicalize + build_csr producing the
 * reference's zero-terminated CSR byte-for-byte). Implemented in
 * paper_2009_07929_b200/csrc/graph_host.cpp, shipped as libktg_graph.so
 * (no CUDA dependency, usable on CPU-only hosts).
 *
 * Reference interfaces restated:
 *   ktgg_csr_from_pairs_*  <- ktruss::canonicalize (edge_list.hpp:51-53,
 *                             edge_list.cpp:62-103) followed by
 *                             ktruss::build_csr (csr.hpp:27, csr.cpp:10-32)
 */
#ifndef KTG_GRAPH_H
#define KTG_GRAPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  KTGG_OK = 0,
  KTGG_ERR_INVALID_PARAMETER = 1,
  KTGG_ERR_INVALID_INPUT = 3,
  KTGG_ERR_EMPTY_GRAPH = 4,
  KTGG_ERR_CORRUPT_CACHE = 5,
  KTGG_ERR_IO = 6,
  KTGG_ERR_OOM = 7
};

typedef struct ktgg_raw ktgg_raw; /* raw u32 label pairs, pre-canonicalization */
typedef struct ktgg_csr ktgg_csr; /* canonical zero-terminated CSR */

typedef struct {
  uint64_t live_edges;
  uint32_t max_out_degree;
  uint64_t tail_elements;  /* sum_v d+(d+-1)/2   (a12 tails)  */
  uint64_t cross_elements; /* sum_v d+ * d-      (A22 rows)   */
  uint64_t L;              /* tail + cross                     */
  uint64_t sum_dout_sq;
} ktgg_work;

const char* ktgg_last_error(void);

/* R-MAT: ef*2^scale draws with mt19937_64(seed), 53-bit
 * uniforms against (a, a+b, a+b+c), then a Fisher-Yates relabel drawn from
 * mt19937_64(seed ^ 0xABCDEF). */
int ktgg_rmat_raw(uint32_t scale, uint32_t edgefactor, uint64_t seed, double a, double b, double c,
                  ktgg_raw** out);
/* Erdős–Rényi: m draws of (rng()%2^log_n, rng()%2^log_n). */
int ktgg_er_raw(uint32_t log_n, uint64_t m, uint64_t seed, ktgg_raw** out);
uint64_t ktgg_raw_count(const ktgg_raw* r);
const uint32_t* ktgg_raw_pairs(const ktgg_raw* r);
void ktgg_raw_free(ktgg_raw* r);

/* canonicalize + build_csr. Errors: KTGG_ERR_EMPTY_GRAPH (no non-loop pair),
 * KTGG_ERR_INVALID_INPUT (> 2^32-1 slots or ids). */
int ktgg_csr_from_raw(const ktgg_raw* r, ktgg_csr** out);
int ktgg_csr_from_pairs_u32(const uint32_t* pairs, uint64_t m, ktgg_csr** out);
int ktgg_csr_from_pairs_u64(const uint64_t* pairs, uint64_t m, ktgg_csr** out);
uint32_t ktgg_csr_n(const ktgg_csr* c);
uint64_t ktgg_csr_slots(const ktgg_csr* c);
/* row_ptr: n+2 entries, col: slots entries, original_ids: n+1 entries ([0]
 * unused); any pointer may be NULL. */
void ktgg_csr_copy(const ktgg_csr* c, uint32_t* row_ptr, uint32_t* col, uint64_t* original_ids);
void ktgg_csr_free(ktgg_csr* c);

/* ZTCSR1 binary cache <- write_csr_cache / read_csr_cache (csr_cache.hpp:16-21,
 * csr_cache.cpp:71-111): "ZTCSR1\0\0" | u32 n | u64 slots | row_ptr | col_idx,
 * little-endian. The reader validates like the reference (KTGG_ERR_CORRUPT_CACHE
 * with the reference's messages). */
int ktgg_write_csr_cache(const char* path, const uint32_t* row_ptr, uint32_t n, const uint32_t* col,
                         uint64_t slots);
int ktgg_read_csr_cache(const char* path, ktgg_csr** out);

/* validate_csr (csr.hpp:32, csr.cpp:34-80): KTGG_OK or KTGG_ERR_INVALID_INPUT
 * with the reference's message for the first violation. */
int ktgg_validate_csr(const uint32_t* row_ptr, uint64_t rp_len, uint32_t n, const uint32_t* col, uint64_t slots);

/* Closed-form merge work of one support pass over the live graph. */
void ktgg_round_work(const uint32_t* row_ptr, uint32_t n, const uint32_t* col, ktgg_work* w);

#ifdef __cplusplus
}
#endif
#endif
