/*
 * ktg.h -- C ABI of the B200-native Eager K-truss engine (libktg.so).
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (/root/reference/proj) exposes it as a C++ static-library API; each ktg_*
 * entry point below replaces one of those functions with identical argument
 * meaning, in-place mutation rules and error behaviour (errors come back as
 * status codes; the C++ shim paper_2009_07929_b200/shim/ktruss_shim.cpp and
 * the Python host layer paper_2009_07929_b200/truss.py rethrow them as the
 * reference's exception types):
 *
 *   ktg_compute_supports  <- ktruss::compute_supports   include/ktruss/support.hpp:52-54,
 *                                                       src/support.cpp:93-132
 *   ktg_reset_supports    <- ktruss::reset_supports     support.hpp:56, support.cpp:134-136
 *   ktg_intersect_tails   <- ktruss::intersect_tails    support.hpp:44-45, support.cpp:64-91
 *   ktg_prune_edges       <- ktruss::prune_edges        include/ktruss/truss.hpp:38-39,
 *                                                       src/truss.cpp:9-37
 *   ktg_run_fixpoint      <- ktruss::detail::run_fixpoint truss.hpp:62-63, truss.cpp:41-53
 *   ktg_ktruss            <- ktruss::ktruss             truss.hpp:44-45, truss.cpp:57-71
 *   ktg_kmax_search       <- ktruss::kmax_search        truss.hpp:56, truss.cpp:73-103
 *
 * Data model (csr.hpp:17-23): upper-triangular zero-terminated CSR; vertex
 * ids 1..n, 0 is the sentinel; row_ptr has n+2 u32 entries, col_idx has
 * `slots` u32 entries; supports has one u32 per slot.
 *
 * All pointers in the ktg_* calls above are HOST pointers (like the
 * reference's std::vectors); host<->device copies happen inside. The
 * ktg_engine_* calls keep a graph resident in HBM across calls (the
 * device-resident path the benchmark times).
 *
 * Threading: calls on distinct engines may run concurrently; one engine must
 * not be used from two threads at once. No call retains caller pointers.
 */
#ifndef KTG_H
#define KTG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KTG_OK = 0,
  KTG_ERR_INVALID_PARAMETER = 1, /* ktruss::InvalidParameterError            */
  KTG_ERR_SUPPORT_OVERFLOW = 2,  /* ktruss::SupportOverflowError; slot via ktg_last_error_slot() */
  KTG_ERR_INVALID_INPUT = 3,     /* ktruss::InvalidInputError                */
  KTG_ERR_CORRUPT_CACHE = 4,     /* ktruss::CorruptCacheError                */
  KTG_ERR_EMPTY_GRAPH = 8,       /* ktruss::EmptyGraphError                  */
  KTG_ERR_CUDA = 5,              /* CUDA runtime / NCCL failure              */
  KTG_ERR_NO_DEVICE = 6,         /* no usable sm_100 device                  */
  KTG_ERR_OOM = 7                /* device or host allocation failed         */
} ktg_status;

/* Per-round observer (truss.hpp:25-26): called on the calling thread after
 * every prune with HOST copies of the pruned col_idx and the supports that
 * drove the round. Test-only: it forces a host-driven loop with a D2H copy
 * per round. */
typedef void (*ktg_round_cb)(const uint32_t* col_idx, const uint32_t* supports, uint64_t slots,
                             uint64_t removed, void* user);

/* Strategy (support.hpp:12-16). Every value runs the same device path; the
 * results are identical by the reference's own contract. */
enum { KTG_STRATEGY_SERIAL = 0, KTG_STRATEGY_COARSE = 1, KTG_STRATEGY_FINE = 2 };

/* flags */
enum {
  KTG_FLAG_HOST_LOOP = 1u << 0,     /* host-driven fixpoint loop instead of the
                                       device-resident CUDA-graph while loop  */
  KTG_FLAG_NAIVE_SUPPORT = 1u << 1, /* thread-per-slot merge kernel (paper
                                       Listing 1), for cross-checking only    */
  KTG_FLAG_COLLECT_WORK = 1u << 2,  /* record per-round closed-form work L_r,
                                       live edges and triangles (extra kernels) */
  KTG_FLAG_TIME_SUPPORT = 1u << 3,  /* host loop; CUDA events around every
                                       support launch (ktg_round_work.support_ms) */
  KTG_FLAG_LABEL_ORDER = 1u << 4,   /* run the fixpoint on the caller's (label-
                                       ordered) CSR instead of the internal
                                       degree-ordered working copy */
  KTG_FLAG_RECOMPUTE = 1u << 5,     /* recompute every round's supports from
                                       scratch (reset + computeSupports,
                                       truss.cpp:44-46) instead of carrying
                                       them: the default working-layout run
                                       decrements the supports of triangles
                                       that lose an edge whenever that is
                                       cheaper (same S, same rounds) */
  KTG_FLAG_NO_DEGREE_BOUND = 1u << 6 /* carried runs from the pristine graph
                                       skip round-0 pivots that cannot reach a
                                       possible survivor (support <= min
                                       degree - 1); this flag turns that off
                                       (results are identical either way) */
};

typedef struct {
  uint32_t struct_size;   /* sizeof(ktg_options)                              */
  int32_t device;         /* CUDA ordinal; -1 = current device                */
  uint32_t strategy;      /* KTG_STRATEGY_*; accepted, see above              */
  uint32_t width_bits;    /* 32 (SupportWidth::Bits32) or 16 (Bits16)         */
  uint32_t flags;         /* KTG_FLAG_*                                       */
  void* stream;           /* cudaStream_t to run on; NULL = engine-owned      */
  ktg_round_cb observer;  /* optional, test-only                             */
  void* observer_user;
} ktg_options;

/* Fills *o with the defaults (device -1, Fine, 32-bit, no flags). */
void ktg_options_init(ktg_options* o);

/* Message / overflow slot of the last failing call on this thread. */
const char* ktg_last_error(void);
uint64_t ktg_last_error_slot(void);

/* Library / device probe: 1 if an sm_100 device is visible, else 0. */
int ktg_device_available(void);
const char* ktg_version(void);
/* Slots per support-task chunk (the multi-GPU task partition unit). */
uint32_t ktg_task_chunk(void);

/* ---------------------------------------------------------------------- */
/* Reference-shaped entry points (host buffers)                            */
/* ---------------------------------------------------------------------- */

/* compute_supports: adds each live slot's triangle count into supports
 * (which the reference requires to be zero on entry) and returns the
 * triangle total. width_bits 16 -> KTG_ERR_SUPPORT_OVERFLOW naming the first
 * slot above 65535 (support.cpp:53-60). s_len must equal slots. */
ktg_status ktg_compute_supports(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx,
                                uint64_t slots, uint32_t* supports, uint64_t s_len,
                                const ktg_options* opt, uint64_t* triangles);

/* reset_supports: zero-fills supports[0..s_len). */
void ktg_reset_supports(uint32_t* supports, uint64_t s_len);

/* intersect_tails: merge of the pivot row tail with the predecessor's row;
 * bumps both matching slots in supports, returns the match count in *found. */
ktg_status ktg_intersect_tails(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx,
                               uint64_t slots, uint32_t pivot_slot, uint32_t predecessor,
                               uint32_t* supports, uint32_t* found);

/* prune_edges: in-place stable per-row compaction of col_idx keeping slots
 * with supports >= k-2; returns the removed count. supports is not touched.
 * k < 2 or s_len != slots -> KTG_ERR_INVALID_PARAMETER. */
ktg_status ktg_prune_edges(const uint32_t* row_ptr, uint32_t n, uint32_t* col_idx, uint64_t slots,
                           const uint32_t* supports, uint64_t s_len, uint32_t k,
                           const ktg_options* opt, uint64_t* removed);

/* detail::run_fixpoint: {reset, compute, prune} until a round removes
 * nothing, mutating col_idx and supports in place (supports ends as the
 * converged round's counts). Writes min(iterations, hist_cap) removal counts
 * to removed_hist; the last is 0. */
ktg_status ktg_run_fixpoint(const uint32_t* row_ptr, uint32_t n, uint32_t* col_idx, uint64_t slots,
                            uint32_t* supports, uint64_t s_len, uint32_t k, const ktg_options* opt,
                            uint64_t* removed_hist, uint32_t hist_cap, uint32_t* iterations);

/* ktruss: fixpoint on a private copy (col_idx is not mutated); the surviving
 * edges come back as parallel (u, v, support) arrays in lexicographic order
 * (extract_edges, csr.cpp:93-106). edge_cap must be >= the live edge count
 * of the input; *num_edges receives the survivor count. */
ktg_status ktg_ktruss(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots,
                      uint32_t k, const ktg_options* opt, uint32_t* out_u, uint32_t* out_v,
                      uint32_t* out_support, uint64_t edge_cap, uint64_t* num_edges,
                      uint64_t* removed_hist, uint32_t hist_cap, uint32_t* iterations);

/* kmax_search: largest k with a non-empty k-truss, plus that truss (same
 * output convention as ktg_ktruss). Empty graph -> KTG_ERR_INVALID_PARAMETER. */
ktg_status ktg_kmax_search(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx,
                           uint64_t slots, const ktg_options* opt, uint32_t* k_max,
                           uint32_t* out_u, uint32_t* out_v, uint32_t* out_support,
                           uint64_t edge_cap, uint64_t* num_edges, uint64_t* removed_hist,
                           uint32_t hist_cap, uint32_t* iterations);

/* ---------------------------------------------------------------------- */
/* Device-resident engine                                                  */
/* ---------------------------------------------------------------------- */

typedef struct ktg_engine ktg_engine;

typedef struct {
  uint32_t iterations;       /* rounds of the last fixpoint                  */
  uint64_t live_edges;       /* survivors after the last fixpoint            */
  uint64_t triangles;        /* triangle total of the converged round        */
  uint32_t max_support;      /* max S of the first round (kmax bound)        */
  double device_ms;          /* CUDA-event time of the last run              */
  uint32_t carried;          /* 1: supports can be carried across rounds (the
                                default path's structures are resident); 0:
                                every round recomputes (KTG_FLAG_RECOMPUTE,
                                label order, or the carried-support structures
                                did not fit in device memory at load)       */
} ktg_run_info;

/* Per-round closed-form work, recorded with KTG_FLAG_COLLECT_WORK. */
typedef struct {
  uint64_t live_edges;  /* live edges entering the round            */
  uint64_t L;           /* sum_v d+(d+-1)/2 + d+ d-    */
  uint64_t triangles;   /* triangles found in the round              */
  uint64_t removed;     /* edges pruned by the round                 */
  double support_ms;    /* support kernel time (KTG_FLAG_TIME_SUPPORT) */
  uint32_t full_pass;   /* 1: the round ran a full support pass; 0: its
                           supports were carried from the previous round */
  uint32_t pad;
  uint64_t L_tail;      /* the a12-tail part of L: sum_v d+(d+-1)/2       */
  uint64_t delta_cost;  /* carried runs: sum of min(du, dv) over removals  */
  uint64_t keep_cost;   /* carried runs: the same over the survivors       */
  uint32_t delta_pieces;/* carried runs: long intersections queued         */
  uint32_t carried;     /* carried runs: 1 if the round carried its S      */
} ktg_round_work;

ktg_status ktg_engine_create(const ktg_options* opt, ktg_engine** out);
void ktg_engine_destroy(ktg_engine* e);

/* Uploads a graph (host pointers) and keeps a pristine copy in HBM. */
ktg_status ktg_engine_load(ktg_engine* e, const uint32_t* row_ptr, uint32_t n,
                           const uint32_t* col_idx, uint64_t slots);
/* Same, from device pointers (D2D). */
ktg_status ktg_engine_load_device(ktg_engine* e, const uint32_t* d_row_ptr, uint32_t n,
                                  const uint32_t* d_col_idx, uint64_t slots);
/* ZTCSR1 cache file straight into HBM (read_csr_cache, csr_cache.hpp:19-21,
 * csr_cache.cpp:80-111): streamed through pinned staging buffers, structural
 * invariants validated on the device. Errors: KTG_ERR_CORRUPT_CACHE with the
 * reference's messages. */
ktg_status ktg_engine_load_cache(ktg_engine* e, const char* path);
/* canonicalize + build_csr on the device (edge_list.cpp:62-103, csr.cpp:10-32):
 * m raw (label, label) pairs as u64 (host or device pointer) -> the
 * reference's canonical zero-terminated CSR, loaded into the engine (CUB radix
 * sorts + unique, binary-search relabel). Errors: KTG_ERR_EMPTY_GRAPH,
 * KTG_ERR_INVALID_INPUT (> 2^32-1 slots / ids). */
ktg_status ktg_engine_build_csr(ktg_engine* e, const uint64_t* pairs, uint64_t m, int pairs_on_device);
ktg_status ktg_engine_csr_info(ktg_engine* e, uint32_t* n, uint64_t* slots);
/* The loaded graph (pristine) to host; original_ids (n+1 u64, [0] unused)
 * only for graphs built by ktg_engine_build_csr. Any pointer may be NULL. */
ktg_status ktg_engine_read_csr(ktg_engine* e, uint32_t* row_ptr, uint32_t* col_idx, uint64_t* original_ids);
/* Restores the pristine col_idx and zeroes both support buffers (async on
 * the engine stream). */
ktg_status ktg_engine_reset(ktg_engine* e);
/* Runs the fixpoint at k on the resident graph (from its current state).
 * Asynchronous unless removed_hist/iterations are requested: pass NULL/0 to
 * leave the result on the device and just enqueue. */
ktg_status ktg_engine_run(ktg_engine* e, uint32_t k, uint64_t* removed_hist, uint32_t hist_cap,
                          uint32_t* iterations);
/* One support pass (no reset, no prune) over the resident graph into the
 * current support buffer; optional triangle total (synchronises). */
ktg_status ktg_engine_support_pass(ktg_engine* e, uint64_t* triangles);
ktg_status ktg_engine_sync(ktg_engine* e);
ktg_status ktg_engine_info(ktg_engine* e, ktg_run_info* info);
/* Per-round records of the last run (KTG_FLAG_COLLECT_WORK / _TIME_SUPPORT). Returns the
 * number of rounds written. */
uint32_t ktg_engine_round_work(ktg_engine* e, ktg_round_work* out, uint32_t cap);
/* Copies the current col_idx / supports (converged buffer) to host. */
ktg_status ktg_engine_read(ktg_engine* e, uint32_t* col_idx, uint32_t* supports);
/* Device pointers of the current state and the engine stream. */
ktg_status ktg_engine_device_state(ktg_engine* e, uint32_t** d_col_idx, uint32_t** d_supports,
                                   void** stream);
/* Survivors of the resident graph as (u, v, support), lexicographic; device
 * compaction, D2H of the survivors only. */
ktg_status ktg_engine_extract(ktg_engine* e, uint32_t* out_u, uint32_t* out_v,
                              uint32_t* out_support, uint64_t edge_cap, uint64_t* num_edges);

/* Multi-GPU, host-driven exchange: every full support pass
 * covers this rank's share of the support tasks only -- in carried-support
 * runs (the default) a contiguous range of the A22 tasks split by a prefix
 * sum of their exact work on the pristine graph, computed once per load; in
 * KTG_FLAG_RECOMPUTE runs a
 * work-balanced range of chunk tasks -- and the caller all-reduces the
 * support buffer through the allreduce callback on the engine stream. The
 * callback runs after every FULL support pass only (carried rounds are
 * replicated on every rank and need no exchange); it sums S only, and the
 * engine derives the round's triangle count from the summed S in carried
 * runs (in recompute runs with the callback, info.triangles is this rank's
 * partial count). world == 1 restores single-GPU operation. Standalone
 * support passes (ktg_engine_support_pass, compute_supports, the kmax bound)
 * are never partitioned: every rank computes the whole pass. */
typedef int (*ktg_allreduce_cb)(uint32_t* d_buf, uint64_t count, void* stream, void* user);
ktg_status ktg_engine_set_partition(ktg_engine* e, uint32_t rank, uint32_t world,
                                    ktg_allreduce_cb allreduce, void* user);

/* Native NCCL variant: the engine all-reduces its partial supports (u32 sum)
 * and the round's triangle count (u64 sum) itself with ncclAllReduce on the
 * engine stream, over NVLink/NVSwitch. Rank 0 creates the id with
 * ktg_nccl_unique_id and ships the 128 bytes to every rank (e.g. through
 * torch.distributed); every rank then calls ktg_engine_set_nccl
 * (collective: blocks until all ranks joined). libnccl.so.2 is loaded with
 * dlopen on first use. */
ktg_status ktg_nccl_unique_id(uint8_t* out_128_bytes);
ktg_status ktg_engine_set_nccl(ktg_engine* e, uint32_t rank, uint32_t world, const uint8_t* unique_id);

/* Fused multi-GPU support pass (reduce-scatter fused into the
 * support kernel): the support buffers are split into `world` contiguous
 * owned spans (span = ceil(slots / world) slots); rank r's k_support_chunked
 * sends every increment straight to the owner's buffer with atomics on
 * NVLink peer memory, so no separate reduce step runs. peer_s0/peer_s1 hold
 * every rank's support buffers (ktg_engine_support_buffers on each rank,
 * mapped into this process: cudaIpcOpenMemHandle across processes, or plain
 * pointers for ranks sharing a process/device); entry `rank` must be this
 * engine's own. The exchange callback runs on the calling thread of the
 * host-driven loop: phase 0 before each support pass (wait for the stream,
 * then for every rank: each rank's previous prune zeroed the buffer the
 * others now add into), phase 1 after it (wait for the stream and every
 * rank, copy every other rank's owned span of the current buffer into
 * d_supports, replace *d_triangles (device u64) by the sum over ranks, and
 * wait again before returning). Call after loading the graph. */
typedef int (*ktg_peer_cb)(int phase, uint32_t* d_supports, uint64_t slots, uint64_t span,
                           unsigned long long* d_triangles, void* stream, void* user);
ktg_status ktg_engine_support_buffers(ktg_engine* e, uint32_t** d_s0, uint32_t** d_s1, uint64_t* slots);
ktg_status ktg_engine_set_peers(ktg_engine* e, uint32_t rank, uint32_t world, uint32_t* const* peer_s0,
                                uint32_t* const* peer_s1, ktg_peer_cb cb, void* user);
/* cudaMemcpyAsync(cudaMemcpyDefault) + stream synchronize: a helper for
 * exchange callbacks written in a host language without CUDA bindings. */
ktg_status ktg_device_copy(void* dst, const void* src, uint64_t bytes, void* stream);
/* CUDA IPC of support buffers between rank processes (64-byte handles):
 * ktg_ipc_handle on the owner, ktg_ipc_open on every peer (peer access is
 * enabled lazily; NVLink peer memory on one node), ktg_ipc_close when done. */
ktg_status ktg_ipc_handle(const void* d_ptr, uint8_t* out_64_bytes);
ktg_status ktg_ipc_open(const uint8_t* handle_64_bytes, void** d_ptr);
ktg_status ktg_ipc_close(void* d_ptr);

/* Peer group (the device-resident partitioned fixpoint): the
 * exchange runs as kernels over NVLink peer memory inside the fixpoint's
 * CUDA graph, so a partitioned fixpoint is ONE graph launch with no host
 * round trip per round:
 *   full pass   this rank's work-balanced range of the A22 tasks, then a
 *               device barrier, a reduce of this rank's span of S over every
 *               rank's partial buffer written back to every rank (reduce-
 *               scatter + all-gather in one kernel), and a second barrier;
 *   carried     the round's removed edges are sharded by a hash of the edge
 *   round       id; each rank finds the lost triangles of its share, applies
 *               the decrements locally and lists them in its exchange area;
 *               after a device barrier every rank applies its peers' lists.
 *               Compaction stays replicated (deterministic, same on every rank).
 * Setup (after ktg_engine_load, collective): every rank allocates its area
 * with ktg_engine_group_area, shares it and its support buffers
 * (ktg_engine_support_buffers) with the peers (ktg_ipc_handle / ktg_ipc_open
 * across processes, plain pointers within one), then calls
 * ktg_engine_set_group with the tables of every rank's area / S0 / S1 mapped
 * into this process (own entry at `rank`), then all ranks meet in a host
 * barrier before the first run. Every rank must run the same sequence of
 * fixpoints (same k). A rank that stops joining barriers makes its peers fail
 * with KTG_ERR_CUDA ("peer group barrier timed out") after 120 s. Loading
 * another graph leaves the group (set it up again). */
ktg_status ktg_engine_group_area(ktg_engine* e, void** d_area, uint64_t* bytes);
ktg_status ktg_engine_set_group(ktg_engine* e, uint32_t rank, uint32_t world, void* const* areas,
                                uint32_t* const* peer_s0, uint32_t* const* peer_s1);

#ifdef __cplusplus
}
#endif
#endif
