// Device kernels of the B200 Eager K-truss engine (sm_100a).
//
// Hot path per round:
//   k_plan_count / k_plan_write  -- split the slot space into support tasks
//   k_support_chunked            -- computeSupports (support.cpp:93-132 semantics)
//   k_prune_light / k_prune_heavy-- pruneEdges (truss.cpp:9-37) fused with the
//                                   support reset of the next round
//   k_control                    -- removal history + device-side while flag
//                                   (run_fixpoint, truss.cpp:41-53)
//
// All arithmetic is integer; every count the reference keeps in u64 is u64
// here. Support increments are commutative atomics, so the result is
// bit-identical to the reference for any schedule.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ktg {

constexpr int kChunk = 512;          // slots per staged chunk (P)
constexpr int kSupportThreads = 256; // threads per support CTA
constexpr int kPruneThreads = 256;
constexpr int kHeavyRow = 2048;      // rows longer than this are pruned by a CTA
// Heavy rows are few (the hubs), so their CTA-per-row kernels run 1024-wide:
// a row takes 4x fewer dependent tile steps than with 256 threads.
constexpr int kSymHeavyThreads = 1024;
constexpr uint32_t kClipMin = 16;    // clip N+(j) by binary search above this degree
constexpr uint32_t kScanRatio = 4;   // scan N+(j) if |N+(j)| <= ratio * |tail|
constexpr int kHistCap = 1 << 16;    // recorded rounds per fixpoint

// Device-resident loop state (one per engine).
struct DevState {
  unsigned long long removed;        // edges pruned this round
  unsigned long long triangles;      // triangles found this round
  unsigned long long last_triangles; // triangles of the last completed round
  unsigned long long live;           // live edges
  unsigned long long overflow_slot;  // min slot with S > 65535 (Bits16)
  unsigned int parity;               // support buffer of the current round
  unsigned int iter;                 // completed rounds
  unsigned int threshold;            // k - 2
  unsigned int task_next;            // support work counter
  unsigned int npairs;               // off-diagonal tasks this round
  unsigned int nheavy;               // heavy rows queued for CTA prune
  unsigned int error;                // nonzero stops the loop
  unsigned int max_support;          // max S seen by k_max_support
  unsigned int width16;              // check supports against 65535
  unsigned int pad;
  unsigned long long pairs_needed;   // off-diagonal task capacity (load time)
  // incremental rounds (working layout, see k_mark / k_delta)
  unsigned int inc;                  // 1: supports are carried across rounds when cheaper
  unsigned int mode;                 // this round: 0 = recompute supports, 1 = carried (delta)
  unsigned int nrq;                  // delta tasks queued by k_mark this round
  unsigned int pad3;
  unsigned int pad2;
  double delta_ratio;                // carry when delta_cost <= delta_ratio * keep_cost
  unsigned long long sum_s;          // sum of S over live edges (k_mark): 3 * triangles
  unsigned long long delta_cost;     // sum over removed edges of min(du, dv)
  unsigned long long keep_cost;      // sum over surviving edges of min(du, dv)
  unsigned long long live_cost;      // keep_cost carried to the next round
  unsigned int carry;                // this round carries supports (k_decide)
  unsigned int fpar;                 // frontier queue consumed this round
  unsigned int nfq[2];               // frontier queue lengths
  unsigned int nqrow, nqsym;         // rows queued for compaction this round
  unsigned int nheavy_sym;           // long symmetric rows queued for CTA compaction
  unsigned int h0;                   // round 0 from pristine: first rank of degree >= k-1 (0: off)
  unsigned int pristine;             // this round runs on the pristine working layout
  unsigned int last_nrq;             // statistics of the last completed round:
  unsigned int last_carry;           //   queued delta pieces, whether it carried,
  unsigned long long last_dcost;     //   its delta cost and keep cost
  unsigned long long last_kcost;
  double delta_ratio0;               // the same for round 0 of a run from the pristine graph
  unsigned int dq_lo, dq_hi;         // this rank's diagonal support tasks: chunks [dq_lo, dq_hi)
  unsigned long long rq_cap;         // delta piece queue capacity (a round that could exceed it recomputes)
  unsigned int a22_lo, a22_hi;       // k_a22_split's result (read back into Graph::a22_lo/hi)
  unsigned int xepoch;               // peer group: barriers passed (never reset by a run)
  unsigned int pad4;
};

constexpr unsigned int kErrGroupTimeout = 2;  // DevState::error: a peer never reached a barrier

// Peer group (multi-GPU, ktg_engine_set_group): the exchange area each rank
// keeps in its own HBM and every rank maps (CUDA IPC / peer access).
constexpr int kMaxGroup = 64;
struct XArea {
  unsigned int flags[kMaxGroup];  // barrier: the epoch rank q has reached (written by q)
  unsigned long long tri;         // this rank's partial triangle count of the current full pass
  unsigned int cnt[2];            // lengths of this rank's decrement lists (round parity)
  unsigned int pad[28];
  // followed by 2 lists of `cap` edge ids: the surviving edges this rank's
  // share of a carried round decremented
};
static_assert(sizeof(XArea) % 16 == 0, "lists start 16-byte aligned");
__host__ __device__ __forceinline__ uint32_t* xlist(XArea* a, uint64_t cap, uint32_t par) {
  return reinterpret_cast<uint32_t*>(a + 1) + par * cap;
}

struct Graph {
  const uint32_t* row_ptr;  // n+2
  uint32_t* col;            // slots (+pad)
  uint32_t* S0;             // support buffers (ping-pong)
  uint32_t* S1;
  uint32_t* deg;            // live out-degree per row, n+2
  const uint32_t* chunk_row;// row containing the last slot of each chunk
  uint2* pairs;             // off-diagonal tasks (q, q2)
  uint32_t* pair_counts;    // per-chunk off-diagonal task count
  uint32_t* heavy_rows;     // rows queued for CTA prune
  DevState* st;
  unsigned long long* hist; // removal count per round
  uint32_t n;
  uint32_t nchunks;
  uint64_t slots;
  uint32_t rank;            // multi-GPU task split
  uint32_t world;
  uint32_t scan_ratio;      // SCAN N+(j) when |N+(j)| <= ratio * |tail|
  uint32_t* payload;        // per-slot id compacted along with col (working layout) or null
  // fused reduce-scatter (multi-GPU, ktg_engine_set_peers): every support
  // increment goes straight to the owner rank's buffer (slot / span) over
  // NVLink peer memory; npeer = 0 keeps local increments
  uint32_t* const* peer0;   // per rank: its S0 (device pointers, peer-mapped)
  uint32_t* const* peer1;   // per rank: its S1
  uint64_t span;            // slots owned per rank
  uint32_t npeer;
  // peer group: this rank's exchange area (null: no group); a carried
  // round's removals are sharded by owner_of(edge id) and every decrement is
  // also listed for the peers (k_xapply)
  XArea* xa;
  uint64_t xcap;
  // multi-rank full passes: this rank's A22 tasks [a22_lo, a22_hi), split by
  // the pristine graph's exact task work (k_support_a22<true> + k_a22_split,
  // once per load)
  uint32_t a22_lo, a22_hi;
};

// Rank owning removed edge id in a sharded carried round (a hash, so the
// split does not follow the caller's row order).
__host__ __device__ __forceinline__ uint32_t owner_of(uint32_t id, uint32_t world) {
  return (uint32_t)(((uint64_t)(id * 2654435761u) * world) >> 32);
}

// One support increment: local buffer, or the owning rank's buffer when the
// support pass is fused with the reduce-scatter.
__device__ __forceinline__ void sadd(const Graph& g, uint32_t* __restrict__ S, uint64_t slot, uint32_t v) {
  if (g.npeer == 0) {
    atomicAdd(S + slot, v);
    return;
  }
  uint32_t* const* tab = g.st->parity ? g.peer1 : g.peer0;
  atomicAdd(tab[(uint32_t)(slot / g.span)] + slot, v);
}

// Symmetric adjacency of the working layout for incremental rounds: row v
// lists every live neighbour of v (in-neighbours then out-neighbours, so the
// row is ascending) with the edge's id (its caller slot, = payload of the
// oriented entry). Rows are compacted as edges die; symdeg is the live length.
struct Sym {
  const unsigned long long* ptr;  // n+2 row offsets
  uint32_t* nbr;
  uint32_t* eid;
  uint32_t* deg;                  // live length of each row
  uint8_t* dead;                  // per edge id: removed (sticky within a fixpoint)
  uint8_t* rdirty;                // per vertex: its working row lost an edge this round
  uint8_t* sdirty;                // per vertex: its symmetric row lost an edge this round
  uint32_t* qsym;                 // symmetric rows to compact this round
  uint32_t* qrow;                 // oriented (working) rows to compact this round
  uint32_t* heavy;                // symmetric rows longer than kHeavyRow (CTA compaction)
  uint32_t* pos_of;               // per edge id: current working slot of the edge
  const uint32_t* erow;           // per edge id: its working (oriented) row
  uint32_t* fq0;                  // frontier queues (edge ids whose carried
  uint32_t* fq1;                  //   support crossed below k-2), ping-pong
  uint4* rq;                      // delta tasks {slot, u, v, piece}
};

constexpr uint32_t kDeadMark = 0x80000000u;  // col mark of an edge removed this round
constexpr int kDeltaPiece = 64;              // smaller-list elements per delta task

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t* cur_S(const Graph& g) { return g.st->parity ? g.S1 : g.S0; }
__device__ __forceinline__ uint32_t* other_S(const Graph& g) { return g.st->parity ? g.S0 : g.S1; }


// ---------------------------------------------------------------------------
// Setup kernels
// ---------------------------------------------------------------------------

// validate_csr (csr.cpp:34-80) per-row checks on the device, warp per row:
// first violation in reference order, packed row << 3 | code into *first
// (atomicMin keeps the lowest row). Codes: 1 no sentinel slot, 2 no zero at
// the row end, 3 nonzero after a zero, 4 not strictly ascending above the
// vertex, 5 beyond n.
// Live out-degree per row, thread per row: a valid row is nonzeros then
// zeros, so its first zero is found by a binary search inside the row
// (O(n log d) instead of a search over row_ptr per row end).
__global__ void k_row_deg(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, uint32_t n,
                          uint32_t* __restrict__ deg, DevState* st) {
  unsigned long long live = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x + 1; v <= n; v += gridDim.x * blockDim.x) {
    uint32_t lo = row_ptr[v], hi = row_ptr[v + 1];
    const uint32_t b = lo;
    while (lo < hi) {  // first zero in [lo, hi)
      const uint32_t mid = (lo + hi) >> 1;
      if (col[mid] != 0) lo = mid + 1; else hi = mid;
    }
    deg[v] = lo - b;
    live += lo - b;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
  if ((threadIdx.x & 31) == 0 && live) atomicAdd(&st->live, live);
}

__global__ void k_validate_rows(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, uint32_t n,
                                uint64_t slots, unsigned long long* first) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t v = warp + 1; v <= n; v += nwarps) {
    const uint32_t b = row_ptr[v], e = row_ptr[v + 1];
    uint32_t code = 0;
    if (b >= e) code = 1;
    else if (e > slots || col[e - 1] != 0) code = 2;  // e > slots: the reference reads past col (UB)
    else {
      uint32_t prev = v;      // value of the previous nonzero slot (or v)
      bool zero_seen = false;
      for (uint32_t off = b; off < e && code == 0; off += 32) {
        const uint32_t x = off + lane;
        const bool in = x < e;
        const uint32_t w = in ? col[x] : 0u;
        const unsigned zm = __ballot_sync(0xffffffffu, in && w == 0);
        const bool zero_before = zero_seen || (zm & ((1u << lane) - 1u));
        uint32_t pw = __shfl_up_sync(0xffffffffu, w, 1);
        if (lane == 0) pw = prev;
        // the previous slot is nonzero whenever this one is checked for order
        uint32_t c = 0;
        if (in && w != 0) {
          if (zero_before) c = 3;
          else if (w <= pw) c = 4;
          else if (w > n) c = 5;
        }
        const unsigned bm = __ballot_sync(0xffffffffu, c != 0);
        if (bm) code = __shfl_sync(0xffffffffu, c, __ffs(bm) - 1);
        zero_seen = zero_seen || zm;
        prev = __shfl_sync(0xffffffffu, w, 31);
      }
    }
    if (lane == 0 && code) atomicMin(first, ((unsigned long long)v << 3) | code);
  }
}

// Row containing the last slot of every chunk (fixed for the graph's life).
__global__ void k_chunk_rows(const uint32_t* __restrict__ row_ptr, uint32_t n, uint64_t slots,
                             uint32_t nchunks, uint32_t* __restrict__ chunk_row) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nchunks) return;
  const uint64_t e64 = umin64((uint64_t)(q + 1) * kChunk, slots) - 1;
  const uint32_t e = (uint32_t)e64;
  // upper_bound(row_ptr[0..n+2), e) - 1
  uint32_t lo = 0, hi = n + 2;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= e) lo = mid + 1; else hi = mid;
  }
  chunk_row[q] = lo - 1;
}

// ---------------------------------------------------------------------------
// Planning: task list for the support kernel
// ---------------------------------------------------------------------------
// A task (q, q2) processes the pivots of chunk q against the a12 tails that
// lie in chunk q2 (staged in shared memory). Diagonal tasks (q, q) cover every
// pivot whose tail starts in its own chunk; only the last row of chunk q can
// extend past it, and its pivots get one off-diagonal task per further chunk
// its live part reaches.

__global__ void k_plan_count(Graph g, int total) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= g.nchunks || g.st->mode) return;
  const uint32_t i = g.chunk_row[q];
  uint32_t cnt = 0;
  if (i >= 1) {
    const uint64_t le = (uint64_t)g.row_ptr[i] + g.deg[i];  // live end (exclusive)
    const uint64_t e = umin64((uint64_t)(q + 1) * kChunk, g.slots);
    if (le > e) cnt = (uint32_t)((le - 1) / kChunk - q);
  }
  g.pair_counts[q] = cnt;
  if (total && cnt) atomicAdd(&g.st->pairs_needed, (unsigned long long)cnt);
}

// Single CTA: exclusive scan of pair_counts, write the pair list, reset the
// task counter. 1024 threads.
__global__ void __launch_bounds__(1024) k_plan_write(Graph g) {
  __shared__ uint32_t warp_sums[32];
  if (g.st->mode) return;  // supports carried this round
  const uint32_t tid = threadIdx.x;
  const uint32_t Q = g.nchunks;
  const uint32_t per = (Q + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(tid * per, Q), hi = min(lo + per, Q);
  uint32_t local = 0;
  for (uint32_t q = lo; q < hi; ++q) local += g.pair_counts[q];
  // block exclusive scan of `local`
  const int lane = tid & 31, wid = tid >> 5;
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;  // inclusive
  }
  __syncthreads();
  uint32_t off = x - local + (wid ? warp_sums[wid - 1] : 0);
  for (uint32_t q = lo; q < hi; ++q) {
    const uint32_t c = g.pair_counts[q];
    for (uint32_t t = 1; t <= c; ++t) g.pairs[off++] = make_uint2(q, q + t);
  }
  if (tid == blockDim.x - 1) {
    g.st->npairs = off;
    g.st->task_next = 0;
    g.st->dq_lo = 0;  // one rank: every diagonal task (k_rank_range narrows it)
    g.st->dq_hi = Q;
  }
}

// Multi-GPU work-balanced split: estimated work of diagonal
// task q = sum over its live pivots s of (tail inside the chunk + 1 +
// live out-degree of col[s]); CTA per chunk, next zeros from a backward
// scan of the staged chunk. cost[Q] = 0 so an exclusive scan ends in the
// total. oracle/ktruss_oracle.c:orc_task_cost restates it.
__global__ void __launch_bounds__(kChunk) k_task_cost(Graph g, unsigned long long* __restrict__ cost) {
  __shared__ uint32_t nz[kChunk];
  __shared__ unsigned long long red[kChunk / 32];
  const uint32_t q = blockIdx.x, x = threadIdx.x;
  if (q >= g.nchunks) {
    if (q == g.nchunks && x == 0) cost[q] = 0;
    return;
  }
  const uint64_t p0 = (uint64_t)q * kChunk;
  const uint32_t plen = (uint32_t)umin64(kChunk, g.slots - p0);
  const uint32_t v = x < plen ? g.col[p0 + x] : 0u;
  nz[x] = (x < plen && v != 0) ? kChunk : x;  // zero (or past the end): its own index
  __syncthreads();
  // next zero at or after x: suffix minimum (Hillis-Steele, log2(kChunk) steps)
  for (uint32_t o = 1; o < kChunk; o <<= 1) {
    const uint32_t y = x + o < kChunk ? nz[x + o] : (uint32_t)kChunk;
    __syncthreads();
    nz[x] = min(nz[x], y);
    __syncthreads();
  }
  unsigned long long c = 0;
  if (x < plen && v != 0) c = (unsigned long long)(min(nz[x], plen) - x - 1) + 1ull + g.deg[v];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((x & 31) == 0) red[x >> 5] = c;
  __syncthreads();
  if (x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kChunk / 32; ++w) t += red[w];
    cost[q] = t;
  }
}

// This rank's diagonal chunks: chunk q goes to rank min(world-1,
// pre[q] * world / total) (pre = exclusive prefix of the task costs), which
// is non-decreasing in q, so every rank owns one contiguous range.
__global__ void k_rank_range(Graph g, const unsigned long long* __restrict__ pre) {
  const uint32_t Q = g.nchunks;
  const unsigned long long T = pre[Q];
  auto owner = [&](uint32_t q) -> uint32_t {
    if (T == 0) return 0u;
    const unsigned long long r = pre[q] * g.world / T;
    return (uint32_t)(r < g.world - 1 ? r : g.world - 1);
  };
  auto first = [&](uint32_t r) -> uint32_t {  // first q with owner(q) >= r
    if (r == 0) return 0u;
    if (r >= g.world) return Q;
    uint32_t lo = 0, hi = Q;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (owner(mid) < r) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  g.st->dq_lo = first(g.rank);
  g.st->dq_hi = first(g.rank + 1);
}

// ---------------------------------------------------------------------------
// Support kernel
// ---------------------------------------------------------------------------
constexpr int kFilterBits = 1 << 15;     // membership filter over (value, row run)
constexpr int kStrip = 512;              // flat elements a warp takes per grab (16 per lane)
constexpr int kQueue = 64;               // per-warp queue of filter positives
constexpr int kBuckets = kChunk / 4;     // position hash: kBuckets x 8 slots (load <= 0.5)
constexpr int kStash = 32;               // overflow entries of full buckets

struct SupportSmem {
  uint32_t A[kChunk];          // staged slots col[a0 .. a0+alen)
  uint32_t cntA[kChunk];       // pending increments of staged slots
  union {
    uint16_t nz[2 * kChunk];   // prologue: next zero at or after x (alen if none)
    uint32_t cntP[kChunk];     // work loop: pending pivot counts (off-diagonal)
  };
  uint32_t pref[kChunk + 1];   // exclusive prefix of per-pivot cost
  uint32_t b0[kChunk];         // clipped N+(j) range [b0, b1)
  uint32_t b1[kChunk];
  uint16_t te[kChunk];         // tail end (relative to a0) | 0x8000 if SCAN mode
  uint32_t filt[kFilterBits / 32];
  uint32_t qk[kSupportThreads / 32][kQueue];   // queued (value, col position, pivot)
  uint32_t qpos[kSupportThreads / 32][kQueue];
  uint16_t qp[kSupportThreads / 32][kQueue];
  __align__(16) uint32_t hkey[kBuckets][8];   // staged value (0 = empty)
  __align__(16) uint32_t hmeta[kBuckets][8];  // row-run end << 16 | position
  uint32_t hcnt[kBuckets];
  uint32_t skey[kStash], smeta[kStash];
  uint32_t nstash;
  uint32_t red[kSupportThreads / 32];
  uint32_t task;
  uint32_t next;               // flat work counter of the current task
};

__device__ __forceinline__ uint32_t filt_hash(uint32_t k, uint32_t te) {
  return ((k ^ (te * 0x85EBCA6Bu)) * 2654435761u) >> (32 - 15);
}

__device__ __forceinline__ uint32_t bucket_of(uint32_t k, uint32_t te) {
  return (((k ^ (te * 0x85EBCA6Bu)) * 2654435761u) >> 16) % kBuckets;
}

// Position of value k in the row run ending at te, at or after tb; kChunk if
// absent. One bucket read (2 x 128-bit); only an overflowed bucket consults
// the stash.
template <typename Smem>
__device__ __forceinline__ uint32_t hash_find(const Smem& s, uint32_t k, uint32_t tb, uint32_t te) {
  const uint32_t b = bucket_of(k, te);
  const uint4 k0 = *reinterpret_cast<const uint4*>(&s.hkey[b][0]);
  const uint4 k1 = *reinterpret_cast<const uint4*>(&s.hkey[b][4]);
  uint32_t m = (k0.x == k) | ((k0.y == k) << 1) | ((k0.z == k) << 2) | ((k0.w == k) << 3) |
               ((k1.x == k) << 4) | ((k1.y == k) << 5) | ((k1.z == k) << 6) | ((k1.w == k) << 7);
  while (m) {
    const int i = __ffs(m) - 1;
    m &= m - 1;
    const uint32_t meta = s.hmeta[b][i];
    const uint32_t pos = meta & 0xffffu;
    if ((meta >> 16) == te && pos >= tb) return pos;
  }
  if (s.hcnt[b] <= 8) return kChunk;
  const uint32_t ns = min(s.nstash, (uint32_t)kStash);
  for (uint32_t i = 0; i < ns; ++i) {
    if (s.skey[i] == k) {
      const uint32_t meta = s.smeta[i];
      const uint32_t pos = meta & 0xffffu;
      if ((meta >> 16) == te && pos >= tb) return pos;
    }
  }
  return kChunk;
}

// Branchless lower_bound over a sorted run a[0, n) (n >= 1 not required):
// first index with a[i] >= key, n if none.
__device__ __forceinline__ uint32_t lb_smem(const uint32_t* a, uint32_t n, uint32_t key) {
  if (n == 0) return 0;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (base[half] < key) ? base + half : base;
    n -= half;
  }
  return (uint32_t)(base - a) + (*base < key);
}

__device__ __forceinline__ uint32_t lb_global(const uint32_t* __restrict__ a, uint32_t lo, uint32_t hi, uint32_t key) {
  uint32_t n = hi - lo;
  if (n == 0) return lo;
  const uint32_t* base = a + lo;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (__ldg(base + half) < key) ? base + half : base;
    n -= half;
  }
  return (uint32_t)(base - a) + (__ldg(base) < key);
}


// Block-wide exclusive scan of one u32 per thread; returns the prefix, total
// in *total. Uses red as scratch.
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t* red, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = kSupportThreads / 32;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < NW ? red[lane] : 0;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) red[lane] = w;
  }
  __syncthreads();
  const uint32_t r = x - v + (wid ? red[wid - 1] : 0);
  *total = red[NW - 1];
  __syncthreads();
  return r;
}

// Confirms one queued filter positive: binary search of k in the pivot's
// tail; on a match bumps the tail slot (smem), the A22 slot (global) and the
// pivot count (smem).
__device__ __forceinline__ bool confirm(const Graph& g, SupportSmem& s, uint32_t* __restrict__ S, uint32_t* cntPiv,
                                        bool diag,
                                        uint32_t k, uint32_t pos, uint32_t p) {
  const uint32_t te = s.te[p] & 0x7fffu;
  const uint32_t tb = diag ? p + 1 : 0;
  uint32_t x;
  if (s.nstash <= (uint32_t)kStash) {
    x = hash_find(s, k, tb, te);
  } else {
    x = tb + lb_smem(s.A + tb, te - tb, k);
    if (!(x < te && s.A[x] == k)) x = kChunk;
  }
  if (x < (uint32_t)kChunk) {
    atomicAdd(&s.cntA[x], 1u);
    sadd(g, S, pos, 1u);
    atomicAdd(&cntPiv[p], 1u);
    return true;
  }
  return false;
}

// Persistent CTAs pull tasks (q, q2) off a counter. Per task:
//   1. stage chunk q2 of col in smem, find the next zero of every position,
//      set a membership-filter bit for every (value, row-run end) pair;
//   2. per pivot slot s=(i,j) in chunk q: its a12 tail within the staged chunk
//      [tb, te); clip N+(j) to the tail's value range; choose SCAN (read the
//      clipped N+(j) coalesced and test each element against the filter) or
//      ITERATE (binary-search each tail element in N+(j)) by cost;
//   3. flatten all pivots' work with a prefix sum; warps grab strips of it
//      dynamically; each lane caches its pivot's descriptor in registers;
//      SCAN elements that pass the filter (~hits + 1.5% false positives) are
//      queued per warp and confirmed 32 at a time by a (value, row-run) bucket
//      hash that returns the tail position in one bucket read;
//   4. a match (i,j,k) adds 1 to S[slot(i,k)] (smem), S[slot(j,k)] (global
//      red.add) and the pivot's count (smem); smem counts are flushed once.
// Semantically each pivot slot gets exactly intersect_tails' matches
// (support.cpp:64-91) plus the pivot add (support.cpp:122).
#ifndef KTG_CHUNKED_MINB
#define KTG_CHUNKED_MINB 6  // 6 CTAs / SM at <= 40 registers: s24 pass 579 -> 379 ms (the 64-register build ran 4)
#endif
__global__ void __launch_bounds__(kSupportThreads, KTG_CHUNKED_MINB)
k_support_chunked(Graph g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SupportSmem& s = *reinterpret_cast<SupportSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kSupportThreads / 32;
  constexpr int EPT = kChunk / kSupportThreads;
  constexpr int FPT = kFilterBits / 32 / kSupportThreads;
  if (g.st->mode) return;  // supports carried this round (incremental mode)
  uint32_t* __restrict__ S = cur_S(g);
  const uint32_t* __restrict__ col = g.col;
  // this rank's tasks: off-diagonal pairs t = l * world + rank, then its
  // diagonal chunk range [dq_lo, dq_hi) densest (highest) first
  const uint32_t npairs = g.st->npairs;
  const uint32_t noff = npairs > g.rank ? (npairs - g.rank + g.world - 1) / g.world : 0u;
  const uint32_t dq_lo = g.st->dq_lo, dq_hi = g.st->dq_hi;
  const uint32_t ntasks = noff + (dq_hi - dq_lo);
  const uint32_t ratio = g.scan_ratio;
  const uint32_t h0 = g.st->h0;  // pivots (i, j) with j < h0 cannot matter (see k_heavy_rank)
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned long long tri_local = 0;

  for (;;) {
    if (tid == 0) {
      s.task = atomicAdd(&g.st->task_next, 1u);
      s.next = 0;
      s.nstash = 0;
    }
#pragma unroll
    for (int e = 0; e < FPT; ++e) s.filt[tid * FPT + e] = 0;
    for (uint32_t b = tid; b < (uint32_t)kBuckets; b += kSupportThreads) {
      s.hcnt[b] = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) s.hkey[b][e] = 0;
    }
    __syncthreads();
    const uint32_t local = s.task;
    if (local >= ntasks) break;
    uint32_t q, q2;
    if (local < noff) {
      const uint2 pr = g.pairs[local * g.world + g.rank];
      q = pr.x;
      q2 = pr.y;
    } else {
      q = q2 = dq_hi - 1 - (local - noff);  // dense (high-rank) chunks first
    }
    const bool diag = q == q2;
    const uint64_t a0 = (uint64_t)q2 * kChunk;
    const uint32_t alen = (uint32_t)umin64(kChunk, g.slots - a0);
    const uint64_t p0 = (uint64_t)q * kChunk;
    const uint32_t plen = (uint32_t)umin64(kChunk, g.slots - p0);
    uint32_t pstart = 0;
    if (!diag) {
      const uint32_t rs = g.row_ptr[g.chunk_row[q]];
      pstart = rs > p0 ? (uint32_t)(rs - p0) : 0;
    }

    // 1. stage + zero counters
    uint32_t first_zero = 0xffffffffu;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t x = tid * EPT + e;
      const uint32_t v = x < alen ? col[a0 + x] : 0u;
      s.A[x] = v;
      s.cntA[x] = 0;
      if (v == 0 && x < alen && first_zero == 0xffffffffu) first_zero = x;
    }
    // next-zero: exclusive suffix-min of first_zero over higher threads; filter bits
    {
      uint32_t m = first_zero;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, m, o);
        if (lane + o < 32) m = min(m, y);
      }
      if (lane == 0) s.red[wid] = m;
      __syncthreads();
      uint32_t carry = 0xffffffffu;
      for (int w = wid + 1; w < NW; ++w) carry = min(carry, s.red[w]);
      const uint32_t incl_next = __shfl_down_sync(0xffffffffu, m, 1);
      if (lane < 31) carry = min(carry, incl_next);
      uint32_t cur = min(carry, alen);
#pragma unroll
      for (int e = EPT - 1; e >= 0; --e) {
        const uint32_t x = tid * EPT + e;
        const uint32_t v = s.A[x];
        if (x < alen && v == 0) cur = x;
        s.nz[x] = (uint16_t)min(cur, (uint32_t)kChunk);
        if (v != 0) {
          const uint32_t h = filt_hash(v, cur);
          atomicOr(&s.filt[h >> 5], 1u << (h & 31));
          const uint32_t b = bucket_of(v, cur);
          const uint32_t at = atomicAdd(&s.hcnt[b], 1u);
          const uint32_t meta = (cur << 16) | x;
          if (at < 8) {
            s.hkey[b][at] = v;
            s.hmeta[b][at] = meta;
          } else {
            const uint32_t z = atomicAdd(&s.nstash, 1u);
            if (z < kStash) {
              s.skey[z] = v;
              s.smeta[z] = meta;
            }
          }
        }
      }
    }
    __syncthreads();

    // 2. per-pivot descriptors
    uint32_t cost[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t x = tid * EPT + e;
      uint32_t c = 0;
      if (x >= pstart && x < plen) {
        const uint32_t j = diag ? s.A[x] : col[p0 + x];
        const uint32_t tb_ = diag ? x + 1 : 0;
        if (j >= h0 && j != 0 && tb_ < alen) {
          const uint32_t te_ = s.nz[tb_];
          if (te_ > tb_) {
            const uint32_t dj = g.deg[j];
            if (dj) {
              const uint32_t bs = g.row_ptr[j];
              uint32_t b0_ = bs, b1_ = bs + dj;
              if (dj > kClipMin) {
                b0_ = lb_global(col, bs, b1_, s.A[tb_]);
                b1_ = lb_global(col, b0_, b1_, s.A[te_ - 1] + 1);
              }
              const uint32_t blen = b1_ - b0_;
              if (blen) {
                const uint32_t tlen = te_ - tb_;
                const bool scan = blen <= tlen * ratio;
                c = scan ? blen : tlen;
                s.b0[x] = b0_;
                s.b1[x] = b1_;
                s.te[x] = (uint16_t)(te_ | (scan ? 0x8000u : 0u));
              }
            }
          }
        }
      }
      cost[e] = c;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) mine += cost[e];
    uint32_t W;
    uint32_t run = block_exscan(mine, s.red, &W);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      s.pref[tid * EPT + e] = run;
      run += cost[e];
    }
    if (tid == 0) s.pref[kChunk] = W;
    __syncthreads();
    if (!diag) {  // cntP aliases nz, which is dead from here on
#pragma unroll
      for (int e = 0; e < EPT; ++e) s.cntP[tid * EPT + e] = 0;
      __syncthreads();
    }

    // 3. flattened element work, strips grabbed dynamically by warps
    uint32_t* __restrict__ cntPiv = diag ? s.cntA : s.cntP;
    uint32_t* qk = s.qk[wid];
    uint32_t* qpos = s.qpos[wid];
    uint16_t* qp = s.qp[wid];
    uint32_t qn = 0;
    for (;;) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&s.next, (uint32_t)kStrip);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= W) break;
      const uint32_t lim = min(base + (uint32_t)kStrip, W);
      uint32_t p;
      {
        uint32_t lo = 0, hi = kChunk;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s.pref[mid + 1] <= base) lo = mid + 1; else hi = mid;
        }
        p = lo;
      }
      uint32_t pe = s.pref[p + 1], pb = s.pref[p];
      uint32_t db0 = s.b0[p], db1 = s.b1[p], dte = s.te[p];
      bool dscan = dte & 0x8000u;
      dte &= 0x7fffu;
      for (uint32_t f0 = base; f0 < lim; f0 += 32) {
        const uint32_t f = f0 + lane;
        bool pos_flag = false;
        uint32_t k = 0, pos = 0;
        if (f < lim) {
          if (f >= pe) {
            do {
              ++p;
              pe = s.pref[p + 1];
            } while (pe <= f);
            pb = s.pref[p];
            db0 = s.b0[p];
            db1 = s.b1[p];
            dte = s.te[p];
            dscan = dte & 0x8000u;
            dte &= 0x7fffu;
          }
          const uint32_t o = f - pb;
          if (dscan) {
            pos = db0 + o;
            k = col[pos];
            const uint32_t h = filt_hash(k, dte);
            pos_flag = (s.filt[h >> 5] >> (h & 31)) & 1u;
          } else {
            const uint32_t x = (diag ? p + 1 : 0) + o;
            const uint32_t kk = s.A[x];
            const uint32_t y = lb_global(col, db0, db1, kk);
            if (y < db1 && __ldg(col + y) == kk) {
              atomicAdd(&s.cntA[x], 1u);
              sadd(g, S, y, 1u);
              atomicAdd(&cntPiv[p], 1u);
              ++tri_local;
            }
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, pos_flag);
        if (pos_flag) {
          const uint32_t slot = qn + __popc(m & lt_mask);
          qk[slot] = k;
          qpos[slot] = pos;
          qp[slot] = (uint16_t)p;
        }
        qn += __popc(m);
        if (qn >= 32) {
          __syncwarp();
          const uint32_t e = qn - 32 + lane;
          tri_local += confirm(g, s, S, cntPiv, diag, qk[e], qpos[e], qp[e]);
          qn -= 32;
          __syncwarp();
        }
      }
    }
    __syncwarp();
    if (lane < qn) tri_local += confirm(g, s, S, cntPiv, diag, qk[lane], qpos[lane], qp[lane]);
    __syncthreads();

    // 4. flush smem counts
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t x = tid * EPT + e;
      const uint32_t ca = s.cntA[x];
      if (ca) sadd(g, S, a0 + x, ca);
      if (!diag) {
        const uint32_t cp = s.cntP[x];
        if (cp) sadd(g, S, p0 + x, cp);
      }
    }
    __syncthreads();
  }

  // triangle total (u64)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tri_local += __shfl_xor_sync(0xffffffffu, tri_local, o);
  if (lane == 0 && tri_local) atomicAdd(&g.st->triangles, tri_local);
}

// ---------------------------------------------------------------------------
// A22-staged support pass (working layout with the symmetric adjacency)
// ---------------------------------------------------------------------------
// The same triangles and increments as k_support_chunked, enumerated from the
// other side. In degree order the a12 tails are the short side of almost
// every intersection (R-MAT s20: sum of tails 1.23e9 against 4.42e9 A22-row
// elements), so a task stages a 512-slot chunk of A22 rows N+(j) in shared
// memory -- hashed by (value, row run) -- and streams the tail of every pivot
// (i, j) whose j has a run in the chunk, probing each tail element once.
// Pivots come from a static in-edge list (edge ids grouped by j); the
// current slot of a pivot is pos_of[id] and dead ids are skipped, so the list
// never needs rebuilding as rounds prune. A triangle (i, j, c) adds 1 to the
// A22 slot (j, c) and the pivot (i, j) in shared memory and red.adds the tail
// slot (i, c) once. Tasks are (chunk, batch of kA22Batch pivots), static.
#ifndef KTG_A22_UNROLL
#define KTG_A22_UNROLL 4
#endif
constexpr int kA22Batch = 256;
#ifndef KTG_A22_LIGHT
#define KTG_A22_LIGHT 1    // round-0 light pivots skip their increments
#endif
#ifndef KTG_A22_TABLE
// 1,920 slots (load <= 0.27): with the aliased step-1/2 arrays the CTA needs
// 26.7 KB, so 6 CTAs fit the 164 KB shared-memory carveout and L1 keeps 92 KB
// for the re-read tail rows (2,048 slots cross into the 196 KB carveout:
// 163 vs 155 ms per s24 pass; 1,216 with the 132 KB carveout: 163 ms)
#define KTG_A22_TABLE 1920
#endif
#ifndef KTG_A22_UNION
#define KTG_A22_UNION 1
#endif
constexpr int kA22TableBits = 11;          // top hash bits when the table size is a power of two
#ifndef KTG_A22_STRIP
#define KTG_A22_STRIP 512
#endif
constexpr int kA22Strip = KTG_A22_STRIP;   // flat tail elements a warp takes per grab (at most)
#ifndef KTG_A22_STRIP_ADAPT
#define KTG_A22_STRIP_ADAPT 1  // strips halve (down to 128) while a batch has < 4 per warp (balance at the barrier)
#endif
constexpr int kA22Table = KTG_A22_TABLE;     // slots (a power of two uses the top hash bits)
constexpr int kA22Unroll = KTG_A22_UNROLL;     // tail elements per lane per step (loads in flight)
constexpr int kA22FiltWords = 512;         // 16K filter bits for <= 512 entries (~3% false positives)

struct A22 {
  const uint32_t* pe;        // in-edge ids, grouped by j (pristine in-lists)
  const uint2* pin_p;        // the same pivots in the pristine graph: {slot, row i}
  const uint32_t* pin_end;   // ... and the end of row i's live part (its tail end)
  const uint32_t* pin_off;   // n+2: start of j's in-list in pe
  const uint32_t* jfirst;    // per chunk: row holding the chunk's first slot
  const uint2* tasks;        // (chunk, batch)
  uint32_t ntasks;
};

struct A22Smem {
#if KTG_A22_UNION
  // steps 1-2 only (rte, roff) alias step 3+ only (A, filt): dead before the
  // staging starts, so the CTA stays under the shared-memory size that leaves
  // the most L1 for the re-read tails at 6 CTAs per SM
  union {
    uint32_t rte[kChunk + 2];        // per row of the chunk: run [tb, te) as tb << 16 | te, or ~0
    uint32_t A[kChunk];
  };
  union {
    uint32_t roff[kChunk + 2];       // pin_off of the chunk's rows (+1)
    uint32_t filt[kA22FiltWords];    // membership bits of (value, run end): most misses stop here
  };
  uint32_t cntA[kChunk];
#else
  uint32_t A[kChunk];
  uint32_t cntA[kChunk];
  uint32_t rte[kChunk + 2];          // per row of the chunk: run [tb, te) as tb << 16 | te, or ~0
  uint32_t roff[kChunk + 2];         // pin_off of the chunk's rows (+1)
#endif
  uint32_t ps[kA22Batch];            // pivot slot (i, j)
  uint32_t plo[kA22Batch];           // first tail slot probed
  uint32_t prun[kA22Batch];          // j's run tb << 16 | te
  uint32_t cntP[kA22Batch];
  uint32_t pref[kA22Batch + 1];
#if !KTG_A22_UNION
  uint32_t filt[kA22FiltWords];      // membership bits of (value, run end): most misses stop here
#endif
  uint2 tab[kA22Table];              // open addressing: {value (0 = empty), chunk position}
  uint32_t red[kSupportThreads / 32];
  uint32_t task;
  uint32_t next;
};

// Shared-memory accesses of the probe loop by 32-bit shared-window address
// (base = the static A22Smem's cvta offset, a uniform constant). Through the
// lambdas' generic references the compiler rebuilt the window base with an
// S2R SR_CgaCtaId + LEA before every filter / table / counter access of the
// probe path (20 S2R in the kernel, each a short-scoreboard round trip).
#ifndef KTG_A22_ASMSMEM
#define KTG_A22_ASMSMEM 1
#endif
// The static A22Smem is the kernel's only shared variable: it starts right
// after the 1 KB the hardware reserves, and a launch without clusters has CTA
// id 0 in its cluster, so its shared-window address is this constant (the
// kernel traps if not). A literal keeps the compiler from rebuilding it.
constexpr uint32_t kA22SmemBase = 0x400;
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void reds_inc(uint32_t a) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a) : "memory");
}

// One multiplicative hash of (value, run end): the table slot takes its top
// kA22TableBits bits, the filter bit a fold of the rest.
__device__ __forceinline__ uint32_t a22_mix(uint32_t v, uint32_t te) {
  return (v ^ (te * 0x85EBCA6Bu)) * 2654435761u;
}
__device__ __forceinline__ uint32_t a22_slot(uint32_t h) {
  if ((kA22Table & (kA22Table - 1)) == 0) return h >> (32 - kA22TableBits);
  return (uint32_t)(((uint64_t)h * kA22Table) >> 32);  // range reduction for other sizes
}
__device__ __forceinline__ uint32_t a22_next(uint32_t h) {
  if ((kA22Table & (kA22Table - 1)) == 0) return (h + 1) & (kA22Table - 1);
  return h + 1 == (uint32_t)kA22Table ? 0u : h + 1;
}
__device__ __forceinline__ uint32_t a22_fbit(uint32_t h) { return (h ^ (h >> 15)) & (kA22FiltWords * 32 - 1); }
// KTG_A22_HASH2: the same (value, run end) key hashed with one IMAD per tail
// element. The run word's contribution rk = run * kA22RunMul keeps only the
// run end te (bits 0-15: kA22RunMul is a multiple of 2^16, so the tb / flag
// bits vanish) and is formed once per pivot in the advance; h = c * kA22Mul +
// rk. Filter word = top 9 bits, bit 31 - (h & 31) (the funnel shift's own wrap); the
// positive path re-reads the pivot's run word for tb / te / the light flag.
// (The old mix: 4 instructions for the key, 6 for the filter bit.)
#ifndef KTG_A22_HASH2
#define KTG_A22_HASH2 1
#endif
#ifndef KTG_A22_UNILOOP
#define KTG_A22_UNILOOP 1  // step loop with a warp-uniform trip count (lanes past lim carry out-of-range elements)
#endif
#if KTG_A22_HASH2 && !KTG_A22_ASMSMEM
#error "KTG_A22_HASH2 is implemented on the KTG_A22_ASMSMEM probe path"
#endif
constexpr uint32_t kA22Mul = 2654435761u;
constexpr uint32_t kA22RunMul = ((0x85EBCA6Bu * 2654435761u) & 0xffffu) << 16;  // odd << 16: te -> bijective offset
static_assert(kA22FiltWords == 512, "HASH2 takes the filter word from the top 9 hash bits");
__device__ __forceinline__ uint32_t a22_h2(uint32_t v, uint32_t rk) { return v * kA22Mul + rk; }

// COST = true (multi-rank runs, before every full pass): steps 1-2 only, over
// all tasks; wcost[t] = the task's flattened tail work W, the weights of the
// work-balanced split of the tasks across ranks (k_a22_split).
#ifndef KTG_A22_MINB
#define KTG_A22_MINB 6
#endif
template <bool COST>
__global__ void __launch_bounds__(kSupportThreads, KTG_A22_MINB)  // 6 CTAs/SM (smem-bound): <= 40 registers
k_support_a22(Graph g, Sym y, A22 a, unsigned long long* __restrict__ wcost) {
  if (g.st->mode) return;  // supports carried this round
  // static (not dynamic) shared memory: constant-offset LDS addressing
  __shared__ __align__(16) A22Smem s;
  const uint32_t tid = threadIdx.x;
#if KTG_A22_ASMSMEM
  if (tid == 0 && (uint32_t)__cvta_generic_to_shared(&s) != kA22SmemBase) __trap();
#endif
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kSupportThreads / 32;
  constexpr int EPT = kChunk / kSupportThreads;
  uint32_t* __restrict__ S = cur_S(g);
  const uint32_t* __restrict__ col = g.col;
  const uint32_t h0 = g.st->h0;
  const bool pristine = g.st->pristine;
  unsigned long long tri_local = 0;
  auto claim = [&]() {  // (thread 0) the CTA's next task into s.task, s.next = 0
    // multi-rank runs: this rank's contiguous, work-balanced task range
    const bool part = g.world > 1 && !COST;
    const uint32_t tt = atomicAdd(&g.st->task_next, 1u) + (part ? g.a22_lo : 0u);
    s.task = tt < (part ? g.a22_hi : a.ntasks) ? tt : 0xffffffffu;
    s.next = 0;
  };

  for (;;) {
    if (tid == 0) claim();
    __syncthreads();
    const uint32_t t = s.task;
    if (t == 0xffffffffu) break;
    const uint2 tk = a.tasks[a.ntasks - 1 - t];  // dense (high-rank) chunks first
    const uint32_t q = tk.x;
    const uint64_t a0 = (uint64_t)q * kChunk;
    const uint32_t alen = (uint32_t)umin64(kChunk, g.slots - a0);
    const uint32_t jf = a.jfirst[q], jl = g.chunk_row[q];
    const uint32_t nrows = jl - jf + 1;

    // 1. rows of the chunk (live run inside the chunk, in-list offsets) and
    //    the batch's pivot descriptors, before anything is staged: batches
    //    whose pivots are all dead cost only this
    for (uint32_t r = tid; r <= nrows; r += kSupportThreads) {
      const uint32_t j = jf + r;
      s.roff[r] = a.pin_off[j];
      if (r < nrows) {
        const uint64_t rb = g.row_ptr[j], re = rb + g.deg[j];
        const uint64_t lo = rb > a0 ? rb : a0, hi = re < a0 + alen ? re : a0 + alen;
        // tb << 16 | te, bit 30: j's row continues outside the chunk (its
        // pivots' tails get clipped to the run's value range)
        s.rte[r] = (lo < hi && j >= h0 && j != 0)
                       ? (uint32_t)((lo - a0) << 16 | (hi - a0)) | ((rb < a0 || re > a0 + alen) ? 0x40000000u : 0u)
                       : 0xffffffffu;
      }
    }
    __syncthreads();

    // 2. pivot descriptors of this batch: slot, tail (clipped to the run's
    //    value range when j's row continues outside the chunk)
    const uint32_t k0 = s.roff[0] + tk.y * kA22Batch;
    const uint32_t k1 = min(k0 + kA22Batch, s.roff[nrows]);
    uint32_t cost = 0;
    s.cntP[tid] = 0;
    if (k0 + tid < k1) {
      const uint32_t k = k0 + tid;
      // row of pivot k: last r with roff[r] <= k
      uint32_t lo = 0, hi = nrows;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s.roff[mid] <= k) lo = mid; else hi = mid;
      }
      const uint32_t run = s.rte[lo];
      bool live = false;
      uint32_t ps = 0, i = 0, iend = 0;
      if (run != 0xffffffffu) {
        if (pristine) {  // static {slot, row} and row end: no dead / pos_of / erow / row gathers
          const uint2 pv = a.pin_p[k];
          ps = pv.x, i = pv.y, live = true;
          iend = a.pin_end[k];
        } else {
          const uint32_t id = a.pe[k];
          live = !y.dead[id];
          if (live) {
            ps = y.pos_of[id], i = y.erow[id];
            iend = g.row_ptr[i] + g.deg[i];
          }
        }
      }
      if (live) {
        uint32_t tlo = ps + 1, thi = iend;
        const uint32_t tb = (run >> 16) & 0x3fffu, te = run & 0xffffu;
        if (run & 0x40000000u) {  // partial run: clip the tail
          tlo = lb_global(col, tlo, thi, col[a0 + tb]);
          thi = lb_global(col, tlo, thi, col[a0 + te - 1] + 1);
        }
        if (thi > tlo) {
          cost = thi - tlo;
          s.ps[tid] = ps;
          s.plo[tid] = tlo;
          // pristine round 0 with the degree bound: rows below h0 go in this
          // round whatever their counts (k_mark), so the pivot (i, j) and its
          // tail slots (i, c) need no increments; bit 31 of the run marks it
          s.prun[tid] = run | ((KTG_A22_LIGHT && i < h0) ? 0x80000000u : 0u);
        }
      }
    }
    uint32_t W;
    const uint32_t run0 = block_exscan(cost, s.red, &W);
    s.pref[tid] = run0;
    if (tid == 0) s.pref[kA22Batch] = W;
    if (COST) {
      if (tid == 0) wcost[t] = W;
      continue;
    }
    if (W == 0) continue;  // no live pivot reaches this chunk (uniform; nothing staged yet)

    // 3. stage the chunk, next zeros, (value, run end) hash -- as k_support_chunked
    for (uint32_t b = tid; b < (uint32_t)kA22Table; b += kSupportThreads) s.tab[b] = make_uint2(0, 0);
    for (uint32_t b = tid; b < (uint32_t)kA22FiltWords; b += kSupportThreads) s.filt[b] = 0;
    uint32_t first_zero = 0xffffffffu;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t x = tid * EPT + e;
      const uint32_t v = x < alen ? col[a0 + x] : 0u;
      s.A[x] = v;
      s.cntA[x] = 0;
      if (v == 0 && x < alen && first_zero == 0xffffffffu) first_zero = x;
    }
    {
      uint32_t m = first_zero;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, m, o);
        if (lane + o < 32) m = min(m, v);
      }
      if (lane == 0) s.red[wid] = m;
      __syncthreads();
      uint32_t carry = 0xffffffffu;
      for (int w = wid + 1; w < NW; ++w) carry = min(carry, s.red[w]);
      const uint32_t incl_next = __shfl_down_sync(0xffffffffu, m, 1);
      if (lane < 31) carry = min(carry, incl_next);
      uint32_t cur = min(carry, alen);
#pragma unroll
      for (int e = EPT - 1; e >= 0; --e) {
        const uint32_t x = tid * EPT + e;
        const uint32_t v = s.A[x];
        if (x < alen && v == 0) cur = x;
        if (v != 0) {  // claim the first free slot from home (values are >= 1)
#if KTG_A22_HASH2
          const uint32_t hh = a22_h2(v, cur * kA22RunMul);
          atomicOr(&s.filt[hh >> 23], 0x80000000u >> (hh & 31));
#else
          const uint32_t hh = a22_mix(v, cur);
          const uint32_t fb = a22_fbit(hh);
          atomicOr(&s.filt[fb >> 5], 1u << (fb & 31));
#endif
          uint32_t h = a22_slot(hh);
          while (atomicCAS(&s.tab[h].x, 0u, v) != 0u) h = a22_next(h);
#if KTG_A22_HASH2
          // payload: x's byte offset in cntA | its run's rk (te * kA22RunMul,
          // bits 16-31) -- a probe matches on (value, rk) without the run bounds
          s.tab[h].y = (x << 2) | (cur * kA22RunMul);
#else
          s.tab[h].y = x;
#endif
        }
      }
    }
    __syncthreads();

    // 4. flattened tail elements, strips grabbed dynamically by warps
    uint32_t tri_task = 0;
    for (;;) {
      uint32_t base = 0;
      // (short batches: half strips, so the 8 warps reach the barrier together)
      // (big batches: 512-element strips, fewer grabs and pivot searches)
      uint32_t strip = kA22Strip;
      if (KTG_A22_STRIP_ADAPT)
        while (strip > 128u && W < 4u * NW * strip) strip >>= 1;
      if (lane == 0) base = atomicAdd(&s.next, strip);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= W) break;
      const uint32_t lim = min(base + strip, W);
      // pivot holding base: p = #{q in [1, kA22Batch) : pref[q] <= base}
      // (pref ascends), two ballots over groups of 8 instead of a search
      static_assert(kA22Batch == 256, "two-level ballot assumes 32 groups of 8");
      uint32_t p;
      {
        const uint32_t g = __popc(__ballot_sync(0xffffffffu, lane < 31 && s.pref[8 * (lane + 1)] <= base));
        const uint32_t c2 = __popc(__ballot_sync(0xffffffffu, lane < 7 && s.pref[8 * g + 1 + lane] <= base));
        p = 8 * g + c2;
      }
      uint32_t pe_ = s.pref[p + 1], pb = s.pref[p], plo = s.plo[p], prun = s.prun[p];
#if KTG_A22_ASMSMEM
      constexpr uint32_t sb = kA22SmemBase;  // checked against &s at kernel entry
      constexpr uint32_t oF = offsetof(A22Smem, filt), oT = offsetof(A22Smem, tab), oA = offsetof(A22Smem, cntA),
                         oP = offsetof(A22Smem, cntP), oR = offsetof(A22Smem, pref), oL = offsetof(A22Smem, plo),
                         oU = offsetof(A22Smem, prun);
#if KTG_A22_HASH2
      // table probe of a filter hit: tail element c (hash hh) of the pivot
      // pl (index | light flag << 31). The entry matches on its value and its
      // run's rk = hh - c * kA22Mul: inside one chunk a value's run end
      // identifies its row (runs are the maximal nonzero stretches). The
      // triangle count comes from the cntA flush.
      auto probe = [&](uint32_t c, uint32_t slot, uint32_t hh, uint32_t rk, uint32_t pl) {
        for (uint32_t h = a22_slot(hh);; h = a22_next(h)) {
          const uint2 e = lds_v2(sb + oT + (h << 3));
          if (e.x == 0) break;
          if (e.x == c && (e.y ^ rk) < 0x10000u) {
            reds_inc(sb + oA + (e.y & 0xffffu));
            if (!KTG_A22_LIGHT || (int32_t)pl >= 0) {
              atomicAdd(&S[slot], 1u);
              reds_inc(sb + oP + (pl << 2));  // (the flag shifts out)
            }
            break;
          }
        }
      };
#else
      auto probe = [&](uint32_t c, uint32_t slot, uint32_t run, uint32_t pp) {
        const uint32_t tb = (run >> 16) & 0x3fffu, te = run & 0xffffu;
        const uint32_t hh = a22_mix(c, te);
        const uint32_t fb = a22_fbit(hh);
        if (lds_u32(sb + oF + ((fb >> 5) << 2)) & (1u << (fb & 31))) {
          uint32_t x = kChunk;
          for (uint32_t h = a22_slot(hh);; h = a22_next(h)) {
            const uint2 e = lds_v2(sb + oT + (h << 3));
            if (e.x == 0) break;
            if (e.x == c && e.y - tb < te - tb) {
              x = e.y;
              break;
            }
          }
          if (x < (uint32_t)kChunk) {
            reds_inc(sb + oA + (x << 2));
            if (!KTG_A22_LIGHT || !(run >> 31)) {
              atomicAdd(&S[slot], 1u);
              reds_inc(sb + oP + (pp << 2));
            }
            ++tri_task;
          }
        }
      };
#endif
#if KTG_A22_HASH2
      // p carries the pivot's light flag in bit 31 (its run word's bit 31:
      // round-0 rows below h0) and prun the pivot's rk from here on
      p |= prun & 0x80000000u;
      prun *= kA22RunMul;
      auto advance = [&](uint32_t f) {
        if (f >= pe_) {
          p &= 0x7fffffffu;
          do {
            ++p;
            pe_ = lds_u32(sb + oR + ((p + 1) << 2));
          } while (pe_ <= f);
          pb = lds_u32(sb + oR + (p << 2));
          plo = lds_u32(sb + oL + (p << 2));
          prun = lds_u32(sb + oU + (p << 2));
          p |= prun & 0x80000000u;
          prun *= kA22RunMul;
        }
      };
#else
      auto advance = [&](uint32_t f) {
        if (f >= pe_) {
          do {
            ++p;
            pe_ = lds_u32(sb + oR + ((p + 1) << 2));
          } while (pe_ <= f);
          pb = lds_u32(sb + oR + (p << 2));
          plo = lds_u32(sb + oL + (p << 2));
          prun = lds_u32(sb + oU + (p << 2));
        }
      };
#endif
#else
      // (value, run) lookup of tail element c of pivot pp: the value may also
      // sit in other rows' runs
      auto probe = [&](uint32_t c, uint32_t slot, uint32_t run, uint32_t pp) {
        const uint32_t tb = (run >> 16) & 0x3fffu, te = run & 0xffffu;
        const uint32_t hh = a22_mix(c, te);
        const uint32_t fb = a22_fbit(hh);
        if (s.filt[fb >> 5] & (1u << (fb & 31))) {
          uint32_t x = kChunk;
          for (uint32_t h = a22_slot(hh);; h = a22_next(h)) {
            const uint2 e = s.tab[h];
            if (e.x == 0) break;
            if (e.x == c && e.y - tb < te - tb) {
              x = e.y;
              break;
            }
          }
          if (x < (uint32_t)kChunk) {
            atomicAdd(&s.cntA[x], 1u);
            if (!KTG_A22_LIGHT || !(run >> 31)) {
              atomicAdd(&S[slot], 1u);
              atomicAdd(&s.cntP[pp], 1u);
            }
            ++tri_task;
          }
        }
      };
      auto advance = [&](uint32_t f) {
        if (f >= pe_) {
          do {
            ++p;
            pe_ = s.pref[p + 1];
          } while (pe_ <= f);
          pb = s.pref[p];
          plo = s.plo[p];
          prun = s.prun[p];
        }
      };
#endif
      // kA22Unroll elements per lane per step, every load issued before any probe
#if KTG_A22_HASH2
      auto step = [&](const uint32_t f) {
        uint32_t sl[kA22Unroll], ru[kA22Unroll], pv[kA22Unroll], cv[kA22Unroll];
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u) {
          const uint32_t fu = f + 32 * u;
          if (fu < lim) advance(fu);
          sl[u] = plo + (fu - pb), ru[u] = prun, pv[u] = p;
        }
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u) cv[u] = (f + 32 * u < lim) ? col[sl[u]] : 0u;
        // the kA22Unroll hashes and filter reads as independent chains (the
        // filter bit 31 - (h & 31) lands in the sign: one funnel shift and a
        // sign test); only the hits go on to the table probe
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u) ru[u] = a22_h2(cv[u], ru[u]);
        bool hit[kA22Unroll];
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u) {
          const uint32_t w = lds_u32(sb + oF + ((ru[u] >> 23) << 2));
          hit[u] = f + 32 * u < lim && (int32_t)__funnelshift_l(0u, w, ru[u]) < 0;
        }
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u)
          if (hit[u]) probe(cv[u], sl[u], ru[u], ru[u] - cv[u] * kA22Mul, pv[u]);

      };
#if KTG_A22_UNILOOP
      for (uint32_t f0 = base; f0 < lim; f0 += 32 * kA22Unroll) step(f0 + lane);  // warp-uniform trip count
#else
      for (uint32_t f = base + lane; f < lim; f += 32 * kA22Unroll) step(f);
#endif
#else
      for (uint32_t f = base + lane; f < lim; f += 32 * kA22Unroll) {
        uint32_t sl[kA22Unroll], ru[kA22Unroll], pv[kA22Unroll], cv[kA22Unroll];
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u) {
          const uint32_t fu = f + 32 * u;
          if (fu < lim) advance(fu);
          sl[u] = plo + (fu - pb), ru[u] = prun, pv[u] = p;
        }
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u) cv[u] = (f + 32 * u < lim) ? col[sl[u]] : 0u;
#pragma unroll
        for (int u = 0; u < kA22Unroll; ++u)
          if (f + 32 * u < lim) probe(cv[u], sl[u], ru[u], pv[u]);
      }
#endif
    }
    tri_local += tri_task;
    __syncthreads();

    // 5. flush shared counts (A22 slots, pivots); every triangle found bumped
    //    exactly one A22 count (the HASH2 probe counts triangles here)
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t x = tid * EPT + e;
      const uint32_t ca = s.cntA[x];
      if (ca) atomicAdd(&S[a0 + x], ca);
      if (KTG_A22_HASH2) tri_local += ca;
    }
    {
      const uint32_t cp = s.cntP[tid];
      if (cp) atomicAdd(&S[s.ps[tid]], cp);
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tri_local += __shfl_xor_sync(0xffffffffu, tri_local, o);
  if (lane == 0 && tri_local) atomicAdd(&g.st->triangles, tri_local);
}

// Load time: row holding each chunk's first slot.
__global__ void k_chunk_first(const uint32_t* __restrict__ row_ptr, uint32_t n, uint64_t slots, uint32_t nchunks,
                              uint32_t* __restrict__ jfirst) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nchunks) return;
  const uint32_t e = (uint32_t)((uint64_t)q * kChunk);
  uint32_t lo = 0, hi = n + 2;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= e) lo = mid + 1; else hi = mid;
  }
  jfirst[q] = max(lo - 1, 1u);
}

// Load time: batches per chunk (pivots into the chunk's rows / kA22Batch).
__global__ void k_a22_count(const uint32_t* __restrict__ jfirst, const uint32_t* __restrict__ chunk_row,
                            const uint32_t* __restrict__ pin_off, uint32_t nchunks, uint32_t* __restrict__ cnt) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q > nchunks) return;
  if (q == nchunks) {
    cnt[q] = 0;
    return;
  }
  const uint32_t k0 = pin_off[jfirst[q]], k1 = pin_off[chunk_row[q] + 1];
  cnt[q] = (k1 - k0 + kA22Batch - 1) / kA22Batch;
}

__global__ void k_a22_fill(const uint32_t* __restrict__ cnt_off, uint32_t nchunks, uint2* __restrict__ tasks) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nchunks) return;
  const uint32_t o = cnt_off[q], c = cnt_off[q + 1] - o;
  for (uint32_t b = 0; b < c; ++b) tasks[o + b] = make_uint2(q, b);
}

// Multi-rank split, computed once per load on the pristine
// graph (round 0 dominates every fixpoint): rank r takes the contiguous tasks
// [lo, hi) whose exclusive work prefix pre[t] (over k_support_a22<true>'s
// costs, pre[ntasks] = total) falls in [total*r/world, total*(r+1)/world);
// every rank computes the same split from the same replicated state.
__global__ void k_a22_split(DevState* st, const unsigned long long* __restrict__ pre, uint32_t ntasks,
                            uint32_t rank, uint32_t world) {
  const unsigned long long total = pre[ntasks];
  auto first_at = [&](unsigned long long bound) {  // first t with pre[t] >= bound
    uint32_t lo = 0, hi = ntasks;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pre[mid] < bound) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const unsigned long long b0 = (unsigned long long)((__uint128_t)total * rank / world);
  const unsigned long long b1 = (unsigned long long)((__uint128_t)total * (rank + 1) / world);
  st->a22_lo = rank == 0 ? 0u : first_at(b0);
  st->a22_hi = rank + 1 == world ? ntasks : first_at(b1);
  st->task_next = 0;
}

// Paper Listing 1 / support.cpp:115-127 as written: one thread per slot,
// sequential two-pointer merge. Cross-check kernel only.
__global__ void k_support_naive(Graph g) {
  uint32_t* __restrict__ S = cur_S(g);
  const uint32_t* __restrict__ col = g.col;
  unsigned long long tri = 0;
  for (uint64_t slot = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; slot < g.slots;
       slot += (uint64_t)gridDim.x * blockDim.x) {
    if ((slot % g.world) != g.rank) continue;
    const uint32_t pred = col[slot];
    if (pred == 0) continue;
    uint32_t a = (uint32_t)slot + 1, b = g.row_ptr[pred], found = 0;
    uint32_t ca = col[a], cb = col[b];
    while (ca != 0 && cb != 0) {
      if (ca == cb) {
        atomicAdd(&S[a], 1u);
        atomicAdd(&S[b], 1u);
        ++found;
        ca = col[++a];
        cb = col[++b];
      } else if (cb > ca) {
        ca = col[++a];
      } else {
        cb = col[++b];
      }
    }
    if (found) atomicAdd(&S[slot], found);
    tri += found;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tri += __shfl_xor_sync(0xffffffffu, tri, o);
  if ((threadIdx.x & 31) == 0 && tri) atomicAdd(&g.st->triangles, tri);
}

// intersect_tails for one pivot (support.cpp:64-91), as written: the
// single-slot unit-test surface of the reference API.
__global__ void k_intersect_one(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                                uint32_t* __restrict__ S, uint32_t pivot, uint32_t pred, uint32_t* found) {
  uint32_t a = pivot + 1, b = row_ptr[pred], f = 0;
  while (col[a] != 0 && col[b] != 0) {
    if (col[a] == col[b]) {
      atomicAdd(&S[a], 1u);
      atomicAdd(&S[b], 1u);
      ++f;
      ++a;
      ++b;
    } else if (col[b] > col[a]) {
      ++a;
    } else {
      ++b;
    }
  }
  *found = f;
}

// First slot whose support exceeds 65535 (check_16bit, support.cpp:53-60),
// in the CALLER's slot numbering (payload maps working slots back), packed
// as slot << 32 | count so one atomicMin keeps the reference's first slot.
__global__ void k_check16(Graph g) {
  const uint32_t* __restrict__ S = cur_S(g);
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < g.slots;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = S[x];
    if (v > 0xFFFFu) {
      const unsigned long long slot = g.payload ? g.payload[x] : x;
      atomicMin(&g.st->overflow_slot, (slot << 32) | v);
      g.st->error = 1;
    }
  }
}

__global__ void k_max_support(Graph g) {
  const uint32_t* __restrict__ S = cur_S(g);
  uint32_t m = 0;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < g.slots;
       x += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, S[x]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&g.st->max_support, m);
}

// ---------------------------------------------------------------------------
// Prune (truss.cpp:9-37) fused with the next round's support reset
// ---------------------------------------------------------------------------
// Per row: stable compaction of live slots with S >= k-2 (ballot + popc),
// zero-fill of the vacated tail, new live degree. With `fused_reset`:
//   * the other support buffer (next round's) is zeroed over the row's live
//     prefix -- the only slots the previous round could have written, since
//     this row's vacated tail was zeroed when it was vacated;
//   * the current buffer is zeroed over the vacated tail (a round that removes
//     anything is not the converged one, so those counts are never returned).
// Without it (host loop / observer) S is left untouched, as in the reference.
// MODE 0 (prune): keep live slots with S >= k-2; the optional payload (slot
// ids of the working layout) moves with col.
// MODE 1 (publish): keep slots whose col is nonzero, moving S0 along -- the
// caller-layout compaction after a degree-ordered fixpoint (see ktg_engine.cu).
template <int MODE>
__global__ void __launch_bounds__(kPruneThreads)
k_prune_light(Graph g, int fused_reset) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t* __restrict__ S = MODE ? g.S0 : cur_S(g);
  uint32_t* __restrict__ So = other_S(g);
  uint32_t* __restrict__ col = g.col;
  uint32_t* __restrict__ pay = g.payload;
  const uint32_t thr = g.st->threshold;
  unsigned long long removed = 0;
  for (uint32_t v = warp + 1; v <= g.n; v += nwarps) {
    const uint32_t d = g.deg[v];
    if (d == 0) continue;
    if (d > (uint32_t)kHeavyRow) {
      if (lane == 0) {
        const uint32_t at = atomicAdd(&g.st->nheavy, 1u);
        g.heavy_rows[at] = v;
      }
      continue;
    }
    const uint32_t base = g.row_ptr[v];
    uint32_t write = 0;
    for (uint32_t off = 0; off < d; off += 32) {
      const uint32_t idx = off + lane;
      const bool live = idx < d;
      const uint32_t c = live ? col[base + idx] : 0u;
      const uint32_t sv = live ? S[base + idx] : 0u;
      const uint32_t pv = (live && pay) ? pay[base + idx] : 0u;
      const bool keep = MODE ? (live && c != 0) : (live && sv >= thr);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      __syncwarp();  // every lane's loads precede any lane's in-place store
      const uint32_t at = base + write + __popc(m & ((1u << lane) - 1u));
      if (keep) {
        col[at] = c;
        if (MODE) S[at] = sv;
        if (pay) pay[at] = pv;
      }
      if (!MODE && fused_reset && live) So[base + idx] = 0;
      write += __popc(m);
    }
    for (uint32_t x = write + lane; x < d; x += 32) {
      col[base + x] = 0;
      if (MODE || fused_reset) S[base + x] = 0;
    }
    if (lane == 0) {
      g.deg[v] = write;
      removed += d - write;
    }
  }
  if (!MODE && lane == 0 && removed) atomicAdd(&g.st->removed, removed);
}

// CTA per heavy row (queued by k_prune_light): same compaction with a
// block-wide scan over tiles of 4 * kPruneThreads slots.
template <int MODE>
__global__ void __launch_bounds__(kSymHeavyThreads)
k_prune_heavy(Graph g, int fused_reset) {
  __shared__ uint32_t red[kSymHeavyThreads / 32];
  __shared__ uint32_t tot_s;
  constexpr int EPT = 4;
  constexpr int TILE = EPT * kSymHeavyThreads;
  const uint32_t tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kSymHeavyThreads / 32;
  uint32_t* __restrict__ S = MODE ? g.S0 : cur_S(g);
  uint32_t* __restrict__ So = other_S(g);
  uint32_t* __restrict__ col = g.col;
  uint32_t* __restrict__ pay = g.payload;
  const uint32_t thr = g.st->threshold;
  const uint32_t nheavy = g.st->nheavy;
  unsigned long long removed = 0;
  for (uint32_t h = blockIdx.x; h < nheavy; h += gridDim.x) {
    const uint32_t v = g.heavy_rows[h];
    const uint32_t d = g.deg[v];
    const uint32_t base = g.row_ptr[v];
    uint32_t write = 0;
    for (uint32_t off = 0; off < d; off += TILE) {
      uint32_t c[EPT], sv[EPT], pv[EPT];
      bool keep[EPT];
      uint32_t cnt = 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const uint32_t idx = off + tid * EPT + e;
        const bool live = idx < d;
        c[e] = live ? col[base + idx] : 0u;
        sv[e] = live ? S[base + idx] : 0u;
        pv[e] = (live && pay) ? pay[base + idx] : 0u;
        keep[e] = MODE ? (live && c[e] != 0) : (live && sv[e] >= thr);
        cnt += keep[e];
        if (!MODE && fused_reset && live) So[base + idx] = 0;
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) red[wid] = x;
      __syncthreads();  // also: every thread has read its tile before writes
      if (wid == 0) {
        uint32_t w = lane < NW ? red[lane] : 0;
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += y;
        }
        if (lane < NW) red[lane] = w;
        if (lane == NW - 1) tot_s = w;
      }
      __syncthreads();
      uint32_t pos = write + x - cnt + (wid ? red[wid - 1] : 0);
#pragma unroll
      for (int e = 0; e < EPT; ++e)
        if (keep[e]) {
          col[base + pos] = c[e];
          if (MODE) S[base + pos] = sv[e];
          if (pay) pay[base + pos] = pv[e];
          ++pos;
        }
      write += tot_s;
      __syncthreads();
    }
    for (uint32_t x = write + tid; x < d; x += blockDim.x) {
      col[base + x] = 0;
      if (MODE || fused_reset) S[base + x] = 0;
    }
    if (tid == 0) {
      g.deg[v] = write;
      removed += d - write;
    }
    __syncthreads();
  }
  if (!MODE && tid == 0 && removed) atomicAdd(&g.st->removed, removed);
}

// ---------------------------------------------------------------------------
// Incremental rounds (working layout): carry supports across rounds
// ---------------------------------------------------------------------------
// A round's supports S_r are exact for the round's graph G_r. Instead of
// recomputing S_{r+1} from scratch, every triangle of G_r that loses an edge
// in round r is found once from one of its removed edges and the surviving
// edges of that triangle lose 1. What is left is exactly the support in
// G_{r+1} -- the same integers the reference's reset + computeSupports
// produces (truss.cpp:44-46), so (col, S, removed per round) stay
// bit-identical; only the work changes. Per round the device picks the
// cheaper of carrying (delta_cost) and a full pass on the survivors
// (keep_cost), see k_decide.
//
// Round r, mode 0 (after a full support pass): k_mark scans every live edge.
// Round r, mode 1 (supports carried from r-1): the removals are exactly the
// edges whose carried support crossed below k-2 during r-1's k_delta, which
// queued them (frontier); k_mark_frontier handles only those. Rows that lose
// an edge are queued once (flag bits) for compaction, so a round costs
// O(removed + their triangles), not O(m).

// Append val to a global queue; one atomic per group of threads that reach
// the call together (queues are filled from divergent code).
__device__ __forceinline__ void append_coalesced(uint32_t* cnt, uint32_t* q, uint32_t val) {
  namespace cg = cooperative_groups;
  cg::coalesced_group grp = cg::coalesced_threads();
  uint32_t base = 0;
  if (grp.thread_rank() == 0) base = atomicAdd(cnt, grp.size());
  base = grp.shfl(base, 0);
  q[base + grp.thread_rank()] = val;
}

// Removal of edge id at working slot p = (u, v): col mark, dead flag, the
// far endpoint's symmetric row flagged (the caller flags row u). Flags are
// plain byte stores (every writer stores 1); k_queues turns them into the
// compaction queues. Returns min(du, dv) (the edge's delta cost).
template <bool READ_FIRST>
__device__ __forceinline__ uint32_t mark_removed(const Graph& g, const Sym& y, uint32_t p, uint32_t u, uint32_t v,
                                                 uint32_t id) {
  g.col[p] = v | kDeadMark;
  y.dead[id] = 1;
  // full marks flag hubs from many rows at once: read first, store once
  if (!READ_FIRST || !y.sdirty[v]) y.sdirty[v] = 1;
  return min(y.deg[u], y.deg[v]);
}

// Mode 0: thread per slot, every live edge (row of a slot by a binary search
// among the rows of its chunk; working rows are short in degree order, so a
// warp per row would idle most lanes); S < k-2 is removed (truss.cpp:31).
// Removed edge ids are queued on this round's frontier list (empty after a
// full pass), block-aggregated, for k_delta. Totals removed, sum S (3T of
// G_r), delta cost and keep cost.
__global__ void __launch_bounds__(kPruneThreads)
k_mark(Graph g, Sym y) {
  if (g.st->mode != 0) return;
  __shared__ uint32_t wcnt[kPruneThreads / 32];
  __shared__ uint32_t qbase;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t* __restrict__ S = cur_S(g);
  const uint32_t thr = g.st->threshold;
  const uint32_t h0 = g.st->h0;
  const uint32_t fpar = g.st->fpar;
  uint32_t* __restrict__ fq = fpar ? y.fq1 : y.fq0;
  unsigned long long removed = 0, sum_s = 0, dcost = 0, kcost = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x; b0 < g.slots; b0 += stride) {
    const uint64_t p = b0 + threadIdx.x;
    bool rm = false;  // queued for k_delta: removed with triangles to carry
    uint32_t id = 0;
    const uint32_t v = p < g.slots ? g.col[p] : 0u;
    if (v != 0) {
      const uint32_t q = (uint32_t)(p / kChunk);
      uint32_t lo = q ? g.chunk_row[q - 1] : 0u, hi = g.chunk_row[q] + 1;
      while (lo < hi) {  // row u = upper_bound(row_ptr, p) - 1
        const uint32_t mid = (lo + hi) >> 1;
        if (g.row_ptr[mid] <= (uint32_t)p) lo = mid + 1; else hi = mid;
      }
      const uint32_t u = lo - 1;
      const uint32_t sv = u < h0 ? 0u : S[p];  // rows below h0 go whatever their count
      sum_s += sv;
      if (sv < thr || u < h0) {
        ++removed;
        id = g.payload[p];
        const uint32_t c = mark_removed<true>(g, y, (uint32_t)p, u, v, id);
        // S = 0 (exact above h0): the edge closes no triangle, nothing to
        // carry -- it is neither costed nor queued for k_delta
        rm = u < h0 || sv != 0;
        if (rm) dcost += c;
        if (!y.rdirty[u]) y.rdirty[u] = 1;
        if (!y.sdirty[u]) y.sdirty[u] = 1;
      } else {
        kcost += min(y.deg[u], y.deg[v]);
      }
    }
    // block-aggregated append of the removed ids to the frontier list
    const unsigned m = __ballot_sync(0xffffffffu, rm);
    if (lane == 0) wcnt[wid] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < kPruneThreads / 32; ++w) {
        const uint32_t c = wcnt[w];
        wcnt[w] = t;
        t += c;
      }
      qbase = t ? atomicAdd(&g.st->nfq[fpar], t) : 0u;
    }
    __syncthreads();
    if (rm) fq[qbase + wcnt[wid] + __popc(m & ((1u << lane) - 1u))] = id;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum_s += __shfl_xor_sync(0xffffffffu, sum_s, o);
    dcost += __shfl_xor_sync(0xffffffffu, dcost, o);
    kcost += __shfl_xor_sync(0xffffffffu, kcost, o);
    removed += __shfl_xor_sync(0xffffffffu, removed, o);
  }
  if (lane == 0) {
    if (sum_s) atomicAdd(&g.st->sum_s, sum_s);
    if (dcost) atomicAdd(&g.st->delta_cost, dcost);
    if (kcost) atomicAdd(&g.st->keep_cost, kcost);
    if (removed) atomicAdd(&g.st->removed, removed);
  }
}

// Mode 1: thread per frontier edge (queued by the previous round's k_delta).
__global__ void __launch_bounds__(kPruneThreads)
k_mark_frontier(Graph g, Sym y) {
  if (g.st->mode != 1) return;
  const uint32_t par = g.st->fpar;
  const uint32_t nf = g.st->nfq[par];
  const uint32_t* __restrict__ fq = par ? y.fq1 : y.fq0;
  const int lane = threadIdx.x & 31;
  unsigned long long dcost = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    const uint32_t id = fq[i];
    const uint32_t p = y.pos_of[id];
    const uint32_t u = y.erow[id];
    const uint32_t c = mark_removed<false>(g, y, p, u, g.col[p], id);
    if (cur_S(g)[p] != 0) dcost += c;  // carried S is exact: S = 0 closes no triangle
    y.rdirty[u] = 1;
    y.sdirty[u] = 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dcost += __shfl_xor_sync(0xffffffffu, dcost, o);
  if (lane == 0 && dcost) atomicAdd(&g.st->delta_cost, dcost);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g.st->removed, (unsigned long long)nf);
}

// Thread per vertex: flagged rows -> compaction queues (ballot-aggregated
// appends, vertex order), flags cleared.
__global__ void k_queues(Graph g, Sym y) {
  if (g.st->removed == 0) return;
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t n_round = (g.n + stride - 1) / stride * stride;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    const uint32_t v = i + 1;
    bool r = false, sy = false;
    if (v <= g.n) {
      r = y.rdirty[v];
      sy = y.sdirty[v];
      if (r) y.rdirty[v] = 0;
      if (sy) y.sdirty[v] = 0;
    }
    const unsigned mr = __ballot_sync(0xffffffffu, r), ms = __ballot_sync(0xffffffffu, sy);
    uint32_t br = 0, bs = 0;
    if (lane == 0) {
      if (mr) br = atomicAdd(&g.st->nqrow, (uint32_t)__popc(mr));
      if (ms) bs = atomicAdd(&g.st->nqsym, (uint32_t)__popc(ms));
    }
    br = __shfl_sync(0xffffffffu, br, 0);
    bs = __shfl_sync(0xffffffffu, bs, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (r) y.qrow[br + __popc(mr & lt)] = v;
    if (sy) y.qsym[bs + __popc(ms & lt)] = v;
  }
}

// Round 0 of a fixpoint from the pristine graph (ranks ascend by undirected
// degree, so symdeg_p is non-decreasing in rank): an edge (u, v), u < v,
// has S <= min(du, dv) - 1 = du - 1, so every edge of a row u with
// du < k-1 goes in round 0 whatever its count (truss.cpp:31), and a triangle
// matters for a possible survivor only through pivots (i, j) with j heavy
// (dj >= k-1; then the tail and N+(j) are heavy too). h0 = first heavy
// rank: k_support_chunked skips pivots j < h0, k_mark removes rows u < h0.
// The round's removals (count and set) and every later round are unchanged.
__global__ void k_heavy_rank(DevState* st, const uint32_t* __restrict__ symdeg_p, uint32_t n) {
  const uint32_t need = st->threshold + 1;  // k - 1
  uint32_t lo = 1, hi = n + 1;              // first rank r in [1, n] with symdeg_p[r] >= need
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (symdeg_p[mid] < need) lo = mid + 1; else hi = mid;
  }
  st->h0 = lo;
  st->pristine = 1;
}

__global__ void k_set_pristine(DevState* st) { st->pristine = 1; }

// One thread: this round's removal count is final; choose carry vs recompute.
__global__ void k_decide(DevState* st, XArea* xa, unsigned long long xcap) {
  if (st->mode == 1) st->keep_cost = st->live_cost > st->delta_cost ? st->live_cost - st->delta_cost : 0;
  // pieces queued <= delta_cost / kDeltaPiece + removed: carry only if they
  // fit; peer group: the decrements (<= 2 per lost triangle <= 2 delta_cost)
  // must fit this round's list
  st->carry = (st->inc && st->removed != 0 &&
               (double)st->delta_cost <= (st->pristine ? st->delta_ratio0 : st->delta_ratio) * (double)st->keep_cost &&
               st->delta_cost / kDeltaPiece + st->removed <= st->rq_cap && (!xa || 2 * st->delta_cost <= xcap))
                  ? 1u
                  : 0u;
  if (xa) xa->cnt[st->iter & 1u] = 0;  // peers read the other parity's list (k_xapply)
}

__device__ __forceinline__ uint32_t lb_run(const uint32_t* __restrict__ a, uint32_t n, uint32_t key) {
  if (n == 0) return 0;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (__ldg(base + half) < key) ? base + half : base;
    n -= half;
  }
  return (uint32_t)(base - a) + (__ldg(base) < key);
}

// Surviving edge id at slot p loses one triangle; queue it for the next
// round when its support crosses below k-2 (exactly once: S only drops by 1).
__device__ __forceinline__ void drop_support(const Graph& g, const Sym& y, uint32_t* __restrict__ S,
                                             uint32_t* __restrict__ fq_next, uint32_t* cnt_next, uint32_t thr,
                                             uint32_t id) {
  const uint32_t old = atomicSub(&S[y.pos_of[id]], 1u);
  if (old == thr) append_coalesced(cnt_next, fq_next, id);
  if (g.xa) {  // peer group: the peers apply the same decrement (k_xapply)
    const uint32_t par = g.st->iter & 1u;
    append_coalesced(&g.xa->cnt[par], xlist(g.xa, g.xcap, par), id);
  }
}

// Triangles of G_r through the removed edge e = (u, v) at working slot p:
// each element w of elements [lo, hi) of the shorter symmetric row is
// binary-searched in the longer one (warp-cooperative, lanes over elements).
// A common neighbour w closes {e, (u,w), (v,w)}; the triangle is handled by
// its removed edge with the smallest id (so once), and each surviving edge
// of it loses 1.
__device__ __forceinline__ void delta_edge(const Graph& g, const Sym& y, uint32_t* __restrict__ S,
                                           uint32_t* __restrict__ fq_next, uint32_t* cnt_next, uint32_t thr,
                                           uint32_t p, uint32_t u, uint32_t v, uint32_t lo, uint32_t hi) {
  const int lane = threadIdx.x & 31;
  const uint32_t e = g.payload[p];
  const uint32_t du = y.deg[u], dv = y.deg[v];
  const bool su = du <= dv;
  const uint32_t la = su ? du : dv, lb = su ? dv : du;
  const unsigned long long oa = y.ptr[su ? u : v], ob = y.ptr[su ? v : u];
  const uint32_t* __restrict__ A = y.nbr + oa;
  const uint32_t* __restrict__ B = y.nbr + ob;
  hi = min(hi, la);
  if (lo >= hi) return;
  const uint32_t bmin = B[0], bmax = B[lb - 1];
  // long B: lane l holds the last element of bucket l of 32 equal buckets,
  // so an element's bucket comes from 5 shuffles and its global binary
  // search covers lb/32 entries (5 fewer dependent loads per element)
  const bool coarse = lb >= 256;
  const uint32_t samp = coarse ? B[(uint32_t)(((uint64_t)(lane + 1) * lb) >> 5) - 1] : 0u;
  for (uint32_t b0 = lo; b0 < hi; b0 += 32) {  // warp-uniform trip count (shuffles)
    const uint32_t i = b0 + lane;
    const bool act = i < hi;
    const uint32_t w = act ? A[i] : 0u;
    uint32_t jlo = 0, jn = lb;
    if (coarse) {
      uint32_t k = 0;  // first bucket whose last element >= w (w <= bmax = last of bucket 31)
#pragma unroll
      for (uint32_t step = 16; step; step >>= 1) {
        const uint32_t sv = __shfl_sync(0xffffffffu, samp, k + step - 1);
        if (sv < w) k += step;
      }
      jlo = (uint32_t)(((uint64_t)k * lb) >> 5);
      jn = (uint32_t)(((uint64_t)(k + 1) * lb) >> 5) - jlo;
    }
    if (!act || w < bmin || w > bmax) continue;
    const uint32_t j = jlo + lb_run(B + jlo, jn, w);
    if (j < lb && B[j] == w) {
      const uint32_t ea = y.eid[oa + i], eb = y.eid[ob + j];
      const bool da = y.dead[ea], db = y.dead[eb];
      if ((da && ea < e) || (db && eb < e)) continue;
      if (!da) drop_support(g, y, S, fq_next, cnt_next, thr, ea);
      if (!db) drop_support(g, y, S, fq_next, cnt_next, thr, eb);
    }
  }
}

constexpr uint32_t kDeltaInline = kDeltaPiece;  // longer intersections are queued as pieces

// Warp per removed edge: after a full mark, rows are scanned for marked
// slots; after a carried round, the frontier list is the removal set.
// Intersections up to kDeltaInline elements run inline; longer ones are
// queued as kDeltaPiece pieces {slot, u, v, piece} for k_delta_big.
__global__ void __launch_bounds__(kPruneThreads)
k_delta(Graph g, Sym y) {
  if (!g.st->carry) return;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t* __restrict__ S = cur_S(g);
  const uint32_t thr = g.st->threshold;
  const uint32_t par = g.st->fpar ^ 1u;  // next round's frontier
  uint32_t* __restrict__ fq_next = par ? y.fq1 : y.fq0;
  uint32_t* cnt_next = &g.st->nfq[par];
  const uint32_t h0 = g.st->h0;
  auto edge = [&](uint32_t p, uint32_t u, uint32_t v) {
    // S of a removed edge is its exact triangle count in G_r (rows below h0
    // of a pristine round 0 excepted): S = 0 means no triangle loses an edge
    if (u >= h0 && S[p] == 0) return;
    if (g.xa && owner_of(g.payload[p], g.world) != g.rank) return;  // a peer's share
    const uint32_t mn = min(y.deg[u], y.deg[v]);
    if (mn <= kDeltaInline) {
      delta_edge(g, y, S, fq_next, cnt_next, thr, p, u, v, 0, mn);
    } else if (lane == 0) {
      const uint32_t np = (mn + kDeltaPiece - 1) / kDeltaPiece;
      const uint32_t at = atomicAdd(&g.st->nrq, np);
      for (uint32_t t = 0; t < np; ++t) y.rq[at + t] = make_uint4(p, u, v, t);
    }
  };
  {  // the removal set: queued by k_mark (mode 0) or by the last k_delta (mode 1)
    const uint32_t fpar = g.st->fpar;
    const uint32_t nf = g.st->nfq[fpar];
    const uint32_t* __restrict__ fq = fpar ? y.fq1 : y.fq0;
    for (uint32_t i = warp; i < nf; i += nwarps) {
      const uint32_t id = fq[i];
      const uint32_t p = y.pos_of[id];
      edge(p, y.erow[id], g.col[p] & ~kDeadMark);
    }
  }
}

// Warp per queued piece of a long intersection.
__global__ void __launch_bounds__(kPruneThreads)
k_delta_big(Graph g, Sym y) {
  if (!g.st->carry) return;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t* __restrict__ S = cur_S(g);
  const uint32_t thr = g.st->threshold;
  const uint32_t par = g.st->fpar ^ 1u;
  uint32_t* __restrict__ fq_next = par ? y.fq1 : y.fq0;
  uint32_t* cnt_next = &g.st->nfq[par];
  const uint32_t ntask = g.st->nrq;
  for (uint32_t t = warp; t < ntask; t += nwarps) {
    const uint4 q = y.rq[t];
    delta_edge(g, y, S, fq_next, cnt_next, thr, q.x, q.y, q.z, q.w * kDeltaPiece, (q.w + 1) * kDeltaPiece);
  }
}

// ---------------------------------------------------------------------------
// Peer group exchange (multi-GPU, ktg_engine_set_group): collectives as
// kernels over NVLink peer memory, so a partitioned fixpoint stays one
// CUDA-graph launch with no host round trip per round.
//   full pass: [this rank's A22 tasks] -> k_xbar -> k_xreduce (rank r sums
//              every rank's partial S over its span and writes the sum back
//              to every rank) -> k_xbar
//   carried round: k_delta on this rank's removals -> k_xbar -> k_xapply
//              (every peer's listed decrements applied locally)
// Every rank runs the same control flow on replicated state, so all ranks
// meet the same barriers in the same order.
// ---------------------------------------------------------------------------
struct XGroup {
  XArea* const* area;      // per rank, peer-mapped (own at [rank])
  uint32_t* const* S0;     // per rank: its support buffers (peer-mapped)
  uint32_t* const* S1;
  uint32_t rank, world;
  uint64_t cap;            // entries per decrement list
  uint64_t span;           // slots reduced per rank (multiple of 4)
};

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// WHEN 0: after a carried run's full pass (mode 0); 1: in a carrying round;
// 2: every round (recompute runs). One thread: publish (optionally) the
// round's partial triangle count, signal every rank, wait for every rank.
// A peer that never arrives (crashed rank) stops the loop after 120 s with
// kErrGroupTimeout instead of hanging the device.
template <int WHEN>
__global__ void k_xbar(DevState* st, XGroup x, int publish_tri) {
  if (WHEN == 0 && (st->mode != 0 || !st->inc)) return;
  if (WHEN == 1 && !st->carry) return;
  if (threadIdx.x != 0 || st->error) return;
  XArea* own = x.area[x.rank];
  if (publish_tri) *reinterpret_cast<volatile unsigned long long*>(&own->tri) = st->triangles;
  const unsigned int ep = ++st->xepoch;
  __threadfence_system();
  for (uint32_t q = 0; q < x.world; ++q) st_release_sys(&x.area[q]->flags[x.rank], ep);
  const unsigned long long t0 = globaltimer_ns();
  for (uint32_t q = 0; q < x.world; ++q) {
    while ((int)(ld_acquire_sys(&own->flags[q]) - ep) < 0) {
      __nanosleep(128);
      if (globaltimer_ns() - t0 > 120000000000ull) {
        st->error = kErrGroupTimeout;
        return;
      }
    }
  }
  __threadfence_system();
}

// Rank r's span of the support buffer: sum of every rank's partial counts,
// written back to every rank (reduce-scatter + all-gather in one pass over
// peer memory); block 0 also totals the round's triangle count.
__global__ void k_xreduce(Graph g, XGroup x, int inc) {
  if (inc && g.st->mode != 0) return;
  if (g.st->error) return;
  uint32_t* const* tab = g.st->parity ? x.S1 : x.S0;
  const uint64_t lo = (uint64_t)x.rank * x.span;
  const uint64_t hi = umin64(g.slots, lo + x.span);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t = 0;
    for (uint32_t q = 0; q < x.world; ++q) t += *reinterpret_cast<volatile unsigned long long*>(&x.area[q]->tri);
    g.st->triangles = t;
  }
  if (lo >= hi) return;
  const uint64_t n4 = (hi - lo) / 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint32_t q = 0; q < x.world; ++q) {
      const uint4 v = __ldcv(reinterpret_cast<const uint4*>(tab[q] + lo) + i);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
    for (uint32_t q = 0; q < x.world; ++q) __stcg(reinterpret_cast<uint4*>(tab[q] + lo) + i, acc);
  }
  for (uint64_t i = lo + 4 * n4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi; i += stride) {
    uint32_t acc = 0;
    for (uint32_t q = 0; q < x.world; ++q) acc += __ldcv(tab[q] + i);
    for (uint32_t q = 0; q < x.world; ++q) __stcg(tab[q] + i, acc);
  }
}

// Carrying round, after k_xbar<1>: every peer's decrements of this round
// applied to the local supports (frontier crossings queued as in k_delta).
__global__ void __launch_bounds__(kPruneThreads)
k_xapply(Graph g, Sym y, XGroup x) {
  if (!g.st->carry || g.st->error) return;
  uint32_t* __restrict__ S = cur_S(g);
  const uint32_t thr = g.st->threshold;
  const uint32_t par = g.st->fpar ^ 1u;
  uint32_t* __restrict__ fq_next = par ? y.fq1 : y.fq0;
  uint32_t* cnt_next = &g.st->nfq[par];
  const uint32_t lp = g.st->iter & 1u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t q = 0; q < x.world; ++q) {
    if (q == x.rank) continue;
    XArea* a = x.area[q];
    const uint32_t n = *reinterpret_cast<volatile unsigned int*>(&a->cnt[lp]);
    const uint32_t* list = xlist(a, x.cap, lp);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const uint32_t id = __ldcv(list + i);
      const uint32_t old = atomicSub(&S[y.pos_of[id]], 1u);
      if (old == thr) append_coalesced(cnt_next, fq_next, id);
    }
  }
}

// Oriented rows that lost an edge: stable compaction of (col, id) and, when
// the round carries supports, S; pos_of follows every moved edge. Warp per
// queued row up to kHeavyRow (HEAVY = 0), CTA per longer row (HEAVY = 1).
// Stable in-place compaction of one oriented row [base, base + d) by a group
// of GS lanes: live entries (no dead mark) move down with their id and,
// when the round carries, their S; pos_of follows; the vacated tail is
// zeroed. Returns the new length.
template <int GS>
__device__ __forceinline__ uint32_t row_compact(const Graph& g, const Sym& y, uint32_t* __restrict__ S, bool carry,
                                                uint32_t base, uint32_t d, uint32_t gl, unsigned gmask) {
  uint32_t write = 0;
  for (uint32_t off = 0; off < d; off += GS) {
    const uint32_t idx = off + gl;
    const bool live = idx < d;
    const uint32_t c = live ? g.col[base + idx] : 0u;
    const uint32_t sv = (live && carry) ? S[base + idx] : 0u;
    const uint32_t pv = live ? g.payload[base + idx] : 0u;
    const bool keep = live && !(c & kDeadMark);
    uint32_t x = keep;
#pragma unroll
    for (int o = 1; o < GS; o <<= 1) {
      const uint32_t t = __shfl_up_sync(gmask, x, o, GS);
      if (gl >= (uint32_t)o) x += t;
    }
    const uint32_t total = __shfl_sync(gmask, x, GS - 1, GS);
    if (keep) {
      const uint32_t pos = write + x - 1;
      g.col[base + pos] = c;
      if (carry) S[base + pos] = sv;
      g.payload[base + pos] = pv;
      if (pos != idx) y.pos_of[pv] = base + pos;
    }
    write += total;
  }
  for (uint32_t x = write + gl; x < d; x += GS) {
    g.col[base + x] = 0;
    if (carry) S[base + x] = 0;
  }
  return write;
}

template <int HEAVY>
__global__ void __launch_bounds__(HEAVY ? kSymHeavyThreads : kPruneThreads)
k_inc_rows(Graph g, Sym y) {
  if (!HEAVY) {
    // a warp takes 4 queued rows: rows of <= 32 entries by one 8-lane group
    // each, longer ones by the whole warp, rows above kHeavyRow by the CTA
    // kernel (HEAVY = 1)
    if (g.st->removed == 0) return;
    const bool carry = g.st->carry;
    uint32_t* __restrict__ S = cur_S(g);
    const uint32_t lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const unsigned gmask = 0xffu << (grp * 8);
    const uint32_t nq = g.st->nqrow;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    if (nq <= nwarps) {  // few rows (late carried rounds): one warp each, all in parallel
      for (uint32_t h = warp; h < nq; h += nwarps) {
        const uint32_t u = y.qrow[h], d = g.deg[u];
        if (d > (uint32_t)kHeavyRow) {
          if (lane == 0) g.heavy_rows[atomicAdd(&g.st->nheavy, 1u)] = u;
          continue;
        }
        const uint32_t nd = row_compact<32>(g, y, S, carry, g.row_ptr[u], d, lane, 0xffffffffu);
        if (lane == 0) g.deg[u] = nd;
      }
      return;
    }
    for (uint32_t h0 = warp * 4; h0 < nq; h0 += nwarps * 4) {  // warp-uniform
      const uint32_t h = h0 + grp;
      const uint32_t u = h < nq ? y.qrow[h] : 0u;
      const uint32_t d = h < nq ? g.deg[u] : 0u;
      if (h < nq && d <= 32) {
        const uint32_t nd = row_compact<8>(g, y, S, carry, g.row_ptr[u], d, gl, gmask);
        if (gl == 0) g.deg[u] = nd;
      } else if (h < nq && d > (uint32_t)kHeavyRow && gl == 0) {
        g.heavy_rows[atomicAdd(&g.st->nheavy, 1u)] = u;
      }
      __syncwarp();
      unsigned lm = __ballot_sync(0xffffffffu, gl == 0 && h < nq && d > 32 && d <= (uint32_t)kHeavyRow);
      while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t uu = __shfl_sync(0xffffffffu, u, src), dd = __shfl_sync(0xffffffffu, d, src);
        const uint32_t nd = row_compact<32>(g, y, S, carry, g.row_ptr[uu], dd, lane, 0xffffffffu);
        if (lane == 0) g.deg[uu] = nd;
      }
    }
    return;
  }
  constexpr int EPT = HEAVY ? 4 : 1;
  constexpr int BT = HEAVY ? kSymHeavyThreads : kPruneThreads;
  constexpr int NW = BT / 32;
  __shared__ uint32_t red[NW];
  __shared__ uint32_t tot_s;
  if (g.st->removed == 0) return;
  const bool carry = g.st->carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t nq = HEAVY ? g.st->nheavy : g.st->nqrow;
  const uint32_t* __restrict__ queue = HEAVY ? g.heavy_rows : y.qrow;
  uint32_t* __restrict__ S = cur_S(g);
  uint32_t* __restrict__ col = g.col;
  uint32_t* __restrict__ pay = g.payload;
  const uint32_t first = HEAVY ? blockIdx.x : (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t step = HEAVY ? gridDim.x : (gridDim.x * blockDim.x) >> 5;
  for (uint32_t h = first; h < nq; h += step) {
    const uint32_t u = queue[h];
    const uint32_t d = g.deg[u];
    if (!HEAVY && d > (uint32_t)kHeavyRow) {  // long row: CTA kernel
      if (lane == 0) g.heavy_rows[atomicAdd(&g.st->nheavy, 1u)] = u;
      continue;
    }
    const uint32_t base = g.row_ptr[u];
    uint32_t write = 0;
    constexpr uint32_t TILE = HEAVY ? EPT * BT : 32;
    for (uint32_t off = 0; off < d; off += TILE) {
      uint32_t c[EPT], sv[EPT], pv[EPT];
      bool keep[EPT];
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t idx = off + (HEAVY ? threadIdx.x * EPT + k : lane);
        const bool live = idx < d;
        c[k] = live ? col[base + idx] : 0u;
        sv[k] = (live && carry) ? S[base + idx] : 0u;
        pv[k] = live ? pay[base + idx] : 0u;
        keep[k] = live && !(c[k] & kDeadMark);
        cnt += keep[k];
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      uint32_t pos, total;
      if (HEAVY) {
        if (lane == 31) red[wid] = x;
        __syncthreads();  // also: every thread has read its tile before writes
        if (wid == 0) {
          uint32_t w = lane < NW ? red[lane] : 0;
#pragma unroll
          for (int o = 1; o < NW; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
          }
          if (lane < NW) red[lane] = w;
          if (lane == NW - 1) tot_s = w;
        }
        __syncthreads();
        pos = write + x - cnt + (wid ? red[wid - 1] : 0);
        total = tot_s;
      } else {
        __syncwarp();  // every lane's loads precede any lane's in-place store
        pos = write + x - cnt;
        total = __shfl_sync(0xffffffffu, x, 31);
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t idx = off + (HEAVY ? threadIdx.x * EPT + k : lane);
        if (keep[k]) {
          col[base + pos] = c[k];
          if (carry) S[base + pos] = sv[k];
          pay[base + pos] = pv[k];
          if (pos != idx) y.pos_of[pv[k]] = base + pos;
          ++pos;
        }
      }
      write += total;
      if (HEAVY) __syncthreads();
    }
    for (uint32_t x = write + (HEAVY ? threadIdx.x : lane); x < d; x += (HEAVY ? blockDim.x : 32)) {
      col[base + x] = 0;
      if (carry) S[base + x] = 0;
    }
    if (HEAVY ? threadIdx.x == 0 : lane == 0) g.deg[u] = write;
    if (HEAVY) __syncthreads();
  }
}

// Stable in-place compaction of one symmetric row by a group of GS lanes
// (GS = 8 or 32, `gl` = lane in the group, `gmask` = the group's lanes):
// drops entries whose edge is dead, returns the new length.
template <int GS>
__device__ __forceinline__ uint32_t sym_compact(const Sym& y, unsigned long long base, uint32_t d, uint32_t gl,
                                                unsigned gmask) {
  uint32_t write = 0;
  for (uint32_t off = 0; off < d; off += GS) {
    const uint32_t idx = off + gl;
    const bool live = idx < d;
    const uint32_t w = live ? y.nbr[base + idx] : 0u;
    const uint32_t ev = live ? y.eid[base + idx] : 0u;
    const bool keep = live && !y.dead[ev];
    uint32_t x = keep;
#pragma unroll
    for (int o = 1; o < GS; o <<= 1) {
      const uint32_t t = __shfl_up_sync(gmask, x, o, GS);
      if (gl >= (uint32_t)o) x += t;
    }
    const uint32_t total = __shfl_sync(gmask, x, GS - 1, GS);
    if (keep) {
      y.nbr[base + write + x - 1] = w;
      y.eid[base + write + x - 1] = ev;
    }
    write += total;
  }
  return write;
}

// Symmetric rows that lost an edge drop their dead entries (stable).
// HEAVY = 0: a warp takes 4 queued rows; rows of <= 32 entries (most of them
// in degree order) are compacted by one 8-lane group each, longer ones by the
// whole warp, rows above kHeavyRow go to the CTA kernel (HEAVY = 1).
template <int HEAVY>
__global__ void __launch_bounds__(HEAVY ? kSymHeavyThreads : kPruneThreads)
k_inc_sym(Graph g, Sym y) {
  if (!HEAVY) {
    if (g.st->removed == 0) return;
    const uint32_t lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const unsigned gmask = 0xffu << (grp * 8);
    const uint32_t nq = g.st->nqsym;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    if (nq <= nwarps) {  // few rows (late carried rounds): one warp each, all in parallel
      for (uint32_t h = warp; h < nq; h += nwarps) {
        const uint32_t v = y.qsym[h], d = y.deg[v];
        if (d > (uint32_t)kHeavyRow) {
          if (lane == 0) y.heavy[atomicAdd(&g.st->nheavy_sym, 1u)] = v;
          continue;
        }
        const uint32_t nd = sym_compact<32>(y, y.ptr[v], d, lane, 0xffffffffu);
        if (lane == 0) y.deg[v] = nd;
      }
      return;
    }
    for (uint32_t h0 = warp * 4; h0 < nq; h0 += nwarps * 4) {  // warp-uniform
      const uint32_t h = h0 + grp;
      const uint32_t v = h < nq ? y.qsym[h] : 0u;
      const uint32_t d = h < nq ? y.deg[v] : 0u;
      if (h < nq && d <= 32) {
        const uint32_t nd = sym_compact<8>(y, y.ptr[v], d, gl, gmask);
        if (gl == 0) y.deg[v] = nd;
      } else if (h < nq && d > (uint32_t)kHeavyRow && gl == 0) {
        y.heavy[atomicAdd(&g.st->nheavy_sym, 1u)] = v;
      }
      __syncwarp();
      unsigned lm = __ballot_sync(0xffffffffu, gl == 0 && h < nq && d > 32 && d <= (uint32_t)kHeavyRow);
      while (lm) {  // the warp's medium rows, one at a time, all 32 lanes
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t vv = __shfl_sync(0xffffffffu, v, src), dd = __shfl_sync(0xffffffffu, d, src);
        const uint32_t nd = sym_compact<32>(y, y.ptr[vv], dd, lane, 0xffffffffu);
        if (lane == 0) y.deg[vv] = nd;
      }
    }
    return;
  }
  constexpr int EPT = HEAVY ? 4 : 1;
  constexpr int BT = HEAVY ? kSymHeavyThreads : kPruneThreads;
  constexpr int NW = BT / 32;
  __shared__ uint32_t red[NW];
  __shared__ uint32_t tot_s;
  if (g.st->removed == 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t nq = HEAVY ? g.st->nheavy_sym : g.st->nqsym;
  const uint32_t* __restrict__ queue = HEAVY ? y.heavy : y.qsym;
  const uint32_t first = HEAVY ? blockIdx.x : (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t step = HEAVY ? gridDim.x : (gridDim.x * blockDim.x) >> 5;
  for (uint32_t h = first; h < nq; h += step) {
    const uint32_t v = queue[h];
    const uint32_t d = y.deg[v];
    if (!HEAVY && d > (uint32_t)kHeavyRow) {  // long row: CTA kernel
      if (lane == 0) y.heavy[atomicAdd(&g.st->nheavy_sym, 1u)] = v;
      continue;
    }
    const unsigned long long base = y.ptr[v];
    uint32_t write = 0;
    constexpr uint32_t TILE = HEAVY ? EPT * BT : 32;
    for (uint32_t off = 0; off < d; off += TILE) {
      uint32_t w[EPT], ev[EPT];
      bool keep[EPT];
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t idx = off + (HEAVY ? threadIdx.x * EPT + k : lane);
        const bool live = idx < d;
        w[k] = live ? y.nbr[base + idx] : 0u;
        ev[k] = live ? y.eid[base + idx] : 0u;
        keep[k] = live && !y.dead[ev[k]];
        cnt += keep[k];
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      uint32_t pos, total;
      if (HEAVY) {
        if (lane == 31) red[wid] = x;
        __syncthreads();
        if (wid == 0) {
          uint32_t s = lane < NW ? red[lane] : 0;
#pragma unroll
          for (int o = 1; o < NW; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
          }
          if (lane < NW) red[lane] = s;
          if (lane == NW - 1) tot_s = s;
        }
        __syncthreads();
        pos = write + x - cnt + (wid ? red[wid - 1] : 0);
        total = tot_s;
      } else {
        __syncwarp();
        pos = write + x - cnt;
        total = __shfl_sync(0xffffffffu, x, 31);
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (keep[k]) {
          y.nbr[base + pos] = w[k];
          y.eid[base + pos] = ev[k];
          ++pos;
        }
      write += total;
      if (HEAVY) __syncthreads();
    }
    if (HEAVY ? threadIdx.x == 0 : lane == 0) y.deg[v] = write;
    if (HEAVY) __syncthreads();
  }
}

// Publish after a carried run, one pass per caller row: caller slot s
// survives iff its edge is not dead; survivors are compacted stably from the
// pristine row (the composition of every round's prune, truss.cpp:26-35) and
// take their support from the working slot pos_of[s]. Warp per row up to
// kHeavyRow (HEAVY = 0, longer rows queued), CTA per longer row (HEAVY = 1).
// One caller row by a group of GS lanes (GS = 8 or 32): survivors of the
// pristine row [base, base + d) compacted stably with their supports, the
// rest zeroed; returns the new length.
template <int GS>
__device__ __forceinline__ uint32_t publish_row(const Graph& c, const uint32_t* __restrict__ col_p,
                                                const uint8_t* __restrict__ dead,
                                                const uint32_t* __restrict__ pos_of,
                                                const uint32_t* __restrict__ Sw, uint32_t base, uint32_t d,
                                                uint32_t gl, unsigned gmask) {
  uint32_t write = 0;
  for (uint32_t off = 0; off < d; off += GS) {
    const uint32_t idx = off + gl;
    const bool keep = idx < d && !dead[base + idx];
    const uint32_t cv = keep ? col_p[base + idx] : 0u;
    const uint32_t sv = keep ? Sw[pos_of[base + idx]] : 0u;
    uint32_t x = keep;
#pragma unroll
    for (int o = 1; o < GS; o <<= 1) {
      const uint32_t t = __shfl_up_sync(gmask, x, o, GS);
      if (gl >= (uint32_t)o) x += t;
    }
    const uint32_t total = __shfl_sync(gmask, x, GS - 1, GS);
    if (keep) {
      c.col[base + write + x - 1] = cv;
      c.S0[base + write + x - 1] = sv;
    }
    write += total;
  }
  for (uint32_t x = write + gl; x < d; x += GS) {
    c.col[base + x] = 0;
    c.S0[base + x] = 0;
  }
  return write;
}

template <int HEAVY>
__global__ void __launch_bounds__(HEAVY ? kSymHeavyThreads : kPruneThreads)
k_publish_inc(Graph c, const uint32_t* __restrict__ col_p, const uint32_t* __restrict__ deg_p,
              const uint8_t* __restrict__ dead, const uint32_t* __restrict__ pos_of,
              const uint32_t* __restrict__ Sw) {
  if (!HEAVY) {
    // a warp takes 4 caller rows: rows of <= 32 pristine entries by one 8-lane
    // group each, longer ones by the whole warp, rows above kHeavyRow by the
    // CTA kernel (HEAVY = 1)
    const uint32_t lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const unsigned gmask = 0xffu << (grp * 8);
    const uint32_t nq = c.n;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t h0 = warp * 4; h0 < nq; h0 += nwarps * 4) {  // warp-uniform
      const uint32_t h = h0 + grp;
      const uint32_t r = h + 1;
      const uint32_t d = h < nq ? deg_p[r] : 0u;
      if (d != 0 && d <= 32) {
        const uint32_t nd = publish_row<8>(c, col_p, dead, pos_of, Sw, c.row_ptr[r], d, gl, gmask);
        if (gl == 0) c.deg[r] = nd;
      } else if (d > (uint32_t)kHeavyRow && gl == 0) {
        c.heavy_rows[atomicAdd(&c.st->nheavy, 1u)] = r;
      }
      __syncwarp();
      unsigned lm = __ballot_sync(0xffffffffu, gl == 0 && d > 32 && d <= (uint32_t)kHeavyRow);
      while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t rr = __shfl_sync(0xffffffffu, r, src), dd = __shfl_sync(0xffffffffu, d, src);
        const uint32_t nd = publish_row<32>(c, col_p, dead, pos_of, Sw, c.row_ptr[rr], dd, lane, 0xffffffffu);
        if (lane == 0) c.deg[rr] = nd;
      }
    }
    return;
  }
  constexpr int EPT = HEAVY ? 4 : 1;
  constexpr int BT = HEAVY ? kSymHeavyThreads : kPruneThreads;
  constexpr int NW = BT / 32;
  __shared__ uint32_t red[NW];
  __shared__ uint32_t tot_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t nq = HEAVY ? c.st->nheavy : c.n;
  const uint32_t first = HEAVY ? blockIdx.x : (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t step = HEAVY ? gridDim.x : (gridDim.x * blockDim.x) >> 5;
  for (uint32_t h = first; h < nq; h += step) {
    const uint32_t r = HEAVY ? c.heavy_rows[h] : h + 1;
    const uint32_t d = deg_p[r];
    if (d == 0) continue;
    if (!HEAVY && d > (uint32_t)kHeavyRow) {
      if (lane == 0) c.heavy_rows[atomicAdd(&c.st->nheavy, 1u)] = r;
      continue;
    }
    const uint32_t base = c.row_ptr[r];
    uint32_t write = 0;
    constexpr uint32_t TILE = HEAVY ? EPT * BT : 32;
    for (uint32_t off = 0; off < d; off += TILE) {
      uint32_t cv[EPT], sv[EPT];
      bool keep[EPT];
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t idx = off + (HEAVY ? threadIdx.x * EPT + k : lane);
        keep[k] = idx < d && !dead[base + idx];
        cv[k] = keep[k] ? col_p[base + idx] : 0u;
        sv[k] = keep[k] ? Sw[pos_of[base + idx]] : 0u;
        cnt += keep[k];
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      uint32_t pos, total;
      if (HEAVY) {
        if (lane == 31) red[wid] = x;
        __syncthreads();
        if (wid == 0) {
          uint32_t w = lane < NW ? red[lane] : 0;
#pragma unroll
          for (int o = 1; o < NW; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
          }
          if (lane < NW) red[lane] = w;
          if (lane == NW - 1) tot_s = w;
        }
        __syncthreads();
        pos = write + x - cnt + (wid ? red[wid - 1] : 0);
        total = tot_s;
      } else {
        pos = write + x - cnt;
        total = __shfl_sync(0xffffffffu, x, 31);
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (keep[k]) {
          c.col[base + pos] = cv[k];
          c.S0[base + pos] = sv[k];
          ++pos;
        }
      write += total;
      if (HEAVY) __syncthreads();
    }
    for (uint32_t x = write + (HEAVY ? threadIdx.x : lane); x < d; x += (HEAVY ? blockDim.x : 32)) {
      c.col[base + x] = 0;
      c.S0[base + x] = 0;
    }
    if (HEAVY ? threadIdx.x == 0 : lane == 0) c.deg[r] = write;
    if (HEAVY) __syncthreads();
  }
}

// A recompute round follows: zero S (the next full pass accumulates into it).
__global__ void k_inc_zero(Graph g) {
  if (g.st->removed == 0 || g.st->carry) return;
  uint4* S4 = reinterpret_cast<uint4*>(cur_S(g));
  const uint64_t n4 = (g.slots + 3) / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    S4[i] = make_uint4(0, 0, 0, 0);
}

// End of an incremental round: removal history, live count, the next round's
// mode and frontier, the while condition. S stays in one buffer.
__global__ void k_control_inc(DevState* st, unsigned long long* hist, cudaGraphConditionalHandle handle,
                              int use_cond) {
  const unsigned long long removed = st->removed;
  const uint32_t it = st->iter;
  if (it < (uint32_t)kHistCap) hist[it] = removed;
  st->iter = it + 1;
  st->live -= removed;
  if (st->mode == 0) st->last_triangles = st->sum_s / 3;
  st->live_cost = st->keep_cost;
  st->last_nrq = st->nrq;
  st->last_carry = st->carry;
  st->last_dcost = st->delta_cost;
  st->last_kcost = st->keep_cost;
  st->mode = st->carry;
  st->h0 = 0;  // round 0 only
  st->pristine = 0;
  st->nfq[st->fpar] = 0;
  st->fpar ^= 1u;
  st->carry = 0;
  st->triangles = 0;
  st->sum_s = 0;
  st->delta_cost = 0;
  st->keep_cost = 0;
  st->nrq = 0;
  st->nqrow = 0;
  st->nqsym = 0;
  st->nheavy_sym = 0;
  st->removed = 0;
  st->task_next = 0;
  st->nheavy = 0;
  const bool cont = removed != 0 && st->error == 0;
  if (use_cond) cudaGraphSetConditional(handle, cont ? 1u : 0u);
}

// T of the converged graph (sum of its supports / 3) after a carried run.
__global__ void k_inc_triangles(Graph g) {
  const uint32_t* __restrict__ S = cur_S(g);
  unsigned long long s = 0;
  const uint4* S4 = reinterpret_cast<const uint4*>(S);
  const uint64_t n4 = (g.slots + 3) / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 q = S4[i];
    s += (unsigned long long)q.x + q.y + q.z + q.w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(&g.st->sum_s, s);
}

__global__ void k_inc_triangles_done(DevState* st) {
  st->last_triangles = st->sum_s / 3;
  st->sum_s = 0;
}

__global__ void k_u64_to_u32(const unsigned long long* __restrict__ a, uint32_t n, uint32_t* __restrict__ b) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = (uint32_t)a[i];
}

// ---------------------------------------------------------------------------
// canonicalize + build_csr on the device
// ---------------------------------------------------------------------------
// Same result as edge_list.cpp:62-103 + csr.cpp:10-32: self-loops dropped,
// labels relabelled 1..n by ascending original label, edges oriented u < v,
// deduplicated, rows sorted; one zero sentinel per row. Self-loops / padding
// become the ~0 sentinel key, which sorts last and is cut off.

__global__ void k_pair_labels(const unsigned long long* __restrict__ pairs, uint64_t m,
                              unsigned long long* __restrict__ labels) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long a = pairs[2 * i], b = pairs[2 * i + 1];
    const bool loop = a == b;
    labels[2 * i] = loop ? ~0ull : a;
    labels[2 * i + 1] = loop ? ~0ull : b;
  }
}

__device__ __forceinline__ uint32_t label_rank(const unsigned long long* __restrict__ lab, uint32_t n,
                                               unsigned long long x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (lab[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo + 1;
}

__global__ void k_pair_keys(const unsigned long long* __restrict__ pairs, uint64_t m,
                            const unsigned long long* __restrict__ lab, uint32_t n,
                            unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a == b) {
      keys[i] = ~0ull;
      continue;
    }
    const uint32_t u = label_rank(lab, n, a), v = label_rank(lab, n, b);
    keys[i] = ((unsigned long long)min(u, v) << 32) | max(u, v);
  }
}

__global__ void k_key_rows(const unsigned long long* __restrict__ keys, uint64_t m, uint32_t* __restrict__ cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[(uint32_t)(keys[i] >> 32)], 1u);
}

// sorted unique keys -> col (slot = idx + u - 1, one sentinel per earlier row)
__global__ void k_key_fill(const unsigned long long* __restrict__ keys, uint64_t m, uint32_t* __restrict__ col) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    col[i + (uint32_t)(k >> 32) - 1] = (uint32_t)k;
  }
}

// ---------------------------------------------------------------------------
// Degree-ordered working layout
// ---------------------------------------------------------------------------
// Vertices are ranked by (undirected degree, id); every edge is oriented from
// lower to higher rank. Supports and trusses are orientation invariant, so the
// fixpoint runs on this layout and the caller's layout is rebuilt from it at
// the end (k_scatter_live + k_prune_*<1>) byte-identically.

__global__ void k_rank_keys(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ din, uint32_t n,
                            unsigned long long* __restrict__ keys) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x + 1; v <= n; v += gridDim.x * blockDim.x)
    keys[v - 1] = ((unsigned long long)(deg[v] + din[v]) << 32) | v;
}

__global__ void k_rank_assign(const unsigned long long* __restrict__ sorted, uint32_t n, uint32_t* __restrict__ rank,
                              uint32_t* __restrict__ symdeg_w) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long k = sorted[i];
    rank[(uint32_t)k] = i + 1;
    symdeg_w[i + 1] = (uint32_t)(k >> 32);  // undirected degree of rank i + 1
  }
}

// Edge keys (a << B | b, a < b ranks) with the caller slot as value,
// slot-parallel (the row of a live slot by binary search over row_ptr);
// offs = exclusive prefix of the caller live degrees.
__global__ void k_edge_keys(Graph g, const uint32_t* __restrict__ rank, const uint32_t* __restrict__ offs,
                            uint32_t B, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                            uint32_t* __restrict__ erow) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < g.slots;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = g.col[x];
    if (c == 0) continue;
    // row = upper_bound(row_ptr, x) - 1, inside the rows of x's chunk
    const uint32_t q = (uint32_t)(x / kChunk);
    uint32_t lo = q ? g.chunk_row[q - 1] : 0u, hi = g.chunk_row[q] + 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (g.row_ptr[mid] <= (uint32_t)x) lo = mid + 1; else hi = mid;
    }
    const uint32_t u = lo - 1;
    const uint32_t o = offs[u] + ((uint32_t)x - g.row_ptr[u]);
    const uint32_t ru = rank[u], rv = rank[c];
    const uint32_t a = min(ru, rv), b = max(ru, rv);
    keys[o] = ((unsigned long long)a << B) | b;
    vals[o] = (uint32_t)x;
    if (erow) erow[x] = a;  // working row of edge id x (caller order: coalesced)
  }
}

// Working out-degree of each rank r from the (a, b)-sorted edge keys: the
// length of r's key run (two lower bounds), instead of one atomic per edge.
__global__ void k_run_counts(const unsigned long long* __restrict__ keys, uint64_t m, uint32_t n, uint32_t B,
                             uint32_t* __restrict__ cnt) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x + 1; r <= n; r += gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = m;
    const unsigned long long k0 = (unsigned long long)r << B;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < k0) lo = mid + 1; else hi = mid;
    }
    const uint64_t first = lo;
    hi = m;
    const unsigned long long k1 = (unsigned long long)(r + 1) << B;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < k1) lo = mid + 1; else hi = mid;
    }
    cnt[r] = (uint32_t)(lo - first);
  }
}

// row sizes (out-degree + sentinel) for the working row_ptr scan
__global__ void k_row_sizes(const uint32_t* __restrict__ cnt, uint32_t n, uint32_t* __restrict__ sizes) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n + 2; i += gridDim.x * blockDim.x)
    sizes[i] = (i >= 1 && i <= n) ? cnt[i] + 1 : 0;
}

// sorted (key, caller slot) -> working col / id; slot = idx + a - 1 because
// every earlier row adds one sentinel.
__global__ void k_fill_working(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                               uint64_t m, uint32_t B, uint32_t* __restrict__ col_w, uint32_t* __restrict__ id_w) {
  const unsigned long long mask = (1ull << B) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const uint32_t a = (uint32_t)(k >> B);
    const uint64_t slot = i + a - 1;
    col_w[slot] = (uint32_t)(k & mask);
    id_w[slot] = vals[i];
  }
}

#ifndef KTG_FILL_UNROLL
#define KTG_FILL_UNROLL 4
#endif
constexpr int kFillUnroll = KTG_FILL_UNROLL;  // load-time fill passes: entries per thread per step

// Working layout + symmetric rows in one pass (carried-support runs): per
// rank r, din_w = undirected degree - out-degree; the u64 sizes for the
// symmetric-row offsets (tot | din) scans.
__global__ void k_sym_sizes(const uint32_t* __restrict__ symdeg_w, const uint32_t* __restrict__ cntw, uint32_t n,
                            uint32_t* __restrict__ din_w, unsigned long long* __restrict__ sz,
                            const uint32_t* __restrict__ row_ptr_w, uint32_t* __restrict__ rend) {
  const uint32_t nb = n + 2;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nb; r += gridDim.x * blockDim.x) {
    const uint32_t tot = (r >= 1 && r <= n) ? symdeg_w[r] : 0u;
    const uint32_t dout = (r >= 1 && r <= n) ? cntw[r] : 0u;
    din_w[r] = tot - dout;
    sz[r] = tot;
    sz[nb + r] = tot - dout;
    rend[r] = row_ptr_w[r] + dout;  // end of working row r's live part (k_fill_in_all's pin_end)
  }
}

// Sorted (a << B | b, caller slot) entry i of the working edges: writes the
// working col/id, pos_of of the edge id, the out-part of symmetric row
// a, and the in-list key (b, a << 32 | working slot) of entry i (entries stay
// in (a, b) order, so a stable sort by b alone yields ascending in-lists);
// totals the delta queue capacity (one task per kDeltaPiece elements of
// min(du, dv) per edge: degrees only shrink, so no round queues more).
__global__ void k_fill_all(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t m,
                           uint32_t B, const uint32_t* __restrict__ row_ptr_w, uint32_t* __restrict__ col_w,
                           uint32_t* __restrict__ id_w, const uint32_t* __restrict__ din_w,
                           const uint32_t* __restrict__ symdeg_w, Sym y, uint32_t* __restrict__ ikeys,
                           unsigned long long* __restrict__ ivals, unsigned long long* __restrict__ cap) {
  const unsigned long long mask = (1ull << B) - 1;
  unsigned long long c = 0;
  // kFillUnroll entries per thread per step, each phase's loads issued for
  // all of them before any use (the pass is latency-bound on the per-row
  // gathers and the scattered pos_of store, not on its streaming bytes)
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < m; i0 += kFillUnroll * stride) {
    unsigned long long k[kFillUnroll];
    uint32_t id[kFillUnroll], a[kFillUnroll], b[kFillUnroll];
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      k[u] = i < m ? keys[i] : 0ull;
      id[u] = i < m ? vals[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) a[u] = (uint32_t)(k[u] >> B), b[u] = (uint32_t)(k[u] & mask);
    unsigned long long base[kFillUnroll];
    uint32_t rw[kFillUnroll], da[kFillUnroll], db[kFillUnroll];
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) {
      if (i0 + u * stride < m) {
        base[u] = y.ptr[a[u]] + din_w[a[u]];
        rw[u] = row_ptr_w[a[u]];
        da[u] = symdeg_w[a[u]];
        db[u] = symdeg_w[b[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < m) {
        const uint32_t slot = (uint32_t)(i + a[u] - 1);
        col_w[slot] = b[u];
        id_w[slot] = id[u];
        y.pos_of[id[u]] = slot;  // erow[id] = a was written by k_edge_keys
        const unsigned long long dst = base[u] + (slot - rw[u]);
        y.nbr[dst] = b[u];
        y.eid[dst] = id[u];
        ikeys[i] = b[u];
        ivals[i] = ((unsigned long long)a[u] << 32) | slot;
        c += (min(da[u], db[u]) + kDeltaPiece - 1) / kDeltaPiece;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cap, c);
}

// Sorted in-list entry i (key b, value a << 32 | working slot): position
// i - inoff[b] of symmetric row b's in-part; also the i-th entry of the A22
// in-edge list (edge id) and its pristine {slot, row} record.
__global__ void k_fill_in_all(const uint32_t* __restrict__ vkeys, const unsigned long long* __restrict__ vals,
                              uint64_t m, const unsigned long long* __restrict__ inoff,
                              const uint32_t* __restrict__ id_w, Sym y, uint32_t* __restrict__ pe,
                              uint2* __restrict__ pin_p, uint32_t* __restrict__ pin_end,
                              const uint32_t* __restrict__ rend) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < m; i0 += kFillUnroll * stride) {
    uint32_t b[kFillUnroll], a[kFillUnroll], slot[kFillUnroll];
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      unsigned long long pv = 0;
      b[u] = 0;
      if (i < m) b[u] = vkeys[i], pv = vals[i];
      a[u] = (uint32_t)(pv >> 32), slot[u] = (uint32_t)pv;
    }
    uint32_t id[kFillUnroll], end[kFillUnroll];
    unsigned long long dst[kFillUnroll];
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < m) {
        id[u] = id_w[slot[u]];
        dst[u] = y.ptr[b[u]] + (i - inoff[b[u]]);
        end[u] = rend[a[u]];  // one gather (row_ptr_w + out-degree precombined)
      }
    }
#pragma unroll
    for (int u = 0; u < kFillUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < m) {
        y.nbr[dst[u]] = a[u];
        y.eid[dst[u]] = id[u];
        pe[i] = id[u];
        pin_p[i] = make_uint2(slot[u], a[u]);
        pin_end[i] = end[u];
      }
    }
  }
}

// Publish, step 1: every live working slot writes its caller slot's pristine
// column and its support into the (zeroed) caller arrays.
__global__ void k_scatter_live(Graph w, const uint32_t* __restrict__ col_pristine, uint32_t* __restrict__ col_out,
                               uint32_t* __restrict__ S_out, int add) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t* __restrict__ Sw = cur_S(w);
  for (uint32_t a = warp + 1; a <= w.n; a += nwarps) {
    const uint32_t d = w.deg[a], base = w.row_ptr[a];
    for (uint32_t x = lane; x < d; x += 32) {
      const uint32_t id = w.payload[base + x];
      if (col_out) col_out[id] = col_pristine[id];
      if (add) S_out[id] += Sw[base + x];
      else S_out[id] = Sw[base + x];
    }
  }
}

// ---------------------------------------------------------------------------
// Loop control
// ---------------------------------------------------------------------------
__global__ void k_begin(DevState* st, uint32_t threshold, uint32_t width16, int parity, uint32_t inc,
                        double delta_ratio, double delta_ratio0) {
  st->inc = inc;
  st->mode = 0;
  st->nrq = 0;
  st->carry = 0;
  st->fpar = 0;
  st->nfq[0] = st->nfq[1] = 0;
  st->nqrow = st->nqsym = 0;
  st->nheavy_sym = 0;
  st->h0 = 0;
  st->pristine = 0;
  st->live_cost = 0;
  st->delta_ratio = delta_ratio;
  st->delta_ratio0 = delta_ratio0;
  st->sum_s = 0;
  st->delta_cost = 0;
  st->keep_cost = 0;
  st->removed = 0;
  st->triangles = 0;
  st->last_triangles = 0;
  st->overflow_slot = ~0ull;
  st->parity = parity < 0 ? (st->parity ^ 1u) : (unsigned)parity;
  st->iter = 0;
  st->threshold = threshold;
  st->task_next = 0;
  st->nheavy = 0;
  st->error = 0;
  st->max_support = 0;
  st->width16 = width16;
}

// End of round: record removed, advance parity unless converged, and (graph
// mode) set the while-node condition -- no host round trip per iteration.
__global__ void k_control(DevState* st, unsigned long long* hist, cudaGraphConditionalHandle handle,
                          int use_cond) {
  const unsigned long long removed = st->removed;
  const uint32_t it = st->iter;
  if (it < (uint32_t)kHistCap) hist[it] = removed;
  st->iter = it + 1;
  st->live -= removed;
  st->last_triangles = st->triangles;
  st->triangles = 0;
  st->removed = 0;
  st->task_next = 0;
  st->nheavy = 0;
  const bool cont = removed != 0 && st->error == 0;
  if (cont) st->parity ^= 1u;
  if (use_cond) cudaGraphSetConditional(handle, cont ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// Per-round closed-form work, optional
// ---------------------------------------------------------------------------
// Live in-degree: slot-parallel (a row's live slots are its nonzero ones;
// label-order hub rows are too long for a warp per row).
__global__ void k_work_din(Graph g, uint32_t* __restrict__ din) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < g.slots;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = g.col[x];
    if (c) atomicAdd(&din[c], 1u);
  }
}

__global__ void k_work_L(Graph g, const uint32_t* __restrict__ din, unsigned long long* out) {
  unsigned long long L = 0, Lt = 0;  // L, and its a12-tail part sum_v d+(d+-1)/2
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x + 1; v <= g.n; v += gridDim.x * blockDim.x) {
    const unsigned long long d = g.deg[v];
    const unsigned long long t = d * (d ? d - 1 : 0) / 2;
    L += t + d * din[v];
    Lt += t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    L += __shfl_xor_sync(0xffffffffu, L, o);
    Lt += __shfl_xor_sync(0xffffffffu, Lt, o);
  }
  if ((threadIdx.x & 31) == 0 && L) atomicAdd(out, L);
  if ((threadIdx.x & 31) == 0 && Lt) atomicAdd(out + 1, Lt);
}

// ---------------------------------------------------------------------------
// Extraction (extract_edges, csr.cpp:93-106): survivors as (u, v, S)
// ---------------------------------------------------------------------------
__global__ void k_extract(Graph g, const uint32_t* __restrict__ S, const unsigned long long* __restrict__ offs,
                          uint32_t* __restrict__ u, uint32_t* __restrict__ v, uint32_t* __restrict__ sup) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = warp + 1; r <= g.n; r += nwarps) {
    const uint32_t d = g.deg[r], base = g.row_ptr[r];
    const unsigned long long o = offs[r];
    for (uint32_t x = lane; x < d; x += 32) {
      u[o + x] = r;
      v[o + x] = g.col[base + x];
      sup[o + x] = S[base + x];
    }
  }
}

}  // namespace ktg
