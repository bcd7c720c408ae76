// B200-native Eager K-truss engine: device-resident state, the fixpoint
// driver and the C ABI declared in include/ktg.h.
//
// Two CSR layouts live on the device:
//   caller layout  -- the reference's zero-terminated, label-ordered CSR
//                     exactly as passed in (csr.hpp:17-23); outputs are
//                     always returned in it;
//   working layout -- the same graph re-oriented by ascending (degree, id)
//                     rank, carrying each entry's caller
//                     slot id. Supports and truss membership do not depend
//                     on orientation, and every prune is a stable per-row
//                     compaction, so the fixpoint runs here (L is 4.3x
//                     smaller at R-MAT s20, max out-degree 672 vs 43,600)
//                     and the caller layout is rebuilt once at convergence
//                     ("publish": scatter survivors + stable compaction).
//                     Byte-identical to running on the caller layout.
// KTG_FLAG_LABEL_ORDER or an observer runs on the caller layout directly.
//
// Loop structure (run_fixpoint, /root/reference/proj/src/truss.cpp:41-53):
//   graph mode (default): one CUDA graph whose single node is a conditional
//     WHILE node; its body is {plan, support, [check16], prune, control}. The
//     control kernel records the round's removal count and sets the while
//     condition on the device (cudaGraphSetConditional), so a whole fixpoint
//     is one graph launch with no host synchronisation per round.
//   host mode (observer, multi-GPU all-reduce, work statistics): the same
//     kernels launched per round from the host, reading `removed` back.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/ktg.h"
#include "ktg_kernels.cuh"

using namespace ktg;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_err_slot = 0;

ktg_status fail(ktg_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define KTG_CUDA(call)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      return fail(_e == cudaErrorMemoryAllocation ? KTG_ERR_OOM : KTG_ERR_CUDA,              \
                  std::string(#call) + ": " + cudaGetErrorString(_e));                       \
    }                                                                                        \
  } while (0)

#define KTG_TRY(expr)                  \
  do {                                 \
    ktg_status _s = (expr);            \
    if (_s != KTG_OK) return _s;       \
  } while (0)

// Growable device buffer (allocations are reused across loads).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;  // bytes
  ktg_status ensure(size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (p && cap >= bytes) return KTG_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    KTG_CUDA(cudaMalloc(&p, bytes));
    cap = bytes;
    return KTG_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// NCCL, loaded on first use (dlopen, so the library has no link-time NCCL
// dependency; under PyTorch this resolves to the already-loaded libnccl.so.2).
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.errorString;
    }
  }
  return api.ok ? &api : nullptr;
}

// One CSR orientation resident in HBM.
struct Layout {
  uint32_t n = 0;
  uint64_t slots = 0;
  uint32_t nchunks = 0;
  uint64_t live_pristine = 0;
  bool ready = false;
  bool has_pristine = false;
  bool has_payload = false;
  DBuf<uint32_t> row_ptr, col, col_p, S0, S1, deg, deg_p, chunk_row, pair_counts, heavy, id, id_p;
  DBuf<uint2> pairs;
  void release() {
    for (DBuf<uint32_t>* b : {&row_ptr, &col, &col_p, &S0, &S1, &deg, &deg_p, &chunk_row, &pair_counts, &heavy,
                              &id, &id_p})
      b->release();
    pairs.release();
    ready = false;
  }
};

}  // namespace

struct ktg_engine {
  ktg_options opt{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;

  Layout cl;               // caller layout
  Layout wl;               // degree-ordered working layout
  bool reoriented = false; // fixpoints of the current graph run on wl
  bool caller_stale = false;

  // reorientation / statistics scratch
  DBuf<uint32_t> din, rank, offs, cntw, sizes, vals, vals_sorted, symdeg_w;
  DBuf<unsigned long long> keys, keys_sorted, ex_offs;
  DBuf<unsigned char> cub_tmp;
  DBuf<uint32_t> ex_out;
  DBuf<unsigned long long> orig_ids;
  bool has_orig_ids = false;

  // incremental rounds: symmetric adjacency of the working layout (+ pristine
  // copies), per-edge dead flags and positions, delta task queue
  DBuf<unsigned long long> sym_ptr, sym_sizes;
  DBuf<unsigned long long> task_cost, task_pre;  // multi-GPU task split (per chunk)
  DBuf<uint32_t> sym_nbr, sym_eid, sym_nbr_p, sym_eid_p, sym_deg, sym_deg_p, pos_of, pos_of_p, erow, qsym,
      qrow, fq0, fq1, sym_heavy;
  DBuf<uint8_t> dead, rdirty, sdirty;
  DBuf<uint4> rq;
  uint64_t sym_entries = 0, rq_cap = 0;
  // A22-staged support pass: in-edge ids by j, their offsets, chunk first
  // rows, (chunk, batch) tasks
  DBuf<uint32_t> a22_pe, a22_off, a22_jfirst, a22_cnt;
  DBuf<uint2> a22_tasks, a22_pin;
  DBuf<uint32_t> a22_pin_end;  // pristine pivots: end of the pivot row's live part
  uint32_t a22_ntasks = 0;
  // multi-rank full passes: per-task work (k_support_a22<true>) and its
  // exclusive prefix (ntasks + 1 entries; cost[ntasks] stays 0)
  DBuf<unsigned long long> a22_cost, a22_pre;
  uint32_t a22_lo = 0, a22_hi = 0;  // this rank's task range (world > 1)
  bool a22_ready = false;
  bool a22_off_env = false;   // KTG_SUPPORT=chunked: keep k_support_chunked in carried runs
  int a22_grid = 0;
  size_t a22_smem = 0;
  bool sym_ready = false;
  bool inc_active = false;    // the current fixpoint carries supports
  bool pristine = false;      // the working layout holds the pristine graph (after load / reset)
  double delta_ratio = 0.0625;  // carry when delta_cost <= ratio * keep_cost (s20 sweep calibration, scripts/ratio_scan.py)
  double delta_ratio0 = 0.03;   // the same for round 0 from the pristine graph (same calibration)

  unsigned long long* d_workL = nullptr;
  DevState* d_st = nullptr;
  unsigned long long* d_hist = nullptr;
  DevState* h_st = nullptr;  // pinned mirror

  int support_grid = 0;
  int prune_grid = 0;
  int heavy_grid = 0;
  size_t support_smem = 0;

  cudaGraphExec_t exec = nullptr;
  const void* exec_key[4] = {nullptr, nullptr, nullptr, nullptr};
  uint64_t exec_key2[4] = {0, 0, 0, 0};

  uint32_t rank_id = 0, world = 1;
  uint32_t scan_ratio = kScanRatio;
  ktg_allreduce_cb allreduce = nullptr;
  void* allreduce_user = nullptr;
  // fused reduce-scatter (ktg_engine_set_peers): [S0 of every rank | S1 of
  // every rank] as device pointers, the owned span, the exchange callback
  DBuf<uint32_t*> peer_tab;
  uint32_t npeer = 0;
  uint64_t peer_span = 0;
  ktg_peer_cb peer_cb = nullptr;
  void* peer_user = nullptr;
  ncclComm_t nccl = nullptr;
  // peer group (ktg_engine_set_group): own exchange area, device tables of
  // every rank's area and support buffers, list capacity, reduce span
  bool group = false;
  DBuf<unsigned char> xarea;
  DBuf<void*> xtab;
  uint64_t xcap = 0, xspan = 0;

  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;
  bool ran = false;  // a fixpoint has recorded ev0 / ev1
  ktg_run_info info{};
  std::vector<ktg_round_work> work;

  Layout& act() { return reoriented ? wl : cl; }

  Graph graph_of(Layout& L) const {
    Graph g;
    g.row_ptr = L.row_ptr.p;
    g.col = L.col.p;
    g.S0 = L.S0.p;
    g.S1 = L.S1.p;
    g.deg = L.deg.p;
    g.chunk_row = L.chunk_row.p;
    g.pairs = L.pairs.p;
    g.pair_counts = L.pair_counts.p;
    g.heavy_rows = L.heavy.p;
    g.st = d_st;
    g.hist = d_hist;
    g.n = L.n;
    g.nchunks = L.nchunks;
    g.slots = L.slots;
    g.rank = rank_id;
    g.world = world;
    g.scan_ratio = scan_ratio;
    g.payload = L.has_payload ? L.id.p : nullptr;
    g.peer0 = npeer ? peer_tab.p : nullptr;
    g.peer1 = npeer ? peer_tab.p + npeer : nullptr;
    g.span = peer_span;
    g.npeer = npeer;
    g.xa = (group && world > 1) ? reinterpret_cast<XArea*>(xarea.p) : nullptr;
    g.xcap = xcap;
    g.a22_lo = a22_lo;
    g.a22_hi = a22_hi;
    return g;
  }

  Sym sym() {
    Sym y;
    y.ptr = sym_ptr.p;
    y.nbr = sym_nbr.p;
    y.eid = sym_eid.p;
    y.deg = sym_deg.p;
    y.dead = dead.p;
    y.rdirty = rdirty.p;
    y.sdirty = sdirty.p;
    y.qsym = qsym.p;
    y.qrow = qrow.p;
    y.heavy = sym_heavy.p;
    y.pos_of = pos_of.p;
    y.erow = erow.p;
    y.fq0 = fq0.p;
    y.fq1 = fq1.p;
    y.rq = rq.p;
    return y;
  }

  XGroup xgroup() {
    XGroup x;
    void** t = xtab.p;
    x.area = reinterpret_cast<XArea* const*>(t);
    x.S0 = reinterpret_cast<uint32_t* const*>(t + world);
    x.S1 = reinterpret_cast<uint32_t* const*>(t + 2 * (size_t)world);
    x.rank = rank_id;
    x.world = world;
    x.cap = xcap;
    x.span = xspan;
    return x;
  }

  // The carried-support structures only (symmetric rows, per-edge maps,
  // frontier / delta queues, A22 plan).
  void release_sym() {
    for (DBuf<uint32_t>* b : {&sym_nbr, &sym_eid, &sym_nbr_p, &sym_eid_p, &sym_deg, &sym_deg_p, &pos_of, &pos_of_p,
                              &erow, &qsym, &qrow, &fq0, &fq1, &sym_heavy, &a22_pe, &a22_off, &a22_jfirst,
                              &a22_cnt})
      b->release();
    sym_ptr.release();
    sym_sizes.release();
    dead.release();
    rdirty.release();
    sdirty.release();
    rq.release();
    a22_tasks.release();
    a22_pin.release();
    a22_pin_end.release();
    a22_cost.release();
    a22_pre.release();
    sym_ready = false;
    a22_ready = false;
  }

  void free_all() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    cl.release();
    wl.release();
    for (DBuf<uint32_t>* b : {&din, &rank, &offs, &cntw, &sizes, &vals, &vals_sorted, &symdeg_w, &ex_out})
      b->release();
    keys.release();
    keys_sorted.release();
    ex_offs.release();
    orig_ids.release();
    cub_tmp.release();
    for (DBuf<uint32_t>* b : {&sym_nbr, &sym_eid, &sym_nbr_p, &sym_eid_p, &sym_deg, &sym_deg_p, &pos_of, &pos_of_p,
                              &erow, &qsym, &qrow, &fq0, &fq1, &sym_heavy, &a22_pe, &a22_off, &a22_jfirst,
                              &a22_cnt})
      b->release();
    sym_ptr.release();
    sym_sizes.release();
    task_cost.release();
    task_pre.release();
    peer_tab.release();
    xarea.release();
    xtab.release();
    group = false;
    dead.release();
    rdirty.release();
    sdirty.release();
    rq.release();
    a22_tasks.release();
    a22_cost.release();
    a22_pre.release();
    a22_pin.release();
    a22_pin_end.release();
    sym_ready = false;
    a22_ready = false;
  }
};

namespace {

bool flag(const ktg_engine* e, uint32_t f) { return (e->opt.flags & f) != 0; }

ktg_status engine_init(const ktg_options* opt, ktg_engine* e) {
  if (opt) {
    if (opt->struct_size != sizeof(ktg_options))
      return fail(KTG_ERR_INVALID_PARAMETER, "ktg_options.struct_size mismatch");
    e->opt = *opt;
  } else {
    ktg_options_init(&e->opt);
  }
  if (e->opt.width_bits != 32 && e->opt.width_bits != 16)
    return fail(KTG_ERR_INVALID_PARAMETER, "width_bits must be 16 or 32");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(KTG_ERR_NO_DEVICE, "no CUDA device visible (the engine has no CPU fallback)");
  }
  if (e->opt.device >= 0) KTG_CUDA(cudaSetDevice(e->opt.device));
  KTG_CUDA(cudaGetDevice(&e->device));
  cudaDeviceProp prop;
  KTG_CUDA(cudaGetDeviceProperties(&prop, e->device));
  if (prop.major != 10)
    return fail(KTG_ERR_NO_DEVICE, std::string("device ") + prop.name +
                                       " is not sm_100 (this build targets sm_100a only)");
  e->num_sms = prop.multiProcessorCount;
  if (const char* r = getenv("KTG_SCAN_RATIO")) e->scan_ratio = (uint32_t)std::max(1, atoi(r));
  if (const char* r = getenv("KTG_DELTA_RATIO")) e->delta_ratio = e->delta_ratio0 = std::max(0.0, atof(r));
  if (const char* r = getenv("KTG_DELTA_RATIO0")) e->delta_ratio0 = std::max(0.0, atof(r));
  if (e->opt.stream) {
    e->stream = static_cast<cudaStream_t>(e->opt.stream);
  } else {
    KTG_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    e->own_stream = true;
  }
  KTG_CUDA(cudaMalloc(&e->d_st, sizeof(DevState)));
  KTG_CUDA(cudaMemset(e->d_st, 0, sizeof(DevState)));
  KTG_CUDA(cudaMalloc(&e->d_hist, sizeof(unsigned long long) * kHistCap));
  KTG_CUDA(cudaMalloc(&e->d_workL, 2 * sizeof(unsigned long long)));
  KTG_CUDA(cudaMallocHost(&e->h_st, sizeof(DevState)));
  std::memset(e->h_st, 0, sizeof(DevState));
  KTG_CUDA(cudaEventCreate(&e->ev0));
  KTG_CUDA(cudaEventCreate(&e->ev1));
  KTG_CUDA(cudaEventCreate(&e->evs0));
  KTG_CUDA(cudaEventCreate(&e->evs1));

  e->support_smem = sizeof(SupportSmem);
  KTG_CUDA(cudaFuncSetAttribute(k_support_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)e->support_smem));
  int per_sm = 0;
  KTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_support_chunked, kSupportThreads,
                                                         e->support_smem));
  e->support_grid = std::max(1, per_sm) * e->num_sms;
  int per_sm_p = 0;
  KTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_p, k_prune_light<0>, kPruneThreads, 0));
  e->prune_grid = std::max(1, per_sm_p) * e->num_sms;
  e->heavy_grid = 2 * e->num_sms;
  e->a22_smem = 0;  // static shared memory (sizeof(A22Smem) < 48 KB)
  int per_sm_a = 0;
  // L1 / shared-memory split of the A22 pass: the driver's default keeps the
  // rest of the SM's 256 KB as L1, which caches the re-read tail rows (a
  // forced 100% carveout measured 163 -> 227 ms per s24 pass); the
  // KTG_A22_CARVEOUT env knob (percent) is for A/B runs only
  if (const char* cv = std::getenv("KTG_A22_CARVEOUT")) {
    const int pct = std::atoi(cv);
    KTG_CUDA(cudaFuncSetAttribute(k_support_a22<false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    KTG_CUDA(cudaFuncSetAttribute(k_support_a22<true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  }
  KTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_a, k_support_a22<false>, kSupportThreads, e->a22_smem));
  e->a22_grid = std::max(1, per_sm_a) * e->num_sms;
  if (const char* v = getenv("KTG_SUPPORT")) e->a22_off_env = std::string(v) == "chunked";
  return KTG_OK;
}

ktg_status read_state(ktg_engine* e) {
  KTG_CUDA(cudaMemcpyAsync(e->h_st, e->d_st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  return KTG_OK;
}

__global__ void k_set_live(DevState* st, unsigned long long live) { st->live = live; }
__global__ void k_reset_state(DevState* st) {
  const unsigned int ep = st->xepoch;
  DevState z{};
  *st = z;
  st->xepoch = ep;
}
__global__ void k_set_rqcap(DevState* st, unsigned long long cap) { st->rq_cap = cap; }
__global__ void k_clear_heavy(DevState* st) { st->nheavy = 0; }

// Per-layout structures once L.row_ptr / L.col hold a CSR: live degrees,
// chunk rows, off-diagonal task capacity, pristine copies.
ktg_status prepare_layout(ktg_engine* e, Layout& L, bool keep_pristine, const uint32_t* known_deg = nullptr,
                          uint64_t known_live = 0) {
  const size_t nb = (size_t)L.n + 2;
  const size_t sb = L.slots + 4;  // +16 B: vector-load padding
  L.nchunks = (uint32_t)((L.slots + kChunk - 1) / kChunk);
  KTG_TRY(L.S0.ensure(sb));
  KTG_TRY(L.S1.ensure(sb));
  KTG_TRY(L.deg.ensure(nb));
  KTG_TRY(L.deg_p.ensure(nb));
  KTG_TRY(L.chunk_row.ensure(L.nchunks));
  KTG_TRY(L.pair_counts.ensure(L.nchunks));
  KTG_TRY(L.heavy.ensure(nb));
  KTG_CUDA(cudaMemsetAsync(L.col.p + L.slots, 0, 16, e->stream));
  KTG_CUDA(cudaMemsetAsync(L.S0.p, 0, sb * 4, e->stream));
  KTG_CUDA(cudaMemsetAsync(L.S1.p, 0, sb * 4, e->stream));
  // fresh loop state; the peer-group barrier epoch survives (the peers'
  // flags in this engine's exchange area hold epochs of earlier barriers)
  k_reset_state<<<1, 1, 0, e->stream>>>(e->d_st);
  if (known_deg) {  // the builder counted every row (working layout: out-degrees)
    KTG_CUDA(cudaMemcpyAsync(L.deg.p, known_deg, nb * 4, cudaMemcpyDeviceToDevice, e->stream));
    k_set_live<<<1, 1, 0, e->stream>>>(e->d_st, known_live);
  } else {
    KTG_CUDA(cudaMemsetAsync(L.deg.p, 0, nb * 4, e->stream));
    k_row_deg<<<(L.n + 255) / 256, 256, 0, e->stream>>>(L.row_ptr.p, L.col.p, L.n, L.deg.p, e->d_st);
  }
  k_chunk_rows<<<(L.nchunks + 255) / 256, 256, 0, e->stream>>>(L.row_ptr.p, L.n, L.slots, L.nchunks,
                                                              L.chunk_row.p);
  KTG_CUDA(cudaGetLastError());
  KTG_CUDA(cudaMemcpyAsync(L.deg_p.p, L.deg.p, nb * 4, cudaMemcpyDeviceToDevice, e->stream));
  L.has_pristine = keep_pristine;
  if (keep_pristine) {
    KTG_TRY(L.col_p.ensure(sb));
    KTG_CUDA(cudaMemcpyAsync(L.col_p.p, L.col.p, sb * 4, cudaMemcpyDeviceToDevice, e->stream));
    if (L.has_payload) {
      KTG_TRY(L.id_p.ensure(sb));
      KTG_CUDA(cudaMemcpyAsync(L.id_p.p, L.id.p, L.slots * 4, cudaMemcpyDeviceToDevice, e->stream));
    }
  }
  // The pristine plan is the largest (live ends only shrink as rows are
  // pruned); k_plan_count totals it on the device.
  Graph g = e->graph_of(L);
  k_plan_count<<<(L.nchunks + 255) / 256, 256, 0, e->stream>>>(g, 1);
  KTG_CUDA(cudaGetLastError());
  KTG_TRY(read_state(e));
  KTG_TRY(L.pairs.ensure(e->h_st->pairs_needed));
  L.live_pristine = e->h_st->live;
  L.ready = true;
  return KTG_OK;
}

// KTG_LOAD_TIMING=1: per-phase wall times of the host-buffer path on stderr
// (debug; synchronises the stream at every mark, so never on in a benchmark).
struct PhaseTimer {
  cudaStream_t s;
  bool on;
  double last = 0;
  explicit PhaseTimer(cudaStream_t st) : s(st), on(getenv("KTG_LOAD_TIMING") != nullptr) {}
  void operator()(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double now =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (last != 0) fprintf(stderr, "ktg: %-28s %8.3f ms\n", what, now - last);
    last = now;
  }
};

ktg_status sym_alloc(ktg_engine* e, uint64_t m);

// Degree-ordered working layout from the caller layout's current state; with
// `with_sym` (carried-support runs) the same pass also writes the symmetric
// rows, pos_of/erow and the A22 in-edge list (build_sym finishes them).
ktg_status build_working(ktg_engine* e, bool with_sym) {
  Layout& C = e->cl;
  Layout& W = e->wl;
  const uint32_t n = C.n;
  const uint64_t m = C.live_pristine;  // live edges of the loaded caller CSR
  const size_t nb = (size_t)n + 2;
  W.n = n;
  W.slots = m + n;
  W.has_payload = true;
  KTG_TRY(W.row_ptr.ensure(nb));
  KTG_TRY(W.col.ensure(W.slots + 4));
  KTG_TRY(W.id.ensure(W.slots + 4));
  KTG_TRY(e->din.ensure(nb));
  KTG_TRY(e->rank.ensure(nb));
  KTG_TRY(e->offs.ensure(nb));
  KTG_TRY(e->cntw.ensure(nb));
  KTG_TRY(e->sizes.ensure(nb));
  KTG_TRY(e->symdeg_w.ensure(nb));
  KTG_TRY(e->keys.ensure(std::max<uint64_t>(m, n)));
  KTG_TRY(e->keys_sorted.ensure(std::max<uint64_t>(m, n)));
  KTG_TRY(e->vals.ensure(m));
  KTG_TRY(e->vals_sorted.ensure(m));
  Graph g = e->graph_of(C);
  const cudaStream_t s = e->stream;
  // undirected degree = out (deg) + in (din)
  KTG_CUDA(cudaMemsetAsync(e->din.p, 0, nb * 4, s));
  KTG_CUDA(cudaMemsetAsync(e->cntw.p, 0, nb * 4, s));
  KTG_CUDA(cudaMemsetAsync(e->symdeg_w.p, 0, nb * 4, s));
  PhaseTimer mk(s);
  mk("bw start");
  k_work_din<<<e->prune_grid, kPruneThreads, 0, s>>>(g, e->din.p);
  k_rank_keys<<<4 * e->num_sms, 256, 0, s>>>(C.deg.p, e->din.p, n, e->keys.p);
  KTG_CUDA(cudaGetLastError());
  // ranks: sort (degree, id) ascending
  uint32_t deg_bits = 1;
  while ((1ull << deg_bits) <= 2ull * m + 1) ++deg_bits;
  size_t tmp = 0, tmp2 = 0, tmp3 = 0;
  KTG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, e->keys.p, e->keys_sorted.p, (int)n, 0, 32 + deg_bits, s));
  uint32_t B = 1;
  while ((1ull << B) <= n) ++B;
  KTG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, e->keys.p, e->keys_sorted.p, e->vals.p,
                                           e->vals_sorted.p, (int64_t)m, 0, 2 * B, s));
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp3, e->sizes.p, W.row_ptr.p, (int)nb, s));
  tmp = std::max(tmp, std::max(tmp2, tmp3));
  if (with_sym) {
    size_t t4 = 0, t5 = 0;
    KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t4, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                           (int)nb, s));
    // in-lists: a STABLE sort of the working edges (emitted in (a, b) order)
    // by b alone keeps every in-list ascending in a -- B key bits, not 2B
    KTG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t5, e->vals.p, e->vals_sorted.p, e->keys.p,
                                             e->keys_sorted.p, (int64_t)m, 0, (int)B, s));
    tmp = std::max(tmp, std::max(t4, t5));
  }
  KTG_TRY(e->cub_tmp.ensure(tmp));
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceRadixSort::SortKeys(e->cub_tmp.p, tmp, e->keys.p, e->keys_sorted.p, (int)n, 0,
                                          32 + deg_bits, s));
  k_rank_assign<<<4 * e->num_sms, 256, 0, s>>>(e->keys_sorted.p, n, e->rank.p, e->symdeg_w.p);
  mk("bw: degrees + rank sort");
  // edge keys in caller row order, then sort by (a, b)
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, C.deg.p, e->offs.p, (int)nb, s));
  if (with_sym) {
    KTG_TRY(sym_alloc(e, m));
    // pos_of is indexed by caller slot: sentinel slots are never written by
    // k_fill_all; define them (initcheck-clean pristine copy)
    KTG_CUDA(cudaMemsetAsync(e->pos_of.p, 0xff, C.slots * 4, s));
  }
  k_edge_keys<<<e->prune_grid, kPruneThreads, 0, s>>>(g, e->rank.p, e->offs.p, B, e->keys.p, e->vals.p,
                                                      with_sym ? e->erow.p : nullptr);
  KTG_CUDA(cudaGetLastError());
  mk("bw: edge keys");
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceRadixSort::SortPairs(e->cub_tmp.p, tmp, e->keys.p, e->keys_sorted.p, e->vals.p,
                                           e->vals_sorted.p, (int64_t)m, 0, 2 * B, s));
  mk("bw: (a, b) sort");
  k_run_counts<<<(n + 255) / 256, 256, 0, s>>>(e->keys_sorted.p, m, n, B, e->cntw.p);
  // working row_ptr = exclusive scan of (out-degree + sentinel)
  k_row_sizes<<<4 * e->num_sms, 256, 0, s>>>(e->cntw.p, n, e->sizes.p);
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, e->sizes.p, W.row_ptr.p, (int)nb, s));
  KTG_CUDA(cudaMemsetAsync(W.col.p, 0, W.slots * 4, s));
  KTG_CUDA(cudaMemsetAsync(W.id.p, 0, W.slots * 4, s));  // sentinel slots carry id 0 (initcheck-clean copies)
  mk("bw: row sizes + scan");
  if (!with_sym) {
    k_fill_working<<<8 * e->num_sms, 256, 0, s>>>(e->keys_sorted.p, e->vals_sorted.p, m, B, W.col.p, W.id.p);
    KTG_CUDA(cudaGetLastError());
    return prepare_layout(e, W, true, e->cntw.p, m);
  }
  unsigned long long* sz = e->sym_sizes.p;  // [tot | din | - | inoff | -] x nb
  // (e->sizes is free after the row_ptr scan: it takes the working row ends)
  k_sym_sizes<<<4 * e->num_sms, 256, 0, s>>>(e->symdeg_w.p, e->cntw.p, n, e->din.p, sz, W.row_ptr.p, e->sizes.p);
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, sz, e->sym_ptr.p, (int)nb, s));
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, sz + nb, sz + 3 * nb, (int)nb, s));
  KTG_CUDA(cudaMemsetAsync(e->d_workL, 0, 8, s));
  Sym y = e->sym();
  k_fill_all<<<8 * e->num_sms, 256, 0, s>>>(e->keys_sorted.p, e->vals_sorted.p, m, B, W.row_ptr.p, W.col.p,
                                            W.id.p, e->din.p, e->symdeg_w.p, y, e->vals.p, e->keys.p,
                                            e->d_workL);
  KTG_CUDA(cudaGetLastError());
  mk("bw: fill rows + sym");
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceRadixSort::SortPairs(e->cub_tmp.p, tmp, e->vals.p, e->vals_sorted.p, e->keys.p,
                                           e->keys_sorted.p, (int64_t)m, 0, (int)B, s));
  mk("bw: in-list sort");
  k_fill_in_all<<<8 * e->num_sms, 256, 0, s>>>(e->vals_sorted.p, e->keys_sorted.p, m, sz + 3 * nb, W.id.p, y,
                                               e->a22_pe.p, e->a22_pin.p, e->a22_pin_end.p, e->sizes.p);
  KTG_CUDA(cudaGetLastError());
  KTG_CUDA(cudaMemcpyAsync(e->sym_deg.p, e->symdeg_w.p, nb * 4, cudaMemcpyDeviceToDevice, s));
  mk("bw: in-list fill");
  const ktg_status pst = prepare_layout(e, W, true, e->cntw.p, m);
  mk("bw: prepare working layout");
  return pst;
}

// Static structures of the A22-staged support pass (after build_sym): the
// pristine in-lists as edge ids, each chunk's first row, (chunk, batch) tasks.
ktg_status build_a22(ktg_engine* e) {
  Layout& W = e->wl;
  const uint32_t n = W.n;
  const uint64_t m = W.live_pristine;
  const size_t nb = (size_t)n + 2;
  const uint32_t Q = W.nchunks;
  const cudaStream_t s = e->stream;
  e->a22_ready = false;
  KTG_TRY(e->a22_pin.ensure(m));
  KTG_TRY(e->a22_off.ensure(nb));
  KTG_TRY(e->a22_jfirst.ensure(Q));
  KTG_TRY(e->a22_cnt.ensure((size_t)Q + 1));
  Sym y = e->sym();
  // a22_pe (the sorted in-list ids) and a22_pin were written by k_fill_in_all
  k_u64_to_u32<<<4 * e->num_sms, 256, 0, s>>>(e->sym_sizes.p + 3 * nb, (uint32_t)nb, e->a22_off.p);
  k_chunk_first<<<(Q + 255) / 256, 256, 0, s>>>(W.row_ptr.p, n, W.slots, Q, e->a22_jfirst.p);
  k_a22_count<<<(Q + 256) / 256, 256, 0, s>>>(e->a22_jfirst.p, W.chunk_row.p, e->a22_off.p, Q, e->a22_cnt.p);
  KTG_CUDA(cudaGetLastError());
  size_t tmp = 0;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, e->a22_cnt.p, e->a22_cnt.p, (int)Q + 1, s));
  KTG_TRY(e->cub_tmp.ensure(tmp));
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, e->a22_cnt.p, e->a22_cnt.p, (int)Q + 1, s));
  uint32_t total = 0;
  KTG_CUDA(cudaMemcpyAsync(&total, e->a22_cnt.p + Q, 4, cudaMemcpyDeviceToHost, s));
  KTG_CUDA(cudaStreamSynchronize(s));
  KTG_TRY(e->a22_tasks.ensure(std::max<uint32_t>(total, 1)));
  k_a22_fill<<<(Q + 255) / 256, 256, 0, s>>>(e->a22_cnt.p, Q, e->a22_tasks.p);
  KTG_CUDA(cudaGetLastError());
  e->a22_ntasks = total;
  // the multi-rank split's buffers (and scan scratch) exist before any
  // fixpoint is captured into a graph
  KTG_TRY(e->a22_cost.ensure((size_t)total + 1));
  KTG_TRY(e->a22_pre.ensure((size_t)total + 1));
  KTG_CUDA(cudaMemsetAsync(e->a22_cost.p, 0, ((size_t)total + 1) * 8, s));
  tmp = 0;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, e->a22_cost.p, e->a22_pre.p, (int)total + 1, s));
  KTG_TRY(e->cub_tmp.ensure(tmp));
  e->a22_ready = true;
  return KTG_OK;
}

__global__ void k_cost_state(DevState* st) {  // a pristine full-pass round for the cost pass
  st->mode = 0;
  st->pristine = 1;
  st->h0 = 0;
  st->task_next = 0;
}

// Multi-rank runs: split the A22 tasks across ranks by the exact work of
// every task on the pristine graph (steps 1-2 of the pass over all tasks,
// prefix sum, k_a22_split), once per load or partition change. Round 0 of
// every fixpoint from pristine is the dominant full pass; later full passes
// reuse the split (balance approximate, results exact either way). The loop
// state fields touched are reset by k_begin before every run.
ktg_status a22_rank_split(ktg_engine* e) {
  e->a22_lo = 0;
  e->a22_hi = e->a22_ntasks;
  if (e->world <= 1 || !e->a22_ready || !e->reoriented) return KTG_OK;
  Layout& W = e->wl;
  Graph g = e->graph_of(W);
  const cudaStream_t s = e->stream;
  A22 a{e->a22_pe.p, e->a22_pin.p, e->a22_pin_end.p, e->a22_off.p, e->a22_jfirst.p, e->a22_tasks.p, e->a22_ntasks};
  k_cost_state<<<1, 1, 0, s>>>(e->d_st);
  k_support_a22<true><<<e->a22_grid, kSupportThreads, e->a22_smem, s>>>(g, e->sym(), a, e->a22_cost.p);
  size_t tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, e->a22_cost.p, e->a22_pre.p, (int)e->a22_ntasks + 1, s));
  k_a22_split<<<1, 1, 0, s>>>(e->d_st, e->a22_pre.p, e->a22_ntasks, e->rank_id, e->world);
  KTG_CUDA(cudaGetLastError());
  KTG_TRY(read_state(e));
  e->a22_lo = e->h_st->a22_lo;
  e->a22_hi = e->h_st->a22_hi;
  if (e->exec) cudaGraphExecDestroy(e->exec);  // the range is baked into the graph's kernel arguments
  e->exec = nullptr;
  return KTG_OK;
}

// Buffers of the symmetric adjacency (build_working fills them when it
// builds with_sym): row v = sorted in-neighbours ++ out-neighbours (working
// row v), each with the edge id; pos_of / erow per edge id; the A22 in-edge
// list and its pristine {slot, row} records.
ktg_status sym_alloc(ktg_engine* e, uint64_t m) {
  const size_t nb = (size_t)e->cl.n + 2;
  e->sym_ready = false;
  e->sym_entries = 2 * m;
  KTG_TRY(e->sym_ptr.ensure(nb));
  KTG_TRY(e->sym_sizes.ensure(5 * nb));
  KTG_TRY(e->sym_nbr.ensure(2 * m));
  KTG_TRY(e->sym_eid.ensure(2 * m));
  KTG_TRY(e->sym_nbr_p.ensure(2 * m));
  KTG_TRY(e->sym_eid_p.ensure(2 * m));
  KTG_TRY(e->sym_deg.ensure(nb));
  KTG_TRY(e->sym_deg_p.ensure(nb));
  KTG_TRY(e->rdirty.ensure(nb));
  KTG_TRY(e->sdirty.ensure(nb));
  KTG_TRY(e->qsym.ensure(nb));
  KTG_TRY(e->qrow.ensure(nb));
  KTG_TRY(e->sym_heavy.ensure(nb));
  KTG_TRY(e->fq0.ensure(m));
  KTG_TRY(e->fq1.ensure(m));
  KTG_TRY(e->pos_of.ensure(e->cl.slots));
  KTG_TRY(e->pos_of_p.ensure(e->cl.slots));
  KTG_TRY(e->erow.ensure(e->cl.slots));
  KTG_TRY(e->dead.ensure(e->cl.slots));
  KTG_TRY(e->a22_pe.ensure(m));
  KTG_TRY(e->a22_pin.ensure(m));
  KTG_TRY(e->a22_pin_end.ensure(m));
  return KTG_OK;
}

// Finishes the symmetric adjacency written by build_working(with_sym):
// pristine copies, per-round flags, the delta queue capacity k_fill_all
// totalled, then the A22 plan.
ktg_status build_sym(ktg_engine* e) {
  const uint64_t m = e->wl.live_pristine;
  const size_t nb = (size_t)e->cl.n + 2;
  const cudaStream_t s = e->stream;
  KTG_CUDA(cudaMemcpyAsync(e->sym_nbr_p.p, e->sym_nbr.p, 2 * m * 4, cudaMemcpyDeviceToDevice, s));
  KTG_CUDA(cudaMemcpyAsync(e->sym_eid_p.p, e->sym_eid.p, 2 * m * 4, cudaMemcpyDeviceToDevice, s));
  KTG_CUDA(cudaMemcpyAsync(e->sym_deg_p.p, e->sym_deg.p, nb * 4, cudaMemcpyDeviceToDevice, s));
  KTG_CUDA(cudaMemcpyAsync(e->pos_of_p.p, e->pos_of.p, e->cl.slots * 4, cudaMemcpyDeviceToDevice, s));
  KTG_CUDA(cudaMemsetAsync(e->dead.p, 0, e->cl.slots, s));
  KTG_CUDA(cudaMemsetAsync(e->rdirty.p, 0, nb, s));
  KTG_CUDA(cudaMemsetAsync(e->sdirty.p, 0, nb, s));
  unsigned long long cap = 0;
  KTG_CUDA(cudaMemcpyAsync(&cap, e->d_workL, 8, cudaMemcpyDeviceToHost, s));
  KTG_CUDA(cudaStreamSynchronize(s));
  // the exact worst case (every edge's pieces at pristine degrees) can be
  // tens of GB on dense graphs; cap the queue at one piece per edge -- a
  // round whose removals could need more recomputes instead (k_decide)
  cap = std::min<unsigned long long>(cap, std::max<unsigned long long>(1ull << 20, m));
  e->rq_cap = cap;
  KTG_TRY(e->rq.ensure(cap));
  k_set_rqcap<<<1, 1, 0, s>>>(e->d_st, cap);
  KTG_CUDA(cudaGetLastError());
  e->sym_ready = true;
  e->pristine = true;
  return build_a22(e);
}


// Uploads (host or device source) into the caller layout; builds the working
// layout unless the label order is requested. Buffers are reused when the
// new graph fits (the host-buffer entry points keep one cached engine per
// thread, so repeated calls allocate nothing and reuse the fixpoint graph).
ktg_status engine_load(ktg_engine* e, const uint32_t* row_ptr, uint32_t n, const uint32_t* col, uint64_t slots,
                       cudaMemcpyKind kind, bool keep_pristine, bool allow_reorient) {
  if (n == 0) return fail(KTG_ERR_INVALID_INPUT, "csr has no vertices");
  if (slots > 0xFFFFFFFFull) return fail(KTG_ERR_INVALID_INPUT, "slot count exceeds 32-bit offsets");
  if (slots < n) return fail(KTG_ERR_INVALID_INPUT, "row_ptr end does not match slot count");
  Layout& C = e->cl;
  C.ready = false;
  e->wl.ready = false;
  // a peer group survives a reload only if the peers' tables still describe
  // this engine's buffers (same allocations, same slot count, lists large
  // enough) -- every rank reloading the same graph, as a multi-GPU e2e does
  const bool had_group = e->group;
  const uint32_t g_rank = e->rank_id, g_world = e->world;
  const void* g_bufs[3] = {e->act().S0.p, e->act().S1.p, (void*)e->act().slots};
  if (had_group) {
    e->group = false;
    e->world = 1;
    e->rank_id = 0;
  }
  if (row_ptr || col) e->has_orig_ids = false;
  C.n = n;
  C.slots = slots;
  C.has_payload = false;
  e->reoriented = allow_reorient && !flag(e, KTG_FLAG_LABEL_ORDER) && e->opt.observer == nullptr;
  e->caller_stale = false;
  KTG_TRY(C.row_ptr.ensure((size_t)n + 2));
  KTG_TRY(C.col.ensure(slots + 4));
  PhaseTimer mark(e->stream);
  mark("start");
  if (row_ptr) KTG_CUDA(cudaMemcpyAsync(C.row_ptr.p, row_ptr, ((size_t)n + 2) * 4, kind, e->stream));
  if (col) KTG_CUDA(cudaMemcpyAsync(C.col.p, col, slots * 4, kind, e->stream));
  mark("upload");
  KTG_TRY(prepare_layout(e, C, keep_pristine || e->reoriented));
  mark("caller layout");
  if (e->reoriented) {
    // carried-support runs need the symmetric rows (col marks use the top bit)
    const bool with_sym = !flag(e, KTG_FLAG_RECOMPUTE) && n <= 0x7fffffffu;
    e->sym_ready = false;
    ktg_status st = build_working(e, with_sym);
    mark("working layout (+ symmetric rows)");
    if (st == KTG_OK && with_sym) st = build_sym(e);
    mark("A22 plan");
    if (st == KTG_ERR_OOM && with_sym) {
      // the carried-support structures (symmetric rows, per-edge maps, A22
      // plan, delta queues) do not fit next to the graph: drop them and run
      // this graph the paper's way, a full support pass every round
      cudaGetLastError();
      e->release_sym();
      st = build_working(e, false);
    }
    KTG_TRY(st);
  }
  if (had_group && e->act().S0.p == g_bufs[0] && e->act().S1.p == g_bufs[1] &&
      (void*)e->act().slots == g_bufs[2] && e->xcap >= e->act().live_pristine) {
    e->group = true;
    e->world = g_world;
    e->rank_id = g_rank;
  }
  return a22_rank_split(e);  // partitioned engines: this graph's task split
}

const char* kValidateMsg[6] = {"", " owns no sentinel slot", " does not end in a zero slot",
                               " has a nonzero after a zero slot",
                               " entries are not strictly ascending above the vertex",
                               " references vertex beyond n"};

// ZTCSR1 file -> HBM (csr_cache.cpp:80-111 semantics and messages), streamed
// through two pinned staging buffers; invariants validated on the device.
ktg_status load_cache(ktg_engine* e, const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(KTG_ERR_INVALID_PARAMETER, std::string("cannot open ") + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  static const char kMagic[8] = {'Z', 'T', 'C', 'S', 'R', '1', '\0', '\0'};
  char magic[8];
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
    return fail(KTG_ERR_CORRUPT_CACHE, "bad cache magic");
  uint32_t n = 0;
  uint64_t slots = 0;
  if (std::fread(&n, 4, 1, f) != 1 || std::fread(&slots, 8, 1, f) != 1)
    return fail(KTG_ERR_CORRUPT_CACHE, "truncated cache header");
  if (n == 0 || slots < n || slots > 0xFFFFFFFFull) return fail(KTG_ERR_CORRUPT_CACHE, "implausible cache dimensions");
  Layout& C = e->cl;
  KTG_TRY(C.row_ptr.ensure((size_t)n + 2));
  KTG_TRY(C.col.ensure(slots + 4));
  constexpr size_t kStage = size_t{32} << 20;
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto release = [&]() {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventSynchronize(done[i]), cudaEventDestroy(done[i]);
      if (stage[i]) cudaFreeHost(stage[i]);
    }
  };
  ktg_status st = KTG_OK;
  for (int i = 0; i < 2 && st == KTG_OK; ++i) {
    if (cudaMallocHost(&stage[i], kStage) != cudaSuccess || cudaEventCreate(&done[i]) != cudaSuccess)
      st = fail(KTG_ERR_OOM, "pinned staging allocation failed");
  }
  // stream row_ptr then col_idx through the staging buffers
  struct Seg {
    char* dst;
    uint64_t bytes;
  } segs[2] = {{reinterpret_cast<char*>(C.row_ptr.p), ((uint64_t)n + 2) * 4},
               {reinterpret_cast<char*>(C.col.p), slots * 4}};
  int buf = 0;
  for (int sgi = 0; sgi < 2 && st == KTG_OK; ++sgi) {
    for (uint64_t off = 0; off < segs[sgi].bytes && st == KTG_OK;) {
      const size_t len = (size_t)std::min<uint64_t>(kStage, segs[sgi].bytes - off);
      cudaEventSynchronize(done[buf]);
      if (std::fread(stage[buf], 1, len, f) != len) {
        st = fail(KTG_ERR_CORRUPT_CACHE, "truncated cache payload");
        break;
      }
      if (cudaMemcpyAsync(segs[sgi].dst + off, stage[buf], len, cudaMemcpyHostToDevice, e->stream) != cudaSuccess ||
          cudaEventRecord(done[buf], e->stream) != cudaSuccess)
        st = fail(KTG_ERR_CUDA, "cache upload failed");
      off += len;
      buf ^= 1;
    }
  }
  if (st == KTG_OK && std::fgetc(f) != EOF) st = fail(KTG_ERR_CORRUPT_CACHE, "trailing bytes after cache payload");
  release();
  if (st != KTG_OK) return st;
  uint32_t head[2] = {0, 0}, last = 0;
  KTG_CUDA(cudaMemcpy(head, C.row_ptr.p, 8, cudaMemcpyDeviceToHost));
  KTG_CUDA(cudaMemcpy(&last, C.row_ptr.p + n + 1, 4, cudaMemcpyDeviceToHost));
  if (last != slots) return fail(KTG_ERR_CORRUPT_CACHE, "row_ptr end does not match slot count");
  if (head[0] != 0 || head[1] != 0)
    return fail(KTG_ERR_CORRUPT_CACHE, "cache violates csr invariants: phantom vertex 0 must own no slots");
  unsigned long long* d_first = nullptr;
  KTG_CUDA(cudaMalloc(&d_first, 8));
  unsigned long long first = ~0ull;
  cudaMemcpy(d_first, &first, 8, cudaMemcpyHostToDevice);
  k_validate_rows<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(C.row_ptr.p, C.col.p, n, slots, d_first);
  cudaError_t ve = cudaGetLastError();
  if (ve == cudaSuccess) ve = cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, e->stream);
  if (ve == cudaSuccess) ve = cudaStreamSynchronize(e->stream);
  cudaFree(d_first);
  if (ve != cudaSuccess) return fail(KTG_ERR_CUDA, std::string("cache validation: ") + cudaGetErrorString(ve));
  if (first != ~0ull)
    return fail(KTG_ERR_CORRUPT_CACHE, "cache violates csr invariants: row " + std::to_string(first >> 3) +
                                           kValidateMsg[first & 7]);
  return engine_load(e, nullptr, n, nullptr, slots, cudaMemcpyDeviceToDevice, true, true);
}

// Caller-layout support buffer holding the current result.
uint32_t* caller_S(ktg_engine* e) {
  if (e->reoriented) return e->cl.S0.p;
  return e->h_st->parity ? e->cl.S1.p : e->cl.S0.p;
}

// Rebuilds the caller layout from the working layout's live set (enqueued,
// no host sync): zero, scatter (pristine column, support) by caller slot, then
// stable per-row compaction over each row's pristine extent.
ktg_status publish(ktg_engine* e) {
  if (!e->reoriented || !e->caller_stale) return KTG_OK;
  Layout& C = e->cl;
  const cudaStream_t s = e->stream;
  if (e->sym_ready && e->inc_active) {
    // every caller slot knows its fate (dead flag) and its working slot:
    // one stable compaction pass from the pristine rows
    Graph g = e->graph_of(C);
    k_clear_heavy<<<1, 1, 0, s>>>(e->d_st);
    k_publish_inc<0><<<e->prune_grid, kPruneThreads, 0, s>>>(g, C.col_p.p, C.deg_p.p, e->dead.p, e->pos_of.p,
                                                            e->wl.S0.p);
    k_publish_inc<1><<<e->heavy_grid, kSymHeavyThreads, 0, s>>>(g, C.col_p.p, C.deg_p.p, e->dead.p, e->pos_of.p,
                                                            e->wl.S0.p);
    k_clear_heavy<<<1, 1, 0, s>>>(e->d_st);
    KTG_CUDA(cudaGetLastError());
    e->caller_stale = false;
    return KTG_OK;
  }
  KTG_CUDA(cudaMemsetAsync(C.col.p, 0, C.slots * 4, s));
  KTG_CUDA(cudaMemsetAsync(C.S0.p, 0, C.slots * 4, s));
  k_scatter_live<<<e->prune_grid, kPruneThreads, 0, s>>>(e->graph_of(e->wl), C.col_p.p, C.col.p, C.S0.p, 0);
  KTG_CUDA(cudaMemcpyAsync(C.deg.p, C.deg_p.p, ((size_t)C.n + 2) * 4, cudaMemcpyDeviceToDevice, s));
  k_clear_heavy<<<1, 1, 0, s>>>(e->d_st);
  Graph g = e->graph_of(C);
  k_prune_light<1><<<e->prune_grid, kPruneThreads, 0, s>>>(g, 0);
  k_prune_heavy<1><<<e->heavy_grid, kSymHeavyThreads, 0, s>>>(g, 0);
  k_clear_heavy<<<1, 1, 0, s>>>(e->d_st);
  KTG_CUDA(cudaGetLastError());
  e->caller_stale = false;
  return KTG_OK;
}

// Support task plan of a k_support_chunked round: off-diagonal pairs, and
// with world > 1 this rank's work-balanced range of diagonal tasks (prefix
// sum of per-chunk work estimates; partitioned loops are host-driven, so the
// buffers may grow here).
ktg_status plan_tasks(ktg_engine* e, Layout& L, const Graph& g) {
  const cudaStream_t s = e->stream;
  k_plan_count<<<(L.nchunks + 255) / 256, 256, 0, s>>>(g, 0);
  k_plan_write<<<1, 1024, 0, s>>>(g);
  if (e->world > 1) {
    const size_t nq = (size_t)L.nchunks + 1;
    KTG_TRY(e->task_cost.ensure(nq));
    KTG_TRY(e->task_pre.ensure(nq));
    size_t tmp = 0;
    KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, e->task_cost.p, e->task_pre.p, (int)nq, s));
    KTG_TRY(e->cub_tmp.ensure(tmp));
    tmp = e->cub_tmp.cap;
    k_task_cost<<<(unsigned)nq, kChunk, 0, s>>>(g, e->task_cost.p);
    KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, e->task_cost.p, e->task_pre.p, (int)nq, s));
    k_rank_range<<<1, 1, 0, s>>>(g, e->task_pre.p);
  }
  KTG_CUDA(cudaGetLastError());
  return KTG_OK;
}

// Enqueue one round on the active layout:
// plan -> support -> [check16] -> [allreduce] -> prune -> control.
ktg_status enqueue_round(ktg_engine* e, bool graph_mode, cudaGraphConditionalHandle handle,
                         cudaEvent_t sup0 = nullptr, cudaEvent_t sup1 = nullptr) {
  Layout& L = e->act();
  Graph g = e->graph_of(L);
  const cudaStream_t s = e->stream;
  const int fused = graph_mode ? 1 : 0;
  const bool a22 = e->inc_active && e->a22_ready && !e->a22_off_env;
  if (!a22) {
    KTG_TRY(plan_tasks(e, L, g));
  }
  if (sup0) KTG_CUDA(cudaEventRecord(sup0, s));
  if (a22) {
    A22 a{e->a22_pe.p, e->a22_pin.p, e->a22_pin_end.p, e->a22_off.p, e->a22_jfirst.p, e->a22_tasks.p, e->a22_ntasks};
    k_support_a22<false><<<e->a22_grid, kSupportThreads, e->a22_smem, s>>>(g, e->sym(), a, nullptr);
  } else if (flag(e, KTG_FLAG_NAIVE_SUPPORT)) {
    k_support_naive<<<4 * e->num_sms, 256, 0, s>>>(g);
  } else {
    const bool exch = !graph_mode && e->npeer > 1 && e->peer_cb;
    // fused path: every rank's previous prune (which zeroes this round's
    // buffer) must be done before any rank adds into it
    if (exch && e->peer_cb(0, nullptr, L.slots, e->peer_span, nullptr, s, e->peer_user) != 0)
      return fail(KTG_ERR_CUDA, "peer exchange callback failed (round start)");
    k_support_chunked<<<e->support_grid, kSupportThreads, e->support_smem, s>>>(g);
  }
  if (sup1) KTG_CUDA(cudaEventRecord(sup1, s));
  const bool grp = e->group && e->world > 1;
  if (grp) {
    // device-side all-reduce of the partial supports over peer memory: carried
    // runs after full passes only, recompute runs every round
    const XGroup x = e->xgroup();
    if (e->inc_active) {
      k_xbar<0><<<1, 32, 0, s>>>(e->d_st, x, 1);
      k_xreduce<<<4 * e->num_sms, 256, 0, s>>>(g, x, 1);
      k_xbar<0><<<1, 32, 0, s>>>(e->d_st, x, 0);
    } else {
      k_xbar<2><<<1, 32, 0, s>>>(e->d_st, x, 1);
      k_xreduce<<<4 * e->num_sms, 256, 0, s>>>(g, x, 0);
      k_xbar<2><<<1, 32, 0, s>>>(e->d_st, x, 0);
    }
  }
  if (e->inc_active) {
    if (!grp && !graph_mode && e->world > 1 && e->h_st->mode == 0 && (e->nccl || e->allreduce)) {
      // multi-rank carried run: this full pass covered this rank's A22
      // tasks only; sum the partial supports, then every rank runs the same
      // deterministic mark / delta / compaction on identical data
      uint32_t* buf = e->h_st->parity ? L.S1.p : L.S0.p;
      if (e->nccl) {
        NcclApi* api = nccl_api();
        const ncclResult_t r = api->allReduce(buf, buf, L.slots, ncclUint32, ncclSum, e->nccl, e->stream);
        if (r != ncclSuccess) return fail(KTG_ERR_CUDA, std::string("ncclAllReduce: ") + api->errorString(r));
      } else if (e->allreduce(buf, L.slots, e->stream, e->allreduce_user) != 0) {
        return fail(KTG_ERR_CUDA, "allreduce callback failed");
      }
    }
    // mark -> [carry: delta] -> compact rows (col, ids, carried S) -> compact
    // symmetric rows -> control (next round's mode, while condition)
    const Sym y = e->sym();
    k_mark<<<e->prune_grid, kPruneThreads, 0, s>>>(g, y);
    k_mark_frontier<<<e->prune_grid, kPruneThreads, 0, s>>>(g, y);
    k_decide<<<1, 1, 0, s>>>(e->d_st, grp ? reinterpret_cast<XArea*>(e->xarea.p) : nullptr, e->xcap);
    k_queues<<<4 * e->num_sms, 256, 0, s>>>(g, y);
    k_delta<<<e->prune_grid, kPruneThreads, 0, s>>>(g, y);
    k_delta_big<<<e->prune_grid, kPruneThreads, 0, s>>>(g, y);
    if (grp) {  // every rank's listed decrements reach every rank
      const XGroup x = e->xgroup();
      k_xbar<1><<<1, 32, 0, s>>>(e->d_st, x, 0);
      k_xapply<<<e->prune_grid, kPruneThreads, 0, s>>>(g, y, x);
    }
    k_inc_rows<0><<<e->prune_grid, kPruneThreads, 0, s>>>(g, y);
    k_inc_rows<1><<<e->heavy_grid, kSymHeavyThreads, 0, s>>>(g, y);
    k_inc_sym<0><<<e->prune_grid, kPruneThreads, 0, s>>>(g, y);
    k_inc_sym<1><<<e->heavy_grid, kSymHeavyThreads, 0, s>>>(g, y);
    k_inc_zero<<<4 * e->num_sms, 256, 0, s>>>(g);
    k_control_inc<<<1, 1, 0, s>>>(e->d_st, e->d_hist, handle, graph_mode ? 1 : 0);
    KTG_CUDA(cudaGetLastError());
    return KTG_OK;
  }
  if (e->opt.width_bits == 16) k_check16<<<4 * e->num_sms, 256, 0, s>>>(g);
  KTG_CUDA(cudaGetLastError());
  if (grp) {
    // exchanged above
  } else if (!graph_mode && e->npeer > 1 && e->peer_cb) {
    // fused path: the support kernel already sent every increment to its
    // owner; the callback waits for all ranks, all-gathers the owned spans
    // and sums the round's triangle count
    uint32_t* buf = e->h_st->parity ? L.S1.p : L.S0.p;
    if (e->peer_cb(1, buf, L.slots, e->peer_span, &e->d_st->triangles, s, e->peer_user) != 0)
      return fail(KTG_ERR_CUDA, "peer exchange callback failed (all-gather)");
  } else if (!graph_mode && (e->nccl || (e->world > 1 && e->allreduce))) {
    // partial supports of this rank's task share -> full supports everywhere
    uint32_t* buf = e->h_st->parity ? L.S1.p : L.S0.p;
    if (e->nccl) {
      NcclApi* api = nccl_api();
      ncclResult_t r = api->allReduce(buf, buf, L.slots, ncclUint32, ncclSum, e->nccl, e->stream);
      if (r == ncclSuccess)
        r = api->allReduce(&e->d_st->triangles, &e->d_st->triangles, 1, ncclUint64, ncclSum, e->nccl, e->stream);
      if (r != ncclSuccess) return fail(KTG_ERR_CUDA, std::string("ncclAllReduce: ") + api->errorString(r));
    } else if (e->allreduce(buf, L.slots, e->stream, e->allreduce_user) != 0) {
      return fail(KTG_ERR_CUDA, "allreduce callback failed");
    }
  }
  k_prune_light<0><<<e->prune_grid, kPruneThreads, 0, s>>>(g, fused);
  k_prune_heavy<0><<<e->heavy_grid, kSymHeavyThreads, 0, s>>>(g, fused);
  k_control<<<1, 1, 0, s>>>(e->d_st, e->d_hist, handle, graph_mode ? 1 : 0);
  KTG_CUDA(cudaGetLastError());
  return KTG_OK;
}

ktg_status build_graph(ktg_engine* e) {
  Layout& L = e->act();
  const void* key[4] = {L.col.p, L.id.p, L.S0.p, L.pairs.p};
  const uint64_t key2[4] = {L.slots, L.n,
                            (uint64_t)(flag(e, KTG_FLAG_NAIVE_SUPPORT) ? 1 : 0) | ((uint64_t)e->group << 1) |
                                ((uint64_t)e->world << 8) | ((uint64_t)e->rank_id << 32),
                            (uint64_t)e->opt.width_bits | ((uint64_t)e->reoriented << 8) |
                                ((uint64_t)e->scan_ratio << 16) | ((uint64_t)e->inc_active << 48)};
  if (e->exec && std::equal(key, key + 4, e->exec_key) && std::equal(key2, key2 + 4, e->exec_key2))
    return KTG_OK;
  if (e->exec) cudaGraphExecDestroy(e->exec);
  e->exec = nullptr;
  cudaGraph_t graph;
  KTG_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle handle;
  KTG_CUDA(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
  alignas(cudaGraphNodeParams) unsigned char cp_buf[sizeof(cudaGraphNodeParams)];
  std::memset(cp_buf, 0, sizeof(cp_buf));
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_buf);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  KTG_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  KTG_CUDA(cudaStreamBeginCaptureToGraph(e->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const ktg_status st = enqueue_round(e, true, handle);
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(e->stream, &captured);
  if (st != KTG_OK) {
    cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess) {
    cudaGraphDestroy(graph);
    return fail(KTG_ERR_CUDA, std::string("capture of the round body failed: ") + cudaGetErrorString(ce));
  }
  const cudaError_t ie = cudaGraphInstantiate(&e->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return fail(KTG_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
  std::copy(key, key + 4, e->exec_key);
  std::copy(key2, key2 + 4, e->exec_key2);
  return KTG_OK;
}

// Prepares the device state for a fixpoint at k. parity < 0 switches to the
// other support buffer on the device (it is all zero whenever the previous
// run converged, see k_prune_light), parity >= 0 selects it explicitly.
// Incremental rounds (supports carried across rounds when cheaper) run on the
// working layout of a single-rank engine with 32-bit widths and no observer;
// KTG_FLAG_RECOMPUTE keeps the paper's full pass every round.
bool inc_eligible(const ktg_engine* e) {
  return e->reoriented && e->sym_ready && !flag(e, KTG_FLAG_RECOMPUTE) && !flag(e, KTG_FLAG_NAIVE_SUPPORT) &&
         e->opt.width_bits == 32 && e->opt.observer == nullptr && e->npeer <= 1 &&
         (e->world == 1 || e->nccl != nullptr || e->allreduce != nullptr || e->group);
}

ktg_status begin_run(ktg_engine* e, uint32_t k, int parity) {
  e->inc_active = inc_eligible(e);
  if (e->inc_active) {
    // one support buffer; round 0 is a full pass into a zeroed S0
    KTG_CUDA(cudaMemsetAsync(e->wl.S0.p, 0, e->wl.slots * 4, e->stream));
    parity = 0;
  }
  k_begin<<<1, 1, 0, e->stream>>>(e->d_st, k >= 2 ? k - 2 : 0, e->opt.width_bits == 16 ? 1 : 0, parity,
                                  e->inc_active ? 1u : 0u, e->delta_ratio,
                                  e->delta_ratio0);
  if (e->inc_active && e->pristine) {
    if (!flag(e, KTG_FLAG_NO_DEGREE_BOUND))
      k_heavy_rank<<<1, 1, 0, e->stream>>>(e->d_st, e->sym_deg_p.p, e->wl.n);
    else
      k_set_pristine<<<1, 1, 0, e->stream>>>(e->d_st);
  }
  e->pristine = false;
  KTG_CUDA(cudaGetLastError());
  return KTG_OK;
}

ktg_status collect_work(ktg_engine* e, ktg_round_work* w) {
  Layout& L = e->act();
  Graph g = e->graph_of(L);
  KTG_TRY(e->din.ensure((size_t)L.n + 2));
  KTG_CUDA(cudaMemsetAsync(e->din.p, 0, ((size_t)L.n + 2) * 4, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_workL, 0, 16, e->stream));
  k_work_din<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(g, e->din.p);
  k_work_L<<<4 * e->num_sms, 256, 0, e->stream>>>(g, e->din.p, e->d_workL);
  KTG_CUDA(cudaGetLastError());
  unsigned long long L2[2] = {0, 0}, live = 0;
  KTG_CUDA(cudaMemcpyAsync(L2, e->d_workL, 16, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaMemcpyAsync(&live, &e->d_st->live, 8, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  w->L = L2[0];
  w->L_tail = L2[1];
  w->live_edges = live;
  return KTG_OK;
}

// After a carried run: T of the converged graph from its supports.
ktg_status inc_finish(ktg_engine* e) {
  if (!e->inc_active) return KTG_OK;
  k_inc_triangles<<<4 * e->num_sms, 256, 0, e->stream>>>(e->graph_of(e->wl));
  k_inc_triangles_done<<<1, 1, 0, e->stream>>>(e->d_st);
  KTG_CUDA(cudaGetLastError());
  return KTG_OK;
}

// The fixpoint on the active layout. Expects begin_run() already enqueued.
// Publishes the caller layout afterwards (enqueued).
ktg_status run_loop(ktg_engine* e, bool want_sync) {
  Layout& L = e->act();
  const bool timing = flag(e, KTG_FLAG_TIME_SUPPORT);
  const bool recording = timing || flag(e, KTG_FLAG_COLLECT_WORK);
  const bool host_loop =
      flag(e, KTG_FLAG_HOST_LOOP) || e->opt.observer || (e->world > 1 && !e->group) || e->nccl || recording;
  e->work.clear();
  e->caller_stale = true;
  e->ran = true;  // ev0 / ev1 bracket a run from here on
  KTG_CUDA(cudaEventRecord(e->ev0, e->stream));
  if (!host_loop) {
    KTG_TRY(build_graph(e));
    KTG_CUDA(cudaGraphLaunch(e->exec, e->stream));
    KTG_TRY(inc_finish(e));
    KTG_TRY(publish(e));
    KTG_CUDA(cudaEventRecord(e->ev1, e->stream));
    if (!want_sync) return KTG_OK;
    return read_state(e);
  }
  std::vector<uint32_t> h_col, h_S;
  if (e->opt.observer) {
    h_col.resize(L.slots);
    h_S.resize(L.slots);
  }
  KTG_TRY(read_state(e));  // parity of round 0
  for (uint32_t round = 0;; ++round) {
    // Host loop keeps S semantics of the reference: the round's buffer is
    // zeroed up front (reset_supports), prune leaves S untouched.
    uint32_t* Sc = e->h_st->parity ? L.S1.p : L.S0.p;
    if (!e->inc_active) KTG_CUDA(cudaMemsetAsync(Sc, 0, L.slots * 4, e->stream));
    ktg_round_work w{};
    w.full_pass = e->h_st->mode == 0 ? 1u : 0u;  // state read after the previous round
    if (flag(e, KTG_FLAG_COLLECT_WORK)) KTG_TRY(collect_work(e, &w));
    KTG_TRY(enqueue_round(e, false, 0, timing ? e->evs0 : nullptr, timing ? e->evs1 : nullptr));
    KTG_TRY(read_state(e));
    unsigned long long removed = 0;
    if (round < (uint32_t)kHistCap) KTG_CUDA(cudaMemcpy(&removed, e->d_hist + round, 8, cudaMemcpyDeviceToHost));
    if (recording) {
      w.triangles = e->h_st->last_triangles;
      w.removed = removed;
      w.delta_cost = e->h_st->last_dcost;
      w.keep_cost = e->h_st->last_kcost;
      w.delta_pieces = e->h_st->last_nrq;
      w.carried = e->h_st->last_carry;
      if (timing) {
        float ms = 0;
        KTG_CUDA(cudaEventElapsedTime(&ms, e->evs0, e->evs1));
        w.support_ms = ms;
      }
      e->work.push_back(w);
    }
    if (e->opt.observer) {  // label layout only (see engine_load)
      const uint32_t par = removed != 0 && e->h_st->error == 0 ? (e->h_st->parity ^ 1u) : e->h_st->parity;
      KTG_CUDA(cudaMemcpy(h_col.data(), L.col.p, L.slots * 4, cudaMemcpyDeviceToHost));
      KTG_CUDA(cudaMemcpy(h_S.data(), par ? L.S1.p : L.S0.p, L.slots * 4, cudaMemcpyDeviceToHost));
      e->opt.observer(h_col.data(), h_S.data(), L.slots, removed, e->opt.observer_user);
    }
    if (removed == 0 || e->h_st->error) break;
  }
  KTG_TRY(inc_finish(e));
  KTG_TRY(publish(e));
  KTG_CUDA(cudaEventRecord(e->ev1, e->stream));
  return read_state(e);
}

ktg_status overflow_error(ktg_engine* e) {
  if (e->h_st->error == kErrGroupTimeout)
    return fail(KTG_ERR_CUDA, "peer group barrier timed out (a rank stopped joining the fixpoint)");
  const unsigned long long key = e->h_st->overflow_slot;
  const uint64_t slot = key >> 32;
  const uint32_t cnt = (uint32_t)(key & 0xffffffffull);
  g_err_slot = slot;
  return fail(KTG_ERR_SUPPORT_OVERFLOW,
              "16-bit support overflow at slot " + std::to_string(slot) + " (count " + std::to_string(cnt) + ")");
}

ktg_status finish_info(ktg_engine* e) {
  float ms = 0;
  if (e->ran && cudaEventElapsedTime(&ms, e->ev0, e->ev1) != cudaSuccess) {
    cudaGetLastError();
    ms = 0;
  }
  e->info.iterations = e->h_st->iter;
  e->info.live_edges = e->h_st->live;
  e->info.triangles = e->h_st->last_triangles;
  e->info.device_ms = ms;
  e->info.carried = (e->reoriented && e->sym_ready && !flag(e, KTG_FLAG_RECOMPUTE)) ? 1u : 0u;
  if (e->h_st->error) return overflow_error(e);
  return KTG_OK;
}

ktg_status copy_hist(ktg_engine* e, uint64_t* hist, uint32_t cap, uint32_t* iterations) {
  const uint32_t it = e->h_st->iter;
  if (iterations) *iterations = it;
  const uint32_t m = std::min<uint32_t>(std::min<uint32_t>(it, cap), (uint32_t)kHistCap);
  if (hist && m) KTG_CUDA(cudaMemcpy(hist, e->d_hist, (size_t)m * 8, cudaMemcpyDeviceToHost));
  return KTG_OK;
}

// One support pass on the active layout into its (parity) buffer, no reset.
// add_to_caller: scatter-add the working supports into the caller's S0
// (ktg_compute_supports accumulates like the reference).
ktg_status support_pass(ktg_engine* e, int parity, uint64_t* triangles, bool max_support, bool add_to_caller) {
  Layout& L = e->act();
  // A standalone pass (compute_supports, the kmax_search bound) is never
  // partitioned: every rank of a partitioned engine computes all tasks, so
  // T, max S and S are whole-graph values on every rank without an exchange.
  struct Solo {
    ktg_engine* e;
    uint32_t rank, world, npeer;
    ~Solo() { e->rank_id = rank, e->world = world, e->npeer = npeer; }
  } solo{e, e->rank_id, e->world, e->npeer};
  e->rank_id = 0, e->world = 1, e->npeer = 0;  // (graph_of: no group area at world 1)
  Graph g = e->graph_of(L);
  e->inc_active = false;
  k_begin<<<1, 1, 0, e->stream>>>(e->d_st, 0, e->opt.width_bits == 16 ? 1 : 0, parity, 0u, e->delta_ratio, e->delta_ratio0);
  KTG_TRY(plan_tasks(e, L, g));
  if (flag(e, KTG_FLAG_NAIVE_SUPPORT))
    k_support_naive<<<4 * e->num_sms, 256, 0, e->stream>>>(g);
  else
    k_support_chunked<<<e->support_grid, kSupportThreads, e->support_smem, e->stream>>>(g);
  if (e->opt.width_bits == 16) k_check16<<<4 * e->num_sms, 256, 0, e->stream>>>(g);
  if (max_support) k_max_support<<<4 * e->num_sms, 256, 0, e->stream>>>(g);
  KTG_CUDA(cudaGetLastError());
  if (e->reoriented) {
    if (add_to_caller) {
      k_scatter_live<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(g, nullptr, nullptr, e->cl.S0.p, 1);
      KTG_CUDA(cudaGetLastError());
    } else {
      e->caller_stale = true;
    }
  }
  KTG_TRY(read_state(e));
  if (triangles) *triangles = e->h_st->triangles;
  e->info.max_support = e->h_st->max_support;
  if (e->h_st->error) return overflow_error(e);
  return KTG_OK;
}

ktg_status extract(ktg_engine* e, uint32_t* u, uint32_t* v, uint32_t* s, uint64_t cap, uint64_t* num) {
  PhaseTimer mark(e->stream);
  mark("start");
  KTG_TRY(publish(e));
  mark("extract: publish");
  KTG_TRY(read_state(e));
  Layout& C = e->cl;
  const uint64_t live = e->h_st->live;
  if (num) *num = live;
  if (live == 0) return KTG_OK;
  if (live > cap) return fail(KTG_ERR_INVALID_PARAMETER, "edge_cap is smaller than the survivor count");
  // row offsets = exclusive prefix of the caller live degrees (device scan)
  const size_t nb = (size_t)C.n + 2;
  KTG_TRY(e->offs.ensure(nb));
  KTG_TRY(e->ex_offs.ensure(nb));
  KTG_TRY(e->ex_out.ensure(live * 3));
  size_t tmp = 0;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, C.deg.p, e->ex_offs.p, (int)nb, e->stream));
  KTG_TRY(e->cub_tmp.ensure(tmp));
  tmp = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, tmp, C.deg.p, e->ex_offs.p, (int)nb, e->stream));
  uint32_t* out = e->ex_out.p;
  k_extract<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(e->graph_of(C), caller_S(e), e->ex_offs.p, out,
                                                           out + live, out + 2 * live);
  KTG_CUDA(cudaGetLastError());
  mark("extract: compaction");
  KTG_CUDA(cudaMemcpyAsync(u, out, live * 4, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaMemcpyAsync(v, out + live, live * 4, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaMemcpyAsync(s, out + 2 * live, live * 4, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  mark("extract: D2H");
  return KTG_OK;
}

ktg_status reset(ktg_engine* e) {
  Layout& L = e->act();
  if (!L.ready) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  if (!L.has_pristine) return fail(KTG_ERR_INVALID_PARAMETER, "engine was loaded without a pristine copy");
  const cudaStream_t s = e->stream;
  KTG_CUDA(cudaMemcpyAsync(L.col.p, L.col_p.p, L.slots * 4, cudaMemcpyDeviceToDevice, s));
  if (L.has_payload) KTG_CUDA(cudaMemcpyAsync(L.id.p, L.id_p.p, L.slots * 4, cudaMemcpyDeviceToDevice, s));
  KTG_CUDA(cudaMemcpyAsync(L.deg.p, L.deg_p.p, ((size_t)L.n + 2) * 4, cudaMemcpyDeviceToDevice, s));
  KTG_CUDA(cudaMemsetAsync(L.S0.p, 0, L.slots * 4, s));
  KTG_CUDA(cudaMemsetAsync(L.S1.p, 0, L.slots * 4, s));
  if (e->reoriented && e->sym_ready) {
    const size_t nb = (size_t)L.n + 2;
    KTG_CUDA(cudaMemcpyAsync(e->sym_nbr.p, e->sym_nbr_p.p, e->sym_entries * 4, cudaMemcpyDeviceToDevice, s));
    KTG_CUDA(cudaMemcpyAsync(e->sym_eid.p, e->sym_eid_p.p, e->sym_entries * 4, cudaMemcpyDeviceToDevice, s));
    KTG_CUDA(cudaMemcpyAsync(e->sym_deg.p, e->sym_deg_p.p, nb * 4, cudaMemcpyDeviceToDevice, s));
    KTG_CUDA(cudaMemcpyAsync(e->pos_of.p, e->pos_of_p.p, e->cl.slots * 4, cudaMemcpyDeviceToDevice, s));
    KTG_CUDA(cudaMemsetAsync(e->dead.p, 0, e->cl.slots, s));
    KTG_CUDA(cudaMemsetAsync(e->rdirty.p, 0, nb, s));
    KTG_CUDA(cudaMemsetAsync(e->sdirty.p, 0, nb, s));
  }
  k_set_live<<<1, 1, 0, s>>>(e->d_st, L.live_pristine);
  KTG_CUDA(cudaGetLastError());
  if (e->reoriented) e->caller_stale = true;
  e->pristine = true;
  return KTG_OK;
}

// Engine for the host-pointer entry points: one cached engine per thread
// and device (buffers and the instantiated fixpoint graph are reused across
// calls); a caller-supplied stream gets a private engine.
struct TmpEngine {
  ktg_engine* e = nullptr;
  bool owned = false;
  ~TmpEngine() {
    if (owned) ktg_engine_destroy(e);
  }
};

// One cached engine per (thread, device) for the host-buffer entry points;
// destroyed when the thread exits (a thread pool sweeping K values keeps its
// engines warm, and no engine outlives its thread).
struct ThreadEngines {
  ktg_engine* e[64] = {};
  ktg_engine*& operator[](int i) { return e[i]; }
  ~ThreadEngines();
};
thread_local ThreadEngines t_cached;

ktg_status tmp_engine(const ktg_options* opt, const uint32_t* row_ptr, uint32_t n, const uint32_t* col,
                      uint64_t slots, bool pristine, bool allow_reorient, TmpEngine& t) {
  ktg_options o;
  if (opt) {
    if (opt->struct_size != sizeof(ktg_options))
      return fail(KTG_ERR_INVALID_PARAMETER, "ktg_options.struct_size mismatch");
    o = *opt;
  } else {
    ktg_options_init(&o);
  }
  if (o.width_bits != 32 && o.width_bits != 16) return fail(KTG_ERR_INVALID_PARAMETER, "width_bits must be 16 or 32");
  int dev = o.device;
  if (dev < 0) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      return fail(KTG_ERR_NO_DEVICE, "no CUDA device visible (the engine has no CPU fallback)");
    }
    KTG_CUDA(cudaGetDevice(&dev));
  }
  if (o.stream == nullptr && dev >= 0 && dev < 64) {
    if (!t_cached[dev]) {
      ktg_options base = o;
      base.flags = 0;
      base.observer = nullptr;
      base.device = dev;
      KTG_TRY(ktg_engine_create(&base, &t_cached[dev]));
    }
    t.e = t_cached[dev];
    t.owned = false;
    KTG_CUDA(cudaSetDevice(dev));
    const cudaStream_t keep = t.e->stream;
    t.e->opt = o;
    t.e->opt.device = dev;
    t.e->opt.stream = nullptr;
    t.e->stream = keep;
  } else {
    KTG_TRY(ktg_engine_create(&o, &t.e));
    t.owned = true;
  }
  return engine_load(t.e, row_ptr, n, col, slots, cudaMemcpyHostToDevice, pristine, allow_reorient);
}

}  // namespace

extern "C" {

void ktg_options_init(ktg_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(ktg_options);
  o->device = -1;
  o->strategy = KTG_STRATEGY_FINE;
  o->width_bits = 32;
}

const char* ktg_last_error(void) { return g_err.c_str(); }
uint64_t ktg_last_error_slot(void) { return g_err_slot; }
const char* ktg_version(void) { return "ktg 0.2 (sm_100a)"; }
uint32_t ktg_task_chunk(void) { return (uint32_t)kChunk; }

int ktg_device_available(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int d = 0; d < count; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) return 1;
  }
  return 0;
}

ktg_status ktg_engine_create(const ktg_options* opt, ktg_engine** out) {
  ktg_engine* e = new (std::nothrow) ktg_engine;
  if (!e) return fail(KTG_ERR_OOM, "host allocation failed");
  const ktg_status st = engine_init(opt, e);
  if (st != KTG_OK) {
    ktg_engine_destroy(e);
    return st;
  }
  *out = e;
  return KTG_OK;
}

void ktg_engine_destroy(ktg_engine* e) {
  if (!e) return;
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->nccl && nccl_api()) nccl_api()->commDestroy(e->nccl);
  e->free_all();
  if (e->d_st) cudaFree(e->d_st);
  if (e->d_hist) cudaFree(e->d_hist);
  if (e->d_workL) cudaFree(e->d_workL);
  if (e->h_st) cudaFreeHost(e->h_st);
  for (cudaEvent_t ev : {e->ev0, e->ev1, e->evs0, e->evs1})
    if (ev) cudaEventDestroy(ev);
  if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

ktg_status ktg_engine_load(ktg_engine* e, const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx,
                           uint64_t slots) {
  return engine_load(e, row_ptr, n, col_idx, slots, cudaMemcpyHostToDevice, true, true);
}

ktg_status ktg_engine_load_device(ktg_engine* e, const uint32_t* d_row_ptr, uint32_t n,
                                  const uint32_t* d_col_idx, uint64_t slots) {
  return engine_load(e, d_row_ptr, n, d_col_idx, slots, cudaMemcpyDeviceToDevice, true, true);
}

ktg_status ktg_engine_load_cache(ktg_engine* e, const char* path) { return load_cache(e, path); }

ktg_status ktg_engine_build_csr(ktg_engine* e, const uint64_t* pairs, uint64_t m, int pairs_on_device) {
  if (m == 0) return fail(KTG_ERR_EMPTY_GRAPH, "no edges survive canonicalization");
  const cudaStream_t s = e->stream;
  DBuf<unsigned long long> dpairs, lab, lab2, keys2;
  auto cleanup = [&]() {
    dpairs.release();
    lab.release();
    lab2.release();
    keys2.release();
  };
  struct Guard {
    std::function<void()> f;
    ~Guard() { f(); }
  } guard{cleanup};
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(pairs);
  if (!pairs_on_device) {
    KTG_TRY(dpairs.ensure(2 * m));
    KTG_CUDA(cudaMemcpyAsync(dpairs.p, pairs, 2 * m * 8, cudaMemcpyHostToDevice, s));
    src = dpairs.p;
  }
  // 1. labels of non-loop pairs, sorted + unique
  KTG_TRY(lab.ensure(2 * m));
  KTG_TRY(lab2.ensure(2 * m));
  k_pair_labels<<<8 * e->num_sms, 256, 0, s>>>(src, m, lab.p);
  KTG_CUDA(cudaGetLastError());
  size_t t1 = 0, t2 = 0;
  KTG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, lab.p, lab2.p, (int64_t)(2 * m), 0, 64, s));
  KTG_CUDA(cub::DeviceSelect::Unique(nullptr, t2, lab2.p, lab.p, e->d_workL, (int64_t)(2 * m), s));
  KTG_TRY(e->cub_tmp.ensure(std::max(t1, t2)));
  t1 = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceRadixSort::SortKeys(e->cub_tmp.p, t1, lab.p, lab2.p, (int64_t)(2 * m), 0, 64, s));
  t2 = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceSelect::Unique(e->cub_tmp.p, t2, lab2.p, lab.p, e->d_workL, (int64_t)(2 * m), s));
  unsigned long long nl = 0, last = 0;
  KTG_CUDA(cudaMemcpyAsync(&nl, e->d_workL, 8, cudaMemcpyDeviceToHost, s));
  KTG_CUDA(cudaStreamSynchronize(s));
  if (nl) KTG_CUDA(cudaMemcpy(&last, lab.p + nl - 1, 8, cudaMemcpyDeviceToHost));
  if (nl && last == ~0ull) --nl;  // drop the self-loop sentinel
  if (nl == 0) return fail(KTG_ERR_EMPTY_GRAPH, "no edges survive canonicalization");
  if (nl > 0xFFFFFFFEull) return fail(KTG_ERR_INVALID_INPUT, "vertex count exceeds 32-bit id space");
  const uint32_t n = (uint32_t)nl;
  // 2. relabel + orient -> (u, v) keys, sorted + unique
  KTG_TRY(keys2.ensure(m));
  k_pair_keys<<<8 * e->num_sms, 256, 0, s>>>(src, m, lab.p, n, lab2.p);
  KTG_CUDA(cudaGetLastError());
  t1 = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceRadixSort::SortKeys(e->cub_tmp.p, t1, lab2.p, keys2.p, (int64_t)m, 0, 64, s));
  t2 = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceSelect::Unique(e->cub_tmp.p, t2, keys2.p, lab2.p, e->d_workL, (int64_t)m, s));
  unsigned long long me = 0;
  KTG_CUDA(cudaMemcpyAsync(&me, e->d_workL, 8, cudaMemcpyDeviceToHost, s));
  KTG_CUDA(cudaStreamSynchronize(s));
  if (me) KTG_CUDA(cudaMemcpy(&last, lab2.p + me - 1, 8, cudaMemcpyDeviceToHost));
  if (me && last == ~0ull) --me;
  if (me + n > 0xFFFFFFFFull) return fail(KTG_ERR_INVALID_INPUT, "graph exceeds 2^32-1 CSR slots");
  // 3. rows: sizes (out-degree + sentinel), exclusive scan, fill
  Layout& C = e->cl;
  const uint64_t slots = me + n;
  KTG_TRY(C.row_ptr.ensure((size_t)n + 2));
  KTG_TRY(C.col.ensure(slots + 4));
  KTG_TRY(e->cntw.ensure((size_t)n + 2));
  KTG_TRY(e->sizes.ensure((size_t)n + 2));
  KTG_CUDA(cudaMemsetAsync(e->cntw.p, 0, ((size_t)n + 2) * 4, s));
  k_key_rows<<<8 * e->num_sms, 256, 0, s>>>(lab2.p, me, e->cntw.p);
  k_row_sizes<<<4 * e->num_sms, 256, 0, s>>>(e->cntw.p, n, e->sizes.p);
  KTG_CUDA(cudaGetLastError());
  size_t t3 = 0;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, e->sizes.p, C.row_ptr.p, (int)(n + 2), s));
  KTG_TRY(e->cub_tmp.ensure(t3));
  t3 = e->cub_tmp.cap;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, t3, e->sizes.p, C.row_ptr.p, (int)(n + 2), s));
  KTG_CUDA(cudaMemsetAsync(C.col.p, 0, slots * 4, s));
  k_key_fill<<<8 * e->num_sms, 256, 0, s>>>(lab2.p, me, C.col.p);
  KTG_CUDA(cudaGetLastError());
  // original ids (labels) kept for ktg_engine_read_csr
  KTG_TRY(e->orig_ids.ensure((size_t)n + 1));
  KTG_CUDA(cudaMemsetAsync(e->orig_ids.p, 0, 8, s));
  KTG_CUDA(cudaMemcpyAsync(e->orig_ids.p + 1, lab.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
  e->has_orig_ids = true;
  return engine_load(e, nullptr, n, nullptr, slots, cudaMemcpyDeviceToDevice, true, true);
}

ktg_status ktg_engine_csr_info(ktg_engine* e, uint32_t* n, uint64_t* slots) {
  if (!e->cl.ready) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  *n = e->cl.n;
  *slots = e->cl.slots;
  return KTG_OK;
}

ktg_status ktg_engine_read_csr(ktg_engine* e, uint32_t* row_ptr, uint32_t* col_idx, uint64_t* original_ids) {
  if (!e->cl.ready) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  Layout& C = e->cl;
  const uint32_t* src = C.has_pristine ? C.col_p.p : C.col.p;  // the loaded (pristine) graph
  if (row_ptr) KTG_CUDA(cudaMemcpy(row_ptr, C.row_ptr.p, ((size_t)C.n + 2) * 4, cudaMemcpyDeviceToHost));
  if (col_idx) KTG_CUDA(cudaMemcpy(col_idx, src, C.slots * 4, cudaMemcpyDeviceToHost));
  if (original_ids) {
    if (!e->has_orig_ids) return fail(KTG_ERR_INVALID_PARAMETER, "graph was not built by ktg_engine_build_csr");
    KTG_CUDA(cudaMemcpy(original_ids, e->orig_ids.p, ((size_t)C.n + 1) * 8, cudaMemcpyDeviceToHost));
  }
  return KTG_OK;
}

ktg_status ktg_engine_reset(ktg_engine* e) { return reset(e); }

ktg_status ktg_engine_run(ktg_engine* e, uint32_t k, uint64_t* removed_hist, uint32_t hist_cap,
                          uint32_t* iterations) {
  if (!e->act().ready) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  KTG_TRY(begin_run(e, k, -1));
  const bool want = removed_hist != nullptr || iterations != nullptr;
  KTG_TRY(run_loop(e, want));
  if (!want) return KTG_OK;
  KTG_TRY(finish_info(e));
  return copy_hist(e, removed_hist, hist_cap, iterations);
}

ktg_status ktg_engine_support_pass(ktg_engine* e, uint64_t* triangles) {
  if (!e->act().ready) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  return support_pass(e, -1, triangles, true, false);
}

ktg_status ktg_engine_sync(ktg_engine* e) {
  KTG_TRY(read_state(e));
  return finish_info(e);
}

ktg_status ktg_engine_info(ktg_engine* e, ktg_run_info* info) {
  *info = e->info;
  return KTG_OK;
}

uint32_t ktg_engine_round_work(ktg_engine* e, ktg_round_work* out, uint32_t cap) {
  const uint32_t m = std::min<uint32_t>(cap, (uint32_t)e->work.size());
  for (uint32_t i = 0; i < m; ++i) out[i] = e->work[i];
  return m;
}

ktg_status ktg_engine_read(ktg_engine* e, uint32_t* col_idx, uint32_t* supports) {
  KTG_TRY(publish(e));
  KTG_TRY(read_state(e));
  Layout& C = e->cl;
  if (col_idx) KTG_CUDA(cudaMemcpy(col_idx, C.col.p, C.slots * 4, cudaMemcpyDeviceToHost));
  if (supports) KTG_CUDA(cudaMemcpy(supports, caller_S(e), C.slots * 4, cudaMemcpyDeviceToHost));
  return KTG_OK;
}

ktg_status ktg_engine_device_state(ktg_engine* e, uint32_t** d_col_idx, uint32_t** d_supports, void** stream) {
  KTG_TRY(publish(e));
  KTG_TRY(read_state(e));
  if (d_col_idx) *d_col_idx = e->cl.col.p;
  if (d_supports) *d_supports = caller_S(e);
  if (stream) *stream = e->stream;
  return KTG_OK;
}

ktg_status ktg_engine_extract(ktg_engine* e, uint32_t* out_u, uint32_t* out_v, uint32_t* out_support,
                              uint64_t edge_cap, uint64_t* num_edges) {
  return extract(e, out_u, out_v, out_support, edge_cap, num_edges);
}

// Exactly one exchange is active per engine: installing one drops the others
// (an NCCL communicator, the fused peer exchange, the allreduce callback).
static void drop_exchanges(ktg_engine* e, bool nccl, bool peers, bool cb) {
  if (nccl && e->nccl) {
    if (NcclApi* api = nccl_api()) api->commDestroy(e->nccl);
    e->nccl = nullptr;
  }
  if (peers) {
    e->npeer = 0;
    e->peer_cb = nullptr;
    e->peer_user = nullptr;
    e->group = false;
  }
  if (cb) {
    e->allreduce = nullptr;
    e->allreduce_user = nullptr;
  }
}

ktg_status ktg_engine_set_partition(ktg_engine* e, uint32_t rank, uint32_t world, ktg_allreduce_cb allreduce,
                                    void* user) {
  if (world == 0 || rank >= world) return fail(KTG_ERR_INVALID_PARAMETER, "rank must be < world");
  if (world > 1 && !allreduce) return fail(KTG_ERR_INVALID_PARAMETER, "world > 1 needs an allreduce callback");
  drop_exchanges(e, true, true, true);
  e->rank_id = rank;
  e->world = world;
  e->allreduce = allreduce;
  e->allreduce_user = user;
  KTG_TRY(a22_rank_split(e));
  if (e->exec) cudaGraphExecDestroy(e->exec);
  e->exec = nullptr;
  return KTG_OK;
}

ktg_status ktg_nccl_unique_id(uint8_t* out) {
  NcclApi* api = nccl_api();
  if (!api) return fail(KTG_ERR_CUDA, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  const ncclResult_t r = api->getUniqueId(&id);
  if (r != ncclSuccess) return fail(KTG_ERR_CUDA, std::string("ncclGetUniqueId: ") + api->errorString(r));
  std::memcpy(out, &id, sizeof(id));
  return KTG_OK;
}

ktg_status ktg_engine_support_buffers(ktg_engine* e, uint32_t** s0, uint32_t** s1, uint64_t* slots) {
  Layout& L = e->act();
  if (!L.ready) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  if (s0) *s0 = L.S0.p;
  if (s1) *s1 = L.S1.p;
  if (slots) *slots = L.slots;
  return KTG_OK;
}

ktg_status ktg_engine_set_peers(ktg_engine* e, uint32_t rank, uint32_t world, uint32_t* const* peer_s0,
                                uint32_t* const* peer_s1, ktg_peer_cb cb, void* user) {
  if (world == 0 || rank >= world) return fail(KTG_ERR_INVALID_PARAMETER, "rank must be < world");
  Layout& L = e->act();
  if (!L.ready) return fail(KTG_ERR_INVALID_PARAMETER, "load the graph before ktg_engine_set_peers");
  if (world > 1 && (!peer_s0 || !peer_s1 || !cb))
    return fail(KTG_ERR_INVALID_PARAMETER, "world > 1 needs peer buffers and an exchange callback");
  if (world > 1 && (peer_s0[rank] != L.S0.p || peer_s1[rank] != L.S1.p))
    return fail(KTG_ERR_INVALID_PARAMETER, "peer tables must hold this engine's own support buffers at its rank");
  drop_exchanges(e, true, true, false);
  e->rank_id = rank;
  e->world = world;
  e->allreduce = nullptr;
  e->npeer = world > 1 ? world : 0;
  e->peer_span = (L.slots + world - 1) / world;
  e->peer_cb = cb;
  e->peer_user = user;
  if (world > 1) {
    std::vector<uint32_t*> tab(2 * (size_t)world);
    for (uint32_t r = 0; r < world; ++r) {
      tab[r] = peer_s0[r];
      tab[world + r] = peer_s1[r];
    }
    KTG_TRY(e->peer_tab.ensure(tab.size()));
    KTG_CUDA(cudaMemcpy(e->peer_tab.p, tab.data(), tab.size() * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  }
  if (e->exec) cudaGraphExecDestroy(e->exec);
  e->exec = nullptr;
  return KTG_OK;
}

__global__ void k_set_xepoch(DevState* st, unsigned int v) { st->xepoch = v; }

ktg_status ktg_engine_group_area(ktg_engine* e, void** d_area, uint64_t* bytes) {
  Layout& L = e->act();
  if (!L.ready) return fail(KTG_ERR_INVALID_PARAMETER, "load the graph before ktg_engine_group_area");
  // one list entry per pristine live edge: a carrying round lists at most
  // 2 * delta_cost decrements and k_decide recomputes instead when that
  // could exceed it
  const uint64_t cap = std::max<uint64_t>(L.live_pristine, 1024);
  const size_t need = sizeof(XArea) + 2 * cap * sizeof(uint32_t);
  KTG_TRY(e->xarea.ensure(need));
  KTG_CUDA(cudaMemsetAsync(e->xarea.p, 0, sizeof(XArea), e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  e->xcap = cap;
  if (d_area) *d_area = e->xarea.p;
  if (bytes) *bytes = need;
  return KTG_OK;
}

ktg_status ktg_engine_set_group(ktg_engine* e, uint32_t rank, uint32_t world, void* const* areas,
                                uint32_t* const* peer_s0, uint32_t* const* peer_s1) {
  if (world == 0 || rank >= world) return fail(KTG_ERR_INVALID_PARAMETER, "rank must be < world");
  if (world > (uint32_t)kMaxGroup) return fail(KTG_ERR_INVALID_PARAMETER, "peer group larger than 64 ranks");
  Layout& L = e->act();
  if (!L.ready) return fail(KTG_ERR_INVALID_PARAMETER, "load the graph before ktg_engine_set_group");
  drop_exchanges(e, true, true, true);
  e->rank_id = 0;
  e->world = 1;
  if (e->exec) cudaGraphExecDestroy(e->exec);
  e->exec = nullptr;
  if (world == 1) return KTG_OK;
  if (!areas || !peer_s0 || !peer_s1) return fail(KTG_ERR_INVALID_PARAMETER, "world > 1 needs the peer tables");
  if (!e->xarea.p || e->xcap == 0 || areas[rank] != e->xarea.p)
    return fail(KTG_ERR_INVALID_PARAMETER, "area table must hold this engine's ktg_engine_group_area at its rank");
  if (peer_s0[rank] != L.S0.p || peer_s1[rank] != L.S1.p)
    return fail(KTG_ERR_INVALID_PARAMETER, "peer tables must hold this engine's own support buffers at its rank");
  std::vector<void*> tab(3 * (size_t)world);
  for (uint32_t r = 0; r < world; ++r) {
    tab[r] = areas[r];
    tab[world + r] = peer_s0[r];
    tab[2 * (size_t)world + r] = peer_s1[r];
  }
  KTG_TRY(e->xtab.ensure(tab.size()));
  KTG_CUDA(cudaMemcpy(e->xtab.p, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice));
  KTG_CUDA(cudaMemsetAsync(e->xarea.p, 0, sizeof(XArea), e->stream));
  k_set_xepoch<<<1, 1, 0, e->stream>>>(e->d_st, 0u);
  KTG_CUDA(cudaGetLastError());
  e->xspan = ((L.slots + world - 1) / world + 3) / 4 * 4;
  e->rank_id = rank;
  e->world = world;
  e->group = true;
  KTG_TRY(a22_rank_split(e));
  // recompute runs plan a work-balanced chunk split every round inside the
  // captured graph: size its buffers now
  const size_t nq = (size_t)L.nchunks + 1;
  KTG_TRY(e->task_cost.ensure(nq));
  KTG_TRY(e->task_pre.ensure(nq));
  size_t tmp = 0;
  KTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, e->task_cost.p, e->task_pre.p, (int)nq, e->stream));
  KTG_TRY(e->cub_tmp.ensure(tmp));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  return KTG_OK;
}

ktg_status ktg_ipc_handle(const void* d_ptr, uint8_t* out_64_bytes) {
  cudaIpcMemHandle_t h;
  KTG_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(out_64_bytes, &h, sizeof(h));
  return KTG_OK;
}

ktg_status ktg_ipc_open(const uint8_t* handle_64_bytes, void** d_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle_64_bytes, sizeof(h));
  KTG_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return KTG_OK;
}

ktg_status ktg_ipc_close(void* d_ptr) {
  KTG_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return KTG_OK;
}

ktg_status ktg_device_copy(void* dst, const void* src, uint64_t bytes, void* stream) {
  KTG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  KTG_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return KTG_OK;
}

ktg_status ktg_engine_set_nccl(ktg_engine* e, uint32_t rank, uint32_t world, const uint8_t* unique_id) {
  if (world == 0 || rank >= world) return fail(KTG_ERR_INVALID_PARAMETER, "rank must be < world");
  NcclApi* api = nccl_api();
  if (!api) return fail(KTG_ERR_CUDA, "libnccl.so.2 not loadable");
  drop_exchanges(e, true, true, true);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  KTG_CUDA(cudaSetDevice(e->device));
  const ncclResult_t r = api->commInitRank(&e->nccl, (int)world, id, (int)rank);
  if (r != ncclSuccess) {
    e->nccl = nullptr;
    return fail(KTG_ERR_CUDA, std::string("ncclCommInitRank: ") + api->errorString(r));
  }
  e->rank_id = rank;
  e->world = world;
  e->allreduce = nullptr;
  if (e->exec) cudaGraphExecDestroy(e->exec);
  e->exec = nullptr;
  return a22_rank_split(e);
}

// ---------------------------------------------------------------------------
// Reference-shaped entry points (host buffers)
// ---------------------------------------------------------------------------

void ktg_reset_supports(uint32_t* supports, uint64_t s_len) {
  if (supports && s_len) std::memset(supports, 0, s_len * 4);
}

ktg_status ktg_compute_supports(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots,
                                uint32_t* supports, uint64_t s_len, const ktg_options* opt,
                                uint64_t* triangles) {
  if (s_len != slots) return fail(KTG_ERR_INVALID_PARAMETER, "support array does not match slot count");
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, true, t));
  ktg_engine* e = t.e;
  // accumulate onto the caller's counts, like the reference (which requires
  // them zero but adds into whatever is there)
  KTG_CUDA(cudaMemcpyAsync(e->cl.S0.p, supports, slots * 4, cudaMemcpyHostToDevice, e->stream));
  uint64_t tri = 0;
  const ktg_status st = support_pass(e, 0, &tri, false, true);
  if (st != KTG_OK && st != KTG_ERR_SUPPORT_OVERFLOW) return st;
  // (label layout: the pass accumulated into cl.S0 directly)
  KTG_CUDA(cudaMemcpy(supports, e->cl.S0.p, slots * 4, cudaMemcpyDeviceToHost));
  if (st != KTG_OK) return st;
  if (triangles) *triangles = tri;
  return KTG_OK;
}

ktg_status ktg_intersect_tails(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots,
                               uint32_t pivot_slot, uint32_t predecessor, uint32_t* supports, uint32_t* found) {
  if (pivot_slot >= slots || predecessor == 0 || predecessor > n)
    return fail(KTG_ERR_INVALID_PARAMETER, "pivot slot / predecessor out of range");
  TmpEngine t;
  KTG_TRY(tmp_engine(nullptr, row_ptr, n, col_idx, slots, false, false, t));
  ktg_engine* e = t.e;
  Layout& C = e->cl;
  KTG_CUDA(cudaMemcpyAsync(C.S0.p, supports, slots * 4, cudaMemcpyHostToDevice, e->stream));
  uint32_t* d_found = C.heavy.p;  // scratch
  k_intersect_one<<<1, 1, 0, e->stream>>>(C.row_ptr.p, C.col.p, C.S0.p, pivot_slot, predecessor, d_found);
  KTG_CUDA(cudaGetLastError());
  KTG_CUDA(cudaMemcpyAsync(supports, C.S0.p, slots * 4, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaMemcpyAsync(found, d_found, 4, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  return KTG_OK;
}

ktg_status ktg_prune_edges(const uint32_t* row_ptr, uint32_t n, uint32_t* col_idx, uint64_t slots,
                           const uint32_t* supports, uint64_t s_len, uint32_t k, const ktg_options* opt,
                           uint64_t* removed) {
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  if (s_len != slots) return fail(KTG_ERR_INVALID_PARAMETER, "support array does not match slot count");
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, false, t));
  ktg_engine* e = t.e;
  Layout& C = e->cl;
  KTG_CUDA(cudaMemcpyAsync(C.S0.p, supports, slots * 4, cudaMemcpyHostToDevice, e->stream));
  KTG_TRY(begin_run(e, k, 0));
  Graph g = e->graph_of(C);
  k_prune_light<0><<<e->prune_grid, kPruneThreads, 0, e->stream>>>(g, 0);
  k_prune_heavy<0><<<e->heavy_grid, kSymHeavyThreads, 0, e->stream>>>(g, 0);
  KTG_CUDA(cudaGetLastError());
  KTG_TRY(read_state(e));
  KTG_CUDA(cudaMemcpy(col_idx, C.col.p, slots * 4, cudaMemcpyDeviceToHost));
  if (removed) *removed = e->h_st->removed;
  return KTG_OK;
}

ktg_status ktg_run_fixpoint(const uint32_t* row_ptr, uint32_t n, uint32_t* col_idx, uint64_t slots,
                            uint32_t* supports, uint64_t s_len, uint32_t k, const ktg_options* opt,
                            uint64_t* removed_hist, uint32_t hist_cap, uint32_t* iterations) {
  if (s_len != slots) return fail(KTG_ERR_INVALID_PARAMETER, "support array does not match slot count");
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, true, t));
  ktg_engine* e = t.e;
  KTG_TRY(begin_run(e, k, 0));
  KTG_TRY(run_loop(e, true));
  const ktg_status st = finish_info(e);
  // write back the (possibly partially pruned) state even on overflow
  KTG_CUDA(cudaMemcpy(col_idx, e->cl.col.p, slots * 4, cudaMemcpyDeviceToHost));
  KTG_CUDA(cudaMemcpy(supports, caller_S(e), slots * 4, cudaMemcpyDeviceToHost));
  if (st != KTG_OK) return st;
  return copy_hist(e, removed_hist, hist_cap, iterations);
}

ktg_status ktg_ktruss(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots, uint32_t k,
                      const ktg_options* opt, uint32_t* out_u, uint32_t* out_v, uint32_t* out_support,
                      uint64_t edge_cap, uint64_t* num_edges, uint64_t* removed_hist, uint32_t hist_cap,
                      uint32_t* iterations) {
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, true, t));
  ktg_engine* e = t.e;
  PhaseTimer mark(e->stream);
  mark("start");
  KTG_TRY(begin_run(e, k, 0));
  KTG_TRY(run_loop(e, true));
  KTG_TRY(finish_info(e));
  KTG_TRY(copy_hist(e, removed_hist, hist_cap, iterations));
  mark("ktruss: fixpoint");
  const ktg_status st = extract(e, out_u, out_v, out_support, edge_cap, num_edges);
  mark("ktruss: publish + extract");
  return st;
}

ktg_status ktg_kmax_search(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots,
                           const ktg_options* opt, uint32_t* k_max, uint32_t* out_u, uint32_t* out_v,
                           uint32_t* out_support, uint64_t edge_cap, uint64_t* num_edges,
                           uint64_t* removed_hist, uint32_t hist_cap, uint32_t* iterations) {
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, true, true, t));
  ktg_engine* e = t.e;
  if (e->cl.live_pristine == 0) return fail(KTG_ERR_INVALID_PARAMETER, "kmax_search needs a non-empty graph");
  // Bound pass (truss.cpp:77-80): one support pass on the pristine graph.
  KTG_TRY(reset(e));
  KTG_TRY(support_pass(e, 0, nullptr, true, false));
  const uint32_t max_support = e->info.max_support;
  auto probe = [&](uint32_t k, uint64_t* live) -> ktg_status {
    KTG_TRY(reset(e));
    KTG_TRY(begin_run(e, k, 0));
    KTG_TRY(run_loop(e, true));
    KTG_TRY(finish_info(e));
    *live = e->h_st->live;
    return KTG_OK;
  };
  uint32_t lo = 2;
  if (max_support > 0) {
    // binary search over [3, max+2], every probe from pristine (truss.cpp:87-101)
    lo = 3;
    uint32_t hi = max_support + 2;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo + 1) / 2;
      uint64_t live = 0;
      KTG_TRY(probe(mid, &live));
      if (live == 0) hi = mid - 1; else lo = mid;
    }
  }
  // the winning truss (deterministic, so re-running it equals keeping it)
  uint64_t live = 0;
  KTG_TRY(probe(lo, &live));
  *k_max = lo;
  KTG_TRY(copy_hist(e, removed_hist, hist_cap, iterations));
  return extract(e, out_u, out_v, out_support, edge_cap, num_edges);
}

}  // extern "C"

namespace {
ThreadEngines::~ThreadEngines() {
  for (ktg_engine*& x : e)
    if (x) {
      ktg_engine_destroy(x);
      x = nullptr;
    }
}
}  // namespace
