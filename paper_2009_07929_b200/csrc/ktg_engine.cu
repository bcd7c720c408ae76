// B200-native Eager K-truss engine: device-resident state, the fixpoint
// driver and the C ABI declared in include/ktg.h.
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

#include <algorithm>
#include <cstdio>
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

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

}  // namespace

struct ktg_engine {
  ktg_options opt{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;

  uint32_t n = 0;
  uint64_t slots = 0;
  uint32_t nchunks = 0;
  uint64_t live_pristine = 0;
  bool has_graph = false;
  bool pristine_valid = false;
  size_t cap_row_ptr = 0, cap_col = 0, cap_colp = 0, cap_S0 = 0, cap_S1 = 0, cap_deg = 0, cap_degp = 0,
         cap_chunk_row = 0, cap_pair_counts = 0, cap_heavy = 0, cap_pairs = 0;

  uint32_t* d_row_ptr = nullptr;
  uint32_t* d_col = nullptr;
  uint32_t* d_col_pristine = nullptr;
  uint32_t* d_S0 = nullptr;
  uint32_t* d_S1 = nullptr;
  uint32_t* d_deg = nullptr;
  uint32_t* d_deg_pristine = nullptr;
  uint32_t* d_chunk_row = nullptr;
  uint32_t* d_pair_counts = nullptr;
  uint32_t* d_heavy = nullptr;
  uint2* d_pairs = nullptr;
  uint32_t* d_din = nullptr;  // work statistics scratch
  unsigned long long* d_workL = nullptr;
  DevState* d_st = nullptr;
  unsigned long long* d_hist = nullptr;
  DevState* h_st = nullptr;  // pinned mirror

  int support_grid = 0;
  int prune_grid = 0;
  int heavy_grid = 0;
  size_t support_smem = 0;

  cudaGraphExec_t exec = nullptr;
  int exec_naive = -1, exec_w16 = -1;
  uint64_t exec_slots = 0;
  uint32_t exec_n = 0;
  const void* exec_col = nullptr;

  uint32_t rank = 0, world = 1;
  ktg_allreduce_cb allreduce = nullptr;
  void* allreduce_user = nullptr;

  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;
  ktg_run_info info{};
  std::vector<ktg_round_work> work;

  Graph dev_graph() const {
    Graph g;
    g.row_ptr = d_row_ptr;
    g.col = d_col;
    g.S0 = d_S0;
    g.S1 = d_S1;
    g.deg = d_deg;
    g.chunk_row = d_chunk_row;
    g.pairs = d_pairs;
    g.pair_counts = d_pair_counts;
    g.heavy_rows = d_heavy;
    g.st = d_st;
    g.hist = d_hist;
    g.n = n;
    g.nchunks = nchunks;
    g.slots = slots;
    g.rank = rank;
    g.world = world;
    return g;
  }

  void free_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    cap_row_ptr = cap_col = cap_colp = cap_S0 = cap_S1 = cap_deg = cap_degp = cap_chunk_row = 0;
    cap_pair_counts = cap_heavy = cap_pairs = 0;
    dfree(d_row_ptr);
    dfree(d_col);
    dfree(d_col_pristine);
    dfree(d_S0);
    dfree(d_S1);
    dfree(d_deg);
    dfree(d_deg_pristine);
    dfree(d_chunk_row);
    dfree(d_pair_counts);
    dfree(d_heavy);
    dfree(d_pairs);
    dfree(d_din);
    has_graph = false;
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
  if (e->opt.stream) {
    e->stream = static_cast<cudaStream_t>(e->opt.stream);
  } else {
    KTG_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    e->own_stream = true;
  }
  KTG_CUDA(cudaMalloc(&e->d_st, sizeof(DevState)));
  KTG_CUDA(cudaMemset(e->d_st, 0, sizeof(DevState)));
  KTG_CUDA(cudaMalloc(&e->d_hist, sizeof(unsigned long long) * kHistCap));
  KTG_CUDA(cudaMalloc(&e->d_workL, sizeof(unsigned long long)));
  KTG_CUDA(cudaMallocHost(&e->h_st, sizeof(DevState)));
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
  KTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_p, k_prune_light, kPruneThreads, 0));
  e->prune_grid = std::max(1, per_sm_p) * e->num_sms;
  e->heavy_grid = 2 * e->num_sms;
  return KTG_OK;
}

ktg_status read_state(ktg_engine* e) {
  KTG_CUDA(cudaMemcpyAsync(e->h_st, e->d_st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  return KTG_OK;
}

template <typename T>
ktg_status ensure(T*& p, size_t& cap, size_t bytes) {
  if (p && cap >= bytes) return KTG_OK;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  KTG_CUDA(cudaMalloc(&p, bytes));
  cap = bytes;
  return KTG_OK;
}

// Uploads (host or device source) and prepares the per-graph structures.
// Device buffers are reused when the new graph fits (the host-buffer entry
// points keep one cached engine per thread, so repeated calls do no
// allocation and reuse the instantiated CUDA graph).
ktg_status engine_load(ktg_engine* e, const uint32_t* row_ptr, uint32_t n, const uint32_t* col,
                       uint64_t slots, cudaMemcpyKind kind, bool keep_pristine) {
  if (n == 0) return fail(KTG_ERR_INVALID_INPUT, "csr has no vertices");
  if (slots > 0xFFFFFFFFull) return fail(KTG_ERR_INVALID_INPUT, "slot count exceeds 32-bit offsets");
  if (slots < n) return fail(KTG_ERR_INVALID_INPUT, "row_ptr end does not match slot count");
  e->has_graph = false;
  e->n = n;
  e->slots = slots;
  e->nchunks = (uint32_t)((slots + kChunk - 1) / kChunk);
  const size_t nb = (size_t)(n + 2) * 4;
  const size_t sb = (size_t)slots * 4 + 16;  // +16: vector-load padding
  KTG_TRY(ensure(e->d_row_ptr, e->cap_row_ptr, nb));
  KTG_TRY(ensure(e->d_col, e->cap_col, sb));
  KTG_TRY(ensure(e->d_S0, e->cap_S0, sb));
  KTG_TRY(ensure(e->d_S1, e->cap_S1, sb));
  KTG_TRY(ensure(e->d_deg, e->cap_deg, nb));
  KTG_TRY(ensure(e->d_deg_pristine, e->cap_degp, nb));
  KTG_TRY(ensure(e->d_chunk_row, e->cap_chunk_row, (size_t)e->nchunks * 4));
  KTG_TRY(ensure(e->d_pair_counts, e->cap_pair_counts, (size_t)e->nchunks * 4));
  KTG_TRY(ensure(e->d_heavy, e->cap_heavy, nb));
  KTG_CUDA(cudaMemcpyAsync(e->d_row_ptr, row_ptr, nb, kind, e->stream));
  KTG_CUDA(cudaMemcpyAsync(e->d_col, col, (size_t)slots * 4, kind, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_col + slots, 0, 16, e->stream));
  e->pristine_valid = false;
  if (keep_pristine) {
    KTG_TRY(ensure(e->d_col_pristine, e->cap_colp, sb));
    KTG_CUDA(cudaMemcpyAsync(e->d_col_pristine, e->d_col, sb, cudaMemcpyDeviceToDevice, e->stream));
    e->pristine_valid = true;
  }
  KTG_CUDA(cudaMemsetAsync(e->d_S0, 0, sb, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_S1, 0, sb, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_deg, 0, nb, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_st, 0, sizeof(DevState), e->stream));
  k_init_deg<<<4 * e->num_sms, 256, 0, e->stream>>>(e->d_row_ptr, e->d_col, n, slots, e->d_deg, e->d_st);
  KTG_CUDA(cudaGetLastError());
  k_chunk_rows<<<(e->nchunks + 255) / 256, 256, 0, e->stream>>>(e->d_row_ptr, n, slots, e->nchunks,
                                                               e->d_chunk_row);
  KTG_CUDA(cudaGetLastError());
  KTG_CUDA(cudaMemcpyAsync(e->d_deg_pristine, e->d_deg, nb, cudaMemcpyDeviceToDevice, e->stream));
  // Off-diagonal task capacity: the pristine plan is the largest (live ends
  // only shrink as rows are pruned); k_plan_count totals it on the device.
  Graph g = e->dev_graph();
  k_plan_count<<<(e->nchunks + 255) / 256, 256, 0, e->stream>>>(g, 1);
  KTG_CUDA(cudaGetLastError());
  KTG_TRY(read_state(e));
  KTG_TRY(ensure(e->d_pairs, e->cap_pairs, sizeof(uint2) * std::max<uint64_t>(1, e->h_st->pairs_needed)));
  e->live_pristine = e->h_st->live;
  e->has_graph = true;
  return KTG_OK;
}

// Enqueue one round: plan -> support -> [check16] -> [allreduce] -> prune -> control.
ktg_status enqueue_round(ktg_engine* e, bool graph_mode, cudaGraphConditionalHandle handle,
                         cudaEvent_t sup0 = nullptr, cudaEvent_t sup1 = nullptr) {
  Graph g = e->dev_graph();
  const cudaStream_t s = e->stream;
  const int fused = graph_mode ? 1 : 0;
  k_plan_count<<<(e->nchunks + 255) / 256, 256, 0, s>>>(g, 0);
  k_plan_write<<<1, 1024, 0, s>>>(g);
  if (sup0) KTG_CUDA(cudaEventRecord(sup0, s));
  if (flag(e, KTG_FLAG_NAIVE_SUPPORT)) {
    k_support_naive<<<4 * e->num_sms, 256, 0, s>>>(g);
  } else {
    k_support_chunked<<<e->support_grid, kSupportThreads, e->support_smem, s>>>(g);
  }
  if (sup1) KTG_CUDA(cudaEventRecord(sup1, s));
  if (e->opt.width_bits == 16) k_check16<<<4 * e->num_sms, 256, 0, s>>>(g);
  KTG_CUDA(cudaGetLastError());
  if (!graph_mode && e->world > 1 && e->allreduce) {
    // partial supports -> full supports on every rank
    uint32_t* buf = e->h_st->parity ? e->d_S1 : e->d_S0;
    if (e->allreduce(buf, e->slots, e->stream, e->allreduce_user) != 0)
      return fail(KTG_ERR_CUDA, "allreduce callback failed");
    // triangle counter is per-rank partial; fine (reported from rank sum by caller)
  }
  k_prune_light<<<e->prune_grid, kPruneThreads, 0, s>>>(g, fused);
  k_prune_heavy<<<e->heavy_grid, kPruneThreads, 0, s>>>(g, fused);
  k_control<<<1, 1, 0, s>>>(e->d_st, e->d_hist, handle, graph_mode ? 1 : 0);
  KTG_CUDA(cudaGetLastError());
  return KTG_OK;
}

ktg_status build_graph(ktg_engine* e) {
  const int naive = flag(e, KTG_FLAG_NAIVE_SUPPORT) ? 1 : 0;
  const int w16 = e->opt.width_bits == 16 ? 1 : 0;
  if (e->exec && e->exec_naive == naive && e->exec_w16 == w16 && e->exec_n == e->n &&
      e->exec_slots == e->slots && e->exec_col == e->d_col)
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
  e->exec_naive = naive;
  e->exec_w16 = w16;
  e->exec_n = e->n;
  e->exec_slots = e->slots;
  e->exec_col = e->d_col;
  return KTG_OK;
}

__global__ void k_set_live(DevState* st, unsigned long long live) { st->live = live; }

// Prepares the device state for a fixpoint at k. parity < 0 switches to the
// other support buffer on the device (it is all zero whenever the previous
// run converged, see k_prune_light), parity >= 0 selects it explicitly.
ktg_status begin_run(ktg_engine* e, uint32_t k, int parity) {
  k_begin<<<1, 1, 0, e->stream>>>(e->d_st, k >= 2 ? k - 2 : 0, e->opt.width_bits == 16 ? 1 : 0, parity);
  KTG_CUDA(cudaGetLastError());
  return KTG_OK;
}

ktg_status collect_work(ktg_engine* e, ktg_round_work* w) {
  Graph g = e->dev_graph();
  if (!e->d_din) KTG_CUDA(cudaMalloc(&e->d_din, (size_t)(e->n + 2) * 4));
  KTG_CUDA(cudaMemsetAsync(e->d_din, 0, (size_t)(e->n + 2) * 4, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_workL, 0, 8, e->stream));
  k_work_din<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(g, e->d_din);
  k_work_L<<<4 * e->num_sms, 256, 0, e->stream>>>(g, e->d_din, e->d_workL);
  KTG_CUDA(cudaGetLastError());
  unsigned long long L = 0, live = 0;
  KTG_CUDA(cudaMemcpyAsync(&L, e->d_workL, 8, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaMemcpyAsync(&live, &e->d_st->live, 8, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  w->L = L;
  w->live_edges = live;
  return KTG_OK;
}

// The fixpoint. Expects begin_run() already enqueued.
ktg_status run_loop(ktg_engine* e, bool want_sync) {
  const bool timing = flag(e, KTG_FLAG_TIME_SUPPORT);
  const bool recording = timing || flag(e, KTG_FLAG_COLLECT_WORK);
  const bool host_loop = flag(e, KTG_FLAG_HOST_LOOP) || e->opt.observer || (e->world > 1) || recording;
  e->work.clear();
  KTG_CUDA(cudaEventRecord(e->ev0, e->stream));
  if (!host_loop) {
    KTG_TRY(build_graph(e));
    KTG_CUDA(cudaGraphLaunch(e->exec, e->stream));
    KTG_CUDA(cudaEventRecord(e->ev1, e->stream));
    if (!want_sync) return KTG_OK;
    return read_state(e);
  }
  std::vector<uint32_t> h_col, h_S;
  if (e->opt.observer) {
    h_col.resize(e->slots);
    h_S.resize(e->slots);
  }
  KTG_TRY(read_state(e));  // parity of round 0
  for (uint32_t round = 0;; ++round) {
    // Host loop keeps S semantics of the reference: the round's buffer is
    // zeroed up front (reset_supports), prune leaves S untouched.
    uint32_t* Sc = e->h_st->parity ? e->d_S1 : e->d_S0;
    KTG_CUDA(cudaMemsetAsync(Sc, 0, (size_t)e->slots * 4, e->stream));
    ktg_round_work w{};
    if (flag(e, KTG_FLAG_COLLECT_WORK)) KTG_TRY(collect_work(e, &w));
    KTG_TRY(enqueue_round(e, false, 0, timing ? e->evs0 : nullptr, timing ? e->evs1 : nullptr));
    // removed of this round is hist[round]; read the whole state
    KTG_TRY(read_state(e));
    unsigned long long removed = 0;
    if (round < (uint32_t)kHistCap) {
      KTG_CUDA(cudaMemcpy(&removed, e->d_hist + round, 8, cudaMemcpyDeviceToHost));
    }
    if (recording) {
      w.triangles = e->h_st->last_triangles;
      w.removed = removed;
      if (timing) {
        float ms = 0;
        KTG_CUDA(cudaEventElapsedTime(&ms, e->evs0, e->evs1));
        w.support_ms = ms;
      }
      e->work.push_back(w);
    }
    if (e->opt.observer) {
      // S of the round: the buffer before control flipped parity
      const uint32_t par = removed != 0 && e->h_st->error == 0 ? (e->h_st->parity ^ 1u) : e->h_st->parity;
      KTG_CUDA(cudaMemcpy(h_col.data(), e->d_col, (size_t)e->slots * 4, cudaMemcpyDeviceToHost));
      KTG_CUDA(cudaMemcpy(h_S.data(), par ? e->d_S1 : e->d_S0, (size_t)e->slots * 4, cudaMemcpyDeviceToHost));
      e->opt.observer(h_col.data(), h_S.data(), e->slots, removed, e->opt.observer_user);
    }
    if (removed == 0 || e->h_st->error) break;
  }
  KTG_CUDA(cudaEventRecord(e->ev1, e->stream));
  return read_state(e);
}

ktg_status finish_info(ktg_engine* e) {
  float ms = 0;
  KTG_CUDA(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  e->info.iterations = e->h_st->iter;
  e->info.live_edges = e->h_st->live;
  e->info.triangles = e->h_st->last_triangles;
  e->info.device_ms = ms;
  if (e->h_st->error) {
    const uint64_t slot = e->h_st->overflow_slot;
    uint32_t cnt = 0;
    const uint32_t* Sc = e->h_st->parity ? e->d_S1 : e->d_S0;
    cudaMemcpy(&cnt, Sc + slot, 4, cudaMemcpyDeviceToHost);
    g_err_slot = slot;
    return fail(KTG_ERR_SUPPORT_OVERFLOW, "16-bit support overflow at slot " + std::to_string(slot) +
                                              " (count " + std::to_string(cnt) + ")");
  }
  return KTG_OK;
}

ktg_status copy_hist(ktg_engine* e, uint64_t* hist, uint32_t cap, uint32_t* iterations) {
  const uint32_t it = e->h_st->iter;
  if (iterations) *iterations = it;
  const uint32_t m = std::min<uint32_t>(std::min<uint32_t>(it, cap), (uint32_t)kHistCap);
  if (hist && m) KTG_CUDA(cudaMemcpy(hist, e->d_hist, (size_t)m * 8, cudaMemcpyDeviceToHost));
  return KTG_OK;
}

// One support pass into the current (parity) buffer, no reset.
ktg_status support_pass(ktg_engine* e, int parity, uint64_t* triangles, bool max_support) {
  Graph g = e->dev_graph();
  k_begin<<<1, 1, 0, e->stream>>>(e->d_st, 0, e->opt.width_bits == 16 ? 1 : 0, parity);
  k_plan_count<<<(e->nchunks + 255) / 256, 256, 0, e->stream>>>(g, 0);
  k_plan_write<<<1, 1024, 0, e->stream>>>(g);
  if (flag(e, KTG_FLAG_NAIVE_SUPPORT))
    k_support_naive<<<4 * e->num_sms, 256, 0, e->stream>>>(g);
  else
    k_support_chunked<<<e->support_grid, kSupportThreads, e->support_smem, e->stream>>>(g);
  if (e->opt.width_bits == 16) k_check16<<<4 * e->num_sms, 256, 0, e->stream>>>(g);
  if (max_support) k_max_support<<<4 * e->num_sms, 256, 0, e->stream>>>(g);
  KTG_CUDA(cudaGetLastError());
  KTG_TRY(read_state(e));
  if (triangles) *triangles = e->h_st->triangles;
  e->info.max_support = e->h_st->max_support;
  if (e->h_st->error) {
    const uint64_t slot = e->h_st->overflow_slot;
    uint32_t cnt = 0;
    cudaMemcpy(&cnt, (e->h_st->parity ? e->d_S1 : e->d_S0) + slot, 4, cudaMemcpyDeviceToHost);
    g_err_slot = slot;
    return fail(KTG_ERR_SUPPORT_OVERFLOW, "16-bit support overflow at slot " + std::to_string(slot) +
                                              " (count " + std::to_string(cnt) + ")");
  }
  return KTG_OK;
}

ktg_status extract(ktg_engine* e, uint32_t* u, uint32_t* v, uint32_t* s, uint64_t cap, uint64_t* num) {
  KTG_TRY(read_state(e));
  const uint64_t live = e->h_st->live;
  if (num) *num = live;
  if (live == 0) return KTG_OK;
  if (live > cap) return fail(KTG_ERR_INVALID_PARAMETER, "edge_cap is smaller than the survivor count");
  // row offsets (exclusive prefix of deg) on the host from a deg copy: the
  // survivors of a converged truss are what remains, O(n) bytes.
  std::vector<uint32_t> deg(e->n + 2);
  KTG_CUDA(cudaMemcpyAsync(deg.data(), e->d_deg, (size_t)(e->n + 2) * 4, cudaMemcpyDeviceToHost, e->stream));
  KTG_CUDA(cudaStreamSynchronize(e->stream));
  std::vector<unsigned long long> offs(e->n + 2, 0);
  unsigned long long acc = 0;
  for (uint32_t r = 1; r <= e->n; ++r) {
    offs[r] = acc;
    acc += deg[r];
  }
  unsigned long long* d_offs = nullptr;
  uint32_t* d_out = nullptr;
  KTG_CUDA(cudaMalloc(&d_offs, (size_t)(e->n + 2) * 8));
  KTG_CUDA(cudaMalloc(&d_out, (size_t)live * 12));
  KTG_CUDA(cudaMemcpyAsync(d_offs, offs.data(), (size_t)(e->n + 2) * 8, cudaMemcpyHostToDevice, e->stream));
  k_extract<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(e->dev_graph(), d_offs, d_out, d_out + live,
                                                           d_out + 2 * live);
  cudaError_t ke = cudaGetLastError();
  if (ke == cudaSuccess) ke = cudaMemcpyAsync(u, d_out, live * 4, cudaMemcpyDeviceToHost, e->stream);
  if (ke == cudaSuccess) ke = cudaMemcpyAsync(v, d_out + live, live * 4, cudaMemcpyDeviceToHost, e->stream);
  if (ke == cudaSuccess) ke = cudaMemcpyAsync(s, d_out + 2 * live, live * 4, cudaMemcpyDeviceToHost, e->stream);
  if (ke == cudaSuccess) ke = cudaStreamSynchronize(e->stream);
  cudaFree(d_offs);
  cudaFree(d_out);
  if (ke != cudaSuccess) return fail(KTG_ERR_CUDA, std::string("extract: ") + cudaGetErrorString(ke));
  return KTG_OK;
}

ktg_status reset(ktg_engine* e) {
  if (!e->has_graph) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  if (!e->pristine_valid) return fail(KTG_ERR_INVALID_PARAMETER, "engine was loaded without a pristine copy");
  const size_t sb = (size_t)e->slots * 4;
  KTG_CUDA(cudaMemcpyAsync(e->d_col, e->d_col_pristine, sb, cudaMemcpyDeviceToDevice, e->stream));
  KTG_CUDA(cudaMemcpyAsync(e->d_deg, e->d_deg_pristine, (size_t)(e->n + 2) * 4, cudaMemcpyDeviceToDevice,
                           e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_S0, 0, sb, e->stream));
  KTG_CUDA(cudaMemsetAsync(e->d_S1, 0, sb, e->stream));
  k_set_live<<<1, 1, 0, e->stream>>>(e->d_st, e->live_pristine);
  KTG_CUDA(cudaGetLastError());
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

thread_local ktg_engine* t_cached[64] = {};

ktg_status tmp_engine(const ktg_options* opt, const uint32_t* row_ptr, uint32_t n, const uint32_t* col,
                      uint64_t slots, bool pristine, TmpEngine& t) {
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
  return engine_load(t.e, row_ptr, n, col, slots, cudaMemcpyHostToDevice, pristine);
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
const char* ktg_version(void) { return "ktg 0.1 (sm_100a)"; }

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
  e->free_graph();
  dfree(e->d_st);
  dfree(e->d_hist);
  dfree(e->d_workL);
  if (e->h_st) cudaFreeHost(e->h_st);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->evs0) cudaEventDestroy(e->evs0);
  if (e->evs1) cudaEventDestroy(e->evs1);
  if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

ktg_status ktg_engine_load(ktg_engine* e, const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx,
                           uint64_t slots) {
  return engine_load(e, row_ptr, n, col_idx, slots, cudaMemcpyHostToDevice, true);
}

ktg_status ktg_engine_load_device(ktg_engine* e, const uint32_t* d_row_ptr, uint32_t n,
                                  const uint32_t* d_col_idx, uint64_t slots) {
  return engine_load(e, d_row_ptr, n, d_col_idx, slots, cudaMemcpyDeviceToDevice, true);
}

ktg_status ktg_engine_reset(ktg_engine* e) { return reset(e); }

ktg_status ktg_engine_run(ktg_engine* e, uint32_t k, uint64_t* removed_hist, uint32_t hist_cap,
                          uint32_t* iterations) {
  if (!e->has_graph) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  KTG_TRY(begin_run(e, k, -1));
  const bool want = removed_hist != nullptr || iterations != nullptr;
  KTG_TRY(run_loop(e, want));
  if (!want) return KTG_OK;
  KTG_TRY(finish_info(e));
  return copy_hist(e, removed_hist, hist_cap, iterations);
}

ktg_status ktg_engine_support_pass(ktg_engine* e, uint64_t* triangles) {
  if (!e->has_graph) return fail(KTG_ERR_INVALID_PARAMETER, "engine has no graph loaded");
  return support_pass(e, -1, triangles, true);
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
  KTG_TRY(read_state(e));
  if (col_idx) KTG_CUDA(cudaMemcpy(col_idx, e->d_col, (size_t)e->slots * 4, cudaMemcpyDeviceToHost));
  if (supports)
    KTG_CUDA(cudaMemcpy(supports, e->h_st->parity ? e->d_S1 : e->d_S0, (size_t)e->slots * 4,
                        cudaMemcpyDeviceToHost));
  return KTG_OK;
}

ktg_status ktg_engine_device_state(ktg_engine* e, uint32_t** d_col_idx, uint32_t** d_supports, void** stream) {
  KTG_TRY(read_state(e));
  if (d_col_idx) *d_col_idx = e->d_col;
  if (d_supports) *d_supports = e->h_st->parity ? e->d_S1 : e->d_S0;
  if (stream) *stream = e->stream;
  return KTG_OK;
}

ktg_status ktg_engine_extract(ktg_engine* e, uint32_t* out_u, uint32_t* out_v, uint32_t* out_support,
                              uint64_t edge_cap, uint64_t* num_edges) {
  return extract(e, out_u, out_v, out_support, edge_cap, num_edges);
}

ktg_status ktg_engine_set_partition(ktg_engine* e, uint32_t rank, uint32_t world, ktg_allreduce_cb allreduce,
                                    void* user) {
  if (world == 0 || rank >= world) return fail(KTG_ERR_INVALID_PARAMETER, "rank must be < world");
  if (world > 1 && !allreduce) return fail(KTG_ERR_INVALID_PARAMETER, "world > 1 needs an allreduce callback");
  e->rank = rank;
  e->world = world;
  e->allreduce = allreduce;
  e->allreduce_user = user;
  if (e->exec) cudaGraphExecDestroy(e->exec);
  e->exec = nullptr;
  return KTG_OK;
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
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, t));
  // accumulate onto the caller's counts, like the reference (which requires
  // them zero but adds into whatever is there)
  KTG_CUDA(cudaMemcpyAsync(t.e->d_S0, supports, slots * 4, cudaMemcpyHostToDevice, t.e->stream));
  uint64_t tri = 0;
  const ktg_status st = support_pass(t.e, 0, &tri, false);
  if (st != KTG_OK) return st;
  KTG_CUDA(cudaMemcpy(supports, t.e->d_S0, slots * 4, cudaMemcpyDeviceToHost));
  if (triangles) *triangles = tri;
  return KTG_OK;
}

ktg_status ktg_intersect_tails(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots,
                               uint32_t pivot_slot, uint32_t predecessor, uint32_t* supports, uint32_t* found) {
  if (pivot_slot >= slots || predecessor == 0 || predecessor > n)
    return fail(KTG_ERR_INVALID_PARAMETER, "pivot slot / predecessor out of range");
  TmpEngine t;
  KTG_TRY(tmp_engine(nullptr, row_ptr, n, col_idx, slots, false, t));
  ktg_engine* e = t.e;
  KTG_CUDA(cudaMemcpyAsync(e->d_S0, supports, slots * 4, cudaMemcpyHostToDevice, e->stream));
  uint32_t* d_found = e->d_heavy;  // scratch
  k_intersect_one<<<1, 1, 0, e->stream>>>(e->d_row_ptr, e->d_col, e->d_S0, pivot_slot, predecessor, d_found);
  KTG_CUDA(cudaGetLastError());
  KTG_CUDA(cudaMemcpyAsync(supports, e->d_S0, slots * 4, cudaMemcpyDeviceToHost, e->stream));
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
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, t));
  ktg_engine* e = t.e;
  KTG_CUDA(cudaMemcpyAsync(e->d_S0, supports, slots * 4, cudaMemcpyHostToDevice, e->stream));
  KTG_TRY(begin_run(e, k, 0));
  Graph g = e->dev_graph();
  k_prune_light<<<e->prune_grid, kPruneThreads, 0, e->stream>>>(g, 0);
  k_prune_heavy<<<e->heavy_grid, kPruneThreads, 0, e->stream>>>(g, 0);
  KTG_CUDA(cudaGetLastError());
  KTG_TRY(read_state(e));
  KTG_CUDA(cudaMemcpy(col_idx, e->d_col, slots * 4, cudaMemcpyDeviceToHost));
  if (removed) *removed = e->h_st->removed;
  return KTG_OK;
}

ktg_status ktg_run_fixpoint(const uint32_t* row_ptr, uint32_t n, uint32_t* col_idx, uint64_t slots,
                            uint32_t* supports, uint64_t s_len, uint32_t k, const ktg_options* opt,
                            uint64_t* removed_hist, uint32_t hist_cap, uint32_t* iterations) {
  if (s_len != slots) return fail(KTG_ERR_INVALID_PARAMETER, "support array does not match slot count");
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, t));
  ktg_engine* e = t.e;
  KTG_TRY(begin_run(e, k, 0));
  KTG_TRY(run_loop(e, true));
  const ktg_status st = finish_info(e);
  // write back the (possibly partially pruned) state even on overflow
  KTG_CUDA(cudaMemcpy(col_idx, e->d_col, slots * 4, cudaMemcpyDeviceToHost));
  KTG_CUDA(cudaMemcpy(supports, e->h_st->parity ? e->d_S1 : e->d_S0, slots * 4, cudaMemcpyDeviceToHost));
  if (st != KTG_OK) return st;
  return copy_hist(e, removed_hist, hist_cap, iterations);
}

ktg_status ktg_ktruss(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots, uint32_t k,
                      const ktg_options* opt, uint32_t* out_u, uint32_t* out_v, uint32_t* out_support,
                      uint64_t edge_cap, uint64_t* num_edges, uint64_t* removed_hist, uint32_t hist_cap,
                      uint32_t* iterations) {
  if (k < 2) return fail(KTG_ERR_INVALID_PARAMETER, "k must be >= 2");
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, false, t));
  ktg_engine* e = t.e;
  KTG_TRY(begin_run(e, k, 0));
  KTG_TRY(run_loop(e, true));
  KTG_TRY(finish_info(e));
  KTG_TRY(copy_hist(e, removed_hist, hist_cap, iterations));
  return extract(e, out_u, out_v, out_support, edge_cap, num_edges);
}

ktg_status ktg_kmax_search(const uint32_t* row_ptr, uint32_t n, const uint32_t* col_idx, uint64_t slots,
                           const ktg_options* opt, uint32_t* k_max, uint32_t* out_u, uint32_t* out_v,
                           uint32_t* out_support, uint64_t edge_cap, uint64_t* num_edges,
                           uint64_t* removed_hist, uint32_t hist_cap, uint32_t* iterations) {
  TmpEngine t;
  KTG_TRY(tmp_engine(opt, row_ptr, n, col_idx, slots, true, t));
  ktg_engine* e = t.e;
  if (e->live_pristine == 0) return fail(KTG_ERR_INVALID_PARAMETER, "kmax_search needs a non-empty graph");
  // Bound pass (truss.cpp:77-80): one support pass on the pristine graph.
  KTG_TRY(reset(e));
  KTG_TRY(support_pass(e, 0, nullptr, true));
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
