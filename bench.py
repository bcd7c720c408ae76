#!/usr/bin/env python
"""K-truss benchmark on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): R-MAT scale-20 edgefactor-16 (Graph500
a/b/c, seed 42), K sweep 3..K_max. One step = the whole
sweep, every K from the pristine graph exactly as the reference's
ktruss(graph, k) would run it (truss.cpp:57-71) -- no state carried between
K values. Metric: edges/s = (#K * m) / sweep time, m = original canonical
edges (bench.cpp:45); time-to-fixpoint per K is reported alongside.

  value    device-resident sweep: graph in HBM, per K a D2D restore of the
           pristine col_idx + the device-side fixpoint (CUDA-graph while loop),
           CUDA events on the engine stream, max over ranks.
  e2e      the same sweep through the reference-shaped C ABI with HOST
           buffers (ktg_ktruss: H2D of the CSR, fixpoint, D2H of the truss)
           per K, from pinned memory.
  roofline the support kernel (k_support_a22): algorithmic bytes of
           SURVEY.md §8(d) per launch / its CUDA-event duration (host-driven
           instrumented pass, sampled K values).
  cpu_baseline  the reference library itself (oracle/_ref, Strategy::Fine,
           all host threads) on a bounded sample of the same sweep.

--impl reference times only the reference CPU implementation (rank 0).
Multi-GPU (torchrun): the K values are split across ranks (independent
fixpoints on a replicated graph; no data-path collective), strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "K-truss time-to-fixpoint (ms) & edges/sec at 1/2/4/8 B200; achieved HBM GB/s"
# K_max of the pinned configs (reference-measured; also
# asserted by tests/test_gpu_large.py) -- lets the reference arm skip its
# ~200 s CPU kmax_search.
KNOWN_KMAX = {(14, 16, 42): 79, (20, 16, 42): 304, (24, 16, 42): 935, ("er", 22, 16, 42): 3,
              ("cliques", 22, 32, 42): 1057, ("cliques", 24, 32, 42): 1654}


def make_graph(args):
    import paper_2009_07929_b200 as kt
    if args.graph == "er":
        return kt.erdos_renyi(args.scale, args.ef << args.scale, args.seed)
    if args.graph == "cliques":
        return kt.rmat_cliques(args.scale, args.ef, args.seed)
    return kt.rmat(args.scale, args.ef, args.seed)


def kmax_key(args):
    if args.graph != "rmat":
        return (args.graph, args.scale, args.ef, args.seed)
    return (args.scale, args.ef, args.seed)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--kstride", type=int, default=1, help="K sweep stride (1 = every K)")
    ap.add_argument("--concurrency", type=int, default=4,
                    help="sweep mode: resident engines (graph copies) per GPU running K values "
                         "concurrently on their own streams")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="sweep", choices=["sweep", "fixpoint"],
                    help="sweep: K sweep 3..K_max (K split across ranks); fixpoint: one fixpoint per step "
                         "at --k (0 = K_max), edge-partitioned over NCCL across ranks")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="fixpoint mode, N>1: ncclAllReduce of partial supports, or the reduce-scatter fused "
                         "into the support kernel (peer atomics + span all-gather over CUDA IPC)")
    ap.add_argument("--graph", default="rmat", choices=["rmat", "er", "cliques"],
                    help="er: Erdős–Rényi with 2^scale vertices and ef*2^scale draws (SURVEY §8(d)); "
                         "cliques: R-MAT plus planted cliques of 128..1024 (configs[4])")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed
    region."""

    REASONS = {
        0x0000000000000002: "applications_clocks",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_model() -> str:
    """The host CPU's model name (the reference timing's hardware)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def k_values(kmax: int, stride: int):
    ks = list(range(3, kmax + 1, stride))
    if ks[-1] != kmax:
        ks.append(kmax)
    return ks


def support_bytes(w, n, slots):
    """Algorithmic bytes of one support launch: list reads
    4*L_r, pivot scan 4*slots, IA 4*(n+2), 3 atomic u32 per triangle."""
    return 4 * w["L"] + 4 * slots + 4 * (n + 2) + 12 * w["triangles"]


def executed_bytes(w, n, slots, m):
    """Bytes k_support_a22 itself moves per launch: the a12 tails it streams
    (4*L_tail), the staged A22 chunks (4*slots), the pivot records (8 per
    live edge), row offsets/degrees (8*(n+2)) and 3 u32 atomics per
    triangle."""
    return 4 * w["L_tail"] + 4 * slots + 8 * m + 8 * (n + 2) + 12 * w["triangles"]


def fixpoint_bytes(work, n, slots):
    """Per-fixpoint algorithmic bytes B of SURVEY.md §8(d) (support + the
    16 B/slot prune)."""
    return sum(support_bytes(w, n, slots) + 16 * slots for w in work)


def cpu_sample(g, ks, budget_s, threads):
    """The reference library (oracle/_ref) on a bounded, evenly spread sample
    of the sweep's K values; every K from pristine; run_fixpoint timed only
    (bench.cpp:33-40). Returns (edges/s, sample description, ms list)."""
    import oracle
    R = oracle.ref()
    # spread: K=3 (heaviest), K_max, then bisecting the range
    cand = [ks[0], ks[-1]]
    step = max(1, len(ks) // 2)
    while step >= 1 and len(cand) < len(ks):
        for i in range(0, len(ks), step):
            if ks[i] not in cand:
                cand.append(ks[i])
        step //= 2
    t_total, done = 0.0, []
    for k in cand:
        _, _, _, ms = R.run_fixpoint(g, k, 2, threads)
        done.append((k, ms))
        t_total += ms / 1e3
        if t_total >= budget_s:
            break
    m = g.num_edges
    tot_ms = sum(ms for _, ms in done)
    return m * len(done) / (tot_ms / 1e3), done


def run_reference(args):
    """--impl reference: the reference's own CPU implementation only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import paper_2009_07929_b200 as kt
    g = kt.rmat(args.scale, args.ef, args.seed)
    key = (args.scale, args.ef, args.seed)
    if key not in KNOWN_KMAX:
        print(json.dumps({"impl": "reference", "unavailable": f"no pinned K_max for {key}"}))
        return
    ks = k_values(KNOWN_KMAX[key], args.kstride)
    R = oracle.ref()
    threads = os.cpu_count() or 1
    # evenly spread K order so any step count samples the whole sweep
    order = []
    stride = max(1, len(ks) // max(1, args.steps + args.warmup))
    for off in range(stride):
        order.extend(ks[off::stride])
    times = []
    for i in range(args.warmup + args.steps):
        k = order[i % len(order)]
        _, _, _, ms = R.run_fixpoint(g, k, 2, threads)
        if i >= args.warmup:
            times.append((k, ms))
    mean_ms = sum(ms for _, ms in times) / len(times)
    value = g.num_edges / (mean_ms / 1e3)
    sample = f"one pristine fixpoint per step, K in {[k for k, _ in times]}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": f"rmat-s{args.scale}-ef{args.ef} K-sweep 3..{ks[-1]} (pristine per K)",
                   "n": g.num_vertices, "m": g.num_edges, "k_values": len(ks), "parallelism": "cpu-omp"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "fixpoint":
        return run_fixpoint_mode(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2009_07929_b200 as kt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    t0 = time.time()
    g = kt.rmat(args.scale, args.ef, args.seed)
    gen_s = time.time() - t0
    n, slots, m = g.num_vertices, g.total_slots(), g.num_edges

    stream = torch.cuda.Stream()
    eng = kt.Engine(g, stream=stream.cuda_stream)
    kmax = eng.kmax()  # untimed, as run_bench resolves K_max (bench.cpp:25)
    ks = k_values(kmax, args.kstride)
    # K split across ranks: greedy by a cost proxy (K=3 is the heaviest)
    mine = ks[rank::world]

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    # P resident engines, each a full copy of the graph on its own stream,
    # take the K values round-robin: the tail of one fixpoint (short,
    # launch-latency-bound carried rounds) overlaps another's full passes
    P = max(1, args.concurrency)
    side_streams = [torch.cuda.Stream() for _ in range(P - 1)]
    engs = [eng] + [kt.Engine(g, stream=st.cuda_stream) for st in side_streams]
    all_streams = [stream] + side_streams

    def sweep(kset):
        for i, k in enumerate(kset):
            e = engs[i % P]
            e.reset()
            e.run(k, sync=False)

    launches_per_k = {}
    rounds_per_k = {}
    live_per_k = {}
    latency_ms = {}
    # one synchronous pass: iterations per K (for the launch count) + checks
    for k in mine:
        eng.reset()
        h = eng.run(k)
        # k_set_live + k_begin + 13 per round (A22-staged support, mark x2, decide,
        # queues, delta, rows x2, sym x2, zero, control; the ones a round does
        # not need exit at once) + 2 triangle total + 4 publish
        launches_per_k[k] = 2 + 13 * len(h) + 2 + 4
        rounds_per_k[k] = len(h)
        live_per_k[k] = eng.info()["live_edges"]
        latency_ms[k] = eng.info()["device_ms"]

    for _ in range(args.warmup):
        sweep(mine)
    torch.cuda.synchronize()

    step_ms = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush between timed steps (not timed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for st in side_streams:  # every engine starts after the flush and e0
                st.wait_event(e0)
            sweep(mine)
            for st in side_streams:  # e1 after every engine's last fixpoint
                done = torch.cuda.Event()
                done.record(st)
                stream.wait_event(done)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier()
    # every engine's last fixpoint of the timed sweep left the same survivor
    # count as the one-at-a-time pass (the concurrent engines share nothing)
    conc_ok = True
    for i, e in enumerate(engs):
        last = [k for j, k in enumerate(mine) if j % P == i]
        if last:
            e.sync()  # reads the device state of its last (asynchronous) fixpoint
            conc_ok &= e.info()["live_edges"] == live_per_k[last[-1]]
    ms_per_step = allmax(sum(step_ms) / len(step_ms))
    lat_mean = allmax(sum(latency_ms.values()) / max(1, len(latency_ms)))
    total_k = len(ks)
    value = total_k * m / (ms_per_step / 1e3)

    # ---- secondary: incremental sweep, one GPU, untimed by the
    # contract; each K starts from the previous truss (same survivors/supports)
    incr = None
    if world == 1:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.reset()
        iters, same = 0, True
        for k in ks:
            h = eng.run(k)
            iters += len(h)
            same &= eng.info()["live_edges"] == live_per_k.get(k, eng.info()["live_edges"])
        e1.record(stream)
        e1.synchronize()
        incr_ms = e0.elapsed_time(e1)
        incr = {"ms": incr_ms, "value": total_k * m / (incr_ms / 1e3), "unit": "edges/s", "rounds": iters,
                "pristine_rounds": sum(rounds_per_k.values()),
                "survivors_equal_pristine": bool(same),
                "note": "each K from the (K-1)-truss; not the headline (value is pristine per K)"}

    # ---- end to end through the reference-shaped C ABI (host buffers) ----
    pin_keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True),
                torch.empty(slots, dtype=torch.int32, pin_memory=True))
    pin_rp = pin_keep[0].numpy().view(np.uint32)
    pin_col = pin_keep[1].numpy().view(np.uint32)
    pin_rp[:] = g.row_ptr
    pin_col[:] = g.col_idx
    hg = kt.ZeroTerminatedCsr(n, pin_rp, pin_col)
    e2e_ms, d2h = [], 0
    if mine:  # untimed warm-up call: the cached host-API engine and the pinned result pool
        kt.ktruss(hg, mine[0])
    barrier()
    for _ in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        d2h = 0
        for k in mine:
            r = kt.ktruss(hg, k)
            d2h += r.nbytes + 8 * r.iterations
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t) * 1e3)
    barrier()
    e2e_step_ms = allmax(sum(e2e_ms) / len(e2e_ms))
    h2d = allsum(len(mine) * (n + 2 + slots) * 4)
    d2h = allsum(d2h)

    # ---- roofline of the support kernel (instrumented, untimed) ----
    roof = None
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            peak, peak_src = float(peaks["hbm_gbs"]), "measured"
        except Exception:
            peak, peak_src = 6650.0, "fallback"
        sample_k = sorted(set([ks[0]] + ks[len(ks) // 4::max(1, len(ks) // 4)] + [ks[-1]]))
        # the headline path's support kernel (k_support_a22) on the rounds
        # that run a full pass; no round-0 degree bound here, so every launch
        # is a whole-graph pass whose algorithmic bytes are the §8(d) formula
        ew = kt.Engine(g, kt.TrussOptions(no_degree_bound=True), collect_work=True)
        et = kt.Engine(g, kt.TrussOptions(no_degree_bound=True), time_support=True)
        tot_b = tot_ms = tot_x = 0.0
        n_launch = 0
        fix_b = 0.0
        for k in sample_k:
            ew.reset()
            ew.run(k)
            work = ew.round_work()
            et.reset()
            et.run(k)
            tw = et.round_work()
            for w, t in zip(work, tw):
                if not t["full_pass"]:  # supports carried: the launch exits at once
                    continue
                tot_b += support_bytes(w, n, slots)
                tot_x += executed_bytes(w, n, slots, w["live_edges"])
                tot_ms += t["support_ms"]
                n_launch += 1
            fix_b += fixpoint_bytes(work, n, slots)
        ew.close()
        et.close()
        achieved = tot_b / (tot_ms / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "support_traffic.json")
        if os.path.exists(tp):
            try:
                tj = json.load(open(tp))
                traffic = tj.get(f"rmat-s{args.scale}-ef{args.ef}")
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": peak_src, "kernel": "k_support_a22",
                "launches_measured": n_launch, "sample_k": sample_k,
                "bytes_per_launch_avg": tot_b / max(1, n_launch),
                "ms_per_launch_avg": tot_ms / max(1, n_launch),
                "executed_bytes_per_launch_avg": tot_x / max(1, n_launch),
                "executed_frac": round(tot_x / (tot_ms / 1e3) / 1e9 / peak, 4),
                "note": "achieved = SURVEY §8(d) algorithmic bytes (full merge view, 4 B per list element of "
                        "L) / time; the kernel itself reads only the a12 tails (executed bytes = "
                        "4*L_tail + 4*slots staged + 8*m pivot records + 12*T)"}

    # ---- CPU baseline: the reference library on the host cores ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            v, done = cpu_sample(g, ks, args.cpu_budget_s, threads)
            cpu = {"value": v, "unit": "edges/s", "cores": threads, "kind": "reference",
                   "sample": "reference run_fixpoint (Strategy::Fine) from pristine at K in "
                             f"{[k for k, _ in done]} ({', '.join(f'{ms:.0f}' for _, ms in done)} ms)",
                   "cpu": cpu_model()}
        except Exception as ex:  # reference library not built
            cpu = {"value": None, "unit": "edges/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    launches = args.steps * sum(launches_per_k.values())
    launches = int(allsum(launches))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {
                "workload": f"rmat-s{args.scale}-ef{args.ef} K-sweep 3..{kmax} (pristine per K)",
                "graph": f"R-MAT scale {args.scale} edgefactor {args.ef} seed {args.seed} "
                         "(a,b,c)=(.57,.19,.19), Fisher-Yates relabel",
                "n": n, "m": m, "slots": slots, "k_max": kmax, "k_values": total_k,
                "kstride": args.kstride,
                "concurrency": f"{P} resident engines per GPU on their own streams, K values round-robin",
                "concurrent_results_match": bool(conc_ok),
                "l2": "512 MiB memset between timed steps (col_idx 65 MB < L2); per-K D2D restore",
                "parallelism": f"k-split x{world}" if world > 1 else "single",
            },
            # one fixpoint at a time on one engine (CUDA events, the sync pass)
            "time_to_fixpoint_ms_mean": lat_mean,
            # the sweep's throughput: step time per K value
            "sweep_ms_per_k": ms_per_step / total_k * world,
            "me_per_s": value / 1e6,
            "e2e": {"value": total_k * m / (e2e_step_ms / 1e3), "unit": "edges/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": e2e_step_ms, "api": "ktg_ktruss (host buffers, pinned)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "incremental_sweep": incr,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "gen_s": round(gen_s, 2),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    for e in engs[1:]:
        e.close()
    if world > 1:
        dist.destroy_process_group()


def cpu_port_sample(g, k, budget_s, threads, world_parts=64):
    """CPU baseline for graphs too large to run whole within the budget: the
    C port (oracle/ktruss_oracle.c, OpenMP) restricted to 1/world_parts of
    the engine's support tasks of the pristine round-1 pass, scaled back up.
    Returns (edges/s estimate for the fixpoint's round 1 only, description)."""
    import time as _t

    import oracle
    P = oracle.port()
    t0 = _t.perf_counter()
    P.support_tasks(g, 0, world_parts)
    dt = (_t.perf_counter() - t0) * world_parts
    return g.num_edges / dt, (f"C port, support tasks t%{world_parts}==0 of the pristine round-1 pass "
                              f"(single thread), scaled x{world_parts}: {dt:.1f} s per support pass; "
                              "lower bound on the fixpoint time")


def run_fixpoint_mode(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2009_07929_b200 as kt
    from paper_2009_07929_b200 import dist as kd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t0 = time.time()
    g = make_graph(args)
    gen_s = time.time() - t0
    n, slots, m = g.num_vertices, g.total_slots(), g.num_edges
    stream = torch.cuda.Stream()
    eng = kt.Engine(g, stream=stream.cuda_stream)
    k = args.k or KNOWN_KMAX.get(kmax_key(args)) or eng.kmax()
    if world > 1:
        if args.exchange == "fused":
            kd.engine_join_fused(eng)
        else:
            kd.engine_join(eng)
    eng.reset()
    hist = eng.run(k)
    # carried-support rounds (13 launches per round + 2 + 4), also across
    # ranks with the NCCL exchange; the fused peer exchange recomputes every
    # round (6 per round + 5 publish)
    fused = world > 1 and args.exchange == "fused"
    launches = (2 + 6 * len(hist) + 5) if fused else (2 + 13 * len(hist) + 2 + 4)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        eng.reset()
        eng.run(k, sync=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            eng.reset()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.run(k, sync=False)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = kd.max_over_ranks(sum(step_ms) / len(step_ms), dev)
    value = m / (ms / 1e3)
    # e2e: the engine's public API from pinned host buffers each step
    keep = (torch.empty(n + 2, dtype=torch.int32, pin_memory=True), torch.empty(slots, dtype=torch.int32,
                                                                                 pin_memory=True))
    keep[0].numpy().view(np.uint32)[:] = g.row_ptr
    keep[1].numpy().view(np.uint32)[:] = g.col_idx
    hg = kt.ZeroTerminatedCsr(n, keep[0].numpy().view(np.uint32), keep[1].numpy().view(np.uint32))
    eng.load(hg)  # untimed warm-up of the same sequence (pinned result pool)
    eng.run(k)
    edges = eng.extract()
    del edges
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.load(hg)
    eng.run(k)
    edges = eng.extract()
    torch.cuda.synchronize()
    e2e_ms = kd.max_over_ranks((time.perf_counter() - t) * 1e3, dev)
    roof = None
    cpu = None
    if rank == 0:
        try:
            peak, src = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
        except Exception:
            peak, src = 6650.0, "fallback"
        # full support passes every round (recompute mode): each launch is a
        # whole-graph pass whose algorithmic bytes are the §8(d) formula
        # one rank: the carried-support path's k_support_a22 (full-pass rounds,
        # no round-0 degree bound); ranks > 1 recompute with k_support_chunked
        ro = kt.TrussOptions(no_degree_bound=True) if world == 1 else kt.TrussOptions(recompute=True)
        ew = kt.Engine(g, ro, collect_work=True)
        et = kt.Engine(g, ro, time_support=True)
        ew.reset(); ew.run(k); w = ew.round_work()
        et.reset(); et.run(k); tw = et.round_work()
        ew.close(); et.close()
        full = [(x, t) for x, t in zip(w, tw) if t["full_pass"]]  # carried rounds skip the kernel
        tb = sum(support_bytes(x, n, slots) for x, _ in full)
        tm = sum(t["support_ms"] for _, t in full)
        achieved = tb / (tm / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_source": src,
                "kernel": "k_support_a22" if world == 1 else "k_support_chunked",
                "launches_measured": len(full)}
        if world == 1 and not args.no_cpu_baseline:
            v, desc = cpu_port_sample(g, k, args.cpu_budget_s, 1)
            cpu = {"value": v, "unit": "edges/s", "cores": 1, "kind": "port", "sample": desc}
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": (f"er-2^{args.scale}-{args.ef}x K={k} fixpoint" if args.graph == "er" else
                                    f"rmat-s{args.scale}-ef{args.ef}+cliques(128..1024) K={k} fixpoint"
                                    if args.graph == "cliques" else
                                    f"rmat-s{args.scale}-ef{args.ef} K={k} fixpoint"),
                       "n": n, "m": m, "slots": slots, "k": k, "rounds": len(hist),
                       "l2": "512 MiB memset between timed steps; inputs > L2" if slots * 4 > 126e6 else
                             "512 MiB memset between timed steps",
                       "parallelism": (f"edge-partitioned x{world} (" + ("support kernel fused with the reduce-scatter, span "
                                                                     "all-gather per round" if args.exchange == "fused" else
                                                                     "A22 tasks split by rank, ncclAllReduce of S after each full pass, "
                                                                     "carried rounds replicated") + ")")
                       if world > 1
                                      else "single"},
            "time_to_fixpoint_ms": ms, "me_per_s": value / 1e6,
            "e2e": {"value": m / (e2e_ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": (n + 2 + slots) * 4,
                    "d2h_bytes_per_step": int(edges.nbytes), "ms_per_step": e2e_ms,
                    "api": "Engine.load (pinned host) + run + extract"},
            "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches * args.steps,
            "clocks": clocks.summary(), "gen_s": round(gen_s, 2),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
