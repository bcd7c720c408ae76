"""Summarise an ncu report (raw page) and/or a launch-list CSV into profiles/.

usage: python scripts/ncu_summary.py --rep gpurun_out/x.ncu-rep --out profiles/name
       python scripts/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/name
"""
import argparse, collections, csv, io, json, subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_op_red.sum",
    "lts__t_sectors_op_atom.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        nm = r[ki].split("(")[0]
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(t for _, t in agg.values())
    return [{"kernel": k, "launches": c, "total_ms": t / 1e6, "share": t / tot}
            for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    doc = {"title": a.title}
    md = [f"# {a.title}\n"]
    if a.rep:
        doc["ncu_full"] = rep(a.rep)
        for d in doc["ncu_full"]:
            md.append(f"## {d['kernel'][:100]}\n\n| metric | value |\n|---|---|")
            md += [f"| {k} | {v} |" for k, v in d.items() if k != "kernel"]
            md.append("")
    if a.launches:
        doc["launches"] = launches(a.launches)
        md.append("## launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        md.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
        md += [f"| {d['kernel']} | {d['launches']} | {d['total_ms']:.3f} | {100*d['share']:.1f}% |" for d in doc["launches"]]
    json.dump(doc, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))
