"""Per-round kernel times from an ncu launch-list CSV (host-loop profile run):
one line per round with the main kernels' microseconds."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0].replace("ktg::", "").replace("void ", ""), float(d["Metric Value"]) / 1000))
fix = -1; rnd = None; rounds = []
for k, us in out:
    if k == "k_begin":
        fix += 1
    if k in ("k_plan_count", "k_support_a22") and fix >= 0 and (rnd is None or "k_control_inc" in rnd or "k_control" in rnd):
        rnd = collections.OrderedDict(); rounds.append((fix, rnd))
    if rnd is not None:
        rnd[k] = rnd.get(k, 0) + us
keys = ["k_support_a22", "k_support_chunked", "k_mark", "k_mark_frontier", "k_queues", "k_delta", "k_delta_big",
        "k_inc_rows<0>", "k_inc_rows<1>", "k_inc_sym<0>", "k_inc_sym<1>", "k_inc_zero", "k_publish_inc<0>",
        "k_publish_inc<1>"]
short = ["a22", "chunk", "mark", "mfr", "q", "delta", "dbig", "rows", "rowsH", "sym", "symH", "zero", "pub", "pubH"]
print("fx rd " + " ".join(f"{s:>7s}" for s in short) + "   total")
for i, (f, r) in enumerate(rounds):
    tot = sum(r.values())
    print(f"{f:2d} {i:2d} " + " ".join(f"{r.get(k, 0):7.1f}" for k in keys) + f" {tot:7.1f}")
