"""Per-kernel totals from an ncu launch-list CSV; with --second, only the
launches after the midpoint marker kernel's second occurrence."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"][:90], float(d["Metric Value"]) / 1000))
if len(sys.argv) > 2:
    marker = sys.argv[2]
    idx = [i for i, (k, _) in enumerate(out) if k.startswith(marker)]
    out = out[idx[1]:] if len(idx) > 1 else out
tot = sum(us for _, us in out)
for k, us in out:
    print(f"{us:9.1f}  {k}")
print(f"total {tot:.1f} us over {len(out)} launches")
