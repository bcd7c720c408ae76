"""Mean DRAM bytes per full-pass k_support_a22 launch from an ncu CSV
(metrics dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum)
-> profiles/support_traffic.json (read by bench.py's roofline.traffic)."""
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launch = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if "k_support_a22" not in d["Kernel Name"]:
            continue
        v = float(d["Metric Value"])
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        launch.setdefault(d["ID"], {})[d["Metric Name"]] = v * scale
full = [x for x in launch.values() if x.get("gpu__time_duration.sum", 0) > 50e3]  # > 50 us: a full pass ran
rd = sum(x["dram__bytes_read.sum"] for x in full) / len(full)
wr = sum(x["dram__bytes_write.sum"] for x in full) / len(full)
out = {"rmat-s20-ef16": rd + wr, "launches": len(full), "read_bytes_mean": rd, "write_bytes_mean": wr,
       "_note": "mean dram__bytes_read.sum+dram__bytes_write.sum per full-pass k_support_a22 launch (fixpoints "
                "K=3,78,153,228,303,304 from pristine, carried supports, no round-0 degree bound, host loop, ncu "
                "--clock-control none, cold-cache serialised); scripts/traffic_run.py + traffic_summary.py"}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(out)
