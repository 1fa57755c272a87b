"""profiles/r02/traffic.json from an ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum CSV:
per-launch DRAM bytes of a kernel over a bench step (bench.py's roofline.traffic).
usage: traffic_json.py CSV WORKLOAD KERNEL SHOTS [LAUNCHES_PER_STEP]"""
import csv
import json
import os
import sys
from collections import defaultdict


def main():
    csv_path, workload, kernel, shots = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    byid = defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        d = dict(zip(rows[hdr], r))
        if kernel not in d.get("Kernel Name", ""):
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20, "GB": 1 << 30}.get(unit, 1)
        byid[d["ID"]][d["Metric Name"]] = v * scale
        names[d["ID"]] = d["Kernel Name"]
    # the timed step's launches: the first `per_step` of the kernel in launch order (bench.py
    # --steps 1 --warmup 0 runs the step before its end-to-end leg)
    ids = sorted(byid, key=int)
    if len(sys.argv) > 5:
        ids = ids[:int(sys.argv[5])]
    launches = len(ids)
    rd = sum(byid[i].get("dram__bytes_read.sum", 0) for i in ids)
    wr = sum(byid[i].get("dram__bytes_write.sum", 0) for i in ids)
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02", "traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data[workload] = {"kernel": kernel, "shots": shots, "launches_per_step": launches,
                      "dram_bytes_per_launch": (rd + wr) / max(launches, 1), "dram_bytes_per_step": rd + wr,
                      "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:{kernel} "
                                f"(bench.py --steps 1, {workload}, {shots} shots): read {rd / 1e9:.3f} GB + write "
                                f"{wr / 1e9:.3f} GB over {launches} launches; {os.path.basename(csv_path)}"}
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(data[workload]))


if __name__ == "__main__":
    main()
