"""Summarise ncu launch captures (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum on k1_flow / k2_flow, one bench
config per CSV) into profiles/<round>_traffic.json, the DRAM bytes per launch
bench.py reports as roofline.traffic / frac_dram.
Usage: python tools/traffic_json.py r2 gpurun_out/r2b_traffic_*.csv"""
import csv
import io
import json
import os
import re
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    txt = open(path).read()
    body = txt[txt.index('"ID"'):]
    per = {}
    for r in csv.DictReader(io.StringIO(body)):
        per.setdefault(r["ID"], {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(per.values())


def main():
    tag, files = sys.argv[1], sys.argv[2:]
    out = {}
    for f in files:
        cfg = re.search(r"traffic_(\w+)\.csv", f).group(1)
        rows = parse(f)
        if not rows:
            continue
        rd = [r["dram__bytes_read.sum"] for r in rows]
        wr = [r["dram__bytes_write.sum"] for r in rows]
        du = [r["gpu__time_duration.sum"] for r in rows]
        out[cfg] = {"kernel": rows[0]["kernel"], "launches_captured": len(rows), "launches_per_apply": 1,
                    "dram_read_bytes_per_launch": statistics.median(rd),
                    "dram_write_bytes_per_launch": statistics.median(wr),
                    "dram_bytes_per_launch": statistics.median([a + b for a, b in zip(rd, wr)]),
                    "duration_ns_median": statistics.median(du),
                    "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                              f"--clock-control none -k regex:'k1_flow|k2_flow' -s 4 -c 2 python bench.py --config {cfg} "
                              f"--steps 2 --warmup 4 (cold-cache, serialised launches)"}
    path = os.path.join(ROOT, "profiles", f"{tag}_traffic.json")
    try:  # configs not captured this time keep their previous record
        prev = json.load(open(path))
    except (OSError, ValueError):
        prev = {}
    prev.update(out)
    out = prev
    json.dump(out, open(path, "w"), indent=1, sort_keys=True)
    for k, v in sorted(out.items()):
        print(k, v["kernel"], v["dram_bytes_per_launch"] / 1e6, "MB", v["duration_ns_median"] / 1e3, "us")


if __name__ == "__main__":
    main()
