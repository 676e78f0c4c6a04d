"""profiles/traffic.json from ncu launch lists (dram__bytes_read.sum +
dram__bytes_write.sum per launch): bench.py's `roofline.traffic` source.

  python scripts/traffic_table.py <config> <launch_list.csv> [commit]

Per kernel name (namespace and template arguments stripped) the median DRAM
bytes per launch and the launch count; merged into profiles/traffic.json under
the config, with the capture file and the commit it was taken at.
"""
import csv
import json
import os
import re
import statistics
import subprocess
import sys

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name: str) -> str:
    n = name.split("(")[0]
    n = re.sub(r"<.*>", "", n)
    return n.replace("void ", "").strip().split("::")[-1]


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    commit = sys.argv[3] if len(sys.argv) > 3 else subprocess.run(
        ["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
    lines = [l for l in open(path) if l.startswith('"')]
    by = {}
    for r in csv.DictReader(lines):
        by.setdefault(int(r["ID"]), {})[r["Metric Name"]] = r
    per = {}
    for k in sorted(by):
        v = by[k]
        if "dram__bytes_read.sum" not in v:
            continue
        rd = float(v["dram__bytes_read.sum"]["Metric Value"]) * SC[v["dram__bytes_read.sum"]["Metric Unit"]]
        wr = float(v["dram__bytes_write.sum"]["Metric Value"]) * SC[v["dram__bytes_write.sum"]["Metric Unit"]]
        per.setdefault(short(v["dram__bytes_read.sum"]["Kernel Name"]), []).append(rd + wr)
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    table = json.load(open(out_path)) if os.path.exists(out_path) else {}
    table[cfg] = {k: {"dram_bytes_per_launch": statistics.median(v), "launches": len(v),
                      "source": os.path.relpath(path, os.path.dirname(out_path)), "commit": commit}
                  for k, v in per.items()}
    json.dump(table, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(table[cfg], indent=1))


if __name__ == "__main__":
    main()
