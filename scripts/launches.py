"""Per-launch table from an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])."""
import csv, sys
SC = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}
f = sys.argv[1]
lines = [l for l in open(f) if l.startswith('"')]
by = {}
for r in csv.DictReader(lines):
    by.setdefault(int(r["ID"]), {})[r["Metric Name"]] = r
tot = 0
for k in sorted(by):
    v = by[k]
    t = float(v["gpu__time_duration.sum"]["Metric Value"]) * SC[v["gpu__time_duration.sum"]["Metric Unit"]]
    tot += t
    extra = ""
    if "dram__bytes_read.sum" in v:
        rd = float(v["dram__bytes_read.sum"]["Metric Value"]) * SC[v["dram__bytes_read.sum"]["Metric Unit"]]
        wr = float(v["dram__bytes_write.sum"]["Metric Value"]) * SC[v["dram__bytes_write.sum"]["Metric Unit"]]
        extra = "R %7.1f MB W %7.1f MB %5.2f TB/s" % (rd / 1e6, wr / 1e6, (rd + wr) / t / 1e12)
    r = v["gpu__time_duration.sum"]
    print("%3d %-45s %-14s %-12s s%-3s %9.1f us %s" % (k, r["Kernel Name"][:45], r["Grid Size"], r["Block Size"],
                                                     r["Stream"], t * 1e6, extra))
print("total %.1f us" % (tot * 1e6))
