"""Summarise gpurun_out/ test logs and bench lines (run here after a gpurun call)."""
import glob, json, os, sys
root = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for f in ("gpu_tests.log", "quick_tests.log", "smoke.log"):
    p = os.path.join(root, f)
    if os.path.exists(p):
        lines = open(p).read().strip().splitlines()
        fails = [l for l in lines if l.startswith("FAILED") or "Error" in l[:40]]
        print(f, "|", " / ".join(lines[-2:]), "|", *fails[:5])
for p in sorted(glob.glob(os.path.join(root, "bench_*.log")) + glob.glob(os.path.join(root, "bench_*.json"))):
    for l in open(p):
        if l.startswith("{"):
            d = json.loads(l)
            if "roofline" not in d:
                print(os.path.basename(p), l.strip()[:300])
                continue
            r = d["roofline"]
            e = d.get("e2e") or {}
            print(os.path.splitext(os.path.basename(p))[0][6:], "ms/step %.3f" % d["ms_per_step"], "paths/s %.4g" % d["value"],
                  {k: round(v, 3) for k, v in d["phase_ms"].items()},
                  r["bound"], "%.1f %s frac %.3f" % (r["achieved"], r["unit"], r["frac"]),
                  "e2e_ms", e.get("ms_per_step"), "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
