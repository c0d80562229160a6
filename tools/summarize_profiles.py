"""Turns a gpurun_out profiling directory (tools/gpu_profile.sh) into the
committed summaries under profiles/:
  <tag>_launches_summary.txt  every launch of `bench.py --steps 1 --warmup 1 --no-extra`
                              (gpu__time_duration + DRAM bytes, cold-cache,
                              serialised: shares, not absolutes)
  <tag>_ncu_full_summary.txt  --set full metrics of the top kernels
  traffic.json                per-kernel DRAM bytes per launch (bench.py
                              reads it for roofline.traffic)
usage: python tools/summarize_profiles.py gpurun_out/r1g r1 [pcg_iterations_of_captured_launch]"""
import collections, csv, io, json, os, subprocess, sys

src, tag = sys.argv[1], sys.argv[2]
pcg_its = int(sys.argv[3]) if len(sys.argv) > 3 else None
os.makedirs("profiles", exist_ok=True)


def short(name):
    import re
    base = name.split("(")[0]
    m = re.search(r"(k_\w+(<[^>]*>)?)\s*$", base)
    return m.group(1) if m else base.replace("void ", "")


rows = [r for r in csv.reader(open(os.path.join(src, "launches.csv"))) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[idi]] = short(r[ki])
    except ValueError:
        pass
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
with open(f"profiles/{tag}_launches_summary.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            "--clock-control none\n# command: python bench.py --steps 1 --warmup 1 --no-cpu-baseline "
            "--no-e2e --no-extra  (config 3, 1 B200): setup + 3 whole LM solves\n# per-launch times are "
            "cold-cache and serialised: compare shares, not absolutes\n")
    f.write(f"# total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches\n")
    f.write(f"{'launches':>8} {'total_us':>10} {'share':>6} {'DRAM_MB':>9}  kernel\n")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{v[0]:8d} {v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[2] / 1e6:9.1f}  {k}\n")

raw = subprocess.run(["ncu", "-i", os.path.join(src, "full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
traffic = {}
with open(f"profiles/{tag}_ncu_full_summary.txt", "w") as f:
    f.write(f"# ncu --set full --clock-control none, config 3, LM iteration 4 kernels (+ LM 5 head)\n"
            f"# source: {src}/full.ncu-rep\n")
    for r in rr[2:]:
        name = short(r[h.index("Kernel Name")])
        vals = {w: r[h.index(w)] for w in want if w in h}
        f.write(name + "\n")
        for w, v in vals.items():
            f.write(f"    {w:62s} {v} {units[h.index(w)]}\n")
        if name not in traffic:
            mb = float(vals["dram__bytes_read.sum"]) + float(vals["dram__bytes_write.sum"])
            scale = 1e6 if units[h.index("dram__bytes_read.sum")].lower().startswith("mbyte") else 1.0
            traffic[name] = {"dram_bytes_per_launch": mb * scale,
                             "duration_ms": float(vals["gpu__time_duration.sum"]) *
                             (1.0 if units[h.index("gpu__time_duration.sum")] == "ms" else 1e-3)}
if pcg_its and "k_pcg3" in traffic:
    traffic["k_pcg3"]["pcg_iterations"] = pcg_its
    traffic["k_pcg3"]["dram_bytes_per_pcg_iteration"] = traffic["k_pcg3"]["dram_bytes_per_launch"] / pcg_its
json.dump({"source": f"{src}/full.ncu-rep (ncu --set full, config 3, LM iteration 4)",
           "kernels": traffic}, open("profiles/traffic.json", "w"), indent=1)
print(open(f"profiles/{tag}_launches_summary.txt").read()[:2500])
print(json.dumps(traffic, indent=1)[:1500])
