"""Write profiles/traffic.json (read by bench.py for roofline.traffic) from an `ncu --set
full` capture of scripts/profile_step.py (one grouped launch = one bench step):
  python scripts/make_traffic.py gpurun_out/r02_v1_step.ncu-rep profiles/r02_v1_step_details.csv [srchash file]
The source hash of the captured build is taken from the capture's <tag>_srchash.txt
(written on the GPU box by scripts/round_capture.sh) when given, else from this tree."""
import csv, io, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

rep, details = sys.argv[1], sys.argv[2]
metrics = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct," \
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
col = {h: i for i, h in enumerate(hdr)}


def val(r, m):
    return float(r[col[m]]) * scale.get(units[col[m]], 1)


launches = [{"kernel": r[col["Kernel Name"]], "grid": r[col["Grid Size"]],
             "us": round(val(r, "gpu__time_duration.sum"), 3),
             "dram_bytes": int(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")),
             "dram_pct": float(r[col["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]]),
             "l2_hit_pct": float(r[col["lts__t_sector_hit_rate.pct"]])} for r in data]
out = {"source": f"ncu --set full --clock-control none, {details} ({len(launches)} launches = one bench step)",
       "kernel": launches[0]["kernel"] if launches else None,
       "dram_bytes_per_step": sum(l["dram_bytes"] for l in launches),
       "ncu_kernel_us_per_step": round(sum(l["us"] for l in launches), 3),
       "workload": "resnet50-grad-set 8 virtual ranks dims 2x4 avg, grouped",
       "source_hash": (open(sys.argv[3]).read().strip() if len(sys.argv) > 3 else __import__("bench").source_hash()),
       "launches": launches}
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out["dram_bytes_per_step"], out["ncu_kernel_us_per_step"])
