"""Summarize the ncu captures of tools/ncu_round.sh into profiles/ (tracked)."""
import csv
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.environ.get("OUT_DIR", "profiles")

# ---- launch list (cold-cache, serialised): shares per kernel family for the second (steady) step
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
launches = [(int(r[ii]), r[ki], float(r[vi])) for r in rows[hdr + 1:] if len(r) > vi]
half = len(launches) // 2
step = launches[half:]  # second iteration of the 3-shape step
fam = {}
for _, name, ns in step:
    key = name.split("(")[0].replace("void ", "")
    key = ("k_gemm_mxf4" if "k_gemm" in key else "k_tcq_dual" if "k_tcq_dual" in key else
           "k_tcq_xq" if "k_tcq_xq" in key else
           "k_quant" if "k_quant" in key else "k_signs" if "k_signs" in key else
           "k_zero_tiles" if "k_zero_tiles" in key else "torch/other")
    fam[key] = fam.get(key, 0.0) + ns
total = sum(fam.values())
with open(f"{out_dir}/{tag}_launch_shares.json", "w") as f:
    json.dump({"source": f"ncu --metrics gpu__time_duration.sum --clock-control none, tools/prof_step.py "
                         f"--all-shapes (one bench step, second iteration)",
               "total_us": round(total / 1e3, 1),
               "by_family_us": {k: round(v / 1e3, 1) for k, v in sorted(fam.items(), key=lambda x: -x[1])},
               "by_family_share": {k: round(v / total, 4) for k, v in fam.items()},
               "launches": [{"name": n[:90], "us": round(t / 1e3, 2)} for _, n, t in step]}, f, indent=1)

# ---- full capture: per-kernel key metrics
import os

rep_dir = os.environ.get("REP_DIR", "gpurun_out")
raw = subprocess.run(["ncu", "-i", f"{rep_dir}/full_{tag}.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
H = rr[0]
want = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
}
units = rr[1]
kern = []
for r in rr[2:]:
    d = {"kernel": r[H.index("Kernel Name")][:80]}
    for k, v in want.items():
        if k in H:
            i = H.index(k)
            val = r[i].replace(",", "")
            try:
                x = float(val)
            except ValueError:
                continue
            u = units[i]
            if u in ("Mbyte", "MB"):
                x *= 1e6
            elif u in ("Gbyte", "GB"):
                x *= 1e9
            elif u in ("Kbyte", "KB"):
                x *= 1e3
            elif u == "nsecond":
                x /= 1e3
            elif u == "usecond":
                pass
            elif u == "msecond":
                x *= 1e3
            d[v] = round(x, 3)
    kern.append(d)
gemms = [k for k in kern if "gemm" in k["kernel"]]
traffic = sum(k.get("dram_read", 0) + k.get("dram_write", 0) for k in gemms) / max(1, len(gemms))
with open(f"{out_dir}/{tag}_ncu_full_summary.json", "w") as f:
    json.dump({"source": "ncu --set full --clock-control none -k regex:k_gemm|k_quant|k_tcq -s 18 -c 18 "
                         "tools/prof_step.py --all-shapes (one full bench step)", "kernels": kern}, f, indent=1)
with open(f"{out_dir}/ncu_traffic.json", "w") as f:
    json.dump({"gemm_dram_bytes_per_launch": round(traffic), "launches": len(gemms),
               "source": f"profiles/{tag}_ncu_full_summary.json (avg dram read+write over the step's GEMMs)"}, f,
              indent=1)
print(json.dumps({k: round(v / 1e3, 1) for k, v in fam.items()}), round(total / 1e3, 1))
for k in kern:
    print(k)
