"""Turn scripts/profile_r02.sh output (gpurun_out/prof2) into committed
summaries under profiles/ (round tag r02): bench lines, the reference arm,
the ncu launch list of the default bench command, ncu --set full of the top
kernel (raw + details), the per-direction DRAM metrics, the per-config DRAM
traffic bench.py reads (profiles/ncu_traffic.json) and the sanitizer log."""
import csv
import io
import json
import os
import shutil
import subprocess

SRC, TAG = "gpurun_out/prof2", "r02"
os.makedirs("profiles", exist_ok=True)


def metrics(path):
    """{metric: value} of the one profiled launch in an ncu --csv log."""
    lines = [l for l in open(path).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    out = {}
    for r in rows[1:]:
        v = r[h.index("Metric Value")].replace(",", "")
        try:
            out[r[h.index("Metric Name")]] = float(v)
        except ValueError:
            out[r[h.index("Metric Name")]] = v
    return out


def bench(path):
    for line in open(path).read().splitlines():
        if line.startswith("{"):
            return json.loads(line)
    return None


split, traffic = {}, {}
for c in ["C3", "C2", "C4", "C5", "C1"]:
    for g in ["all", "x", "yz"]:
        p = f"{SRC}/split_{c}_{g}.csv"
        if not os.path.exists(p):
            continue
        m = metrics(p)
        b = bench(p)
        alg = b["roofline"]["algorithmic_bytes_per_launch"]
        t = m["gpu__time_duration.sum"] * 1e-9
        rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
        e = {"ncu_duration_us": round(t * 1e6, 2), "dram_read": rd, "dram_write": wr,
             "dram_bytes": rd + wr, "algorithmic_bytes": alg, "traffic_over_algorithmic": round((rd + wr) / alg, 3),
             "dram_gbs_under_ncu": round((rd + wr) / t / 1e9, 1),
             "dram_cycles_active_pct": m["dram__cycles_active.avg.pct_of_peak_sustained_elapsed"],
             "lts_sectors_op_read": m["lts__t_sectors_op_read.sum"], "lts_sectors_op_write": m["lts__t_sectors_op_write.sum"],
             "achieved_occupancy_pct": m["sm__warps_active.avg.pct_of_peak_sustained_active"],
             "theoretical_occupancy_pct": m["sm__maximum_warps_per_active_cycle_pct"],
             "ngrow": b["config"]["nghost"], "tags": b["config"]["tags_this_rank"]}
        split.setdefault(c, {})[g] = e
        if g == "all":
            traffic[c] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_duration_s": t,
                          "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": round((rd + wr) / alg, 3),
                          "dram_gbs_under_ncu": round((rd + wr) / t / 1e9, 1),
                          "lts_op_read_sectors": m["lts__t_sectors_op_read.sum"],
                          "lts_op_write_sectors": m["lts__t_sectors_op_write.sum"],
                          "warps_active_pct": m["sm__warps_active.avg.pct_of_peak_sustained_active"],
                          "source": f"profiles/{TAG}_ncu_split.json (ncu --metrics, one ghx_copy_kernel launch, "
                                    "--clock-control none)"}
json.dump(split, open(f"profiles/{TAG}_ncu_split.json", "w"), indent=1)
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)

for f in os.listdir(SRC):
    if f.startswith("bench_") and f.endswith(".json"):
        shutil.copy(f"{SRC}/{f}", f"profiles/{TAG}_{f}")
    if f.startswith("launches_") and f.endswith(".csv"):
        shutil.copy(f"{SRC}/{f}", f"profiles/{TAG}_{f}")
if os.path.exists(f"{SRC}/sanitizer.txt"):
    shutil.copy(f"{SRC}/sanitizer.txt", f"profiles/{TAG}_sanitizer.txt")
for f in ("pcie_seam_probe.txt", "pcie_ring_probe.txt"):
    if os.path.exists(f"gpurun_out/{f}"):
        shutil.copy(f"gpurun_out/{f}", f"profiles/{TAG}_{f}")

for c in ["C3", "C2"]:
    rep = f"{SRC}/full_{c}.ncu-rep"
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    with open(f"profiles/{TAG}_ncu_full_{c}_raw.csv", "w") as fo:
        w = csv.writer(fo)
        w.writerow(["metric", "unit", "value"])
        for k, uu, vv in zip(h, u, v):
            if any(s in k for s in ("dram__", "lts__t_sectors", "lts__t_sector_hit", "sm__warps_active",
                                    "launch__", "gpu__time_duration", "sm__throughput", "l1tex__t_sectors_pipe_lsu",
                                    "smsp__average_warps_issue_stalled", "sm__maximum_warps")):
                w.writerow([k, uu, vv])
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(f"profiles/{TAG}_ncu_full_{c}_details.csv", "w").write(det)
print(json.dumps({c: {g: (e["ncu_duration_us"], e["traffic_over_algorithmic"], e["dram_gbs_under_ncu"],
                          e["dram_cycles_active_pct"]) for g, e in v.items()} for c, v in split.items()}, indent=1))
