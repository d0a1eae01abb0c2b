"""Turn a profile_round.sh output (gpurun_out/prof) into committed summaries
under profiles/ (round tag as argv[1])."""
import csv, io, json, os, shutil, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = "gpurun_out/prof"
os.makedirs("profiles", exist_ok=True)
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TU = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
traffic = {}
for c in ["C1", "C2", "C3", "C4", "C5"]:
    p = f"{src}/traffic_{c}.csv"
    if not os.path.exists(p):
        continue
    lines = [l for l in open(p).read().splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    m = {r[rows[0].index("Metric Name")]: (float(r[rows[0].index("Metric Value")].replace(",", "")),
                                           r[rows[0].index("Metric Unit")]) for r in rows[1:]}
    rd = m["dram__bytes_read.sum"][0] * UNIT[m["dram__bytes_read.sum"][1]]
    wr = m["dram__bytes_write.sum"][0] * UNIT[m["dram__bytes_write.sum"][1]]
    t = m["gpu__time_duration.sum"]
    b = json.load(open(f"{src}/bench_{c}.json"))
    alg = b["roofline"]["algorithmic_bytes_per_launch"]
    traffic[c] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                  "ncu_duration_s": t[0] * TU.get(t[1], 1e-9), "algorithmic_bytes_per_launch": alg,
                  "traffic_over_algorithmic": round((rd + wr) / alg, 3),
                  "dram_gbs_under_ncu": round((rd + wr) / (t[0] * TU.get(t[1], 1e-9)) / 1e9, 1),
                  "lts_tex_read_sectors": m["lts__t_sectors_srcunit_tex_op_read.sum"][0],
                  "lts_tex_write_sectors": m["lts__t_sectors_srcunit_tex_op_write.sum"][0],
                  "warps_active_pct": m["sm__warps_active.avg.pct_of_peak_sustained_active"][0]}
    shutil.copy(f"{src}/bench_{c}.json", f"profiles/{tag}_bench_{c}.json")
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
for f in os.listdir(src):
    if f.startswith("bench_amr_") and f.endswith(".json"):
        shutil.copy(f"{src}/{f}", f"profiles/{tag}_{f}")
    if f in ("traffic_interp.csv", "traffic_avgdown.csv", "traffic_advance.csv"):
        name = {"traffic_interp.csv": "interp", "traffic_avgdown.csv": "avgdown", "traffic_advance.csv": "advance"}[f]
        shutil.copy(f"{src}/{f}", f"profiles/{tag}_ncu_{name}_kernel.csv")
    if (f.startswith("seam_probe_") or f.startswith("pcie_probe")) and f.endswith(".txt"):
        shutil.copy(f"{src}/{f}", f"profiles/{tag}_{f}")
    if f.startswith("launches_") and f.endswith(".csv"):
        shutil.copy(f"{src}/{f}", f"profiles/{tag}_{f}")
    if f.startswith("bench_ref_") and f.endswith(".json"):
        shutil.copy(f"{src}/{f}", f"profiles/{tag}_{f.replace('bench_ref', 'bench_reference')}")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for c in ["C2", "C3", "C4", "C5", "advance"]:
    rep = f"{src}/full_{c}.ncu-rep"
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    with open(f"profiles/{tag}_ncu_full_{c}_raw.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit", "value"])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                w.writerow([k, u[i], v[i]])
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hh = rows[0]
    with open(f"profiles/{tag}_ncu_full_{c}_details.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["section", "metric", "unit", "value"])
        for row in rows[1:]:
            d = dict(zip(hh, row))
            w.writerow([d.get("Section Name", ""), d.get("Metric Name", ""), d.get("Metric Unit", ""),
                        d.get("Metric Value", "")])
for c, t in traffic.items():
    b = json.load(open(f"profiles/{tag}_bench_{c}.json"))
    print(c, b["ms_per_step"], b["value"], b["roofline"]["frac"], round(t["dram_bytes_per_launch"] / 1e9, 3),
          t["traffic_over_algorithmic"], b["e2e"]["value"], (b.get("cpu_baseline") or {}).get("value"),
          b["clocks"])
