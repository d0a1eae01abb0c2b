"""Per-process, per-launch summary of an `ncu --csv --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` log:
    python scripts/parse_ncu_launches.py LOG [last_k]"""
import collections
import csv
import io
import sys


def launches(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    if not rows:
        return {}
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    d = collections.defaultdict(dict)
    for r in rows[1:]:
        key = (r[ix["Process ID"]], int(r[ix["ID"]]))
        d[key][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    per = collections.defaultdict(list)
    for (pid, i), m in sorted(d.items()):
        per[pid].append((m["gpu__time_duration.sum"] / 1e3, (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / 1e6))
    return per


if __name__ == "__main__":
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for pid, lst in launches(sys.argv[1]).items():
        print(pid, [f"{t:.1f}us/{b:.0f}MB" for t, b in lst[-k:]])
