"""Summarise ncu captures for profiles/: key metrics + stall reasons of a --set full
report, and per-kernel shares of a --metrics gpu__time_duration.sum launch list.

python tools/ncu_summary.py report <file.ncu-rep> [--json out.json]
python tools/ncu_summary.py launches <file.csv>"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3}


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        stalls = {}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                d[h] = f"{v} {u}".strip()
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    if float(v) > 0:
                        stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v))
                except ValueError:
                    pass
        rb = [float(v) * SCALE.get(u, 1) for h, u, v in zip(hdr, units, vals) if h == "dram__bytes_read.sum"]
        wb = [float(v) * SCALE.get(u, 1) for h, u, v in zip(hdr, units, vals) if h == "dram__bytes_write.sum"]
        d["dram_bytes_total"] = (rb[0] if rb else 0) + (wb[0] if wb else 0)
        tot = sum(stalls.values()) or 1
        d["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1e-9)
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "total_ms": round(v[1] * 1e3, 4), "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    res = report(path) if kind == "report" else launches(path)
    txt = json.dumps(res, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt + "\n")
    print(txt)
