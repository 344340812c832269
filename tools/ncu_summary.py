"""Summarise an ncu --set full report (raw page) for the pseudo-flow kernel into profiles/.
usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep out.json [algorithmic_bytes_per_launch] [workload] [tile_x tile_y zchunk] [--traffic]"""
import csv
import io
import json
import subprocess
import sys

argv = [a for a in sys.argv if a != "--traffic"]
rep, out = argv[1], argv[2]
alg = float(argv[3]) if len(argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__warps_launched.sum", "sm__cycles_elapsed.avg.per_second"]
res = []
for r in data:
    d = {}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            d[w] = r[i] + (f" {units[i]}" if units[i] else "")
    # stall reasons
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                if float(r[i]) > 0:
                    d.setdefault("stalls", {})[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
            except ValueError:
                pass
    res.append(d)
summary = {"report": rep, "kernels": res}
if alg and res:
    def nbytes(s):
        v, u = s.split()[0].replace(",", ""), s.split()[1] if len(s.split()) > 1 else "byte"
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        return float(v) * mul
    k = res[-1]
    rb = nbytes(k["dram__bytes_read.sum"])
    wb = nbytes(k["dram__bytes_write.sum"])
    summary["dram_bytes_per_launch"] = rb + wb
    summary["algorithmic_bytes_per_launch"] = alg
    summary["traffic_over_algorithmic"] = (rb + wb) / alg
if len(argv) > 4:
    summary["workload"] = argv[4]
if len(argv) > 5:
    summary["kernel_config"] = [int(v) for v in argv[5:8]]
# the source state this capture measured (bench.py reports the traffic only for the same sources)
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from bench import source_hash  # noqa: E402
summary["src_hash"] = source_hash()
json.dump(summary, open(out, "w"), indent=1)
if "--traffic" in sys.argv and alg and res:
    # merge into profiles/ncu_traffic.json (one entry per workload + kernel)
    import os
    tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    ents = [e for e in tj.get("entries", []) if not (e.get("workload") == summary.get("workload") and
                                                      e.get("kernel") == res[-1].get("Kernel Name"))]
    ents.append({"workload": summary.get("workload"), "kernel": res[-1].get("Kernel Name"),
                 "src_hash": summary["src_hash"], "dram_bytes_per_launch": summary["dram_bytes_per_launch"],
                 "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": summary["traffic_over_algorithmic"],
                 "gpu__time_duration": res[-1].get("gpu__time_duration.sum"), "report": rep})
    json.dump({"note": "ncu --set full, one launch each (tools/ncu_summary.py --traffic); bench.py uses an entry only "
                       "when its src_hash matches the current sources", "entries": ents}, open(tp, "w"), indent=1)
print(json.dumps(summary, indent=1)[:4000])
