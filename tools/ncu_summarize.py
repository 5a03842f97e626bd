"""Summarise a gpurun ncu capture into profiles/: the per-kernel launch list of one bench
step (ncu --metrics gpu__time_duration.sum) and the key --set full metrics of the hot kernels.

    python tools/ncu_summarize.py TAG [OUT.json]
reads gpurun_out/TAG_launches.csv and gpurun_out/TAG_prof.ncu-rep.
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1]
out_path = sys.argv[2] if len(sys.argv) > 2 else f"profiles/ncu_summary_{tag}.json"

# ---- launch list (cold-cache, serialised: use the SHARE of the step, not absolute times)
agg = defaultdict(list)
try:  # the launch list is optional (a full capture of selected kernels alone has none)
    rows = list(csv.reader(open(f"gpurun_out/{tag}_launches.csv")))
except OSError:
    rows = []
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r]
if hi:
    hi = hi[0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            unit = r[ui]
            us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
            name = r[ki].split("(")[0].replace("void ", "")
            agg[name].append(us)
total = sum(sum(v) for v in agg.values()) or 1.0
launches = [{"kernel": k, "launches": len(v), "total_us": round(sum(v), 1), "avg_us": round(sum(v) / len(v), 1),
             "share": round(sum(v) / total, 4)} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]

# ---- full-set metrics of the captured kernels
raw = subprocess.run(["ncu", "-i", f"gpurun_out/{tag}_prof.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
kernels = {}
if rr:
    hdr = rr[0]
    want = {
        "duration_us": ("gpu__time_duration.sum", 1e3),
        "dram_read_MB": ("dram__bytes_read.sum", 1.0),
        "dram_write_MB": ("dram__bytes_write.sum", 1.0),
        "dmma_pipe_active_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
        "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
        "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
        "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
        "registers": ("launch__registers_per_thread", 1.0),
        "smem_per_block_KB": ("launch__shared_mem_per_block_dynamic", 1.0),
        "grid": ("launch__grid_size", 1.0),
        "block": ("launch__block_size", 1.0),
    }
    units = rr[1]
    for row in rr[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        ent = {}
        for key, (metric, scale) in want.items():
            if metric in d:
                try:
                    v = float(d[metric].replace(",", ""))
                except ValueError:
                    continue
                un = u.get(metric, "")
                if metric.startswith("dram__bytes"):
                    v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(un, 1.0)
                elif metric == "gpu__time_duration.sum":
                    v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(un, 1.0)
                    scale = 1.0
                elif metric == "launch__shared_mem_per_block_dynamic":
                    v = v * {"byte": 1.0 / 1024, "Kbyte": 1.0}.get(un, 1.0)
                ent[key] = round(v * scale, 3)
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        ent["top_stalls_pct"] = {k: round(100 * s / tot, 1) for s, k in sorted(stalls, reverse=True)[:5]}
        if "dram_read_MB" in ent and "dram_write_MB" in ent and ent["dram_read_MB"] == ent["dram_read_MB"] \
                and ent["dram_write_MB"] == ent["dram_write_MB"]:  # (not NaN)
            ent["dram_bytes_per_launch"] = int(round((ent["dram_read_MB"] + ent["dram_write_MB"]) * 1e6))
        kernels.setdefault(name, ent)

json.dump({"source": f"gpurun_out/{tag}_prof.ncu-rep (ncu --set full --clock-control none) and "
                     f"gpurun_out/{tag}_launches.csv (ncu --metrics gpu__time_duration.sum --clock-control none)",
           "launch_list_total_us": round(total, 1), "launch_list": launches, "kernels": kernels},
          open(out_path, "w"), indent=1)
print(open(out_path).read())
