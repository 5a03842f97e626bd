"""Summarise an ncu --page source (sass) CSV: top instructions by excessive shared wavefronts and by stall samples."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}


def num(r, k):
    try:
        return float(r[ix[k]])
    except ValueError:
        return 0.0


tot_ex = sum(num(r, "L1 Wavefronts Shared Excessive") for r in data)
print("total excessive shared wavefronts", tot_ex)
for r in sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:12]:
    print(f"{num(r, 'L1 Wavefronts Shared Excessive'):12.0f} {num(r, 'L1 Wavefronts Shared'):12.0f} {r[ix['Address']][-5:]} {r[ix['Source']].strip()}")
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
print("total stall samples", tot)
stall_cols = [h for h in hdr if h.startswith("stall_")]
agg = {h: sum(num(r, h) for r in data) for h in stall_cols}
for h, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {h:32s} {v / tot * 100:5.1f}%")
for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:15]:
    print(f"{num(r, 'Warp Stall Sampling (All Samples)'):8.0f} {r[ix['Address']][-5:]} {r[ix['Source']].strip()}")
