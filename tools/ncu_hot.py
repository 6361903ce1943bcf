"""Developer tool: the hottest SASS lines (warp-stall samples) of one kernel
in an .ncu-rep, with the CUDA source line each maps to."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
sass = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                      capture_output=True, text=True).stdout.splitlines()))
hdr = sass[1]
rows = [dict(zip(hdr, r)) for r in sass[2:] if len(r) == len(hdr)]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
print(f"total samples {tot}")
for r in rows[:top]:
    n = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{100 * n / max(1, tot):5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:90]}")
