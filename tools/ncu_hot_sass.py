"""Developer tool: top SASS instructions by warp-stall samples from an
.ncu-rep (ncu -i REP --page source --print-source sass), with instruction
counts -- where a kernel's time goes."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, ist, iex = (hdr.index("Address"), hdr.index("Source"),
                      hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"))
recs = []
for k, r in enumerate(rows[2:]):
    if len(r) != len(hdr):
        continue
    try:
        recs.append((int(r[ist]), k, r[isrc].strip(), int(r[iex])))
    except ValueError:
        pass
tot = sum(x[0] for x in recs)
print(f"total samples {tot}")
for s, k, src, ex in sorted(recs, reverse=True)[:top]:
    print(f"{100.0 * s / tot:6.2f}%  #{k:5d}  exec {ex:>11d}  {src}")
