"""Summarise an ncu --csv launch list (developer tool): per-launch rows over a
threshold and per-kernel totals."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
min_id = int(sys.argv[2]) if len(sys.argv) > 2 else 0
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 100.0
hdr, recs = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        recs.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = {}
for (i, k), m in sorted(recs.items()):
    if i < min_id:
        continue
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    name = k.split("(")[0].replace("bfb::<unnamed>::", "").replace("void ", "")
    if t > thr:
        print(f"{i:>5} {name:34s} {t:10.1f} us  rd {m.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB"
              f"  wr {m.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")
    tot[name] = tot.get(name, 0) + t
print("--- totals (us)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:12.1f}  {k}")
