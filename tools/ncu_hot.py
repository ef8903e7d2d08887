"""Summarise an ncu source page (cuda,sass CSV) into per-source-line stall samples.

    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_hot.py x.csv [top]
"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = collections.OrderedDict()
cur_file = ""
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[2] == "-":  # source line row with aggregated metrics
        key = (cur_file, int(r[0]))
        s = float(r[4] or 0)
        ex = float(r[7] or 0)
        agg[key] = (s, ex, r[1].strip()[:90])
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (s, ex, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{s/tot*100:5.1f}% {int(s):7d} inst={int(ex):9d} {f}:{ln:<4d} {src}")
