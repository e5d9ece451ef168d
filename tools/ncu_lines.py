"""Per-source-line instruction and stall-sample shares from an ncu source page:
ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv;
python tools/ncu_lines.py X.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None
agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if len(r) < 10 or r[0] in ('Line No', '') or r[2] != '-':
        continue
    try:
        samp, ie = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    agg[(cur, int(r[0]))] = (r[1].strip()[:100], samp, ie)
ts = sum(v[1] for v in agg.values()) or 1
ti = sum(v[2] for v in agg.values()) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][1] / ts + kv[1][2] / ti))[:top]:
    print(f"{k[0]}:{k[1]:>5}  instr {100 * v[2] / ti:5.1f}%  samples {100 * v[1] / ts:5.1f}%  {v[0]}")
