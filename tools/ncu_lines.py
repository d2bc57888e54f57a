"""Aggregate an ncu `--page source --print-source cuda,sass --csv` dump by CUDA source line."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = "?"; hdr = None; agg = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[2] != "-":   # sass line rows repeat: only take cuda line rows (Address == '-')
        continue
    try:
        s = float(r[4] or 0); i = float(r[7] or 0)
    except ValueError:
        continue
    agg[(cur_file, r[0])] = (s, i, r[1][:100])
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot:.0f}, warp instructions {toti:.3e}")
byfile = defaultdict(lambda: [0, 0])
for (f, l), v in agg.items():
    byfile[f][0] += v[0]; byfile[f][1] += v[1]
for f, v in sorted(byfile.items(), key=lambda x: -x[1][0]):
    print(f"  {f:24s} samples {100*v[0]/tot:5.1f}%  instr {100*v[1]/toti:5.1f}%")
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*v[0]/tot:5.1f}% {100*v[1]/toti:5.1f}%  {f}:{l}: {v[2]}")
