"""Per-CUDA-line stall-reason breakdown from an ncu `--page source --print-source cuda,sass --csv` dump."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = "?"; hdr = None; agg = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[2] != "-": continue
    try: samp = float(r[4] or 0)
    except ValueError: continue
    st = {}
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try: st[name[6:]] = float(r[k] or 0)
            except ValueError: pass
    agg[(cur, r[0])] = (samp, st, r[1][:80])
tot = sum(v[0] for v in agg.values()) or 1
glob = {}
for v in agg.values():
    for k, x in v[1].items(): glob[k] = glob.get(k, 0) + x
gt = sum(glob.values()) or 1
print("kernel-wide:", ", ".join(f"{k} {100*x/gt:.0f}%" for k, x in sorted(glob.items(), key=lambda z: -z[1])[:8]))
for (f, l), v in sorted(agg.items(), key=lambda z: -z[1][0])[:top]:
    st = sorted(v[1].items(), key=lambda z: -z[1])[:3]
    ss = sum(v[1].values()) or 1
    print(f"{100*v[0]/tot:5.1f}% {f}:{l:5s} [{', '.join(f'{k} {100*x/ss:.0f}%' for k, x in st)}] {v[2]}")
