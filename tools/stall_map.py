"""Per-function stall-reason map of the lockstep kernel from an ncu source-page
SASS CSV (--page source --csv --print-source sass) joined with nvdisasm -g line
info. Usage: stall_map.py <sass.csv> <nvdisasm_g.sass> [reason ...]"""
import collections, csv, re, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
col = {k: i for i, k in enumerate(h)}
want = sys.argv[3:] or ["stall_wait", "stall_no_inst", "stall_selected", "stall_short_sb", "stall_branch_resolving", "stall_long_sb"]
line_of = {}
cur = None
for ln in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (Path(m.group(1)).name, int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
spans = collections.defaultdict(list)
src_dir = Path(__file__).resolve().parents[1] / "paper_2509_23384_b200" / "csrc" / "device"
for f in src_dir.glob("*.cu*"):
    for i, l in enumerate(f.read_text().splitlines(), 1):
        m = re.match(r"^(?:static |template.*)?\s*__device__[^(]*?(\w+)\(", l) or \
            re.match(r"^extern \"C\" __global__[^(]*?(\w+)\(", l)
        if m:
            spans[f.name].append((i, m.group(1)))
def func_of(fl):
    if fl is None:
        return "?"
    f, l = fl
    best = f"{f}:?"
    for start, name in spans.get(f, []):
        if start <= l:
            best = f"{f}:{name}"
    return best
base = None
agg = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try:
        a = int(r[0], 16)
    except ValueError:
        continue
    base = a if base is None else base
    fn = func_of(line_of.get(a - base))
    agg[fn]["exec"] += int(r[col["Instructions Executed"]] or 0)
    agg[fn]["bytes"] += 16
    for k in want:
        agg[fn][k] += int(r[col[k]] or 0)
tot = collections.Counter()
for v in agg.values():
    tot.update(v)
act = sum(tot[k] for k in want)
print(f"{'function':48s} {'act%':>6s} " + " ".join(f"{k[6:14]:>8s}" for k in want) + "   exec%  codeKB")
for fn, v in sorted(agg.items(), key=lambda kv: -sum(kv[1][k] for k in want))[:40]:
    a = sum(v[k] for k in want)
    print(f"{fn[:48]:48s} {100*a/act:6.2f} " + " ".join(f"{100*v[k]/act:8.2f}" for k in want) +
          f"  {100*v['exec']/tot['exec']:6.2f} {v['bytes']/1024:7.1f}")
