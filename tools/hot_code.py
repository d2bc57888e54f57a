"""Hot-code map of the lockstep kernel: joins ncu per-instruction execution
counts (--page source --print-source sass CSV) with nvdisasm -g line info of
the same cubin, then aggregates executed instructions and code bytes by
source function. Usage: hot_code.py <ncu_sass.csv> <nvdisasm_g.sass>"""
import collections, csv, re, sys
from pathlib import Path

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, ie = h.index("Address"), h.index("Instructions Executed")
isamp = h.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ia], 16), int(r[ie]), int(r[isamp])))
    except ValueError:
        pass
base = recs[0][0]
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
# function spans per source file
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
ex = collections.Counter(); sz = collections.Counter(); st = collections.Counter()
for a, e, s in recs:
    fn = func_of(line_of.get(a - base))
    ex[fn] += e; sz[fn] += 16; st[fn] += s
tot = sum(ex.values()); tots = sum(st.values())
print(f"{'function':52s} {'exec%':>6s} {'stall%':>6s} {'code KB':>8s}")
for fn, e in ex.most_common(40):
    print(f"{fn:52s} {100*e/tot:6.2f} {100*st[fn]/tots:6.2f} {sz[fn]/1024:8.1f}")
