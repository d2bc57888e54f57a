"""SASS code bytes of a cubin by source function, from `nvdisasm -gi` inline
line info: each instruction is charged to the innermost frame in this
repo's sources (intrinsics such as __shfl_sync are charged to their caller).
Usage: code_size_map.py <nvdisasm_gi.sass> [top] [fn,fn,...: show their inline callers]"""
import collections, re, sys
from pathlib import Path

DEV = Path(__file__).resolve().parents[1] / "paper_2509_23384_b200" / "csrc" / "device"
pat = re.compile(r'//## File "([^"]+)", line (\d+)')
instr = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/")
fdef = re.compile(r"^(?:static\s+)?(?:template\s*<[^>]*>\s*)?(?:__device__|__global__)[^(;]*?\b(\w+)\s*\(")
src = {}


def func_of(fn, ln):
    if fn not in src:
        p = DEV / fn
        src[fn] = p.read_text().split("\n") if p.exists() else []
    lines = src[fn]
    for i in range(min(ln - 1, len(lines) - 1), -1, -1):
        m = fdef.match(lines[i])
        if m:
            return m.group(1)
    return "?"


block, in_block, frames = [], False, None
by_func, by_shfl, callers = collections.Counter(), collections.Counter(), collections.Counter()
want = set(sys.argv[3].split(",")) if len(sys.argv) > 3 else set()
total = 0
for line in open(sys.argv[1]):
    m = pat.search(line)
    if m:
        if not in_block:
            block, in_block = [], True
        block.append((m.group(1), int(m.group(2))))
        continue
    if instr.match(line):
        if in_block:
            frames, in_block = block, False
        total += 1
        if not frames:
            continue
        ours = [(f.split("/")[-1], n) for f, n in frames if "/root/repo" in f or "paper_2509" in f]
        key = (ours[0][0], func_of(*ours[0])) if ours else ("?", "?")
        by_func[key] += 1
        if key[1] in want:
            callers[(key[1],) + tuple(func_of(*o) for o in ours[1:4])] += 1
        if "sm_30_intrinsics" in frames[0][0] or "sm_80_rt" in frames[0][0]:
            by_shfl[key] += 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"{total} instructions ({16 * total / 1024:.0f} KB); warp intrinsics (shuffles, reduces) "
      f"{16 * sum(by_shfl.values()) / 1024:.0f} KB")
print(f"{'function':48s} {'code KB':>8s} {'of which intrinsics':>20s}")
for k, v in by_func.most_common(top):
    print(f"{k[0] + ':' + k[1]:48s} {16 * v / 1024:8.1f} {16 * by_shfl[k] / 1024:20.1f}")
for k, v in callers.most_common(30):
    print(f"{16 * v / 1024:7.1f} KB  " + " <- ".join(k))
