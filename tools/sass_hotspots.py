"""Dev: join an ncu source page (SASS, --page source --csv --print-source sass)
with nvdisasm -gi line info: stall samples and instructions executed per
source function / line.
    python tools/sass_hotspots.py <engine.sass> <kernel mangled name> <sass.csv>"""
import csv
import re
import sys
from collections import defaultdict

sass_path, kname, csv_path = sys.argv[1:4]
lines = open(sass_path).read().split("\n")
# all text sections: kernel + noinline callees (ncu lists them in one address space)
loc = {}     # (section, offset) -> innermost (file, line)
order = []   # sections in file order with their instruction offsets
sec = None
cur = None
first_of_group = True
for ln in lines:
    m = re.match(r"\s*\.section\s+\.text\.([^,\s]+)", ln)
    if m:
        sec = m.group(1)
        order.append([sec, []])
        continue
    m = re.match(r"\s*//## File \"(.+?)\", line (\d+)", ln)
    if m:
        if first_of_group:
            cur = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
            first_of_group = False
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and sec:
        off = int(m.group(1), 16)
        loc[(sec, off)] = cur
        order[-1][1].append(off)
        first_of_group = True
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ia, isamp, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
data = rows[2:]
base = int(data[0][ia], 16)
ksec = next(i for i, (s, _) in enumerate(order) if s == kname)
# csv addresses are contiguous per function; map by walking sections from the kernel
by_line = defaultdict(lambda: [0, 0, 0])
tot_s = tot_e = 0
# assume csv rows are kernel instructions first (offset = addr - base)
kern_offs = set(order[ksec][1])
miss = 0
for r in data:
    off = int(r[ia], 16) - base
    s, e = int(r[isamp] or 0), int(r[iex] or 0)
    tot_s += s
    tot_e += e
    L = loc.get((kname, off))
    if L is None:
        miss += 1
        L = ("?", 0)
    a = by_line[L]
    a[0] += s
    a[1] += e
    a[2] += 1
print(f"rows {len(data)} kernel instrs {len(kern_offs)} unmapped {miss} samples {tot_s} executed {tot_e}")
src = {}
def text(f, n):
    if f not in src:
        try:
            src[f] = open(f"/root/repo/paper_2601_22705_b200/csrc/{f}").read().split("\n")
        except OSError:
            src[f] = []
    t = src[f]
    return t[n - 1].strip()[:70] if 0 < n <= len(t) else ""
top = sorted(by_line.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 60]
for (f, n), (s, e, k) in top:
    print(f"{100*s/tot_s:5.1f}% {100*e/max(tot_e,1):5.1f}%ex {k:4d}i {f}:{n} {text(f, n)}")

# per enclosing function (by definition line ranges in each file)
import bisect
fdefs = {}
for f in {k[0] for k in by_line}:
    t = src.get(f) or (text(f, 1) and src[f]) or []
    starts = []
    for i, l in enumerate(t, 1):
        m = re.match(r"^(?:template.*)?(?:__device__|__global__|static __device__).*?(\w+)\(", l)
        if m:
            starts.append((i, m.group(1)))
    fdefs[f] = starts
agg = defaultdict(lambda: [0, 0, 0])
for (f, n), (s, e, k) in by_line.items():
    st = fdefs.get(f, [])
    j = bisect.bisect_right([a for a, _ in st], n) - 1
    name = f + ":" + (st[j][1] if j >= 0 else "?")
    a = agg[name]
    a[0] += s; a[1] += e; a[2] += k
print("\nper function: stall% exec% static-instrs")
for name, (s, e, k) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
    print(f"{100*s/tot_s:5.1f}% {100*e/max(tot_e,1):5.1f}%ex {k:5d}i {16*k/1024:6.1f}KB {name}")
