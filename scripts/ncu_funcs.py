"""Instructions / stall samples per source function (engine .cu) from an ncu
report; usage: ncu_funcs.py REP SRC [tiles]"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep, srcf = sys.argv[1], sys.argv[2]
tiles = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; fname = '?'; agg = []
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or not r or not r[0].isdigit(): continue
    back = lambda name: r[len(r) - (len(hdr) - hdr.index(name))]
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    agg.append((fname, int(r[0]), f(back("Instructions Executed")), f(back("Warp Stall Sampling (All Samples)"))))
src = open(srcf).read().split('\n')
funcs = []
for i, l in enumerate(src, 1):
    m2 = re.search(r'(?:__device__ __forceinline__ [\w:<>*]+ |__global__ void (?:__launch_bounds__\([^)]*\) )?)(\w+)\(', l)
    if m2: funcs.append((i, m2.group(1)))
    if l.startswith('  auto ') and '= [&]' in l: funcs.append((i, 'lambda:' + l.split()[1]))
def fn_of(line):
    best = '?'
    for i, n in funcs:
        if i <= line: best = n
    return best
ti = sum(a[2] for a in agg) or 1; ts = sum(a[3] for a in agg) or 1
d = defaultdict(lambda: [0.0, 0.0])
base = srcf.split('/')[-1]
for fname, line, ie, st in agg:
    key = fn_of(line) if fname == base else fname
    d[key][0] += ie; d[key][1] += st
for k, (v, s) in sorted(d.items(), key=lambda kv: -kv[1][0])[:18]:
    print(f"{100*v/ti:5.1f}% inst {v/tiles:7.1f}/unit {100*s/ts:5.1f}% stall  {k}")
