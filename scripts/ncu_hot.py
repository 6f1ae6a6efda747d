"""Per-CUDA-line instruction and stall totals from an ncu report
(needs -lineinfo).  usage: ncu_hot.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; fname = "?"; agg = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    back = lambda name: r[len(r) - (len(hdr) - hdr.index(name))]  # robust to split source text
    ie = f(back("Instructions Executed"))
    st = f(back("Warp Stall Sampling (All Samples)"))
    agg.append((ie, st, f"{fname}:{r[0]}", r[1][:100]))
ti = sum(a[0] for a in agg) or 1; ts = sum(a[1] for a in agg) or 1
print(f"total warp-instr {ti:.4e}, stall samples {ts:.0f}")
for ie, st, where, s in sorted(agg, key=lambda a: -a[0])[:top]:
    print(f"{100*ie/ti:5.1f}% inst {100*st/ts:5.1f}% stall {where:22s} {s}")
print("--- by stall")
for ie, st, where, s in sorted(agg, key=lambda a: -a[1])[:12]:
    print(f"{100*ie/ti:5.1f}% inst {100*st/ts:5.1f}% stall {where:22s} {s}")
