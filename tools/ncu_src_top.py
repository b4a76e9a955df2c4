"""Developer tool: per-source-line instruction and stall-sample shares of one kernel in an
ncu report (`ncu -i REP --page source --csv --print-source cuda,sass`).
argv: report.ncu-rep [top=40]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


cur, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not r[0].isdigit() or hdr is None:
        continue
    v = num(r[hdr.index("Instructions Executed")])
    s = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    if v or s:
        agg[(cur, int(r[0]))] = (v, s, r[1].strip()[:90])
tv = sum(a[0] for a in agg.values()) or 1
ts = sum(a[1] for a in agg.values()) or 1
print(f"instructions {tv:.0f}, stall samples {ts:.0f}")
for (f, ln), (v, s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{f}:{ln:<5d} {100 * v / tv:5.1f}% instr {100 * s / ts:5.1f}% samples  {src}")
