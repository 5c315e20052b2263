"""Per-source-line instruction and stall-sample totals of an ncu capture
(needs -lineinfo and --import-source on):

    python tools/ncu_lines.py capture.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
fname = ""
lines = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "Line No"):
        d = dict(zip(range(len(r)), r))
        try:
            inst = int(r[hdr.index("Instructions Executed")])
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        lines.append((inst, samp, f"{fname}:{r[0]}", r[1].strip()[:90]))
ti = sum(l[0] for l in lines) or 1
ts = sum(l[1] for l in lines) or 1
print(f"total inst {ti}  samples {ts}")
print("-- by instructions")
for l in sorted(lines, reverse=True)[:top]:
    print(f"{100*l[0]/ti:5.1f}% i {100*l[1]/ts:5.1f}% s  {l[2]:14s} {l[3]}")
print("-- by stall samples")
for l in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"{100*l[0]/ti:5.1f}% i {100*l[1]/ts:5.1f}% s  {l[2]:14s} {l[3]}")
