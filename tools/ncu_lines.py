"""Per-source-line totals from `ncu --page source --csv --print-source cuda,sass`
(instructions executed, warp-stall samples), top N lines.
usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N] [SKIP]"""
import csv
import io
import os
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
fname, h, recs = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Name":
        fname = os.path.basename(r[1])
    elif r[:2] == ["Line No", "Source"]:
        h = r
        ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    elif h and r and r[0].isdigit():
        try:
            recs.append((fname, int(r[0]), r[1], int(r[ie] or 0), int(r[ws] or 0)))
        except ValueError:
            pass
ti, ts = sum(x[3] for x in recs) or 1, sum(x[4] for x in recs) or 1
print(f"total warp instructions {ti:,}  stall samples {ts:,}")
for f, ln, src, i, s in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{f[:10]:10s}:{ln:<5d} {100*i/ti:5.1f}% inst {100*s/ts:5.1f}% stall  {src.strip()[:80]}")
