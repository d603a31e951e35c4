"""Per-SASS-instruction hot spots of one kernel from an ncu report: shared-memory excess
wavefronts (bank conflicts) and warp-stall samples, with the CUDA source line each belongs to.
usage: python tools/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [N] [SKIP]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Address")
ix = {k: h.index(k) for k in h}
recs = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(h)]


def num(r, k):
    try:
        return float(r[ix[k]] or 0)
    except ValueError:
        return 0.0


tot_ex = sum(num(r, "L1 Wavefronts Shared Excessive") for r in recs)
tot_wf = sum(num(r, "L1 Wavefronts Shared") for r in recs)
tot_st = sum(num(r, "Warp Stall Sampling (All Samples)") for r in recs) or 1
print(f"shared wavefronts {tot_wf:,.0f}  excessive {tot_ex:,.0f}  stall samples {tot_st:,.0f}")
print("-- top excessive shared wavefronts")
for r in sorted(recs, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:top]:
    if num(r, "L1 Wavefronts Shared Excessive") <= 0:
        break
    print(f"{r[0]} {num(r, 'L1 Wavefronts Shared Excessive'):>14,.0f} of {num(r, 'L1 Wavefronts Shared'):>14,.0f}  {r[1][:70]}")
print("-- stall samples by opcode")
by = {}
for r in recs:
    op = r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]
    by[op] = by.get(op, 0) + num(r, "Warp Stall Sampling (All Samples)")
for k, v in sorted(by.items(), key=lambda x: -x[1])[:top]:
    print(f"  {k:30s} {100 * v / tot_st:5.1f}%")
