"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of one
steady-state c4 iteration from an `ncu --set full` report made by
tools/ncu_full.sh (13 launches in iteration order: S plan, S/2 strip plan, update), written as the JSON that
bench.py reads for the roofline's `traffic` field.

  python tools/traffic_from_ncu.py gpurun_out/p.ncu-rep profiles/r1/traffic.json
"""
import csv
import io
import json
import subprocess
import sys

ORDER = ["H_fft_rows", "H_fft_cols", "H_fft_rows_inv", "H_fft2_rows", "H_fft2_cols", "H_fft2_rows_inv",
         "HT_fft_rows", "HT_fft_cols", "HT_fft_rows_inv", "HT_fft2_rows", "HT_fft2_cols", "HT_fft2_rows_inv",
         "update_from_g"]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    ir, iw, it = (hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
    res = {"source": rep, "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)",
           "kernels": {}}
    for name, r in zip(ORDER, data):
        b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
        res["kernels"][name] = {"kernel": r[ki][:80], "bytes": b, "ncu_ms": float(r[it]) * tscale[units[it]]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
