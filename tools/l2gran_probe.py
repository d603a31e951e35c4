"""A/B of cudaLimitMaxL2FetchGranularity (device-wide hint: 32 / 64 / 128 bytes fetched from
DRAM per L2 miss) on the c4 iteration: the column passes read 64-byte row segments at a
large stride, the row passes and K4 stream contiguously.  Prints ms per iteration (CUDA
events on the library stream) and per-kernel ms for each setting.  Not a benchmark line.
usage: python tools/l2gran_probe.py [config] [steps]"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1705_06603_b200 import deblur as D  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rt = ctypes.CDLL("libcudart.so.12")
LIMIT = 0x05                                           # cudaLimitMaxL2FetchGranularity
pb = synth.make_config(k)
for gran in (0, 32, 64, 128, 0):
    torch.cuda.set_device(0)
    if gran:
        rc = rt.cudaDeviceSetLimit(LIMIT, ctypes.c_size_t(gran))
        assert rc == 0, rc
    cur = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(cur), LIMIT)
    with D.Deblur.from_problem(pb) as dev:
        st = torch.cuda.ExternalStream(dev.stream)
        dev.iterate(6)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        dev.iterate(steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        dev.set_profiling(True)
        dev.reset_stats()
        dev.iterate(steps)
        torch.cuda.synchronize()
        ks = {n: v[1] / v[0] for n, v in dev.kernel_stats().items() if v[0] > 0 and "fft2" not in n}
    print(f"== set {gran or 'default'} (limit reads {cur.value}): {ms:.3f} ms/it  " +
          "  ".join(f"{n} {t:.3f}" for n, t in ks.items()), flush=True)
