import time, sys, torch, numpy as np
sys.path.insert(0, '.')
import synth
from paper_1705_06603_b200 import deblur as D
pb = synth.make_config(4)
dev = D.Deblur.from_problem(pb)
y = torch.from_numpy(pb.y).pin_memory(); img = torch.empty((pb.ny, pb.nx)).pin_memory()
for rep in range(3):
    t0 = time.perf_counter(); dev.reset(y.numpy()); t1 = time.perf_counter(); dev.iterate(20); t2 = time.perf_counter(); dev.get_image(out=img.numpy()); t3 = time.perf_counter()
    print(f"reset {t1-t0:.3f}  iterate20 {t2-t1:.3f}  get_image {t3-t2:.3f}")
