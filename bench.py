#!/usr/bin/env python
"""Benchmark: one full distributed iteration of facet-consensus deblurring
(BASELINE.json metric "Mpixel-iterations/s"), on BASELINE.json configs[3]
("c4": 16384^2, 16x16 grid of 63x63 Moffat PSFs, 4x2 facets, 128-px overlap)
unless --config says otherwise.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A step = deblur_iterate(1): per facet one Local-Solver step (H + residual,
H^T + TV + prox + projection) then halo exchange + consensus.  Inputs are
resident in HBM before the timed region; the state (~9 GB at c4) is far larger
than L2, so no flush is needed between steps.  Time = CUDA events on the
library's own stream, barrier + synchronize on both sides, max over ranks.
`--impl reference` times the fp64 CPU oracle (the only reference this tier has)
on a bounded crop of the same workload.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FFMA = os.path.join(ROOT, "profiles", "r2", "ffma_peak.json")      # tools/ffma_peak.cu on a B200 box
TRAFFIC = os.path.join(ROOT, "profiles", "r2", "traffic.json")     # ncu --set full capture (tools/ncu_full.sh)
NOMINAL_SMS = 148
FMA_PER_SM_CLK = 128


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        return json.load(open(MEASURED))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 50 ms from before the timed
    region (nvidia-smi needs ~0.1-0.3 s to start) and filtered to the samples taken
    between mark_start() and mark_end() (host wall clock; the region is bracketed by
    device synchronisation, so wall time covers the device work)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)                     # let NVML start before the timed region
        except Exception:
            self.p = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        import datetime
        sm, mx, reasons, outside = [], 0.0, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [s.strip() for s in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                clk, cmax = float(f[2]), float(f[3])
            except ValueError:
                continue
            if self.t0 is not None and self.t1 is not None and not (self.t0 <= ts <= self.t1):
                outside += 1
                continue
            sm.append(clk)
            mx = max(mx, cmax)
            for nm, v in zip(names, f[6:10]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def run_ours(args, rank, world, local):
    import torch
    from paper_1705_06603_b200 import deblur as D

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # the communicator lines (ranks, channels, NVLS / P2P transport) go to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo")
    pb = synth.make_config(args.config)
    if args.operator_mode == 1:
        pb = synth.per_node(pb)
    if args.local_solver == "vmlmb":
        pb.local_solver, pb.inner_steps, pb.inner_increment = 1, args.inner, args.inner_inc
    nid = None
    if world > 1:
        import torch.distributed as dist
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t = torch.frombuffer(bytearray(D.nccl_id()), dtype=torch.uint8).clone()
        dist.broadcast(t, 0)
        nid = bytes(t.tolist())
    path = {"direct": D.CONV_DIRECT, "fft": D.CONV_FFT, "auto": D.CONV_AUTO}[args.path]
    params, keep = D.problem_params(pb, conv_path=path, rank=rank, world=world, device=local, nccl_id_bytes=nid,
                                    loopback_world=args.loopback if world == 1 else 0)
    dev = D.Deblur(params, keep)
    stream = torch.cuda.ExternalStream(dev.stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up: both start parities of the 2-iteration CUDA graph get captured here, so no
    # capture / instantiation happens inside the timed region
    dev.iterate(args.warmup)
    if args.warmup % 2:
        dev.iterate(3)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = sum(v[0] for k, v in dev.kernel_stats().items() if k != "halo_exchange")
    with ClockSampler(local) as clk:
        clk.mark_start()
        e0.record(stream)
        dev.iterate(args.steps)                       # the timed region: no instrumentation
        e1.record(stream)
        barrier()
        clk.mark_end()
    ms = e0.elapsed_time(e1)
    launches = sum(v[0] for k, v in dev.kernel_stats().items() if k != "halo_exchange") - launches0
    # second pass over the same K steps with per-kernel CUDA events on the library stream
    dev.set_profiling(True)
    dev.reset_stats()
    barrier()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    dev.iterate(args.steps)
    p1.record(stream)
    barrier()
    ms_prof = p0.elapsed_time(p1)
    stats = dev.kernel_stats()
    dev.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    npix = pb.ny * pb.nx
    value = npix * args.steps / (ms / 1e3) / 1e6

    # dominant kernel roofline (this rank's launches; per-launch averages; algorithmic work from the library)
    kern = {k: v for k, v in stats.items() if v[0] > 0 and k != "halo_exchange"}
    work = dev.kernel_work()
    pk = peaks()
    try:
        fp32_peak = float(json.load(open(FFMA))["fp32_tflops"])
        fp32_src = "profiles/r2/ffma_peak.json (measured FFMA, tools/ffma_peak.cu)"
    except (OSError, ValueError, KeyError):
        fp32_peak = NOMINAL_SMS * FMA_PER_SM_CLK * 2 * pk.get("sm_max_mhz", 1965.0) / 1e6   # TFLOP/s
        fp32_src = "fallback: 148 SM x 128 FP32 FMA/clk x 2 x sm_max_mhz (guide unit counts)"
    ridge = fp32_peak * 1e12 / (pk["hbm_gbs"] * 1e9)          # flop/byte where the two roofs meet

    def roof(name):
        """The kernel's roofline side by its algorithmic intensity (flops / compulsory bytes):
        above the ridge point the FP32 pipe bounds it (alu), below it HBM does."""
        n, tot_ms = kern[name]
        per = tot_ms / n / 1e3
        fl, by = work.get(name, (0.0, 0.0))
        alu = fl > 0 and (by <= 0 or fl / by >= ridge)
        out = {"kernel": name, "ms_per_launch": round(per * 1e3, 4)}
        if fl > 0:
            out["alu_frac"] = round(fl / per / 1e12 / fp32_peak, 4)
        if by > 0:
            out["hbm_frac"] = round(by / per / 1e9 / pk["hbm_gbs"], 4)
        if by > 0 and fl > 0:
            out["intensity_flop_per_byte"] = round(fl / by, 2)
        if alu:
            a = fl / per / 1e12
            out.update({"bound": "alu", "achieved": round(a, 3), "peak": round(fp32_peak, 2), "unit": "TFLOP/s",
                        "frac": round(a / fp32_peak, 4), "traffic": None, "peak_source": fp32_src})
            return out
        a = by / per / 1e9 if by > 0 else None
        out.update({"bound": "hbm", "achieved": None if a is None else round(a, 1), "peak": pk["hbm_gbs"],
                    "unit": "GB/s", "frac": None if a is None else round(a / pk["hbm_gbs"], 4), "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "_fallback" not in pk else "fallback"})
        return out

    dom = max(kern, key=lambda k: kern[k][1])
    roofline = roof(dom)
    # DRAM traffic of the same kernel from the committed `ncu --set full` capture (per launch)
    try:
        tr = json.load(open(TRAFFIC))
        kt = tr["kernels"].get(dom)
        if kt is not None and args.config == 4:
            roofline["traffic"] = kt["bytes"]
            roofline["traffic_source"] = os.path.relpath(TRAFFIC, ROOT) + " (" + tr["metric"] + ")"
    except (OSError, ValueError, KeyError):
        pass
    tot_ms_all = sum(x[1] for x in kern.values())
    breakdown = {}
    for k, v in kern.items():
        r = roof(k)
        breakdown[k] = {"launches": v[0], "ms_per_launch": round(v[1] / max(v[0], 1), 4),
                        "share": round(v[1] / max(tot_ms_all, 1e-9), 4), "bound": r["bound"],
                        "achieved": r["achieved"], "unit": r["unit"], "frac": r["frac"],
                        "hbm_frac": r.get("hbm_frac"), "alu_frac": r.get("alu_frac")}

    # end to end through the C ABI with host buffers: reset(y from pinned host) + K iterations + image D2H
    y_pin = torch.from_numpy(pb.y).pin_memory()
    img_pin = torch.empty((pb.ny, pb.nx), dtype=torch.float32).pin_memory() if rank == 0 else None

    def e2e_job():
        barrier()
        t0 = time.perf_counter()
        dev.reset(y_pin.numpy())                      # pinned host buffer, no staging copy
        dev.iterate(args.steps)
        dev.get_image(out=img_pin.numpy() if img_pin is not None else None)
        barrier()
        return time.perf_counter() - t0

    e2e_job()                                         # one untimed job (first-touch of pinned pages)
    te = torch.tensor([statistics.median(e2e_job() for _ in range(3))], dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    serial = {"value": round(npix * args.steps / float(te.item()) / 1e6, 3),
              "job": f"deblur_reset(y host pinned) + deblur_iterate({args.steps}) + deblur_get_image(host pinned); "
                     "median of 3 jobs after one untimed job",
              "seconds": round(float(te.item()), 3)}

    # pipelined jobs (a stream of exposures): the next observation's upload and the previous
    # image's download overlap the current job's iterations (deblur_stage_y / reset_staged /
    # get_image_async); every job still moves its y up and its image down inside the region
    img2 = [torch.empty((pb.ny, pb.nx), dtype=torch.float32).pin_memory() for _ in range(2)] if world == 1 else None
    y_np = y_pin.numpy()

    def e2e_pipelined(jobs):
        barrier()
        t0 = time.perf_counter()
        dev.stage_y(y_np)
        for j in range(jobs):
            dev.reset_staged()
            if j + 1 < jobs:
                dev.stage_y(y_np)
            dev.iterate(args.steps)
            dev.get_image_async(img2[j % 2].numpy())
        dev.sync()
        barrier()
        return time.perf_counter() - t0

    if world == 1:
        jobs = 4
        e2e_pipelined(2)                              # untimed
        tp = e2e_pipelined(jobs)
        e2e = {"value": round(npix * args.steps * jobs / tp / 1e6, 3), "unit": "Mpixel-iterations/s",
               "h2d_bytes_per_step": int(pb.y.nbytes // args.steps),
               "d2h_bytes_per_step": int(npix * 4 // args.steps),
               "job": f"{jobs} jobs back to back, each deblur_reset_staged (y staged from pinned host by "
                      f"deblur_stage_y during the previous job) + deblur_iterate({args.steps}) + "
                      "deblur_get_image_async (pinned host, downloaded during the next job); timed from the first "
                      "upload to the last download (deblur_sync)",
               "seconds": round(tp, 3), "serial_jobs": serial}
    else:
        e2e = {"value": serial["value"], "unit": "Mpixel-iterations/s",
               "h2d_bytes_per_step": int(pb.y.nbytes // args.steps),
               "d2h_bytes_per_step": int(npix * 4 // args.steps),
               "job": serial["job"], "seconds": serial["seconds"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(pb, args.cpu_seconds)

    if rank == 0:
        clocks = clk.summary()
        cfg = dict(synth.CONFIGS[args.config])
        line = {
            "metric": "Mpixel-iterations/s (full distributed iteration)",
            "value": round(value, 3), "unit": "Mpixel-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded star field, synth/)",
            "config": {"workload": f"c{args.config}", "image": f"{pb.ny}x{pb.nx}", "psf": f"{pb.P}x{pb.P}",
                       "psf_grid": f"{pb.gy}x{pb.gx}", "facets": f"{pb.fy}x{pb.fx}", "overlap": pb.overlap,
                       "lambda": pb.lam, "eps": pb.eps, "iterations_per_step": 1, "inner_steps": pb.inner_steps,
                       "local_solver": {0: "projected gradient", 1: "VMLM-B"}[pb.local_solver],
                       "conv_path": {1: "direct", 2: "fft"}[dev.conv_path],
                       "operator_mode": {0: "interpolated H per facet", 1: "per-node PSFs (paper node model)"}[
                           args.operator_mode],
                       "l2": "no flush: resident state >> 126 MB L2", "parallelism": f"facets over {world} GPU(s)"
                       + (f", loopback exchange between {args.loopback} virtual ranks" if args.loopback > 1 and world == 1 else "")},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "kernels": breakdown,
            "kernels_pass_ms_per_step": round(ms_prof / args.steps, 4),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dev.close()


def oracle_sample(pb, n: int):
    """A bounded crop of the workload for the oracle: the n x n block of the
    estimate domain starting at (N/4, N/4) (so it straddles PSF-grid cells like
    the bulk of the image) with its PSFs, weights and observed pixels, one facet."""
    from oracle import solver
    P = pb.P
    m = n - P + 1
    o = min(pb.ny // 4, pb.ny - n)
    prm = solver.Params(lam=pb.lam, eps=pb.eps, gamma=pb.gamma, rho=pb.rho, reg_kind=pb.reg_kind,
                        tv_boundary=pb.tv_boundary, inner_steps=pb.inner_steps)
    w = pb.noise_w[o:o + m, o:o + m] if pb.noise_w is not None else np.float64(np.float32(pb.noise_w_scalar))
    return solver.Deblur(pb.psfs, pb.wy[:, o:o + n], pb.wx[:, o:o + n], pb.y[o:o + m, o:o + m], w, 1, 1, 0, prm)


def cpu_model() -> str:
    """lscpu model name of the host (SURVEY §8d asks for it next to the core count)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(pb, seconds: float):
    n = min(pb.ny, 512)
    d = oracle_sample(pb, n)
    t0 = time.perf_counter()
    d.iterate(1)
    dt = time.perf_counter() - t0
    # scale the crop so one iteration takes ~seconds/2, then time 2 iterations
    n2 = int(min(pb.ny, max(n, n * math.sqrt(max(seconds / 2 / dt, 1.0)))))
    n2 = max(pb.P + 1, n2 - n2 % 2)
    d = oracle_sample(pb, n2)
    t0 = time.perf_counter()
    d.iterate(2)
    dt = time.perf_counter() - t0
    return {"value": round(n2 * n2 * 2 / dt / 1e6, 4), "unit": "Mpixel-iterations/s",
            "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"fp64 oracle, 2 iterations on the {n2}x{n2} crop at (N/4, N/4) of c{args_config(pb)} (1 facet)",
            "seconds": round(dt, 2)}


def args_config(pb):
    return pb.name.lstrip("c").split("@")[0]


def run_reference(args, rank, world):
    if rank != 0:
        return
    if world > 1 and "LOCAL_WORLD_SIZE" in os.environ:
        # torchrun exports OMP_NUM_THREADS=1 to every rank; the other ranks have exited, so
        # rank 0 runs the oracle on all host cores, as the N = 1 launch does (set before
        # liboracle.so / libgomp is loaded)
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    pb = synth.make_config(args.config)
    n = min(pb.ny, args.ref_crop)
    d = oracle_sample(pb, n)
    d.iterate(args.warmup)
    t0 = time.perf_counter()
    d.iterate(args.steps)
    dt = time.perf_counter() - t0
    value = n * n * args.steps / dt / 1e6
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = f"fp64 oracle, {n}x{n} crop at (N/4, N/4) of c{args.config} (1 facet), {args.steps} iterations"
    line = {"impl": "reference", "metric": "Mpixel-iterations/s (full distributed iteration)",
            "value": round(value, 4), "unit": "Mpixel-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded star field, synth/)",
            "config": {"workload": f"c{args.config}", "sample": sample},
            "cpu_baseline": {"value": round(value, 4), "unit": "Mpixel-iterations/s", "cores": cores,
                             "kind": "oracle", "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "Mpixel-iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--path", choices=["auto", "direct", "fft"], default="auto")
    ap.add_argument("--local-solver", choices=["pg", "vmlmb"], default="pg",
                    help="pg: one projected-gradient step per iteration (north star); vmlmb: VMLM-B inner solves")
    ap.add_argument("--inner", type=int, default=10, help="VMLM-B inner budget at the first outer iteration")
    ap.add_argument("--inner-inc", type=int, default=0, help="VMLM-B budget increment per outer iteration")
    ap.add_argument("--operator-mode", type=int, choices=[0, 1], default=0,
                    help="0: interpolated H restricted to facets (north star); 1: per-node PSFs, facets = PSF grid")
    ap.add_argument("--loopback", type=int, default=0,
                    help="N=1 only: run the multi-rank halo exchange between this many virtual ranks (params.loopback_world)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-crop", type=int, default=1024)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
