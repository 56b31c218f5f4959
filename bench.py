#!/usr/bin/env python
"""bench.py -- throughput of the shearlet dec -> hard-threshold -> rec hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2d512|3d192|2d1024x64|3d128|2d256]
                    [--impl ours|reference]

Default workload (BASELINE.json configs[1], the metric's 2D config): 512^2
frames, nScales=4 shear levels [1,1,2,2] (R=49 shearlets), one step =
decompose -> hard_threshold(defaults_2d(40), RMS-scaled) -> reconstruct of a
batch of 8 distinct noisy cartoon frames (each frame's 103 MB coefficient
stack is materialised in HBM, so a step moves ~2.5 GB > L2; L2 is also flushed
between timed steps). Metric: frames/s (whole job, summed over ranks).

Multi-GPU (torchrun, one rank per GPU, NCCL): 2D frames are replicas/shards by
image (no collective); 3D shards the filter bank by shearlet index, broadcasts
the input volume and NCCL-reduces the reconstruction partial sums.

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference library compiled with our FFTW-API shim, all host
threads) on the same config, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
FP64_PEAK_TFLOPS = 34.0  # measured: tools/fp64_peak.cu (DFMA loop, 64 FMA/clk/SM at 1965 MHz)

CONFIGS = {
    # name: (dims, levels, schedule kind, sigma, frames per step per rank, seed base)
    "2d512": dict(dims=(512, 512), levels=[1, 1, 2, 2], sigma=40.0, batch=8, unit="frames/s",
                  metric="2D 512^2 dec+thr+rec frames/s (nScales=4, R=49)", baseline_cfg=1),
    "2d512_nostack": dict(dims=(512, 512), levels=[1, 1, 2, 2], sigma=40.0, batch=8, unit="frames/s", nostack=True,
                          metric="2D 512^2 denoise frames/s, coefficient stack not materialised (nScales=4, R=49)",
                          baseline_cfg=1),
    "2d256": dict(dims=(256, 256), levels=[1, 1], sigma=40.0, batch=32, unit="frames/s",
                  metric="2D 256^2 dec+rec frames/s (nScales=2, R=17)", baseline_cfg=0),
    "2d1024x64": dict(dims=(1024, 1024), levels=[1, 1, 2, 2], sigma=40.0, batch=64, unit="frames/s",
                      metric="2D 1024^2 x64 dec+thr+rec frames/s (R=49, sharded by image)", baseline_cfg=2),
    "3d128": dict(dims=(128, 128, 128), levels=[1, 1], sigma=40.0, batch=1, unit="vols/s",
                  metric="3D 128^3 dec+thr+rec vols/s (nScales=2, R=99)", baseline_cfg=3),
    "3d192": dict(dims=(192, 192, 192), levels=[1, 1, 2], sigma=40.0, batch=1, unit="vols/s",
                  metric="3D 192^3 dec+thr+rec vols/s (nScales=3 SL3D_2, R=292)", baseline_cfg=4),
    "3d192sl1": dict(dims=(192, 192, 192), levels=[0, 0, 1], sigma=40.0, batch=1, unit="vols/s",
                     metric="3D 192^3 dec+thr+rec vols/s (nScales=3 SL3D_1, R=76)", baseline_cfg=4),
    "3d256": dict(dims=(256, 256, 256), levels=[1, 1], sigma=40.0, batch=1, unit="vols/s",
                  metric="3D 256^3 dec+thr+rec vols/s (nScales=2, R=99)", baseline_cfg=None),
}


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def schedule_for(P, cfg):
    n = len(cfg["levels"])
    return P.ThresholdSchedule.defaults_2d(cfg["sigma"], n) if len(cfg["dims"]) == 2 else \
        P.ThresholdSchedule.defaults_3d(cfg["sigma"], n)


def make_inputs(gen_cartoon, add_noise, cfg, count, seed0):
    dims = cfg["dims"]
    clean = gen_cartoon(dims[0])
    return [add_noise(clean, cfg["sigma"], seed0 + i) for i in range(count)]


def algorithmic_bytes(cfg, R, frames):
    """Compulsory HBM bytes of one dec+thr+rec per frame with the stack
    materialised (SURVEY.md 8(d) with our real-valued filter representation):
    16 N (f read + f_rec write) + 16 R N (band write in dec + read in rec)
    + 16 R Nh (real psi half-spectrum read in dec and in rec; 2D) or the
    3D factor tables (L2-resident, counted once) + 8 N (W half read)."""
    dims = cfg["dims"]
    N = int(np.prod(dims))
    Nh = N // dims[-1] * (dims[-1] // 2 + 1)
    if len(dims) == 2:
        if cfg.get("nostack"):  # stack never written: f/f_rec + real psi halves read twice
            return frames * (16 * N + 16 * R * Nh)
        return frames * (16 * N + 16 * R * N + 16 * R * Nh)
    return frames * (16 * N + 16 * R * N + 8 * Nh)


def algorithmic_flops(cfg, R):
    """(2R+2) real-input FFTs at 2.5 N log2 N plus 14 flops per
    half-spectrum point per band (conj-multiply + multiply-add), per frame."""
    dims = cfg["dims"]
    N = int(np.prod(dims))
    Nh = N // dims[-1] * (dims[-1] // 2 + 1)
    return (2 * R + 2) * 2.5 * N * np.log2(N) + R * Nh * 14


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # wait for the first sample so the timed region is covered from its start
            t0 = time.time()
            self.first = self.proc.stdout.readline() if self.proc.stdout else ""
            while not self.first and time.time() - t0 < 5:
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU reference
def cpu_reference(cfg, seconds=12.0, steps=5, warmup=1):
    """The reference's own CPU path (oracle/_ref, all host threads): `warmup`
    untimed then up to `steps` timed single-frame (or single-volume)
    dec+thr+rec runs, stopping early once `seconds` of timed work is done (a
    bounded sample; at least one timed run). Falls back to the numpy oracle
    port when oracle/_ref is not built."""
    from oracle import ref
    dims, levels = cfg["dims"], cfg["levels"]
    cores = os.cpu_count() or 1
    n = len(levels)
    K = ([2.5] * (n - 1) + [3.8]) if len(dims) == 2 else ([3.0] * (n - 1) + [4.0])
    if ref.available():
        kind = "reference"
        sysr = ref.RefSystem2D(*dims, levels) if len(dims) == 2 else ref.RefSystem3D(dims, levels)
        clean = ref.cartoon(dims[0]) if len(dims) == 2 else ref.cartoon_volume(dims[0])
        x = ref.add_noise(clean, cfg["sigma"], 7)
        run = lambda: sysr.denoise(x, K, cfg["sigma"], threads=0)  # noqa: E731
    else:
        from oracle import shearlet_np as O
        kind = "port"
        cores = 1
        if len(dims) == 2:
            so = O.build_system_2d(*dims, levels)
            x = O.cartoon(dims[0]) + 40.0
            run = lambda: O.inverse_2d(O.hard_threshold(O.forward_2d(x, so), so.index, 0, so.filter_norms, K,  # noqa
                                                        cfg["sigma"]), so)
        else:
            so = O.build_system_3d(dims, levels)
            x = np.full(dims, 40.0)
            run = lambda: O.inverse_3d(O.hard_threshold(O.forward_3d(x, so), so.index, 0, so.filter_norms, K,  # noqa
                                                        cfg["sigma"]), so)
    nwarm = max(0, warmup) if len(dims) == 2 else 0  # a 3D volume is a long sample already
    for _ in range(nwarm):
        run()  # first-touch page faults, FFT plan creation
    times = []
    while True:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
        if sum(times) > seconds or len(times) >= max(1, steps):
            break
    total = sum(times)
    unit1 = "frame" if len(dims) == 2 else "volume"
    return {"value": len(times) / total, "unit": cfg["unit"], "cores": cores, "kind": kind,
            "sample": f"{len(times)} timed x 1 {unit1} dec+thr+rec (of {steps} requested, capped at ~{seconds:.0f} s) "
                      f"after {nwarm} warm-up, threads=0 (all {os.cpu_count()} host cores)"
                      + ("" if kind == "reference" else " [numpy port: oracle/_ref not built]")
                      + "; FFT = our FFTW-API shim (no libfftw3 in the image)"}


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="2d512", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        res = cpu_reference(cfg, seconds=60.0, steps=args.steps, warmup=args.warmup)
        line = {"metric": cfg["metric"], "value": res["value"], "unit": cfg["unit"], "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / res["value"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference phantoms + seeded Gaussian noise)", "impl": "reference",
                "config": {"workload": args.config, "dims": list(cfg["dims"]), "shear_levels": cfg["levels"]},
                "cpu_baseline": res,
                "e2e": {"value": res["value"], "unit": cfg["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_1402_5670_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    dims = cfg["dims"]
    is3d = len(dims) == 3
    prof = P.ScaleProfile.from_levels(cfg["levels"])
    sch = schedule_for(P, cfg)
    R_full = P.redundancy_3d(prof) if is3d else P.redundancy_2d(prof)

    # ---- work partition
    nstreams = int(os.environ.get("SLB_STREAMS", "6"))
    if is3d:
        # shearlet-index sharding: contiguous balanced band ranges
        lo, hi = R_full * rank // world, R_full * (rank + 1) // world
        sysg = P.build_system_3d(dims, prof, device=local, shard=(lo, hi) if world > 1 else None)
        frames = 1
        scaling = "strong"  # one volume per step whatever the rank count
    else:
        sysg = P.build_system_2d(*dims, prof, device=local)
        sysg.set_streams(nstreams)
        if cfg.get("nostack"):
            sysg.set_stack_output(False)  # reported separately from the materialised-stack metric
        if args.config == "2d1024x64":
            frames = cfg["batch"] // world  # fixed total batch sharded by image
            scaling = "strong"
        else:
            frames = cfg["batch"]  # per-rank batch fixed (replicas)
            scaling = "weak"

    gen = P.cartoon_volume if is3d else P.cartoon
    host_in = make_inputs(gen, P.add_gaussian_noise, cfg, frames, 1000 * rank)
    d_in = [torch.from_numpy(x).to(dev) for x in host_in]
    d_out = [torch.empty_like(x) for x in d_in]
    N = int(np.prod(dims))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream_ptr = lambda: P._stream_ptr(local)  # noqa: E731
    K = np.ascontiguousarray(sch.per_scale_factors, dtype=np.float64)
    import ctypes as C
    Kp = K.ctypes.data_as(C.POINTER(C.c_double))
    L = P.lib()

    d_in_b = torch.stack(d_in)
    d_out_b = torch.empty_like(d_in_b)

    def step():
        if not is3d:
            # batched denoise: frames spread over the handle's internal streams,
            # each frame's stack materialised in that stream's workspace
            P._check(L.sl_denoise_batch_dev(sysg.handle, C.c_void_p(d_in_b.data_ptr()), frames,
                                            C.c_void_p(d_out_b.data_ptr()), Kp, len(K), float(sch.sigma), 1,
                                            stream_ptr()))
            return
        for i in range(frames):
            x = d_in[i]
            if world > 1:
                dist.broadcast(x, src=0)
            # fused denoise of this rank's bands (dec rows + threshold + rec rows in one
            # pass, stack materialised); on a shard the output is the partial reconstruction
            P._check(L.sl_denoise_dev(sysg.handle, C.c_void_p(x.data_ptr()), C.c_void_p(d_out[i].data_ptr()),
                                      Kp, len(K), float(sch.sigma), 1, stream_ptr()))
            if world > 1:
                dist.reduce(d_out[i], dst=0, op=dist.ReduceOp.SUM)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    launches0 = sysg.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush.zero_()  # evict L2 between timed steps (outside the timed interval)
            starts[k].record()
            step()
            ends[k].record()
        barrier()
    launches = sysg.launch_count() - launches0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    total_units = (frames * world if not is3d else 1) * args.steps
    value = total_units / (ms_total / 1000.0)

    # ---- instrumented pass: per-kernel device time (CUDA events on the launch
    # stream), frames serialised on one stream so kernel durations do not overlap
    sysg.set_streams(1)
    sysg.set_profiling(True)
    for k in range(max(2, args.steps // 2)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    stats = sysg.pass_stats()
    sysg.set_profiling(False)
    sysg.set_streams(nstreams)

    # ---- end to end through the public API with host buffers (pinned)
    pinned_in = torch.from_numpy(np.stack(host_in)).pin_memory()
    pinned_out = torch.empty_like(pinned_in).pin_memory()
    barrier()
    e2e_times = []
    for k in range(max(3, args.steps // 2) + 1):
        barrier()
        t0 = time.perf_counter()
        if not is3d:
            P._check(L.sl_denoise_batch_host(sysg.handle, P._dp(pinned_in.numpy()), frames, P._dp(pinned_out.numpy()),
                                             Kp, len(K), float(sch.sigma), 1))
        else:
            for i in range(frames):
                xd = pinned_in[i].to(dev, non_blocking=True)
                if world > 1:
                    dist.broadcast(xd, src=0)
                od = P.denoise(xd, sysg, sch)
                if world > 1:
                    dist.reduce(od, dst=0, op=dist.ReduceOp.SUM)
                pinned_out[i].copy_(od)
        torch.cuda.synchronize()
        if k > 0:
            e2e_times.append(time.perf_counter() - t0)
    te = torch.tensor([float(np.median(e2e_times))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = (frames * world if not is3d else 1) / float(te.item())

    if rank == 0:
        peak, peak_kind = hbm_peak()
        R = R_full
        nbytes = algorithmic_bytes(cfg, R, 1)
        # dominant kernel by device time
        dom = max(stats.items(), key=lambda kv: kv[1][0]) if stats else ("none", (0.0, 0))
        dom_name, (dom_ms, dom_n, dom_units) = dom
        per_unit = pass_bytes(dom_name, dims)
        dom_bytes = per_unit * dom_units / max(dom_n, 1) if per_unit else None
        dom_avg_s = dom_ms / max(dom_n, 1) / 1000.0
        achieved = (dom_bytes / dom_avg_s / 1e9) if dom_avg_s > 0 and dom_bytes else None
        traffic = measured_traffic(args.config, dom_name, dom_units / max(dom_n, 1))
        # per-rank compulsory bytes per step: `frames` frames (2D) or 1/world of a volume's bands (3D)
        path_gbs = nbytes * (1.0 / world if is3d else frames) / (ms_step / 1000.0) / 1e9
        line = {
            "metric": cfg["metric"], "value": value, "unit": cfg["unit"], "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference cartoon phantom + seeded Gaussian noise (sigma 40)",
            "config": {"workload": args.config, "dims": list(dims), "shear_levels": cfg["levels"], "R": R_full,
                       "frames_per_step_per_rank": frames, "threshold": "defaults (RMS-scaled)",
                       "l2": "flushed between timed steps (256 MB write); stack per frame > L2",
                       "parallelism": (f"shearlet-shard{world}" if is3d else f"dp{world}")},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "bytes_per_launch": dom_bytes, "avg_launch_ms": dom_avg_s * 1000.0,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
            "path_roofline": {"bytes_per_unit": nbytes, "achieved": path_gbs, "frac": path_gbs / peak,
                              "note": "whole dec+thr+rec step: compulsory HBM bytes / device time"},
            "fp64": {"flops_per_unit": algorithmic_flops(cfg, R),
                     "achieved_tflops": algorithmic_flops(cfg, R) * (1.0 / world if is3d else frames)
                     / (ms_step / 1000.0) / 1e12,
                     "peak_tflops": FP64_PEAK_TFLOPS,
                     "frac": algorithmic_flops(cfg, R) * (1.0 / world if is3d else frames) / (ms_step / 1000.0)
                     / 1e12 / FP64_PEAK_TFLOPS,
                     "note": "per GPU; SURVEY 8(d) flop count; peak measured by tools/fp64_peak.cu"},
            "kernels": {k: {"ms_total": v[0], "launches": v[1], "bands": v[2]} for k, v in sorted(stats.items())},
            "gpu_launches": int(launches),
            "e2e": {"value": e2e_value, "unit": cfg["unit"], "h2d_bytes_per_step": frames * N * 8,
                    "d2h_bytes_per_step": frames * N * 8,
                    "api": ("sl_denoise_batch_host (pinned host in/out; H2D in frame order on a copy stream, fused dec/thr/rec on 3 compute streams, D2H in frame order on a second copy stream)" if not is3d else "denoise (sl_denoise_dev) with pinned H2D/D2H")},
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_reference(cfg, seconds=12.0, steps=10, warmup=1)
            except Exception as e:  # reported, never fatal
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measured_traffic(config, pass_name, bands_per_launch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    pass, from the committed ncu --set full summary (profiles/traffic.json,
    written by tools/ncu_summary.py traffic; cold-cache per-band bytes scaled to
    this run's bands per launch), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            e = json.load(fh)[config][pass_name]
        return e["dram_bytes_per_band"] * bands_per_launch
    except (OSError, KeyError, ValueError):
        return None


def pass_bytes(name, dims):
    """Bytes at the boundary of each pass per band (or spectrum) processed, for
    the current multi-pass design."""
    N = int(np.prod(dims))
    Nh = N // dims[-1] * (dims[-1] // 2 + 1)
    # 3D band group (csrc/fast3d_host.cuh fast3d_group): ~6 GB of rotated intermediate, >= 16
    G3 = int(os.environ.get("SLB_G3", "0")) or max(16, int(6 * 2 ** 30 / (16 * Nh)))
    return None if name == "none" else {
        # generic path
        "rows_c2r_thr": 16 * Nh + 8 * N,          # intermediate read + band write, per band
        "rows_c2r": 16 * Nh + 8 * N,
        "rows_r2c": 8 * N + 16 * Nh,
        "lines_decmul": 16 * Nh + 8 * Nh + 16 * Nh,  # F + psi (real) + intermediate write
        "lines_recmul": 16 * Nh + 8 * Nh + 16 * Nh,
        "lines_plain": 32 * Nh,
        "lines_divw": 32 * Nh + 8 * Nh,
        "reduce_bands": 16 * Nh,
        # fast 2D path (fast2d.cuh)
        "f2_rows_r2c": 8 * N + 16 * Nh,           # band rows read + column-major half write
        "f2_rows_c2r_thr": 16 * Nh + 8 * N,       # half read + thresholded band write
        "f2_rows_c2r": 16 * Nh + 8 * N,
        "f2_rows_fused": 16 * Nh + 8 * N + 16 * Nh,  # half read, thresholded band write, rec half write
        "f3_rows_fused": 16 * Nh + 8 * N + 16 * Nh,
        "f2_cols_dec": 8 * Nh + 16 * Nh,          # real psi + half write (F re-reads hit L2)
        "f2_cols_rec": 16 * Nh + 8 * Nh,          # half read + real psi (slot writes / final sum amortised)
        "f2_cols_fwd": 32 * Nh,
        "f2_cols_final": 32 * Nh + 8 * Nh,
        # fast 3D path (fast3d.cuh); psi synthesised from L2-resident tables
        "f3_rows_r2c": 8 * N + 16 * Nh,
        "f3_rows_c2r_thr": 16 * Nh + 8 * N,
        "f3_rows_c2r": 16 * Nh + 8 * N,
        "f3_axis1": 32 * Nh,
        "f3_ax0_dec": 16 * Nh + 16 * Nh / G3,     # rotated write + F read once per band group
        "f3_ax0_rec": 16 * Nh + 32 * Nh / G3,     # rotated read + accumulator RMW once per group
        "f3_ax0_fwd": 32 * Nh,
        "f3_ax0_final": 40 * Nh,
    }.get(name, None)


if __name__ == "__main__":
    main()
