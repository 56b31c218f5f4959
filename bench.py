#!/usr/bin/env python
"""bench.py -- throughput of the shearlet dec -> hard-threshold -> rec hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2d512|3d192|...]
                    [--impl ours|reference] [--no-3d] [--no-cpu-baseline]

BASELINE.json's metric has two halves; the default run measures both:
  * the headline line: 2D 512^2 (configs[1]), nScales=4 shear levels
    [1,1,2,2] (R=49); one step = decompose -> hard_threshold(defaults_2d(40),
    RMS-scaled) -> reconstruct of a streamed batch of 32 distinct noisy cartoon
    frames through the fused device batch (sl_denoise_batch_dev: lock-step
    frame pairs over the handle's streams, each frame's 103 MB thresholded
    stack materialised in HBM);
  * "workloads": {"3d192": ...}: 3D 192^3 SL3D_2 [1,1,2] (R=292, configs[4]),
    one step = the fused denoise of one noisy cartoon volume (sl_denoise_dev,
    16.5 GB stack materialised), timed the same way.
Each entry also reports the lone-frame (b = 1) fused denoise, the unfused
operators the reference's callers hit (sl_sheardec_threshold_dev +
sl_shearrec_dev = hard_threshold(forward) then inverse), the system build
time, the dominant kernel's roofline (live CUDA events) and the whole path's
HBM / FP64 fractions by SURVEY 8(d)'s byte and flop counts.

Timing: CUDA events on the launch stream around each step, L2 flushed
(256 MB write) between steps outside the timed interval, W >= 3 warm-up
steps, barrier + synchronize on both sides, max over ranks; nvidia-smi clocks
sampled during the timed region. e2e = the same metric through the host
entry points with pinned host in/out, copies inside the timed region.

Multi-GPU (torchrun, one rank per GPU): 2D frames are replicas (weak scaling,
no collective); 3D shards the filter bank by shearlet index through the
library's own NCCL communicator (sl_comm_create / sl_system_set_comm /
sl_denoise_dist_dev: broadcast of the volume, sharded fused denoise, reduce of
the half-spectrum accumulators, root-only final inverse FFT).

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference library compiled with our FFTW-API shim, all host
threads) on the same configs, rank 0 only, same JSON keys.
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
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
SMS = 148
FP64_FLOP_PER_CLK_SM = 128  # 64 DFMA / clk / SM (tools/fp64_peak.cu measured 34 TF at 1965 MHz under load)

CONFIGS = {
    # name: dims, shear levels, sigma, frames per step per rank, unit, metric
    "2d512": dict(dims=(512, 512), levels=[1, 1, 2, 2], sigma=40.0, batch=32, unit="frames/s",
                  metric="2D 512^2 dec+thr+rec frames/s (nScales=4, R=49)", baseline_cfg=1),
    "2d512_nostack": dict(dims=(512, 512), levels=[1, 1, 2, 2], sigma=40.0, batch=32, unit="frames/s", nostack=True,
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
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def fp64_peak_tflops(sm_mhz):
    """Theoretical DFMA peak at the sampled max SM clock: 148 SMs x 64 FMA x 2."""
    return SMS * FP64_FLOP_PER_CLK_SM * (sm_mhz or 1965.0) * 1e6 / 1e12


def config_dict(name, cfg, frames, world):
    """The `config` object both arms print (same keys and values)."""
    return {"workload": name, "dims": list(cfg["dims"]), "shear_levels": cfg["levels"],
            "frames_per_step_per_rank": frames, "threshold": "defaults_2d/3d(40), RMS-scaled",
            "l2": "flushed between timed steps (256 MB write); per-frame stack > L2",
            "parallelism": (f"shearlet-shard{world}" if len(cfg["dims"]) == 3 else f"dp{world}")}


def schedule_for(P, cfg):
    n = len(cfg["levels"])
    return P.ThresholdSchedule.defaults_2d(cfg["sigma"], n) if len(cfg["dims"]) == 2 else \
        P.ThresholdSchedule.defaults_3d(cfg["sigma"], n)


# ------------------------------------------------------------------ accounting
def _sizes(dims):
    N = int(np.prod(dims))
    return N, N // dims[-1] * (dims[-1] // 2 + 1)


def table_bytes(cfg, R):
    """3D factor tables (ĝ + Φ̂ planes, L2-resident): counted once per call."""
    dims = cfg["dims"]
    if len(dims) == 2:
        return 0
    n = dims[0]
    K = [2 ** (lv) for lv in cfg["levels"]]
    return sum((2 * k + 1) * n * n * 16 for k in K)


def path_bytes(cfg, R, frames, kind, group=1):
    """Compulsory HBM bytes of one call of `frames` frames.
    kind "fused": the fused denoise as timed -- f read + f_rec write (16 N),
    thresholded stack written once (8 R N, 0 when not materialised), real ψ̂
    halves read in dec and in rec once per lock-step group (2D: 16 R Nh per
    group of `group` frames) or the 3D factor tables + W half (8 Nh).
    kind "decrec": forward -> hard_threshold -> inverse through the
    materialised stack (the reference's operators): the stack is written and
    read back (16 R N), ψ̂ read per frame."""
    dims = cfg["dims"]
    N, Nh = _sizes(dims)
    stack_w = 0 if cfg.get("nostack") else 8 * R * N
    if len(dims) == 2:
        if kind == "fused":
            ngroups = -(-frames // group)
            return frames * (16 * N + stack_w) + ngroups * 16 * R * Nh
        return frames * (16 * N + 16 * R * N + 16 * R * Nh)
    T = table_bytes(cfg, R)
    if kind == "fused":
        return frames * (16 * N + stack_w + 8 * Nh) + T
    return frames * (16 * N + 16 * R * N + 8 * Nh) + T


def algorithmic_flops(cfg, R):
    """(2R+2) real-input FFTs at 2.5 N log2 N plus 14 flops per
    half-spectrum point per band (conj-multiply + multiply-add), per frame."""
    N, Nh = _sizes(cfg["dims"])
    return (2 * R + 2) * 2.5 * N * np.log2(N) + R * Nh * 14


def pass_bytes(name, dims, G3=None):
    """I/O bytes at the boundary of each pass per band (or spectrum) processed,
    for the kernel design in DESIGN.md section 4."""
    N, Nh = _sizes(dims)
    if G3 is None:
        G3 = max(16, int(6 * 2 ** 30 / (16 * Nh)))
    return None if name == "none" else {
        # generic path
        "rows_c2r_thr": 16 * Nh + 8 * N, "rows_c2r": 16 * Nh + 8 * N, "rows_r2c": 8 * N + 16 * Nh,
        "lines_decmul": 16 * Nh + 8 * Nh + 16 * Nh, "lines_recmul": 16 * Nh + 8 * Nh + 16 * Nh,
        "lines_plain": 32 * Nh, "lines_divw": 32 * Nh + 8 * Nh, "reduce_bands": 16 * Nh,
        # fast 2D path (fast2d.cuh, fast2d_fused.cuh)
        "f2_rows_r2c": 8 * N + 16 * Nh,             # band rows read + column-major half write
        "f2_rows_c2r_thr": 16 * Nh + 8 * N,         # half read + thresholded band write
        "f2_rows_c2r": 16 * Nh + 8 * N,
        "f2_rows_fused": 16 * Nh + 8 * N + 16 * Nh,  # half read, thresholded band write, rec half write
        "f2_cols_dec": 8 * Nh + 16 * Nh,            # real psi + half write (F re-reads hit L2)
        "f2_cols_rec": 16 * Nh + 8 * Nh,            # half read + real psi (slot writes / final sum amortised)
        "f2_cols_fwd": 32 * Nh, "f2_cols_final": 32 * Nh + 8 * Nh,
        # fast 3D path (fast3d.cuh); psi synthesised from L2-resident tables
        "f3_rows_fused": 16 * Nh + 8 * N + 16 * Nh,
        "f3_rows_r2c": 8 * N + 16 * Nh, "f3_rows_c2r_thr": 16 * Nh + 8 * N, "f3_rows_c2r": 16 * Nh + 8 * N,
        "f3_axis1": 32 * Nh,
        "f3_ax0_dec": 16 * Nh + 16 * Nh / G3,       # rotated write + F read once per band group
        "f3_ax0_rec": 16 * Nh + 32 * Nh / G3,       # rotated read + accumulator RMW once per group
        "f3_ax0_fwd": 32 * Nh, "f3_ax0_final": 40 * Nh,
        # three-pass 3D path (fast3d_split.cuh)
        "f3s_dec": 16 * Nh + 16 * Nh / G3,          # Z write (+ F once per group)
        "f3s_mid": 16 * Nh + 8 * N + 16 * Nh,       # Z read, thresholded band write, Z' write
        "f3s_rec": 16 * Nh + 32 * Nh / G3,          # Z' read (+ accumulator RMW once per group)
        # shear-group passes A / C (fast3d_group.cuh): F read and accumulator
        # RMW once per shear group (~8 bands at SL3D_2), charged here per band
        "f3g_dec": 16 * Nh + 16 * Nh / 8,           # Z write (+ F once per group)
        "f3g_rec": 16 * Nh + 32 * Nh / 8,           # Z' read (+ accumulator RMW once per group)
        "f3_transpose": 32 * Nh,
    }.get(name, None)


def measured_traffic(config, pass_name, bands_per_launch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    pass, from the committed ncu --set full summary (profiles/traffic.json,
    cold-cache per-band bytes scaled to this run's bands per launch), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            e = json.load(fh)[config][pass_name]
        return e["dram_bytes_per_band"] * bands_per_launch
    except (OSError, KeyError, ValueError):
        return None


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
            t0 = time.time()  # wait for the first sample so the timed region is covered from its start
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
    dec+thr+rec runs, stopping once `seconds` of timed work is done (a
    bounded sample; at least one timed run), plus its system build time.
    Falls back to the numpy oracle port when oracle/_ref is not built."""
    from oracle import ref
    dims, levels = cfg["dims"], cfg["levels"]
    cores = os.cpu_count() or 1
    n = len(levels)
    K = ([2.5] * (n - 1) + [3.8]) if len(dims) == 2 else ([3.0] * (n - 1) + [4.0])
    build_s = None
    if ref.available():
        kind = "reference"
        t0 = time.perf_counter()
        sysr = ref.RefSystem2D(*dims, levels) if len(dims) == 2 else ref.RefSystem3D(dims, levels)
        build_s = time.perf_counter() - t0
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
            "build_s": build_s,
            "sample": f"{len(times)} timed x 1 {unit1} dec+thr+rec (of {steps} requested, capped at ~{seconds:.0f} s) "
                      f"after {nwarm} warm-up, threads=0 (all {os.cpu_count()} host cores)"
                      + ("" if kind == "reference" else " [numpy port: oracle/_ref not built]")
                      + "; FFT = our FFTW-API shim (no libfftw3 in the image)"}


# ------------------------------------------------------------------ GPU workload
class Ctx:
    def __init__(self, world, rank, local):
        self.world, self.rank, self.local = world, rank, local


def run_workload(name, steps, warmup, ctx, want_cpu):
    import ctypes as C
    import torch
    import torch.distributed as dist
    import paper_1402_5670_b200 as P

    cfg = CONFIGS[name]
    world, rank, local = ctx.world, ctx.rank, ctx.local
    dev = torch.device("cuda", local)
    dims = cfg["dims"]
    is3d = len(dims) == 3
    prof = P.ScaleProfile.from_levels(cfg["levels"])
    sch = schedule_for(P, cfg)
    R_full = P.redundancy_3d(prof) if is3d else P.redundancy_2d(prof)

    # ---- system build (timed: the reference times build_system_* separately)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if is3d:
        sysg = P.build_system_3d(dims, prof, device=local)
    else:
        sysg = P.build_system_2d(*dims, prof, device=local)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    comm = None
    if world > 1:
        # the library's own NCCL communicator (sl_comm_create): 3D shards the
        # bank by shearlet index (broadcast f, accumulator reduce inside the
        # library); 2D batches keep the bank and shard by image
        from paper_1402_5670_b200 import dist as PD
        comm = PD.library_comm(local)
        PD.attach(sysg, comm)
    nstreams = int(os.environ.get("SLB_STREAMS", "6"))
    if is3d:
        frames, scaling = 1, "strong"  # one volume per step whatever the rank count
    else:
        sysg.set_streams(nstreams)
        if name == "2d1024x64":
            frames, scaling = cfg["batch"] // world, "strong"  # fixed total batch sharded by image
        else:
            frames, scaling = cfg["batch"], "weak"  # per-rank batch fixed (replicas)
    if cfg.get("nostack"):
        sysg.set_stack_output(False)  # reported separately from the materialised-stack metric

    gen = P.cartoon_volume if is3d else P.cartoon
    clean = gen(dims[0])
    host_in = [P.add_gaussian_noise(clean, cfg["sigma"], 1000 * rank + i) for i in range(frames)]
    d_in_b = torch.from_numpy(np.stack(host_in)).to(dev)
    d_out_b = torch.empty_like(d_in_b)
    N = int(np.prod(dims))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    K = np.ascontiguousarray(sch.per_scale_factors, dtype=np.float64)
    Kp = K.ctypes.data_as(C.POINTER(C.c_double))
    L = P.lib()
    sg = float(sch.sigma)

    def sp():
        return P._stream_ptr(local)

    def step_fused():
        if not is3d:
            # batched fused denoise: lock-step frame pairs spread over the handle's streams
            P._check(L.sl_denoise_batch_dev(sysg.handle, C.c_void_p(d_in_b.data_ptr()), frames,
                                            C.c_void_p(d_out_b.data_ptr()), Kp, len(K), sg, 1, sp()))
            return
        for i in range(frames):
            x, o = d_in_b[i], d_out_b[i]
            if world > 1:  # in-library NCCL broadcast + sharded denoise + accumulator reduce
                P._check(L.sl_denoise_dist_dev(sysg.handle, C.c_void_p(x.data_ptr()), C.c_void_p(o.data_ptr()),
                                               Kp, len(K), sg, 1, 0, sp()))
            else:
                P._check(L.sl_denoise_dev(sysg.handle, C.c_void_p(x.data_ptr()), C.c_void_p(o.data_ptr()),
                                          Kp, len(K), sg, 1, sp()))

    def step_lone():  # b = 1: one frame through sl_denoise_dev
        P._check(L.sl_denoise_dev(sysg.handle, C.c_void_p(d_in_b[0].data_ptr()), C.c_void_p(d_out_b[0].data_ptr()),
                                  Kp, len(K), sg, 1, sp()))

    stack = torch.empty((sysg.n_bands,) + tuple(dims), dtype=torch.float64, device=dev)

    def step_unfused():  # forward + fused hard_threshold, then inverse, through the stack
        P._check(L.sl_sheardec_threshold_dev(sysg.handle, C.c_void_p(d_in_b[0].data_ptr()),
                                             C.c_void_p(stack.data_ptr()), Kp, len(K), sg, 1, sp()))
        P._check(L.sl_shearrec_dev(sysg.handle, C.c_void_p(stack.data_ptr()), sysg.n_bands,
                                   C.c_void_p(d_out_b[0].data_ptr()), sp()))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def timed(fn, k, w, clk=None):
        for _ in range(w):
            fn()
        barrier()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        l0 = sysg.launch_count()
        if clk:
            clk.__enter__()
        barrier()
        for j in range(k):
            flush.zero_()  # evict L2 between timed steps (outside the timed interval)
            starts[j].record()
            fn()
            ends[j].record()
        barrier()
        if clk:
            clk.__exit__()
        launches = sysg.launch_count() - l0
        ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / k, launches

    clk = ClockSampler(local)
    ms_step, launches = timed(step_fused, steps, warmup, clk)
    units_step = frames * world if not is3d else 1
    value = units_step / (ms_step / 1000.0)
    k_side = max(3, min(steps, 20 if is3d else 50))
    ms_lone, _ = timed(step_lone, k_side, 2) if (not is3d and world == 1) else (ms_step, None)
    ms_unf, _ = timed(step_unfused, k_side, 2) if world == 1 else (None, None)
    del stack
    torch.cuda.empty_cache()

    # ---- instrumented pass: per-kernel device time (CUDA events on the launch
    # stream), frames serialised on one stream so kernel durations do not overlap
    sysg.set_streams(1)
    sysg.set_profiling(True)
    for _ in range(max(2, min(steps, 10) // 2)):
        flush.zero_()
        step_fused()
    torch.cuda.synchronize()
    stats = sysg.pass_stats()
    sysg.set_profiling(False)
    sysg.set_streams(nstreams)

    # ---- end to end through the public API with host buffers (pinned)
    pinned_in = torch.from_numpy(np.stack(host_in)).pin_memory()
    pinned_out = torch.empty_like(pinned_in).pin_memory()
    barrier()
    e2e_times = []
    for k in range(max(3, min(steps, 20 if is3d else 100) // 2) + 1):
        barrier()
        t0 = time.perf_counter()
        if not is3d:
            P._check(L.sl_denoise_batch_host(sysg.handle, P._dp(pinned_in.numpy()), frames, P._dp(pinned_out.numpy()),
                                             Kp, len(K), sg, 1))
        else:
            for i in range(frames):
                xd = pinned_in[i].to(dev, non_blocking=True)
                od = P.denoise_dist(xd, sysg, sch) if world > 1 else P.denoise(xd, sysg, sch)
                pinned_out[i].copy_(od)
        torch.cuda.synchronize()
        if k > 0:
            e2e_times.append(time.perf_counter() - t0)
    te = torch.tensor([float(np.median(e2e_times))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units_step / float(te.item())
    if rank != 0:
        return None

    peak, peak_src = hbm_peak()
    clocks = clk.summary()
    fp64_peak = fp64_peak_tflops(clocks.get("sm_max_mhz"))
    R = R_full
    share = (1.0 / world) if is3d else 1.0  # per-GPU share of a volume's bands
    group = min(4, frames) if (not is3d and frames > 1) else 1  # lock-step groups of 4 frames in the device batch
    fused_b = path_bytes(cfg, R, frames, "fused", group) * share
    lone_b = path_bytes(cfg, R, 1, "fused") * share
    unf_b = path_bytes(cfg, R, 1, "decrec") * share
    flops = algorithmic_flops(cfg, R) * share

    def frac(nbytes, ms):
        gbs = nbytes / (ms / 1000.0) / 1e9
        return {"bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peak}

    # dominant kernel by device time (serialised instrumented pass)
    dom_name, (dom_ms, dom_n, dom_units) = max(stats.items(), key=lambda kv: kv[1][0]) if stats else \
        ("none", (0.0, 0, 0))
    per_unit = pass_bytes(dom_name, dims)
    dom_bytes = per_unit * dom_units / max(dom_n, 1) if per_unit else None
    dom_avg_s = dom_ms / max(dom_n, 1) / 1000.0
    achieved = (dom_bytes / dom_avg_s / 1e9) if dom_avg_s > 0 and dom_bytes else None
    step_ms_serial = sum(v[0] for v in stats.values()) / max(1, max(2, min(steps, 10) // 2))
    out = {
        "metric": cfg["metric"], "value": value, "unit": cfg["unit"], "n_gpus": world, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference cartoon phantom + seeded Gaussian noise (sigma 40)",
        "config": config_dict(name, cfg, frames, world),
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": measured_traffic(name, dom_name, dom_units / max(dom_n, 1)),
                     "bytes_per_launch": dom_bytes, "avg_launch_ms": dom_avg_s * 1000.0,
                     "share_of_serial_step": (dom_ms / max(1, max(2, min(steps, 10) // 2))) / step_ms_serial
                     if step_ms_serial > 0 else None,
                     "peak_source": peak_src,
                     "note": "achieved = the pass's I/O bytes per launch (DESIGN.md 4) / its live CUDA-event "
                             "launch time; traffic = ncu dram bytes of the same kernel (profiles/traffic.json)"},
        "path_roofline": {
            "fused_denoise": dict(frac(fused_b, ms_step), frames_per_call=frames, lockstep_group=group,
                                  note="timed path: f + f_rec, stack written once (never read back), "
                                       "psi halves per lock-step group (2D) / factor tables + W (3D)"),
            "lone_frame": dict(frac(lone_b, ms_lone), ms=ms_lone, units_per_s=(1 if is3d else 1) / (ms_lone / 1e3),
                               note="b = 1 through sl_denoise_dev"),
            "dec_rec_unfused": (dict(frac(unf_b, ms_unf), ms=ms_unf, units_per_s=1.0 / (ms_unf / 1e3),
                                     note="sl_sheardec_threshold_dev + sl_shearrec_dev: stack written and read back")
                                if ms_unf else None),
        },
        "fp64": {"flops_per_unit": algorithmic_flops(cfg, R), "achieved_tflops": flops * frames / (ms_step / 1e3) / 1e12
                 if not is3d else flops / (ms_step / 1e3) / 1e12,
                 "peak_tflops": fp64_peak,
                 "note": "per GPU; SURVEY 8(d) flop count; peak = 148 SMs x 128 flop/clk x max SM clock"},
        "build_s": build_s,
        "kernels": {k: {"ms_total": v[0], "launches": v[1], "bands": v[2]} for k, v in sorted(stats.items())},
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_value, "unit": cfg["unit"], "h2d_bytes_per_step": frames * N * 8,
                "d2h_bytes_per_step": frames * N * 8,
                "api": ("sl_denoise_batch_host (pinned host in/out; H2D in frame order on a copy stream, fused "
                        "dec/thr/rec on 4 compute streams (one head frame, then lock-step pairs), D2H in frame "
                        "order on a second copy stream)" if not is3d
                        else "denoise (sl_denoise_dev) with pinned H2D/D2H")},
        "clocks": clocks,
    }
    out["fp64"]["frac"] = out["fp64"]["achieved_tflops"] / fp64_peak
    if world == 1 and want_cpu:
        try:
            out["cpu_baseline"] = cpu_reference(cfg, seconds=12.0, steps=10 if not is3d else 1, warmup=1)
        except Exception as e:  # reported, never fatal
            out["cpu_baseline"] = {"value": None, "error": str(e)}
    if comm is not None:
        sysg.set_comm(None)
    del sysg, comm
    torch.cuda.empty_cache()
    return out


def run_fp32(name, steps, warmup, local):
    """The optional fp32 mode (reported separately, never as the headline):
    2D -- the same lock-step 8-frame fused denoise with every FFT pass in fp32
    (sl_denoise_batch_f32_dev); 3D -- the fused denoise of one volume with the
    three band passes in fp32 (sl_denoise_f32_dev). Device-timed like the
    fp64 lines (L2 flushed between steps)."""
    import ctypes as C
    import torch
    import paper_1402_5670_b200 as P
    cfg = CONFIGS[name]
    dims = cfg["dims"]
    is3d = len(dims) == 3
    dev = torch.device("cuda", local)
    prof = P.ScaleProfile.from_levels(cfg["levels"])
    s = P.build_system_3d(dims, prof, device=local, dtype="f32") if is3d else \
        P.build_system_2d(*dims, prof, device=local, dtype="f32")
    sch = schedule_for(P, cfg)
    frames = 1 if is3d else cfg["batch"]
    gen = P.cartoon_volume if is3d else P.cartoon
    x = torch.from_numpy(np.stack([P.add_gaussian_noise(gen(dims[0]), cfg["sigma"], i) for i in range(frames)]))
    x = x.to(dev).float()
    o = torch.empty_like(x)
    K = np.ascontiguousarray(sch.per_scale_factors, dtype=np.float64)
    Kp = K.ctypes.data_as(C.POINTER(C.c_double))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def step():
        if is3d:
            P._check(P.lib().sl_denoise_f32_dev(s.handle, C.c_void_p(x.data_ptr()), None, C.c_void_p(o.data_ptr()),
                                                Kp, len(K), float(sch.sigma), 1, P._stream_ptr(local)))
        else:
            P._check(P.lib().sl_denoise_batch_f32_dev(s.handle, C.c_void_p(x.data_ptr()), frames, None,
                                                      C.c_void_p(o.data_ptr()), Kp, len(K), float(sch.sigma), 1,
                                                      P._stream_ptr(local)))
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    R = P.redundancy_3d(prof) if is3d else P.redundancy_2d(prof)
    nbytes = path_bytes(cfg, R, frames, "fused", 1 if is3d else 2) / 2  # fp32: every term halved
    peak, _ = hbm_peak()
    gbs = nbytes / (ms / 1e3) / 1e9
    del s
    torch.cuda.empty_cache()
    return {"metric": cfg["metric"] + ", fp32 mode", "value": frames / (ms / 1e3), "unit": cfg["unit"],
            "ms_per_step": ms, "steps": steps, "dtype": "f32",
            "path_roofline": {"bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peak},
            "note": "optional fp32 mode (within 1e-5 of the fp64 reference, tests/test_gpu_fp32.py); not the headline"}


# ------------------------------------------------------------------ main
def reference_line(name, steps, warmup, ngpus):
    cfg = CONFIGS[name]
    res = cpu_reference(cfg, seconds=60.0 if len(cfg["dims"]) == 2 else 240.0,
                        steps=steps if len(cfg["dims"]) == 2 else 1, warmup=warmup)
    frames = cfg["batch"] if name != "2d1024x64" else cfg["batch"] // max(1, ngpus)
    return {"metric": cfg["metric"], "value": res["value"], "unit": cfg["unit"], "n_gpus": ngpus,
            "ms_per_step": 1000.0 / res["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic: reference cartoon phantom + seeded Gaussian "
            "noise (sigma 40)", "impl": "reference", "config": config_dict(name, cfg, frames, ngpus),
            "build_s": res.get("build_s"), "cpu_baseline": res,
            "e2e": {"value": res["value"], "unit": cfg["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="2d512", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-3d", action="store_true", help="skip the nested 3d192 workload of the default run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nested = args.config == "2d512" and not args.no_3d

    if args.impl == "reference":
        if rank != 0:
            return
        line = reference_line(args.config, args.steps, args.warmup, args.gpus)
        line.update(steps=args.steps, warmup=args.warmup)
        if nested:
            line["workloads"] = {"3d192": reference_line("3d192", args.steps, args.warmup, args.gpus)}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Ctx(world, rank, local)
    line = run_workload(args.config, args.steps, args.warmup, ctx, not args.no_cpu_baseline)
    if nested:
        k3 = max(3, min(args.steps, 20))
        w3 = run_workload("3d192", k3, max(3, args.warmup), ctx, not args.no_cpu_baseline)
        if rank == 0:
            w3["steps"], w3["warmup"] = k3, max(3, args.warmup)
            line["workloads"] = {"3d192": w3}
            if world == 1:
                line["workloads"]["2d512_f32"] = run_fp32("2d512", args.steps, max(3, args.warmup), local)
                line["workloads"]["3d192_f32"] = run_fp32("3d192", k3, max(3, args.warmup), local)
    if rank == 0:
        line.update(steps=args.steps, warmup=args.warmup)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
