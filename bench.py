#!/usr/bin/env python
"""Benchmark: integral histograms/s and output GB/s (% of HBM) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the north-star's 70 % target config):
1920x1080 uint8 frames, 32 uniform bins, a batch of 64 frames per step,
frame-sharded across the N ranks (strong scaling: 64 frames in total).
Synthetic frames are ``synth_image(1920, 1080, k)`` for k = 0..63 (the
reference bench's generator, bench.py:59-62).

One JSON line on rank 0.  ``value`` is device-resident throughput (frames
already in HBM, outputs written to HBM), CUDA-event timed, max over ranks;
``e2e`` is the same metric through the host-buffer public API
(pipeline.FramePipeline: pinned H2D of the frames, kernels, pinned D2H of
the 17 GB result, all inside the timed region).

``--impl reference`` times the reference algorithm on the host CPU: the
oracle's C port of the reference's fastest strategy, cross-weave
(strategies.py:129-150), with every host thread, on a bounded sample of the
same workload (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WIDTH, HEIGHT, BINS, FRAMES = 1920, 1080, 32, 64
WORKLOAD = "1920x1080 u8 frames, 32 uniform bins, 64-frame batch (BASELINE cfg2), frame-sharded"
METRIC = "integral histograms/sec"
UNIT = "hist/s"
ALG_BYTES_PER_HIST = WIDTH * HEIGHT + 256 + 4 * BINS * WIDTH * HEIGHT
OUT_BYTES_PER_HIST = 4 * BINS * WIDTH * HEIGHT


def synth_image(width, height, seed):
    """bench.py:59-62 of the reference: default_rng(SeedSequence([seed, W, H]))."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, width, height]))
    return rng.integers(0, 256, size=(height, width), dtype=np.uint8)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per k2_scan launch from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        return d.get("k2_scan_hd_bytes_per_frame")
    except Exception:
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 5 ms while
    the timed region runs (the recipe's nvidia-smi fields, read directly)."""

    REASONS = {  # nvmlClocksEventReason* bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        import pynvml as N

        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            try:
                bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            except AttributeError:
                bits = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            for name, bit in self.REASONS.items():
                if bits & bit:
                    self.reasons.add(name)
            self._stop.wait(0.005)

    def __enter__(self):
        self.thread = threading.Thread(target=self._safe_run, daemon=True)
        self.thread.start()
        return self

    def _safe_run(self):
        try:
            self._run()
        except Exception as exc:  # NVML missing: report, do not fail the bench
            self.error = repr(exc)

    def __exit__(self, *exc):
        self._stop.set()
        self.thread.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "error": getattr(self, "error", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference_sample(frames_idx, threads=0):
    """Oracle C port of the reference cross-weave on the host; returns seconds
    and the number of histograms computed."""
    from oracle import oracle as O

    lut = O.np_uniform_table(BINS)
    imgs = [synth_image(WIDTH, HEIGHT, k) for k in frames_idx]
    t0 = time.perf_counter()
    for img in imgs:
        O.compute_crossweave(img, lut, BINS, threads)
    return time.perf_counter() - t0, len(imgs)


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host CPU (rank 0 only)."""
    if rank != 0:
        return
    from oracle import oracle as O

    cores = O.max_threads()
    per_step = args.ref_frames
    idx = list(range(per_step))
    for _ in range(args.warmup):
        cpu_reference_sample(idx[:1])
    times = []
    for _ in range(args.steps):
        dt, n = cpu_reference_sample(idx)
        times.append(dt)
    total = sum(times)
    value = per_step * args.steps / total
    sample = (f"{per_step} of the 64 HD frames per step (seeds 0..{per_step - 1}), "
              f"C port of reference compute_crossweave (strategies.py:129-150), {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_block(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "output_gbs": value * OUT_BYTES_PER_HIST / 1e9,
    }
    print(json.dumps(line), flush=True)


def config_block(world):
    return {"workload": WORKLOAD, "width": WIDTH, "height": HEIGHT, "bins": BINS,
            "frames_per_step": FRAMES, "parallelism": f"frame-shard x{world}",
            "l2": "no flush: per-step output 17 GB >> 126 MB L2 (inputs 133 MB > L2)"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1711_01919_b200 as ih
    from paper_1711_01919_b200 import device, pipeline, sharding

    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    spec = ih.BinSpec.uniform(BINS)

    def reduce_max(vals):
        """Max over ranks (NCCL needs CUDA tensors; gloo is used only for the
        single-GPU path test of this code)."""
        if world == 1:
            return list(vals)
        on = dev if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor(list(vals), dtype=torch.float64, device=on)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()
    f0, f1 = sharding.frame_shards(FRAMES, world)[rank]
    nloc = f1 - f0
    host_frames = np.stack([synth_image(WIDTH, HEIGHT, k) for k in range(f0, f1)])
    d_frames = torch.from_numpy(host_frames).to(dev)
    out = device.empty_output(nloc, BINS, HEIGHT, WIDTH, dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        device.prepare(d_frames, spec.table, BINS, stream=stream)
        ev_mid.record(stream)
        device.scan(d_frames, spec.table, BINS, out, stream=stream)

    plan = device.plan(nloc, HEIGHT, WIDTH, BINS, aligned16=d_frames.data_ptr() % 16 == 0)
    launches_per_step = plan["launches"]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    ev_mid = torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        step()
    barrier()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(dev_index) as clocks:
        barrier()
        for k in range(args.steps):
            starts[k].record(stream)
            ev_mid = mids[k]
            step()
            ends[k].record(stream)
        barrier()
    total_ms = starts[0].elapsed_time(ends[-1])
    scan_ms = sum(mids[k].elapsed_time(ends[k]) for k in range(args.steps)) / args.steps
    prep_ms = sum(starts[k].elapsed_time(mids[k]) for k in range(args.steps)) / args.steps

    # ---- parity spot check of the timed output (frame f0), outside the timed region
    import zlib

    with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as fh:
        gold = json.load(fh)["1920x1080x32_frames"]
    crc_ok = f"{zlib.crc32(out[0].cpu().numpy().tobytes()):08x}" == gold[f0]

    # ---- e2e through the host-buffer API (pinned H2D + kernels + pinned D2H)
    e2e = None
    if args.e2e_steps > 0:
        pipe = pipeline.FramePipeline(nloc, HEIGHT, WIDTH, spec, chunk=args.chunk)
        h_in = pipeline.pinned_empty((nloc, HEIGHT, WIDTH), dtype=torch.uint8)
        h_in.copy_(torch.from_numpy(host_frames))
        h_out = pipeline.pinned_empty((nloc, BINS, HEIGHT, WIDTH))
        pipe.run(h_in, h_out)  # warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            pipe.run(h_in, h_out)
        barrier()
        e2e_s = reduce_max([time.perf_counter() - t0])[0]
        e2e = {"value": FRAMES * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(pipe.h2d_bytes) * world,
               "d2h_bytes_per_step": int(pipe.d2h_bytes) * world,
               "steps": args.e2e_steps, "timer": "host perf_counter around synchronized steps"}
        crc_ok = crc_ok and f"{zlib.crc32(h_out[0].numpy().tobytes()):08x}" == gold[f0]
        # the e2e roofline: a plain pinned D2H copy of one output slice (PCIe bound)
        probe = out[: min(nloc, 4)].view(torch.int32)
        dst = h_out[: probe.shape[0]].view(torch.int32)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        for _ in range(3):
            dst.copy_(probe, non_blocking=True)
        torch.cuda.synchronize(dev)
        d2h_gbs = 3 * probe.numel() * 4 / (time.perf_counter() - t1) / 1e9
        e2e["d2h_copy_gbs"] = d2h_gbs
        e2e["e2e_out_gbs"] = e2e["value"] * OUT_BYTES_PER_HIST / 1e9 / world
        e2e["frac_of_d2h_copy"] = e2e["e2e_out_gbs"] / d2h_gbs
        del h_out, h_in, pipe

    total_ms, scan_ms, prep_ms, bad = reduce_max([total_ms, scan_ms, prep_ms,
                                                  0.0 if crc_ok else 1.0])
    if rank != 0:
        return
    value = FRAMES * args.steps / (total_ms / 1000.0)
    peak, peak_src = measured_peaks()
    achieved = nloc * ALG_BYTES_PER_HIST / (scan_ms / 1000.0) / 1e9
    traffic = committed_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_block(world),
        "output_gbs": value * OUT_BYTES_PER_HIST / 1e9,
        "hbm_frac_step": value * ALG_BYTES_PER_HIST / 1e9 / peak / world,
        "roofline": {"bound": "hbm", "kernel": "k2_scan", "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (traffic * nloc if traffic else None),
                     "alg_bytes_per_launch": nloc * ALG_BYTES_PER_HIST,
                     "launch_ms": scan_ms, "prepare_ms": prep_ms},
        "gpu_launches": launches_per_step * args.steps,
        "plan": plan,
        "parity": "frame 0 crc32 == reference golden" if not bad else "MISMATCH",
        "clocks": clocks.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and args.cpu_baseline_frames > 0:
        from oracle import oracle as O

        dt, n = cpu_reference_sample(range(args.cpu_baseline_frames))
        line["cpu_baseline"] = {
            "value": n / dt, "unit": UNIT, "cores": O.max_threads(), "kind": "port",
            "sample": f"{n} HD frames (seeds 0..{n - 1}) through the C port of reference "
                      f"compute_crossweave (strategies.py:129-150), all host threads"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=4, help="frames per pipelined e2e chunk")
    ap.add_argument("--cpu-baseline-frames", type=int, default=64)
    ap.add_argument("--ref-frames", type=int, default=16, help="frames per reference-arm step")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = os.environ.get("IH_BENCH_BACKEND", "nccl")  # gloo: 1-GPU path test only
        dev_index = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(dev_index)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
