#!/usr/bin/env python
"""Benchmark: integral histograms/s and output GB/s (% of HBM) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 512|hd64|4k128|8k256] [--gather] [--dry-run]

`--gpus N` is authoritative: under torchrun WORLD_SIZE must equal N; run
directly with N > 1, bench.py re-launches itself under torch.distributed.run
with N ranks (and exits non-zero when fewer than N GPUs are visible).

`512` is configs[1] (512x512x32, one image per step, a replica per GPU;
CUDA-graph replayed steps, eager calls reported beside them).
Default workload (BASELINE.json configs[2], the north-star's 70 % target
config): 1920x1080 uint8 frames, 32 uniform bins, a batch of 64 frames per
step, frame-sharded across the N ranks (strong scaling: 64 frames in total).
`4k128` / `8k256` are configs[3] / configs[4]: one image per step, the bin
dimension sharded across ranks (each rank computes a contiguous bin slab, no
collective on the data path; `--gather` additionally times an NCCL gather of
the slabs onto rank 0, reported separately).  Synthetic images are
``synth_image(W, H, k)`` (the reference bench's generator, bench.py:59-62).

One JSON line on rank 0.  ``value`` is device-resident throughput (images in
HBM, outputs written to HBM), CUDA-event timed, max over ranks; ``e2e`` is the
same metric through the host-buffer public API (pipeline.FramePipeline: pinned
H2D of the images, kernels, pinned D2H of the whole result, all inside the
timed region).

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
import zlib
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "integral histograms/sec"
UNIT = "hist/s"


@dataclass(frozen=True)
class Workload:
    key: str
    width: int
    height: int
    bins: int
    frames: int  # integral histograms per step
    shard: str   # "frames" | "bins"
    desc: str

    @property
    def alg_bytes(self) -> int:  # u8 read + LUT + u32 write, one full histogram
        return self.width * self.height + 256 + 4 * self.bins * self.width * self.height

    @property
    def out_bytes(self) -> int:
        return 4 * self.bins * self.width * self.height


WORKLOADS = {
    "512": Workload("512", 512, 512, 32, 1, "replicas",
                    "512x512 u8 image, 32 uniform bins, one image per step (BASELINE cfg1), "
                    "one replica per GPU"),
    "hd64": Workload("hd64", 1920, 1080, 32, 64, "frames",
                     "1920x1080 u8 frames, 32 uniform bins, 64-frame batch (BASELINE cfg2), "
                     "frame-sharded"),
    "4k128": Workload("4k128", 3840, 2160, 128, 1, "bins",
                      "3840x2160 u8 image, 128 uniform bins (BASELINE cfg3), bin-sharded"),
    "8k256": Workload("8k256", 8192, 8192, 256, 1, "bins",
                      "8192x8192 u8 image, 256 uniform bins (BASELINE cfg4), bin-sharded"),
}


def synth_image(width, height, seed):
    """bench.py:59-62 of the reference: default_rng(SeedSequence([seed, W, H]))."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, width, height]))
    return rng.integers(0, 256, size=(height, width), dtype=np.uint8)


def uniform_table(bins):
    return ((np.arange(256) * bins) // 256).astype(np.uint8)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(wl: Workload, plan: dict):
    """dram__bytes_read.sum + dram__bytes_write.sum per histogram of k2_scan from
    the committed ncu --set full capture (profiles/ncu_traffic.json), or None
    when there is none for this workload or it was taken with a different
    launch plan (segments / column tiles) than the one this run uses."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            e = json.load(fh)["per_histogram"][wl.key]
    except Exception:
        return None
    if e.get("column_tiles", 1) != plan.get("column_tiles", 1):
        return None
    # captured per segment count without tail split or skew: both only move
    # rows between segments, so the DRAM bytes of the same count are the same
    # (the reads are the image plus one carry table per segment)
    # (keys "<n>/kb2": the bin-pair grouping, two bins per scan CTA)
    key = str(plan.get("segments")) + ("/kb2" if plan.get("bins_per_cta") == 2 else "")
    cap = e.get("by_segments", {}).get(key)
    return cap["bytes"] if cap else None


CSV_EXTRA = "devices,alg_bytes,gbs,frac_of_peak,ncu_dram_bytes,host_cpu"


def write_csv(path: str, line: dict, wl: Workload) -> None:
    """Append the run as one row of the reference's CSV schema
    (pkg/src/inthist/bench.py:24) plus the BASELINE.md 4.5 roofline columns;
    per-histogram figures (median_ms = 1000 / aggregate hist/s)."""
    from paper_1711_01919_b200.harness import CSV_HEADER

    new = not os.path.exists(path)
    v = line["value"]
    ms = 1000.0 / v
    crc = golden().get(f"{wl.width}x{wl.height}x{wl.bins}", {}).get("crc", "")
    tr = line["roofline"].get("traffic")
    hists = line["config"]["histograms_per_step"]
    row = [line.get("impl", "single_pass"), wl.width, wl.height, wl.bins, 0, 0, line["steps"],
           f"{ms:.6f}", f"{ms:.6f}", f"{v:.6f}", crc if line.get("parity", "").startswith(
               ("rank-0 output crc32 ==", "output crc32 ==")) else "",
           line["n_gpus"], wl.alg_bytes, f"{v * wl.alg_bytes / 1e9:.1f}",
           f"{line['hbm_frac_step']:.4f}", f"{tr / hists:.0f}" if tr else "",
           '"' + line["config"]["host_cpu"] + '"']
    with open(path, "a") as fh:
        if new:
            fh.write(CSV_HEADER + "," + CSV_EXTRA + "\n")
        fh.write(",".join(str(x) for x in row) + "\n")


def golden():
    with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as fh:
        return json.load(fh)


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

    def _sample(self):
        N = self._nvml
        self.samples.append(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM))
        try:
            bits = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except AttributeError:
            bits = N.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for name, bit in self.REASONS.items():
            if bits & bit:
                self.reasons.add(name)

    def _loop(self):
        try:
            while not self._stop.wait(0.005):
                self._sample()
        except Exception as exc:
            self.error = repr(exc)

    def __enter__(self):
        self._nvml = None
        try:  # NVML initialised here, so the first sample is at the region's start
            import pynvml as N

            N.nvmlInit()
            self._nvml = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
            self._sample()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception as exc:  # NVML missing: report, do not fail the bench
            self.error = repr(exc)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self.thread.join(timeout=5)
            try:
                self._sample()  # and one at its end
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "error": getattr(self, "error", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU side
def cpu_sample(wl: Workload, budget_s: float = 20.0):
    """The oracle's C port of the reference cross-weave on all host threads, on a
    bounded sample of the workload.  Returns (hist/s, cores, sample text)."""
    from oracle import oracle as O

    cores = O.max_threads()
    lut = uniform_table(wl.bins)
    if wl.shard == "replicas":  # one small image per step: repeat it within the budget
        img = synth_image(wl.width, wl.height, 0)
        t1 = time.perf_counter()
        O.compute_crossweave(img, lut, wl.bins)
        per = max(time.perf_counter() - t1, 1e-6)
        n = int(max(1, min(10000, budget_s / per)))
        t1 = time.perf_counter()
        for _ in range(n):
            O.compute_crossweave(img, lut, wl.bins)
        dt = time.perf_counter() - t1
        return n / dt, cores, (f"{n} repetitions of synth_image({wl.width}, {wl.height}, 0) "
                               f"x {wl.bins} bins, C port of reference compute_crossweave "
                               f"(strategies.py:129-150), {cores} threads")
    if wl.shard == "frames":
        # size the sample from one timed frame so it stays within the budget
        first = synth_image(wl.width, wl.height, 0)
        t1 = time.perf_counter()
        O.compute_crossweave(first, lut, wl.bins)
        per = max(time.perf_counter() - t1, 1e-6)
        n = int(max(1, min(wl.frames, budget_s / per)))
        imgs = [synth_image(wl.width, wl.height, k) for k in range(n)]
        t1 = time.perf_counter()
        for img in imgs:
            O.compute_crossweave(img, lut, wl.bins)
        dt = time.perf_counter() - t1
        return n / dt, cores, (f"{n} of the {wl.frames} frames (seeds 0..{n - 1}), C port of "
                               f"reference compute_crossweave (strategies.py:129-150), "
                               f"{cores} threads")
    # one big image: time a 16-bin slab (the LUT maps every other bin out of range)
    img = synth_image(wl.width, wl.height, 0)
    nb = min(16, wl.bins)
    slab_lut = np.where(lut < nb, lut, 255).astype(np.uint8)
    t1 = time.perf_counter()
    O.compute_crossweave(img, slab_lut, nb)
    dt = time.perf_counter() - t1
    return (nb / wl.bins) / dt, cores, (
        f"bins 0..{nb - 1} of the {wl.bins}-bin tensor of synth_image seed 0, scaled by "
        f"{nb}/{wl.bins}; C port of reference compute_crossweave, {cores} threads")


def config_block(wl: Workload, world: int):
    kind = {"frames": "frame-shard", "bins": "bin-shard", "replicas": "replica"}[wl.shard]
    l2 = (f"no flush: per-step output {wl.frames * wl.out_bytes / 1e9:.1f} GB >> 126 MB L2"
          if wl.frames * wl.out_bytes > 126e6 else
          f"no flush: steps rotate over {SMALL_BUFFERS} input/output buffer sets "
          f"({SMALL_BUFFERS * (wl.alg_bytes) / 1e6:.0f} MB > 126 MB L2)")
    return {"workload": wl.desc, "key": wl.key, "width": wl.width, "height": wl.height,
            "bins": wl.bins, "histograms_per_step": step_histograms(wl, world),
            "parallelism": f"{kind} x{world}", "l2": l2, "host_cpu": cpu_model()}


SMALL_BUFFERS = 8  # cfg1: buffer sets the steps rotate over (> L2 in total)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} threads)"
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def run_reference(args, wl: Workload, rank, world):
    """--impl reference: the reference algorithm on the host CPU (rank 0 only)."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample(wl, budget_s=0.2)
    budget = min(args.ref_budget, 150.0 / args.steps)  # whole run within a few minutes
    samples = [cpu_sample(wl, budget_s=budget) for _ in range(args.steps)]
    value = statistics.median(v for v, _, _ in samples)
    _, cores, sample = samples[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * wl.frames / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_block(wl, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "output_gbs": value * wl.out_bytes / 1e9,
    }
    print(json.dumps(line), flush=True)


def rank_share(wl: Workload, rank: int, world: int):
    """This rank's frames [f0, f1) x bins [b0, b1): contiguous frame runs
    (frame-sharded), bin slabs (bin-sharded, reference streaming.py:81-82), or
    the whole workload per rank (replicas)."""
    from paper_1711_01919_b200 import sharding

    if wl.shard == "frames":
        f0, f1 = sharding.frame_shards(wl.frames, world)[rank]
        return f0, f1, 0, wl.bins
    if wl.shard == "bins":
        b0, b1 = sharding.bin_slabs(wl.bins, world)[rank]
        return 0, wl.frames, b0, b1
    return 0, wl.frames, 0, wl.bins


def step_histograms(wl: Workload, world: int) -> int:
    """Integral histograms all ranks complete per step."""
    return wl.frames * world if wl.shard == "replicas" else wl.frames


def run_dry(args, wl: Workload, rank, world):
    """--dry-run: the N-rank plumbing without device work.  Each rank takes its
    share, 'runs' for a rank-dependent host delay, and the step time is the max
    over ranks -- the same reduction run_ours applies to its CUDA-event times."""
    import torch
    import torch.distributed as dist

    share = rank_share(wl, rank, world)
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    ms = 1000.0 * (time.perf_counter() - t0)
    shares = [share]
    rank_ms = [ms]
    if world > 1:
        shares = [None] * world
        dist.all_gather_object(shares, share)
        rank_ms = [None] * world
        dist.all_gather_object(rank_ms, ms)
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": UNIT,
                          "n_gpus": world, "ms_per_step": ms, "rank_ms": rank_ms,
                          "shares": [list(x) for x in shares],
                          "histograms_per_step": step_histograms(wl, world),
                          "config": config_block(wl, world)}), flush=True)


# ------------------------------------------------------------------ GPU side
def run_ours(args, wl: Workload, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1711_01919_b200 as ih
    from paper_1711_01919_b200 import device, sharding

    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    spec = ih.BinSpec.uniform(wl.bins)

    def reduce_max(vals):
        """Max over ranks (NCCL needs CUDA tensors; gloo is used only for the
        single-GPU path test of this code)."""
        if world == 1:
            return list(vals)
        on = dev if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor(list(vals), dtype=torch.float64, device=on)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # this rank's share: frames [f0, f1) x bins [b0, b1); --share-of N times
    # rank 0's share of an N-GPU run on this one GPU
    pw = args.share_of if args.share_of else world
    if wl.shard == "frames":
        f0, f1 = sharding.frame_shards(wl.frames, pw)[rank]
        b0, b1 = 0, wl.bins
    else:
        f0, f1 = 0, wl.frames
        b0, b1 = sharding.bin_slabs(wl.bins, pw)[rank]
    nloc, nb = f1 - f0, b1 - b0
    active = nloc > 0 and nb > 0
    host = np.stack([synth_image(wl.width, wl.height, k) for k in range(f0, max(f1, f0 + 1))])
    d_img = torch.from_numpy(host).to(dev)
    out = device.empty_output(max(nloc, 1), max(nb, 1), wl.height, wl.width, dev)
    stream = torch.cuda.current_stream(dev)
    brange = (b0, b1) if active else None
    tuned = None

    def set_hint(c):  # an autotune candidate [segments, tail_pct, tail_div, flags, ms]
        device.set_plan_hint(nloc, wl.height, wl.width, nb, c[0], c[1], c[2], skew=bool(c[3] & 4),
                             kb=2 if c[3] & 8 else 4 if c[3] & 16 else 0)

    # Steps are pipelined the way a video stream runs: the prepass of batch k+1
    # (k2_colcounts: reads only the images) runs on a side stream into the
    # other of two workspaces while batch k's scan (write-bound) runs, and the
    # scans of consecutive batches alternate between two streams and two
    # output buffers, so batch k+1's first CTAs fill the SMs batch k's
    # finished CTAs leave (the tail of a grid, DESIGN 8.1).  Every step still
    # executes both phases over its full batch; --no-overlap serialises all.
    # scans on high-priority streams, prepasses on a low-priority one: the
    # block scheduler fills SMs with scan CTAs first and the prepasses take the
    # gaps (same box, 100 steps: 4K x 128 4-way share 0.843-0.852 -> 0.859,
    # others within noise; IH_BENCH_PRIO=0 restores equal priorities)
    prio = os.environ.get("IH_BENCH_PRIO", "1") == "1" and args.overlap
    side = torch.cuda.Stream(dev, priority=0)
    nws = max(1, device.workspace_bytes(max(nloc, 1), wl.height, wl.width, max(nb, 1)))
    outs, sstreams = [out], [torch.cuda.Stream(dev, priority=-1) if prio else stream]
    if args.overlap and active:
        free, _ = torch.cuda.mem_get_info(dev)
        if free > out.numel() * 4 + (8 << 30):  # a second output buffer fits
            outs.append(device.empty_output(nloc, nb, wl.height, wl.width, dev))
            sstreams.append(torch.cuda.Stream(dev, priority=-1 if prio else 0))
    # prepasses run AHEAD steps ahead of the scans (one workspace each in
    # flight): with two scan streams, batch k+1's carries are ready when batch
    # k's first CTAs retire, so its scan can start in their slots
    ahead = 2 if len(outs) > 1 else 1
    if args.autotune and active:  # measured row-segment count for this shape (warm-up phase)
        # the whole call (prepare + scan): tuning the scan alone picked many
        # short segments whose prepass, even overlapped, cost more (HD x8:
        # step 0.80 vs 0.88; profiles/r01f/autotune_objective.txt)
        objective = "call"
        tuned = device.autotune(nloc, wl.height, wl.width, wl.bins, bin_range=brange, device=dev,
                                images=d_img[:nloc], out=out[:nloc], objective=objective)
        tuned["objective"] = objective
        # workspaces for every candidate the pipelined refinement below may pick
        for c in tuned["ranked"][:args.refine]:
            set_hint(c)
            nws = max(nws, device.workspace_bytes(nloc, wl.height, wl.width, nb))
        set_hint(tuned["ranked"][0])
    wss = [torch.empty(nws, dtype=torch.uint8, device=dev) for _ in range(ahead + 1)]

    def run_steps(n, ev_scan0=None, ev_scan1=None):
        """Issue n steps; returns per-step (scan start, scan end) events."""
        before = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        after = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        prep_done = [torch.cuda.Event() for _ in range(n)]

        nw = len(wss)

        def issue_prep(k):
            s_prep = side if args.overlap else stream
            if args.overlap:
                s_prep.wait_event(kick)
                if k >= nw:
                    s_prep.wait_event(after[k - nw])  # workspace k % nw is free again
            if active:
                device.prepare(d_img, spec.table, wl.bins, bin_range=brange, stream=s_prep,
                               workspace=wss[k % nw])
            prep_done[k].record(s_prep)

        kick = torch.cuda.Event()
        kick.record(stream)
        for s_k in sstreams:
            if s_k is not stream:
                s_k.wait_event(kick)
        for k in range(min(ahead, n)):
            issue_prep(k)
        for k in range(n):
            s_k = sstreams[k % len(sstreams)]
            s_k.wait_event(prep_done[k])
            before[k].record(s_k)
            if active:
                device.scan(d_img, spec.table, wl.bins, outs[k % len(outs)], bin_range=brange,
                            stream=s_k, workspace=wss[k % nw])
            after[k].record(s_k)
            if k + ahead < n:
                issue_prep(k + ahead)
        for s_k in sstreams:
            if s_k is not stream:
                stream.wait_stream(s_k)
        return before, after

    def isolated_scan_ms(n=5):
        """Average k2_scan launch with nothing else running (the roofline's
        per-launch time: consecutive launches overlap in the pipelined steps)."""
        if not active:
            return 0.0
        device.prepare(d_img, spec.table, wl.bins, bin_range=brange, stream=stream,
                       workspace=wss[0])
        device.scan(d_img, spec.table, wl.bins, out, bin_range=brange, stream=stream,
                    workspace=wss[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        tot = 0.0
        for _ in range(n):
            e0.record(stream)
            device.scan(d_img, spec.table, wl.bins, out, bin_range=brange, stream=stream,
                        workspace=wss[0])
            e1.record(stream)
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
        return tot / n

    if tuned is not None and len(outs) > 1 and args.refine > 1:
        # pipelined refinement: the call-timed ranking misorders plans whose
        # scans overlap differently in these steps (8 HD frames: bin pairs 2 %
        # faster per call, 4 % slower per pipelined step; profiles/r02m/), so
        # the top candidates run a few real steps each and the fastest is kept
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps_ms = []
        for c in tuned["ranked"][:args.refine]:
            set_hint(c)
            run_steps(2)
            e0.record(stream)
            run_steps(6)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            steps_ms.append((e0.elapsed_time(e1) / 6, c))
        best = min(steps_ms, key=lambda x: x[0])[1]
        set_hint(best)
        tuned["pipelined_refine_ms"] = [[round(ms, 4)] + c[:4] for ms, c in steps_ms]
        tuned["chosen"] = best[:4]
    plan = device.plan(nloc, wl.height, wl.width, nb,
                       aligned16=d_img.data_ptr() % 16 == 0) if active else {"launches": 0}
    run_steps(args.warmup)
    barrier()
    with ClockSampler(dev_index) as clocks:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        befores, afters = run_steps(args.steps)
        t_end.record(stream)
        barrier()
    total_ms = t_start.elapsed_time(t_end)
    overlapped_ms = sum(b.elapsed_time(a) for b, a in zip(befores, afters)) / args.steps
    scan_ms = isolated_scan_ms() if len(outs) > 1 else overlapped_ms
    n_out_buffers = len(outs)
    del outs[1:]  # free the second output buffer before the checks, queries and e2e
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    prep_ms = max(0.0, total_ms / args.steps - scan_ms)  # exposed (not overlapped) part

    # ---- parity spot check of the timed output, outside the timed region
    gold = golden()
    crc_ok = True
    if active:
        if wl.key == "hd64":
            crc_ok = f"{zlib.crc32(out[0].cpu().numpy().tobytes()):08x}" == \
                gold["1920x1080x32_frames"][f0]
        else:
            planes = gold[f"{wl.width}x{wl.height}x{wl.bins}"]["plane_crc"]
            crc_ok = f"{zlib.crc32(out[0, 0].cpu().numpy().tobytes()):08x}" == planes[b0]

    # ---- cfg4's batched region queries (K3) on this rank's slab: Q = 65,536
    # inclusive regions drawn as acceptance C4 does, timed apart
    queries = None
    if wl.key == "8k256" and active:
        rng = np.random.default_rng(20260823 + 4)
        Q = 65536
        rr = np.sort(rng.integers(0, wl.height, (Q, 2)), axis=1)
        cc = np.sort(rng.integers(0, wl.width, (Q, 2)), axis=1)
        regs = torch.from_numpy(np.stack([rr[:, 0], cc[:, 0], rr[:, 1], cc[:, 1]], 1)
                                .astype(np.int32)).to(dev)
        slab = out[0]
        res_q = torch.empty((Q, nb), dtype=torch.uint64, device=dev)
        for _ in range(3):
            device.region_histograms(slab, regs, out=res_q)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(10):
            device.region_histograms(slab, regs, out=res_q)
        e1.record()
        torch.cuda.synchronize(dev)
        q_ms = reduce_max([e0.elapsed_time(e1) / 10])[0]
        # spot check against the four-corner formula on the host for a few queries
        t_host = slab[:, :, :].view(torch.int32)
        ok = True
        for k in (0, 1, Q // 2, Q - 1):
            r0, c0, r1, c1 = (int(x) for x in regs[k].tolist())
            corners = [(r1, c1, 1), (r0 - 1, c1, -1), (r1, c0 - 1, -1), (r0 - 1, c0 - 1, 1)]
            want = sum(sgn * t_host[:, a, b].to(torch.int64).remainder(1 << 32)
                       for a, b, sgn in corners if a >= 0 and b >= 0)
            ok = ok and bool(torch.equal(res_q[k].view(torch.int64).cpu(), want.cpu()))
        queries = {"kernel": "k3_region_histograms", "Q": Q, "bins": nb, "ms": q_ms,
                   "region_histograms_per_s": Q / (q_ms / 1e3), "spot_check": ok}
        crc_ok = crc_ok and ok

    # ---- optional gather of bin slabs onto rank 0 (not part of the metric)
    gather_ms = None
    if args.gather and wl.shard == "bins" and world > 1:
        barrier()
        g_start = time.perf_counter()
        full = sharding.gather_slabs(out[0] if active else None, wl.bins, wl.height, wl.width,
                                     rank, world)
        barrier()
        gather_ms = reduce_max([1000 * (time.perf_counter() - g_start)])[0]
        del full

    # ---- e2e through the host-buffer API (pinned H2D + kernels + pinned D2H)
    e2e = None
    if args.e2e_steps > 0 and active:
        try:
            e2e = run_e2e(args, wl, spec, host, nloc, (b0, b1), out, dev, barrier, reduce_max,
                          world)
            crc_ok = crc_ok and e2e.pop("_crc_ok")
        except (RuntimeError, MemoryError) as exc:  # e.g. pinned allocation failure
            e2e = {"value": None, "unit": UNIT, "error": repr(exc)[:200]}

    # ---- same-run write-only ceiling (outside the timed region, after every
    # check that reads `out`): the best of a 32-bit fill and a memset over up
    # to 4 GiB of the output buffer
    write_gbs = None
    if active:
        flat = out.view(torch.int32).view(-1)[: 1 << 30]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 0.0
        for op in (lambda: flat.fill_(0x01020304), lambda: flat.zero_()):
            op()
            torch.cuda.synchronize(dev)
            e0.record()
            for _ in range(5):
                op()
            e1.record()
            torch.cuda.synchronize(dev)
            best = max(best, 5 * flat.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
        write_gbs = best

    total_ms, scan_ms, prep_ms, bad = reduce_max([total_ms, scan_ms, prep_ms,
                                                  0.0 if crc_ok else 1.0])
    if rank != 0:
        return
    value = wl.frames * args.steps / (total_ms / 1000.0)
    peak, peak_src = measured_peaks()
    alg_launch = nloc * (wl.width * wl.height + 256 + 4 * nb * wl.width * wl.height)
    achieved = alg_launch / (scan_ms / 1000.0) / 1e9
    traffic = committed_traffic(wl, plan)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_block(wl, world),
        "output_gbs": value * wl.out_bytes / 1e9,
        "hbm_frac_step": value * wl.alg_bytes / 1e9 / peak / world,
        "roofline": {"bound": "hbm", "kernel": "k2_scan", "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (traffic * nloc if traffic and nb == wl.bins else None),
                     "write_ceiling_gbs": write_gbs,
                     "frac_of_write_ceiling": (achieved / write_gbs if write_gbs else None),
                     "alg_bytes_per_launch": alg_launch, "launch_ms": scan_ms,
                     "prepare_exposed_ms": prep_ms, "rank0_share": [f0, f1, b0, b1],
                     "launch_timer": ("isolated k2_scan launches (CUDA events, after the timed "
                                      "steps): in the pipelined steps consecutive scans overlap"
                                      if n_out_buffers > 1 else "CUDA events around each timed scan"),
                     "pipelined_scan_span_ms": overlapped_ms},
        "pipelined_steps": bool(args.overlap),
        "output_buffers": n_out_buffers,
        "gpu_launches": plan["launches"] * args.steps,
        "plan": plan,
        "autotune": tuned,
        "parity": "rank-0 output crc32 == reference golden" if not bad else "MISMATCH",
        "clocks": clocks.summary(),
    }
    if traffic is None:
        line["roofline"]["traffic_note"] = ("no committed ncu capture of this workload with "
                                            "this launch plan (profiles/ncu_traffic.json)")
    if args.share_of:
        share_bytes = nloc * (wl.width * wl.height + 256 + 4 * nb * wl.width * wl.height)
        line["hbm_frac_step"] = share_bytes * args.steps / (total_ms / 1e3) / 1e9 / peak
        line["metric"] = (METRIC + f" (projected {args.share_of}-GPU job: rank 0's share timed "
                          "alone on this GPU)")
        line["emulated_share"] = {
            "of_gpus": args.share_of, "rank": 0, "frames": [f0, f1], "bins": [b0, b1],
            "per_gpu_hbm_frac_step": share_bytes * args.steps / (total_ms / 1e3) / 1e9 / peak,
            "note": "no other rank ran; the projection assumes every rank's share takes as long "
                    "(equal shares, no inter-GPU traffic on the data path)"}
    if gather_ms is not None:
        line["gather_ms"] = gather_ms
    if queries is not None:
        line["queries"] = queries
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and args.cpu_baseline:
        v, cores, sample = cpu_sample(wl, budget_s=args.ref_budget)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if args.csv:
        write_csv(args.csv, line, wl)


def run_small(args, wl: Workload, rank, world, local_rank):
    """cfg1 (512x512x32): one image per step -- a 33.8 MB problem whose kernels
    run for a few microseconds, so the step is launch-bound unless the launches
    are pre-recorded.  Each rank (a replica) cycles over SMALL_BUFFERS
    (input, output, workspace) sets, > L2 in total.  ``value`` replays the
    steps from CUDA graphs (8 one-image calls per graph, every call still one
    full integral histogram); ``eager`` is the same K steps as plain
    device.integral_histogram calls (preallocated output and workspace)."""
    import torch
    import torch.distributed as dist

    from paper_1711_01919_b200 import device, pipeline

    import paper_1711_01919_b200 as ih

    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    spec = ih.BinSpec.uniform(wl.bins)
    lut = spec.table
    nbuf = SMALL_BUFFERS
    host = synth_image(wl.width, wl.height, 0)
    imgs = [device.upload_image(host, dev) for _ in range(nbuf)]
    outs = [device.empty_output(1, wl.bins, wl.height, wl.width, dev)[0] for _ in range(nbuf)]
    nws = max(16, device.workspace_bytes(1, wl.height, wl.width, wl.bins))
    wss = [torch.empty(nws, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
    plan = device.plan(1, wl.height, wl.width, wl.bins)
    stream = torch.cuda.Stream(dev)

    def reduce_max(vals):
        if world == 1:
            return list(vals)
        on = dev if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor(list(vals), dtype=torch.float64, device=on)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def call(k, s=None):
        device.integral_histogram(imgs[k], lut, wl.bins, out=outs[k], workspace=wss[k],
                                  stream=s if s is not None else stream)

    # independent images are served `inflight` at a time (a serving process
    # with concurrent requests): call k runs on branch stream k % inflight, so
    # one image's launch chain overlaps the others'; every call is still one
    # full integral histogram with its own input, output and workspace
    inflight = max(1, min(args.inflight, nbuf))
    branches = [torch.cuda.Stream(dev) for _ in range(inflight)]

    def all_calls():
        for b in branches:
            b.wait_stream(stream)
        for k in range(nbuf):
            call(k, branches[k % inflight])
        for b in branches:
            stream.wait_stream(b)

    with torch.cuda.stream(stream):
        for k in range(nbuf):  # warm: attributes, plan caches
            call(k)
    torch.cuda.synchronize(dev)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        return g

    g_all = capture(all_calls)
    g_one = [capture(lambda k=k: call(k)) for k in range(nbuf)]
    g_scan = capture(lambda: [device.scan(imgs[k], lut, wl.bins, outs[k], workspace=wss[k],
                                          stream=stream) for k in range(nbuf)])

    def graph_steps(n):
        with torch.cuda.stream(stream):
            for _ in range(n // nbuf):
                g_all.replay()
            for k in range(n % nbuf):
                g_one[k].replay()

    def eager_steps(n):
        for i in range(n):
            call(i % nbuf)

    def timed(fn, n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        fn(n)
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1)

    graph_steps(max(args.warmup, nbuf))
    eager_steps(max(args.warmup, nbuf))
    barrier()
    with ClockSampler(dev_index) as clocks:
        total_ms = timed(graph_steps, args.steps)
    eager_ms = timed(eager_steps, args.steps)
    # the scan kernel alone, back to back inside one graph (nbuf launches per replay)
    reps = max(1, args.steps // nbuf)

    def scan_steps(n):
        with torch.cuda.stream(stream):
            for _ in range(n):
                g_scan.replay()

    scan_ms = timed(scan_steps, reps) / (reps * nbuf)
    gold = golden()["512x512x32"]["crc"]
    crc_ok = all(f"{zlib.crc32(o.cpu().numpy().tobytes()):08x}" == gold for o in outs[:2])

    e2e = None
    if args.e2e_steps > 0:
        pipe = pipeline.FramePipeline(1, wl.height, wl.width, spec, chunk=1)
        h_in = pipeline.pinned_empty((1, wl.height, wl.width), dtype=torch.uint8)
        h_in.copy_(torch.from_numpy(host[None]))
        h_out = pipeline.pinned_empty((1, wl.bins, wl.height, wl.width))
        n_e2e = max(args.e2e_steps, 20)
        for _ in range(3):
            pipe.run(h_in, h_out)
        barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            pipe.run(h_in, h_out)
        barrier()
        e2e_s = reduce_max([time.perf_counter() - t0])[0]
        crc_ok = crc_ok and f"{zlib.crc32(h_out.numpy().tobytes()):08x}" == gold
        e2e = {"value": world * n_e2e / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(pipe.h2d_bytes) * world,
               "d2h_bytes_per_step": int(pipe.d2h_bytes) * world, "steps": n_e2e,
               "timer": "host perf_counter around synchronized steps"}

    total_ms, eager_ms, scan_ms, bad = reduce_max([total_ms, eager_ms, scan_ms,
                                                   0.0 if crc_ok else 1.0])
    if rank != 0:
        return
    per_step = total_ms / args.steps
    value = world * args.steps / (total_ms / 1000.0)
    peak, peak_src = measured_peaks()
    alg = wl.alg_bytes
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": dict(config_block(wl, world), timing="CUDA-graph replay, 8 one-image calls "
                       f"per graph, {inflight} in flight on parallel branches; eager: the same "
                       "steps as plain API calls on one stream", inflight=inflight),
        "output_gbs": value * wl.out_bytes / 1e9,
        "hbm_frac_step": alg / (per_step / 1e3) / 1e9 / peak,
        "us_per_call_graph": 1000.0 * per_step,
        "eager": {"value": world * args.steps / (eager_ms / 1000.0), "unit": UNIT,
                  "us_per_call": 1000.0 * eager_ms / args.steps},
        "roofline": {"bound": "hbm", "kernel": "k2_scan", "achieved": alg / (scan_ms / 1e3) / 1e9,
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": alg / (scan_ms / 1e3) / 1e9 / peak, "traffic": None,
                     "alg_bytes_per_launch": alg, "launch_ms": scan_ms,
                     "launch_timer": "CUDA events around graphs of 8 back-to-back scan launches"},
        "gpu_launches": plan["launches"] * args.steps,
        "plan": plan,
        "parity": "output crc32 == reference golden 53891c64" if not bad else "MISMATCH",
        "clocks": clocks.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and args.cpu_baseline:
        v, cores, sample = cpu_sample(wl, budget_s=args.ref_budget)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if args.csv:
        write_csv(args.csv, line, wl)


def run_e2e(args, wl, spec, host, nloc, brange, out, dev, barrier, reduce_max, world):
    """Host buffers in, host buffers out, through pipeline.FramePipeline."""
    import torch

    from paper_1711_01919_b200 import pipeline

    b0, b1 = brange
    pipe = pipeline.FramePipeline(nloc, wl.height, wl.width, spec, chunk=args.chunk,
                                  bin_range=(b0, b1))
    h_in = pipeline.pinned_empty((nloc, wl.height, wl.width), dtype=torch.uint8)
    h_in.copy_(torch.from_numpy(host[:nloc]))
    h_out = pipeline.pinned_empty((nloc, b1 - b0, wl.height, wl.width))
    pipe.run(h_in, h_out)  # warm-up
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        pipe.run(h_in, h_out)
    barrier()
    e2e_s = reduce_max([time.perf_counter() - t0])[0]
    res = {"value": wl.frames * args.e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(pipe.h2d_bytes) * world,
           "d2h_bytes_per_step": int(pipe.d2h_bytes) * world,
           "steps": args.e2e_steps, "timer": "host perf_counter around synchronized steps"}
    res["_crc_ok"] = bool(torch.equal(h_out[0, 0].view(torch.int32),
                                      out[0, 0].view(torch.int32).cpu()))
    # the e2e roofline: a plain pinned D2H copy of one output slice (PCIe bound)
    probe = out[: min(nloc, 4)].view(torch.int32)
    dst = h_out[: probe.shape[0]].view(torch.int32)
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    for _ in range(3):
        dst.copy_(probe, non_blocking=True)
    torch.cuda.synchronize(dev)
    d2h_gbs = 3 * probe.numel() * 4 / (time.perf_counter() - t1) / 1e9
    res["d2h_copy_gbs"] = d2h_gbs
    res["e2e_out_gbs_per_gpu"] = pipe.d2h_bytes * args.e2e_steps / e2e_s / 1e9
    res["frac_of_d2h_copy"] = res["e2e_out_gbs_per_gpu"] / d2h_gbs
    del h_out, h_in, pipe
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hd64", choices=sorted(WORKLOADS))
    ap.add_argument("--frames", type=int, default=0, help="override histograms per step")
    ap.add_argument("--gather", action="store_true", help="time an NCCL gather of bin slabs")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=4, help="frames per pipelined e2e chunk")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--refine", type=int, default=4,
                    help="autotune candidates re-timed as pipelined steps (1: call ranking only)")
    ap.add_argument("--no-autotune", dest="autotune", action="store_false",
                    help="keep the planner's heuristic row-segment count")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false",
                    help="run each step's prepass and scan back to back on one stream")
    ap.add_argument("--ref-budget", type=float, default=10.0,
                    help="seconds of CPU work per reference sample (bounded)")
    ap.add_argument("--inflight", type=int, default=4,
                    help="cfg1: independent one-image calls in flight (graph branches)")
    ap.add_argument("--share-of", type=int, default=0,
                    help="time rank 0's share of an N-GPU run on this single GPU (per-GPU share "
                         "evidence when only one GPU exists; not the job metric)")
    ap.add_argument("--csv", default="",
                    help="also append the run to this CSV (reference schema + roofline columns)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / partition / max-over-ranks plumbing only (no GPU work; "
                         "CPU tests of the N>1 path)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    wl = WORKLOADS[args.workload]
    if args.frames:  # sizing experiments, e.g. the per-GPU share of an N-GPU run
        wl = Workload(wl.key, wl.width, wl.height, wl.bins, args.frames, wl.shard,
                      wl.desc + f" [frames overridden: {args.frames}]")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1 and args.impl == "ours":
        # `--gpus N` without a launcher: start N ranks ourselves (the driver's
        # torchrun form sets WORLD_SIZE and lands in the branch below)
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if launched and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; they must agree",
              file=sys.stderr)
        sys.exit(2)
    if args.share_of and (world > 1 or args.share_of < 1 or wl.key == "512"):
        print("bench.py: --share-of emulates one rank's share of a frame- or bin-sharded "
              "workload on a single process", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return
    backend = os.environ.get("IH_BENCH_BACKEND", "nccl")  # gloo: 1-GPU / CPU path tests only
    if not args.dry_run:
        import torch

        ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if ndev < 1 or (backend == "nccl" and ndev < world):
            print(f"bench.py: {world} rank(s) need {world} CUDA device(s), {ndev} visible "
                  f"(one process per GPU; no CPU fallback)", file=sys.stderr)
            sys.exit(3)
    if world > 1:
        import torch
        import torch.distributed as dist

        if backend == "nccl" and not args.dry_run:
            dev_index = local_rank % torch.cuda.device_count()
            torch.cuda.set_device(dev_index)
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            if not args.dry_run:
                torch.cuda.set_device(local_rank % torch.cuda.device_count())
            dist.init_process_group("gloo")
    try:
        if args.dry_run:
            run_dry(args, wl, rank, world)
        elif wl.key == "512":
            run_small(args, wl, rank, world, local_rank)
        else:
            run_ours(args, wl, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


def self_launch(args) -> int:
    """Re-run this command under torch.distributed.run with --gpus ranks (one
    process per GPU, rendezvous on 127.0.0.1); returns the launcher's exit code."""
    import socket
    import subprocess

    if not args.dry_run and os.environ.get("IH_BENCH_BACKEND", "nccl") == "nccl":
        import torch

        ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if ndev < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {ndev} visible",
                  file=sys.stderr)
            return 3
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


if __name__ == "__main__":
    main()
