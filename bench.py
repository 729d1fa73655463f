#!/usr/bin/env python
"""Throughput of the B200-native Smol preprocessing hot path.

A "step" is one smol_preproc_run over one batch: every step of the hot path
(dequantize, scaled IDCT, upsample, colour, resize+crop, normalize, NCHW
store) for every image of the batch, in one fused kernel launch.  Default
workload: BASELINE.json configs[1] = c2, 256 ImageNet-shaped 500x375 4:2:0
images, full-scale decode, short side 256, centre crop 224, fp32 NCHW.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl smol|reference]

N > 1: launched by torchrun, one process per GPU; every rank processes its
own batch (images are independent; no data-path collective: weak scaling).
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "preprocessed images/sec"
UNIT = "images/s"
L2_BYTES = 126 * 2 ** 20


def _traffic(cfg_name: str, layout: str):
    """ncu DRAM bytes per launch of the fused kernel for this workload, from
    the committed capture summary (profiles/traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(f"{cfg_name}/{layout}")
        return None if t is None else float(t["read"] + t["write"])
    except Exception:
        return None


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()                       # wait for the sampler to be running
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.start = len(self.lines)           # samples before the timed region are dropped
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            # a timed region shorter than the sampling period still gets the
            # sample that closes it (clocks decay over >100 ms after work ends)
            t0 = time.time()
            while len(self.lines) <= self.start and time.time() - t0 < 0.2 and self.proc.poll() is None:
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "start", 0):]:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def _cpu_baseline(cfg, imgs, qt, budget_s: float, max_images: int):
    """The oracle as it stands, on this host's cores, over a bounded sample."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    oracle.build()
    po = oracle.params_from_config(cfg)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.run_image(po, imgs[0], qt)
    t1 = time.perf_counter() - t0
    n = int(max(1, min(max_images, round(budget_s * cores / max(t1, 1e-6)))))   # ~budget_s of CPU work
    sample = [imgs[i % len(imgs)] for i in range(n)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(lambda im: oracle.run_image(po, im, qt), sample))
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"{n} {cfg.name} images ({cfg.width}x{cfg.height}, cycling the batch), "
                      f"thread pool of {cores} over images, {dt:.1f} s wall",
            "seconds": dt}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm)."""
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    imgs, qt = synth.distinct_images(cfg, n_distinct=min(cfg.n, 16))
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    oracle.build()
    po = oracle.params_from_config(cfg)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.run_image(po, imgs[0], qt)
    t1 = time.perf_counter() - t0
    total_budget = 150.0                       # seconds for the whole K + W run
    per_step = total_budget / max(1, args.steps + args.warmup)
    n = int(max(1, min(cfg.n, per_step * cores / max(t1, 1e-6))))
    sample = [imgs[i % len(imgs)] for i in range(n)]
    ex = ThreadPoolExecutor(cores)
    for _ in range(args.warmup):
        list(ex.map(lambda im: oracle.run_image(po, im, qt), sample))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        list(ex.map(lambda im: oracle.run_image(po, im, qt), sample))
    dt = time.perf_counter() - t0
    ex.shutdown()
    value = n * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_name(cfg), "sample_per_step": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"{n} images of {cfg.name} per step, thread pool of {cores}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _eq4(args, plan, batches, reps, out, stream, nloc, t_pre):
    """Eq. 4 beside the measurement: T_exec of ResNet-50
    on this GPU (torchvision architecture, random init: no weights offline;
    fp16, channels_last, CUDA graph, the same batch), the measured pipelined
    throughput (preprocessing of batch k+1 on one stream overlapping the DNN
    on batch k on another, double-buffered), and the predictions of min()
    (Eq. 4), sum and exec-only with their errors."""
    import torch
    import torchvision
    from paper_2007_13005_b200 import throughput as tpm
    torch.backends.cudnn.benchmark = True
    model = torchvision.models.resnet50(weights=None).cuda().eval().half().to(memory_format=torch.channels_last)
    bufs = [out, torch.empty_like(out)]
    xs = [torch.empty(out.shape, device="cuda", dtype=torch.half).to(memory_format=torch.channels_last)
          for _ in range(2)]
    side = torch.cuda.Stream()
    graphs = []
    with torch.inference_mode():
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                model(xs[0].copy_(bufs[0]))
        torch.cuda.current_stream().wait_stream(side)
        for i in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                model(xs[i].copy_(bufs[i]))        # dtype/layout conversion is part of the DNN step
            graphs.append(g)
    torch.cuda.synchronize()
    k_exec = 20
    dnn = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(dnn):
        for k in range(3):
            graphs[k % 2].replay()
        e0.record(dnn)
        for k in range(k_exec):
            graphs[k % 2].replay()
        e1.record(dnn)
    torch.cuda.synchronize()
    t_exec = nloc * k_exec / (e0.elapsed_time(e1) / 1e3)
    # pipelined: preprocessing (stream `stream`) -> DNN (stream `dnn`), two buffers
    k_pipe = 20
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for f in free:
        f.record(dnn)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p0.record(stream)
    for k in range(k_pipe):
        b = k % 2
        stream.wait_event(free[b])
        plan.run(batches[k % reps], out=bufs[b], stream=stream)
        ready[b].record(stream)
        dnn.wait_event(ready[b])
        with torch.cuda.stream(dnn):
            graphs[b].replay()
        free[b].record(dnn)
    stream.wait_stream(dnn)
    p1.record(stream)
    torch.cuda.synchronize()
    t_pipe = nloc * k_pipe / (p0.elapsed_time(p1) / 1e3)
    return {"t_preproc": t_pre, "t_exec": t_exec, "pipelined_measured": t_pipe,
            "dnn": f"ResNet-50 (torchvision architecture, random init), fp16 channels_last, CUDA graph, "
                   f"batch {nloc}, incl. the NCHW->fp16 channels_last conversion of the preprocessed batch",
            "models": tpm.model_errors(t_pipe, t_pre, [t_exec]),
            "note": "Eq. 4 min() assumes the two stages run on disjoint resources (the paper's CPU "
                    "preprocessing + GPU DNN); here both share one B200, where the sum model applies"}


def _workload_name(cfg):
    out = "x".join(str(v) for v in (3,) + cfg.out_hw)
    return (f"{cfg.name}: {cfg.n} x {cfg.width}x{cfg.height} 4:2:0 JPEG coefficients (q{cfg.quality}), "
            f"decode scale 1/{cfg.scale_denom}, "
            + (f"resize short {cfg.resize_short}, crop {cfg.crop_w}x{cfg.crop_h}" if cfg.resize_mode == "short"
               else f"resize {cfg.resize_w}x{cfg.resize_h}")
            + f" -> {cfg.out_dtype} NCHW {out}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="smol", choices=["smol", "reference"])
    ap.add_argument("--replicas", type=int, default=0, help="rotating input replicas (0 = auto: > L2)")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--tile-rows", type=int, default=0)
    ap.add_argument("--eq4", action="store_true",
                    help="also measure ResNet-50 on this GPU and pipelined preprocessing+DNN (Eq. 4 report)")
    ap.add_argument("--batch", type=int, default=0, help="images per GPU (0 = the config's N)")
    ap.add_argument("--layout", default="dense", choices=["dense", "packed"],
                    help="coefficient block layout (packed: only the coefficients the scale uses)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2007_13005_b200 as smol

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    cfg = synth.CONFIGS[args.config]
    params = smol.params_from_config(cfg, tile_rows=args.tile_rows, layout=args.layout)
    # weak scaling: a global batch of cfg.n images per GPU, partitioned into
    # contiguous ROI-balanced ranges (one per rank); no data-path collective
    from paper_2007_13005_b200 import shard
    per_gpu = args.batch or cfg.n
    all_imgs, qt = synth.batch_images(cfg, n=per_gpu * world)
    lo, hi = shard.partition(shard.roi_weights(params, all_imgs), world)[rank]
    imgs = all_imgs[lo:hi]
    nloc = len(imgs)
    plan = smol.Plan(params, max(nloc, 1))
    arena_bytes = smol.batch_for(params, imgs[:1], qt).coef_bytes * len(imgs)
    reps = args.replicas or max(2, int(np.ceil(1.5 * L2_BYTES / max(arena_bytes, 1))) + 1)
    batches = [smol.batch_for(params, imgs, qt) for _ in range(reps)]
    out = plan.new_output(nloc)
    stream = torch.cuda.Stream()

    # algorithmic bytes per image: ROI coefficients + output tensor
    g = smol.geometry(params, cfg.width, cfg.height)
    out_bytes = 3 * g["OH"] * g["OW"] * (2 if cfg.out_dtype == "f16" else 4)
    alg_bytes_img = g["roi_coef_bytes"] + out_bytes
    alg_bytes_launch = alg_bytes_img * nloc

    def step(k, o=out):
        plan.run(batches[k % reps], out=o, stream=stream)

    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            step(k)
    torch.cuda.synchronize()

    # ---- timed region: K steps --------------------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for k in range(args.steps):
            step(k)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_max = shard.max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    value = len(all_imgs) * args.steps / (ms_max / 1e3)

    # ---- per-launch kernel duration (events bracket each launch) ------------
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 50))]
    for k, (a, b) in enumerate(evs):
        a.record(stream)
        step(k)
        b.record(stream)
    torch.cuda.synchronize()
    launch_ms = statistics.median(a.elapsed_time(b) for a, b in evs)

    # ---- end to end: pinned host inputs -> device -> result read ------------
    # Two public entry points: smol_preproc_run_compact (compact records, one
    # DMA + expand kernel; the headline e2e) and smol_preproc_run_host (dense
    # ROI block rows gathered over PCIe).  At scale 1/8 the packed DC plane is
    # already smaller than a compact record, so run_host is the e2e path there.
    res_host = torch.empty((1,) + tuple(out.shape[1:]), dtype=out.dtype, pin_memory=True)

    def e2e_time(host_batches):
        for k in range(6):
            plan.run(host_batches[k % 2], out=out, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.e2e_steps):
            plan.run(host_batches[k % 2], out=out, stream=stream)
            with torch.cuda.stream(stream):
                res_host.copy_(out[:1], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = shard.max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, device="cuda")
        return len(all_imgs) / (ms / 1e3)

    gather_value = e2e_time([smol.batch_for(params, imgs, qt, location="pinned") for _ in range(2)])
    gather_h2d = g["roi_coef_bytes"] * len(all_imgs)
    use_compact = cfg.scale_denom != 8
    if use_compact:
        cbs = [smol.CompactBatch(params, imgs, qt, location="pinned") for _ in range(2)]
        compact_value = e2e_time(cbs)
        compact_h2d = cbs[0].arena_bytes * world
    d2h = int(res_host.numel() * res_host.element_size()) * world
    if use_compact:
        e2e = {"value": compact_value, "unit": UNIT, "h2d_bytes_per_step": compact_h2d, "d2h_bytes_per_step": d2h,
               "path": "smol_preproc_run_compact: compact records (ROI blocks, nonzero used coefficients) "
                       "in pinned host memory -> one H2D DMA + expand kernel + fused kernel; D2H of one "
                       "image's output as the step's result read",
               "run_host": {"value": gather_value, "h2d_bytes_per_step": gather_h2d,
                            "path": "dense ROI block rows gathered from pinned host memory"}}
    else:
        e2e = {"value": gather_value, "unit": UNIT, "h2d_bytes_per_step": gather_h2d, "d2h_bytes_per_step": d2h,
               "path": "smol_preproc_run_host: ROI block rows of the packed DC plane gathered from pinned "
                       "host memory; D2H of one image's output as the step's result read"}

    if rank == 0:
        peak, peak_src = _peaks()
        achieved = alg_bytes_launch / (launch_ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.out_dtype if False else "f32",
            "data": "synthetic (seeded natural-image JPEG coefficients, synth/)",
            "config": {"workload": _workload_name(cfg), "batch_per_gpu": nloc,
                       "global_batch": len(all_imgs), "parallelism": f"image shards x{world}, no collective",
                       "l2": f"inputs larger than L2: {reps} rotating replicas of the "
                             f"{arena_bytes / 1e6:.0f} MB coefficient arena",
                       "alg_bytes_per_image": alg_bytes_img,
                       "roi_coef_bytes_per_image": g["roi_coef_bytes"],
                       "coef_stats": synth.coef_stats(imgs[:min(len(imgs), 64)]),
                       "tile_rows": plan.params.tile_rows, "coef_layout": args.layout},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(cfg.name, args.layout), "peak_source": peak_src,
                         "kernel": ("smol_thumb_kernel" if cfg.scale_denom == 8 and args.layout == "packed"
                                    else "smol_fused_kernel"), "launch_ms": launch_ms,
                         "alg_bytes_per_launch": alg_bytes_launch},
            "e2e": e2e,
            "gpu_launches": args.steps * plan.launches_per_run(),
        }
        line["dtype"] = "f32" if cfg.out_dtype == "f32" else "f16"
        c = clk.summary()
        if c:
            line["clocks"] = c
        if args.eq4 and world == 1:
            try:
                line["eq4"] = _eq4(args, plan, batches, reps, out, stream, nloc, value)
            except Exception as e:  # noqa: BLE001
                line["eq4"] = {"error": repr(e)}
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = _cpu_baseline(cfg, imgs[:64], qt, args.cpu_budget, 16 * cfg.n)
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    plan.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
