#!/usr/bin/env python3
"""Benchmark of the Scanner (arXiv 1805.07339) HIST + shot-diff hot path on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` (torchrun for
N > 1) prints ONE JSON line on rank 0. A step is one pass of the whole hot path
(sample -> per-channel histogram -> [-1,0] shot-diff, + NCCL all-gather of the
result columns when N > 1) over the BASELINE config C2 (1920x1080 RGB8,
16,384 frames, Stride 1), frames already resident in HBM, captured once per rank
as a CUDA graph and replayed. Strong scaling by default: at N GPUs the 16,384
frames are split contiguously (2,048 per GPU at N = 8, each shard with its
recomputed 1-frame halo, BASELINE "frames sharded with 1-frame halo");
`--scaling weak` runs the config N times over instead. `--impl reference` times
the CPU oracle (the reference arm for this tier) instead.
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

METRIC = "sampled frames/sec (histogram+shotdiff) at 1/2/4/8 B200; % of HBM peak GB/s"
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--mode", default="shots", help="synthetic content: shots|uniform|constant|xgrad")
    ap.add_argument("--frames", type=int, default=0,
                    help="limit positions (debug; 0 = the whole config; per GPU under weak scaling)")
    ap.add_argument("--e2e-frames", type=int, default=1024, help="positions per e2e step from pinned host memory")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU-baseline budget (oracle, rank 0, N=1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-frames-per-step", type=int, default=64)
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only to exercise N>1 on one GPU")
    ap.add_argument("--round-frames", type=int, default=0,
                    help="process a rank's shard in rounds of this many positions (input + output > HBM, e.g. C5 "
                         "at N = 1); generation between rounds is untimed, timed steps are summed over rounds")
    ap.add_argument("--gather", default="auto", choices=["auto", "nccl", "p2p"],
                    help="N > 1 result exchange: p2p = fused into the histogram / shot-diff kernels over peer "
                         "memory (scn_run_hist_shotdiff_to); nccl = one NCCL all_gather of the result block; "
                         "auto (default) = p2p for the hist + shot-diff step (NCCL if a rank cannot map its "
                         "peers), nccl for the other ops")
    ap.add_argument("--cuts", type=int, default=0,
                    help="NEXT N3: add the bounded-state adaptive cut detector with warmup W to the step")
    ap.add_argument("--bins", type=int, default=0, help="override the config's bins per channel (NEXT N4: 256)")
    ap.add_argument("--montage", type=int, default=0,
                    help="NEXT N1: time the two-job shot montage with this many tiles per canvas row (N = 1)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong (default) = the config itself split contiguously over N GPUs (BASELINE C2: "
                         "16,384 frames sharded with 1-frame halo); weak = each GPU processes one config's worth "
                         "(the config's input N times over)")
    ap.add_argument("--shape", default="", help="override the config's frame size, WxH (e.g. 1366x768)")
    ap.add_argument("--no-graph", action="store_true", help="launch each step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--force-graph", action="store_true",
                    help="try graph capture even with gloo (test of the capture-failure fallback)")
    ap.add_argument("--joint", type=int, default=0,
                    help="NEXT N4 joint-colour histogram with J bins per channel (J^3 bins) instead of the "
                         "config's ops (N = 1)")
    ap.add_argument("--hist-impl", type=int, default=0,
                    help="scn_set_hist_impl: 0 lane-private pair keys (default), 1 K2a match per byte, 2 K2a' packed")
    ap.add_argument("--graph", default="f", choices=["f", "e"],
                    help="f: sample -> hist -> [-1,0] (default); e: hist -> [-1,0] -> sample (NEXT N2, N = 1)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def stop(self, window=None):
        """Clock statistics over the samples taken inside `window` = (t0, t1) wall seconds (the
        timed region; all samples if the region was too short to catch one)."""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        picked = [p for t, p in self.samples if window is None or window[0] <= t <= window[1] + 0.15]
        in_window = bool(picked) and window is not None
        if not picked:
            picked = [p for _, p in self.samples]
        for s in picked:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
            except ValueError:
                continue
            for i, n in enumerate(names):
                if s[3 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "timed region" if in_window else "whole sampling run (timed region shorter than a sample)"}


def traffic_from_profile(frames: int, F: int, kernel: str, lib_version: str):
    """dram bytes per launch from a committed ncu --set full summary of this kernel at this
    frame size (profiles/ncu_<kernel>[_<tag>]_summary.json; bytes/frame x frames), the
    summary's source, and whether the capture's git SHA is the library's (scn_version)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_{kernel}*_summary.json"))):
        d = json.load(open(p))
        bpf = d.get("dram_bytes_per_frame")
        if bpf and d.get("frame_bytes") == F and d.get("kernel") == kernel:
            sha = d.get("git_sha")
            match = bool(sha) and sha[:12] in lib_version
            if not match:
                print(f"warning: {os.path.basename(p)} was captured at {sha} but the library is {lib_version}",
                      file=sys.stderr)
            return float(bpf) * frames, {"source": d.get("source", p), "summary": os.path.relpath(p, ROOT),
                                         "capture_sha": sha, "matches_library": match}
    return None, None


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------
def host_frames(wl, positions, plan_):
    import scn_synth
    spec = wl.spec()
    part, row, _ = plan_
    out = np.empty((len(positions), wl.height, wl.width, 3), dtype=np.uint8)
    for i, p in enumerate(positions):
        out[i] = spec.frame(int(part[p]), int(row[p]))
    return out


def oracle_plan(wl):
    import oracle
    import scn_synth
    vids, rows, seg = [], [], []
    for v in range(wl.n_videos):
        k = wl.sampling[0]
        if k == "stride":
            r = oracle.sample_stride(wl.rows_per_video, wl.sampling[1])
        elif k == "range":
            r = oracle.sample_range(wl.rows_per_video, wl.sampling[1], wl.sampling[2])
        else:
            r = oracle.sample_gather(wl.rows_per_video,
                                     scn_synth.gather_rows(wl.sampling[1], wl.rows_per_video, wl.sampling[2]))
        vids += [v] * len(r)
        rows += r.tolist()
        seg += [1] + [0] * (len(r) - 1) if len(r) else []
    return np.array(vids, np.int32), np.array(rows, np.int64), np.array(seg, np.uint8)


def time_oracle(frames: np.ndarray, bins: int, budget_s: float):
    import oracle
    n_done, t_used = 0, 0.0
    while t_used < budget_s:
        t0 = time.perf_counter()
        oracle.hist_diff_frames(frames, bins)
        t_used += time.perf_counter() - t0
        n_done += len(frames)
    return n_done, t_used


def time_oracle_all_cores(frames: np.ndarray, bins: int, budget_s: float, threads: int):
    """The unmodified single-threaded oracle run as `threads` independent instances over
    disjoint frames (ctypes releases the GIL), wall-clock timed: frames/s on all host cores."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    per = max(1, len(frames) // threads)
    chunks = [frames[(i * per) % len(frames):(i * per) % len(frames) + per] for i in range(threads)]
    done = [0] * threads
    stop = time.perf_counter() + budget_s

    def work(i):
        while time.perf_counter() < stop:
            oracle.hist_diff_frames(chunks[i], bins)
            done[i] += len(chunks[i])

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return sum(done), time.perf_counter() - t0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import scn_synth
    import oracle  # noqa: F401  (reference arm = the CPU oracle, as it stands)
    wl = scn_synth.WORKLOADS[args.config]
    plan_ = oracle_plan(wl)  # the oracle's own sampling: no product code on the reference arm
    n = max(1, args.ref_frames_per_step)
    frames = host_frames(wl, list(range(n)), plan_)
    import oracle as _o
    from concurrent.futures import ThreadPoolExecutor
    threads = min(os.cpu_count() or 1, n)
    parts = np.array_split(np.arange(n), threads)

    def one_step(pool):  # the step's frames split over `threads` independent oracle instances
        list(pool.map(lambda idx: _o.hist_diff_frames(frames[idx[0]:idx[-1] + 1], wl.bins), parts))

    with ThreadPoolExecutor(threads) as pool:
        for _ in range(args.warmup):
            one_step(pool)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(pool)
        dt = time.perf_counter() - t0
    fps = n * args.steps / dt
    sample = (f"positions 0..{n - 1} of {args.config} ({wl.width}x{wl.height}) per step, frames generated on the host "
              f"(untimed), split over {threads} independent instances of the single-threaded C oracle")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": wl.name, "frames_per_step": n, "bins": wl.bins, "ops": "hist+shotdiff"},
        "cpu_baseline": {"value": fps, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_graph_e(args):
    """NEXT N2 (fig:sampling-e): HIST over the exact required set R = S U (S-1), then D'[j] from row pairs."""
    import torch

    import scn_harness
    import scn_synth
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    wl = scn_synth.WORKLOADS[args.config]
    st = torch.cuda.current_stream(dev)
    job = scn_harness.StencilJob(wl, -1, device=dev, stream=st, spec=wl.spec(mode=args.mode))
    out = job.alloc_outputs()
    for _ in range(max(args.warmup, 0)):
        job.run(out)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(st)
    for k in range(args.steps):
        ev[k][0].record(st)
        launches += job.run(out)
        ev[k][1].record(st)
    t1.record(st)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / args.steps
    peak, peak_src = load_peaks()
    alg = job.R * (wl.frame_bytes + 3 * wl.bins * 4)
    line = {"metric": METRIC, "value": job.M / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl.name + " graph e (hist -> [-1,0] -> sample)", "frames": job.M,
                       "required_frames": job.R, "bins": wl.bins, "ops": "hist(R)+diff_pairs"},
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                         "algorithmic_bytes_per_step": alg},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches}
    print(json.dumps(line), flush=True)
    job.close()
    return 0


def run_montage(args):
    """NEXT N1: job 1 (hist + shot-diff over the film) -> D to host -> shot starts -> job 2
    (gather keyframes, 2x downsample into a montage canvas). Timed end to end on the stream,
    host selection included."""
    import torch

    import scn_harness
    import scn_synth
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    wl = scn_synth.WORKLOADS[args.config]
    st = torch.cuda.current_stream(dev)
    pl = scn_harness.plan(wl)
    M = len(pl[1]) if args.frames <= 0 else min(args.frames, len(pl[1]))
    pl = tuple(x[:M] for x in pl)
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, device=dev, stream=st, plan_=pl,
                                spec=wl.spec(mode=args.mode))
    out = job.alloc_outputs(("hist", "shotdiff"), wl.bins)
    tau = wl.width * wl.height
    for _ in range(max(args.warmup, 1)):
        canvas, pos = scn_harness.shot_montage(job, args.montage, tau, out=out)
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        canvas, pos = scn_harness.shot_montage(job, args.montage, tau, out=out)
        b.record(st)
        torch.cuda.synchronize(dev)
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    line = {"metric": METRIC, "value": M / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl.name + " two-job shot montage (NEXT N1)", "frames": M,
                       "keyframes": int(len(pos)), "canvas": list(canvas.shape), "cols": args.montage,
                       "ops": "job1 hist+shotdiff -> D2H -> select -> job2 gather+downsample montage"},
            "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": None,
            "step_ms_min": min(ts)}
    print(json.dumps(line), flush=True)
    job.close()
    return 0


def run_joint(args):
    """NEXT N4, joint-colour variant: scn_run_hist_shotdiff_joint (J bins per channel, J^3 counters
    per frame, then the [-1,0] L1 shot-diff over them) over the config's sampled frames,
    device-resident, N = 1."""
    import torch

    import paper_1805_07339_b200 as scn
    import scn_harness
    import scn_synth
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    wl = _apply_shape(scn_synth.WORKLOADS[args.config], args)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    pl = scn_harness.plan(wl)
    M = len(pl[1]) if args.frames <= 0 else min(args.frames, len(pl[1]))
    pl = tuple(x[:M] for x in pl)
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=False, device=dev, stream=st, plan_=pl,
                                spec=wl.spec(mode=args.mode))
    J = args.joint
    out = torch.empty((max(M, 1), J ** 3), dtype=torch.int32, device=dev)
    diff = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
    scratch = torch.empty(J ** 3, dtype=torch.int32, device=dev)

    def step():
        scn.scn_run_hist_shotdiff_joint(job.seq, 0, M, J, out, diff, scratch, st)

    for _ in range(max(args.warmup, 0)):
        step()
    launches = scn.scn_last_launch_count()
    torch.cuda.synchronize(dev)
    props = torch.cuda.get_device_properties(dev)
    clocks = ClockSampler(f"GPU-{props.uuid}" if getattr(props, "uuid", None) else "0")
    clocks.start()
    time.sleep(0.3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    w0 = time.time()
    ev[0].record(st)
    for k in range(args.steps):
        step()
        ev[k + 1].record(st)
    torch.cuda.synchronize(dev)
    clk = clocks.stop((w0, time.time()))
    ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    step_ms = float(np.mean(ms))
    peak, peak_src = load_peaks()
    # histogram: frame read + row write; shot-diff: two row reads + D write (SURVEY §8(d) per frame)
    alg = M * (wl.frame_bytes + J ** 3 * 4 * 3 + 4)
    ach = alg / (step_ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": M / (step_ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl.name + f" joint-colour histogram J={J} (NEXT N4)", "frames": M,
                       "width": wl.width, "height": wl.height, "joint_bins": J ** 3, "content": args.mode,
                       "ops": "hist_joint+shotdiff_joint", "l2": "no flush: input %.1f GB >> 126 MB L2" % (M * wl.frame_bytes / 1e9)},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": None, "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
                         "kernel": "hist_tma_kernel<7,16> + shotdiff_kernel (whole step incl. memset)",
                         **stream_ceiling(False, ach)},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches * args.steps, "clocks": clk,
            "step_ms_min": float(min(ms)), "library": scn.scn_version()}
    print(json.dumps(line), flush=True)
    job.close()
    return 0


def run_rounds(args):
    """SURVEY §8(d) residency: a shard larger than HBM is processed in rounds (the paper's I/O
    packets). Each round materialises its positions (untimed), then W warm-up + K timed
    steps run over that round; a step of the whole job = the sum of the rounds' step times."""
    import torch

    import paper_1805_07339_b200 as scn
    import scn_harness
    import scn_synth
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    wl = scn_synth.WORKLOADS[args.config]
    st = torch.cuda.current_stream(dev)
    pl = scn_harness.plan(wl)
    M = len(pl[1]) if args.frames <= 0 else min(args.frames, len(pl[1]))
    pl = tuple(x[:M] for x in pl)
    K = args.round_frames
    do_ds, do_diff = "downsample" in wl.ops, "shotdiff" in wl.ops
    ops = tuple(o for o in ("hist", "shotdiff", "downsample") if o == "hist" or o in wl.ops)
    round_ms, hist_ms, buf, launches = [], [], None, 0
    for r0 in range(0, M, K):
        r1 = min(M, r0 + K)
        job = scn_harness.DeviceJob(wl, r0, r1, with_halo=True, device=dev, stream=st, plan_=pl, buf=buf,
                                    spec=wl.spec(mode=args.mode))
        buf = job.buf
        out = job.alloc_outputs(ops, wl.bins)

        def step(ev=None):
            nonlocal launches
            if ev is not None:
                ev[0].record(st)
            if do_ds:
                scn.scn_run_hist_downsample(job.seq, r0, r1, wl.bins, out["hist"], out["ds"], st)
            else:
                scn.scn_run_histogram(job.seq, r0, r1, wl.bins, out["hist"], st)
            launches += scn.scn_last_launch_count() if ev is not None else 0
            if ev is not None:
                ev[1].record(st)
            if do_diff:
                scn.scn_run_shotdiff(job.seq, r0, r1, wl.bins, out["hist"], out["diff"], out["scratch"], st)
                launches += scn.scn_last_launch_count() if ev is not None else 0

        for _ in range(max(args.warmup, 0)):
            step()
        torch.cuda.synchronize(dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for k in range(args.steps):
            step(evs[k])
        b_.record(st)
        torch.cuda.synchronize(dev)
        round_ms.append(a.elapsed_time(b_) / args.steps)
        hist_ms.append(float(np.mean([x.elapsed_time(y) for x, y in evs])))
        job.close()
        del out
    ms = sum(round_ms)
    peak, peak_src = load_peaks()
    F = wl.frame_bytes
    ds_b = (wl.width // 2) * (wl.height // 2) * 3 if do_ds else 0
    alg = M * (F + 3 * wl.bins * 4 + ds_b)
    ach = alg / (sum(hist_ms) / 1e3) / 1e9
    line = {"metric": METRIC, "value": M / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl.name, "frames": M, "rounds": len(round_ms), "round_frames": K,
                       "ops": "+".join(ops), "round_ms": round_ms,
                       "l2": "no flush: inputs per round >> 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": None, "peak_source": peak_src, "algorithmic_bytes_per_step": alg},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches}
    print(json.dumps(line), flush=True)
    return 0


def _apply_shape(wl, args):
    import dataclasses
    if args.bins:
        wl = dataclasses.replace(wl, bins=args.bins)
    if args.shape:
        w, h = (int(x) for x in args.shape.lower().split("x"))
        wl = dataclasses.replace(wl, name=f"{wl.name} @{w}x{h}", width=w, height=h)
    return wl


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1805_07339_b200 as scn
    import scn_harness
    import scn_synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus={args.gpus}; using WORLD_SIZE", file=sys.stderr)
    dev_index = local % max(torch.cuda.device_count(), 1)  # == local on a multi-GPU box
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if args.dist_backend == "nccl":
            # NCCL's INIT log names the communicator size ("nranks N"), so a run's rank count is checkable
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout for the JSON line
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    scn.scn_set_hist_impl(args.hist_impl)

    wl = scn_synth.WORKLOADS[args.config]
    if args.scaling == "weak":
        wl = wl.weak(world)  # per-GPU work fixed at one config as N grows
    wl = _apply_shape(wl, args)
    plan_ = scn_harness.plan(wl)
    # --frames limits one config's worth (per GPU under weak scaling)
    lim = args.frames * (world if args.scaling == "weak" else 1)
    M = len(plan_[1]) if args.frames <= 0 else min(lim, len(plan_[1]))
    plan_ = (plan_[0][:M], plan_[1][:M], plan_[2][:M])
    b, e = scn.scn_shard_range(M, world, rank)
    n = e - b
    bins = wl.bins
    # one non-default stream for everything (CUDA graphs cannot capture the legacy stream);
    # made current so torch's collectives and graph replays are ordered on it too
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    cut_w = args.cuts
    jb = b
    if cut_w > 0:  # NEXT N3: the shard starts W positions early (warmup), computed and discarded
        meta = scn_harness._build_seq(wl)
        jb = scn.scn_seq_warmup_begin(meta, b, cut_w)
        scn.scn_seq_destroy(meta)
    job = scn_harness.DeviceJob(wl, jb, e, with_halo=True, spec=wl.spec(mode=args.mode), device=dev, stream=stream,
                                plan_=plan_)
    d_cut = torch.empty(max(n, 1), dtype=torch.uint8, device=dev) if cut_w > 0 else None
    do_diff, do_ds = "shotdiff" in wl.ops, "downsample" in wl.ops
    ops = tuple(o for o in ("hist", "shotdiff", "downsample") if o == "hist" or o in wl.ops)
    out = job.alloc_outputs(ops, bins)
    fusable = do_diff and not do_ds and not cut_w  # the step scn_run_hist_shotdiff_to covers
    if args.gather == "p2p" and not fusable:
        raise SystemExit("--gather p2p covers the hist + shot-diff step only")
    p2p = world > 1 and (args.gather == "p2p" or (args.gather == "auto" and fusable))
    gather_note = None
    peer = None
    if p2p:  # the fused peer-memory gather, or NCCL if any rank cannot map its peers' columns
        err = None
        try:
            peer = scn_harness.PeerColumns(M, bins, dist, dev)
        except Exception as ex:  # noqa: BLE001 (reported in the JSON line)
            err = f"{type(ex).__name__}: {ex}"[:200]
        bad = torch.tensor([0.0 if err is None else 1.0], dtype=torch.float64, device=dev)
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if float(bad[0]):
            if peer is not None:
                peer.close(barrier=False)
            dist.barrier()  # every rank, mapped or not, before the columns are dropped
            peer, p2p = None, False
            gather_note = "p2p unavailable, fell back to NCCL all_gather: " + (err or "failed on another rank")
    gather = scn_harness.ColumnGather(M, world, bins, dev, dist) if world > 1 and peer is None else None
    if gather is not None and jb == b:  # the kernels write straight into the all-gather's send block
        out["hist"] = gather.hist
        if do_diff:
            out["diff"] = gather.diff
    launches = [0]

    def compute():
        if peer is not None:  # HIST + shot-diff writing this rank's rows into every rank's columns
            scn.scn_run_hist_shotdiff_to(job.seq, b, e, bins, peer.hist_ptrs, peer.diff_ptrs, rank, out["scratch"],
                                         stream)
            launches[0] += scn.scn_last_launch_count()
            return
        if do_ds:  # HIST + 2x downsample in one read of each frame (reading Q12)
            scn.scn_run_hist_downsample(job.seq, jb, e, bins, out["hist"], out["ds"], stream)
            launches[0] += scn.scn_last_launch_count()
            if do_diff:
                scn.scn_run_shotdiff(job.seq, jb, e, bins, out["hist"], out["diff"], out["scratch"], stream)
                launches[0] += scn.scn_last_launch_count()
        elif do_diff:  # the shard's halo frame rides in the same histogram launch
            scn.scn_run_hist_shotdiff(job.seq, jb, e, bins, out["hist"], out["diff"], out["scratch"], stream)
            launches[0] += scn.scn_last_launch_count()
        else:
            scn.scn_run_histogram(job.seq, jb, e, bins, out["hist"], stream)
            launches[0] += scn.scn_last_launch_count()
        if cut_w > 0:
            scn.scn_run_adaptive_cuts(job.seq, b, e, cut_w, out["diff"], 4, 1, wl.width * wl.height // 8, d_cut,
                                      stream)
            launches[0] += scn.scn_last_launch_count()

    def exchange():
        if gather is not None:
            gather.gather(out["hist"][b - jb:], out["diff"][b - jb:] if do_diff else None, n)

    def step():
        compute()
        exchange()

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    # One CUDA graph per rank for the step (memset + histogram + shot-diff + all-gather), and
    # two more for the breakdown (compute only, exchange only). gloo collectives run on the
    # host and cannot be captured, so a gloo run (N > 1 ranks sharing one GPU) stays eager.
    # (the fused peer gather has no collective in the step, so it captures under any backend)
    use_graph = not args.no_graph and (world == 1 or args.dist_backend == "nccl" or peer is not None or
                                       args.force_graph)
    graphs, per_step_launches, graph_note = {}, 0, None
    if use_graph:
        try:
            for name, fn in (("step", step), ("compute", compute), ("exchange", exchange)):
                if name == "exchange" and gather is None:
                    continue
                g = torch.cuda.CUDAGraph()
                launches[0] = 0
                # thread_local: only this thread's unsafe calls abort the capture (NCCL's
                # watchdog thread keeps polling its events while we capture)
                with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
                    fn()
                graphs[name] = g
                if name == "step":
                    per_step_launches = launches[0]
            torch.cuda.synchronize(dev)
        except Exception as ex:  # noqa: BLE001 (reported; the step then launches eagerly)
            graph_note = f"graph capture failed, eager launches: {type(ex).__name__}: {ex}"[:200]
            graphs.clear()
            torch.cuda.synchronize(dev)
        if world > 1:  # every rank takes the same path
            ok = torch.tensor([0.0 if graphs else 1.0], dtype=torch.float64, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MAX)
            if float(ok[0]):
                graphs.clear()
                graph_note = graph_note or "graph capture failed on another rank, eager launches"
        use_graph = bool(graphs)
    run = {k: (lambda g=g: g.replay()) for k, g in graphs.items()} if use_graph else \
        {"step": step, "compute": compute, "exchange": exchange}
    if use_graph:
        run["step"]()  # warm replay
        torch.cuda.synchronize(dev)
    launches[0] = 0

    def timed(fn, steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev[0].record(stream)
        for k in range(steps):
            fn()
            ev[k + 1].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]

    props = torch.cuda.get_device_properties(dev)
    gpu_id = f"GPU-{props.uuid}" if getattr(props, "uuid", None) else str(dev_index)
    clocks = ClockSampler(gpu_id)
    clocks.start()
    time.sleep(0.3)  # let nvidia-smi start sampling before the timed region
    w0 = time.time()
    step_ms = timed(run["step"], args.steps)  # the timed region: barrier + sync on both sides
    clk = clocks.stop((w0, time.time()))
    gpu_launches = per_step_launches * args.steps if use_graph else launches[0]
    total_ms = float(sum(step_ms))
    # breakdown (after the timed region): the compute and the exchange alone, same K
    comp_ms = timed(run["compute"], args.steps)
    exch_ms = timed(run["exchange"], args.steps) if gather is not None else [0.0]
    mine = [total_ms / args.steps, float(np.mean(comp_ms)), float(np.mean(exch_ms)), float(min(step_ms)),
            float(statistics.median(step_ms))]
    per_rank = [mine]
    if world > 1:
        allr = torch.zeros((world, len(mine)), dtype=torch.float64, device=dev)
        allr[rank] = torch.tensor(mine, dtype=torch.float64, device=dev)
        dist.all_reduce(allr)  # each rank fills its own row
        per_rank = allr.cpu().tolist()
    ms_per_step = max(r[0] for r in per_rank)  # max over ranks
    hist_ms_max = max(r[1] for r in per_rank)

    # ---- end-to-end through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, wl, plan_, M, world, rank, dev, stream, ops, bins, do_diff, do_ds)

    # ---- CPU baseline: the oracle as it stands, rank 0, N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nfr = 16
            # the oracle's input comes from the host generator (scn_synth), never from the GPU
            frames = host_frames(wl, list(range(b, b + nfr)), plan_)
            n1, t1s = time_oracle(frames, bins, max(2.0, args.cpu_seconds / 3))
            threads = os.cpu_count() or 1
            ndone, tused = time_oracle_all_cores(frames, bins, args.cpu_seconds, threads)
            cpu = {"value": ndone / tused, "unit": UNIT, "cores": threads, "kind": "oracle",
                   "single_core_value": n1 / t1s,
                   "sample": f"positions {b}..{b + nfr - 1} of {args.config} ({wl.width}x{wl.height}), frames "
                             f"generated on the host (untimed); {threads} independent instances of the "
                             f"single-threaded C oracle over disjoint frames, {ndone} frames in {tused:.1f} s wall; "
                             f"one instance alone {n1 / t1s:.1f} frames/s"}
        except Exception as ex:  # noqa: BLE001 (reported in the JSON line, the GPU numbers still print)
            cpu = {"value": None, "kind": "oracle", "error": f"{type(ex).__name__}: {ex}"[:300]}

    if world > 1:
        dist.barrier()
    if rank == 0:
        peak, peak_src = load_peaks()
        F = wl.frame_bytes
        ds_b = (wl.width // 2) * (wl.height // 2) * 3 if do_ds else 0
        halo = job.p0 - job.lo  # the recomputed [-1,0] halo frame of this shard (0 or 1)
        # read each frame once (+ the halo), write counts (+ ds); the timed call also
        # runs the shot-diff (reads 2 rows, writes 4 B per position) when it is fused in
        diff_b = (e - jb) * (2 * 3 * bins * 4 + 4) if (do_diff and not do_ds) else 0
        alg_bytes = (e - jb + halo) * F + (e - jb) * (3 * bins * 4 + ds_b) + diff_b
        # the dominant call's average duration: at N = 1 the timed step IS that call (memset +
        # histogram + shot-diff, replayed from the graph inside the timed region); at N > 1 the
        # step also holds the exchange, so rank 0's compute-alone breakdown over the same K
        launch_ms = per_rank[0][0] if world == 1 else per_rank[0][1]
        achieved = alg_bytes / (launch_ms / 1e3) / 1e9
        traffic, tsrc = traffic_from_profile(n, F, "histds" if do_ds else "hist", scn.scn_version())
        comp = [r[1] for r in per_rank]
        line = {
            "metric": METRIC, "value": M / (ms_per_step / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl.name, "frames": M, "frames_per_gpu": n, "width": wl.width, "height": wl.height,
                       "bins": bins,
                       "sampling": str(wl.sampling[:2] if wl.sampling[0] != "range" else ("range", len(wl.sampling[1]), wl.sampling[2])),
                       "ops": "+".join(ops) + (f"+adaptive_cuts(W={cut_w})" if cut_w else "") +
                              (("+fused_peer_gather" if p2p else "+nccl_allgather") if world > 1 else ""),
                       "content": args.mode, "parallelism": f"dp{world} contiguous shards + 1-frame halo",
                       "hist_variant": scn.scn_hist_variant(bins),
                       "step_launch": "cuda_graph_replay" if use_graph else "eager",
                       "l2": "no flush: per-GPU input %.1f GB >> 126 MB L2" % (n * F / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("hist_tma_kernel<2,8> fused hist+downsample (scn_run_hist_downsample incl. memset)"
                                    if do_ds else "hist_tma_kernel<0,16> + shotdiff_kernel (scn_run_hist_shotdiff "
                                    "incl. memset)" if do_diff else "hist_tma_kernel<0,16> (scn_run_histogram)"),
                         "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": launch_ms,
                         "peak_source": peak_src, "traffic_source": tsrc,
                         # also against the nominal ~8 TB/s, and the second roofline
                         # (shared-atomic throughput of K2) next to its K0-measured capacity
                         "peak_nominal": NOMINAL_HBM_GBPS, "frac_nominal": achieved / NOMINAL_HBM_GBPS,
                         # the measured stream ceiling for this kernel's read:write mix on a B200
                         **stream_ceiling(do_ds, achieved),
                         "shared_atomics": atomic_roofline(bins, (e - jb + halo) * F, hist_ms_max, clk)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clk,
            "step_ms_min": min(r[3] for r in per_rank), "step_ms_median": max(r[4] for r in per_rank),
            # per-rank breakdown (ms per step): the step, its compute alone (memset + histogram +
            # shot-diff), the exchange alone (all-gather), and the fixed cost step - compute
            "breakdown": {"step_ms": [r[0] for r in per_rank], "compute_ms": comp,
                          "gather_ms": [r[2] for r in per_rank],
                          "overhead_ms": [r[0] - r[1] for r in per_rank],
                          "barrier_skew_ms": max(comp) - min(comp)},
            "library": scn.scn_version(),
        }
        if gather_note:
            line["config"]["gather_note"] = gather_note
        if graph_note:
            line["config"]["graph_note"] = graph_note
    graphs.clear()
    job.close()
    if peer is not None:
        peer.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:  # last, after teardown: NCCL's INIT log (stdout) cannot follow the JSON line
        print(json.dumps(line), flush=True)
    return 0


def run_e2e(args, wl, plan_, M, world, rank, dev, stream, ops, bins, do_diff, do_ds):
    """The same metric end to end through scn_run_pipeline_host: each step copies its frames
    from pinned host memory (H2D inside the timed region) and reads the result columns back
    (D2H). A failure on any rank (e.g. pinned-memory exhaustion on an unfamiliar box) is
    reported in the line instead of aborting the run; every rank still joins each
    collective, so a local failure cannot hang the others."""
    import torch
    import torch.distributed as dist

    import paper_1805_07339_b200 as scn
    import scn_harness

    def agree(ok: bool) -> bool:  # all ranks succeeded?
        if world == 1:
            return ok
        f = torch.tensor([0.0 if ok else 1.0], dtype=torch.float64, device=dev)
        dist.all_reduce(f, op=dist.ReduceOp.MAX)
        return float(f[0]) == 0.0

    ne = min(args.e2e_frames * (world if args.scaling == "weak" else 1), M)
    eb, ee = scn.scn_shard_range(ne, world, rank)
    err, hj = None, None
    try:
        hj = scn_harness.HostJob(wl, eb, ee, with_halo=True, device=dev, plan_=plan_, staging_frames=48)
        ne_r = max(ee - eb, 1)
        eo = {"hist": torch.empty((ne_r, 3, bins), dtype=torch.int32, device=dev),
              "diff": torch.empty(ne_r, dtype=torch.int32, device=dev),
              "scratch": torch.empty(3 * bins, dtype=torch.int32, device=dev)}
        if do_ds:
            eo["ds"] = torch.empty((ne_r, wl.height // 2, wl.width // 2, 3), dtype=torch.uint8, device=dev)
        h_out = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in eo.items()
                 if k == "hist" or (k == "diff" and do_diff) or (k == "ds" and do_ds)}
        cs = torch.cuda.Stream(dev)

        def e2e_step():
            hj.run(eo, ops, bins, stream=stream, copy_stream=cs)
            for k, hv in h_out.items():
                hv.copy_(eo[k], non_blocking=True)

        for _ in range(max(args.warmup, 1)):
            e2e_step()
        torch.cuda.synchronize(dev)
    except Exception as ex:  # noqa: BLE001 (reported in the JSON line)
        err = f"{type(ex).__name__}: {ex}"[:300]
    if not agree(err is None):
        if hj is not None:
            hj.close()
        return {"value": None, "unit": UNIT, "error": err or "failed on another rank"}
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ksteps = max(1, min(args.steps, 10))
    e0.record(stream)
    for _ in range(ksteps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    d2h_r = sum(v.numel() * v.element_size() for v in h_out.values())
    te = torch.tensor([e0.elapsed_time(e1), float(d2h_r)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = te.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(te, op=dist.ReduceOp.SUM)
        te[0] = tmax[0]
    hj.close()
    e2e_ms = float(te[0]) / ksteps
    h2d = ne * wl.frame_bytes  # whole job: every rank's frames (each rank copies its shard)
    return {"value": ne / (e2e_ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(te[1]),
            "positions_per_step": ne, "ms_per_step": e2e_ms,
            "h2d_GBps": h2d / (e2e_ms / 1e3) / 1e9,
            "h2d_ceiling_note": "raw pinned H2D on the GPU box measured 55.4-55.6 GB/s per GPU "
                                "(profiles/r01_h2d_ceiling.json)",
            "path": "scn_run_pipeline_host: pinned host frames -> double-buffered H2D (copy stream) -> "
                    "hist+shotdiff kernels -> D2H of the result columns"}



NOMINAL_HBM_GBPS = 8000.0  # B200 nominal HBM3e bandwidth (the north_star's "roughly 8 TB/s")
K0_ATOMS_ILP = 31.8  # conflict-free lane-private red.shared lane-ops / SM-clock (profiles/r01_k0_micro_v2.json)


# Measured HBM stream ceilings on a B200 (no compute): best TMA bulk read ring
# (profiles/r01_k0_micro_v2.json, tma_read_t16384_s6_w17) and TMA bulk load + bulk store
# at 4:1 read:write (profiles/r01_mix_ceiling.json, tma_r4w1_s4) — the mix of the fused
# hist + downsample kernel (F read, F/4 written per frame).
READ_CEILING_GBPS = 7565.8
R4W1_CEILING_GBPS = 7140.5


def stream_ceiling(do_ds, achieved):
    c, src = ((R4W1_CEILING_GBPS, "profiles/r01_mix_ceiling.json tma_r4w1_s4 (TMA load + store, 4:1)") if do_ds else
              (READ_CEILING_GBPS, "profiles/r01_k0_micro_v2.json tma_read_t16384_s6_w17 (TMA read ring)"))
    return {"stream_ceiling": c, "frac_stream_ceiling": achieved / c, "stream_ceiling_source": src}


def atomic_roofline(bins, in_bytes, ms, clk):
    """Shared-atomic side of the histogram: lane-ops per input byte are fixed by the design
    (0.5 with pair keys at B <= 16, 1 with one key per byte), so the achieved rate per SM-clock
    follows from the measured time and the median SM clock under load."""
    per_byte = 0.5 if bins in (1, 2, 4, 8, 16) else 1.0
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz")
    if not mhz or ms <= 0:
        return None
    rate = per_byte * in_bytes / (ms / 1e3) / (148 * mhz * 1e6)
    return {"lane_ops_per_input_byte": per_byte, "lane_ops_per_sm_clk": rate,
            "capacity_lane_ops_per_sm_clk": K0_ATOMS_ILP, "frac": rate / K0_ATOMS_ILP,
            "clock_mhz_used": mhz, "capacity_source": "profiles/r01_k0_micro_v2.json (atoms_ilp_lane_private)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.graph == "e":
        return run_graph_e(args)
    if args.montage > 0:
        return run_montage(args)
    if args.joint > 0:
        return run_joint(args)
    if args.round_frames > 0 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        return run_rounds(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
