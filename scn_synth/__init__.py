"""Seeded synthetic input generator shared by the CUDA path's tests/bench and the oracle.

INPUT ONLY: frames (RGB8 HWC), shot structure, gather index lists and the
workload presets C1-C5 (BASELINE.json ``configs``). It holds none of the
method's arithmetic (no sampling, histogram, difference or downsample).
The C implementation lives in ``scn_synth.h`` / ``synth_host.c`` (host) and
``synth_cuda.cu`` (device fill), so host and device bytes are identical.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST = os.path.join(_HERE, "libscn_synth_host.so")
_CUDA = os.path.join(_HERE, "libscn_synth_cuda.so")

SHOTS, UNIFORM, CONSTANT, XGRAD = 0, 1, 2, 3
MODES = {"shots": SHOTS, "uniform": UNIFORM, "constant": CONSTANT, "xgrad": XGRAD}
DEFAULT_SEED = 180507339


class SynthSpecC(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint32),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("n_cuts", ctypes.c_int32),
        ("cuts", ctypes.POINTER(ctypes.c_int64)),
        ("len_min", ctypes.c_int32),
        ("len_max", ctypes.c_int32),
        ("shared_scene", ctypes.c_int32),
        ("n_videos_scene", ctypes.c_int32),
    ]


class FrameDescC(ctypes.Structure):
    _fields_ = [
        ("video", ctypes.c_int32),
        ("shot", ctypes.c_int32),
        ("t", ctypes.c_int32),
        ("x_offset", ctypes.c_int32),
        ("row", ctypes.c_int64),
    ]


_host = None
_cuda = None


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(_HOST):
            raise RuntimeError(f"{_HOST} missing: run `make -C {os.path.dirname(_HERE)}`")
        L = ctypes.CDLL(_HOST)
        L.synth_describe.restype = FrameDescC
        L.synth_describe.argtypes = [ctypes.POINTER(SynthSpecC), ctypes.c_int32, ctypes.c_int64]
        L.synth_cut_rows.restype = ctypes.c_int64
        L.synth_cut_rows.argtypes = [ctypes.POINTER(SynthSpecC), ctypes.c_int32, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]
        L.synth_fill_frame_host.argtypes = [ctypes.POINTER(SynthSpecC), ctypes.POINTER(FrameDescC),
                                            ctypes.c_void_p]
        L.synth_gather_rows.restype = ctypes.c_int
        L.synth_gather_rows.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.POINTER(ctypes.c_int64)]
        _host = L
    return _host


def cuda_lib():
    global _cuda
    if _cuda is None:
        if not os.path.exists(_CUDA):
            raise RuntimeError(f"{_CUDA} missing: run `make -C {os.path.dirname(_HERE)}`")
        L = ctypes.CDLL(_CUDA)
        L.synth_job_bytes.restype = ctypes.c_size_t
        L.synth_fill_frames_device.restype = ctypes.c_int
        L.synth_fill_frames_device.argtypes = [ctypes.POINTER(SynthSpecC), ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _cuda = L
    return _cuda


class Spec:
    """Content spec of one video family (all tables of a config share it)."""

    def __init__(self, width, height, mode="shots", seed=DEFAULT_SEED, cuts=None, len_min=48, len_max=240,
                 shared_scene=False, n_videos_scene=1):
        self.width, self.height = int(width), int(height)
        self.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        self._cuts = None if cuts is None else np.ascontiguousarray(sorted(cuts), dtype=np.int64)
        self.c = SynthSpecC(
            seed=seed & 0xFFFFFFFF, width=self.width, height=self.height, mode=self.mode,
            n_cuts=-1 if cuts is None else len(self._cuts),
            cuts=(self._cuts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if cuts is not None and len(cuts)
                  else None),
            len_min=len_min, len_max=len_max, shared_scene=int(bool(shared_scene)),
            n_videos_scene=int(n_videos_scene))

    @property
    def frame_bytes(self) -> int:
        return self.width * self.height * 3

    def frame(self, video: int, row: int) -> np.ndarray:
        """Host copy of frame `row` of table `video` as uint8 [H, W, 3]."""
        L = host_lib()
        d = L.synth_describe(ctypes.byref(self.c), video, row)
        out = np.empty((self.height, self.width, 3), dtype=np.uint8)
        L.synth_fill_frame_host(ctypes.byref(self.c), ctypes.byref(d), out.ctypes.data_as(ctypes.c_void_p))
        return out

    def describe(self, video: int, row: int):
        d = host_lib().synth_describe(ctypes.byref(self.c), video, row)
        return {"video": d.video, "shot": d.shot, "t": d.t, "x_offset": d.x_offset, "row": d.row}

    def cut_rows(self, video: int, num_rows: int) -> np.ndarray:
        L = host_lib()
        n = L.synth_cut_rows(ctypes.byref(self.c), video, num_rows, None, 0)
        out = np.zeros(max(n, 1), dtype=np.int64)
        L.synth_cut_rows(ctypes.byref(self.c), video, num_rows, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                         n)
        return out[:n]

    def fill_device(self, videos, rows, dst_ptrs, jobs_ptr: int, stream_ptr: int = 0) -> None:
        """Fill frames on the device: dst_ptrs[i] <- frame rows[i] of table videos[i].

        jobs_ptr: device scratch of len(rows) * job_bytes() bytes (caller-owned)."""
        v = np.ascontiguousarray(videos, dtype=np.int32)
        r = np.ascontiguousarray(rows, dtype=np.int64)
        d = np.ascontiguousarray(dst_ptrs, dtype=np.uint64)
        rc = cuda_lib().synth_fill_frames_device(ctypes.byref(self.c), v.ctypes.data_as(ctypes.c_void_p),
                                                 r.ctypes.data_as(ctypes.c_void_p), d.ctypes.data_as(ctypes.c_void_p),
                                                 len(r), ctypes.c_void_p(jobs_ptr), ctypes.c_void_p(stream_ptr))
        if rc:
            raise RuntimeError(f"synth_fill_frames_device failed: cudaError {rc}")


def job_bytes() -> int:
    return int(cuda_lib().synth_job_bytes())


def gather_rows(seed: int, n: int, k: int) -> np.ndarray:
    """k distinct rows of [0, n), Floyd's algorithm on splitmix64(seed), sorted (reading Q10)."""
    out = np.zeros(max(k, 1), dtype=np.int64)
    rc = host_lib().synth_gather_rows(seed & 0xFFFFFFFFFFFFFFFF, n, k,
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc:
        raise ValueError(f"gather_rows({n}, {k}) failed")
    return out[:k]


# ---------------------------------------------------------------------------
# Workload presets = BASELINE.json "configs"
# ---------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    width: int
    height: int
    n_videos: int
    rows_per_video: int
    sampling: tuple            # ("stride", s) | ("range", blocks, step) | ("gather", seed, k)
    ops: tuple                 # subset of ("hist", "shotdiff", "downsample")
    bins: int = 16
    spec_kw: dict = field(default_factory=dict)

    def spec(self, mode: str | None = None, seed: int = DEFAULT_SEED) -> Spec:
        kw = dict(self.spec_kw)
        if mode is not None:
            kw["mode"] = mode
        return Spec(self.width, self.height, seed=seed, **kw)

    @property
    def frame_bytes(self) -> int:
        return self.width * self.height * 3

    def weak(self, g: int) -> "Workload":
        """The config's input g times over, for weak scaling on g GPUs: one video grows to
        g x its rows (a gather draws g x as many rows), several videos become g x as many
        videos. Contiguous shards of the result hold exactly one config's worth each."""
        import dataclasses
        if g <= 1:
            return self
        if self.n_videos == 1:
            smp = self.sampling
            if smp[0] == "gather":
                smp = (smp[0], smp[1], smp[2] * g)
            return dataclasses.replace(self, name=f"{self.name} x{g} (weak)", rows_per_video=self.rows_per_video * g,
                                       sampling=smp)
        return dataclasses.replace(self, name=f"{self.name} x{g} (weak)", n_videos=self.n_videos * g)


WORKLOADS = {
    "C1": Workload("C1-tiny-64x36-stride1-cuts", 64, 36, 1, 240, ("stride", 1), ("hist", "shotdiff"),
                   spec_kw={"cuts": [57, 131, 198]}),
    "C2": Workload("C2-film-1080p-16384f-stride1", 1920, 1080, 1, 16384, ("stride", 1), ("hist", "shotdiff"),
                   spec_kw={"len_min": 48, "len_max": 240}),
    "C3": Workload("C3-tvnews-640x360-2048x512-stride30", 640, 360, 2048, 512, ("stride", 30), ("hist",),
                   spec_kw={"len_min": 171, "len_max": 512}),
    "C4": Workload("C4-gather-1080p-4096of65536", 1920, 1080, 1, 65536, ("gather", 1805, 4096),
                   ("hist", "downsample"), spec_kw={"len_min": 48, "len_max": 240}),
    "C5": Workload("C5-vr-4k-14x1024-range", 3840, 2160, 14, 1024,
                   ("range", [(128 * k, 128 * k + 64) for k in range(8)], 1), ("downsample", "hist"),
                   spec_kw={"len_min": 48, "len_max": 240, "shared_scene": True, "n_videos_scene": 14}),
}
