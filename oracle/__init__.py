"""CPU oracle for the Scanner (arXiv 1805.07339) HIST / shot-diff / downsample path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product package ``paper_1805_07339_b200`` never imports it and
shares no code with it (the only shared module is the input generator
``scn_synth``).

Thin ctypes wrapper over ``libscn_oracle.so`` (plain single-threaded C,
``oracle/scn_oracle.c``); every function there cites the PAPER.md passage it
follows. Pins: ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

import scn_synth

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libscn_oracle.so")
_lib = None

OK, EINVAL, ERANGE, EUNSUPPORTED = 0, 1, 2, 4


class OracleError(Exception):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what}: status {code}")
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        L = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.oracle_sample_stride.argtypes = [ctypes.c_int64, ctypes.c_int64, i64p, ctypes.c_int64, i64p]
        L.oracle_sample_range.argtypes = [ctypes.c_int64, i64p, ctypes.c_int64, ctypes.c_int64, i64p,
                                          ctypes.c_int64, i64p]
        L.oracle_sample_gather.argtypes = [ctypes.c_int64, i64p, ctypes.c_int64, i64p, ctypes.c_int64, i64p]
        L.oracle_hist.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.oracle_hist_joint.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_void_p]
        L.oracle_run_joint.argtypes = [ctypes.POINTER(scn_synth.SynthSpecC), ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
        L.oracle_shotdiff_joint.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                            ctypes.c_void_p]
        L.oracle_shotdiff.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                      ctypes.c_void_p]
        L.oracle_downsample.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.oracle_run.argtypes = [ctypes.POINTER(scn_synth.SynthSpecC), ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_hist_diff_frames.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_required_rows.argtypes = [i64p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, i64p, ctypes.c_int64,
                                            i64p]
        L.oracle_stencil_then_sample.argtypes = [ctypes.POINTER(scn_synth.SynthSpecC), ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                                 ctypes.c_int32, ctypes.c_void_p]
        L.oracle_adaptive_cuts.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                           ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        L.oracle_shot_starts.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, i64p,
                                         ctypes.c_int64, i64p]
        L.oracle_montage.argtypes = [ctypes.POINTER(scn_synth.SynthSpecC), ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _sample(fn, *args) -> np.ndarray:
    m = ctypes.c_int64(0)
    rc = fn(*args, None, 0, ctypes.byref(m))
    if rc:
        raise OracleError(rc, fn.__name__)
    out = np.zeros(max(m.value, 1), dtype=np.int64)
    rc = fn(*args, _i64p(out), m.value, ctypes.byref(m))
    if rc:
        raise OracleError(rc, fn.__name__)
    return out[: m.value]


def sample_stride(n_rows: int, stride: int) -> np.ndarray:
    """P:L208 stride sampling (reading Q8: from row 0)."""
    return _sample(lib().oracle_sample_stride, n_rows, stride)


def sample_range(n_rows: int, blocks, step: int = 1) -> np.ndarray:
    """P:L208/P:L306 range sampling over half-open blocks [a, b) (reading Q9)."""
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.int64).reshape(-1, 2))
    return _sample(lib().oracle_sample_range, n_rows, _i64p(b), b.shape[0], step)


def sample_gather(n_rows: int, rows) -> np.ndarray:
    """P:L208 index-list sampling, strictly increasing (reading Q10)."""
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    return _sample(lib().oracle_sample_gather, n_rows, _i64p(r), r.shape[0])


def hist(frame: np.ndarray, bins: int = 16) -> np.ndarray:
    """P:L331 per-channel colour histogram of one HWC RGB8 frame -> uint32 [3, bins]."""
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w, c = f.shape
    assert c == 3
    out = np.zeros((3, bins), dtype=np.uint32)
    rc = lib().oracle_hist(_ptr(f), w, h, bins, _ptr(out))
    if rc:
        raise OracleError(rc, "hist")
    return out


def hist_joint(frame: np.ndarray, j: int = 4) -> np.ndarray:
    """NEXT N4 joint-colour histogram of one HWC RGB8 frame -> uint32 [J^3],
    k = bin(R)*J*J + bin(G)*J + bin(B), bin(v) = floor(v*J/256)."""
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w, c = f.shape
    assert c == 3
    out = np.zeros(j ** 3, dtype=np.uint32)
    rc = lib().oracle_hist_joint(_ptr(f), w, h, j, _ptr(out))
    if rc:
        raise OracleError(rc, "hist_joint")
    return out


def run_joint(spec: "scn_synth.Spec", videos, rows, p0: int, p1: int, j: int = 4) -> np.ndarray:
    """Joint-colour histograms of the synthetic frames at sampled positions [p0, p1) -> [n, J^3]."""
    v = np.ascontiguousarray(videos, dtype=np.int32)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    n = p1 - p0
    out = np.zeros((max(n, 1), j ** 3), dtype=np.uint32)
    rc = lib().oracle_run_joint(ctypes.byref(spec.c), _ptr(v), _ptr(r), p0, p1, j, _ptr(out))
    if rc:
        raise OracleError(rc, "run_joint")
    return out[:n]


def shotdiff_joint(hists: np.ndarray, seg_start=None) -> np.ndarray:
    """[-1,0] L1 difference of joint-colour histograms [M, J^3] -> uint32 [M] (0 at segment starts)."""
    hh = np.ascontiguousarray(hists, dtype=np.uint32)
    m, k = hh.shape
    j = round(k ** (1 / 3))
    assert j ** 3 == k
    seg = np.zeros(max(m, 1), dtype=np.uint8)
    if seg_start is not None:
        seg[:m] = np.asarray(seg_start, dtype=np.uint8)
    if m:
        seg[0] = 1
    out = np.zeros(max(m, 1), dtype=np.uint32)
    rc = lib().oracle_shotdiff_joint(_ptr(hh), _ptr(seg), m, j, _ptr(out))
    if rc:
        raise OracleError(rc, "shotdiff_joint")
    return out[:m]


def run_joint_diff(spec: "scn_synth.Spec", videos, rows, seg_start, p0: int, p1: int, j: int = 4):
    """Joint-colour histograms and their [-1,0] shot-diff for positions [p0, p1); position p0's
    stencil neighbour p0-1 (the halo) is included when p0 is not a segment start."""
    seg = np.asarray(seg_start, dtype=np.uint8)
    lo = p0 - 1 if (0 < p0 < len(seg) and not seg[p0]) else p0
    H = run_joint(spec, videos, rows, lo, p1, j)
    D = shotdiff_joint(H, seg[lo:p1])
    return H[p0 - lo:], D[p0 - lo:]


def shotdiff(hists: np.ndarray, seg_start=None) -> np.ndarray:
    """P:L210 + P:L455: [-1,0] stencil L1 histogram difference -> uint32 [M]."""
    hh = np.ascontiguousarray(hists, dtype=np.uint32)
    m = hh.shape[0]
    bins = hh.shape[-1]
    hh = hh.reshape(m, 3 * bins)
    seg = np.zeros(max(m, 1), dtype=np.uint8)
    if seg_start is not None:
        seg[:m] = np.asarray(seg_start, dtype=np.uint8)
    if m:
        seg[0] = 1
    out = np.zeros(max(m, 1), dtype=np.uint32)
    rc = lib().oracle_shotdiff(_ptr(hh), _ptr(seg), m, bins, _ptr(out))
    if rc:
        raise OracleError(rc, "shotdiff")
    return out[:m]


def downsample(frame: np.ndarray) -> np.ndarray:
    """P:L183/P:L335 integer 2x box downsample (reading Q11) -> uint8 [H/2, W/2, 3]."""
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w, _ = f.shape
    out = np.zeros((h // 2, w // 2, 3), dtype=np.uint8)
    rc = lib().oracle_downsample(_ptr(f), w, h, _ptr(out))
    if rc:
        raise OracleError(rc, "downsample")
    return out


def run(spec: "scn_synth.Spec", videos, rows, seg_start, p0: int, p1: int, bins: int = 16,
        want_hist=True, want_diff=True, want_ds=False):
    """Whole-job oracle over synthetic frames for sampled positions [p0, p1).

    videos/rows: per-position (table, row) of the sampled sequence; seg_start:
    per-position first-of-segment flags. Returns (hist [n,3,bins], diff [n], ds [n,H/2,W/2,3]).
    """
    v = np.ascontiguousarray(videos, dtype=np.int32)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    s = np.ascontiguousarray(seg_start, dtype=np.uint8)
    n = p1 - p0
    H = np.zeros((max(n, 1), 3, bins), dtype=np.uint32) if want_hist else None
    D = np.zeros(max(n, 1), dtype=np.uint32) if want_diff else None
    DS = (np.zeros((max(n, 1), spec.height // 2, spec.width // 2, 3), dtype=np.uint8) if want_ds else None)
    rc = lib().oracle_run(ctypes.byref(spec.c), _ptr(v), _ptr(r), _ptr(s), p0, p1, bins,
                          _ptr(H) if H is not None else None, _ptr(D) if D is not None else None,
                          _ptr(DS) if DS is not None else None)
    if rc:
        raise OracleError(rc, "run")
    return (H[:n] if H is not None else None, D[:n] if D is not None else None,
            DS[:n] if DS is not None else None)


def hist_diff_frames(frames: np.ndarray, bins: int = 16, seg_first: bool = True):
    """HIST + shot-diff over pre-generated contiguous frames [n, H, W, 3] (the timed CPU baseline)."""
    f = np.ascontiguousarray(frames, dtype=np.uint8)
    n, h, w, _ = f.shape
    H = np.zeros((max(n, 1), 3, bins), dtype=np.uint32)
    D = np.zeros(max(n, 1), dtype=np.uint32)
    rc = lib().oracle_hist_diff_frames(_ptr(f), n, w, h, bins, int(seg_first), _ptr(H), _ptr(D))
    if rc:
        raise OracleError(rc, "hist_diff_frames")
    return H[:n], D[:n]


def required_rows(rows, offset: int, n_rows: int) -> np.ndarray:
    """NEXT N2: exact HIST input rows for table -> HIST -> [offset,0] stencil -> Sample(rows)."""
    r = np.ascontiguousarray(rows, dtype=np.int64)
    return _sample(lib().oracle_required_rows, _i64p(r) if len(r) else None, len(r), offset, n_rows)


def stencil_then_sample(spec, videos, rows, offset: int, n_rows: int, bins: int = 16) -> np.ndarray:
    """NEXT N2 (fig:sampling-e): D'[j] = L1(H(S_j), H(clamp(S_j + offset))) over original table rows."""
    v = np.ascontiguousarray(videos, dtype=np.int32)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros(max(len(r), 1), dtype=np.uint32)
    rc = lib().oracle_stencil_then_sample(ctypes.byref(spec.c), _ptr(v), _ptr(r), len(r), offset, n_rows, bins,
                                          _ptr(out))
    if rc:
        raise OracleError(rc, "stencil_then_sample")
    return out[: len(r)]


def adaptive_cuts(diff, seg_start, warmup: int, k_num: int, k_den: int, floor: int) -> np.ndarray:
    """NEXT N3: bounded-state adaptive cut detector with warmup W over D -> uint8 [m]."""
    d = np.ascontiguousarray(diff, dtype=np.uint32)
    s = np.ascontiguousarray(seg_start, dtype=np.uint8)
    out = np.zeros(max(len(d), 1), dtype=np.uint8)
    rc = lib().oracle_adaptive_cuts(_ptr(d), _ptr(s), len(d), warmup, k_num, k_den, floor, _ptr(out))
    if rc:
        raise OracleError(rc, "adaptive_cuts")
    return out[: len(d)]


def shot_starts(diff, seg_start, tau: int) -> np.ndarray:
    """NEXT N1: first position of every shot = {p : seg_start[p] or D[p] > tau} (reading Q5)."""
    d = np.ascontiguousarray(diff, dtype=np.uint32)
    s = np.ascontiguousarray(seg_start, dtype=np.uint8)
    return _sample(lib().oracle_shot_starts, _ptr(d), _ptr(s), len(d), tau)


def montage(spec, videos, rows, cols: int) -> np.ndarray:
    """NEXT N1: keyframes (video, row) downsampled 2x and tiled cols per canvas row -> uint8 canvas."""
    v = np.ascontiguousarray(videos, dtype=np.int32)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    k = len(r)
    oh, ow = spec.height // 2, spec.width // 2
    canvas = np.zeros((max(-(-k // cols), 1) * oh, cols * ow, 3), dtype=np.uint8)
    rc = lib().oracle_montage(ctypes.byref(spec.c), _ptr(v), _ptr(r), k, cols, _ptr(canvas))
    if rc:
        raise OracleError(rc, "montage")
    return canvas[: (-(-k // cols)) * oh]
