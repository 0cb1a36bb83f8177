"""Thin Python binding of libscn.so (include/scn.h): same names, argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module converts Python ints / numpy arrays / objects with ``data_ptr()``
(torch tensors) / ``cuda_stream`` (torch streams) to plain C arguments and
raises ``ScnError`` on a non-OK status. There is no fallback: importing fails
loudly if the library is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCN_LIB=tuning loads the measurement build (same kernels + SCN_* environment knobs, `make tuning`)
LIB_PATH = os.path.join(_HERE, "libscn_tuning.so" if os.environ.get("SCN_LIB") == "tuning" else "libscn.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {os.path.dirname(_HERE)}` "
                      "(no CPU fallback exists)")
_lib = ctypes.CDLL(LIB_PATH)

SCN_OK, SCN_EINVAL, SCN_ERANGE, SCN_ECUDA, SCN_EUNSUPPORTED = 0, 1, 2, 3, 4
SCN_MEM_DEVICE, SCN_MEM_HOST = 0, 1
SCN_OP_HIST, SCN_OP_SHOTDIFF, SCN_OP_DOWNSAMPLE = 1, 2, 4
SCN_HIST_LANE_PAIRS, SCN_HIST_MATCH, SCN_HIST_MATCH_PACKED = 0, 1, 2
STATUS_NAMES = {0: "SCN_OK", 1: "SCN_EINVAL", 2: "SCN_ERANGE", 3: "SCN_ECUDA", 4: "SCN_EUNSUPPORTED"}

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_sz = ctypes.c_size_t


class ScnBlock(ctypes.Structure):
    _fields_ = [("start", ctypes.c_int64), ("end", ctypes.c_int64)]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_pp = ctypes.POINTER(_vp)
_sig("scn_last_error", ctypes.c_char_p)
_sig("scn_version", ctypes.c_char_p)
_sig("scn_last_launch_count", _i32)
_sig("scn_set_hist_impl", ctypes.c_int, _i32)
_sig("scn_get_hist_impl", _i32)
_sig("scn_hist_variant", ctypes.c_char_p, _i32)
_sig("scn_table_create", ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _vp, _i64, _vp, _pp)
_sig("scn_table_destroy", None, _vp)
_sig("scn_table_rows", _i64, _vp)
_sig("scn_sample_stride", ctypes.c_int, _vp, _i64, _pp)
_sig("scn_sample_range", ctypes.c_int, _vp, _vp, _i64, _i64, _pp)
_sig("scn_sample_gather", ctypes.c_int, _vp, _vp, _i64, _pp)
_sig("scn_seq_concat", ctypes.c_int, _vp, _i32, _pp)
_sig("scn_seq_length", _i64, _vp)
_sig("scn_seq_rows", ctypes.c_int, _vp, _vp, _vp)
_sig("scn_seq_seg_starts", ctypes.c_int, _vp, _vp)
_sig("scn_shard_range", ctypes.c_int, _i64, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64))
_sig("scn_seq_needs_halo", _i32, _vp, _i64)
_sig("scn_seq_device_bytes", _sz, _vp)
_sig("scn_seq_upload", ctypes.c_int, _vp, _vp, _sz, _vp)
_sig("scn_seq_destroy", None, _vp)
_sig("scn_run_histogram", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp)
_sig("scn_run_histogram_joint", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp)
_sig("scn_run_hist_shotdiff_joint", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp)
_sig("scn_run_shotdiff", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp)
_sig("scn_run_hist_shotdiff", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp)
_sig("scn_run_downsample", ctypes.c_int, _vp, _i64, _i64, _vp, _vp)
_sig("scn_run_hist_downsample", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp, _vp)
_sig("scn_seq_stencil_required", ctypes.c_int, _vp, _i32, _pp, _vp, _vp)
_sig("scn_run_diff_pairs", ctypes.c_int, _vp, _vp, _vp, _i64, _i32, _vp, _vp)
_sig("scn_seq_warmup_begin", _i64, _vp, _i64, _i32)
_sig("scn_run_adaptive_cuts", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _u32, _u32, _u32, _vp, _vp)
_sig("scn_select_shot_starts", ctypes.c_int, _vp, _i64, _i64, _vp, _u32, _vp, _i64, ctypes.POINTER(_i64))
_sig("scn_seq_gather_positions", ctypes.c_int, _vp, _vp, _i64, _pp)
_sig("scn_run_montage", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _i64, _vp)
_sig("scn_run_hist_shotdiff_to", ctypes.c_int, _vp, _i64, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _vp)
_sig("scn_ipc_import", ctypes.c_int, _vp, _i64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64))
_sig("scn_ipc_release", ctypes.c_int, ctypes.c_uint64)
_sig("scn_run_pipeline_host", ctypes.c_int, _vp, _i64, _i64, _i32, _u32, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp)


class ScnError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(rc: int, fn: str) -> None:
    if rc != SCN_OK:
        raise ScnError(rc, fn, (_lib.scn_last_error() or b"").decode())


def _ptr(x) -> int | None:
    """Device/host address of x: int, None, torch tensor (data_ptr) or numpy array."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, np.ndarray):
        return int(x.ctypes.data)
    return int(x)


def _stream(s) -> int | None:
    if s is None:
        return None
    if hasattr(s, "cuda_stream"):
        return int(s.cuda_stream) or None
    return int(s) or None


def scn_last_error() -> str:
    return (_lib.scn_last_error() or b"").decode()


def scn_version() -> str:
    return _lib.scn_version().decode()


def scn_last_launch_count() -> int:
    return int(_lib.scn_last_launch_count())


def scn_set_hist_impl(impl: int) -> None:
    _check(_lib.scn_set_hist_impl(impl), "scn_set_hist_impl")


def scn_get_hist_impl() -> int:
    return int(_lib.scn_get_hist_impl())


def scn_hist_variant(bins: int) -> str:
    return _lib.scn_hist_variant(bins).decode()


def scn_table_create(num_rows, width, height, channels=3, where=SCN_MEM_DEVICE, base=None, frame_stride_bytes=0,
                     row_ptrs=None):
    rp = None
    if row_ptrs is not None:
        rp = np.ascontiguousarray(row_ptrs, dtype=np.uint64)
    out = _vp()
    rc = _lib.scn_table_create(num_rows, width, height, channels, where, _ptr(base), frame_stride_bytes,
                               None if rp is None else rp.ctypes.data, ctypes.byref(out))
    _check(rc, "scn_table_create")
    return out


def scn_table_destroy(t) -> None:
    _lib.scn_table_destroy(t)


def scn_table_rows(t) -> int:
    return int(_lib.scn_table_rows(t))


def scn_sample_stride(t, stride):
    out = _vp()
    _check(_lib.scn_sample_stride(t, stride, ctypes.byref(out)), "scn_sample_stride")
    return out


def scn_sample_range(t, blocks, step=1):
    arr = (ScnBlock * max(len(blocks), 1))(*[ScnBlock(int(a), int(b)) for a, b in blocks])
    out = _vp()
    _check(_lib.scn_sample_range(t, ctypes.cast(arr, _vp), len(blocks), step, ctypes.byref(out)), "scn_sample_range")
    return out


def scn_sample_gather(t, rows):
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = _vp()
    _check(_lib.scn_sample_gather(t, r.ctypes.data if len(r) else None, len(r), ctypes.byref(out)),
           "scn_sample_gather")
    return out


def scn_seq_concat(parts):
    arr = (_vp * max(len(parts), 1))(*[p.value if isinstance(p, _vp) else p for p in parts])
    out = _vp()
    _check(_lib.scn_seq_concat(ctypes.cast(arr, _vp), len(parts), ctypes.byref(out)), "scn_seq_concat")
    return out


def scn_seq_length(s) -> int:
    return int(_lib.scn_seq_length(s))


def scn_seq_rows(s):
    m = scn_seq_length(s)
    part = np.zeros(max(m, 1), dtype=np.int32)
    row = np.zeros(max(m, 1), dtype=np.int64)
    _check(_lib.scn_seq_rows(s, part.ctypes.data, row.ctypes.data), "scn_seq_rows")
    return part[:m], row[:m]


def scn_seq_seg_starts(s):
    m = scn_seq_length(s)
    f = np.zeros(max(m, 1), dtype=np.uint8)
    _check(_lib.scn_seq_seg_starts(s, f.ctypes.data), "scn_seq_seg_starts")
    return f[:m]


def scn_shard_range(m, world, rank):
    b, e = _i64(), _i64()
    _check(_lib.scn_shard_range(m, world, rank, ctypes.byref(b), ctypes.byref(e)), "scn_shard_range")
    return b.value, e.value


def scn_seq_needs_halo(s, begin) -> int:
    return int(_lib.scn_seq_needs_halo(s, begin))


def scn_seq_device_bytes(s) -> int:
    return int(_lib.scn_seq_device_bytes(s))


def scn_seq_upload(s, d_workspace, nbytes, stream=None) -> None:
    _check(_lib.scn_seq_upload(s, _ptr(d_workspace), nbytes, _stream(stream)), "scn_seq_upload")


def scn_seq_destroy(s) -> None:
    _lib.scn_seq_destroy(s)


def scn_run_histogram(s, begin, end, bins, d_hist, stream=None) -> None:
    _check(_lib.scn_run_histogram(s, begin, end, bins, _ptr(d_hist), _stream(stream)), "scn_run_histogram")


def scn_run_histogram_joint(s, begin, end, bins_per_channel, d_hist, stream=None) -> None:
    _check(_lib.scn_run_histogram_joint(s, begin, end, bins_per_channel, _ptr(d_hist), _stream(stream)),
           "scn_run_histogram_joint")


def scn_run_hist_shotdiff_joint(s, begin, end, bins_per_channel, d_hist, d_diff, d_scratch=None, stream=None) -> None:
    _check(_lib.scn_run_hist_shotdiff_joint(s, begin, end, bins_per_channel, _ptr(d_hist), _ptr(d_diff),
                                            _ptr(d_scratch), _stream(stream)), "scn_run_hist_shotdiff_joint")


def scn_run_shotdiff(s, begin, end, bins, d_hist, d_diff, d_scratch=None, stream=None) -> None:
    _check(_lib.scn_run_shotdiff(s, begin, end, bins, _ptr(d_hist), _ptr(d_diff), _ptr(d_scratch), _stream(stream)),
           "scn_run_shotdiff")


def scn_run_hist_shotdiff(s, begin, end, bins, d_hist, d_diff, d_scratch=None, stream=None) -> None:
    _check(_lib.scn_run_hist_shotdiff(s, begin, end, bins, _ptr(d_hist), _ptr(d_diff), _ptr(d_scratch),
                                      _stream(stream)), "scn_run_hist_shotdiff")


def scn_run_downsample(s, begin, end, d_out, stream=None) -> None:
    _check(_lib.scn_run_downsample(s, begin, end, _ptr(d_out), _stream(stream)), "scn_run_downsample")


def scn_run_hist_downsample(s, begin, end, bins, d_hist, d_out, stream=None) -> None:
    _check(_lib.scn_run_hist_downsample(s, begin, end, bins, _ptr(d_hist), _ptr(d_out), _stream(stream)),
           "scn_run_hist_downsample")


def scn_run_pipeline_host(s, begin, end, bins, ops, d_hist, d_diff, d_out, d_scratch, d_staging, staging_bytes,
                          stream=None, copy_stream=None) -> None:
    _check(_lib.scn_run_pipeline_host(s, begin, end, bins, ops, _ptr(d_hist), _ptr(d_diff), _ptr(d_out),
                                      _ptr(d_scratch), _ptr(d_staging), staging_bytes, _stream(stream),
                                      _stream(copy_stream)), "scn_run_pipeline_host")


def scn_seq_stencil_required(s, offset):
    """NEXT N2: returns (required_seq, pos[M], nbr[M]) for table -> HIST -> [offset,0] stencil -> Sample."""
    m = scn_seq_length(s)
    pos = np.zeros(max(m, 1), dtype=np.int64)
    nbr = np.zeros(max(m, 1), dtype=np.int64)
    out = _vp()
    _check(_lib.scn_seq_stencil_required(s, offset, ctypes.byref(out), pos.ctypes.data, nbr.ctypes.data),
           "scn_seq_stencil_required")
    return out, pos[:m], nbr[:m]


def scn_run_diff_pairs(d_hist, d_a, d_b, n, bins, d_diff, stream=None) -> None:
    _check(_lib.scn_run_diff_pairs(_ptr(d_hist), _ptr(d_a), _ptr(d_b), n, bins, _ptr(d_diff), _stream(stream)),
           "scn_run_diff_pairs")


def scn_seq_warmup_begin(s, begin, warmup) -> int:
    return int(_lib.scn_seq_warmup_begin(s, begin, warmup))


def scn_run_adaptive_cuts(s, begin, end, warmup, d_diff, k_num, k_den, floor, d_cut, stream=None) -> None:
    _check(_lib.scn_run_adaptive_cuts(s, begin, end, warmup, _ptr(d_diff), k_num, k_den, floor, _ptr(d_cut),
                                      _stream(stream)), "scn_run_adaptive_cuts")


def scn_select_shot_starts(s, begin, end, h_diff, tau) -> np.ndarray:
    """NEXT N1: positions in [begin,end) that start a shot (segment start or D > tau)."""
    d = np.ascontiguousarray(h_diff, dtype=np.uint32)
    if end > begin and len(d) < end - begin:
        raise ValueError(f"h_diff holds {len(d)} values, the range [{begin},{end}) needs {end - begin}")
    cnt = _i64()
    _check(_lib.scn_select_shot_starts(s, begin, end, d.ctypes.data, tau, None, 0, ctypes.byref(cnt)),
           "scn_select_shot_starts")
    out = np.zeros(max(cnt.value, 1), dtype=np.int64)
    _check(_lib.scn_select_shot_starts(s, begin, end, d.ctypes.data, tau, out.ctypes.data, cnt.value,
                                       ctypes.byref(cnt)), "scn_select_shot_starts")
    return out[: cnt.value]


def scn_seq_gather_positions(s, positions):
    p = np.ascontiguousarray(positions, dtype=np.int64)
    out = _vp()
    _check(_lib.scn_seq_gather_positions(s, p.ctypes.data if len(p) else None, len(p), ctypes.byref(out)),
           "scn_seq_gather_positions")
    return out


def scn_run_montage(s, begin, end, cols, d_canvas, canvas_pitch, stream=None) -> None:
    _check(_lib.scn_run_montage(s, begin, end, cols, _ptr(d_canvas), canvas_pitch, _stream(stream)),
           "scn_run_montage")


def scn_run_hist_shotdiff_to(s, begin, end, bins, hist_dests, diff_dests, self_index, d_scratch=None,
                             stream=None) -> None:
    """HIST + shot-diff writing rows [begin,end) straight into every rank's result columns."""
    h = np.ascontiguousarray(hist_dests, dtype=np.uint64)
    d = np.ascontiguousarray(diff_dests, dtype=np.uint64)
    if len(h) != len(d):
        raise ValueError(f"{len(h)} histogram destinations but {len(d)} diff destinations")
    _check(_lib.scn_run_hist_shotdiff_to(s, begin, end, bins, h.ctypes.data, d.ctypes.data, len(h), self_index,
                                         _ptr(d_scratch), _stream(stream)), "scn_run_hist_shotdiff_to")


def scn_ipc_import(handle: bytes, offset: int):
    """Map a peer's IPC-exported allocation on the current device -> (base, ptr)."""
    hb = ctypes.create_string_buffer(bytes(handle), 64)
    base, ptr = ctypes.c_uint64(), ctypes.c_uint64()
    _check(_lib.scn_ipc_import(hb, offset, ctypes.byref(base), ctypes.byref(ptr)), "scn_ipc_import")
    return base.value, ptr.value


def scn_ipc_release(base: int) -> None:
    _check(_lib.scn_ipc_release(base), "scn_ipc_release")


__all__ = [n for n in dir() if n.startswith(("scn_", "SCN_"))] + ["ScnError", "ScnBlock", "LIB_PATH"]
