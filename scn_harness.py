"""Harness shared by tests/, bench.py and __graft_entry__.smoke(): builds a
workload's tables and sampled sequence through the product's C ABI, allocates
device memory with torch, materialises only the sampled rows a shard needs
(the paper's sparse decode: "only a sparse set ... must be
computed"; here "decode" is the synthetic fill) and runs the hot path.

It contains no histogram / difference / downsample arithmetic: every compute
step goes through paper_1805_07339_b200 (libscn.so). The oracle is imported
only by the callers that are allowed to use it (tests, smoke, bench baseline).
"""
from __future__ import annotations

import os

import numpy as np
import torch

import paper_1805_07339_b200 as scn
import scn_synth

FAKE_BASE = 1 << 40  # placeholder (never dereferenced) for metadata-only planning tables


def ceil16(x: int) -> int:
    return (x + 15) & ~15


def _sample(t, sampling):
    kind = sampling[0]
    if kind == "stride":
        return scn.scn_sample_stride(t, sampling[1])
    if kind == "range":
        return scn.scn_sample_range(t, sampling[1], sampling[2])
    if kind == "gather":
        rows = scn_synth.gather_rows(sampling[1], scn.scn_table_rows(t), sampling[2])
        return scn.scn_sample_gather(t, rows)
    raise ValueError(kind)


def _build_seq(wl: scn_synth.Workload, row_ptrs_of=None, where=scn.SCN_MEM_DEVICE):
    """Create the per-video tables, sample each and concatenate.

    row_ptrs_of(video) -> uint64[N] row pointers (sparse) or None (placeholder dense)."""
    F16 = ceil16(wl.frame_bytes)
    parts, tables = [], []
    try:
        for v in range(wl.n_videos):
            if row_ptrs_of is None:
                t = scn.scn_table_create(wl.rows_per_video, wl.width, wl.height, 3, where, FAKE_BASE, F16)
            else:
                t = scn.scn_table_create(wl.rows_per_video, wl.width, wl.height, 3, where, None, 0, row_ptrs_of(v))
            tables.append(t)
            parts.append(_sample(t, wl.sampling))
        seq = scn.scn_seq_concat(parts) if len(parts) > 1 else parts.pop()
    finally:
        for p in parts:
            scn.scn_seq_destroy(p)
        for t in tables:
            scn.scn_table_destroy(t)
    return seq


def plan(wl: scn_synth.Workload):
    """Sampled positions of the whole job: (video[M], row[M], seg_start[M])."""
    seq = _build_seq(wl)
    try:
        part, row = scn.scn_seq_rows(seq)
        seg = scn.scn_seq_seg_starts(seq)
    finally:
        scn.scn_seq_destroy(seq)
    return part.astype(np.int32), row, seg


class DeviceJob:
    """Positions [p0, p1) of a workload (plus the [-1,0] halo when asked) resident in HBM."""

    def __init__(self, wl: scn_synth.Workload, p0: int, p1: int, with_halo: bool, spec: scn_synth.Spec | None = None,
                 device="cuda", stream=None, plan_=None, buf: torch.Tensor | None = None):
        self.wl = wl
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.part, self.row, self.seg = plan_ if plan_ is not None else plan(wl)
        self.M = len(self.row)
        self.p0, self.p1 = p0, p1
        halo = 1 if (with_halo and 0 < p0 < self.M and not self.seg[p0]) else 0
        self.lo = p0 - halo
        self.F = wl.frame_bytes
        self.F16 = ceil16(self.F)
        n_mat = p1 - self.lo
        need = max(n_mat, 1) * self.F16
        if buf is not None and buf.numel() >= need:
            self.buf = buf
        else:
            self.buf = torch.empty(need, dtype=torch.uint8, device=self.device)
        base = self.buf.data_ptr()
        addrs = base + np.arange(n_mat, dtype=np.uint64) * np.uint64(self.F16)
        self.spec = spec if spec is not None else wl.spec()
        if n_mat > 0:
            jobs = torch.empty(n_mat * scn_synth.job_bytes(), dtype=torch.uint8, device=self.device)
            with torch.cuda.stream(self.stream):
                self.spec.fill_device(self.part[self.lo:p1], self.row[self.lo:p1], addrs, jobs.data_ptr(),
                                      self.stream.cuda_stream)
            self.stream.synchronize()
            del jobs
        # sparse tables: only positions [lo, p1) resident
        ptrs = {}
        for j in range(self.lo, p1):
            v = int(self.part[j])
            if v not in ptrs:
                ptrs[v] = np.zeros(wl.rows_per_video, dtype=np.uint64)
            ptrs[v][int(self.row[j])] = addrs[j - self.lo]
        zeros = np.zeros(wl.rows_per_video, dtype=np.uint64)
        self.seq = _build_seq(wl, lambda v: ptrs.get(v, zeros))
        self.ws = torch.empty(max(scn.scn_seq_device_bytes(self.seq), 16), dtype=torch.uint8, device=self.device)
        scn.scn_seq_upload(self.seq, self.ws, self.ws.numel(), self.stream)
        self.stream.synchronize()

    def alloc_outputs(self, ops=("hist", "shotdiff"), bins=None):
        bins = bins or self.wl.bins
        n = self.p1 - self.p0
        out = {}
        if "hist" in ops:
            out["hist"] = torch.empty((max(n, 1), 3, bins), dtype=torch.int32, device=self.device)
        if "shotdiff" in ops:
            out["diff"] = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
            out["scratch"] = torch.empty(3 * bins, dtype=torch.int32, device=self.device)
        if "downsample" in ops:
            out["ds"] = torch.empty((max(n, 1), self.wl.height // 2, self.wl.width // 2, 3), dtype=torch.uint8,
                                    device=self.device)
        return out

    def run(self, out, ops=("hist", "shotdiff"), bins=None, fused=True, stream=None):
        """One pass of the hot path over [p0, p1) through the C ABI. Returns kernels launched."""
        bins = bins or self.wl.bins
        st = stream if stream is not None else self.stream
        s, b, e = self.seq, self.p0, self.p1
        launches = 0
        if "hist" in ops and "downsample" in ops and fused:
            scn.scn_run_hist_downsample(s, b, e, bins, out["hist"], out["ds"], st)
            launches += scn.scn_last_launch_count()
            if "shotdiff" in ops:
                scn.scn_run_shotdiff(s, b, e, bins, out["hist"], out["diff"], out["scratch"], st)
                launches += scn.scn_last_launch_count()
        elif "hist" in ops and "shotdiff" in ops and fused:
            scn.scn_run_hist_shotdiff(s, b, e, bins, out["hist"], out["diff"], out["scratch"], st)
            launches += scn.scn_last_launch_count()
        else:
            if "hist" in ops:
                scn.scn_run_histogram(s, b, e, bins, out["hist"], st)
                launches += scn.scn_last_launch_count()
            if "shotdiff" in ops:
                scn.scn_run_shotdiff(s, b, e, bins, out["hist"], out["diff"], out["scratch"], st)
                launches += scn.scn_last_launch_count()
            if "downsample" in ops:
                scn.scn_run_downsample(s, b, e, out["ds"], st)
                launches += scn.scn_last_launch_count()
        return launches

    def close(self):
        if getattr(self, "seq", None) is not None:
            scn.scn_seq_destroy(self.seq)
            self.seq = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostJob:
    """Positions [p0, p1) resident in pinned HOST memory (end-to-end path)."""

    def __init__(self, wl: scn_synth.Workload, p0: int, p1: int, with_halo: bool, device="cuda", plan_=None,
                 staging_frames: int = 32):
        self.wl = wl
        self.device = torch.device(device)
        self.part, self.row, self.seg = plan_ if plan_ is not None else plan(wl)
        self.M = len(self.row)
        self.p0, self.p1 = p0, p1
        halo = 1 if (with_halo and 0 < p0 < self.M and not self.seg[p0]) else 0
        self.lo = p0 - halo
        self.F = wl.frame_bytes
        self.F16 = ceil16(self.F)
        n_mat = p1 - self.lo
        # generate on the device in chunks, copy into pinned host memory (generation is untimed)
        self.host = torch.empty(max(n_mat, 1) * self.F16, dtype=torch.uint8, pin_memory=True)
        chunk = max(1, min(n_mat, (1 << 31) // self.F16))
        spec = wl.spec()
        tmp = torch.empty(chunk * self.F16, dtype=torch.uint8, device=self.device)
        jobs = torch.empty(chunk * scn_synth.job_bytes(), dtype=torch.uint8, device=self.device)
        st = torch.cuda.current_stream(self.device)
        for c0 in range(0, n_mat, chunk):
            k = min(chunk, n_mat - c0)
            addrs = tmp.data_ptr() + np.arange(k, dtype=np.uint64) * np.uint64(self.F16)
            spec.fill_device(self.part[self.lo + c0:self.lo + c0 + k], self.row[self.lo + c0:self.lo + c0 + k],
                             addrs, jobs.data_ptr(), st.cuda_stream)
            self.host[c0 * self.F16:(c0 + k) * self.F16].copy_(tmp[:k * self.F16])
        torch.cuda.synchronize(self.device)
        del tmp, jobs
        haddr = self.host.data_ptr() + np.arange(n_mat, dtype=np.uint64) * np.uint64(self.F16)
        ptrs = {}
        for j in range(self.lo, p1):
            v = int(self.part[j])
            if v not in ptrs:
                ptrs[v] = np.zeros(wl.rows_per_video, dtype=np.uint64)
            ptrs[v][int(self.row[j])] = haddr[j - self.lo]
        zeros = np.zeros(wl.rows_per_video, dtype=np.uint64)
        self.seq = _build_seq(wl, lambda v: ptrs.get(v, zeros), where=scn.SCN_MEM_HOST)
        n = p1 - p0
        self.staging_bytes = ceil16(max(n, 1)) + 2 * staging_frames * self.F16
        self.staging = torch.empty(self.staging_bytes, dtype=torch.uint8, device=self.device)

    def run(self, out, ops=("hist", "shotdiff"), bins=None, stream=None, copy_stream=None):
        bins = bins or self.wl.bins
        mask = ((scn.SCN_OP_HIST if "hist" in ops else 0) | (scn.SCN_OP_SHOTDIFF if "shotdiff" in ops else 0) |
                (scn.SCN_OP_DOWNSAMPLE if "downsample" in ops else 0))
        scn.scn_run_pipeline_host(self.seq, self.p0, self.p1, bins, mask, out.get("hist"), out.get("diff"),
                                  out.get("ds"), out.get("scratch"), self.staging, self.staging_bytes, stream,
                                  copy_stream)
        return scn.scn_last_launch_count()

    def close(self):
        if getattr(self, "seq", None) is not None:
            scn.scn_seq_destroy(self.seq)
            self.seq = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ColumnGather:
    """Final result exchange for N > 1: ONE all-gather of a flat int32
    send block laid out [rows_pad x 3B histogram counters | rows_pad shot-diffs], rows_pad =
    ceil(M/G). The kernels write the shard's H and D straight into the block through the
    `hist` / `diff` views (no pack copies); gather() copies only when handed other buffers.
    NCCL on the GPU box, gloo in the CPU tests; result() unpacks and trims the padding."""

    def __init__(self, M: int, world: int, bins: int, device, dist):
        self.M, self.world, self.bins, self.dist = M, world, bins, dist
        self.rows_pad = max(-(-M // world), 1) if world else 1
        self.spans = [scn.scn_shard_range(M, world, r) for r in range(world)]
        self.K = 3 * bins
        self.block = self.rows_pad * (self.K + 1)
        self.send = torch.zeros(self.block, dtype=torch.int32, device=device)
        self.hist = self.send[: self.rows_pad * self.K].view(self.rows_pad, 3, bins)
        self.diff = self.send[self.rows_pad * self.K:]
        self.all = torch.empty(self.block * world, dtype=torch.int32, device=device)

    def gather(self, hist=None, diff=None, n: int = 0):
        if hist is not None and hist.data_ptr() != self.hist.data_ptr():
            self.hist[:n].copy_(hist[:n].reshape(n, 3, self.bins))
        if diff is not None and diff.data_ptr() != self.diff.data_ptr():
            self.diff[:n].copy_(diff[:n])
        if self.send.is_cuda and self.dist.get_backend() == "gloo":
            # test-only path (several ranks sharing one GPU): gloo gathers host copies
            pa, aa = self.send.cpu(), self.all.cpu()
            self.dist.all_gather_into_tensor(aa, pa)
            self.all.copy_(aa)
            return
        self.dist.all_gather_into_tensor(self.all, self.send)

    def result(self):
        a = self.all.view(self.world, self.block)
        hs, ds = [], []
        for r, (b, e) in enumerate(self.spans):
            hs.append(a[r, : (e - b) * self.K].reshape(e - b, 3, self.bins))
            ds.append(a[r, self.rows_pad * self.K: self.rows_pad * self.K + e - b])
        return torch.cat(hs), torch.cat(ds)


class StencilJob:
    """NEXT N2 (fig:sampling-e): table -> HIST -> [offset,0] stencil -> Sample, over positions
    [p0, p1) of a workload's sampled sequence. Only the exact required set R = S U clamp(S+offset)
     is materialised; one scn_run_histogram over R and one scn_run_diff_pairs."""

    def __init__(self, wl: scn_synth.Workload, offset: int = -1, device="cuda", stream=None, spec=None):
        self.wl, self.offset = wl, offset
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        meta = _build_seq(wl)
        try:
            req_meta, pos, nbr = scn.scn_seq_stencil_required(meta, offset)
            rpart, rrow = scn.scn_seq_rows(req_meta)
            scn.scn_seq_destroy(req_meta)
            self.part, self.row = scn.scn_seq_rows(meta)
        finally:
            scn.scn_seq_destroy(meta)
        self.M, self.R = len(self.row), len(rrow)
        self.F16 = ceil16(wl.frame_bytes)
        self.buf = torch.empty(max(self.R, 1) * self.F16, dtype=torch.uint8, device=self.device)
        addrs = self.buf.data_ptr() + np.arange(self.R, dtype=np.uint64) * np.uint64(self.F16)
        self.spec = spec if spec is not None else wl.spec()
        if self.R:
            jobs = torch.empty(self.R * scn_synth.job_bytes(), dtype=torch.uint8, device=self.device)
            self.spec.fill_device(rpart.astype(np.int32), rrow, addrs, jobs.data_ptr(), self.stream.cuda_stream)
            self.stream.synchronize()
            del jobs
        ptrs = {}
        for j in range(self.R):
            v = int(rpart[j])
            if v not in ptrs:
                ptrs[v] = np.zeros(wl.rows_per_video, dtype=np.uint64)
            ptrs[v][int(rrow[j])] = addrs[j]
        zeros = np.zeros(wl.rows_per_video, dtype=np.uint64)
        self.seq = _build_seq(wl, lambda v: ptrs.get(v, zeros))
        self.req, pos, nbr = scn.scn_seq_stencil_required(self.seq, offset)
        self.ws = torch.empty(max(scn.scn_seq_device_bytes(self.req), 16), dtype=torch.uint8, device=self.device)
        scn.scn_seq_upload(self.req, self.ws, self.ws.numel(), self.stream)
        self.d_pos = torch.from_numpy(pos).to(self.device)
        self.d_nbr = torch.from_numpy(nbr).to(self.device)
        self.stream.synchronize()

    def alloc_outputs(self, bins=None):
        bins = bins or self.wl.bins
        return {"hist_req": torch.empty((max(self.R, 1), 3, bins), dtype=torch.int32, device=self.device),
                "diff": torch.empty(max(self.M, 1), dtype=torch.int32, device=self.device)}

    def run(self, out, bins=None, stream=None):
        bins = bins or self.wl.bins
        st = stream if stream is not None else self.stream
        scn.scn_run_histogram(self.req, 0, self.R, bins, out["hist_req"], st)
        n = scn.scn_last_launch_count()
        scn.scn_run_diff_pairs(out["hist_req"], self.d_pos, self.d_nbr, self.M, bins, out["diff"], st)
        return n + scn.scn_last_launch_count()

    def close(self):
        for a in ("req", "seq"):
            if getattr(self, a, None) is not None:
                scn.scn_seq_destroy(getattr(self, a))
                setattr(self, a, None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shot_montage(job: "DeviceJob", cols: int, tau: int, out=None, stream=None):
    """NEXT N1: the two-job film summary over a DeviceJob's positions [p0, p1).

    Job 1: HIST + shot-diff; the D column goes to the host, where the first position of
    every shot is selected (D > tau or a table start, reading Q5); job 2: Gather those
    positions and write their 2x downsample as montage tiles. Returns (canvas, positions)."""
    wl = job.wl
    st = stream if stream is not None else job.stream
    if out is None:
        out = job.alloc_outputs(("hist", "shotdiff"), wl.bins)
    b, e = job.p0, job.p1
    scn.scn_run_hist_shotdiff(job.seq, b, e, wl.bins, out["hist"], out["diff"], out["scratch"], st)
    d = torch.empty(max(e - b, 1), dtype=torch.int32, pin_memory=True)
    d.copy_(out["diff"][: max(e - b, 1)], non_blocking=True)
    st.synchronize()
    pos = scn.scn_select_shot_starts(job.seq, b, e, d.numpy().view(np.uint32)[: e - b], tau)
    kseq = scn.scn_seq_gather_positions(job.seq, pos)
    try:
        k = len(pos)
        ws = torch.empty(max(scn.scn_seq_device_bytes(kseq), 16), dtype=torch.uint8, device=job.device)
        scn.scn_seq_upload(kseq, ws, ws.numel(), st)
        oh, ow = wl.height // 2, wl.width // 2
        canvas = torch.empty((max(-(-k // cols), 1) * oh, cols * ow, 3), dtype=torch.uint8, device=job.device)
        scn.scn_run_montage(kseq, 0, k, cols, canvas, cols * ow * 3, st)
        st.synchronize()
    finally:
        scn.scn_seq_destroy(kseq)
    return canvas[: (-(-k // cols)) * oh], pos


class PeerColumns:
    """Full result columns (hist [M,3,B], diff [M]) on every rank, with every peer's columns
    mapped into this process, so scn_run_hist_shotdiff_to can write each rank's rows into all
    of them (the fused result all-gather; NVLink P2P when ranks are on different GPUs).
    Export: torch's storage sharing gives the allocation's cudaIpcMemHandle and the column's
    byte offset; import: scn_ipc_import opens it in THIS rank's device context with lazy peer
    access."""

    def __init__(self, M: int, bins: int, dist, device):
        self.dist = dist
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.hist = torch.zeros((max(M, 1), 3, bins), dtype=torch.int32, device=device)
        self.diff = torch.zeros(max(M, 1), dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)

        def export(t):
            st = t.untyped_storage()
            _, handle, _, off = st._share_cuda_()[:4]
            handle = bytes(handle)
            # torch prefixes the 64-byte cudaIpcMemHandle_t with [version byte] + a segment-type byte
            # ('c' = plain cudaMalloc segment; expandable segments use another format)
            tag_at = len(handle) - 65
            if tag_at in (0, 1):
                if handle[tag_at:tag_at + 1] != b"c":
                    raise RuntimeError(f"PeerColumns needs cudaMalloc segments (handle tag "
                                       f"{handle[tag_at:tag_at + 1]!r}); unset expandable_segments")
                handle = handle[tag_at + 1:]
            if len(handle) != 64:
                raise RuntimeError(f"unexpected CUDA IPC handle length {len(handle)}")
            return handle, int(off) + t.storage_offset() * t.element_size()

        # every rank joins the exchange even if its own export fails, so a failure on one rank
        # cannot leave the others waiting in the collective
        try:
            if os.environ.get("SCN_TEST_P2P_FAIL_RANK") == str(self.rank):  # test hook: the fallback path
                raise RuntimeError("export disabled by SCN_TEST_P2P_FAIL_RANK")
            mine, err = (export(self.hist), export(self.diff)), None
        except Exception as ex:  # noqa: BLE001 (re-raised on every rank below)
            mine, err = None, f"{type(ex).__name__}: {ex}"
        objs = [None] * self.world
        dist.all_gather_object(objs, mine)
        self.bases = None
        if any(o is None for o in objs):
            raise RuntimeError(err or "a peer could not export its result columns")
        self.bases = []
        self.hist_ptrs, self.diff_ptrs = [], []
        for g, ((hh, ho), (dh, do)) in enumerate(objs):
            if g == self.rank:
                self.hist_ptrs.append(self.hist.data_ptr())
                self.diff_ptrs.append(self.diff.data_ptr())
                continue
            bh, ph = scn.scn_ipc_import(hh, ho)
            self.bases.append(bh)
            if dh == hh:  # both columns in one caching-allocator block: one mapping serves both
                pd = bh + do
            else:
                bd, pd = scn.scn_ipc_import(dh, do)
                self.bases.append(bd)
            self.hist_ptrs.append(ph)
            self.diff_ptrs.append(pd)

    def close(self, barrier: bool = True):
        """Release the peer mappings; with barrier (every rank must call it then), peers drop
        their mappings before owners free the columns."""
        if self.bases is None:
            return
        torch.cuda.synchronize()
        for b in self.bases:
            scn.scn_ipc_release(b)
        self.bases = None
        if barrier:
            self.dist.barrier()
