"""C-ABI host-side tests (no GPU): the library loads, exports every symbol
include/scn.h declares, and its host logic (sampling P:L208, concatenation
P:L181-185 / slices P:L216, shard math and halo P:L214, validation) agrees
with the oracle and the header's error contract. No compute calls."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
import scn_synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = 1 << 40


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "scn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scn_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = _declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(scn.LIB_PATH)
    for name in syms:
        assert hasattr(lib, name), name
        assert hasattr(scn, name), f"binding lacks {name}"


def test_version_and_error_string():
    assert "sm_100a" in scn.scn_version()
    with pytest.raises(scn.ScnError) as e:
        scn.scn_table_create(10, 0, 5, 3, scn.SCN_MEM_DEVICE, FAKE, 16)
    assert e.value.status == scn.SCN_EINVAL
    assert "width" in scn.scn_last_error()


def _table(n, w=8, h=4):
    F16 = (w * h * 3 + 15) & ~15
    return scn.scn_table_create(n, w, h, 3, scn.SCN_MEM_DEVICE, FAKE, F16)


def test_sampling_matches_oracle():
    rng = random.Random(3)
    for _ in range(300):
        n = rng.randint(0, 80)
        t = _table(n)
        s = rng.randint(1, 90)
        q = scn.scn_sample_stride(t, s)
        assert scn.scn_seq_rows(q)[1].tolist() == oracle.sample_stride(n, s).tolist()
        scn.scn_seq_destroy(q)
        cuts = sorted(rng.sample(range(n + 1), k=min(n + 1, 2 * rng.randint(0, 3))))
        blocks = [(cuts[i], cuts[i + 1]) for i in range(0, len(cuts) - 1, 2)]
        k = rng.randint(1, 7)
        q = scn.scn_sample_range(t, blocks, k)
        assert scn.scn_seq_rows(q)[1].tolist() == oracle.sample_range(n, blocks, k).tolist()
        scn.scn_seq_destroy(q)
        rows = sorted(rng.sample(range(n), rng.randint(0, n))) if n else []
        q = scn.scn_sample_gather(t, rows)
        assert scn.scn_seq_rows(q)[1].tolist() == oracle.sample_gather(n, rows).tolist()
        scn.scn_seq_destroy(q)
        scn.scn_table_destroy(t)


@pytest.mark.parametrize("call,status", [
    (lambda t: scn.scn_sample_stride(t, 0), scn.SCN_EINVAL),
    (lambda t: scn.scn_sample_gather(t, [4, 1]), scn.SCN_EINVAL),
    (lambda t: scn.scn_sample_gather(t, [3, 3]), scn.SCN_EINVAL),
    (lambda t: scn.scn_sample_gather(t, [10]), scn.SCN_ERANGE),
    (lambda t: scn.scn_sample_gather(t, [-1]), scn.SCN_ERANGE),
    (lambda t: scn.scn_sample_range(t, [(5, 8), (2, 4)], 1), scn.SCN_EINVAL),
    (lambda t: scn.scn_sample_range(t, [(2, 11)], 1), scn.SCN_ERANGE),
    (lambda t: scn.scn_sample_range(t, [(2, 5)], 0), scn.SCN_EINVAL),
])
def test_sampling_errors(call, status):
    t = _table(10)
    with pytest.raises(scn.ScnError) as e:
        call(t)
    assert e.value.status == status
    scn.scn_table_destroy(t)


def test_table_validation():
    D = scn.SCN_MEM_DEVICE
    bad = [
        dict(num_rows=-1, width=8, height=4, base=FAKE, frame_stride_bytes=96),
        dict(num_rows=4, width=8, height=4, channels=4, base=FAKE, frame_stride_bytes=96),
        dict(num_rows=4, width=8, height=4, base=FAKE, frame_stride_bytes=95),   # < F
        dict(num_rows=4, width=64, height=36, base=FAKE, frame_stride_bytes=6913),  # not multiple of 16
        dict(num_rows=4, width=8, height=4, base=FAKE + 8, frame_stride_bytes=96),  # misaligned base
        dict(num_rows=4, width=8, height=4),                                       # neither base nor rows
        dict(num_rows=4, width=8, height=4, base=FAKE, frame_stride_bytes=96, row_ptrs=[16] * 4),  # both
        dict(num_rows=2, width=8, height=4, row_ptrs=[16, 24]),                    # misaligned row ptr
        dict(num_rows=1, width=40000, height=40000, base=FAKE, frame_stride_bytes=4800000000),  # W*H bound
    ]
    for kw in bad:
        kw.setdefault("channels", 3)
        with pytest.raises(scn.ScnError) as e:
            scn.scn_table_create(where=D, **kw)
        assert e.value.status == scn.SCN_EINVAL, kw
    t = scn.scn_table_create(0, 8, 4, 3, D)  # empty table is valid (reading Q18)
    q = scn.scn_sample_stride(t, 1)
    assert scn.scn_seq_length(q) == 0
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)


def test_concat_segments_and_halo():
    ta, tb = _table(10), _table(7)
    qa, qb = scn.scn_sample_stride(ta, 3), scn.scn_sample_stride(tb, 2)
    q = scn.scn_seq_concat([qa, qb])
    part, row = scn.scn_seq_rows(q)
    assert part.tolist() == [0] * 4 + [1] * 4
    assert row.tolist() == [0, 3, 6, 9, 0, 2, 4, 6]
    assert scn.scn_seq_seg_starts(q).tolist() == [1, 0, 0, 0, 1, 0, 0, 0]
    assert [scn.scn_seq_needs_halo(q, b) for b in range(9)] == [0, 1, 1, 1, 0, 1, 1, 1, 0]
    t3 = scn.scn_table_create(5, 9, 4, 3, scn.SCN_MEM_DEVICE, FAKE, 112)
    q3 = scn.scn_sample_stride(t3, 1)
    with pytest.raises(scn.ScnError) as e:
        scn.scn_seq_concat([qa, q3])  # unequal frame shape
    assert e.value.status == scn.SCN_EINVAL
    for x in (qa, qb, q, q3):
        scn.scn_seq_destroy(x)
    for t in (ta, tb, t3):
        scn.scn_table_destroy(t)


def test_shard_range():
    for m in (0, 1, 7, 240, 16384, 36864):
        for G in (1, 2, 3, 4, 8):
            spans = [scn.scn_shard_range(m, G, r) for r in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(G - 1))
            assert all(e - b in (m // G, m // G + 1) for b, e in spans)
            assert spans == [((r * m) // G, ((r + 1) * m) // G) for r in range(G)]
    for bad in ((10, 0, 0), (10, 2, 2), (10, 2, -1), (-1, 1, 0)):
        with pytest.raises(scn.ScnError):
            scn.scn_shard_range(*bad)


def test_run_validation_without_gpu():
    t = _table(10)
    q = scn.scn_sample_stride(t, 1)
    with pytest.raises(scn.ScnError) as e:
        scn.scn_run_histogram(q, 0, 4, 0, 1 << 20)
    assert e.value.status == scn.SCN_EUNSUPPORTED
    with pytest.raises(scn.ScnError) as e:
        scn.scn_run_histogram(q, 0, 11, 16, 1 << 20)
    assert e.value.status == scn.SCN_ERANGE
    with pytest.raises(scn.ScnError) as e:
        scn.scn_run_histogram(q, 5, 4, 16, 1 << 20)
    assert e.value.status == scn.SCN_EINVAL
    with pytest.raises(scn.ScnError) as e:  # not uploaded
        scn.scn_run_histogram(q, 0, 4, 16, 1 << 20)
    assert e.value.status == scn.SCN_EINVAL
    with pytest.raises(scn.ScnError) as e:  # device sequence on the host pipeline
        scn.scn_run_pipeline_host(q, 0, 4, 16, 1, 1 << 20, None, None, None, 1 << 20, 1 << 20)
    assert e.value.status == scn.SCN_EINVAL
    scn.scn_run_histogram(q, 3, 3, 16, None)  # empty range is a no-op
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)


@pytest.mark.parametrize("name", list(scn_synth.WORKLOADS))
def test_plan_matches_oracle_sampling(name):
    wl = scn_synth.WORKLOADS[name]
    part, row, seg = scn_harness.plan(wl)
    kind = wl.sampling[0]
    per = []
    for v in range(wl.n_videos):
        if kind == "stride":
            r = oracle.sample_stride(wl.rows_per_video, wl.sampling[1])
        elif kind == "range":
            r = oracle.sample_range(wl.rows_per_video, wl.sampling[1], wl.sampling[2])
        else:
            r = oracle.sample_gather(wl.rows_per_video,
                                     scn_synth.gather_rows(wl.sampling[1], wl.rows_per_video, wl.sampling[2]))
        per.append(r)
    assert row.tolist() == np.concatenate(per).tolist()
    assert part.tolist() == np.concatenate([[v] * len(r) for v, r in enumerate(per)]).tolist()
    assert seg.sum() == wl.n_videos
    expect_m = {"C1": 240, "C2": 16384, "C3": 36864, "C4": 4096, "C5": 7168}[name]
    assert len(row) == expect_m


def test_n2_stencil_required_matches_oracle():
    rng = random.Random(91)
    for _ in range(200):
        nv = rng.randint(1, 3)
        parts, tables, expect_rows, S_all = [], [], [], []
        for v in range(nv):
            n = rng.randint(1, 40)
            t = _table(n)
            tables.append(t)
            rows = sorted(rng.sample(range(n), rng.randint(1, n)))
            parts.append(scn.scn_sample_gather(t, rows))
            S_all.append((rows, n))
        q = scn.scn_seq_concat(parts) if nv > 1 else parts[0]
        o = rng.randint(-4, 4)
        req, pos, nbr = scn.scn_seq_stencil_required(q, o)
        rpart, rrow = scn.scn_seq_rows(req)
        seg = scn.scn_seq_seg_starts(req)
        exp_rows, exp_part = [], []
        for v, (rows, n) in enumerate(S_all):
            rr = oracle.required_rows(rows, o, n).tolist()
            exp_rows += rr
            exp_part += [v] * len(rr)
        assert rrow.tolist() == exp_rows and rpart.tolist() == exp_part
        assert seg.sum() == nv
        j = 0
        for v, (rows, n) in enumerate(S_all):
            for r in rows:
                assert rrow[pos[j]] == r and rpart[pos[j]] == v
                assert rrow[nbr[j]] == min(max(r + o, 0), n - 1) and rpart[nbr[j]] == v
                j += 1
        for x in [req] + ([q] if nv > 1 else []) + parts:
            scn.scn_seq_destroy(x)
        for t in tables:
            scn.scn_table_destroy(t)


def test_n3_warmup_begin():
    ta, tb = _table(10), _table(7)
    qa, qb = scn.scn_sample_stride(ta, 1), scn.scn_sample_stride(tb, 1)
    q = scn.scn_seq_concat([qa, qb])  # tables start at positions 0 and 10
    seg = scn.scn_seq_seg_starts(q)
    for b in range(17):
        for w in range(0, 6):
            s0 = max(i for i in range(b + 1) if seg[i]) if b < 17 else b
            assert scn.scn_seq_warmup_begin(q, b, w) == max(s0, b - w), (b, w)
    for x in (qa, qb, q):
        scn.scn_seq_destroy(x)
    scn.scn_table_destroy(ta)
    scn.scn_table_destroy(tb)


def test_n1_select_and_gather_positions_match_oracle():
    rng = np.random.default_rng(8)
    ta, tb = _table(30), _table(25)
    qa, qb = scn.scn_sample_stride(ta, 2), scn.scn_sample_stride(tb, 3)
    q = scn.scn_seq_concat([qa, qb])
    m = scn.scn_seq_length(q)
    seg = scn.scn_seq_seg_starts(q)
    part, row = scn.scn_seq_rows(q)
    for _ in range(50):
        d = rng.integers(0, 100, m).astype(np.uint32)
        tau = int(rng.integers(0, 100))
        b = int(rng.integers(0, m))
        e = int(rng.integers(b, m + 1))
        got = scn.scn_select_shot_starts(q, b, e, d[b:e], tau)
        ref = oracle.shot_starts(d, seg, tau)
        assert got.tolist() == [p for p in ref.tolist() if b <= p < e]
        g = scn.scn_seq_gather_positions(q, got)
        gp, gr = scn.scn_seq_rows(g)
        gs = scn.scn_seq_seg_starts(g)
        assert gr.tolist() == row[got].tolist()
        # parts renumbered in order; a new part starts wherever the table changes
        assert gs.tolist() == [1 if (i == 0 or part[got[i]] != part[got[i - 1]]) else 0 for i in range(len(got))]
        scn.scn_seq_destroy(g)
    with pytest.raises(scn.ScnError) as ex:
        scn.scn_seq_gather_positions(q, [3, 3])
    assert ex.value.status == scn.SCN_EINVAL
    with pytest.raises(scn.ScnError) as ex:
        scn.scn_seq_gather_positions(q, [m])
    assert ex.value.status == scn.SCN_ERANGE
    for x in (qa, qb, q):
        scn.scn_seq_destroy(x)
    scn.scn_table_destroy(ta)
    scn.scn_table_destroy(tb)


def test_plain_c_demo_builds_and_links():
    # the ABI is usable from plain C: examples/scn_demo.c compiles against include/scn.h and links libscn.so
    import subprocess
    r = subprocess.run(["make", "-C", ROOT, "examples/scn_demo"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(os.path.join(ROOT, "examples", "scn_demo"))


def test_nested_concat_keeps_inner_tables():
    ta, tb, tc = _table(6), _table(5), _table(4)
    qa, qb, qc = (scn.scn_sample_stride(t, 2) for t in (ta, tb, tc))
    inner = scn.scn_seq_concat([qa, qb])
    outer = scn.scn_seq_concat([inner, qc])
    part, row = scn.scn_seq_rows(outer)
    assert part.tolist() == [0, 0, 0, 1, 1, 1, 2, 2]
    assert row.tolist() == [0, 2, 4, 0, 2, 4, 0, 2]
    assert scn.scn_seq_seg_starts(outer).tolist() == [1, 0, 0, 1, 0, 0, 1, 0]
    # the stencil closure still resolves rows through each inner table (clamp per table)
    req, pos, nbr = scn.scn_seq_stencil_required(outer, 1)
    rp, rr = scn.scn_seq_rows(req)
    assert rr.tolist() == [0, 1, 2, 3, 4, 5, 0, 1, 2, 3, 4, 0, 1, 2, 3]
    assert rp.tolist() == [0] * 6 + [1] * 5 + [2] * 4
    for x in (qa, qb, qc, inner, outer, req):
        scn.scn_seq_destroy(x)
    for t in (ta, tb, tc):
        scn.scn_table_destroy(t)


def test_pipeline_host_validation_without_gpu():
    F16 = 96
    host = np.zeros(10 * F16, dtype=np.uint8)
    t = scn.scn_table_create(10, 8, 4, 3, scn.SCN_MEM_HOST, host, F16)
    q = scn.scn_sample_stride(t, 1)
    big = 1 << 30

    def run(**kw):
        a = dict(s=q, begin=0, end=10, bins=16, ops=scn.SCN_OP_HIST | scn.SCN_OP_SHOTDIFF, d_hist=big,
                 d_diff=big, d_out=None, d_scratch=big, d_staging=big, staging_bytes=1 << 20)
        a.update(kw)
        with pytest.raises(scn.ScnError) as e:
            scn.scn_run_pipeline_host(a["s"], a["begin"], a["end"], a["bins"], a["ops"], a["d_hist"], a["d_diff"],
                                      a["d_out"], a["d_scratch"], a["d_staging"], a["staging_bytes"])
        return e.value.status

    assert run(ops=8) == scn.SCN_EINVAL                      # unknown op bit
    assert run(ops=scn.SCN_OP_SHOTDIFF) == scn.SCN_EINVAL    # shot-diff needs HIST
    assert run(bins=0) == scn.SCN_EUNSUPPORTED
    assert run(end=11) == scn.SCN_ERANGE
    assert run(begin=5, end=4) == scn.SCN_EINVAL
    assert run(d_hist=None) == scn.SCN_EINVAL
    assert run(staging_bytes=100) == scn.SCN_EINVAL          # < header + 2 frames
    assert run(d_staging=big + 8) == scn.SCN_EINVAL          # not 16-aligned
    assert run(begin=3, d_scratch=None) == scn.SCN_EINVAL    # halo needs scratch
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)
    # a sparse host table with an absent row in the range
    ptrs = np.array([host.ctypes.data + i * F16 if i != 6 else 0 for i in range(10)], dtype=np.uint64)
    t = scn.scn_table_create(10, 8, 4, 3, scn.SCN_MEM_HOST, None, 0, ptrs)
    q = scn.scn_sample_stride(t, 1)
    with pytest.raises(scn.ScnError) as e:
        scn.scn_run_pipeline_host(q, 0, 10, 16, scn.SCN_OP_HIST, big, None, None, None, big, 1 << 20)
    assert e.value.status == scn.SCN_ERANGE
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)


def test_adaptive_cuts_overflow_bound_and_hist_impl_validation():
    # W * (k_num + k_den) must stay < 2^32 so the 64-bit comparison is exact (DESIGN §8 N3)
    t = _table(10)
    q = scn.scn_sample_stride(t, 1)
    scn.scn_run_adaptive_cuts(q, 0, 0, 16, None, 4, 1, 0, None)  # in bounds, empty range: no-op
    for w, kn, kd in ((1 << 16, 1 << 16, 0), (2, (1 << 31), (1 << 31) - 1), (1 << 30, 2, 2)):
        with pytest.raises(scn.ScnError) as e:
            scn.scn_run_adaptive_cuts(q, 0, 0, w, None, kn, max(kd, 1), 0, None)
        assert e.value.status == scn.SCN_EINVAL
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)
    assert scn.scn_get_hist_impl() == scn.SCN_HIST_LANE_PAIRS
    for bad in (-1, 3):
        with pytest.raises(scn.ScnError) as e:
            scn.scn_set_hist_impl(bad)
        assert e.value.status == scn.SCN_EINVAL
    assert scn.scn_hist_variant(16) == "tma_pair_lane_private"
    assert scn.scn_hist_variant(100) == "tma_raw_lane_private_remap"
    assert scn.scn_hist_variant(5) == "tma_pair_bins_lane_private"
    scn.scn_set_hist_impl(scn.SCN_HIST_MATCH_PACKED)
    assert scn.scn_hist_variant(8) == "k2a_packed_match_per_warp"
    assert scn.scn_hist_variant(256) == "tma_raw_lane_private_remap"
    scn.scn_set_hist_impl(scn.SCN_HIST_LANE_PAIRS)


def test_binding_rejects_short_host_arrays():
    t = _table(10)
    q = scn.scn_sample_stride(t, 1)
    with pytest.raises(ValueError):
        scn.scn_select_shot_starts(q, 0, 5, np.zeros(4, np.uint32), 1)
    with pytest.raises(ValueError):
        scn.scn_run_hist_shotdiff_to(q, 0, 0, 16, [1 << 20, 1 << 21], [1 << 22], 0)
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)


def test_product_library_reads_no_environment():
    # the measurement knobs exist only in libscn_tuning.so (-DSCN_TUNING); outside that
    # #ifdef block the product sources call no getenv (cudart_static's own are not ours)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_1805_07339_b200", "csrc", "kernels.cu")).read()
    pre, rest = src.split("#ifdef SCN_TUNING", 1)
    tuning, post = rest.split("#else", 1)
    assert "getenv" in tuning and "getenv" not in pre + post
    assert "getenv" not in open(os.path.join(root, "paper_1805_07339_b200", "csrc", "scn_api.cpp")).read()
