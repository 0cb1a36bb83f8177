"""Property-based checks (hypothesis) of the C-ABI host logic against the oracle and
the definitions (no GPU): sampling, shard partition (Q17), the [-1,0]
halo and bounded-state warmup begin, the stencil-before-sample
required set (NEXT N2) and shot-start selection (NEXT N1)."""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_1805_07339_b200 as scn

FAKE = 1 << 40
SET = settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])


def _table(n):
    return scn.scn_table_create(n, 8, 4, 3, scn.SCN_MEM_DEVICE, FAKE, 96)


@SET
@given(st.integers(0, 5000), st.integers(1, 64))
def test_shard_partition(m, g):
    spans = [scn.scn_shard_range(m, g, r) for r in range(g)]
    assert spans[0][0] == 0 and spans[-1][1] == m
    assert all(spans[i][1] == spans[i + 1][0] for i in range(g - 1))
    assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


@SET
@given(st.integers(0, 300), st.integers(1, 400))
def test_stride_matches_oracle(n, s):
    t = _table(n)
    q = scn.scn_sample_stride(t, s)
    assert scn.scn_seq_rows(q)[1].tolist() == oracle.sample_stride(n, s).tolist()
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)


@SET
@given(st.lists(st.integers(1, 60), min_size=1, max_size=4), st.data())
def test_halo_and_warmup(lengths, data):
    tables = [_table(n) for n in lengths]
    parts = [scn.scn_sample_stride(t, 1) for t in tables]
    q = scn.scn_seq_concat(parts)
    seg = scn.scn_seq_seg_starts(q)
    m = len(seg)
    b = data.draw(st.integers(0, m - 1))
    w = data.draw(st.integers(0, 20))
    assert scn.scn_seq_needs_halo(q, b) == (1 if b > 0 and not seg[b] else 0)
    s0 = max(i for i in range(b + 1) if seg[i])
    assert scn.scn_seq_warmup_begin(q, b, w) == max(s0, b - w)
    for x in parts + [q]:
        scn.scn_seq_destroy(x)
    for t in tables:
        scn.scn_table_destroy(t)


@SET
@given(st.integers(1, 80), st.data())
def test_required_set_matches_oracle(n, data):
    rows = sorted(data.draw(st.sets(st.integers(0, n - 1), min_size=1, max_size=n)))
    o = data.draw(st.integers(-6, 6))
    t = _table(n)
    q = scn.scn_sample_gather(t, rows)
    req, pos, nbr = scn.scn_seq_stencil_required(q, o)
    rr = scn.scn_seq_rows(req)[1]
    assert rr.tolist() == oracle.required_rows(rows, o, n).tolist()
    assert [int(rr[p]) for p in pos] == rows
    assert [int(rr[p]) for p in nbr] == [min(max(r + o, 0), n - 1) for r in rows]
    for x in (req, q):
        scn.scn_seq_destroy(x)
    scn.scn_table_destroy(t)


@SET
@given(st.lists(st.integers(0, 1000), min_size=1, max_size=120), st.integers(0, 1000))
def test_shot_starts_match_oracle(diffs, tau):
    n = len(diffs)
    t = _table(n)
    q = scn.scn_sample_stride(t, 1)
    d = np.array(diffs, np.uint32)
    got = scn.scn_select_shot_starts(q, 0, n, d, tau)
    assert got.tolist() == oracle.shot_starts(d, scn.scn_seq_seg_starts(q), tau).tolist()
    scn.scn_seq_destroy(q)
    scn.scn_table_destroy(t)
