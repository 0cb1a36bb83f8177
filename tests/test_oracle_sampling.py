"""Pins for the oracle's sampling (§3.2; readings Q8-Q10, Q18).

Independent of the oracle's loops: paper examples, hand fixtures, Python's
own range()/set enumeration on tiny tables, and closed-form lengths."""
import json
import math
import os
import random

import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sampling.json")))
STATUS = {"EINVAL": oracle.EINVAL, "ERANGE": oracle.ERANGE}


@pytest.mark.parametrize("case", GOLD["paper"], ids=lambda c: c["cite"])
def test_paper_examples(case):
    rows = oracle.sample_stride(case["n_rows"], case["stride"])
    assert len(rows) == case["length"]


@pytest.mark.parametrize("case", GOLD["stride"])
def test_stride_fixtures(case):
    assert oracle.sample_stride(case["n_rows"], case["stride"]).tolist() == case["rows"]


@pytest.mark.parametrize("case", GOLD["range"])
def test_range_fixtures(case):
    assert oracle.sample_range(case["n_rows"], case["blocks"], case["step"]).tolist() == case["rows"]


@pytest.mark.parametrize("case", GOLD["gather"])
def test_gather_fixtures(case):
    assert oracle.sample_gather(case["n_rows"], case["rows_in"]).tolist() == case["rows"]


@pytest.mark.parametrize("case", GOLD["errors"])
def test_error_fixtures(case):
    with pytest.raises(oracle.OracleError) as e:
        if case["kind"] == "stride":
            oracle.sample_stride(case["n_rows"], case["stride"])
        elif case["kind"] == "gather":
            oracle.sample_gather(case["n_rows"], case["rows_in"])
        else:
            oracle.sample_range(case["n_rows"], case["blocks"], case["step"])
    assert e.value.code == STATUS[case["status"]]


def test_stride_bruteforce():
    for n in range(0, 65):
        for s in range(1, 71):
            got = oracle.sample_stride(n, s).tolist()
            assert got == list(range(0, n, s))
            assert len(got) == math.ceil(n / s)


def _random_blocks(rng, n):
    cuts = sorted(rng.sample(range(0, n + 1), k=min(n + 1, 2 * rng.randint(0, 4))))
    return [(cuts[i], cuts[i + 1]) for i in range(0, len(cuts) - 1, 2)]


def test_range_bruteforce():
    rng = random.Random(7339)
    for _ in range(2000):
        n = rng.randint(0, 64)
        blocks = _random_blocks(rng, n)
        k = rng.randint(1, 9)
        expect = [r for (a, b) in blocks for r in range(a, b, k)]
        got = oracle.sample_range(n, blocks, k).tolist()
        assert got == expect
        assert len(got) == sum(math.ceil((b - a) / k) for a, b in blocks)


def test_gather_bruteforce():
    rng = random.Random(1805)
    for _ in range(500):
        n = rng.randint(1, 64)
        rows = sorted(rng.sample(range(n), rng.randint(0, n)))
        assert oracle.sample_gather(n, rows).tolist() == rows
