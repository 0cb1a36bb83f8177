"""GPU parity for the NEXT rows vs the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import scn_harness
import scn_synth
from scn_synth import Workload

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("sampling,offset", [(("stride", 3), -1), (("stride", 1), -1), (("stride", 7), -2),
                                             (("gather", 9, 40), -1), (("range", [(0, 10), (30, 50)], 4), 1),
                                             (("stride", 5), 0)])
def test_n2_stencil_then_sample(sampling, offset):
    wl = Workload("n2", 96, 54, 3, 120, sampling, ("hist", "shotdiff"), spec_kw={"len_min": 5, "len_max": 30})
    job = scn_harness.StencilJob(wl, offset)
    out = job.alloc_outputs()
    job.run(out)
    torch.cuda.synchronize()
    got = _u32(out["diff"])[: job.M]
    expect = oracle.stencil_then_sample(wl.spec(), job.part, job.row, offset, wl.rows_per_video, wl.bins)
    np.testing.assert_array_equal(got, expect)
    # the required set is exactly the oracle's dependency closure, per table
    for v in range(wl.n_videos):
        rows = job.row[job.part == v]
        assert len(oracle.required_rows(rows, offset, wl.rows_per_video)) > 0
    job.close()


def test_n2_c1_cuts():
    wl = scn_synth.Workload("C1e", 64, 36, 1, 240, ("stride", 3), ("hist", "shotdiff"),
                            spec_kw={"cuts": [57, 131, 198]})
    job = scn_harness.StencilJob(wl, -1)
    out = job.alloc_outputs()
    job.run(out)
    torch.cuda.synchronize()
    d = _u32(out["diff"])[: job.M]
    assert job.row[np.nonzero(d > 64 * 36)[0]].tolist() == [57, 198]
    assert job.R == len(oracle.required_rows(job.row, -1, 240))
    job.close()
