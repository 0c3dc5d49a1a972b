"""Size-threshold search (tools/threshold_search.py): the
selection rule on hand-made rows, and libbpc's host plan at every candidate
threshold (no device): a lower threshold compresses a superset of tensors, so
the per-rank payload never grows, and the plan still matches the oracle's."""
import os
import sys

import pytest

from workloads import config, layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import threshold_search as ts  # noqa: E402


def test_modeled_time_and_choice():
    rows = [{"threshold_bytes": 0, "ms_per_step": 0.30, "payload_bytes": 3_000_000},
            {"threshold_bytes": 1 << 20, "ms_per_step": 0.22, "payload_bytes": 9_000_000},
            {"threshold_bytes": 1 << 24, "ms_per_step": 0.25, "payload_bytes": 60_000_000}]
    # n = 1: no exchange, the device time decides
    assert ts.modeled_ms(0.22, 9_000_000, 1, 900.0) == 0.22
    assert ts.choose(rows, 1, 900.0)["threshold_bytes"] == 1 << 20
    # NVLink (900 GB/s, n = 8): 2 * 9e6 * 7/8 / 9e11 s = 0.0175 ms on top of 0.22
    assert ts.modeled_ms(0.22, 9_000_000, 8, 900.0) == pytest.approx(0.22 + 0.0175)
    assert ts.choose(rows, 8, 900.0)["threshold_bytes"] == 1 << 20
    # the paper's 25 Gb/s network: the payload dominates, compress everything
    assert ts.choose(rows, 8, 3.125)["threshold_bytes"] == 0
    # ties go to the larger threshold
    tie = [dict(rows[1], threshold_bytes=1 << 18), rows[1]]
    assert ts.choose(tie, 1, 900.0)["threshold_bytes"] == 1 << 20


@pytest.fixture(scope="module")
def bpc():
    from paper_2105_07829_b200 import build
    build.build()
    import paper_2105_07829_b200 as P
    return P


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_plan_over_candidates(bpc, name):
    import oracle
    w = config(name)
    numels = w.tensor_numels()
    offs, _ = layout(numels)
    prev = None
    for th in sorted(ts.CANDIDATES, reverse=True):
        cfg = bpc.make_config(numels, offs, w.comp, world_size=8, rank=0, chunk_elems=w.chunk_elems,
                              threshold_bytes=th)
        s, chunks = bpc.plan(cfg)
        raw = [c for c in chunks if c.raw]
        assert all(4 * c.len < th for c in raw)
        assert all(c.raw or 4 * numels[c.tensor] >= th for c in chunks)
        if prev is not None:
            assert s.payload_total <= prev
        prev = s.payload_total
        ocfg = oracle.Cfg.from_workload(config(name, threshold_bytes=th), n=8)
        assert [(c.tensor, c.offset, c.len, c.raw) for c in chunks] == ocfg.plan()
    # threshold 0 compresses every tensor
    assert not raw
