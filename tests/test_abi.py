"""The C ABI library loads and exports every symbol include/bpc.h declares, and
its host-only planning (no device needed) validates configs and lays out the
chunk plan exactly as the oracle's plan (R1, R3, R8; §7 owner map)."""
import os
import re

import numpy as np
import pytest

from workloads import (LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp, config,
                       layout)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bpc():
    from paper_2105_07829_b200 import build
    build.build()
    import paper_2105_07829_b200 as P
    return P


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bpc.h")).read()
    return sorted(set(re.findall(r"\b(bpc_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(bpc):
    names = declared_symbols()
    assert len(names) >= 20
    lib = bpc.lib()
    for n in names:
        assert hasattr(lib, n), f"libbpc.so does not export {n}"
    assert set(names) == set(bpc.EXPORTS)


def test_library_is_sm100a(bpc):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", bpc._bpc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _cfg(bpc, numels, comp, **kw):
    offs, _ = layout(numels)
    return bpc.make_config(numels, offs, comp, **kw)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_plan_matches_oracle_plan(bpc, orc, name):
    w = config(name)
    numels = w.tensor_numels()
    offs, _ = layout(numels)
    cfg = bpc.make_config(numels, offs, w.comp, world_size=8, rank=3, chunk_elems=w.chunk_elems,
                          threshold_bytes=w.threshold_bytes)
    s, chunks = bpc.plan(cfg)
    ocfg = orc.Cfg.from_workload(w, n=8)
    oplan = ocfg.plan()
    assert [(c.tensor, c.offset, c.len, c.raw) for c in chunks] == oplan
    assert [c.payload_bytes for c in chunks] == [b for _, b in ocfg.payload_layout()]
    # SURVEY.md §8 chunk counts (2^18 units, 1 MiB threshold)
    expect = {"C2": (96, 132), "C3": (530, 20), "C4": (458, 130), "C5": (1282, 250)}[name]
    assert (s.num_compressed, s.num_chunks - s.num_compressed) == expect


def test_owner_map_and_segments(bpc):
    w = config("C5")
    numels = w.tensor_numels()
    offs, _ = layout(numels)
    segs = []
    for r in range(8):
        cfg = bpc.make_config(numels, offs, w.comp, world_size=8, rank=r)
        s, chunks = bpc.plan(cfg)
        segs.append((s, chunks))
    owners = [c.owner for c in segs[0][1]]
    for s, chunks in segs:
        assert [c.owner for c in chunks] == owners          # every rank derives the same map
        assert [c.payload_offset for c in chunks] == [c.payload_offset for c in segs[0][1]]
    # each owner's segment is contiguous, 16-byte aligned and sized as its recv slot
    for r in range(8):
        mine = [c for c in segs[0][1] if c.owner == r]
        assert all(c.payload_offset % 16 == 0 for c in mine)
        assert segs[r][0].recv_slot_bytes == sum((c.payload_bytes + 4 + 15) // 16 * 16 for c in mine)
    # LPT balance of the server cost: max/mean close to 1
    cost = np.zeros(8)
    for c in segs[0][1]:
        pb = c.payload_bytes
        cost[c.owner] += (4 * 8 * c.len + 4 * c.len) if c.raw else (8 * pb + 8 * c.len + pb)
    assert cost.max() / cost.mean() < 1.01


@pytest.mark.parametrize("comp,kw,status", [
    (Comp(TOP_K, 2, 1), {}, 4),                       # k fraction > 1 -> K_TOO_LARGE
    (Comp(LINEAR_DITHER, bits=9), {}, 1),             # bits out of range
    (Comp(NATURAL_DITHER, bits=1), {}, 1),
    (Comp(7), {}, 5),                                  # unknown kind
    (Comp(SCALED_SIGN), {"chunk_elems": 3000}, 1),    # not a power of two
    (Comp(SCALED_SIGN), {"chunk_elems": 1 << 20}, 1),  # > 2^18
    (Comp(SCALED_SIGN), {"world_size": 2, "rank": 2}, 1),
])
def test_plan_validation(bpc, comp, kw, status):
    with pytest.raises(bpc.BpcError) as ei:
        bpc.plan(_cfg(bpc, [1000, 300000], comp, **kw))
    assert ei.value.status == status


def test_plan_rejects_bad_tensors(bpc):
    with pytest.raises(bpc.BpcError) as ei:
        bpc.plan(bpc.make_config([10, 0], [0, 16], Comp(SCALED_SIGN)))
    assert ei.value.status == 3                      # EMPTY_BLOCK
    with pytest.raises(bpc.BpcError) as ei:
        bpc.plan(bpc.make_config([10, 10], [0, 6], Comp(SCALED_SIGN)))
    assert ei.value.status == 1                      # misaligned offset
    with pytest.raises(bpc.BpcError) as ei:
        bpc.plan(bpc.make_config([10, 10], [0, 8], Comp(SCALED_SIGN)))
    assert ei.value.status == 2                      # overlap


def test_init_without_gpu_fails_loudly(bpc):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bpc.BpcError) as ei:
        bpc.Context(_cfg(bpc, [1000], Comp(SCALED_SIGN)))
    assert ei.value.status == 8                      # BPC_ERR_CUDA: no CPU fallback
