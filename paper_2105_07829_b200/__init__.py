"""B200-native compressed gradient aggregation + update (arXiv 2105.07829).

The product path is libbpc.so (include/bpc.h): hand-written sm_100a CUDA
kernels + NCCL.  This package is its thin Python binding.  See DESIGN.md.
"""
from __future__ import annotations

from ._bpc import (BUF_M, BUF_P, BUF_RECV, BUF_SEND, BUF_SERVER_ERR, BUF_V, BUF_WORKER_ERR, BpcError,
                   ChunkInfo, Config, Context, EXPORTS, PlanSummary, connect_local, lib, make_config, plan,
                   unique_id)

__all__ = ["Context", "make_config", "plan", "unique_id", "connect_local", "context_for", "BpcError", "lib", "EXPORTS",
           "BUF_SEND", "BUF_RECV", "BUF_P", "BUF_WORKER_ERR", "BUF_SERVER_ERR", "BUF_M", "BUF_V",
           "ChunkInfo", "Config", "PlanSummary"]


def context_for(wcfg, *, rank=0, world_size=None, device=0, stream=None, nccl_id=None, check_finite=0,
                exchange="p2p"):
    """Build a Context for a workloads.Config (shapes, compressor, hyper-parameters)."""
    from workloads import layout
    import torch
    numels = wcfg.tensor_numels()
    offs, _ = layout(numels)
    if stream is None:
        stream = torch.cuda.current_stream(device).cuda_stream
    # chunk_elems = 0 is the oracle's per-tensor unit: unit_mode 1
    cfg = make_config(numels, offs, wcfg.comp, world_size=wcfg.n if world_size is None else world_size,
                      rank=rank, device=device, stream=stream, nccl_id=nccl_id, seed=wcfg.seed,
                      chunk_elems=wcfg.chunk_elems or (1 << 18), unit_mode=1 if wcfg.chunk_elems == 0 else 0,
                      threshold_bytes=wcfg.threshold_bytes, beta1=wcfg.beta1,
                      beta2=wcfg.beta2, eps=wcfg.eps, weight_decay=wcfg.weight_decay,
                      check_finite=check_finite, exchange={"p2p": 0, "nccl": 1, "nvls": 2}[exchange],
                      optimizer={"adam": 0, "lans": 1, "nag": 2}[getattr(wcfg, "optimizer", "adam")],
                      lans_alpha_l=getattr(wcfg, "alpha_l", 0.01), lans_alpha_u=getattr(wcfg, "alpha_u", 10.0),
                      momentum=getattr(wcfg, "momentum", 0.9))
    return Context(cfg)
