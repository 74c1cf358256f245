"""Multi-GPU BC: sources partitioned across ranks, one allreduce of partial BC.

The reference has no distributed path: bc_parallel sums
per-thread buffers in one process (engine.cpp:444-448).  Here each rank
(one process per GPU, torch.distributed / NCCL) holds a full CSR replica,
runs the strided share ``sources[rank::world]`` and the partial node/edge BC
vectors are summed with one ``all_reduce`` -- the path's only exchange step.
Halved normalization is applied once, after the reduce (engine.cpp:451-454).
depth_per_source entries are disjoint per rank (a source runs on exactly one
rank; duplicates land on whichever ranks hold them and agree), so they
combine with MAX.

``compute`` is the per-rank kernel; the default runs the GPU path through the
C ABI.  Tests inject a CPU checker to exercise the sharding and reduction
logic with the gloo backend.
"""
from __future__ import annotations

from dataclasses import replace
from typing import Callable, Optional

import numpy as np


def shard_sources(sources: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Strided partition: spreads per-source cost variance evenly."""
    return np.ascontiguousarray(np.asarray(sources)[rank::world])


def bc_distributed(g, opt=None, compute: Optional[Callable] = None, group=None, device=None):
    """bc_parallel over all ranks of ``group``; every rank returns the full result.

    g: CsrGraph (or anything ``compute`` accepts).  compute(g, opt) -> BcResult
    for the rank's shard with Raw normalization.
    """
    import torch
    import torch.distributed as dist

    from . import BcResult, EngineOptions, GpuGraph, Normalization, _validate

    opt = opt or EngineOptions()
    _validate(opt)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    all_src = np.arange(g.n, dtype=np.uint32) if opt.sources is None else np.asarray(opt.sources, np.int64)
    if len(all_src) and (all_src.min() < 0 or all_src.max() >= g.n):
        raise ValueError("bc_parallel: source id out of range")
    mine = shard_sources(all_src.astype(np.uint32), rank, world)
    local_opt = replace(opt, sources=mine, normalization=Normalization.Raw)
    if compute is None:
        gg = GpuGraph(g, device=-1 if device is None else device)
        try:
            part = gg.bc(local_opt)
        finally:
            gg.close()
    else:
        part = compute(g, local_opt)
    dev = device if device is not None else ("cuda" if torch.cuda.is_available() and
                                            dist.is_initialized() and dist.get_backend(group) == "nccl"
                                            else "cpu")
    node = torch.from_numpy(np.ascontiguousarray(part.node_bc, np.float64)).to(dev)
    depth = torch.from_numpy(np.ascontiguousarray(part.depth_per_source).astype(np.int64)).to(dev)
    edge = torch.from_numpy(np.ascontiguousarray(part.edge_bc, np.float64)).to(dev) if opt.compute_edge_bc else None
    if world > 1:
        dist.all_reduce(node, group=group)
        dist.all_reduce(depth, op=dist.ReduceOp.MAX, group=group)
        if edge is not None:
            dist.all_reduce(edge, group=group)
    scale = 0.5 if opt.normalization == Normalization.Halved else 1.0
    node_np = node.cpu().numpy() * scale
    edge_np = edge.cpu().numpy() * scale if edge is not None else np.zeros(0)
    return BcResult(node_np, edge_np, depth.cpu().numpy().astype(np.uint32), part.elapsed)
