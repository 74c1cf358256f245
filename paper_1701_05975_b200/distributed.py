"""Multi-GPU BC: sources partitioned across ranks, one allreduce of partial BC.

The reference has no distributed path: bc_parallel sums
per-thread buffers in one process (engine.cpp:444-448).  Here each rank
(one process per GPU, torch.distributed / NCCL) holds a full CSR replica,
runs the strided share ``sources[rank::world]`` and the partial node/edge BC
vectors (and depth_per_source) are summed with one ``all_reduce`` of one
fp64 buffer -- the path's only exchange step.
Halved normalization is applied once, after the reduce (engine.cpp:451-454).
depth_per_source: a source's entry is kept only by the rank holding its
first occurrence (duplicates on other ranks agree and are zeroed), so the
same SUM combines it exactly.

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
    dev = device if device is not None else ("cuda" if torch.cuda.is_available() and
                                            dist.is_initialized() and dist.get_backend(group) == "nccl"
                                            else "cpu")
    n, m = int(g.n), int(g.m)
    # ONE all-reduce (SUM) of one fp64 buffer [node | edge | depth]: a source's
    # depth is kept only on the rank owning its first occurrence in the list
    # (repeats carry the same value), so the sum equals it exactly.
    not_mine = None
    if world > 1 and len(all_src):
        first = np.unique(all_src.astype(np.int64), return_index=True)
        not_mine = first[0][first[1] % world != rank]  # the strided shard holding the first occurrence
    width = n + (m if opt.compute_edge_bc else 0) + n
    if compute is None and str(dev).startswith("cuda"):
        # device-resident run (wbc_gpu_bc_device): the partials never leave HBM
        buf = torch.zeros(width, dtype=torch.float64, device=dev)
        d_depth = torch.zeros(n, dtype=torch.int32, device=dev)
        d_src = torch.from_numpy(mine.astype(np.int32)).to(dev)
        tdev = torch.device(dev)
        gg = GpuGraph(g, device=torch.cuda.current_device() if tdev.index is None else tdev.index)
        try:
            if len(mine):
                gg.bc_device(d_src.data_ptr(), len(mine), buf.data_ptr(), d_depth.data_ptr(),
                             buf[n:].data_ptr() if opt.compute_edge_bc else 0, edge_bc=opt.compute_edge_bc,
                             stream=torch.cuda.current_stream(dev).cuda_stream)
            buf[width - n:] = d_depth.to(torch.float64)
            if not_mine is not None and len(not_mine):
                buf[width - n + torch.from_numpy(not_mine).to(dev)] = 0.0
            elapsed = 0.0
        finally:
            gg.close()
    else:
        if compute is None:
            gg = GpuGraph(g, device=-1 if device is None else device)
            try:
                part = gg.bc(local_opt)
            finally:
                gg.close()
        else:
            part = compute(g, local_opt)
        depth = np.asarray(part.depth_per_source, np.float64).copy()
        if not_mine is not None:
            depth[not_mine] = 0.0
        pieces = [np.ascontiguousarray(part.node_bc, np.float64)]
        if opt.compute_edge_bc:
            pieces.append(np.ascontiguousarray(part.edge_bc, np.float64))
        pieces.append(depth)
        buf = torch.from_numpy(np.concatenate(pieces)).to(dev)
        elapsed = part.elapsed
    if world > 1:
        dist.all_reduce(buf, group=group)
    out = buf.cpu().numpy()
    node = out[:n]
    edge = out[n:n + m] if opt.compute_edge_bc else None
    depth_out = out[width - n:]
    scale = 0.5 if opt.normalization == Normalization.Halved else 1.0
    node_np = node * scale
    edge_np = edge * scale if edge is not None else np.zeros(0)
    return BcResult(node_np, edge_np, np.rint(depth_out).astype(np.uint32), elapsed)
