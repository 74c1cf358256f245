"""N>1 path (source partitioning + one allreduce of partial BC) on CPU with
gloo, world_size 2.  The per-rank compute is the oracle standing in for the
GPU kernel; what is tested is the product's sharding/reduction logic in
paper_1701_05975_b200/distributed.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1701_05975_b200 as W
    from paper_1701_05975_b200.distributed import bc_distributed, shard_sources
    from oracle import Oracle
    O = Oracle()

    def oracle_compute(g, opt):
        node, edge, depth = O.bc_eq4(g, sources=opt.sources, edge_bc=opt.compute_edge_bc)
        return W.BcResult(node, edge if edge is not None else np.zeros(0), depth, 0.0)

    el = W.assign_weights(W.gen_kronecker(9, 8.0, 4), 1, 30, 4)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 50, 2)
    src = np.concatenate([src, src[:3]])                 # duplicates count twice
    assert len(shard_sources(src, rank, world)) in (len(src) // world, len(src) // world + 1)
    r = bc_distributed(g, W.EngineOptions(sources=src, compute_edge_bc=True,
                                          normalization=W.Normalization.Halved), compute=oracle_compute)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), node=r.node_bc, edge=r.edge_bc, depth=r.depth_per_source)
    dist.destroy_process_group()


def test_two_rank_gloo(tmp_path, oracle):
    import paper_1701_05975_b200 as W
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    el = W.assign_weights(W.gen_kronecker(9, 8.0, 4), 1, 30, 4)
    g = W.build_csr(el)
    src = W.sample_sources(g.n, 50, 2)
    src = np.concatenate([src, src[:3]])
    node, edge, depth = oracle.bc_eq4(g, sources=src, edge_bc=True, halved=True)
    for rank in (0, 1):
        r = np.load(tmp_path / f"r{rank}.npz")
        tol = lambda a, b: np.abs(a - b) <= np.maximum(1e-12, 1e-9 * np.maximum(np.abs(a), np.abs(b)))
        assert tol(r["node"], node).all() and tol(r["edge"], edge).all()
        assert np.array_equal(r["depth"], depth)
