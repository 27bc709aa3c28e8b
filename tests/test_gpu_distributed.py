"""The subtree-partitioned compressor as a real multi-process program on the
GPU: world 2 over gloo (the one-GPU box has no second device for NCCL), both
ranks running the CUDA engine on cuda:0.  The collective is the host-staged
all-gather (distributed._all_gather_flat); the kernels of the two ranks never
wait on each other.  The gathered factorization must equal the single-GPU
sweep bit for bit (partitioning changes no per-node arithmetic), and the
preallocated DistributedCompressor must reproduce the operator."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASE = dict(n=4096, leaf=32, k=12, r=20, s=60)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _samples():
    from oracle import hbs_oracle as O
    c = CASE
    g = O.baseline_generator(c["n"], c["leaf"], c["k"], seed=0)
    return g, O.samples_from(g, c["s"], 0)


def _worker(rank, world, port, outdir):
    import paper_2205_02990_b200 as hb
    from paper_2205_02990_b200.distributed import DistributedCompressor, SubtreePartition, compress_distributed
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        c = CASE
        tree = hb.build_tree(c["n"], c["leaf"])
        g, samples = _samples()
        part = SubtreePartition(tree, world, rank, c["r"])
        local = [torch.from_numpy(m[part.begin:part.end]).cuda() for m in samples]
        f = compress_distributed(local, tree, hb.CompressionConfig(rank=c["r"], leaf_threshold=c["leaf"]))
        blocks, root = f.gather()
        comp = DistributedCompressor(tree, part, c["s"], device="cuda:0")
        comp.run(*local)
        torch.cuda.synchronize()
        comp.raise_for_status()
        from oracle import hbs_oracle as O
        x = O.gaussian(c["n"], 4, 0, 4)
        ax = comp.operator().apply(torch.from_numpy(x[part.begin:part.end]).cuda()).cpu().numpy()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), root=root, ids=np.array(sorted(blocks)), ax=ax,
                 begin=part.begin, end=part.end,
                 **{f"u{i}": blocks[i][0] for i in blocks}, **{f"v{i}": blocks[i][1] for i in blocks},
                 **{f"d{i}": blocks[i][2] for i in blocks})
    finally:
        dist.destroy_process_group()


def test_two_rank_cuda_engine_bitwise_equals_single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2205_02990_b200 as hb
    from oracle import hbs_oracle as O
    c = CASE
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        outs = [dict(np.load(os.path.join(d, f"rank{i}.npz"))) for i in range(world)]
    g, samples = _samples()
    tree = hb.build_tree(c["n"], c["leaf"])
    f = hb.compress_from_samples(hb.SampleSet(*samples), tree, hb.CompressionConfig(rank=c["r"], leaf_threshold=c["leaf"]))
    for out in outs:
        assert np.array_equal(out["root"], f.root_disc)
        assert len(out["ids"]) == (1 << (tree.depth + 1)) - 2
        for nid in out["ids"]:
            nid = int(nid)
            assert np.array_equal(out[f"u{nid}"], f.u_bases[nid])
            assert np.array_equal(out[f"v{nid}"], f.v_bases[nid])
            assert np.array_equal(out[f"d{nid}"], f.discs[nid])
    x = O.gaussian(c["n"], 4, 0, 4)
    got = np.concatenate([out["ax"] for out in outs])
    want = O.apply(g, x)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10
