"""Multi-process (world_size 2, gloo, CPU) coverage of the batched multi-GPU
path: the batch partition and the single
data-path collective (all-gather of (d, e)).  On the GPU box the same code
runs over NCCL; a single matrix never spans ranks.  The per-rank work here is
the CPU oracle (test infrastructure); the product path needs CUDA."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2510_12705_b200.dist import gather_results, partition


@pytest.mark.parametrize("batch,world", [(64, 1), (64, 2), (64, 8), (5, 2), (3, 4), (0, 2), (7, 3)])
def test_partition_covers_batch_contiguously(batch, world):
    spans = [partition(batch, world, r) for r in range(world)]
    pos = 0
    for start, count in spans:
        assert start == pos and count >= 0
        pos += count
    assert pos == batch
    counts = [c for _, c in spans]
    assert max(counts) - min(counts) <= 1


def test_partition_rejects_bad_arguments():
    with pytest.raises(ValueError):
        partition(4, 0, 0)
    with pytest.raises(ValueError):
        partition(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, tw, batch, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, count = partition(batch, world, rank)
        ds, es = [], []
        for mid in range(start, start + count):
            band = synth.random_band(n, b, "f64", seed=5, matrix_id=mid)
            d, e = oracle.band_to_bidiag(band, b, tw)
            ds.append(d)
            es.append(e)
        d = torch.tensor(np.array(ds).reshape(count, n))
        e = torch.tensor(np.array(es).reshape(count, n - 1))
        D, E = gather_results(d, e, world)
        np.save(os.path.join(outdir, f"D{rank}.npy"), D.numpy())
        np.save(os.path.join(outdir, f"E{rank}.npy"), E.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [5, 4])
def test_gather_results_world2_gloo(tmp_path, batch):
    n, b, tw, world = 48, 6, 3, 2
    mp.spawn(_worker, args=(world, _free_port(), n, b, tw, batch, str(tmp_path)), nprocs=world, join=True)
    ref_d, ref_e = [], []
    for mid in range(batch):
        band = synth.random_band(n, b, "f64", seed=5, matrix_id=mid)
        d, e = oracle.band_to_bidiag(band, b, tw)
        ref_d.append(d)
        ref_e.append(e)
    for r in range(world):   # every rank holds the whole batch, in global matrix order
        assert np.array_equal(np.load(tmp_path / f"D{r}.npy"), np.array(ref_d))
        assert np.array_equal(np.load(tmp_path / f"E{r}.npy"), np.array(ref_e))
