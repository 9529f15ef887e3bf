"""CPU, world_size 2 over gloo: (batch, head) slab partition + gather to rank 0
(SURVEY 8e).  The per-slab compute is the oracle restatement (CPU); on the GPU
box the same host logic drives mha_forward over NCCL."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_12784_b200.shard import gather_to_rank0, run_sharded, shard_range


def test_shard_range_partitions_exactly():
    for bh in (1, 2, 7, 64, 65):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(bh, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == bh
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _oracle_forward(q, k, v):
    from oracle import pyoracle as po
    out, lse = po.attention_ref(q.double().numpy(), k.double().numpy(), v.double().numpy(), False)
    return torch.from_numpy(out), torch.from_numpy(lse)


def _worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, N, d = 2, 3, 32, 16
        g = torch.Generator().manual_seed(0)
        q, k, v = (torch.randn(B, H, N, d, generator=g) for _ in range(3))
        got = run_sharded(_oracle_forward, [q, k, v])
        if rank == 0:
            ref_o, ref_l = _oracle_forward(q.reshape(B * H, 1, N, d), k.reshape(B * H, 1, N, d), v.reshape(B * H, 1, N, d))
            result["ok"] = bool(torch.equal(got[0], ref_o.reshape(B * H, N, d)) and
                                torch.equal(got[1], ref_l.reshape(B * H, N)))
        # uneven gather
        lo, hi = shard_range(5, world, rank)
        local = torch.arange(lo, hi, dtype=torch.float32).unsqueeze(1)
        full = gather_to_rank0(local, 5)
        if rank == 0:
            result["uneven"] = full.squeeze(1).tolist() == [0.0, 1.0, 2.0, 3.0, 4.0]
    finally:
        dist.destroy_process_group()


def test_world2_gloo_shard_and_gather():
    port = 29500 + (os.getpid() % 1000)
    with mp.Manager() as m:
        result = m.dict()
        mp.spawn(_worker, args=(2, port, result), nprocs=2, join=True)
        assert result.get("ok") is True
        assert result.get("uneven") is True
