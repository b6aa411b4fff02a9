"""Multi-process (gloo, CPU) tests of the batch-sharded inference path
(paper_2008_05101_b200/shard.py).  The per-rank network is the C oracle's
ternary body (CPU stand-in for the GPU body, which is tested bit-exact against
the same oracle in test_gpu_net.py) followed by a global-average pool; the
gathered rows on rank 0 must equal the unsharded run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_05101_b200.shard import ShardedForward, max_shard, shard_range
from tests.netspec import tiny_body


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _body_forward(blocks, c, h, w):
    from oracle.oracle import Oracle
    O = Oracle()

    def fwd(x: torch.Tensor) -> torch.Tensor:
        n = x.shape[0]
        if n == 0:
            return torch.zeros((0, blocks[-1]["convs"][-1]["out_c"]), dtype=torch.float32)
        st, out = O.net_body(blocks, x.numpy(), n, c, h, w)
        assert st == 0
        return torch.from_numpy(out.reshape(n, out.shape[1], -1).mean(axis=2, dtype=np.float32))
    return fwd


def _worker(rank, world, port, batch, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blocks, (_, c, h, w), _ = tiny_body(seed=3, n=1)
        rng = np.random.default_rng(11)
        x = torch.from_numpy(np.abs(rng.standard_normal((batch, c, h, w))).astype(np.float32))
        fwd = _body_forward(blocks, c, h, w)
        out_dim = blocks[-1]["convs"][-1]["out_c"]
        sf = ShardedForward(fwd, batch, out_dim, rank, world)
        y = sf(sf.local_slice(x).contiguous())
        if rank == 0:
            ref = fwd(x)
            np.save(result_path, np.stack([y.numpy(), ref.numpy()]))
        else:
            assert y is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(2, 5), (2, 4), (3, 2)])
def test_sharded_body_equals_unsharded(tmp_path, world, batch):
    path = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(world, _free_port(), batch, path), nprocs=world, join=True)
    got, want = np.load(path)
    assert got.shape == (batch, want.shape[1])
    assert np.array_equal(got.view(np.int32), want.view(np.int32))


def test_shard_ranges_partition_the_batch():
    for world in range(1, 9):
        for batch in range(0, 40):
            shards = [shard_range(batch, r, world) for r in range(world)]
            assert sum(s.count for s in shards) == batch
            pos = 0
            for s in shards:
                assert s.start == pos and 0 <= s.count <= max_shard(batch, world)
                pos += s.count
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    # cfg5: ResNet-50 batch 1024 over 1/2/4/8 GPUs -> 1024/512/256/128 per GPU
    assert [shard_range(1024, 0, g).count for g in (1, 2, 4, 8)] == [1024, 512, 256, 128]
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_gather_rejects_wrong_shard_shape():
    sf = ShardedForward(lambda x: x, 4, 3, 0, 1)
    with pytest.raises(ValueError):
        sf.gather(torch.zeros(3, 3))
    assert sf.gather(torch.ones(4, 3)).shape == (4, 3)
