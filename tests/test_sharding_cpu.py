"""Host-side logic of the by-molecule multi-GPU driver, exercised on CPU with gloo, world size 2.

The per-rank evaluation is replaced by a cheap deterministic function of the local atoms (the
real one needs a GPU); what is tested is the partition, the re-based batch codes, and that the
gathered result equals the single-rank result (batch independence)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_17660_b200 import sharding, synth


def fake_step(z, pos, batch, box):
    """Per-sample 'energy' = sum of |r - centroid|^2 * z, 'forces' = pos * z: local per molecule."""
    z = np.asarray(z, dtype=np.float64)
    pos = np.asarray(pos, dtype=np.float64)
    batch = np.asarray(batch)
    assert batch[0] == 0 and np.all(np.diff(batch) >= 0) and np.all(np.diff(batch) <= 1)
    ns = int(batch[-1]) + 1
    cent = np.stack([np.bincount(batch, weights=pos[:, k], minlength=ns) for k in range(3)], 1)
    cent /= np.bincount(batch, minlength=ns)[:, None]
    e = np.bincount(batch, weights=((pos - cent[batch]) ** 2).sum(1) * z, minlength=ns)
    return torch.tensor(e, dtype=torch.float32), torch.tensor(pos * z[:, None], dtype=torch.float32)


def test_partition_tiles_the_batch_and_balances_atoms():
    _, pos, batch, _ = synth.config_d_molecules(97, seed=1)
    for world in (1, 2, 3, 4, 8):
        shards = sharding.shard_by_molecule(batch, world)
        assert shards[0][0] == 0 and shards[-1][1] == len(batch)
        assert shards[0][2] == 0 and shards[-1][3] == int(batch[-1]) + 1
        for a, b in zip(shards[:-1], shards[1:]):
            assert a[1] == b[0] and a[3] == b[2]
        atoms = np.array([s[1] - s[0] for s in shards])
        assert atoms.min() > 0 and atoms.max() - atoms.min() <= 2 * 24
        for a0, a1, s0, s1 in shards:
            assert batch[a0] == s0 and batch[a1 - 1] == s1 - 1      # whole molecules only


def test_more_ranks_than_molecules():
    batch = np.array([0, 0, 0, 1, 1])
    shards = sharding.shard_by_molecule(batch, 4)
    assert shards[0][0] == 0 and shards[-1][1] == 5
    assert sum(s[1] - s[0] for s in shards) == 5


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z, pos, batch, _ = synth.config_d_molecules(41, seed=3)
    e, f = sharding.evaluate_sharded(fake_step, z, pos, batch, None, device="cpu")
    # the resident form used by bench.py (buffers allocated once, all_gather_into_tensor)
    z_l, pos_l, b_l, _ = sharding.local_shard(z, pos, batch, rank, world)
    gather = sharding.ResidentGather(batch, world, rank, "cpu")
    for _ in range(2):
        e2, f2 = gather(*fake_step(z_l, pos_l, b_l, None))
    assert torch.equal(e, e2) and torch.equal(f, f2)
    if rank == 0:
        torch.save((e, f), out)
    dist.destroy_process_group()


def test_gathered_result_equals_single_rank(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    e, f = torch.load(out)
    z, pos, batch, _ = synth.config_d_molecules(41, seed=3)
    e_ref, f_ref = fake_step(z, pos, batch, None)
    assert torch.equal(e, e_ref) and torch.equal(f, f_ref)
