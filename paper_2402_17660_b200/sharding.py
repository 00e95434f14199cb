"""Batched inference sharded by whole molecules over the GPUs of one node.

Samples never interact (cross-batch pairs are rejected in the pair kernels,
``_neighbor_kernels.py:36,134,210``; energies are per-sample sums, ``graphnet.py:411``), so the
batch is cut into contiguous ranges of whole molecules balanced on atom count, every rank
evaluates its range with its own replica of the weights, and there is NO collective in the
step: one ``all_gather`` at the end returns the per-sample energies and per-atom forces to
every rank.  A single large periodic system does not shard ("replicas only").
"""

from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def shard_by_molecule(batch, world_size: int) -> List[Tuple[int, int, int, int]]:
    """Contiguous molecule ranges balanced on atom count.

    Returns one ``(atom_start, atom_end, sample_start, sample_end)`` per rank; every rank gets
    at least one molecule when there are enough, ranges tile the batch exactly."""
    batch = np.asarray(batch)
    n_samples = int(batch[-1]) + 1
    sizes = np.bincount(batch, minlength=n_samples)
    cum = np.concatenate([[0], np.cumsum(sizes)])
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, world_size):
        target = total * r / world_size
        s = int(np.searchsorted(cum, target, side="left"))
        lo = cuts[-1] + 1 if n_samples - cuts[-1] > world_size - r else cuts[-1]
        hi = n_samples - (world_size - r)
        cuts.append(int(min(max(s, lo), max(hi, cuts[-1]))))
    cuts.append(n_samples)
    return [(int(cum[cuts[r]]), int(cum[cuts[r + 1]]), cuts[r], cuts[r + 1]) for r in range(world_size)]


def local_shard(species, positions, batch, rank: int, world_size: int):
    """This rank's atoms with batch codes re-based to start at 0 (system.py:231-235)."""
    a0, a1, s0, s1 = shard_by_molecule(batch, world_size)[rank]
    batch = np.asarray(batch)
    return (np.asarray(species)[a0:a1], np.asarray(positions)[a0:a1], batch[a0:a1] - s0,
            (a0, a1, s0, s1))


def evaluate_sharded(step: Callable, species, positions, batch, box=None, group=None,
                     device: Optional[str] = None):
    """Evaluate a batch of molecules across the ranks of ``torch.distributed``.

    ``step(z, pos, batch, box) -> (energy[n_local_samples], forces[n_local_atoms, 3])`` is the
    per-rank evaluation (``TensorNet.forward`` on the GPU).  Returns the full
    ``(energy[n_samples], forces[N, 3])`` on every rank, gathered once at the end."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shards = shard_by_molecule(batch, world)
    z_l, pos_l, b_l, (a0, a1, s0, s1) = local_shard(species, positions, batch, rank, world)
    if a1 > a0:
        e_l, f_l = step(z_l, pos_l, b_l, box)
        e_l, f_l = torch.as_tensor(e_l), torch.as_tensor(f_l)
    else:
        e_l, f_l = torch.zeros(0), torch.zeros((0, 3))
    if world == 1:
        return e_l, f_l
    dev = e_l.device if device is None else torch.device(device)
    n_samples = int(np.asarray(batch)[-1]) + 1
    n_atoms = len(np.asarray(batch))
    max_s = max(s[3] - s[2] for s in shards)
    max_a = max(s[1] - s[0] for s in shards)
    e_pad = torch.zeros(max_s, dtype=torch.float32, device=dev)
    f_pad = torch.zeros((max_a, 3), dtype=torch.float32, device=dev)
    e_pad[: s1 - s0] = e_l.to(dev, torch.float32)
    f_pad[: a1 - a0] = f_l.to(dev, torch.float32)
    e_all = [torch.empty_like(e_pad) for _ in range(world)]
    f_all = [torch.empty_like(f_pad) for _ in range(world)]
    dist.all_gather(e_all, e_pad, group=group)
    dist.all_gather(f_all, f_pad, group=group)
    energy = torch.empty(n_samples, dtype=torch.float32, device=dev)
    forces = torch.empty((n_atoms, 3), dtype=torch.float32, device=dev)
    for r, (ra0, ra1, rs0, rs1) in enumerate(shards):
        energy[rs0:rs1] = e_all[r][: rs1 - rs0]
        forces[ra0:ra1] = f_all[r][: ra1 - ra0]
    return energy, forces


class ResidentGather:
    """The gather at the end of a sharded step with every buffer allocated once: ``__call__`` takes
    this rank's energies/forces (device tensors) and returns the full ``(energy[n_samples],
    forces[N, 3])`` on every rank.  Two ``all_gather_into_tensor`` calls on padded per-rank slots
    (ranks hold different atom counts), then the slots are packed; no host synchronisation, so a
    benchmark can time K steps back to back with the collective inside the timed region."""

    def __init__(self, batch, world_size: int, rank: int, device, group=None):
        import torch

        self.torch, self.group, self.world, self.rank = torch, group, world_size, rank
        batch = np.asarray(batch)
        self.shards = shard_by_molecule(batch, world_size)
        self.n_samples, self.n_atoms = int(batch[-1]) + 1, len(batch)
        self.max_s = max(s[3] - s[2] for s in self.shards)
        self.max_a = max(s[1] - s[0] for s in self.shards)
        f32 = dict(dtype=torch.float32, device=device)
        self.e_pad = torch.zeros(self.max_s, **f32)
        self.f_pad = torch.zeros((self.max_a, 3), **f32)
        self.e_all = torch.empty(world_size * self.max_s, **f32)
        self.f_all = torch.empty((world_size * self.max_a, 3), **f32)
        self.energy = torch.empty(self.n_samples, **f32)
        self.forces = torch.empty((self.n_atoms, 3), **f32)

    def __call__(self, e_local, f_local):
        import torch.distributed as dist

        a0, a1, s0, s1 = self.shards[self.rank]
        self.e_pad[: s1 - s0].copy_(e_local, non_blocking=True)
        self.f_pad[: a1 - a0].copy_(f_local, non_blocking=True)
        if self.world > 1:
            dist.all_gather_into_tensor(self.e_all, self.e_pad, group=self.group)
            dist.all_gather_into_tensor(self.f_all, self.f_pad, group=self.group)
        else:
            self.e_all.copy_(self.e_pad)
            self.f_all.copy_(self.f_pad)
        for r, (ra0, ra1, rs0, rs1) in enumerate(self.shards):
            self.energy[rs0:rs1] = self.e_all[r * self.max_s: r * self.max_s + rs1 - rs0]
            self.forces[ra0:ra1] = self.f_all[r * self.max_a: r * self.max_a + ra1 - ra0]
        return self.energy, self.forces
