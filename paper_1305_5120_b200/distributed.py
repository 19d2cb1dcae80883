"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL on B200).

The filter is column-separable (core.py:276-283 touches each column on its
own), so the active block is split into contiguous column ranges exactly like
the reference's worker tiles (linalg.py:238-243: bounds[i] = s*i // workers),
H is replicated on every rank and there is no communication inside the
filter. After the filter the shards are all-gathered (NCCL over NVLink) for
CholQR and Rayleigh-Ritz.

All collectives here are plain torch.distributed calls, so the same code runs
on CPU tensors under the gloo backend in the tests (world_size 2).
"""

import torch
import torch.distributed as dist


class ColumnShards:
    """Contiguous split of k columns over ``world`` ranks."""

    def __init__(self, k, world):
        if k < 0 or world < 1:
            raise ValueError("need k >= 0 and world >= 1")
        self.k = int(k)
        self.world = int(world)
        self.bounds = [(self.k * i) // self.world for i in range(self.world + 1)]
        self.widths = [self.bounds[i + 1] - self.bounds[i] for i in range(self.world)]
        self.padded = max(self.widths) if self.widths else 0

    def range(self, rank):
        return self.bounds[rank], self.bounds[rank + 1]

    def owner(self, col):
        for r in range(self.world):
            if self.bounds[r] <= col < self.bounds[r + 1]:
                return r
        raise IndexError(col)

    def all_gather(self, local, gathered, group=None):
        """All-gather (width_r, n) shards into ``gathered`` (padded * world, n).

        Column-major blocks are (cols, rows) tensors, so a shard is a contiguous
        row range and the gather is one flat all_gather_into_tensor."""
        if self.world == 1:
            gathered[: local.shape[0]].copy_(local)
            return gathered
        rank = dist.get_rank(group)
        w = self.widths[rank]
        if local.shape[0] != w:
            raise ValueError(f"rank {rank} shard has {local.shape[0]} columns, expected {w}")
        if w == self.padded and local.is_contiguous():
            send = local
        else:
            send = torch.zeros((self.padded, local.shape[1]), dtype=local.dtype, device=local.device)
            send[:w].copy_(local)
        dist.all_gather_into_tensor(gathered, send, group=group)
        return gathered

    def compact(self, gathered, out):
        """Drop the padding: out (k, n) <- gathered shards in column order."""
        for r in range(self.world):
            lo, hi = self.bounds[r], self.bounds[r + 1]
            out[lo:hi].copy_(gathered[r * self.padded: r * self.padded + (hi - lo)])
        return out

    def gather_block(self, local, group=None):
        """Convenience: full (k, n) block from every rank's shard."""
        n = local.shape[1]
        g = torch.empty((self.padded * self.world, n), dtype=local.dtype, device=local.device)
        self.all_gather(local, g, group)
        out = torch.empty((self.k, n), dtype=local.dtype, device=local.device)
        return self.compact(g, out)


def all_gather_values(vals, shards, group=None):
    """Gather per-rank 1-D float64 vectors (e.g. residual norms of own columns)."""
    if shards.world == 1:
        return vals
    rank = dist.get_rank(group)
    w = shards.widths[rank]
    send = torch.zeros(shards.padded, dtype=torch.float64, device=vals.device)
    send[:w].copy_(vals[:w])
    recv = torch.empty(shards.padded * shards.world, dtype=torch.float64, device=vals.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    out = torch.empty(shards.k, dtype=torch.float64, device=vals.device)
    for r in range(shards.world):
        lo, hi = shards.range(r)
        out[lo:hi].copy_(recv[r * shards.padded: r * shards.padded + hi - lo])
    return out
