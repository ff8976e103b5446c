"""Multi-GPU shot scheduler: one process per GPU, shots sharded in contiguous
blocks, one all-reduce of (gradient, misfit) per gradient evaluation.

The reference's only parallelism is a thread map over shots with a
deterministic pairwise reduction (seisopt/gradients.py:91-95, :40-50,
:150-152).  Here each rank owns a contiguous block of shots, runs them as one
batched launch sequence on its GPU, folds its partial image locally (fold_pad
is linear, so it commutes with the sum) and joins the others with a single
``all_reduce`` over NCCL (NVLink/NVSwitch) -- or gloo in CPU tests.  The AA
optimizer state is replicated: every rank holds the identical reduced
gradient, so no broadcast is needed.
"""

from __future__ import annotations

from dataclasses import dataclass


def shard_bounds(n_shots: int, world: int, rank: int):
    """Contiguous block of shots for ``rank``: sizes differ by at most one,
    the first ``n_shots % world`` ranks take the extra shot."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_shots, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start, count


@dataclass
class ShotShard:
    shot0: int
    count: int
    rank: int = 0
    world: int = 1
    group: object = None

    @staticmethod
    def from_env(n_shots: int, group=None):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            world, rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            world, rank = 1, 0
        s0, cnt = shard_bounds(n_shots, world, rank)
        if cnt == 0:
            raise ValueError(f"rank {rank} owns no shots ({n_shots} shots over {world} ranks)")
        return ShotShard(s0, cnt, rank, world, group)

    def _dist(self):
        import torch.distributed as dist
        return dist if (self.world > 1 and dist.is_initialized()) else None

    def allreduce_(self, tensor):
        dist = self._dist()
        if dist is not None:
            dist.all_reduce(tensor, group=self.group)
        return tensor

    def allreduce_value(self, value: float) -> float:
        import torch
        dist = self._dist()
        if dist is None:
            return float(value)
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, group=self.group)
        return float(t.item())

    def allreduce_value_grad(self, value: float, grad) -> float:
        """Gradient summed in place over the ranks, misfit summed in fp64.

        fp64 gradients carry the misfit in the same buffer (one collective,
        exact).  fp32 gradients are reduced in their own dtype and the misfit
        in a separate fp64 all-reduce, so the value handed to the optimizer's
        Armijo test has the same precision as FwiObjective.value's."""
        import torch
        dist = self._dist()
        if dist is None:
            return float(value)
        flat = grad.reshape(-1)
        if grad.dtype == torch.float64:
            n = flat.numel()
            buf = torch.empty(n + 1, dtype=grad.dtype, device=grad.device)
            buf[:n].copy_(flat)
            buf[n] = float(value)
            dist.all_reduce(buf, group=self.group)
            flat.copy_(buf[:n])
            return float(buf[n].item())
        dist.all_reduce(flat, group=self.group)
        return self.allreduce_value(value)
