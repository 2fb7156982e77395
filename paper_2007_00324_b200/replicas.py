"""Multi-GPU = independent replicas: one process per GPU, one
mesh per process, no data-path collective.  torch.distributed (gloo, host
side: north_star says no NCCL) is used only for the barrier and the max/sum
of per-rank timings, which are taken on each device with CUDA events."""
from __future__ import annotations

import os


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def assign(n_items: int, world: int, rank: int) -> list[int]:
    """Round-robin assignment of independent PSLGs to ranks (config 5)."""
    return list(range(rank, n_items, world))


def replica_seed(base: int, rank: int, item: int = 0) -> int:
    """Distinct PSLG per replica: seed + rank (+ 1000 * item for several per rank)."""
    return base + rank + 1000 * item


class Dist:
    """Barrier + max/sum of host floats over ranks; a no-op for world == 1."""

    def __init__(self, world: int, rank: int, local: int, backend: str = "gloo"):
        self.world, self.rank, self.local, self.backend = world, rank, local, backend
        if world > 1:
            import torch
            import torch.distributed as td
            self.td = td
            if backend == "nccl":
                torch.cuda.set_device(local)
                td.init_process_group("nccl", device_id=torch.device("cuda", local))
                self.dev = torch.device("cuda", local)
            else:
                td.init_process_group(backend)
                self.dev = torch.device("cpu")

    def barrier(self) -> None:
        if self.world > 1:
            self.td.barrier()

    def _reduce(self, x: float, op) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        self.td.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        return self._reduce(x, self.td.ReduceOp.MAX if self.world > 1 else None)

    def sum(self, x: float) -> float:
        return self._reduce(x, self.td.ReduceOp.SUM if self.world > 1 else None)

    def close(self) -> None:
        if self.world > 1:
            self.td.destroy_process_group()


def throughput(steiner_total: float, seconds_max: float) -> float:
    """Whole-job Steiner points/s: all ranks' points over the slowest rank's time."""
    return steiner_total / seconds_max if seconds_max > 0 else 0.0
