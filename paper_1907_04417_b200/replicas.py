"""Multi-GPU plumbing for the benchmark: one process per GPU (torchrun
environment), process-group set-up, barriers and the max-over-ranks of device
times.  The row-partitioned solve itself is paper_1907_04417_b200.distributed.
Backend "nccl" on GPUs, "gloo" in the CPU tests."""

import os


def world():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend, device=None):
    """Initialise the default process group when world_size > 1; returns the
    torch.distributed module or None for a single process."""
    ws, _, _ = world()
    if ws <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl" and device is not None:
        dist.init_process_group(backend, device_id=device)
    else:
        dist.init_process_group(backend)
    return dist


def max_over_ranks(value, dist, device="cpu"):
    """Max of a float over all ranks (identity without a process group)."""
    if dist is None:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def parallelism(world_size):
    return "single GPU" if world_size == 1 else f"{world_size} independent replicas (one per GPU)"


def whole_job_rate(units_per_rank, world_size, t_max):
    """Units processed by all ranks divided by the slowest rank's time."""
    return units_per_rank * world_size / t_max
