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
    """What bench.py --gpus N runs: N = 1 one GPU; N > 1 the row-partitioned
    solve of paper_1907_04417_b200.distributed."""
    if world_size == 1:
        return "single GPU"
    return (f"row-partitioned fine level over {world_size} GPUs (nnz-balanced contiguous row blocks, NCCL halo "
            "exchanges, exact-order Gauss-Seidel pipelined across ranks); coarse levels gathered to GPU 0")
