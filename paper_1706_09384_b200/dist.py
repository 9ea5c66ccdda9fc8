"""Multi-process plumbing for ``bench.py --gpus N`` (one process per GPU).

The H-matvec path runs as independent replicas (the
north star is one GPU; block-row sharding with an all-gather of y is the
recorded next step), so the only collective is the timing reduction: the
device time of the K steps is the MAX over ranks and the aggregate throughput
is (ranks x K x bytes) / that time.
"""

import torch
import torch.distributed as dist


def max_over_ranks(value, device):
    """Max of a float over all ranks (identity when not distributed)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(ms_local, bytes_per_step, steps, device):
    """(aggregate GB/s, max ms) for replicas each doing ``steps`` steps."""
    ws = dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1
    ms = max_over_ranks(ms_local, device)
    return ws * steps * bytes_per_step / (ms * 1e-3) / 1e9, ms
