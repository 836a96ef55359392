"""Replica parallelism for N GPUs.

The path shards only by rows with a per-frame boundary exchange (SURVEY
§8e); until that is built, N GPUs run N independent replicas -- one process
per GPU, each compressing its own field -- and the only collectives are the
barrier around the timed region and the max over ranks of the device time.
These helpers are backend-agnostic so the same code runs under NCCL on the
GPU box and under gloo in the CPU tests.
"""

from __future__ import annotations


def rank_world(env=None):
    import os
    env = os.environ if env is None else env
    return int(env.get("RANK", "0")), int(env.get("WORLD_SIZE", "1"))


def barrier(dist=None, cuda=True):
    if cuda:
        import torch
        torch.cuda.synchronize()
    if dist is not None and dist.is_initialized():
        dist.barrier()
        if cuda:
            import torch
            torch.cuda.synchronize()


def max_over_ranks(x: float, dist=None, device="cuda") -> float:
    """Max of a per-rank scalar (device times are reported as the max)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, dist=None, device="cuda") -> float:
    """Whole-job totals (units processed by all replicas)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
