"""Multi-GPU Monte Carlo: samples shard across ranks, one process per GPU.

The reference's only parallelism is a std::thread pool over sample indices
(montecarlo.cpp:218-245). Here each rank (GPU) takes a contiguous range of
GLOBAL sample indices -- [g*ceil(n/G), min(n, (g+1)*ceil(n/G)))
-- and every random stream is keyed by the global index, so records are
bitwise independent of the number of GPUs. The data path has no collective;
the single exchange is the final gather of the 24-byte per-sample records,
done by the library itself over NCCL (nmpcmc_gpu_run_sharded), after which
K4 computes aggregate_stats in index order exactly like the single-process
call. shard() and gather_records() restate the sharding / gather contract
in Python for the multi-process CPU tests (gloo).
"""
from typing import Optional, Tuple

import numpy as np

from . import abi


def shard(n_sims: int, rank: int, world: int) -> Tuple[int, int]:
    """(first, count) of this rank's contiguous global index range."""
    if n_sims < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard request")
    per = -(-n_sims // world)
    first = min(n_sims, rank * per)
    last = min(n_sims, first + per)
    return first, last - first


def gather_records(local: np.ndarray, n_sims: int, rank: int, world: int, device=None) -> Optional[np.ndarray]:
    """All-gather every rank's records (index order) with torch.distributed;
    returns the full array on every rank. `device` = torch device for NCCL
    (None -> CPU tensors for gloo)."""
    import torch
    import torch.distributed as dist

    per = -(-n_sims // world)
    buf = np.zeros(per, dtype=abi.RECORD_DTYPE)
    buf[: len(local)] = local
    t = torch.from_numpy(buf.view(np.uint8).copy())
    if device is not None:
        t = t.to(device)
    out = torch.empty(world * t.numel(), dtype=torch.uint8, device=t.device)
    dist.all_gather_into_tensor(out, t)
    allrec = np.frombuffer(out.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)
    return allrec[:n_sims].copy()


def run_monte_carlo_distributed(sc, n_sims: int, local_rank: Optional[int] = None, counters: bool = False):
    """run_monte_carlo over all ranks of the default process group, one GPU
    per rank. The data path and the exchange are the library's own C++
    (nmpcmc_gpu_comm_init + nmpcmc_gpu_run_sharded): each rank runs its
    contiguous block, the 24 B records are all-gathered and the work counters
    all-reduced over NCCL inside the library, and K4 computes the aggregate on
    the device. torch.distributed only ships the 128-byte NCCL id from rank 0
    (out of band, as NCCL expects). Every rank returns the same McResult;
    `counters` returns the all-reduced totals dict instead of per-sample rows."""
    import time

    import torch
    import torch.distributed as dist

    from . import engine

    rank, world = dist.get_rank(), dist.get_world_size()
    dev = local_rank if local_rank is not None else torch.cuda.current_device()
    ctx = engine.Context(dev)
    box = [engine.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    ctx.comm_init(box[0], rank, world)
    dist.barrier()
    t0 = time.perf_counter()
    allrec, agg = ctx.run_sharded(sc, 0, n_sims)
    wall = time.perf_counter() - t0
    totals = ctx.last_totals() if counters else None
    return engine.McResult(allrec, agg, wall, totals, 0)
