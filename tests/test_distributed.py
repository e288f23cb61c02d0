"""Multi-rank host logic on CPU (gloo, world_size 2): shard ranges, record
gather and the rank-0 aggregate equal the single-process reference result.
Records come from the CPU oracle here (no GPU); on GPUs the same gather runs
over NCCL (bench.py, distributed.run_monte_carlo_distributed)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, assert_records_equal, load_golden
from paper_2212_02197_b200 import distributed


@pytest.mark.parametrize("n,world", [(10, 2), (11, 2), (7, 3), (1, 4), (0, 2), (30000, 8)])
def test_shard_ranges_cover_exactly(n, world):
    seen = []
    for r in range(world):
        first, count = distributed.shard(n, r, world)
        seen.extend(range(first, first + count))
    assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from conftest import load_golden as lg
    from oracle import lib as O
    from paper_2212_02197_b200 import distributed as D
    from paper_2212_02197_b200 import engine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, _, sc = lg("pi_cfg1")
    n = 50
    first, count = D.shard(n, rank, world)
    # per-rank records from the CPU oracle on this rank's global index range
    rec, _ = O.run_batch(O.ref("xlibm"), sc, first, count, 2) if count else (np.zeros(0, dtype=d["rec_xlibm"].dtype), 0)
    allrec = D.gather_records(rec, n, rank, world, device=None)
    agg = engine.aggregate_stats(allrec)
    np.save(os.path.join(out_dir, f"rec{rank}.npy"), allrec)
    np.save(os.path.join(out_dir, f"agg{rank}.npy"), np.array([agg["mean"], agg["variance"], agg["n_failed"]]))
    dist.destroy_process_group()


@pytest.mark.skipif(not __import__("oracle.lib", fromlist=["x"]).ref_available() and not os.path.isdir("/root/reference"),
                    reason="oracle/_ref not built")
def test_gloo_two_ranks_gather_equals_single_process(tmp_path):
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn")
    d, _, _ = load_golden("pi_cfg1")
    want = d["rec_xlibm"][:50]
    from paper_2212_02197_b200 import engine
    agg = engine.aggregate_stats(want)
    for r in range(world):
        got = np.load(tmp_path / f"rec{r}.npy")
        assert_records_equal(got, want)
        a = np.load(tmp_path / f"agg{r}.npy")
        assert a[0] == agg["mean"] and a[1] == agg["variance"] and a[2] == agg["n_failed"]


@pytest.mark.parametrize("n,world", [(10, 2), (11, 2), (7, 3), (1, 4), (0, 2), (30000, 8), (1000003, 7)])
def test_c_abi_shard_range_matches_python(n, world):
    """nmpcmc_gpu_shard_range (the C++ multi-device / multi-rank split) is
    the same contiguous split as distributed.shard."""
    from paper_2212_02197_b200 import engine
    for r in range(world):
        assert engine.shard_range(n, r, world) == distributed.shard(n, r, world)


def test_multi_device_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2212_02197_b200 import engine
    with pytest.raises(engine.CudaError):
        engine.Context(devices=[0, 1])
