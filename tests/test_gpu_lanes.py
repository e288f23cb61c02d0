"""Pipelined batches (NMPCMC_OPT_LANES = 2): consecutive NMPC/PI launches on
alternating internal streams with separate workspaces give exactly the records
of serial execution, through the device and the async host entry points."""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import assert_records_equal
from paper_2212_02197_b200 import abi, configs

pytestmark = pytest.mark.gpu


def _dev_records(buf):
    return np.frombuffer(buf.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)


def test_lanes_device_path_matches_serial(gpu_ctx):
    sc_n = configs.make_scenario("nmpc", N=30, n_steps=30, perturb=True)
    sc_p = configs.make_scenario("pi", perturb=True)
    want = [gpu_ctx.run(sc, first, 700)[0] for first in (0, 700, 1400) for sc in (sc_n, sc_p)]
    rsz = C.sizeof(abi.SimRecord)
    bufs = [torch.empty(700 * rsz, dtype=torch.uint8, device="cuda") for _ in range(6)]
    torch.cuda.synchronize()  # buffers allocated on torch's stream
    gpu_ctx.set_lanes(2)
    try:
        k = 0
        for first in (0, 700, 1400):
            for sc in (sc_n, sc_p):
                gpu_ctx.run_device(sc, first, 700, bufs[k].data_ptr())
                k += 1
        gpu_ctx.wait()
    finally:
        gpu_ctx.set_lanes(1)
    for got, w in zip(bufs, want):
        assert_records_equal(_dev_records(got), w)


def test_lanes_async_host_path_matches_serial(gpu_ctx):
    sc = configs.make_scenario("nmpc", N=30, n_steps=20, perturb=True)
    want = [gpu_ctx.run(sc, first, 500)[0] for first in (0, 500, 1000)]
    rsz = C.sizeof(abi.SimRecord)
    host = [torch.empty(500 * rsz, dtype=torch.uint8).pin_memory() for _ in range(3)]
    gpu_ctx.set_lanes(2)
    try:
        for i, first in enumerate((0, 500, 1000)):
            gpu_ctx.run_async(sc, first, 500, host[i].data_ptr())
        gpu_ctx.wait()
    finally:
        gpu_ctx.set_lanes(1)
    for h, w in zip(host, want):
        assert_records_equal(np.frombuffer(h.numpy().tobytes(), dtype=abi.RECORD_DTYPE), w)
