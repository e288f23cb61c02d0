"""K4 (statistics on the device) and the multi-GPU C-ABI paths on one B200.

- K4: aggregate_stats / phi_histogram of device-resident records are bitwise
  the reference's host results (montecarlo.cpp:172-211, :268-304);
- multi-device context (nmpcmc_gpu_ctx_create_multi): records are bitwise
  independent of the device list -- [0] exercises a one-rank NCCL-free
  path, [0, 0, 0] three blocks on one GPU with the peer-copy gather --
  and the aggregate equals the single-device one;
- one-process-per-GPU form (comm_init + run_sharded) with one rank.
The NCCL all-gather over distinct GPUs needs >1 GPU; the driver's runs get
one, so it is exercised only on multi-GPU boxes (test skips otherwise)."""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import assert_records_equal, load_golden
from oracle import lib as O
from paper_2212_02197_b200 import abi, configs, engine

pytestmark = pytest.mark.gpu


def _ref_agg(rec):
    """aggregate_stats of the reference build itself (oracle/_ref)."""
    L = O.ref("glibc")
    out = abi.Aggregate()
    L.nmpcmc_ref_aggregate(rec.ctypes.data_as(C.POINTER(abi.SimRecord)), len(rec), C.byref(out))
    return abi.aggregate_to_dict(out)


def _same_agg(a, b):
    for k in a:
        va, vb = np.asarray(a[k], dtype=float), np.asarray(b[k], dtype=float)
        np.testing.assert_array_equal(va, vb, err_msg=k)


def _records_dev(rec):
    t = torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8).copy()).cuda()
    return t


@pytest.mark.parametrize("name", ["pi_cfg1", "nmpc_n30_short", "nmpc_cfg3_full"])
def test_k4_aggregate_and_histogram_bitwise(gpu_ctx, name):
    try:
        d, _, _ = load_golden(name)
    except FileNotFoundError:
        pytest.skip(f"{name} fixture absent")
    rec = np.ascontiguousarray(d["rec_glibc"])
    t = _records_dev(rec)
    for bins in (0, 7):
        agg, h = gpu_ctx.aggregate_device(t.data_ptr(), len(rec), bins=bins)
        _same_agg(agg, engine.aggregate_stats(rec))
        _same_agg(agg, _ref_agg(rec))
        want = engine.phi_histogram(rec["phi"], bins)
        np.testing.assert_array_equal(h.edges, want.edges)
        np.testing.assert_array_equal(h.counts, want.counts)


def test_k4_edge_cases(gpu_ctx):
    """All failed, a single sample, ties, a non-failed infinite phi."""
    base = np.zeros(5, dtype=abi.RECORD_DTYPE)
    cases = []
    a = base.copy(); a["failed"] = 1; a["phi"] = np.nan; cases.append(a)            # all failed
    b = base[:1].copy(); b["phi"] = 3.5; cases.append(b)                               # one sample
    c = base.copy(); c["phi"] = 2.0; cases.append(c)                                   # all equal
    e = base.copy(); e["phi"] = [1.0, np.inf, 2.0, 2.0, 0.5]; cases.append(e)          # inf, not failed
    f = base.copy(); f["phi"] = [1e300, 1e-300, 0.0, 7.0, 1e300]; f["ocp_solves"] = 720; f["ocp_failures"] = [0, 1, 2, 3, 700]
    cases.append(f)
    for rec in cases:
        t = _records_dev(rec)
        agg, h = gpu_ctx.aggregate_device(t.data_ptr(), len(rec), bins=0)
        _same_agg(agg, engine.aggregate_stats(rec))
        want = engine.phi_histogram(rec["phi"], 0)
        np.testing.assert_array_equal(h.edges, want.edges)
        np.testing.assert_array_equal(h.counts, want.counts)


def test_k4_large_random_matches_host(gpu_ctx):
    rng = np.random.default_rng(5)
    n = 300_001
    rec = np.zeros(n, dtype=abi.RECORD_DTYPE)
    rec["phi"] = rng.lognormal(3.0, 1.5, n)
    fail = rng.uniform(size=n) < 0.3
    rec["failed"] = fail
    rec["phi"][fail] = np.nan
    rec["ocp_solves"] = rng.integers(0, 720, n)
    rec["ocp_failures"] = rec["ocp_solves"] // 7
    t = _records_dev(rec)
    agg, h = gpu_ctx.aggregate_device(t.data_ptr(), n, bins=0)
    _same_agg(agg, engine.aggregate_stats(rec))
    want = engine.phi_histogram(rec["phi"], 0)
    np.testing.assert_array_equal(h.edges, want.edges)
    np.testing.assert_array_equal(h.counts, want.counts)


def test_run_aggregate_is_device_k4(gpu_ctx):
    d, _, sc = load_golden("pi_cfg0")
    rec, cnt, agg = gpu_ctx.run(sc, 0, 256, counters=True, aggregate=True)
    assert_records_equal(rec, d["rec_xlibm"])
    _same_agg(agg, engine.aggregate_stats(d["rec_xlibm"]))
    tot = gpu_ctx.last_totals()
    assert tot["control_steps"] == int(cnt["control_steps"].sum())
    h = gpu_ctx.histogram_last(0)
    want = engine.phi_histogram(d["rec_xlibm"]["phi"], 0)
    np.testing.assert_array_equal(h.edges, want.edges)
    np.testing.assert_array_equal(h.counts, want.counts)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("name,n", [("pi_cfg1", 256), ("nmpc_n30_short", 64)])
def test_multi_device_context_bitwise(devices, name, n):
    d, _, sc = load_golden(name)
    ctx = engine.Context(devices=devices)
    assert ctx.num_devices == len(devices)
    assert not ctx.uses_nccl  # one GPU: blocks gathered with peer copies
    rec, cnt, agg = ctx.run(sc, int(d["first"]), n, counters=True, aggregate=True)
    assert_records_equal(rec, d["rec_xlibm"][:n])
    _same_agg(agg, engine.aggregate_stats(d["rec_xlibm"][:n]))
    tot = ctx.last_totals()
    for k in ("control_steps", "shoot_full", "ipm_stage_iters", "qp_solves"):
        assert tot[k] == int(cnt[k].sum()), k
    # async form over the same blocks
    host = torch.empty(n * 24, dtype=torch.uint8).pin_memory()
    ctx.run_async(sc, int(d["first"]), n, host.data_ptr())
    ctx.wait()
    assert_records_equal(np.frombuffer(host.numpy().tobytes(), dtype=abi.RECORD_DTYPE), d["rec_xlibm"][:n])
    ctx.close()


def test_multi_device_traj_sharded():
    d, kw, _ = load_golden("pi_cfg0")
    sc = configs.make_scenario(**kw, record=True)
    one = engine.Context(0)
    r1, t1 = one.run_traj(sc, 0, 5)
    multi = engine.Context(devices=[0, 0])
    r2, t2 = multi.run_traj(sc, 0, 5)
    assert_records_equal(r2, r1)
    np.testing.assert_array_equal(t2, t1)
    np.testing.assert_array_equal(t1[:len(d["traj_xlibm"])], d["traj_xlibm"])


def test_run_sharded_single_rank_with_nccl_id():
    """One rank: comm_init(nranks=1) and run_sharded == run (the NCCL id path
    of the multi-process launch)."""
    d, _, sc = load_golden("pi_cfg1")
    ctx = engine.Context(0)
    uid = engine.nccl_unique_id()
    assert len(uid) == 128
    ctx.comm_init(uid, 0, 1)
    rec, agg = ctx.run_sharded(sc, 0, 200)
    assert_records_equal(rec, d["rec_xlibm"][:200])
    _same_agg(agg, engine.aggregate_stats(d["rec_xlibm"][:200]))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs for an NCCL communicator")
def test_multi_device_nccl_two_gpus():
    d, _, sc = load_golden("nmpc_n30_short")
    ctx = engine.Context(devices=[0, 1])
    assert ctx.uses_nccl
    rec, _, agg = ctx.run(sc, 0, 64, aggregate=True)
    assert_records_equal(rec, d["rec_xlibm"][:64])
    _same_agg(agg, engine.aggregate_stats(d["rec_xlibm"][:64]))
