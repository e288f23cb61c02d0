"""Python host mirror of the reference's Monte Carlo driver API over the C ABI.

Names and semantics follow /root/reference/proj/core/include/nmpcmc/montecarlo.hpp:
  validate_scenario(sc)            montecarlo.hpp:59   -> N_bar, raises on bad config
  run_closed_loop(sc, sim_index)   montecarlo.hpp:92   -> SimResult (+ trajectory)
  run_monte_carlo(sc, n_sims, ...) montecarlo.hpp:121  -> McResult
  aggregate_stats(sims)            montecarlo.hpp:108  -> McAggregate (dict)
  phi_histogram(phi, bins=0)       montecarlo.hpp:141  -> Histogram
Errors raise the reference's exception classes (errors.hpp:9-32). There is no
CPU fallback: without the CUDA library or a GPU these calls raise.
"""
import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi

_LIB_PATH = os.environ.get("NMPCMC_GPU_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libnmpcmc_gpu.so")
_lib = None


class NmpcmcError(RuntimeError):
    pass


class DimensionMismatch(NmpcmcError, ValueError):
    pass


class NotPositiveDefinite(NmpcmcError):
    pass


class NonFiniteState(NmpcmcError):
    pass


class DomainError(NmpcmcError, ValueError):
    pass


class LengthMismatch(NmpcmcError, ValueError):
    pass


class Unsupported(NmpcmcError):
    pass


class CudaError(NmpcmcError):
    pass


_EXC = {1: DimensionMismatch, 2: NotPositiveDefinite, 3: NonFiniteState, 4: DomainError,
        5: LengthMismatch, 6: Unsupported, 7: ValueError, 100: CudaError, 101: CudaError}


def _raise(code: int, msg: str = ""):
    if code != 0:
        cls = _EXC.get(code, NmpcmcError)
        raise cls(f"{abi.STATUS_NAMES.get(code, code)}: {msg}")


def library():
    """Load libnmpcmc_gpu.so (built by build.py / __graft_entry__.build()).

    Fails loudly when the extension is missing -- there is no fallback.
    """
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_2212_02197_b200.build`")
    lib = C.CDLL(_LIB_PATH)
    abi.check_layout(lib)
    S = C.POINTER(abi.Scenario)
    R = C.POINTER(abi.SimRecord)
    W = C.POINTER(abi.WorkCounters)
    A = C.POINTER(abi.Aggregate)
    P = C.c_void_p
    lib.nmpcmc_gpu_abi_version.restype = C.c_int
    lib.nmpcmc_gpu_validate.argtypes = [S, C.POINTER(C.c_int32)]
    lib.nmpcmc_gpu_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
    lib.nmpcmc_gpu_device_count.argtypes = [C.POINTER(C.c_int)]
    lib.nmpcmc_gpu_ctx_destroy.argtypes = [P]
    lib.nmpcmc_gpu_ctx_destroy.restype = None
    lib.nmpcmc_gpu_last_error.argtypes = [P]
    lib.nmpcmc_gpu_last_error.restype = C.c_char_p
    lib.nmpcmc_gpu_set_stream.argtypes = [P, P]
    lib.nmpcmc_gpu_set_option.argtypes = [P, C.c_int32, C.c_int64]
    lib.nmpcmc_gpu_run.argtypes = [P, S, C.c_uint64, C.c_int64, R, W, A]
    lib.nmpcmc_gpu_run_device.argtypes = [P, S, C.c_uint64, C.c_int64, P, P]
    lib.nmpcmc_gpu_run_async.argtypes = [P, S, C.c_uint64, C.c_int64, P, P]
    lib.nmpcmc_gpu_join.argtypes = [P]
    lib.nmpcmc_gpu_solve_ocp_batch.argtypes = [P, S, C.c_int64] + [C.c_void_p] * 9
    lib.nmpcmc_gpu_solve_qp_batch.argtypes = [P, C.c_void_p, C.c_int64] + [C.c_void_p] * 4
    lib.nmpcmc_gpu_wait.argtypes = [P]
    lib.nmpcmc_gpu_traj_rows.argtypes = [S]
    lib.nmpcmc_gpu_traj_rows.restype = C.c_int32
    lib.nmpcmc_gpu_run_traj.argtypes = [P, S, C.c_uint64, C.c_int64, R, C.POINTER(C.c_double)]
    lib.nmpcmc_gpu_aggregate.argtypes = [R, C.c_int64, A]
    lib.nmpcmc_gpu_histogram.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int32,
                                         C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    lib.nmpcmc_gpu_philox_blocks.argtypes = [P, C.POINTER(C.c_uint32), C.c_int64, C.POINTER(C.c_uint32)]
    lib.nmpcmc_gpu_normals.argtypes = [P, C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    lib.nmpcmc_gpu_libm.argtypes = [P, C.c_int32, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double)]
    lib.nmpcmc_gpu_fp64_peak.argtypes = [P, C.c_int, C.POINTER(C.c_double)]
    # K4 (device statistics) and the multi-GPU forms
    lib.nmpcmc_gpu_aggregate_device.argtypes = [P, P, C.c_int64, A, C.c_int32, C.POINTER(C.c_double),
                                                C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    lib.nmpcmc_gpu_last_records.argtypes = [P, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int)]
    lib.nmpcmc_gpu_histogram_last.argtypes = [P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                              C.POINTER(C.c_int32)]
    lib.nmpcmc_gpu_last_totals.argtypes = [P, W]
    lib.nmpcmc_gpu_ctx_create_multi.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(P)]
    lib.nmpcmc_gpu_ctx_num_devices.argtypes = [P]
    lib.nmpcmc_gpu_ctx_uses_nccl.argtypes = [P]
    lib.nmpcmc_gpu_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]
    lib.nmpcmc_gpu_shard_range.restype = None
    lib.nmpcmc_gpu_nccl_unique_id.argtypes = [C.c_void_p]
    lib.nmpcmc_gpu_comm_init.argtypes = [P, C.c_void_p, C.c_int, C.c_int]
    lib.nmpcmc_gpu_run_sharded.argtypes = [P, S, C.c_uint64, C.c_int64, R, A]
    lib.nmpcmc_gpu_allgather_records.argtypes = [P, P, C.c_int64, P]
    _lib = lib
    return lib


def device_count() -> int:
    """Visible CUDA devices (0 without a driver)."""
    n = C.c_int(0)
    library().nmpcmc_gpu_device_count(C.byref(n))
    return n.value


def validate_scenario(sc: abi.Scenario) -> int:
    """validate_scenario (montecarlo.cpp:34-63): returns N_bar or raises."""
    nbar = C.c_int32(0)
    _raise(library().nmpcmc_gpu_validate(C.byref(sc), C.byref(nbar)), "scenario")
    return nbar.value


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def shard_range(n: int, g: int, G: int):
    """(begin, count) of block g of G of [0, n) (nmpcmc_gpu_shard_range, host)."""
    b, c = C.c_int64(0), C.c_int64(0)
    library().nmpcmc_gpu_shard_range(n, g, G, C.byref(b), C.byref(c))
    return b.value, c.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for nmpcmc_gpu_comm_init (create on rank 0, ship to the others)."""
    buf = (C.c_uint8 * 128)()
    _raise(library().nmpcmc_gpu_nccl_unique_id(buf), "NCCL unique id")
    return bytes(buf)


class Context:
    """One device + one CUDA stream (C ABI nmpcmc_gpu_ctx); or, with
    devices=[...], one sub-context per GPU of this process
    (nmpcmc_gpu_ctx_create_multi: runs shard by global index, records are
    gathered over NCCL)."""

    def __init__(self, device: int = 0, devices=None):
        self.lib = library()
        h = C.c_void_p()
        if devices is None:
            _raise(self.lib.nmpcmc_gpu_ctx_create(device, C.byref(h)), f"device {device}")
            self.device = device
        else:
            ids = (C.c_int * len(devices))(*devices)
            rc = self.lib.nmpcmc_gpu_ctx_create_multi(ids, len(devices), C.byref(h))
            if rc != 0:
                _raise(rc, self.lib.nmpcmc_gpu_last_error(None).decode())
            self.device = devices[0]
        self.handle = h

    @property
    def num_devices(self) -> int:
        return self.lib.nmpcmc_gpu_ctx_num_devices(self.handle)

    @property
    def uses_nccl(self) -> bool:
        return self.lib.nmpcmc_gpu_ctx_uses_nccl(self.handle) == 1

    def close(self):
        if self.handle:
            self.lib.nmpcmc_gpu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            _raise(rc, self.lib.nmpcmc_gpu_last_error(self.handle).decode())

    KERNELS = {"warp": 1, "thread": 2, "generic": 3, "generic_warp": 4}

    def set_nmpc_kernel(self, kind: str):
        """'warp' (K3, default), 'generic' (K3g; 'thread' is its alias since
        the one-thread-per-sample K3b was retired) or
        'generic_warp' (K3w) for a one-state controller model; bitwise-
        identical results. A three-state controller model (or N > 255) runs
        K3w, or K3g when 'generic' is selected."""
        self._check(self.lib.nmpcmc_gpu_set_option(self.handle, 1, self.KERNELS[kind]))

    PI_KERNELS = {"auto": 0, "lanes": 1, "ws3": 3, "ws7": 7}

    def set_pi_kernel(self, kind: str):
        """NMPCMC_OPT_PI_KERNEL: 'auto' (default: the warp-specialised kernel,
        one consumer warp of 32 samples with producer warps generating the
        normals ahead), 'lanes' (one thread or 4 lanes per sample), 'ws3' /
        'ws7' (warp-specialised with 3 / 7 producer warps); bitwise-identical
        results."""
        self._check(self.lib.nmpcmc_gpu_set_option(self.handle, 5, self.PI_KERNELS[kind]))

    def set_ctrl_jacobians(self, kind: str):
        """'analytic' (default, make_cstr_model's closed forms) or 'fd': the
        controller model's jacobians by the reference's central differences
        (model.cpp:54-124), as for a Model without analytic jacobians; runs
        on K3w."""
        self._check(self.lib.nmpcmc_gpu_set_option(self.handle, 4, {"analytic": 0, "fd": 1}[kind]))

    def set_stream(self, stream_ptr: int):
        self._check(self.lib.nmpcmc_gpu_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def run(self, sc, first_sim: int, n_sims: int, counters: bool = False, aggregate: bool = False):
        """Records (numpy, index order) and optional work counters; host
        buffers. aggregate=True also returns the device-computed (K4)
        aggregate_stats dict as a third value."""
        rec = np.zeros(n_sims, dtype=abi.RECORD_DTYPE)
        cnt = np.zeros(n_sims, dtype=abi.COUNTERS_DTYPE) if counters else None
        agg = abi.Aggregate() if aggregate else None
        self._check(self.lib.nmpcmc_gpu_run(
            self.handle, C.byref(sc), first_sim, n_sims, _ptr(rec, abi.SimRecord),
            _ptr(cnt, abi.WorkCounters) if cnt is not None else None, C.byref(agg) if agg is not None else None))
        if aggregate:
            return rec, cnt, abi.aggregate_to_dict(agg)
        return rec, cnt

    # ---- K4 statistics on the device
    def aggregate_device(self, records_dev_ptr: int, n: int, bins: Optional[int] = None):
        """aggregate_stats (and phi_histogram when bins is not None) of n
        DEVICE-resident records at records_dev_ptr, on the device."""
        agg = abi.Aggregate()
        edges = np.zeros(201)
        counts = np.zeros(200, dtype=np.int32)
        nb = C.c_int32(0)
        want_h = bins is not None
        self._check(self.lib.nmpcmc_gpu_aggregate_device(
            self.handle, C.c_void_p(records_dev_ptr), n, C.byref(agg), bins or 0,
            _ptr(edges, C.c_double) if want_h else None, _ptr(counts, C.c_int32) if want_h else None,
            C.byref(nb) if want_h else None))
        h = Histogram(edges[: nb.value + 1].copy(), counts[: nb.value].copy()) if want_h else None
        return abi.aggregate_to_dict(agg), h

    def histogram_last(self, bins: int = 0) -> "Histogram":
        """phi_histogram of the last run's records, computed on the device."""
        edges = np.zeros(201)
        counts = np.zeros(200, dtype=np.int32)
        nb = C.c_int32(0)
        self._check(self.lib.nmpcmc_gpu_histogram_last(self.handle, bins, _ptr(edges, C.c_double),
                                                       _ptr(counts, C.c_int32), C.byref(nb)))
        return Histogram(edges[: nb.value + 1].copy(), counts[: nb.value].copy())

    def last_totals(self) -> dict:
        """Work counters of the last run summed over samples, devices, ranks."""
        w = abi.WorkCounters()
        self._check(self.lib.nmpcmc_gpu_last_totals(self.handle, C.byref(w)))
        return {k: int(getattr(w, k)) for k, _ in abi.WorkCounters._fields_}

    # ---- one process per GPU
    def comm_init(self, uid: bytes, rank: int, nranks: int):
        """Join the NCCL communicator of nranks processes (nmpcmc_gpu_comm_init)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.lib.nmpcmc_gpu_comm_init(self.handle, buf, rank, nranks))

    def allgather_records(self, local_dev_ptr: int, chunk: int, all_dev_ptr: int):
        """NCCL all-gather of `chunk` device records per rank (enqueued on the context stream)."""
        self._check(self.lib.nmpcmc_gpu_allgather_records(self.handle, C.c_void_p(local_dev_ptr), chunk,
                                                          C.c_void_p(all_dev_ptr)))

    def run_sharded(self, sc, first_sim: int, n_sims: int, records: bool = True, aggregate: bool = True):
        """This rank's block of [first, first + n), records all-gathered over
        NCCL (every rank gets all n, index order), K4 aggregate."""
        rec = np.zeros(n_sims, dtype=abi.RECORD_DTYPE) if records else None
        agg = abi.Aggregate() if aggregate else None
        self._check(self.lib.nmpcmc_gpu_run_sharded(
            self.handle, C.byref(sc), first_sim, n_sims, _ptr(rec, abi.SimRecord) if rec is not None else None,
            C.byref(agg) if agg is not None else None))
        return rec, (abi.aggregate_to_dict(agg) if agg is not None else None)

    def set_lanes(self, lanes: int):
        """NMPCMC_OPT_LANES: 2 pipelines consecutive batches over two internal
        streams (a batch's drain overlaps the next); 1 = context stream only."""
        self._check(self.lib.nmpcmc_gpu_set_option(self.handle, 3, lanes))

    def run_async(self, sc, first_sim: int, n_sims: int, rec_ptr: int, cnt_ptr: int = 0):
        """Enqueue a batch and the copy of its records (counters) into HOST
        memory at rec_ptr (cnt_ptr); valid after wait(). Pinned memory lets
        consecutive calls overlap."""
        self._check(self.lib.nmpcmc_gpu_run_async(
            self.handle, C.byref(sc), first_sim, n_sims, C.c_void_p(rec_ptr),
            C.c_void_p(cnt_ptr) if cnt_ptr else None))

    def join(self):
        """Order the context stream after all lane work (no host wait)."""
        self._check(self.lib.nmpcmc_gpu_join(self.handle))

    def wait(self):
        self._check(self.lib.nmpcmc_gpu_wait(self.handle))

    def run_device(self, sc, first_sim: int, n_sims: int, rec_ptr: int, cnt_ptr: int = 0):
        """Enqueue on the context stream (or a lane); outputs are device pointers."""
        self._check(self.lib.nmpcmc_gpu_run_device(
            self.handle, C.byref(sc), first_sim, n_sims, C.c_void_p(rec_ptr),
            C.c_void_p(cnt_ptr) if cnt_ptr else None))

    def run_traj(self, sc, first_sim: int, n_sims: int):
        rows = self.lib.nmpcmc_gpu_traj_rows(C.byref(sc))
        if rows < 0:
            validate_scenario(sc)
        rec = np.zeros(n_sims, dtype=abi.RECORD_DTYPE)
        traj = np.zeros((n_sims, rows, 5))
        self._check(self.lib.nmpcmc_gpu_run_traj(self.handle, C.byref(sc), first_sim, n_sims,
                                                 _ptr(rec, abi.SimRecord), _ptr(traj, C.c_double)))
        return rec, traj

    # unit-level entry points
    def philox_blocks(self, ctr_key: np.ndarray) -> np.ndarray:
        ck = np.ascontiguousarray(ctr_key, dtype=np.uint32).reshape(-1, 6)
        out = np.zeros((ck.shape[0], 4), dtype=np.uint32)
        self._check(self.lib.nmpcmc_gpu_philox_blocks(self.handle, _ptr(ck, C.c_uint32), ck.shape[0],
                                                      _ptr(out, C.c_uint32)))
        return out

    def normals(self, seed: int, stream: int, n: int) -> np.ndarray:
        out = np.zeros(n)
        self._check(self.lib.nmpcmc_gpu_normals(self.handle, seed, stream, n, _ptr(out, C.c_double)))
        return out

    def fp64_peak(self, use_fma: bool = True) -> float:
        """Measured FP64 TFLOP/s of this device (roofline denominator)."""
        out = C.c_double(0.0)
        self._check(self.lib.nmpcmc_gpu_fp64_peak(self.handle, 1 if use_fma else 0, C.byref(out)))
        return out.value

    def libm(self, fn: str, x: np.ndarray) -> np.ndarray:
        code = {"exp": 0, "log": 1, "sin": 2, "cos": 3}[fn]
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros_like(x)
        self._check(self.lib.nmpcmc_gpu_libm(self.handle, code, _ptr(x, C.c_double), x.size,
                                             _ptr(out, C.c_double)))
        return out


@dataclass
class SimResult:
    """SimResult (montecarlo.hpp:72-79)."""

    sim_index: int
    phi: float
    failed: bool
    ocp_solves: int
    ocp_failures: int
    status: int = 0
    trajectory: Optional[np.ndarray] = None  # rows x (t, z, z_bar, u, y)


@dataclass
class McResult:
    """McResult (montecarlo.hpp:112-116); records kept as a numpy array."""

    records: np.ndarray
    aggregate: dict
    wall_seconds: float
    counters: Optional[np.ndarray] = None
    first_sim: int = 0

    @property
    def sims(self) -> List[SimResult]:
        r = self.records
        return [SimResult(self.first_sim + i, float(r["phi"][i]), bool(r["failed"][i]),
                          int(r["ocp_solves"][i]), int(r["ocp_failures"][i]), int(r["status"][i]))
                for i in range(len(r))]


_ctx_cache = {}


def _context(device: int) -> Context:
    if device not in _ctx_cache:
        _ctx_cache[device] = Context(device)
    return _ctx_cache[device]


def run_closed_loop(sc, sim_index: int, device: int = 0) -> SimResult:
    """run_closed_loop (montecarlo.cpp:80-157); trajectory when sc.record_trajectories."""
    ctx = _context(device)
    if sc.record_trajectories:
        rec, traj = ctx.run_traj(sc, sim_index, 1)
        t = traj[0]
        t = t[~np.isnan(t[:, 0])]
    else:
        rec, _ = ctx.run(sc, sim_index, 1)
        t = None
    r = rec[0]
    return SimResult(sim_index, float(r["phi"]), bool(r["failed"]), int(r["ocp_solves"]),
                     int(r["ocp_failures"]), int(r["status"]), t)


def run_monte_carlo(sc, n_sims: int, device: int = 0, first_sim: int = 0,
                    counters: bool = False) -> McResult:
    """run_monte_carlo (montecarlo.cpp:213-251) on one GPU: samples
    [first_sim, first_sim + n_sims) in index order, then aggregate_stats."""
    if n_sims < 1:
        raise DomainError("run_monte_carlo: n_sims must be at least 1")
    validate_scenario(sc)
    ctx = _context(device)
    t0 = time.perf_counter()
    rec, cnt = ctx.run(sc, first_sim, n_sims, counters=counters)
    wall = time.perf_counter() - t0
    return McResult(rec, aggregate_stats(rec), wall, cnt, first_sim)


def aggregate_stats(records: np.ndarray) -> dict:
    """aggregate_stats (montecarlo.cpp:172-211), index order."""
    rec = np.ascontiguousarray(records, dtype=abi.RECORD_DTYPE)
    out = abi.Aggregate()
    _raise(library().nmpcmc_gpu_aggregate(_ptr(rec, abi.SimRecord), len(rec), C.byref(out)))
    return abi.aggregate_to_dict(out)


@dataclass
class Histogram:
    """Histogram (montecarlo.hpp:136-141)."""

    edges: np.ndarray = field(default_factory=lambda: np.zeros(0))
    counts: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int32))


def phi_histogram(phi, bins: int = 0) -> Histogram:
    """phi_histogram (montecarlo.cpp:268-304)."""
    v = np.ascontiguousarray(phi, dtype=np.float64)
    edges = np.zeros(201)
    counts = np.zeros(200, dtype=np.int32)
    nb = C.c_int32(0)
    _raise(library().nmpcmc_gpu_histogram(_ptr(v, C.c_double), v.size, bins, _ptr(edges, C.c_double),
                                          _ptr(counts, C.c_int32), C.byref(nb)))
    return Histogram(edges[: nb.value + 1].copy(), counts[: nb.value].copy())
