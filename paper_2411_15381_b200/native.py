"""ctypes binding of libds_b200.so (the C ABI in include/ds_gpu.h).

There is no CPU fallback: if the library is missing or no sm_100 device is
visible, every entry point raises. Status codes map to the exception types the
reference throws (allocator.cpp:12-36, profiles.cpp:20-26,98-100,108-112):

    DS_ERR_INVALID_ARGUMENT -> InvalidArgument  (std::invalid_argument)
    DS_ERR_DOMAIN           -> DomainError      (std::domain_error)
    DS_ERR_INVARIANT        -> InvariantError   (diffserve::InvariantError)
    DS_ERR_OUT_OF_RANGE     -> OutOfRange       (std::out_of_range)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libds_b200.so")


class DsError(RuntimeError):
    status = -1


class InvalidArgument(DsError, ValueError):
    status = abi.ERR_INVALID_ARGUMENT


class DomainError(DsError, ValueError):
    status = abi.ERR_DOMAIN


class InvariantError(DsError):
    status = abi.ERR_INVARIANT


class OutOfRange(DsError, IndexError):
    status = abi.ERR_OUT_OF_RANGE


class CudaError(DsError):
    status = abi.ERR_CUDA


class NoDevice(DsError):
    status = abi.ERR_NO_DEVICE


class CapacityError(DsError):
    status = abi.ERR_CAPACITY


class CommError(DsError):
    status = abi.ERR_COMM


_EXC = {c.status: c for c in (InvalidArgument, DomainError, InvariantError, OutOfRange,
                              CudaError, NoDevice, CapacityError, CommError)}

_lib = None
c_p = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
u64 = ctypes.c_uint64
f64 = ctypes.c_double

# (name, restype, argtypes) for every symbol include/ds_gpu.h declares.
SIGNATURES = [
    ("ds_version", ctypes.c_char_p, []),
    ("ds_last_error", ctypes.c_char_p, []),
    ("ds_ctx_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(c_p)]),
    ("ds_ctx_destroy", ctypes.c_int, [c_p]),
    ("ds_ctx_synchronize", ctypes.c_int, [c_p]),
    ("ds_ctx_launch_count", i64, [c_p]),
    ("ds_ctx_stream", c_p, [c_p]),
    ("ds_ctx_take_error", ctypes.c_int, [c_p, c_p, ctypes.POINTER(i64)]),
    ("ds_plan_batch", ctypes.c_int, [c_p, c_p, i32, c_p, i32, c_p, c_p, i32, c_p]),
    ("ds_plan_batch_device", ctypes.c_int, [c_p, c_p, i32, c_p, i32, c_p, c_p, i32, c_p, c_p]),
    ("ds_plan_validate", ctypes.c_int, [c_p, i32, c_p, i32, c_p, c_p, i32]),
    ("ds_plan_keys", ctypes.c_int, [c_p, c_p, i32, c_p, i32, c_p, c_p, i32, i32, i32, c_p]),
    ("ds_plan_keys_device", ctypes.c_int,
     [c_p, c_p, i32, c_p, i32, c_p, c_p, i32, i32, i32, c_p, c_p]),
    ("ds_plan_from_keys", ctypes.c_int, [c_p, c_p, i32, c_p, i32, c_p, c_p, i32, c_p, c_p]),
    ("ds_plan_from_keys_device", ctypes.c_int,
     [c_p, c_p, i32, c_p, i32, c_p, c_p, i32, c_p, c_p, c_p]),
    ("ds_score_latent", ctypes.c_int, [c_p, c_p, u64, i64, c_p, c_p]),
    ("ds_score_latent_device", ctypes.c_int, [c_p, c_p, u64, i64, c_p, c_p, c_p]),
    ("ds_route", ctypes.c_int, [c_p, c_p, i32, i64, c_p, i32, i64, c_p, c_p]),
    ("ds_route_device", ctypes.c_int, [c_p, c_p, i32, i64, c_p, i32, i64, c_p, c_p, c_p]),
    ("ds_route_scratch_bytes", ctypes.c_size_t, [i64, i32]),
    ("ds_curve_observe", ctypes.c_int, [c_p, c_p, c_p, i32, i64, f64]),
    ("ds_curve_observe_device", ctypes.c_int, [c_p, c_p, c_p, i32, i64, f64, c_p]),
    ("ds_disc_create", ctypes.c_int, [c_p, u64, ctypes.POINTER(c_p)]),
    ("ds_disc_destroy", ctypes.c_int, [c_p]),
    ("ds_disc_export", ctypes.c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    ("ds_disc_score", ctypes.c_int, [c_p, c_p, i64, i32, i32, c_p]),
    ("ds_disc_score_device", ctypes.c_int, [c_p, c_p, i64, i32, i32, c_p, c_p]),
    ("ds_disc_batch_complete_device", ctypes.c_int,
     [c_p, c_p, i64, i32, i32, c_p, c_p, f64, c_p, i32, i64, c_p, c_p, c_p]),
    ("ds_disc_batches_complete_device", ctypes.c_int,
     [c_p, c_p, i64, c_p, i32, i32, i32, c_p, c_p, f64, c_p, i64, c_p, c_p, c_p]),
    ("ds_synth_images_device", ctypes.c_int, [c_p, u64, u64, i64, i32, i32, c_p, c_p]),
    ("ds_generate_arrivals", ctypes.c_int, [c_p, c_p, i32, f64, u64, i32, c_p, i64,
                                            ctypes.POINTER(i64)]),
    ("ds_generate_arrivals_device", ctypes.c_int, [c_p, c_p, i32, f64, u64, i32, c_p, i64,
                                                   ctypes.POINTER(i64), c_p]),
    ("ds_sample_queries", ctypes.c_int, [c_p, c_p, u64, c_p, i64, f64, c_p]),
    ("ds_sample_queries_device", ctypes.c_int, [c_p, c_p, u64, c_p, i64, f64, c_p, c_p]),
    ("ds_format_queries_csv", ctypes.c_int, [c_p, c_p, i64, c_p, i64, ctypes.POINTER(i64)]),
    ("ds_format_intervals_csv", ctypes.c_int, [c_p, c_p, i64, c_p, i64, ctypes.POINTER(i64)]),
    ("ds_format_plans_csv", ctypes.c_int, [c_p, c_p, i64, c_p, i64, ctypes.POINTER(i64)]),
    ("ds_format_queries_csv_device", ctypes.c_int, [c_p, c_p, i64, c_p, i64,
                                                    ctypes.POINTER(i64), c_p]),
    ("ds_format_g6", ctypes.c_int, [c_p, c_p, i64, c_p]),
    # multi-GPU (ds_comm)
    ("ds_comm_nccl_unique_id", ctypes.c_int, [c_p]),
    ("ds_comm_init_nccl", ctypes.c_int, [c_p, i32, i32, c_p, ctypes.POINTER(c_p)]),
    ("ds_comm_wrap_nccl", ctypes.c_int, [c_p, c_p, ctypes.POINTER(c_p)]),
    ("ds_comm_init_all", ctypes.c_int, [c_p, i32, c_p]),
    ("ds_comm_create_host", ctypes.c_int, [c_p, i32, i32, c_p, c_p, ctypes.POINTER(c_p)]),
    ("ds_comm_destroy", ctypes.c_int, [c_p]),
    ("ds_comm_rank", i32, [c_p]),
    ("ds_comm_size", i32, [c_p]),
    ("ds_shard_range", None, [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    ("ds_route_sharded_device", ctypes.c_int,
     [c_p, c_p, c_p, i32, i64, c_p, i32, i64, c_p, c_p, c_p, c_p, c_p]),
    ("ds_queue_gather_device", ctypes.c_int,
     [c_p, c_p, i32, c_p, i64, c_p, i32, c_p, i64, c_p, c_p]),
    ("ds_curve_observe_sharded_device", ctypes.c_int, [c_p, c_p, c_p, c_p, i32, c_p, f64, c_p]),
    ("ds_plan_sharded_device", ctypes.c_int,
     [c_p, c_p, c_p, i32, c_p, i32, c_p, c_p, i32, i32, i32, c_p, c_p]),
    ("ds_comm_gather_device", ctypes.c_int,
     [c_p, c_p, i32, c_p, ctypes.c_size_t, c_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
      c_p]),
]

# ds_comm_ops (include/ds_gpu.h): host-transport callbacks
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_p, c_p, ctypes.c_size_t, c_p)
ALLREDUCE_MIN_U64_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.c_size_t, c_p)
GATHERV_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_p, c_p, ctypes.POINTER(ctypes.c_size_t),
                              ctypes.c_int32, c_p)


class CommOps(ctypes.Structure):
    _fields_ = [("allgather", ALLGATHER_FN), ("allreduce_min_u64", ALLREDUCE_MIN_U64_FN),
                ("gatherv", GATHERV_FN)]


def lib():
    """Load libds_b200.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run __graft_entry__.build() (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != abi.OK:
        msg = lib().ds_last_error().decode(errors="replace")
        raise _EXC.get(status, DsError)(msg)


class Context:
    """One ds_ctx (device + stream). Not thread-safe, like the reference's
    Simulation."""

    def __init__(self, device: int = 0):
        h = c_p()
        check(lib().ds_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            lib().ds_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().ds_ctx_stream(self.handle) or 0

    def launches(self) -> int:
        return int(lib().ds_ctx_launch_count(self.handle))

    def synchronize(self):
        check(lib().ds_ctx_synchronize(self.handle))

    def take_error(self, stream: int = 0) -> int:
        """Raises DomainError if a _device call met a confidence outside
        [0, 1] since the last call (ds_ctx_take_error); returns -1 otherwise."""
        v = i64(-1)
        check(lib().ds_ctx_take_error(self.handle, c_p(stream), ctypes.byref(v)))
        return int(v.value)

    # ---- planner ------------------------------------------------------
    def plan_batch(self, problems: np.ndarray, cascades: np.ndarray, grid_values: np.ndarray,
                   grid_offsets: np.ndarray) -> np.ndarray:
        problems = np.ascontiguousarray(problems, abi.PROBLEM)
        cascades = np.ascontiguousarray(cascades, abi.CASCADE)
        grid_values = np.ascontiguousarray(grid_values, np.float64)
        grid_offsets = np.ascontiguousarray(grid_offsets, np.int32)
        out = np.zeros(len(problems), abi.PLAN)
        check(lib().ds_plan_batch(self.handle, abi.ptr(problems), len(problems),
                                  abi.ptr(cascades), len(cascades), abi.ptr(grid_values),
                                  abi.ptr(grid_offsets), len(grid_offsets) - 1, abi.ptr(out)))
        return out

    def plan_keys(self, problems: np.ndarray, cascades: np.ndarray, grid_values: np.ndarray,
                  grid_offsets: np.ndarray, t_lo: int, t_hi: int) -> np.ndarray:
        """Packed selection keys of the search restricted to grid indices
        [t_lo, t_hi) (uint64; 2**64-1 = none), see ds_plan_keys."""
        problems = np.ascontiguousarray(problems, abi.PROBLEM)
        cascades = np.ascontiguousarray(cascades, abi.CASCADE)
        grid_values = np.ascontiguousarray(grid_values, np.float64)
        grid_offsets = np.ascontiguousarray(grid_offsets, np.int32)
        keys = np.zeros(len(problems), np.uint64)
        check(lib().ds_plan_keys(self.handle, abi.ptr(problems), len(problems), abi.ptr(cascades),
                                 len(cascades), abi.ptr(grid_values), abi.ptr(grid_offsets),
                                 len(grid_offsets) - 1, t_lo, t_hi, abi.ptr(keys)))
        return keys

    def plan_from_keys(self, problems: np.ndarray, cascades: np.ndarray,
                       grid_values: np.ndarray, grid_offsets: np.ndarray,
                       keys: np.ndarray) -> np.ndarray:
        problems = np.ascontiguousarray(problems, abi.PROBLEM)
        cascades = np.ascontiguousarray(cascades, abi.CASCADE)
        grid_values = np.ascontiguousarray(grid_values, np.float64)
        grid_offsets = np.ascontiguousarray(grid_offsets, np.int32)
        keys = np.ascontiguousarray(keys, np.uint64)
        out = np.zeros(len(problems), abi.PLAN)
        check(lib().ds_plan_from_keys(self.handle, abi.ptr(problems), len(problems),
                                      abi.ptr(cascades), len(cascades), abi.ptr(grid_values),
                                      abi.ptr(grid_offsets), len(grid_offsets) - 1,
                                      abi.ptr(keys), abi.ptr(out)))
        return out

    # ---- latent scorer --------------------------------------------------
    def score_latent(self, model: np.ndarray, id0: int, n: int, with_quality: bool = False):
        model = np.ascontiguousarray(model, abi.QUERY_MODEL)
        conf = np.zeros(n, np.float64)
        ql = np.zeros(n, np.float64) if with_quality else None
        check(lib().ds_score_latent(self.handle, abi.ptr(model), id0, n, abi.ptr(conf),
                                    abi.ptr(ql)))
        return (conf, ql) if with_quality else conf

    # ---- workload synthesis ----------------------------------------------
    def generate_arrivals(self, rates, interval_seconds: float, seed: int,
                          mode: int = abi.ARRIVALS_POISSON) -> np.ndarray:
        rates = np.ascontiguousarray(np.atleast_1d(np.asarray(rates, np.float64)))
        n = i64(0)
        check(lib().ds_generate_arrivals(self.handle, abi.ptr(rates), len(rates),
                                         float(interval_seconds), int(seed), int(mode), None, 0,
                                         ctypes.byref(n)))
        out = np.zeros(max(n.value, 1), np.float64)
        check(lib().ds_generate_arrivals(self.handle, abi.ptr(rates), len(rates),
                                         float(interval_seconds), int(seed), int(mode),
                                         abi.ptr(out), len(out), ctypes.byref(n)))
        return out[:n.value]

    def sample_query_records(self, model: np.ndarray, arrivals, slo_seconds: float,
                             id0: int = 0) -> np.ndarray:
        model = np.ascontiguousarray(model, abi.QUERY_MODEL)
        arrivals = np.ascontiguousarray(arrivals, np.float64)
        out = np.zeros(len(arrivals), abi.QUERY)
        check(lib().ds_sample_queries(self.handle, abi.ptr(model), id0, abi.ptr(arrivals),
                                      len(arrivals), float(slo_seconds), abi.ptr(out)))
        return out

    # ---- CSV output ------------------------------------------------------
    def _format_csv(self, fn: str, rows: np.ndarray, dtype) -> bytes:
        rows = np.ascontiguousarray(rows, dtype)
        n = i64(0)
        f = getattr(lib(), fn)
        out = np.empty(len(rows) * 256 + 4096, np.uint8)   # every row fits in 256 bytes
        check(f(self.handle, abi.ptr(rows), len(rows), abi.ptr(out), len(out), ctypes.byref(n)))
        return out[:n.value].tobytes()

    def format_queries_csv(self, records: np.ndarray) -> bytes:
        return self._format_csv("ds_format_queries_csv", records, abi.QUERY_RECORD)

    def format_intervals_csv(self, rows: np.ndarray) -> bytes:
        return self._format_csv("ds_format_intervals_csv", rows, abi.INTERVAL_SNAPSHOT)

    def format_plans_csv(self, rows: np.ndarray) -> bytes:
        return self._format_csv("ds_format_plans_csv", rows, abi.PLAN_LOG_ENTRY)

    def format_g6(self, values) -> np.ndarray:
        """fmt6 of each value as 16-byte NUL-padded slots (np.dtype('S16'))."""
        values = np.ascontiguousarray(values, np.float64)
        out = np.zeros(len(values), "S16")
        check(lib().ds_format_g6(self.handle, abi.ptr(values), len(values), abi.ptr(out)))
        return out

    # ---- router ---------------------------------------------------------
    def route(self, conf: np.ndarray, thresholds, index_base: int = 0, with_lists: bool = True):
        conf = np.ascontiguousarray(conf)
        if conf.dtype == np.float64:
            dt = abi.CONF_F64
        elif conf.dtype == np.float32:
            dt = abi.CONF_F32
        else:
            raise TypeError("confidences must be float64 or float32")
        thr = np.ascontiguousarray(np.atleast_1d(np.asarray(thresholds, np.float64)))
        n, nt = len(conf), len(thr)
        counts = np.zeros(nt, np.int64)
        idx = np.zeros(nt * max(n, 1), np.int64) if with_lists else None
        check(lib().ds_route(self.handle, abi.ptr(conf), dt, n, abi.ptr(thr), nt, index_base,
                             abi.ptr(idx), abi.ptr(counts)))
        if not with_lists:
            return counts, None
        lists = [idx[k * n: k * n + counts[k]].copy() for k in range(nt)]
        return counts, lists

    # ---- deferral curve -------------------------------------------------
    def curve_observe(self, curve: np.ndarray, conf: np.ndarray, decay: float) -> np.ndarray:
        curve = np.array(curve, abi.CURVE)  # copy: the call updates in place
        conf = np.ascontiguousarray(conf)
        dt = abi.CONF_F64 if conf.dtype == np.float64 else abi.CONF_F32
        if conf.dtype not in (np.float64, np.float32):
            raise TypeError("confidences must be float64 or float32")
        check(lib().ds_curve_observe(self.handle, abi.ptr(curve), abi.ptr(conf), dt, len(conf),
                                     decay))
        return curve


class Discriminator:
    """PatchDisc scorer (ds_disc_*), weights generated on the device from a seed."""

    def __init__(self, ctx: Context, weight_seed: int = 2024):
        self.ctx = ctx
        h = c_p()
        check(lib().ds_disc_create(ctx.handle, weight_seed, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().ds_disc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> dict:
        from . import abi as _abi  # noqa: F401
        q1 = np.zeros((768, 256), np.int8)
        s1 = np.zeros(1, np.float32)
        w2 = np.zeros((256, 1024), np.uint16)
        w3 = np.zeros((1024, 256), np.uint16)
        b1 = np.zeros(256, np.float32)
        b2 = np.zeros(1024, np.float32)
        b3 = np.zeros(256, np.float32)
        hw = np.zeros(256, np.float32)
        hb = np.zeros(1, np.float32)
        check(lib().ds_disc_export(self.handle, abi.ptr(q1), abi.ptr(s1), abi.ptr(w2), abi.ptr(w3),
                                   abi.ptr(b1), abi.ptr(b2), abi.ptr(b3), abi.ptr(hw),
                                   abi.ptr(hb)))
        return dict(q1=q1, s1=float(s1[0]), w2=w2, w3=w3, b1=b1, b2=b2, b3=b3, head_w=hw,
                    head_b=float(hb[0]))

    def score(self, images: np.ndarray) -> np.ndarray:
        images = np.ascontiguousarray(images, np.uint8)
        n, h, w, c = images.shape
        if c != 3:
            raise ValueError("images must be NHWC with 3 channels")
        conf = np.zeros(n, np.float32)
        check(lib().ds_disc_score(self.handle, abi.ptr(images), n, h, w, abi.ptr(conf)))
        return conf

    def score_device(self, images_ptr: int, n: int, h: int, w: int, conf_ptr: int,
                     stream: int = 0):
        check(lib().ds_disc_score_device(self.handle, c_p(images_ptr), n, h, w, c_p(conf_ptr),
                                         c_p(stream)))

    def batches_complete_device(self, images_ptr: int, n_images: int, offsets_ptr: int,
                                n_batches: int, h: int, w: int, conf_ptr: int, curve_ptr: int,
                                decay: float, thr_ptr: int, index_base: int, heavy_ptr: int,
                                counts_ptr: int, stream: int = 0):
        """A backlog of light batches in order (ds_disc_batches_complete_device)."""
        check(lib().ds_disc_batches_complete_device(
            self.handle, c_p(images_ptr), n_images, c_p(offsets_ptr), n_batches, h, w,
            c_p(conf_ptr), c_p(curve_ptr), decay, c_p(thr_ptr), index_base, c_p(heavy_ptr),
            c_p(counts_ptr), c_p(stream)))

    def batch_complete_device(self, images_ptr: int, n: int, h: int, w: int, conf_ptr: int,
                              curve_ptr: int, decay: float, thr_ptr: int, nt: int,
                              index_base: int, heavy_ptr: int, counts_ptr: int, stream: int = 0):
        """One light batch (cluster.cpp:288-307): score, observe in order, defer."""
        check(lib().ds_disc_batch_complete_device(
            self.handle, c_p(images_ptr), n, h, w, c_p(conf_ptr), c_p(curve_ptr), decay,
            c_p(thr_ptr), nt, index_base, c_p(heavy_ptr), c_p(counts_ptr), c_p(stream)))


class Comm:
    """A ds_comm: the collectives of the sharded hot path (include/ds_gpu.h
    "multi-GPU"). Made by Comm.nccl (one rank per GPU over NCCL; rank 0's
    unique_id() distributed out of band) or Comm.host (caller callbacks: the
    tests' several ranks on one GPU over gloo, dist.TorchHostOps)."""

    def __init__(self, ctx: Context, handle, keepalive=None):
        self.ctx = ctx
        self.handle = handle
        self._keep = keepalive
        L = lib()
        self.rank = int(L.ds_comm_rank(handle))
        self.size = int(L.ds_comm_size(handle))

    @staticmethod
    def _nccl_first():
        # The library dlopens "libnccl.so.2" and takes the process's copy if
        # one is loaded. torch links its own (newer) NCCL under that soname:
        # import it first, else the system NCCL would be loaded and torch's
        # import would then bind to it (missing symbols).
        try:
            import torch  # noqa: F401
        except ImportError:
            pass

    @staticmethod
    def unique_id() -> bytes:
        Comm._nccl_first()
        buf = (ctypes.c_uint8 * 128)()
        check(lib().ds_comm_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, ctx: Context, nranks: int, rank: int, uid: bytes) -> "Comm":
        if len(uid) != 128:
            raise InvalidArgument("an NCCL unique id is 128 bytes")
        cls._nccl_first()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = c_p()
        check(lib().ds_comm_init_nccl(ctx.handle, nranks, rank, buf, ctypes.byref(h)))
        return cls(ctx, h)

    @classmethod
    def host(cls, ctx: Context, nranks: int, rank: int, impl) -> "Comm":
        """impl.allgather(u8 array) -> u8 array of nranks*len; impl.allreduce_min_u64(u64
        array) in place; impl.gatherv(u8 array, sizes, root) -> u8 array at root."""
        import traceback

        def view(ptr, n, ty=ctypes.c_uint8):
            return np.ctypeslib.as_array((ty * n).from_address(ptr)) if n else \
                np.zeros(0, np.uint8)

        def ag(send, recv, nbytes, user):
            try:
                out = np.ascontiguousarray(impl.allgather(view(send, nbytes).copy()), np.uint8)
                if out.nbytes != nbytes * nranks:
                    return 1
                ctypes.memmove(recv, out.ctypes.data, out.nbytes)
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        def ar(buf, count, user):
            try:
                a = np.ctypeslib.as_array(buf, shape=(count,))
                a[:] = impl.allreduce_min_u64(a.copy())
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        def gv(send, recv, sizes, root, user):
            try:
                sz = [int(sizes[r]) for r in range(nranks)]
                out = impl.gatherv(view(send, sz[rank]).copy(), sz, int(root))
                if rank == root:
                    out = np.ascontiguousarray(out, np.uint8)
                    if out.nbytes != sum(sz):
                        return 1
                    if out.nbytes:
                        ctypes.memmove(recv, out.ctypes.data, out.nbytes)
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        ops = CommOps(ALLGATHER_FN(ag), ALLREDUCE_MIN_U64_FN(ar), GATHERV_FN(gv))
        h = c_p()
        check(lib().ds_comm_create_host(ctx.handle, nranks, rank, ctypes.byref(ops), None,
                                        ctypes.byref(h)))
        return cls(ctx, h, keepalive=ops)

    def close(self):
        if self.handle:
            lib().ds_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def shard_range(n: int, nranks: int, rank: int):
        lo, hi = i64(0), i64(0)
        lib().ds_shard_range(n, nranks, rank, ctypes.byref(lo), ctypes.byref(hi))
        return int(lo.value), int(hi.value)

    # ---- collective calls on device pointers (ints), stream-ordered -----------
    def route(self, conf_ptr, dtype, n_local, thr_ptr, nt, index_base, heavy_ptr, counts_ptr,
              offsets_ptr=0, totals_ptr=0, stream=0):
        check(lib().ds_route_sharded_device(
            self.ctx.handle, self.handle, c_p(conf_ptr), dtype, n_local, c_p(thr_ptr), nt,
            index_base, c_p(heavy_ptr), c_p(counts_ptr), c_p(offsets_ptr or None),
            c_p(totals_ptr or None), c_p(stream or None)))

    def gather_queues(self, root, heavy_ptr, n_local, counts_ptr, nt, global_ptr=0,
                      global_stride=0, global_counts_ptr=0, stream=0):
        check(lib().ds_queue_gather_device(
            self.ctx.handle, self.handle, root, c_p(heavy_ptr or None), n_local, c_p(counts_ptr),
            nt, c_p(global_ptr or None), global_stride, c_p(global_counts_ptr or None),
            c_p(stream or None)))

    def curve_observe(self, curve_ptr, conf_ptr, dtype, shard_sizes, decay, stream=0):
        sizes = np.ascontiguousarray(shard_sizes, np.int64)
        if len(sizes) != self.size:
            raise InvalidArgument("one shard size per rank")
        check(lib().ds_curve_observe_sharded_device(
            self.ctx.handle, self.handle, c_p(curve_ptr), c_p(conf_ptr or None), dtype,
            abi.ptr(sizes), decay, c_p(stream or None)))

    def plan(self, problems_ptr, n, cascades_ptr, n_cascades, grid_ptr, offs_ptr, n_grids, t_lo,
             t_hi, out_ptr, stream=0):
        check(lib().ds_plan_sharded_device(
            self.ctx.handle, self.handle, c_p(problems_ptr), n, c_p(cascades_ptr), n_cascades,
            c_p(grid_ptr), c_p(offs_ptr), n_grids, t_lo, t_hi, c_p(out_ptr), c_p(stream or None)))

    def gather(self, root, send_ptr, nbytes, recv_ptr=0, capacity=0, stream=0) -> int:
        total = ctypes.c_size_t(0)
        check(lib().ds_comm_gather_device(
            self.ctx.handle, self.handle, root, c_p(send_ptr or None), nbytes,
            c_p(recv_ptr or None), capacity, ctypes.byref(total), c_p(stream or None)))
        return int(total.value)
