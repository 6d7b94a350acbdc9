"""ctypes binding of include/dspmv.h -- same names as the C ABI.

Argument marshalling only: numpy arrays / ints / torch tensors (anything with
``data_ptr()``) are turned into pointers and sizes; statuses become
``DspmvError``.  Device work, planning, scheduling and exchange all happen in
``libdspmv.so``.  The library MUST be present (built by ``make`` /
``__graft_entry__.build()``); there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DSPMV_LIB=<variant> selects lib/libdspmv_<variant>.so (e.g. "prof": the
# instrumented build of `make PROFILE=1`); default lib/libdspmv.so
_VAR = os.environ.get("DSPMV_LIB", "")
LIB_PATH = os.path.join(_HERE, "lib", f"libdspmv_{_VAR}.so" if _VAR else "libdspmv.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libdspmv.so not built ({LIB_PATH}); run `make` or __graft_entry__.build()")
lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------- enums
DSPMV_OK, DSPMV_ERR_ARG, DSPMV_ERR_RANGE, DSPMV_ERR_SCHEDULE, DSPMV_ERR_DEADLOCK, \
    DSPMV_ERR_STATE, DSPMV_ERR_CUDA, DSPMV_ERR_NCCL, DSPMV_ERR_OOM = range(9)
STATUS_NAMES = ["OK", "ERR_ARG", "ERR_RANGE", "ERR_SCHEDULE", "ERR_DEADLOCK", "ERR_STATE",
                "ERR_CUDA", "ERR_NCCL", "ERR_OOM"]
DSPMV_F64, DSPMV_F32 = 0, 1
DSPMV_COMM_NCCL, DSPMV_COMM_LOCAL, DSPMV_COMM_HOST = 0, 1, 2
DSPMV_EXCHANGE_COPY, DSPMV_EXCHANGE_PUT, DSPMV_EXCHANGE_NONE = 0, 1, 2
DSPMV_SKERNEL_AUTO, DSPMV_SKERNEL_BLOCK, DSPMV_SKERNEL_STREAM, DSPMV_SKERNEL_STREAM_TMA, DSPMV_SKERNEL_SELL = \
    0, 1, 2, 3, 4
DSPMV_PACK_GATHER, DSPMV_PACK_ALIAS_IF_CONTIGUOUS = 0, 1
DSPMV_ACC_TICKET, DSPMV_ACC_EXPLICIT_IN_END = 0, 1
DSPMV_UNPACK_COPY, DSPMV_UNPACK_FUSED = 0, 1
DSPMV_LONG_ROW_TREE, DSPMV_LONG_ROW_STORED = 0, 1
(DSPMV_OP_START, DSPMV_OP_PACK, DSPMV_OP_SPMV_LOCAL, DSPMV_OP_POST_SEND, DSPMV_OP_POST_RECV,
 DSPMV_OP_WAIT_SEND, DSPMV_OP_WAIT_RECV, DSPMV_OP_UNPACK, DSPMV_OP_SPMV_REMOTE, DSPMV_OP_END,
 DSPMV_OP_EVENT_RECORD, DSPMV_OP_EVENT_SYNC, DSPMV_OP_STREAM_WAIT_EVENT) = range(13)
(DSPMV_HALO_GID, DSPMV_RECV_COUNTS, DSPMV_RECV_DISPL, DSPMV_SEND_COUNTS, DSPMV_SEND_DISPL,
 DSPMV_PACK_MAP, DSPMV_AL_ROWPTR, DSPMV_AL_COL, DSPMV_AR_ROWS, DSPMV_AR_ROWPTR, DSPMV_AR_COL,
 DSPMV_AL_VAL, DSPMV_AR_VAL) = range(13)
DSPMV_MAX_STREAMS, DSPMV_MAX_EVENTS, DSPMV_MAX_OPS = 4, 64, 256
GPU_VERTICES = (DSPMV_OP_PACK, DSPMV_OP_SPMV_LOCAL, DSPMV_OP_UNPACK, DSPMV_OP_SPMV_REMOTE)
VERTEX_NAMES = ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv",
                "Unpack", "y_R", "end"]


class DspmvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 9 else status}: {msg}")


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p)


class dspmv_plan_opts(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("vector_threshold", ctypes.c_int32),
                ("keep_host", ctypes.c_int32), ("comm_priority", ctypes.c_int32),
                ("block_cfg", ctypes.c_int32), ("caller_stream0", ctypes.c_int32),
                ("reserve_sms", ctypes.c_int32), ("exchange", ctypes.c_int32),
                ("s_kernel", ctypes.c_int32), ("pack_mode", ctypes.c_int32),
                ("accumulate_mode", ctypes.c_int32), ("debug_checks", ctypes.c_int32),
                ("unpack_mode", ctypes.c_int32), ("long_row_sum", ctypes.c_int32),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", ctypes.c_void_p)]


class dspmv_plan_info(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64),
                ("row_end", ctypes.c_int64), ("nnz_local", ctypes.c_int64),
                ("nnz_remote", ctypes.c_int64), ("n_remote_rows", ctypes.c_int64),
                ("n_halo", ctypes.c_int64), ("n_send", ctypes.c_int64),
                ("n_recv_peers", ctypes.c_int32), ("n_send_peers", ctypes.c_int32),
                ("n_blocks_local", ctypes.c_int32), ("n_vrows_local", ctypes.c_int32),
                ("n_blocks_remote", ctypes.c_int32), ("n_vrows_remote", ctypes.c_int32),
                ("grid_local", ctypes.c_int32), ("grid_remote", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("ready", ctypes.c_int32),
                ("device_bytes", ctypes.c_int64),
                ("s_kernel_local", ctypes.c_int32), ("s_kernel_remote", ctypes.c_int32),
                ("pack_alias", ctypes.c_int32), ("accumulate_mode", ctypes.c_int32),
                ("unpack_fused", ctypes.c_int32)]


class dspmv_op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("stream", ctypes.c_int32),
                ("event", ctypes.c_int32), ("peer", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_S = ctypes.c_int  # status


def _sig(name, args, res=_S):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("dspmv_last_error", [], ctypes.c_char_p)
_sig("dspmv_version", [], _I)
_sig("dspmv_comm_unique_id", [_P])
_sig("dspmv_comm_create", [_P, _I, _I, _I, _P])
_sig("dspmv_comm_create_local", [_I, _I, _P])
_sig("dspmv_comm_destroy", [_P])
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_sig("dspmv_comm_create_host", [_I, _I, _I, ALLGATHER_FN, _P, _P])
_sig("dspmv_comm_info", [_P, _P, _P, _P])
_sig("dspmv_partition", [_I64, _I, _P])
_sig("dspmv_plan_opts_default", [_P], None)
_sig("dspmv_plan_create", [_P, _I64, _I64, _P, _P, _P, _P, _P])
_sig("dspmv_plan_destroy", [_P])
_sig("dspmv_plan_info_get", [_P, _P])
_sig("dspmv_plan_export", [_P, _I, _P, ctypes.c_size_t, _P])
_sig("dspmv_plan_build_host", [_I, _I64, _P, _P, _P, _I, _P])
_sig("dspmv_host_plan_info", [_P, _I, _P])
_sig("dspmv_host_plan_export", [_P, _I, _I, _P, ctypes.c_size_t, _P])
_sig("dspmv_host_plan_destroy", [_P])
_sig("dspmv_rank_plan_build_host", [_I, _I, _I64, _I64, _P, _P, _P, _I, _P])
_sig("dspmv_host_plan_requests", [_P, _I, _P, ctypes.c_size_t, _P])
_sig("dspmv_host_plan_set_requests", [_P, _P, _P])
_sig("dspmv_layout_host", [_P, ctypes.c_int32, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P])
_sig("dspmv_stream_layout_host", [_P, ctypes.c_int32, _I, _I, _P, _P, _P, _P, _P])
_sig("dspmv_sell_layout_host", [_P, ctypes.c_int32, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P])
_sig("dspmv_schedule_validate", [_P, _I, _I])
_sig("dspmv_schedule_derive", [_P, _P, _I, _P, _I, _P])
_sig("dspmv_schedule_derive_peers", [_P, _P, _P, _I, _I, _P, _I, _P])
_sig("dspmv_schedule_dag", [_P, _I, _P, _P, _I, _P, _P, _I, _P])
_sig("dspmv_schedule_moves", [_P, _I, _P, _I, _I, _P, _I, _P])
_sig("dspmv_schedule_parse", [ctypes.c_char_p, _P, _I, _P, _P])
_sig("dspmv_schedule_format", [_P, _I, _P, ctypes.c_size_t])
_sig("dspmv_schedule_create", [_P, _P, _I, _I, _P])
_sig("dspmv_schedule_destroy", [_P])
_sig("dspmv_schedule_set_timing", [_P, _I])
_sig("dspmv_schedule_set_caller_stream0", [_P, _I])
_sig("dspmv_schedule_op_times", [_P, _P, _I])
_sig("dspmv_schedule_op_timeline", [_P, _P, _P, _I])
_sig("dspmv_apply", [_P, _P, _P, _P])
_sig("dspmv_apply_host", [_P, _P, _P, _P])
_sig("dspmv_apply_graph", [_P, _P, _P, _P])
_sig("dspmv_apply_graph_prepare", [_P, _P, _P, _P])
_sig("dspmv_apply_group", [_P, _I, _P, _P, _P])
_sig("dspmv_apply_graph_group", [_P, _I, _P, _P, _P])
_sig("dspmv_l2_flush", [_I, _P])
_sig("dspmv_launch_count", [_P])
_sig("dspmv_profile_counters", [_P, _I, _I, _P])


def _check(st: int):
    if st != DSPMV_OK:
        raise DspmvError(st, lib.dspmv_last_error().decode(errors="replace"))


def _ptr(a) -> int | None:
    """Pointer of a numpy array, a torch tensor (data_ptr), an int, or None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(a)}")


def _stream(s) -> int | None:
    if s is None or isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


def _ops_array(ops) -> np.ndarray:
    a = np.zeros((len(ops), 4), np.int32)
    for i, o in enumerate(ops):
        o = tuple(o)
        a[i, :len(o)] = o
    return a


# ------------------------------------------------------------------- API
def dspmv_last_error() -> str:
    return lib.dspmv_last_error().decode(errors="replace")


def dspmv_version() -> int:
    return lib.dspmv_version()


def dspmv_partition(n_global: int, nranks: int) -> np.ndarray:
    out = np.zeros(nranks + 1, np.int64)
    _check(lib.dspmv_partition(n_global, nranks, out.ctypes.data))
    return out


def dspmv_comm_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib.dspmv_comm_unique_id(buf))
    return bytes(buf)


def dspmv_comm_create(uid: bytes, nranks: int, rank: int, device: int):
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    h = _P()
    _check(lib.dspmv_comm_create(buf, nranks, rank, device, ctypes.byref(h)))
    h._device = device
    return h


def dspmv_comm_create_local(nranks: int, device: int):
    hs = (_P * nranks)()
    _check(lib.dspmv_comm_create_local(nranks, device, hs))
    out = [_P(h) for h in hs]
    for h in out:
        h._device = device
    return out


def dspmv_comm_create_host(nranks: int, rank: int, device: int, allgather):
    """allgather(send: bytes) -> bytes (nranks*len(send), rank order); e.g.
    backed by torch.distributed (gloo).  The callback object is kept alive
    on the returned handle."""
    def _cb(send, recv, nbytes, ctx):
        try:
            out = allgather(ctypes.string_at(send, nbytes))
            assert len(out) == nranks * nbytes
            ctypes.memmove(recv, out, len(out))
            return 0
        except Exception:  # noqa: BLE001 -- reported to C as a failure status
            return 1
    cb = ALLGATHER_FN(_cb)
    h = _P()
    _check(lib.dspmv_comm_create_host(nranks, rank, device, cb, None, ctypes.byref(h)))
    h._cb = cb
    h._device = device
    return h


def dspmv_comm_destroy(comm):
    _check(lib.dspmv_comm_destroy(comm))


def dspmv_comm_info(comm):
    n, r, k = _I(), _I(), _I()
    _check(lib.dspmv_comm_info(comm, ctypes.byref(n), ctypes.byref(r), ctypes.byref(k)))
    return n.value, r.value, k.value


def _torch_alloc(nbytes, device, ctx):
    try:
        import torch
        return torch.cuda.caching_allocator_alloc(int(nbytes), int(device))
    except Exception:  # noqa: BLE001 -- the library reports ERR_OOM
        return None


def _torch_free(ptr, nbytes, device, ctx):
    import torch
    torch.cuda.caching_allocator_delete(ptr)


_TORCH_ALLOC = ALLOC_FN(_torch_alloc)
_TORCH_FREE = FREE_FN(_torch_free)


def dspmv_plan_create(comm, n_global: int, rowptr, col_global, val, dtype=DSPMV_F64,
                      vector_threshold: int = -1, keep_host: bool = False,
                      comm_priority: bool = True, block_cfg: int = -1,
                      caller_stream0: bool | None = None, reserve_sms: int | None = None,
                      exchange: int = DSPMV_EXCHANGE_COPY, s_kernel: int = DSPMV_SKERNEL_AUTO,
                      pack_mode: int = DSPMV_PACK_GATHER, accumulate_mode: int = DSPMV_ACC_TICKET,
                      debug_checks: bool | None = None, torch_alloc: bool = True,
                      unpack_mode: int = DSPMV_UNPACK_COPY, long_row_sum: int = DSPMV_LONG_ROW_TREE):
    """rowptr int64[n_local+1], col int32[nnz] (global ids), val float64/32.
    torch_alloc: the plan's device memory comes from torch's caching allocator
    (dspmv_plan_opts.alloc/free); False = cudaMalloc inside the library."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col_global, np.int32)
    val = np.ascontiguousarray(val, np.float32 if dtype == DSPMV_F32 else np.float64)
    o = dspmv_plan_opts()
    lib.dspmv_plan_opts_default(ctypes.byref(o))
    o.dtype = dtype
    o.vector_threshold = vector_threshold
    o.keep_host = int(keep_host)
    o.comm_priority = int(comm_priority)
    o.block_cfg = block_cfg
    if caller_stream0 is not None:
        o.caller_stream0 = int(caller_stream0)
    if reserve_sms is not None:
        o.reserve_sms = int(reserve_sms)
    o.exchange = int(exchange)
    o.s_kernel = int(s_kernel)
    o.pack_mode = int(pack_mode)
    o.accumulate_mode = int(accumulate_mode)
    o.unpack_mode = int(unpack_mode)
    o.long_row_sum = int(long_row_sum)
    if debug_checks is not None:
        o.debug_checks = int(debug_checks)
    if torch_alloc:
        o.alloc, o.free = _TORCH_ALLOC, _TORCH_FREE
    h = _P()
    _check(lib.dspmv_plan_create(comm, n_global, len(rowptr) - 1, rowptr.ctypes.data,
                                 col.ctypes.data, val.ctypes.data, ctypes.byref(o),
                                 ctypes.byref(h)))
    info = dspmv_plan_info_get(h)
    # what apply-time argument checks need (dtype, rows, device)
    h._meta = (dtype, int(info["row_end"] - info["row_begin"]), _comm_device(comm))
    return h


def _comm_device(comm):
    return getattr(comm, "_device", None)


def dspmv_plan_destroy(plan):
    _check(lib.dspmv_plan_destroy(plan))


def _info_dict(i: dspmv_plan_info) -> dict:
    return {f: getattr(i, f) for f, _ in dspmv_plan_info._fields_}


def dspmv_plan_info_get(plan) -> dict:
    i = dspmv_plan_info()
    _check(lib.dspmv_plan_info_get(plan, ctypes.byref(i)))
    return _info_dict(i)


_VAL_IDS = (DSPMV_AL_VAL, DSPMV_AR_VAL)


def _export(fn, args, what, dtype):
    need = ctypes.c_size_t()
    _check(fn(*args, what, None, 0, ctypes.byref(need)))
    dt = (np.float32 if dtype == DSPMV_F32 else np.float64) if what in _VAL_IDS else np.int32
    out = np.zeros(need.value // np.dtype(dt).itemsize, dt)
    _check(fn(*args, what, out.ctypes.data, need.value, None))
    return out


def dspmv_plan_export(plan, what: int) -> np.ndarray:
    return _export(lib.dspmv_plan_export, (plan,), what, dspmv_plan_info_get(plan)["dtype"])


def dspmv_plan_build_host(nranks: int, n_global: int, rowptr, col, val=None, dtype=DSPMV_F64):
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    vp = None
    if val is not None:
        val = np.ascontiguousarray(val, np.float32 if dtype == DSPMV_F32 else np.float64)
        vp = val.ctypes.data
    h = _P()
    _check(lib.dspmv_plan_build_host(nranks, n_global, rowptr.ctypes.data, col.ctypes.data, vp,
                                     dtype, ctypes.byref(h)))
    h._dtype = dtype
    return h


def dspmv_host_plan_info(hp, rank: int) -> dict:
    i = dspmv_plan_info()
    _check(lib.dspmv_host_plan_info(hp, rank, ctypes.byref(i)))
    return _info_dict(i)


def dspmv_host_plan_export(hp, rank: int, what: int) -> np.ndarray:
    return _export(lib.dspmv_host_plan_export, (hp, rank), what, getattr(hp, "_dtype", DSPMV_F64))


def dspmv_host_plan_destroy(hp):
    _check(lib.dspmv_host_plan_destroy(hp))


def dspmv_rank_plan_build_host(nranks: int, rank: int, n_global: int, rowptr, col, val=None,
                               dtype=DSPMV_F64):
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    vp = None
    if val is not None:
        val = np.ascontiguousarray(val, np.float32 if dtype == DSPMV_F32 else np.float64)
        vp = val.ctypes.data
    h = _P()
    _check(lib.dspmv_rank_plan_build_host(nranks, rank, n_global, len(rowptr) - 1, rowptr.ctypes.data,
                                          col.ctypes.data, vp, dtype, ctypes.byref(h)))
    h._dtype = dtype
    return h


def dspmv_host_plan_requests(hp, owner: int) -> np.ndarray:
    n = ctypes.c_size_t()
    _check(lib.dspmv_host_plan_requests(hp, owner, None, 0, ctypes.byref(n)))
    out = np.zeros(n.value, np.int32)
    _check(lib.dspmv_host_plan_requests(hp, owner, out.ctypes.data, n.value, None))
    return out


def dspmv_host_plan_set_requests(hp, lists):
    lists = [np.ascontiguousarray(l, np.int32) for l in lists]
    n = len(lists)
    ptrs = (_P * n)(*[l.ctypes.data if len(l) else None for l in lists])
    counts = np.array([len(l) for l in lists], np.int32)
    _check(lib.dspmv_host_plan_set_requests(hp, ptrs, counts.ctypes.data))


def dspmv_layout_host(rowptr, dtype=DSPMV_F64, cfg: int = -1, vthr: int = -1):
    """(s_rows, desc[nb,16], v_rows, cfg_used) of the planner's row layout."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    nr = len(rowptr) - 1
    ns, nb, nv, cu = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib.dspmv_layout_host(rowptr.ctypes.data, nr, dtype, cfg, vthr, None, ctypes.byref(ns), None,
                                 ctypes.byref(nb), None, ctypes.byref(nv), ctypes.byref(cu)))
    s_rows = np.zeros(max(ns.value, 1), np.int32)
    desc = np.zeros(max(nb.value, 1) * 16, np.int32)
    v_rows = np.zeros(max(nv.value, 1), np.int32)
    _check(lib.dspmv_layout_host(rowptr.ctypes.data, nr, dtype, cfg, vthr, s_rows.ctypes.data, ctypes.byref(ns),
                                 desc.ctypes.data, ctypes.byref(nb), v_rows.ctypes.data, ctypes.byref(nv),
                                 ctypes.byref(cu)))
    return s_rows[:ns.value], desc[:nb.value * 16].reshape(-1, 16), v_rows[:nv.value], cu.value


def dspmv_stream_layout_host(rowptr, vthr: int = -1, s_kernel: int = DSPMV_SKERNEL_AUTO):
    """(tiles[nt,2], v_rows, stream_used) of the planner's CSR-stream layout."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    nr = len(rowptr) - 1
    nt, nv, su = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib.dspmv_stream_layout_host(rowptr.ctypes.data, nr, vthr, s_kernel, None, ctypes.byref(nt), None,
                                        ctypes.byref(nv), ctypes.byref(su)))
    tiles = np.zeros(max(nt.value, 1) * 2, np.int32)
    v_rows = np.zeros(max(nv.value, 1), np.int32)
    _check(lib.dspmv_stream_layout_host(rowptr.ctypes.data, nr, vthr, s_kernel, tiles.ctypes.data, ctypes.byref(nt),
                                        v_rows.ctypes.data, ctypes.byref(nv), ctypes.byref(su)))
    return tiles[:2 * nt.value].reshape(-1, 2), v_rows[:nv.value], bool(su.value)


def dspmv_sell_layout_host(rowptr, vthr: int = -1, window: int = -1):
    """The planner's sliced (DSPMV_SKERNEL_SELL) form of the S rows:
    dict(base[ns+1], lane_row[ns,32], lane_len[ns,32], entry_src[nnz_S], chunks[nc+1])."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    nr = len(rowptr) - 1
    ns, ne, nc = ctypes.c_int32(0), ctypes.c_int64(0), ctypes.c_int32(0)
    _check(lib.dspmv_sell_layout_host(rowptr.ctypes.data, nr, vthr, window, None, None, None, None, None,
                                      ctypes.byref(ns), ctypes.byref(ne), ctypes.byref(nc)))
    base = np.zeros(ns.value + 1, np.int32)
    lane_row = np.zeros(max(1, 32 * ns.value), np.int32)
    lane_len = np.zeros(max(1, 32 * ns.value), np.int32)
    src = np.zeros(max(1, ne.value), np.int32)
    chunks = np.zeros(nc.value + 1, np.int32)
    _check(lib.dspmv_sell_layout_host(rowptr.ctypes.data, nr, vthr, window, base.ctypes.data, lane_row.ctypes.data,
                                      lane_len.ctypes.data, src.ctypes.data, chunks.ctypes.data,
                                      ctypes.byref(ns), ctypes.byref(ne), ctypes.byref(nc)))
    n = ns.value
    return dict(base=base, lane_row=lane_row[:32 * n].reshape(n, 32), lane_len=lane_len[:32 * n].reshape(n, 32),
                entry_src=src[:ne.value], chunks=chunks)


def dspmv_schedule_validate(ops, n_streams: int):
    a = _ops_array(ops)
    _check(lib.dspmv_schedule_validate(a.ctypes.data, len(a), n_streams))


def dspmv_schedule_derive(order, streams, n_streams: int) -> np.ndarray:
    order = np.ascontiguousarray(order, np.int32)
    streams = np.ascontiguousarray(streams, np.int32)
    out = np.zeros((DSPMV_MAX_OPS, 4), np.int32)
    n = _I()
    _check(lib.dspmv_schedule_derive(order.ctypes.data, streams.ctypes.data, n_streams,
                                     out.ctypes.data, DSPMV_MAX_OPS, ctypes.byref(n)))
    return out[:n.value].copy()


def dspmv_schedule_derive_peers(order, streams, peers, n_streams: int) -> np.ndarray:
    """Any granularity: order / streams / peers name the DAG vertices (kinds,
    streams of GPU vertices, peer offsets; per destination P:281-284)."""
    order = np.ascontiguousarray(order, np.int32)
    streams = np.ascontiguousarray(streams, np.int32)
    peers = np.ascontiguousarray(peers, np.int32)
    out = np.zeros((DSPMV_MAX_OPS, 4), np.int32)
    n = _I()
    _check(lib.dspmv_schedule_derive_peers(order.ctypes.data, streams.ctypes.data, peers.ctypes.data, len(order),
                                           n_streams, out.ctypes.data, DSPMV_MAX_OPS, ctypes.byref(n)))
    return out[:n.value].copy()


def dspmv_schedule_dag(offsets=()):
    """(vertices [(kind, peer)], edges [(u, v, is_deadlock_edge)]) of the coarse
    DAG (no offsets) or the per-destination DAG of send offsets `offsets`."""
    offs = np.ascontiguousarray(list(offsets), np.int32)
    nv, ne = _I(), _I()
    _check(lib.dspmv_schedule_dag(offs.ctypes.data if len(offs) else None, len(offs), None, None, 0,
                                  ctypes.byref(nv), None, 0, ctypes.byref(ne)))
    kinds = np.zeros(nv.value, np.int32)
    peers = np.zeros(nv.value, np.int32)
    edges = np.zeros((ne.value, 3), np.int32)
    _check(lib.dspmv_schedule_dag(offs.ctypes.data if len(offs) else None, len(offs), kinds.ctypes.data,
                                  peers.ctypes.data, nv.value, ctypes.byref(nv), edges.ctypes.data, ne.value,
                                  ctypes.byref(ne)))
    return list(zip(kinds.tolist(), peers.tolist())), [tuple(e) for e in edges.tolist()]


def dspmv_schedule_moves(prefix, n_streams: int, offsets=()) -> np.ndarray:
    """Legal next ops after a schedule prefix with orderable syncs (R-N5)."""
    offs = np.ascontiguousarray(list(offsets), np.int32)
    a = _ops_array(prefix) if len(prefix) else np.zeros((0, 4), np.int32)
    out = np.zeros((4 * DSPMV_MAX_OPS, 4), np.int32)
    n = _I()
    _check(lib.dspmv_schedule_moves(offs.ctypes.data if len(offs) else None, len(offs),
                                    a.ctypes.data if len(a) else None, len(a), n_streams, out.ctypes.data,
                                    len(out), ctypes.byref(n)))
    return out[:n.value].copy()


def vertex_label(kind: int, peer: int = 0) -> str:
    """"Pack", "Pack[+1]" (per destination)."""
    return VERTEX_NAMES[kind] + (f"[{peer:+d}]" if peer else "")


def dspmv_schedule_parse(text: str):
    out = np.zeros((DSPMV_MAX_OPS, 4), np.int32)
    n, ns = _I(), _I()
    _check(lib.dspmv_schedule_parse(text.encode(), out.ctypes.data, DSPMV_MAX_OPS,
                                    ctypes.byref(n), ctypes.byref(ns)))
    return out[:n.value].copy(), ns.value


def dspmv_schedule_format(ops) -> str:
    a = _ops_array(ops)
    buf = ctypes.create_string_buffer(64 * len(a) + 64)
    _check(lib.dspmv_schedule_format(a.ctypes.data, len(a), buf, len(buf)))
    return buf.value.decode()


def dspmv_schedule_create(plan, ops, n_streams: int):
    a = _ops_array(ops)
    h = _P()
    _check(lib.dspmv_schedule_create(plan, a.ctypes.data, len(a), n_streams, ctypes.byref(h)))
    h._n_ops = len(a)
    h._meta = getattr(plan, "_meta", None)
    return h


def _check_vec(sched, v, name, host: bool):
    """Tensors passed to an apply must match the plan: dtype, >= n_local
    elements, contiguous, on the plan's device (device applies) or in host
    memory (apply_host).  Raw pointers / numpy arrays pass unchecked except
    numpy dtype and length."""
    meta = getattr(sched, "_meta", None)
    if meta is None or v is None or isinstance(v, int):
        return
    dtype, n_local, device = meta
    want = "float32" if dtype == DSPMV_F32 else "float64"
    if isinstance(v, np.ndarray):
        if v.dtype != np.dtype(want) or v.size < n_local or not v.flags.c_contiguous:
            raise DspmvError(DSPMV_ERR_ARG, f"{name}: need a contiguous {want} array of >= {n_local} elements")
        return
    if not hasattr(v, "data_ptr"):
        return
    if str(v.dtype).split(".")[-1] != want or v.numel() < n_local or not v.is_contiguous():
        raise DspmvError(DSPMV_ERR_ARG, f"{name}: need a contiguous {want} tensor of >= {n_local} elements, "
                                        f"got {v.dtype} {tuple(v.shape)}")
    if host and v.is_cuda:
        raise DspmvError(DSPMV_ERR_ARG, f"{name}: apply_host takes host memory")
    if not host and n_local > 0 and (not v.is_cuda or (device is not None and v.device.index != device)):
        raise DspmvError(DSPMV_ERR_ARG, f"{name}: must be on cuda:{device}")


def dspmv_schedule_destroy(sched):
    _check(lib.dspmv_schedule_destroy(sched))


def dspmv_schedule_set_caller_stream0(sched, mode: int):
    """1: schedule stream 0 is the caller's stream; 0: a library stream; -1: the plan's option."""
    _check(lib.dspmv_schedule_set_caller_stream0(sched, int(mode)))


def dspmv_schedule_set_timing(sched, enable):
    """enable: False/True (every GPU op) or a bit mask of (1 << op kind)."""
    _check(lib.dspmv_schedule_set_timing(sched, int(enable)))


def dspmv_schedule_op_times(sched, n: int | None = None) -> np.ndarray:
    n = getattr(sched, "_n_ops", 0) if n is None else n
    out = np.zeros(n, np.float32)
    _check(lib.dspmv_schedule_op_times(sched, out.ctypes.data, n))
    return out


def dspmv_schedule_op_timeline(sched, n: int | None = None):
    """(begin_ms, end_ms) per op relative to START on the caller stream."""
    n = getattr(sched, "_n_ops", 0) if n is None else n
    b = np.zeros(n, np.float32)
    e = np.zeros(n, np.float32)
    _check(lib.dspmv_schedule_op_timeline(sched, b.ctypes.data, e.ctypes.data, n))
    return b, e


def dspmv_apply(sched, x, y, stream=None):
    """x, y: device buffers (torch tensors or raw pointers)."""
    _check_vec(sched, x, "x", False)
    _check_vec(sched, y, "y", False)
    _check(lib.dspmv_apply(sched, _ptr(x), _ptr(y), _stream(stream)))


def dspmv_apply_graph(sched, x, y, stream):
    """GPU-resident (CUDA-graph) execution; stream-ordered, non-blocking."""
    _check_vec(sched, x, "x", False)
    _check_vec(sched, y, "y", False)
    _check(lib.dspmv_apply_graph(sched, _ptr(x), _ptr(y), _stream(stream)))


def dspmv_apply_graph_prepare(sched, x, y, stream):
    """Capture the graph for x/y without launching it (SPMD: agree first)."""
    _check_vec(sched, x, "x", False)
    _check_vec(sched, y, "y", False)
    _check(lib.dspmv_apply_graph_prepare(sched, _ptr(x), _ptr(y), _stream(stream)))


def dspmv_apply_host(sched, x_host, y_host, stream=None):
    """x_host, y_host: host buffers (numpy or pinned torch CPU tensors)."""
    _check_vec(sched, x_host, "x_host", True)
    _check_vec(sched, y_host, "y_host", True)
    _check(lib.dspmv_apply_host(sched, _ptr(x_host), _ptr(y_host), _stream(stream)))


def dspmv_apply_group(scheds, xs, ys, stream=None):
    n = len(scheds)
    for s, x, y in zip(scheds, xs, ys):
        _check_vec(s, x, "x", False)
        _check_vec(s, y, "y", False)
    sa = (_P * n)(*[s.value for s in scheds])
    xa = (_P * n)(*[_ptr(x) for x in xs])
    ya = (_P * n)(*[_ptr(y) for y in ys])
    _check(lib.dspmv_apply_group(sa, n, xa, ya, _stream(stream)))


def dspmv_apply_graph_group(scheds, xs, ys, stream):
    """LOCAL group as ONE CUDA graph (every rank's branch concurrent); stream-ordered."""
    n = len(scheds)
    for s, x, y in zip(scheds, xs, ys):
        _check_vec(s, x, "x", False)
        _check_vec(s, y, "y", False)
    sa = (_P * n)(*[s.value for s in scheds])
    xa = (_P * n)(*[_ptr(x) for x in xs])
    ya = (_P * n)(*[_ptr(y) for y in ys])
    _check(lib.dspmv_apply_graph_group(sa, n, xa, ya, _stream(stream)))


def dspmv_l2_flush(device: int = 0, stream=None):
    _check(lib.dspmv_l2_flush(device, _stream(stream)))


def dspmv_launch_count() -> int:
    c = ctypes.c_uint64()
    _check(lib.dspmv_launch_count(ctypes.byref(c)))
    return c.value


def dspmv_profile_counters(reset: bool = True):
    out = (ctypes.c_ulonglong * 8)()
    n = _I()
    _check(lib.dspmv_profile_counters(out, 8, int(reset), ctypes.byref(n)))
    return list(out)[:n.value]
