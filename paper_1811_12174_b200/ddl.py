"""Thin Python binding of libddl (include/ddl.h).

Argument marshalling only: every step of the all-reduce runs in libddl's sm_100a kernels.
PyTorch supplies device memory, streams and the process group used once to exchange the
cudaIpc handles (never on the data path).  There is no CPU fallback: if libddl.so is
missing, importing this module raises.

Low-level functions carry the C names (``ddl_init``, ``ddl_allreduce``, ...) and take raw
pointers; the classes below wrap them for torch tensors:

* ``Comm``      -- one process per GPU (``init(dims)`` under torchrun).
* ``Loopback``  -- P virtual ranks on one GPU, one launch (tests, 1-GPU benchmark).
* ``local_reduce`` -- K5, out = scale * sum_j ins[j].

``dims`` follow the paper's "2x4" notation when given as a string (outer x inner, e.g.
"2 nodes x 4 GPUs") and are innermost-first when given as a list.
"""
from __future__ import annotations

import ctypes
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DDL_LIB", os.path.join(HERE, "libddl.so"))

SUCCESS, ERR_INVALID_ARGUMENT, ERR_BAD_DIMS, ERR_UNSUPPORTED, ERR_CUDA, ERR_NO_PEER_ACCESS, \
    ERR_NOT_CONNECTED, ERR_TOO_LARGE, ERR_TIMEOUT, ERR_MISMATCH = range(10)
INT32, FLOAT32, BFLOAT16 = 0, 1, 2
SUM, AVG = 0, 1
ALGO_AUTO, ALGO_HIER, ALGO_ONESHOT, ALGO_LL = 0, 1, 2, 3
MAX_RANKS = 16

DTYPE_CODES = {"int32": INT32, "float32": FLOAT32, "bfloat16": BFLOAT16}
OP_CODES = {"sum": SUM, "avg": AVG}


class DDLError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        msg = _lib.ddl_result_string(code).decode()
        extra = _lib.ddl_last_error_string().decode() if code == ERR_CUDA else ""
        super().__init__(f"{what}: {msg}" + (f" ({extra})" if extra else ""))


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libddl.so not built at {LIB_PATH}: run ./build.sh (or __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    c_int, c_size, c_void, c_u64 = ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint64
    ip = ctypes.POINTER(c_int)
    pp = ctypes.POINTER(c_void)
    sig = {
        "ddl_version": (c_int, []),
        "ddl_build_flags": (c_int, []),
        "ddl_result_string": (ctypes.c_char_p, [c_int]),
        "ddl_last_error_string": (ctypes.c_char_p, []),
        "ddl_check_dims": (c_int, [c_int, ip, c_int]),
        "ddl_block_elems": (c_size, [c_size, c_int, c_int]),
        "ddl_plan_group": (c_int, [c_int, ip, c_int, c_int, c_int, ip]),
        "ddl_plan_blocks": (c_int, [c_int, ip, c_int, c_int, c_int, ip, ip]),
        "ddl_plan_barriers": (c_int, [c_int, ip, c_int, c_int, ip, ip, ip]),
        "ddl_plan_traffic": (c_int, [c_size, c_int, c_int, ip, c_int, c_int,
                                     ctypes.POINTER(c_u64), ctypes.POINTER(c_u64)]),
        "ddl_init": (c_int, [pp, c_int, c_int, ip, c_int, c_int, c_size]),
        "ddl_handle_size": (c_size, []),
        "ddl_export_handle": (c_int, [c_void, c_void]),
        "ddl_connect": (c_int, [c_void, c_void]),
        "ddl_buffer": (c_int, [c_void, pp, ctypes.POINTER(c_size)]),
        "ddl_peer_buffer": (c_int, [c_void, c_int, pp, ctypes.POINTER(c_size)]),
        "ddl_peer_copy": (c_int, [c_void, c_int, c_size, c_size, c_size, c_void]),
        "ddl_nvls_blob_size": (c_size, []),
        "ddl_debug_nvls_fd_selftest": (c_int, []),
        "ddl_nvls_prepare": (c_int, [c_void, c_size, c_void]),
        "ddl_nvls_attach": (c_int, [c_void, c_void, c_void]),
        "ddl_nvls_bind": (c_int, [c_void, c_void, c_void]),
        "ddl_nvls_commit": (c_int, [c_void, c_void]),
        "ddl_nvls_buffer": (c_int, [c_void, pp, ctypes.POINTER(c_size), ip]),
        "ddl_allreduce": (c_int, [c_void, c_void, c_size, c_int, c_int, c_void]),
        "ddl_allreduce_many": (c_int, [c_void, pp, ctypes.POINTER(c_size), c_int, c_int, c_int, c_void]),
        "ddl_reduce_scatter": (c_int, [c_void, c_void, c_void, c_size, c_int, c_int, c_void]),
        "ddl_allgather": (c_int, [c_void, c_void, c_void, c_size, c_int, c_void]),
        "ddl_async_error": (c_int, [c_void]),
        "ddl_set_algo": (c_int, [c_void, c_int, c_size]),
        "ddl_set_ll_max": (c_int, [c_void, c_size]),
        "ddl_set_timeout": (c_int, [c_void, c_u64]),
        "ddl_algo_for": (c_int, [c_void, c_size, c_int]),
        "ddl_ctas_for": (c_int, [c_void, c_size, c_int]),
        "ddl_debug_skip_rank": (c_int, [c_void, c_int]),
        "ddl_debug_connect_local": (c_int, [pp, c_int]),
        "ddl_reg_handle_size": (c_size, []),
        "ddl_register_export": (c_int, [c_void, c_void, c_size, c_void]),
        "ddl_register_connect": (c_int, [c_void, c_void, c_void, ip]),
        "ddl_deregister": (c_int, [c_void, c_int]),
        "ddl_debug_register_local": (c_int, [pp, pp, c_size, c_int, ip]),
        "ddl_debug_trace": (c_int, [c_void, c_void, c_size]),
        "ddl_finalize": (c_int, [c_void]),
        "ddl_loopback_init": (c_int, [pp, c_int, ip, c_int, c_int]),
        "ddl_init_loopback": (c_int, [pp, c_int, ip, c_int, c_int, c_size]),
        "ddl_group_allreduce": (c_int, [c_void, pp, c_size, c_int, c_int, c_void]),
        "ddl_group_allreduce_many": (c_int, [c_void, pp, ctypes.POINTER(c_size), c_int, c_int, c_int, c_void]),
        "ddl_group_reduce_scatter": (c_int, [c_void, pp, pp, c_size, c_int, c_int, c_void]),
        "ddl_group_allgather": (c_int, [c_void, pp, pp, c_size, c_int, c_void]),
        "ddl_local_reduce": (c_int, [pp, c_int, c_void, c_size, c_int, ctypes.c_float, c_void]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def has_experimental_kernels() -> bool:
    """PATH 3 (DDL_DYN) / PATH 4 (DDL_STEAL) compiled in (DDL_EXPERIMENTAL=1 bash build.sh)."""
    return bool(_lib.ddl_build_flags() & 1)


def lib() -> ctypes.CDLL:
    return _lib


def _check(code: int, what: str) -> None:
    if code != SUCCESS:
        raise DDLError(code, what)


def _ints(xs) -> ctypes.Array:
    return (ctypes.c_int * max(1, len(xs)))(*xs)


def _ptrs(xs) -> ctypes.Array:
    return (ctypes.c_void_p * max(1, len(xs)))(*xs)


def _sizes(xs) -> ctypes.Array:
    return (ctypes.c_size_t * max(1, len(xs)))(*xs)


def parse_dims(spec, nranks: int | None = None) -> list[int]:
    """'2x4' -> [4, 2] (written outer x inner); a list is already innermost-first;
    None -> [nranks] (one flat dimension)."""
    if spec is None:
        return [int(nranks)]
    if isinstance(spec, str):
        return [int(x) for x in spec.lower().split("x")][::-1]
    return [int(g) for g in spec]


# ---------------------------------------------------------------- host planner queries
def check_dims(nranks: int, dims) -> int:
    return _lib.ddl_check_dims(nranks, _ints(dims), len(dims))


def block_elems(count: int, nranks: int, dtype: str) -> int:
    return _lib.ddl_block_elems(count, nranks, DTYPE_CODES[dtype])


def plan_group(nranks: int, dims, rank: int, d: int) -> list[int]:
    out = (ctypes.c_int * dims[d])()
    _check(_lib.ddl_plan_group(nranks, _ints(dims), len(dims), rank, d, out), "ddl_plan_group")
    return list(out)


def plan_blocks(nranks: int, dims, rank: int, d: int) -> list[int]:
    out = (ctypes.c_int * nranks)()
    nb = ctypes.c_int()
    _check(_lib.ddl_plan_blocks(nranks, _ints(dims), len(dims), rank, d, out, ctypes.byref(nb)),
           "ddl_plan_blocks")
    return list(out[:nb.value])


def plan_barriers(nranks: int, dims, rank: int) -> list[list[int]]:
    nmax = 2 * len(dims) + 1
    peers = (ctypes.c_int * (nmax * nranks))()
    counts = (ctypes.c_int * nmax)()
    nb = ctypes.c_int()
    _check(_lib.ddl_plan_barriers(nranks, _ints(dims), len(dims), rank, peers, counts, ctypes.byref(nb)),
           "ddl_plan_barriers")
    return [list(peers[j * nranks:j * nranks + counts[j]]) for j in range(nb.value)]


def plan_traffic(count: int, dtype: str, nranks: int, dims, rank: int) -> tuple[list[int], list[int]]:
    k = len(dims)
    rs = (ctypes.c_uint64 * k)()
    ag = (ctypes.c_uint64 * k)()
    _check(_lib.ddl_plan_traffic(count, DTYPE_CODES[dtype], nranks, _ints(dims), k, rank, rs, ag),
           "ddl_plan_traffic")
    return list(rs), list(ag)


# ---------------------------------------------------------------- torch helpers
def _torch():
    import torch
    return torch


_DTYPE_NAMES = {}


def dtype_name(t) -> str:
    if not _DTYPE_NAMES:
        torch = _torch()
        _DTYPE_NAMES.update({torch.int32: "int32", torch.float32: "float32", torch.bfloat16: "bfloat16"})
    name = _DTYPE_NAMES.get(t.dtype)
    if name is None:
        raise DDLError(ERR_UNSUPPORTED, f"dtype {t.dtype}")
    return name


_RAW_STREAM = []


def _stream(stream=None, device=None) -> int:
    """cudaStream_t of `stream`, else of the current stream of `device` (default: current
    device).  torch.cuda.current_stream() costs ~3 us per call; the raw-handle query ~0.2."""
    if stream is not None:
        return stream.cuda_stream
    torch = _torch()
    if not _RAW_STREAM:
        _RAW_STREAM.append(getattr(torch._C, "_cuda_getCurrentRawStream", None))
    raw = _RAW_STREAM[0]
    if raw is None:
        return torch.cuda.current_stream(device).cuda_stream
    return raw(torch.cuda.current_device() if device is None else device)


def _require_cuda(t) -> None:
    if not t.is_cuda or not t.is_contiguous():
        raise DDLError(ERR_INVALID_ARGUMENT, "tensors must be contiguous CUDA tensors")


# ---------------------------------------------------------------- multi-process comm
def exchange_handles(dims, mine: bytes, group=None) -> bytes:
    """Bootstrap exchange (never on the data path): all-gather every rank's (dims, handle
    bytes) over the process group, check all ranks agree on dims, return the handles
    concatenated in rank order."""
    import torch.distributed as dist
    n = dist.get_world_size(group)
    allh = [None] * n
    dist.all_gather_object(allh, (list(dims), bytes(mine)), group=group)
    if any(d != list(dims) for d, _ in allh):
        raise DDLError(ERR_MISMATCH, "ranks passed different dims")
    if any(len(b) != len(mine) for _, b in allh):
        raise DDLError(ERR_MISMATCH, "handle sizes differ between ranks")
    return b"".join(b for _, b in allh)


class Comm:
    """One rank of a DDL communicator (one process per GPU).  Collective construction:
    every rank of ``group`` calls ``Comm(dims, ...)``; cudaIpc handles are exchanged with
    ``all_gather_object`` on the (gloo or NCCL) process group -- bootstrap only."""

    def __init__(self, dims=None, group=None, max_bytes: int = 256 << 20, device: int | None = None,
                 nvls_bytes: int | None = None):
        torch = _torch()
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.dims = parse_dims(dims, self.nranks)
        if math.prod(self.dims) != self.nranks:
            raise DDLError(ERR_BAD_DIMS, f"dims {self.dims} vs {self.nranks} ranks")
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _check(_lib.ddl_init(ctypes.byref(h), self.rank, self.nranks, _ints(self.dims), len(self.dims),
                             self.device, max_bytes), "ddl_init")
        self.h = h
        hs = _lib.ddl_handle_size()
        mine = ctypes.create_string_buffer(hs)
        _check(_lib.ddl_export_handle(self.h, mine), "ddl_export_handle")
        blob = ctypes.create_string_buffer(exchange_handles(self.dims, bytes(mine.raw), group), hs * self.nranks)
        _check(_lib.ddl_connect(self.h, blob), "ddl_connect")
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(_lib.ddl_buffer(self.h, ctypes.byref(p), ctypes.byref(n)), "ddl_buffer")
        self.buffer_ptr, self.buffer_bytes = p.value, n.value
        # NVLS phases (ddl_nvls_*): requested with nvls_bytes or DDL_NVLS_BYTES; falls back
        # to the direct phases on every rank if any rank cannot take part
        self.nvls_ptr, self.nvls_bytes, self.nvls_mask, self.nvls_status = 0, 0, 0, "off"
        nb = nvls_bytes if nvls_bytes is not None else int(os.environ.get("DDL_NVLS_BYTES", "0"))
        if nb > 0 and self.nranks > 1:
            self._nvls_setup(nb)

    def _nvls_setup(self, nbytes: int) -> None:
        import torch.distributed as dist
        bs = _lib.ddl_nvls_blob_size()

        def gather(blob):
            allb = [None] * self.nranks
            dist.all_gather_object(allb, bytes(blob.raw), group=self.group)
            return ctypes.create_string_buffer(b"".join(allb), bs * self.nranks)

        mine = ctypes.create_string_buffer(bs)
        _check(_lib.ddl_nvls_prepare(self.h, nbytes, mine), "ddl_nvls_prepare")
        allb = gather(mine)
        for step, fn in (("attach", _lib.ddl_nvls_attach), ("bind", _lib.ddl_nvls_bind)):
            mine = ctypes.create_string_buffer(bs)
            _check(fn(self.h, allb, mine), f"ddl_nvls_{step}")
            allb = gather(mine)
        statuses = [int.from_bytes(allb.raw[r * bs + 8:r * bs + 12], "little", signed=True) for r in range(self.nranks)]
        code = _lib.ddl_nvls_commit(self.h, allb)
        if code == SUCCESS:
            p, n, m = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_int()
            _check(_lib.ddl_nvls_buffer(self.h, ctypes.byref(p), ctypes.byref(n), ctypes.byref(m)), "ddl_nvls_buffer")
            self.nvls_ptr, self.nvls_bytes, self.nvls_mask, self.nvls_status = p.value, n.value, m.value, "on"
        elif code == ERR_UNSUPPORTED:
            self.nvls_status = f"fallback (per-rank setup status {statuses}: see ddl_nvls.h Status)"
        else:
            _check(code, "ddl_nvls_commit")

    def nvls_buffer(self, count: int, dtype, offset_bytes: int = 0):
        """A tensor view of this rank's NVLS buffer (same offset on every rank): all-reduces
        of it run the NVLS phases.  Raises if NVLS is off (see ``nvls_status``)."""
        torch = _torch()
        if not self.nvls_ptr:
            raise DDLError(ERR_UNSUPPORTED, f"NVLS {self.nvls_status}")
        esz = torch.tensor([], dtype=dtype).element_size()
        if offset_bytes % 256 or offset_bytes + count * esz > self.nvls_bytes:
            raise DDLError(ERR_TOO_LARGE, "view outside the NVLS buffer")
        full = _tensor_from_ptr(self.nvls_ptr, self.nvls_bytes, self.device)
        return full[offset_bytes:offset_bytes + count * esz].view(dtype)

    def buffer(self, count: int, dtype, offset_bytes: int = 0):
        """A torch tensor view of the symmetric zero-copy buffer (same offset on every rank)."""
        torch = _torch()
        esz = torch.tensor([], dtype=dtype).element_size()
        if offset_bytes % 256 or offset_bytes + count * esz > self.buffer_bytes:
            raise DDLError(ERR_TOO_LARGE, "view outside the symmetric buffer")
        full = _tensor_from_ptr(self.buffer_ptr, self.buffer_bytes, self.device)
        return full[offset_bytes:offset_bytes + count * esz].view(dtype)

    def peer_copy(self, peer: int, src_offset: int, dst_offset: int, nbytes: int, stream=None) -> None:
        """Enqueue a copy of nbytes from this rank's symmetric buffer into rank ``peer``'s over
        the cudaIpc mapping (copy engines); for measurement only (bench.py's peer-copy peak).
        Raw pointers stay inside the library: a torch view of peer memory would be attributed
        to the peer's device."""
        _check(_lib.ddl_peer_copy(self.h, peer, src_offset, dst_offset, nbytes, _stream(stream, self.device)),
               "ddl_peer_copy")

    def _zero_copy(self, ptr: int, nbytes: int) -> bool:
        """Inside the symmetric buffer or the NVLS buffer (read by peers in place)."""
        return (self.buffer_ptr <= ptr and ptr + nbytes <= self.buffer_ptr + self.buffer_bytes) or \
            (bool(self.nvls_ptr) and self.nvls_ptr <= ptr and ptr + nbytes <= self.nvls_ptr + self.nvls_bytes)

    def all_reduce(self, t, op: str = "sum", stream=None):
        """In-place all-reduce.  A tensor inside the symmetric buffer is reduced zero-copy;
        any other tensor larger than the staging workspace is reduced in workspace-sized
        pieces (each element's result depends only on that element across ranks, so the
        split never changes a bit)."""
        _require_cuda(t)
        dt = DTYPE_CODES[dtype_name(t)]
        nbytes = t.numel() * t.element_size()
        inside = self._zero_copy(t.data_ptr(), nbytes)
        piece = (self.buffer_bytes // t.element_size()) // 256 * 256
        if inside or nbytes <= self.buffer_bytes or piece == 0:
            _check(_lib.ddl_allreduce(self.h, t.data_ptr(), t.numel(), dt, OP_CODES[op],
                                      _stream(stream, t.device.index)), "ddl_allreduce")
            return t
        flat = t.view(-1)
        for lo in range(0, t.numel(), piece):
            part = flat[lo:lo + piece]
            _check(_lib.ddl_allreduce(self.h, part.data_ptr(), part.numel(), dt, OP_CODES[op],
                                      _stream(stream, t.device.index)), "ddl_allreduce")
        return t

    def all_reduce_many(self, ts, op: str = "sum", stream=None):
        """Grouped in-place all-reduce of several tensors of one dtype (e.g. the gradient
        buckets of a step): zero-copy ones share one launch over DDL_CHANNELS channels
        (``ddl_allreduce_many``); results equal one all_reduce per tensor bit for bit.
        Every rank passes the same tensor sizes in the same order."""
        if not ts:
            return ts
        dt = dtype_name(ts[0])
        rest = []
        for t in ts:
            _require_cuda(t)
            if dtype_name(t) != dt:
                raise DDLError(ERR_INVALID_ARGUMENT, "all_reduce_many: mixed dtypes")
            nbytes = t.numel() * t.element_size()
            inside = self._zero_copy(t.data_ptr(), nbytes)
            if not inside and nbytes > self.buffer_bytes:
                self.all_reduce(t, op, stream)   # staged in workspace-sized pieces
            else:
                rest.append(t)
        if rest:
            _check(_lib.ddl_allreduce_many(self.h, _ptrs([t.data_ptr() for t in rest]),
                                           _sizes([t.numel() for t in rest]), len(rest), DTYPE_CODES[dt],
                                           OP_CODES[op], _stream(stream, rest[0].device.index)),
                   "ddl_allreduce_many")
        return ts

    def register(self, t) -> int:
        """Collective: register a persistent device tensor (same size on every rank) so that
        all-reduces on it -- or on a view at the same offset on every rank -- are zero-copy."""
        import torch.distributed as dist
        _require_cuda(t)
        nbytes = t.numel() * t.element_size()
        blob = ctypes.create_string_buffer(_lib.ddl_reg_handle_size())
        _check(_lib.ddl_register_export(self.h, t.data_ptr(), nbytes, blob), "ddl_register_export")
        allb = [None] * self.nranks
        dist.all_gather_object(allb, bytes(blob.raw), group=self.group)
        joined = ctypes.create_string_buffer(b"".join(allb), len(blob.raw) * self.nranks)
        rid = ctypes.c_int()
        _check(_lib.ddl_register_connect(self.h, t.data_ptr(), joined, ctypes.byref(rid)), "ddl_register_connect")
        return rid.value

    def deregister(self, reg_id: int) -> None:
        _check(_lib.ddl_deregister(self.h, reg_id), "ddl_deregister")

    def reduce_scatter(self, out, inp, op: str = "sum", stream=None):
        _require_cuda(out)
        _require_cuda(inp)
        if inp.numel() != out.numel() * self.nranks or inp.dtype != out.dtype:
            raise DDLError(ERR_INVALID_ARGUMENT, "reduce_scatter: inp must hold nranks * out.numel()")
        _check(_lib.ddl_reduce_scatter(self.h, inp.data_ptr(), out.data_ptr(), out.numel(),
                                       DTYPE_CODES[dtype_name(out)], OP_CODES[op],
                                       _stream(stream, out.device.index)),
               "ddl_reduce_scatter")
        return out

    def all_gather(self, out, inp, stream=None):
        _require_cuda(out)
        _require_cuda(inp)
        if out.numel() != inp.numel() * self.nranks or inp.dtype != out.dtype:
            raise DDLError(ERR_INVALID_ARGUMENT, "all_gather: out must hold nranks * inp.numel()")
        _check(_lib.ddl_allgather(self.h, inp.data_ptr(), out.data_ptr(), inp.numel(),
                                  DTYPE_CODES[dtype_name(out)], _stream(stream, out.device.index)), "ddl_allgather")
        return out

    def set_algo(self, algo: int, oneshot_max_bytes: int = 512 << 10) -> None:
        _check(_lib.ddl_set_algo(self.h, algo, oneshot_max_bytes), "ddl_set_algo")

    def set_ll_max(self, ll_max_bytes: int) -> None:
        _check(_lib.ddl_set_ll_max(self.h, ll_max_bytes), "ddl_set_ll_max")

    def algo_for(self, count: int, dtype: str) -> int:
        return _lib.ddl_algo_for(self.h, count, DTYPE_CODES[dtype])

    def async_error(self) -> int:
        return _lib.ddl_async_error(self.h)

    def finalize(self) -> None:
        if self.h:
            import torch.distributed as dist
            _torch().cuda.synchronize()
            dist.barrier(group=self.group)
            _lib.ddl_finalize(self.h)
            self.h = None


def auto_dims(world: int, local_world: int | None = None) -> list[int]:
    """Topology-aware factorisation (the role of ddlrun's topology config files):
    ranks of one node share NVSwitch, where every pair has the same bandwidth, so one flat
    dimension (fewest phases and barriers) is best inside a node -- measured in loopback
    (profiles/r01_loopback_sweep.csv: [8] beats 2x4 and 2x2x2 at every size).  Across nodes
    the node is the outer dimension (see multinode.TwoLevelComm for the off-node fabric)."""
    import os
    if local_world is None:
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    local_world = max(1, min(local_world, world))
    if world % local_world:
        raise DDLError(ERR_BAD_DIMS, f"{world} ranks do not split into nodes of {local_world}")
    nodes = world // local_world
    return [local_world] if nodes == 1 else [local_world, nodes]


def init(dims=None, group=None, max_bytes: int = 256 << 20, nvls_bytes: int | None = None) -> Comm:
    """``ddl.init(dims)``: the analogue of the paper's ``import ddl`` + ``ddlrun`` setup
     under torchrun.  ``dims="auto"`` picks :func:`auto_dims`.  The
    environment variable ``DDL_DIMS`` (e.g. ``2x4``, or ``auto``) overrides ``dims`` -- the
    role of ddlrun's topology configuration -- and must be equal on every rank.
    ``nvls_bytes`` (or DDL_NVLS_BYTES) requests the NVSwitch multicast phases (Comm)."""
    import torch.distributed as dist
    return Comm(resolve_dims(dims, dist.get_world_size(group)), group, max_bytes, nvls_bytes=nvls_bytes)


def resolve_dims(dims, world: int, local_world: int | None = None) -> list[int]:
    """dims as ddl.init takes them, after the DDL_DIMS override: None -> [world], "auto" ->
    auto_dims, "2x4" -> [4, 2], a list as is (innermost first)."""
    import os
    dims = os.environ.get("DDL_DIMS") or dims
    if isinstance(dims, str) and dims == "auto":
        return auto_dims(world, local_world)
    return parse_dims(dims, world)


def _tensor_from_ptr(ptr: int, nbytes: int, device: int):
    """Wrap library-owned device memory as a uint8 torch tensor (no copy, not owned)."""
    torch = _torch()

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                    "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(), device=f"cuda:{device}")


# ---------------------------------------------------------------- loopback (1 GPU)
class Loopback:
    """P virtual ranks on one GPU: the same kernels and barrier protocol as ``Comm``,
    launched once for all ranks (cooperative launch)."""

    def __init__(self, nranks: int, dims=None, device: int | None = None):
        torch = _torch()
        self.nranks = nranks
        self.dims = parse_dims(dims, nranks)
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _check(_lib.ddl_loopback_init(ctypes.byref(h), nranks, _ints(self.dims), len(self.dims), self.device),
               "ddl_loopback_init")
        self.h = h

    def all_reduce(self, bufs, op: str = "sum", stream=None):
        for b in bufs:
            _require_cuda(b)
        _check(_lib.ddl_group_allreduce(self.h, _ptrs([b.data_ptr() for b in bufs]), bufs[0].numel(),
                                        DTYPE_CODES[dtype_name(bufs[0])], OP_CODES[op],
                                        _stream(stream, bufs[0].device.index)),
               "ddl_group_allreduce")
        return bufs

    def all_reduce_many(self, buckets, op: str = "sum", stream=None):
        """Grouped all-reduce: buckets[i][r] is virtual rank r's copy of buffer i (one dtype);
        one cooperative launch for the hierarchical-sized buffers (``ddl_group_allreduce_many``)."""
        if not buckets:
            return buckets
        dt = dtype_name(buckets[0][0])
        ptrs = []
        for b in buckets:
            if len(b) != self.nranks or any(dtype_name(t) != dt or t.numel() != b[0].numel() for t in b):
                raise DDLError(ERR_INVALID_ARGUMENT, "all_reduce_many: one same-size tensor per rank per bucket")
            for t in b:
                _require_cuda(t)
            ptrs += [t.data_ptr() for t in b]
        _check(_lib.ddl_group_allreduce_many(self.h, _ptrs(ptrs), _sizes([b[0].numel() for b in buckets]),
                                             len(buckets), DTYPE_CODES[dt], OP_CODES[op],
                                             _stream(stream, buckets[0][0].device.index)),
               "ddl_group_allreduce_many")
        return buckets

    def reduce_scatter(self, outs, inps, op: str = "sum", stream=None):
        _check(_lib.ddl_group_reduce_scatter(self.h, _ptrs([t.data_ptr() for t in inps]),
                                             _ptrs([t.data_ptr() for t in outs]), outs[0].numel(),
                                             DTYPE_CODES[dtype_name(outs[0])], OP_CODES[op],
                                             _stream(stream, outs[0].device.index)),
               "ddl_group_reduce_scatter")
        return outs

    def all_gather(self, outs, inps, stream=None):
        _check(_lib.ddl_group_allgather(self.h, _ptrs([t.data_ptr() for t in inps]),
                                        _ptrs([t.data_ptr() for t in outs]), inps[0].numel(),
                                        DTYPE_CODES[dtype_name(outs[0])], _stream(stream, outs[0].device.index)),
               "ddl_group_allgather")
        return outs

    def set_algo(self, algo: int, oneshot_max_bytes: int = 512 << 10) -> None:
        _check(_lib.ddl_set_algo(self.h, algo, oneshot_max_bytes), "ddl_set_algo")

    def set_timeout(self, ms: int) -> None:
        _check(_lib.ddl_set_timeout(self.h, ms), "ddl_set_timeout")

    def algo_for(self, count: int, dtype: str) -> int:
        return _lib.ddl_algo_for(self.h, count, DTYPE_CODES[dtype])

    def ctas_for(self, count: int, dtype: str) -> int:
        return _lib.ddl_ctas_for(self.h, count, DTYPE_CODES[dtype])

    def trace(self):
        """[nranks][cmax][128] globaltimer (slot 127: the SM id) stamps of the last call (DDL_TRACE=1 at init)."""
        import numpy as np
        torch = _torch()
        cmax = 4 * torch.cuda.get_device_properties(self.device).multi_processor_count
        out = np.zeros((self.nranks, cmax, 128), dtype=np.uint64)
        _check(_lib.ddl_debug_trace(self.h, out.ctypes.data, out.nbytes), "ddl_debug_trace")
        return out

    def debug_skip_rank(self, r: int) -> None:
        _check(_lib.ddl_debug_skip_rank(self.h, r), "ddl_debug_skip_rank")

    def async_error(self) -> int:
        return _lib.ddl_async_error(self.h)

    def finalize(self) -> None:
        if self.h:
            _lib.ddl_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.finalize()
        except Exception:
            pass


# ---------------------------------------------------------------- in-process group (tests)
class InProcessGroup:
    """P ranks of the MULTI-PROCESS code path inside one process on one GPU (test hook
    ``ddl_debug_connect_local``: peers addressed directly instead of through cudaIpc).
    Each rank's call is launched on its own stream; the P kernels run concurrently."""

    def __init__(self, nranks: int, dims=None, max_bytes: int = 64 << 20, device: int | None = None):
        torch = _torch()
        self.nranks = nranks
        self.dims = parse_dims(dims, nranks)
        self.device = torch.cuda.current_device() if device is None else device
        hs = []
        for r in range(nranks):
            h = ctypes.c_void_p()
            _check(_lib.ddl_init(ctypes.byref(h), r, nranks, _ints(self.dims), len(self.dims), self.device,
                                 max_bytes), "ddl_init")
            hs.append(h)
        self.hs = hs
        _check(_lib.ddl_debug_connect_local(_ptrs([h.value for h in hs]), nranks), "ddl_debug_connect_local")
        self.streams = [torch.cuda.Stream() for _ in range(nranks)]
        self.buf = []
        for h in hs:
            p = ctypes.c_void_p()
            n = ctypes.c_size_t()
            _check(_lib.ddl_buffer(h, ctypes.byref(p), ctypes.byref(n)), "ddl_buffer")
            self.buf.append(_tensor_from_ptr(p.value, n.value, self.device))

    def buffer(self, r: int, count: int, dtype, offset_bytes: int = 0):
        esz = _torch().tensor([], dtype=dtype).element_size()
        return self.buf[r][offset_bytes:offset_bytes + count * esz].view(dtype)

    def register(self, tensors) -> int:
        """Register one tensor per rank (equal sizes) for zero-copy all-reduces."""
        rid = ctypes.c_int()
        nbytes = tensors[0].numel() * tensors[0].element_size()
        _check(_lib.ddl_debug_register_local(_ptrs([h.value for h in self.hs]),
                                             _ptrs([t.data_ptr() for t in tensors]), nbytes, self.nranks,
                                             ctypes.byref(rid)), "ddl_debug_register_local")
        return rid.value

    def _each(self, fn):
        torch = _torch()
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        for r in range(self.nranks):
            fn(r, self.streams[r].cuda_stream)
        for s in self.streams:
            cur.wait_stream(s)

    def all_reduce(self, bufs, op: str = "sum"):
        dt = DTYPE_CODES[dtype_name(bufs[0])]
        self._each(lambda r, s: _check(_lib.ddl_allreduce(self.hs[r], bufs[r].data_ptr(), bufs[r].numel(), dt,
                                                          OP_CODES[op], s), "ddl_allreduce"))
        return bufs

    def all_reduce_many(self, buckets, op: str = "sum"):
        """buckets[i][r]: rank r's tensor of bucket i; every rank calls ddl_allreduce_many."""
        dt = DTYPE_CODES[dtype_name(buckets[0][0])]
        sizes = _sizes([b[0].numel() for b in buckets])
        self._each(lambda r, s: _check(_lib.ddl_allreduce_many(self.hs[r], _ptrs([b[r].data_ptr() for b in buckets]),
                                                               sizes, len(buckets), dt, OP_CODES[op], s),
                                       "ddl_allreduce_many"))
        return buckets

    def reduce_scatter(self, outs, inps, op: str = "sum"):
        dt = DTYPE_CODES[dtype_name(outs[0])]
        self._each(lambda r, s: _check(_lib.ddl_reduce_scatter(self.hs[r], inps[r].data_ptr(), outs[r].data_ptr(),
                                                               outs[r].numel(), dt, OP_CODES[op], s),
                                       "ddl_reduce_scatter"))
        return outs

    def all_gather(self, outs, inps):
        dt = DTYPE_CODES[dtype_name(outs[0])]
        self._each(lambda r, s: _check(_lib.ddl_allgather(self.hs[r], inps[r].data_ptr(), outs[r].data_ptr(),
                                                          inps[r].numel(), dt, s), "ddl_allgather"))
        return outs

    def set_algo(self, algo: int, oneshot_max_bytes: int = 512 << 10) -> None:
        for h in self.hs:
            _check(_lib.ddl_set_algo(h, algo, oneshot_max_bytes), "ddl_set_algo")

    def set_ll_max(self, ll_max_bytes: int) -> None:
        for h in self.hs:
            _check(_lib.ddl_set_ll_max(h, ll_max_bytes), "ddl_set_ll_max")

    def algo_for(self, count: int, dtype: str) -> int:
        return _lib.ddl_algo_for(self.hs[0], count, DTYPE_CODES[dtype])

    def async_error(self) -> int:
        return max(_lib.ddl_async_error(h) for h in self.hs)

    def finalize(self) -> None:
        _torch().cuda.synchronize()
        for h in self.hs:
            _lib.ddl_finalize(h)
        self.hs = []


# ---------------------------------------------------------------- K5
def local_reduce(ins, out, scale: float = 1.0, stream=None):
    """out = scale * sum_j ins[j] (ascending j), the 1-GPU HBM-roofline kernel (launched on
    out's device)."""
    for t in list(ins) + [out]:
        _require_cuda(t)
    torch = _torch()
    dev = out.device.index

    def call():
        _check(_lib.ddl_local_reduce(_ptrs([t.data_ptr() for t in ins]), len(ins), out.data_ptr(), out.numel(),
                                     DTYPE_CODES[dtype_name(out)], float(scale), _stream(stream, dev)),
               "ddl_local_reduce")
    if dev == torch.cuda.current_device():
        call()
    else:
        with torch.cuda.device(dev):
            call()
    return out
