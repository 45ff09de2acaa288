"""CPU ORACLE for PowerAI DDL's topology-aware all-reduce -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.  The product path
(``paper_1811_12174_b200`` + ``libddl.so``) never imports, links or executes it, and this
module imports nothing from the product: the two share no code.  Only
``synthetic_inputs`` (random draws, no arithmetic of the method) feeds both.

What is computed (the method).  PAPER.md §2.1: "decompose one all-reduce
operation into a series of reduce-scatter and all-gather patterns in a topology-aware
fashion"; feature (1): adapt "to the hierarchy of communication bandwidths".  The
ranks are factorised as ``dims = [g_0, ..., g_{k-1}]`` (innermost first, prod = P;
SPEC S:L264-270).  Reduce-scatter runs innermost -> outermost, all-gather outermost ->
innermost.  The plain definition the schedule reaches is
``y[e] = sum_r x_r[e]`` (times 1/P for avg), identical on every rank.

The module is a step-by-step, lockstep simulation of P ranks ("a deterministic
lockstep loop inside one thread"), in the order and notation of SURVEY.md 8(a)/(c):

* coords  c_d(r) = floor(r / G_d) mod g_d,  G_d = prod_{j<d} g_j
* group of r in dim d: m_v = r + (v - c_d(r)) * G_d, v = 0..g_d-1            (a1)
* blocks: q = roundup(ceil(n/P), 16 B / w); block b = [min(n,bq), min(n,(b+1)q))  (a3)
* A_d(r) = {b : c_j(b) = c_j(r) for all j < d}: blocks rank r still reduces before RS d
* RS phase d: for b in A_{d+1}(r): y = ((x_{m_0} + x_{m_1}) + ...) + x_{m_{g-1}}  (a4),
  every add rounded in the accumulator type; last RS phase with g_d > 1 multiplies by
  fl32(1/P) for avg (a5); the result is cast to the I/O type and stored in place.
* AG phase d: copy A_{d+1}(m_v) from every group peer m_v, v != c_d(r)     (a6)

Readings of the paper where it is silent (SURVEY.md 8(c) ledger):
direct within-group fold in ascending c_d (ledger 1); "2x4" means 2 outer x 4 inner, i.e.
dims [4, 2] (ledger 2); strided P-block layout, rank r owns block r (ledger 3); ragged
blocks, no padding (ledger 4); avg = one multiply by fl32(1/P) of the fully reduced fp32
value, fused into the last RS phase whose g_d > 1 (ledger 5); int32 avg rejected (ledger 6);
bf16 accumulates in fp32 within a phase and is rounded RNE to bf16 at every phase boundary
(ledger 7); IEEE RNE everywhere, no FMA, no flush-to-zero (ledger 9); int32 wraps (ledger 11).
NVLS phases (SURVEY.md 8(f) NEXT-1, P:L54 (3) "mix and match" per piece; DESIGN.md reading
15): ``allreduce(..., nvls_dims=...)`` runs those dims' RS phases "in the switch" -- one
admissible result of an unspecified fold order (_switch_sum) -- and ``fold_error_bound``
gives the bound every fold order meets, which is how NVLS results are gated (int32 exact).

Arithmetic: numpy int32 (wrapping) and float32 (IEEE binary32, round-to-nearest-even, no
FTZ) elementwise adds, one per step in the order above.  bf16 rounding is written out on
the bit patterns (RNE, NaN kept quiet).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

INT32, FLOAT32, BFLOAT16 = "int32", "float32", "bfloat16"
DTYPES = (INT32, FLOAT32, BFLOAT16)
ITEMSIZE = {INT32: 4, FLOAT32: 4, BFLOAT16: 2}
STORAGE = {INT32: np.int32, FLOAT32: np.float32, BFLOAT16: np.uint16}   # bf16 held as bit patterns


class DdlOracleError(ValueError):
    pass


class BadDims(DdlOracleError):          # SPEC S:L280-282 "BadArity"
    pass


class LengthMismatch(DdlOracleError):
    pass


class EmptyBuffers(DdlOracleError):     # SPEC S:L333 (no ranks at all)
    pass


class Unsupported(DdlOracleError):      # ledger 6: int32 + avg
    pass


# ----------------------------------------------------------------------------- topology (a1)

def parse_dims(spec) -> list[int]:
    """'2x4' (written outer x inner, as "2 nodes x 4 GPUs") -> [4, 2]
    (innermost first).  A list/tuple is taken as already innermost-first."""
    if isinstance(spec, str):
        parts = [int(p) for p in spec.lower().split("x")]
        return parts[::-1]
    return [int(g) for g in spec]


def validate_dims(dims, nranks: int) -> list[int]:
    """every group_size >= 1 and prod group_size = ranks (else BadArity)."""
    dims = [int(g) for g in dims]
    if nranks < 1:
        raise EmptyBuffers("no ranks")
    if not 1 <= len(dims) <= 8 or any(g < 1 for g in dims) or math.prod(dims) != nranks:
        raise BadDims(f"dims {dims} do not factorise {nranks} ranks")
    return dims


def prefix(dims, d: int) -> int:
    """G_d = prod_{j<d} g_j."""
    return math.prod(dims[:d])


def coord(r: int, d: int, dims) -> int:
    """c_d(r) = floor(r / G_d) mod g_d  (mixed radix, innermost fastest)."""
    return (r // prefix(dims, d)) % dims[d]


def group(r: int, d: int, dims) -> list[int]:
    """Members of r's group in dim d, ordered by their coordinate v = c_d(m_v)."""
    G = prefix(dims, d)
    return [r + (v - coord(r, d, dims)) * G for v in range(dims[d])]


def active_blocks(r: int, d: int, dims) -> list[int]:
    """A_d(r) = {b : c_j(b) = c_j(r) for all j < d}, ascending, written as the definition."""
    P = math.prod(dims)
    return [b for b in range(P) if all(coord(b, j, dims) == coord(r, j, dims) for j in range(d))]


def schedule(dims) -> list[tuple[str, int]]:
    """RS over dims innermost -> outermost, then AG outermost -> innermost.
    A dim with g_d = 1 has no partner and no phase (ledger 13)."""
    live = [d for d, g in enumerate(dims) if g > 1]
    return [("RS", d) for d in live] + [("AG", d) for d in reversed(live)]


# ----------------------------------------------------------------------------- layout (a3)

def block_elems(n: int, nranks: int, dtype: str) -> int:
    """q = roundup(ceil(n/P), V), V = 16 B / w elements (one 128-bit vector)."""
    V = 16 // ITEMSIZE[dtype]
    per = -(-n // nranks)
    return -(-per // V) * V


def block_range(b: int, n: int, q: int) -> tuple[int, int]:
    return min(n, b * q), min(n, (b + 1) * q)


# ----------------------------------------------------------------------------- numerics

def bf16_round(f: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern, IEEE round-to-nearest-even (ties to even), overflow to
    inf, NaN kept NaN (quiet bit set), subnormals kept (no flush)."""
    u = np.asarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) & np.uint64(0xFFFF)
    nan = (u & np.uint64(0x7FFFFFFF)) > np.uint64(0x7F800000)
    r = np.where(nan, ((u >> np.uint64(16)) | np.uint64(0x40)) & np.uint64(0xFFFF), r)
    return r.astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    """bf16 bit pattern -> float32 (exact: bf16 is the upper half of binary32)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def _to_acc(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == BFLOAT16:
        return bf16_to_f32(x)
    return np.array(x, dtype=STORAGE[dtype], copy=True)


def _from_acc(acc: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == BFLOAT16:
        return bf16_round(acc)
    return acc.astype(STORAGE[dtype], copy=False)


def avg_scale(nranks: int) -> np.float32:
    """fl32(1/P), computed once in binary32 (ledger 5)."""
    return np.float32(1.0) / np.float32(nranks)


# ----------------------------------------------------------------------------- schedule

@dataclass
class Traffic:
    """Per-rank byte counters of one call (SPEC S:L371 traffic conservation)."""
    remote_read: list = field(default_factory=list)   # [rank] -> {phase: bytes read from peers}
    local_read: list = field(default_factory=list)
    local_write: list = field(default_factory=list)

    @classmethod
    def new(cls, P: int) -> "Traffic":
        return cls([dict() for _ in range(P)], [dict() for _ in range(P)], [dict() for _ in range(P)])

    def add(self, table: str, r: int, phase, nbytes: int) -> None:
        t = getattr(self, table)[r]
        t[phase] = t.get(phase, 0) + nbytes


def _check_buffers(bufs, dtype: str) -> tuple[int, int]:
    if dtype not in DTYPES:
        raise Unsupported(f"dtype {dtype}")
    if len(bufs) == 0:
        raise EmptyBuffers("no rank buffers")
    n = len(bufs[0])
    if any(len(b) != n for b in bufs):
        raise LengthMismatch("rank buffers differ in length")
    return len(bufs), n


def _switch_sum(vals, dtype):
    """An NVLS phase: the NVSwitch returns the group's sum in an order
    it does not specify (ledger 14: every order is "correct").  The oracle takes one admissible
    result: the binary64 sum of the members' values, rounded once to binary32 (int32: the
    exact sum mod 2^32, which every order reaches).  GPU results of NVLS phases are compared
    with fold_error_bound, never bit for bit (fp32 / bf16)."""
    if dtype == INT32:
        acc = vals[0].astype(np.int64)
        for v in vals[1:]:
            acc = acc + v.astype(np.int64)
        return (acc & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    acc = vals[0].astype(np.float64)
    for v in vals[1:]:
        acc = acc + v.astype(np.float64)
    return acc.astype(np.float32)


def _rs_phases(B, dims, dtype, op, n, q, traffic, nvls_dims=()):
    """one lockstep pass per RS phase, innermost dim first.  Dims in
    nvls_dims reduce "in the switch" (_switch_sum) instead of the ascending direct fold."""
    P = len(B)
    w = ITEMSIZE[dtype]
    live = [d for d, g in enumerate(dims) if g > 1]
    last = live[-1] if live else None
    for d in live:
        snap = [x.copy() for x in B]           # every rank reads the state at phase start
        for r in range(P):
            members = group(r, d, dims)
            for b in active_blocks(r, d + 1, dims):
                lo, hi = block_range(b, n, q)
                if lo == hi:
                    continue
                if d in nvls_dims:
                    acc = _switch_sum([_to_acc(snap[m][lo:hi], dtype) for m in members], dtype)
                else:
                    acc = _to_acc(snap[members[0]][lo:hi], dtype)
                    for v in range(1, len(members)):
                        acc = acc + _to_acc(snap[members[v]][lo:hi], dtype)
                if op == "avg" and d == last:
                    acc = acc * avg_scale(P)
                B[r][lo:hi] = _from_acc(acc, dtype)
                if traffic is not None:
                    nb = (hi - lo) * w
                    traffic.add("remote_read", r, ("RS", d), nb * (len(members) - 1))
                    traffic.add("local_read", r, ("RS", d), nb)
                    traffic.add("local_write", r, ("RS", d), nb)


def _ag_phases(B, dims, dtype, n, q, traffic):
    """all-gather phases, outermost dim first; pure bit copies."""
    P = len(B)
    w = ITEMSIZE[dtype]
    live = [d for d, g in enumerate(dims) if g > 1]
    for d in reversed(live):
        snap = [x.copy() for x in B]
        for r in range(P):
            c = coord(r, d, dims)
            for v, m in enumerate(group(r, d, dims)):
                if v == c:
                    continue
                for b in active_blocks(m, d + 1, dims):
                    lo, hi = block_range(b, n, q)
                    B[r][lo:hi] = snap[m][lo:hi]
                    if traffic is not None and hi > lo:
                        traffic.add("remote_read", r, ("AG", d), (hi - lo) * w)
                        traffic.add("local_write", r, ("AG", d), (hi - lo) * w)


def allreduce(bufs, dims, dtype: str, op: str = "sum", q: int | None = None,
              traffic: Traffic | None = None, nvls_dims=()) -> list[np.ndarray]:
    """ddl_allreduce semantics: returns every rank's buffer after the full schedule
    RS(d=0..k-1) then AG(d=k-1..0).  Inputs are not modified.  nvls_dims: the dims whose
    phases run in the NVSwitch (per-phase algorithm, P:L54 (3)); their RS fold order is the
    switch's (_switch_sum), their AG is the same bit copy."""
    P, n = _check_buffers(bufs, dtype)
    dims = validate_dims(dims, P)
    if op not in ("sum", "avg"):
        raise Unsupported(f"op {op}")
    if op == "avg" and dtype == INT32:
        raise Unsupported("int32 avg is undefined (ledger 6)")
    q = block_elems(n, P, dtype) if q is None else q
    B = [np.array(x, dtype=STORAGE[dtype], copy=True) for x in bufs]
    _rs_phases(B, dims, dtype, op, n, q, traffic, tuple(nvls_dims))
    _ag_phases(B, dims, dtype, n, q, traffic)
    return B


def reduce_scatter(bufs, dims, dtype: str, op: str = "sum", traffic: Traffic | None = None):
    """ddl_reduce_scatter semantics (NCCL layout): n = P * recvcount, block size q =
    recvcount, rank r receives block r = [r*q, (r+1)*q) of the reduced vector."""
    P, n = _check_buffers(bufs, dtype)
    dims = validate_dims(dims, P)
    if n % P:
        raise LengthMismatch("reduce_scatter needs n = P * recvcount")
    if op == "avg" and dtype == INT32:
        raise Unsupported("int32 avg is undefined (ledger 6)")
    q = n // P
    B = [np.array(x, dtype=STORAGE[dtype], copy=True) for x in bufs]
    _rs_phases(B, dims, dtype, op, n, q, traffic)
    return [B[r][r * q:(r + 1) * q].copy() for r in range(P)]


def allgather(sends, dims, dtype: str, traffic: Traffic | None = None):
    """ddl_allgather semantics: rank r's sendcount elements land at [r*q, (r+1)*q) of
    every rank's output, q = sendcount; the AG phases alone."""
    P, q = _check_buffers(sends, dtype)
    dims = validate_dims(dims, P)
    n = P * q
    B = [np.zeros(n, dtype=STORAGE[dtype]) for _ in range(P)]
    for r in range(P):
        B[r][r * q:(r + 1) * q] = sends[r]
    _ag_phases(B, dims, dtype, n, q, traffic)
    return B


def allreduce_sampled(bufs, dims, dtype: str, op: str, idx) -> np.ndarray:
    """Reduced values at element indices ``idx`` only.  The schedule's result at element e
    depends only on (x_0[e], ..., x_{P-1}[e]) and dims -- never on the block e lies in
    (every RS phase folds the same group members in the same order for every block) --
    so running the schedule on the gathered columns gives the same values.  This is pinned
    by tests/test_oracle.py::test_sampled_equals_full."""
    cols = [np.asarray(x)[idx] for x in bufs]
    return allreduce(cols, dims, dtype, op)[0]


def local_reduce(ins, dtype: str, scale: float = 1.0) -> np.ndarray:
    """K5 / SURVEY.md 8(a) a8: out = s * sum_{j<g} in_j over g local buffers, folded in
    ascending j in the accumulator type, one multiply by fl32(s) (skipped when s == 1),
    then the output cast."""
    g, n = _check_buffers(ins, dtype)
    if dtype == INT32 and scale != 1.0:
        raise Unsupported("int32 local reduce takes no scale")
    acc = _to_acc(ins[0], dtype)
    for j in range(1, g):
        acc = acc + _to_acc(ins[j], dtype)
    if scale != 1.0:
        acc = acc * np.float32(scale)
    return _from_acc(acc, dtype)


# ----------------------------------------------------------------------------- plain definition

def naive_sum(bufs, dtype: str) -> np.ndarray:
    """The plain definition y = sum_r x_r, rank by rank in ascending r.
    int32: exact integer sum reduced mod 2^32 (two's complement); fp32/bf16: float32
    left fold (inputs widened exactly), result in float32."""
    if dtype == INT32:
        tot = np.zeros(len(bufs[0]), dtype=np.int64)
        for x in bufs:
            tot = (tot + np.asarray(x, dtype=np.int64)) & 0xFFFFFFFF
        return tot.astype(np.uint32).view(np.int32)
    acc = np.zeros(len(bufs[0]), dtype=np.float32)
    for i, x in enumerate(bufs):
        xf = bf16_to_f32(x) if dtype == BFLOAT16 else np.asarray(x, dtype=np.float32)
        acc = xf.copy() if i == 0 else acc + xf
    return acc


def exact_sum_f64(bufs, dtype: str) -> tuple[np.ndarray, np.ndarray]:
    """fp64 sum and sum of magnitudes, for the Higham-bound tolerance (ledger 8)."""
    xs = [bf16_to_f32(x) if dtype == BFLOAT16 else np.asarray(x, dtype=np.float32) for x in bufs]
    s = np.zeros(len(xs[0]), dtype=np.float64)
    a = np.zeros(len(xs[0]), dtype=np.float64)
    for x in xs:
        s += x.astype(np.float64)
        a += np.abs(x.astype(np.float64))
    return s, a


def fold_error_bound(bufs, dims, dtype: str, op: str = "sum"):
    """(s, bound): the exact (binary64) result s -- the sum, or the sum / P for avg -- and a
    per-element bound on |y - s| that holds for ANY summation order inside the phases (the
    direct ascending folds and the switch's unspecified NVLS folds alike; ledger 8/14).
    fp32: every order is a binary tree of P-1 rounded adds, |err| <= gamma_{P-1} sum|x|
    (Higham 2002, eq. 4.4) with u = 2^-24, plus the avg multiply by fl32(1/P) (2u |s|/P).
    bf16: additionally one RNE to bf16 (u = 2^-8) at each of the k phase boundaries.  A tiny
    absolute term covers subnormal results (no flush: ledger 9)."""
    P = len(bufs)
    s64, a64 = exact_sum_f64(bufs, dtype)
    k = sum(1 for g in dims if g > 1)
    u = 2.0 ** -24
    g = (P - 1) * u / (1 - (P - 1) * u)
    if dtype == BFLOAT16:
        ub = 2.0 ** -8
        bound = (k * ub + g * (1 + ub) ** k) * (1 + ub) ** k * a64
    else:
        bound = g * a64
    tiny = P * 2.0 ** -149
    if op == "avg":
        return s64 / P, bound / P + 3 * u * np.abs(s64) / P + tiny
    return s64, bound + tiny
