"""Pins for the CPU oracle (oracle/ddl_oracle.py) against things other than itself:
the plain definition (naive rank-by-rank sum), closed forms of rank-indexed
inputs, hand-derived worked examples (tests/golden/worked_examples.json), a brute-force
scalar evaluator of the nested fold formula (no buffers, blocks or phases), library bf16
casts, the Higham error bound, and the SPEC's invariants.

A plausible oracle mistake -- a dropped term, a wrong group member or coordinate, a
transposed fold order, a missing phase-boundary rounding, a misplaced avg multiply, a
wrong block range -- fails at least one of these.  CPU only (no GPU marker).
"""
import json
import math
import os
import struct

import ml_dtypes
import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st, HealthCheck

import oracle
import synthetic_inputs as si

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def factorisations(P, maxlen=4):
    """Every ordered factorisation of P into factors >= 2 (plus [1] for P = 1)."""
    if P == 1:
        return [[1]]
    out = []

    def rec(rem, cur):
        if rem == 1:
            out.append(list(cur))
            return
        if len(cur) >= maxlen:
            return
        for f in range(2, rem + 1):
            if rem % f == 0:
                rec(rem // f, cur + [f])
    rec(P, [])
    return out


def factorisations_with_ones(P):
    """Factorisations of P that contain g_d = 1 (a legal dim whose phase is skipped, SPEC
    S:L266 group_size >= 1; ledger 13): a 1 inserted before, between and after the factors
    of every factorisation, plus all-ones padding for P = 1."""
    if P == 1:
        return [[1], [1, 1], [1, 1, 1]]
    out = []
    for f in factorisations(P, 3):
        for pos in range(len(f) + 1):
            out.append(f[:pos] + [1] + f[pos:])
    out.append([1] + factorisations(P, 3)[0] + [1])
    if P == 8:
        out.append([2, 1, 2, 1, 2])
    return out


def same_bits(a, b):
    """Bitwise equality, except every NaN equals every NaN (ledger 10).  uint16 arrays are
    bf16 bit patterns: NaN when (bits & 0x7FFF) > 0x7F80."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype == np.float32:
        na, nb = np.isnan(a), np.isnan(b)
        return bool(np.array_equal(na, nb) and np.array_equal(a.view(np.uint32)[~na], b.view(np.uint32)[~nb]))
    if a.dtype == np.uint16:
        na, nb = (a & 0x7FFF) > 0x7F80, (b & 0x7FFF) > 0x7F80
        return bool(np.array_equal(na, nb) and np.array_equal(a[~na], b[~nb]))
    return bool(np.array_equal(a, b))


# --------------------------------------------------------------------------- brute force
# An independent scalar evaluator of the nested formula
#   S_{d+1}(c_{d+1..}) = fold_{c_d = 0..g_d-1} S_d(c_d, c_{d+1..})
# (SURVEY.md 8(c) "Fold order"): pure Python numbers, one element at a time, rounding done
# with struct (binary32) and ml_dtypes (bfloat16) instead of numpy array arithmetic.  For
# binary32 + and *, computing in binary64 and rounding once is exact-then-rounded because
# 53 >= 2*24 + 2 (double rounding is innocuous).

def fl32(x: float) -> float:
    """Round a Python float to binary32 (RNE).  struct refuses finite values that round past
    the largest binary32; IEEE says they become +-inf (overflow, ledger 9)."""
    try:
        return struct.unpack("<f", struct.pack("<f", x))[0]
    except OverflowError:
        return math.copysign(math.inf, x)


def flbf16(x: float) -> float:
    return float(ml_dtypes.bfloat16(np.float32(x)))


def brute_element(vals, dims, dtype, op):
    P = len(vals)
    if dtype == "int32":
        level = [int(v) for v in vals]
    elif dtype == "bfloat16":
        level = [float(np.uint32(int(v) << 16).view(np.float32)) for v in vals]
    else:
        level = [float(v) for v in vals]
    live = [d for d, g in enumerate(dims) if g > 1]
    for d, g in enumerate(dims):
        if g == 1:
            continue
        nxt = []
        for i in range(len(level) // g):
            grp = level[i * g:(i + 1) * g]        # ranks sharing coords > d, ascending c_d
            acc = grp[0]
            for v in grp[1:]:
                acc = ((acc + v + 2**31) % 2**32) - 2**31 if dtype == "int32" else fl32(acc + v)
            if op == "avg" and d == live[-1]:
                acc = fl32(acc * fl32(1.0 / P))
            if dtype == "bfloat16":
                acc = flbf16(acc)
            nxt.append(acc)
        level = nxt
    (y,) = level
    if dtype == "int32":
        return np.int32(y)
    if dtype == "bfloat16":
        return ml_dtypes.bfloat16(y).view(np.uint16)
    return np.float32(y)


def brute_allreduce(bufs, dims, dtype, op):
    n = len(bufs[0])
    return np.array([brute_element([b[e] for b in bufs], dims, dtype, op) for e in range(n)],
                    dtype=oracle.ddl_oracle.STORAGE[dtype])


# --------------------------------------------------------------------------- topology / schedule

def test_parse_dims_outer_by_inner():
    assert oracle.parse_dims("2x4") == [4, 2]
    assert oracle.parse_dims("2x2x2") == [2, 2, 2]
    assert oracle.parse_dims("8") == [8]
    assert oracle.parse_dims([4, 2]) == [4, 2]


def test_golden_schedules_and_bad_dims():
    g = json.load(open(GOLDEN))
    for s in g["schedules"]:
        dims = oracle.parse_dims(s["spec"]) if "spec" in s else s["dims"]
        assert dims == s["dims"], s["cite"]
        assert [list(p) for p in oracle.schedule(dims)] == s["expect"], s["cite"]
    for b in g["bad_dims"]:
        with pytest.raises(oracle.BadDims):
            oracle.validate_dims(b["dims"], b["nranks"])


def test_golden_tier_between():
    # tier_between(a, b) = innermost dim whose coordinate differs
    for t in json.load(open(GOLDEN))["tier_between"]:
        dims = t["dims"]
        diff = [d for d in range(len(dims)) if oracle.coord(t["a"], d, dims) != oracle.coord(t["b"], d, dims)]
        assert max(diff) == t["tier"], t["cite"]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8, 12, 16, 24, 32])
def test_coords_mixed_radix_roundtrip(P):
    for dims in factorisations(P):
        G = [math.prod(dims[:d]) for d in range(len(dims))]
        for r in range(P):
            c = [oracle.coord(r, d, dims) for d in range(len(dims))]
            assert sum(ci * Gi for ci, Gi in zip(c, G)) == r          # S:L294 bijection
            for d in range(len(dims)):
                grp = oracle.group(r, d, dims)
                assert len(grp) == dims[d] and r in grp
                assert [oracle.coord(m, d, dims) for m in grp] == list(range(dims[d]))
                for m in grp:   # a group differs from r only in coordinate d
                    assert all(oracle.coord(m, j, dims) == c[j] for j in range(len(dims)) if j != d)


@pytest.mark.parametrize("P", [1, 2, 4, 6, 8, 12])
def test_active_blocks_end_at_own_block(P):
    """After all RS phases rank r owns exactly block r; |A_d| = P / G_d."""
    for dims in factorisations(P):
        k = len(dims)
        for r in range(P):
            assert oracle.active_blocks(r, k, dims) == [r]
            for d in range(k + 1):
                assert len(oracle.active_blocks(r, d, dims)) == P // math.prod(dims[:d])
        # within an RS phase, the blocks a rank writes are disjoint from those its group reads from it
        for d in range(k):
            for r in range(P):
                mine = set(oracle.active_blocks(r, d + 1, dims))
                for m in oracle.group(r, d, dims):
                    if m != r:
                        assert mine.isdisjoint(oracle.active_blocks(m, d + 1, dims))


# --------------------------------------------------------------------------- worked examples

def test_golden_worked_examples():
    for ex in json.load(open(GOLDEN))["examples"]:
        dt = ex["dtype"]
        if dt == "bfloat16":
            bufs = [np.array([int(h, 16) for h in x], dtype=np.uint16) for x in ex["inputs_hex"]]
            want = np.array([int(h, 16) for h in ex["expect_all_ranks_hex"]], dtype=np.uint16)
        else:
            st_ = oracle.ddl_oracle.STORAGE[dt]
            bufs = [np.array(x, dtype=st_) for x in ex["inputs"]]
            want = np.array(ex["expect_all_ranks"], dtype=st_)
        out = oracle.allreduce(bufs, ex["dims"], dt, ex["op"])
        for r, y in enumerate(out):
            assert same_bits(y, want), (ex["name"], ex["cite"], r, y, want)
        # and the brute-force evaluator agrees with the hand derivation too
        assert same_bits(brute_allreduce(bufs, ex["dims"], dt, ex["op"]), want), ex["name"]


# --------------------------------------------------------------------------- int32: exact

@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("kind", ["uniform", "fullrange"])
def test_int32_equals_naive_sum(P, kind):
    n = 1003
    bufs = si.rank_buffers("int32", kind, n, P)
    want = oracle.naive_sum(bufs, "int32")
    for dims in factorisations(P):
        out = oracle.allreduce(bufs, dims, "int32")
        for y in out:
            assert np.array_equal(y, want), dims


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_int32_bitmask_closed_form(P):
    n = (1 << 20) + 37      # wraps the (i mod 2^20) field once
    bufs = si.rank_buffers("int32", "bitmask", n, P)
    i = np.arange(n, dtype=np.int64)
    want = (((1 << P) - 1) + P * ((i % (1 << 20)) << 8)) & 0xFFFFFFFF
    want = want.astype(np.uint32).view(np.int32)
    for dims in factorisations(P):
        for y in oracle.allreduce(bufs, dims, "int32"):
            assert np.array_equal(y, want), dims


def test_int32_wrap():
    bufs = [np.full(5, 1 << 30, dtype=np.int32) for _ in range(4)]
    for dims in ([4], [2, 2]):
        for y in oracle.allreduce(bufs, dims, "int32"):
            assert np.all(y == 0)


def test_int32_avg_rejected():
    with pytest.raises(oracle.Unsupported):
        oracle.allreduce([np.zeros(4, np.int32)] * 2, [2], "int32", "avg")


# --------------------------------------------------------------------------- fp32

@pytest.mark.parametrize("P", [2, 3, 4, 6, 8])
def test_fp32_intvalued_exact(P):
    bufs = si.rank_buffers("float32", "intvalued", 777, P)
    s64, _ = oracle.exact_sum_f64(bufs, "float32")
    for dims in factorisations(P):
        for y in oracle.allreduce(bufs, dims, "float32"):
            assert np.array_equal(y.astype(np.float64), s64), dims


@pytest.mark.parametrize("P", [1, 2, 4, 8, 16])
def test_fp32_rankplus1_closed_form(P):
    bufs = si.rank_buffers("float32", "rankplus1", 100, P)
    for dims in factorisations(P):
        assert np.all(oracle.allreduce(bufs, dims, "float32")[P - 1] == P * (P + 1) / 2)
        assert np.all(oracle.allreduce(bufs, dims, "float32", "avg")[0] == (P + 1) / 2)


@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_fp32_flat_dims_is_recursive_summation(P):
    """dims = [P] is textbook recursive summation in ascending rank: bitwise equal to a
    plain float32 left fold (the naive definition)."""
    bufs = si.rank_buffers("float32", "normal", 4099, P)
    want = oracle.naive_sum(bufs, "float32")
    acc = bufs[0].copy()
    for x in bufs[1:]:
        acc = (acc + x).astype(np.float32)
    assert np.array_equal(want, acc)
    for y in oracle.allreduce(bufs, [P], "float32"):
        assert same_bits(y, want)


@pytest.mark.parametrize("P", [2, 4, 8, 16])
def test_fp32_higham_bound(P):
    """|y - s| <= gamma_{P-1} * sum_r |x_r| for any summation order (Higham, recursive
    summation / any tree), gamma_m = m u / (1 - m u), u = 2^-24."""
    bufs = si.rank_buffers("float32", "normal", 20000, P)
    s64, a64 = oracle.exact_sum_f64(bufs, "float32")
    u = 2.0 ** -24
    gam = (P - 1) * u / (1 - (P - 1) * u)
    for dims in factorisations(P):
        y = oracle.allreduce(bufs, dims, "float32")[0].astype(np.float64)
        assert np.all(np.abs(y - s64) <= gam * a64 + 1e-45), dims
        assert np.max(np.abs(y - s64) / a64) < 1e-6       # north_star fp32 tolerance (ledger 8)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_avg_power_of_two_equals_sum_then_scale(P):
    """For P = 2^m, x * 2^-m is exact: fused avg == SPEC's sum-then-scale."""
    bufs = si.rank_buffers("float32", "normal", 3001, P)
    for dims in factorisations(P):
        s = oracle.allreduce(bufs, dims, "float32", "sum")[0]
        a = oracle.allreduce(bufs, dims, "float32", "avg")[0]
        assert np.array_equal(a, (s * np.float32(1.0 / P)).astype(np.float32))
        assert np.array_equal(a, (s / np.float32(P)).astype(np.float32))


# --------------------------------------------------------------------------- bf16

def test_bf16_round_matches_libraries():
    specials = np.array([0.0, -0.0, 1.0, -1.0, 1 + 2**-8, 1 + 3 * 2**-8, 1 + 2**-7 + 2**-8,
                         np.finfo(np.float32).max, -np.finfo(np.float32).max, 3.3895e38, 3.4e38,
                         np.inf, -np.inf, 1e-40, -1e-40, 2**-133, 1.17549435e-38, 65504.0,
                         np.float32(1.00390625), 255.5, 256.5], dtype=np.float32)
    rnd = np.random.Generator(np.random.PCG64(7))
    bits = rnd.integers(0, 1 << 32, size=200000, dtype=np.uint32)
    bits = bits[((bits >> 23) & 0xFF) != 0xFF]                       # finite patterns
    x = np.concatenate([specials, bits.view(np.float32), rnd.standard_normal(50000).astype(np.float32)])
    mine = oracle.bf16_round(x)
    ml = x.astype(ml_dtypes.bfloat16).view(np.uint16)
    th = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, ml)
    assert np.array_equal(mine, th)
    nan_in = np.array([np.nan, -np.nan, np.uint32(0x7F800001).view(np.float32)], dtype=np.float32)
    assert np.all(np.isnan(oracle.bf16_to_f32(oracle.bf16_round(nan_in))))
    back = oracle.bf16_to_f32(mine)
    assert np.array_equal(back, ml.view(ml_dtypes.bfloat16).astype(np.float32), equal_nan=True)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_bf16_error_bound(P):
    """Each phase boundary rounds to bf16 (relative 2^-8 of a partial bounded by sum|x|):
    |y - s| <= (k * 2^-8 + (P-1) * 2^-24 * (1 + 2^-8)^k) * sum|x| + tiny."""
    bufs = si.rank_buffers("bfloat16", "normal", 50000, P)
    s64, a64 = oracle.exact_sum_f64(bufs, "bfloat16")
    for dims in factorisations(P):
        k = len(dims)
        y = oracle.bf16_to_f32(oracle.allreduce(bufs, dims, "bfloat16")[0]).astype(np.float64)
        bound = (k * 2.0**-8 + (P - 1) * 2.0**-24 * (1 + 2.0**-8) ** k) * (1 + 2.0**-8) ** k
        assert np.all(np.abs(y - s64) <= bound * a64 + 1e-38), dims
        # north_star: "bf16 within 1e-2" -- exactly 1e-2, every factorisation (ledger 7/8)
        assert np.max(np.abs(y - s64) / np.maximum(a64, 1e-30)) <= 1e-2, dims


# --------------------------------------------------------------------------- brute-force nested fold

@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("dtype,kind", [("float32", "normal"), ("bfloat16", "normal"), ("int32", "fullrange")])
def test_nested_formula_brute_force(P, dtype, kind):
    n = 37     # spans several blocks and a ragged tail for every P here
    bufs = si.rank_buffers(dtype, kind, n, P)
    for dims in factorisations(P):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            want = brute_allreduce(bufs, dims, dtype, op)
            out = oracle.allreduce(bufs, dims, dtype, op)
            for y in out:
                assert same_bits(y, want), (dims, op)


def test_nested_formula_brute_force_32_ranks():
    for P, dims in [(32, [2, 4, 4]), (32, [8, 4]), (24, [3, 2, 4]), (16, [2, 2, 2, 2])]:
        bufs = si.rank_buffers("float32", "normal", 19, P)
        assert same_bits(oracle.allreduce(bufs, dims, "float32", "avg")[P - 1],
                         brute_allreduce(bufs, dims, "float32", "avg"))
        bb = si.rank_buffers("bfloat16", "normal", 19, P)
        assert same_bits(oracle.allreduce(bb, dims, "bfloat16")[3], brute_allreduce(bb, dims, "bfloat16", "sum"))


@settings(max_examples=500, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(1, 32).flatmap(lambda P: st.tuples(st.just(P), st.sampled_from(factorisations(P, 5)))),
       st.integers(0, 300), st.integers(0, 2**31 - 1))
def test_property_spec_acceptance_5(Pdims, n, seed):
    """random (topology, buffer) instances up to 32 ranks, integer-valued:
    hierarchical == brute-force sum == flat (dims [P]) result."""
    P, dims = Pdims
    bufs = si.rank_buffers("float32", "intvalued", n, P, seed=seed)
    s64, _ = oracle.exact_sum_f64(bufs, "float32")
    h = oracle.allreduce(bufs, dims, "float32")
    f = oracle.allreduce(bufs, [P], "float32")
    for y in h:
        assert np.array_equal(y.astype(np.float64), s64)
    assert np.array_equal(h[0], f[P - 1])


@pytest.mark.parametrize("P", [1, 2, 4, 6, 8])
@pytest.mark.parametrize("dtype,kind", [("float32", "normal"), ("bfloat16", "normal"), ("int32", "fullrange")])
def test_dims_with_unit_factors_brute_force(P, dtype, kind):
    """g_d = 1 dims (SPEC S:L266 group_size >= 1, "1x1 -> empty phase list"; ledger
    13): the oracle on [4,1,2], [1,8], [8,1], [2,1,2,1,2], ... equals the brute-force nested
    fold (which skips a size-1 level), element by element; P = 1 is the identity
    (S:L335)."""
    n = 37
    bufs = si.rank_buffers(dtype, kind, n, P)
    for dims in factorisations_with_ones(P):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            want = brute_allreduce(bufs, dims, dtype, op)
            out = oracle.allreduce(bufs, dims, dtype, op)
            for y in out:
                assert same_bits(y, want), (dims, op)
            if P == 1:
                assert same_bits(out[0], bufs[0]), (dims, op)      # identity, avg scales by 1
            assert len(oracle.schedule(dims)) == 2 * sum(1 for g in dims if g > 1)


def test_unit_dims_schedule_golden():
    """a 1x1 topology has an empty phase list; a g = 1 dim contributes no phase."""
    assert oracle.schedule([1, 1]) == []
    assert oracle.schedule([1]) == []
    assert oracle.schedule([4, 1, 2]) == [("RS", 0), ("RS", 2), ("AG", 2), ("AG", 0)]
    assert oracle.schedule([1, 8]) == [("RS", 1), ("AG", 1)]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_ieee_specials_brute_force(P, dtype):
    """IEEE special values (ledger 9/10): +-0, subnormals (no FTZ/DAZ), +-max, pairwise
    overflow to +-inf, inf - inf = NaN, NaN propagation.  The oracle equals the brute-force
    scalar fold (Python binary64 arithmetic rounded to binary32 by struct -- overflow to
    inf -- and to bf16 by ml_dtypes) for every factorisation, sum and avg."""
    n = 600
    bufs = si.rank_buffers(dtype, "specials", n, P)
    # columns where every rank holds a subnormal or a signed zero (random draws rarely line
    # up across P ranks): chosen bit patterns, no arithmetic
    if dtype == "float32":
        sub = np.array([0x00000001, 0x80000001, 0x007FFFFF, 0x00000003], dtype=np.uint32)
        zero = np.array([0x80000000, 0x80000000, 0x00000000], dtype=np.uint32)
        view = np.uint32
    else:
        sub = np.array([0x0001, 0x8001, 0x007F, 0x0003], dtype=np.uint16)
        zero = np.array([0x8000, 0x8000, 0x0000], dtype=np.uint16)
        view = np.uint16
    for r in range(P):
        v = bufs[r].view(view)
        for c in range(16):
            v[c] = sub[(r + c) % len(sub)] if c < 12 else sub[0]
        for c in range(16, 24):
            v[c] = zero[0] if c < 20 else zero[(r + c) % len(zero)]
    got_any = {"nan": False, "inf": False, "negzero": False, "sub": False}
    for dims in factorisations(P) + ([[4, 1, 2]] if P == 8 else []):
        for op in ("sum", "avg"):
            want = brute_allreduce(bufs, dims, dtype, op)
            out = oracle.allreduce(bufs, dims, dtype, op)
            assert same_bits(out[P - 1], want), (dims, op)
            f = oracle.bf16_to_f32(want) if dtype == "bfloat16" else want
            got_any["nan"] |= bool(np.isnan(f).any())
            got_any["inf"] |= bool(np.isinf(f).any())
            got_any["negzero"] |= bool(((f == 0) & np.signbit(f)).any())
            got_any["sub"] |= bool(((f != 0) & (np.abs(f) < np.float32(1.1754944e-38))).any())
    assert all(got_any.values()), got_any      # the inputs really exercise every special


def test_ieee_specials_closed_forms():
    """Hand-derived special cases, fp32 and bf16, P = 2 and 4: overflow of two finite
    values, signed zeros (+0 + -0 = +0; -0 + -0 = -0), a subnormal sum kept (no FTZ),
    inf + (-inf) = NaN, NaN absorbs inf."""
    mx = np.float32(3.4028235e38)
    tiny = np.uint32(1).view(np.float32)      # smallest subnormal, 1 ulp
    cases = [  # (per-rank values, expected sum)
        ([mx, mx], np.float32(np.inf)),
        ([-mx, -mx], np.float32(-np.inf)),
        ([np.float32(0.0), np.float32(-0.0)], np.float32(0.0)),
        ([np.float32(-0.0), np.float32(-0.0)], np.float32(-0.0)),
        ([tiny, tiny], np.uint32(2).view(np.float32)),      # 1 ulp + 1 ulp = 2 ulp (no FTZ)
        ([np.float32(np.inf), np.float32(-np.inf)], np.float32(np.nan)),
        ([np.float32(np.nan), np.float32(np.inf), np.float32(1), np.float32(2)], np.float32(np.nan)),
        ([mx, mx, -mx, -mx], np.float32(np.nan)),     # (mx+mx) + (-mx-mx) = inf - inf ([2,2])
    ]
    for vals, want in cases:
        P = len(vals)
        bufs = [np.array([v], dtype=np.float32) for v in vals]
        dims = [2] if P == 2 else [2, 2]
        y = oracle.allreduce(bufs, dims, "float32", "sum")[0]
        assert same_bits(y, np.array([want], dtype=np.float32)), (vals, y, want)
        bb = [oracle.bf16_round(b) for b in bufs]      # every value above is bf16-exact
        yb = oracle.allreduce(bb, dims, "bfloat16", "sum")[0]
        assert same_bits(yb, oracle.bf16_round(np.array([want], dtype=np.float32))), (vals, yb)
    # [4] folds ((mx + mx) - mx) - mx = (inf - mx) - mx = inf: the order matters
    y = oracle.allreduce([np.array([v], dtype=np.float32) for v in (mx, mx, -mx, -mx)], [4], "float32")[0]
    assert y[0] == np.inf
    # avg of subnormals: (1 ulp + 2 ulp) * fl32(1/2) = 1.5 ulp -> RNE to 2 ulp (ties to even);
    # a flush-to-zero implementation would give 0
    one, two = np.uint32(1).view(np.float32), np.uint32(2).view(np.float32)
    y = oracle.allreduce([np.array([one], dtype=np.float32), np.array([two], dtype=np.float32)], [2],
                         "float32", "avg")[0]
    assert y.view(np.uint32)[0] == 2


# --------------------------------------------------------------------------- invariants

@pytest.mark.parametrize("P,n", [(4, 1_000_003), (8, 5), (8, 7), (8, 1), (3, 2), (4, 0)])
def test_ragged_and_degenerate(P, n):
    """S:L369 padding transparency: output length = input length; n < P leaves empty blocks."""
    bufs = si.rank_buffers("int32", "uniform", n, P)
    want = oracle.naive_sum(bufs, "int32")
    for dims in factorisations(P)[:3]:
        out = oracle.allreduce(bufs, dims, "int32")
        assert all(len(y) == n for y in out)
        assert all(np.array_equal(y, want) for y in out)


@pytest.mark.parametrize("dtype,kind", [("float32", "normal"), ("bfloat16", "normal")])
def test_replicas_identical_and_deterministic(dtype, kind):
    """S:L441 replica consistency; S:L368 order-fixity (two runs bitwise identical)."""
    P = 8
    bufs = si.rank_buffers(dtype, kind, 2053, P)
    for dims in factorisations(P):
        a = oracle.allreduce(bufs, dims, dtype, "avg")
        b = oracle.allreduce(bufs, dims, dtype, "avg")
        for r in range(P):
            assert same_bits(a[r], a[0]) and same_bits(a[r], b[r])


@pytest.mark.parametrize("P", [2, 4, 8])
def test_reduce_scatter_allgather_compose(P):
    """allgather(reduce_scatter(x)) == allreduce(x); RS slice r == allreduce block r."""
    q = 96                                   # a multiple of the 16-B vector -> same layout
    for dtype, kind in [("float32", "normal"), ("bfloat16", "normal"), ("int32", "fullrange")]:
        bufs = si.rank_buffers(dtype, kind, P * q, P)
        for dims in factorisations(P):
            ops = ["sum"] if dtype == "int32" else ["sum", "avg"]
            for op in ops:
                ar = oracle.allreduce(bufs, dims, dtype, op)
                rs = oracle.reduce_scatter(bufs, dims, dtype, op)
                for r in range(P):
                    assert same_bits(rs[r], ar[r][r * q:(r + 1) * q])
                ag = oracle.allgather(rs, dims, dtype)
                for r in range(P):
                    assert same_bits(ag[r], ar[r])


def test_allgather_is_concatenation():
    P = 8
    sends = [np.arange(10, dtype=np.int32) + 100 * r for r in range(P)]
    for dims in factorisations(P):
        for y in oracle.allgather(sends, dims, "int32"):
            assert np.array_equal(y, np.concatenate(sends))


def test_int32_dims_permutation_invariant():
    P = 8
    bufs = si.rank_buffers("int32", "fullrange", 999, P)
    res = {tuple(d): oracle.allreduce(bufs, d, "int32")[0] for d in factorisations(P)}
    first = next(iter(res.values()))
    assert all(np.array_equal(v, first) for v in res.values())


def test_sampled_equals_full():
    P = 8
    n = 5000
    rnd = np.random.Generator(np.random.PCG64(3))
    idx = np.sort(rnd.choice(n, 300, replace=False))
    for dtype in ("float32", "bfloat16"):
        bufs = si.rank_buffers(dtype, "normal", n, P)
        for dims in ([4, 2], [2, 2, 2], [8]):
            full = oracle.allreduce(bufs, dims, dtype, "avg")[5]
            assert same_bits(oracle.allreduce_sampled(bufs, dims, dtype, "avg", idx), full[idx])


# --------------------------------------------------------------------------- traffic

@pytest.mark.parametrize("P", [2, 4, 8])
def test_traffic_conservation(P):
    n = P * 64
    S = n * 4
    for dims in factorisations(P):
        t = oracle.Traffic.new(P)
        oracle.allreduce(si.rank_buffers("float32", "normal", n, P), dims, "float32", traffic=t)
        for r in range(P):
            assert sum(t.remote_read[r].values()) == 2 * (P - 1) * S // P
            for d, g in enumerate(dims):
                active = S // math.prod(dims[:d])
                assert t.remote_read[r][("RS", d)] == (g - 1) * active // g
                assert t.remote_read[r][("AG", d)] == (g - 1) * active // g


# --------------------------------------------------------------------------- K5 local reduce

def test_local_reduce():
    ins = si.rank_buffers("int32", "fullrange", 1000, 8)
    assert np.array_equal(oracle.local_reduce(ins, "int32"), oracle.naive_sum(ins, "int32"))
    f = si.rank_buffers("float32", "normal", 1000, 5)
    assert np.array_equal(oracle.local_reduce(f, "float32"), oracle.naive_sum(f, "float32"))
    iv = si.rank_buffers("float32", "intvalued", 1000, 4)
    s64, _ = oracle.exact_sum_f64(iv, "float32")
    assert np.array_equal(oracle.local_reduce(iv, "float32", 0.25).astype(np.float64), s64 / 4)
    b = si.rank_buffers("bfloat16", "normal", 1000, 4)
    want = oracle.bf16_round(oracle.naive_sum(b, "bfloat16"))
    assert np.array_equal(oracle.local_reduce(b, "bfloat16"), want)


# --------------------------------------------------------------------------- NVLS phases (NEXT-1)

def _exact_fraction_sum(vals):
    from fractions import Fraction
    return sum((Fraction(float(v)) for v in vals), Fraction(0))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_nvls_int32_exact(P):
    """int32 NVLS phases: every fold order reaches the exact sum mod 2^32 (bit-exact pin)."""
    bufs = si.rank_buffers("int32", "fullrange", 777, P)
    want = oracle.naive_sum(bufs, "int32")
    for dims in factorisations(P):
        live = [d for d, g in enumerate(dims) if g > 1]
        for nv in ([], live, live[:1]):
            out = oracle.allreduce(bufs, dims, "int32", "sum", nvls_dims=nv)
            assert all(np.array_equal(y, want) for y in out), (dims, nv)


def test_nvls_switch_sum_correctly_rounded_flat():
    """dims [P] with its one phase in the switch: the oracle's admissible result is the
    exact sum rounded once to binary32 -- checked with exact rational arithmetic
    (fractions) on every element: |y - s| <= 2^-24 |s| (half an ulp)."""
    P = 8
    bufs = si.rank_buffers("float32", "normal", 400, P)
    y = oracle.allreduce(bufs, [P], "float32", "sum", nvls_dims=[0])[0]
    for e in range(400):
        s = _exact_fraction_sum([b[e] for b in bufs])
        assert abs(float(y[e]) - float(s)) <= 2.0 ** -24 * abs(float(s)) * (1 + 1e-9), e


def test_nvls_two_member_phases_equal_direct():
    """A 2-member phase has only one fold (a + b == b + a exactly, rounded once), so an NVLS
    [2, 2, 2] all-reduce equals the direct one bit for bit (fp32 sum and avg)."""
    bufs = si.rank_buffers("float32", "normal", 1000, 8)
    for op in ("sum", "avg"):
        a = oracle.allreduce(bufs, [2, 2, 2], "float32", op)
        b = oracle.allreduce(bufs, [2, 2, 2], "float32", op, nvls_dims=[0, 1, 2])
        assert all(same_bits(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
@pytest.mark.parametrize("P", [2, 4, 8, 16])
def test_fold_error_bound_holds_for_every_order(dtype, P):
    """fold_error_bound is a valid bound for the direct order, the switch order on any subset
    of dims, and a brute-force fold in REVERSED member order (another admissible tree); and it
    is not vacuous: fp32 stays below north_star's 1e-6 componentwise gate for P <= 16."""
    bufs = si.rank_buffers(dtype, "normal", 3000, P)
    for dims in factorisations(P):
        for op in ("sum", "avg"):
            s, bound = oracle.fold_error_bound(bufs, dims, dtype, op)
            live = [d for d, g in enumerate(dims) if g > 1]
            for nv in ([], live, live[-1:]):
                y = oracle.allreduce(bufs, dims, dtype, op, nvls_dims=nv)[0]
                yf = oracle.bf16_to_f32(y) if dtype == "bfloat16" else y
                assert np.all(np.abs(yf.astype(np.float64) - s) <= bound), (dims, op, nv)
            rev = oracle.allreduce(bufs[::-1], dims, dtype, op)[0]
            rf = oracle.bf16_to_f32(rev) if dtype == "bfloat16" else rev
            assert np.all(np.abs(rf.astype(np.float64) - s) <= bound), (dims, op, "reversed")
            _, a64 = oracle.exact_sum_f64(bufs, dtype)
            if dtype == "float32" and (op == "sum" or P <= 8):   # avg adds 3u|s|/P for the multiply
                mag = a64 / P if op == "avg" else a64
                assert np.all(bound <= 1e-6 * mag + 1e-30)
