"""C ABI: the library loads on a CPU-only box, exports every symbol declared
in include/adct_cuda.h, the ctypes prototypes match the header, and the
host-side logic (quantiser tables, argument validation) behaves.  No CUDA
compute is called here."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import exact
from paper_1702_00817_b200 import _lib, errors, quant

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "adct_cuda.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return re.findall(r"^[a-z_0-9 ]+?\**\s*\b(adct_[a-z0-9_]+)\s*\(", src, flags=re.M)


def test_library_loads_and_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), n
    # and the dynamic symbol table really has them (not just ctypes lookup)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_prototypes_cover_header_exactly():
    assert set(header_functions()) == set(_lib.PROTOTYPES)


def test_struct_sizes_match_header():
    # adct_qtab_t: 10 x 64 int32 + 4 int32 + 64 uint32 (recip_f); adct_plane_t: 2 ptr + 2 int32 + 2 int64
    assert ctypes.sizeof(_lib.QTab) == (11 * 64 + 4) * 4
    assert ctypes.sizeof(_lib.Plane) == 8 + 8 + 4 + 4 + 8 + 8


def test_no_nccl_or_torch_linked():
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "nccl" not in out and "torch" not in out


def test_version_and_strerror():
    L = _lib.lib()
    assert L.adct_version() >= 10000
    assert L.adct_strerror(2).decode() == "retention count must be in [1, 64]"
    assert L.adct_strerror(999).decode() == "unknown error"


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("q", [1, 5, 10, 25, 30, 50, 75, 90, 95, 100])
def test_qtab_from_quality_matches_oracle(q):
    t = quant.quant_table(q)
    assert np.array_equal(quant.qtab_qprime(t), exact.qprime(quant.q50_luma(), q))
    assert np.array_equal(quant.qtab_qprime(t), quant.qprime_for_quality(q))
    qe = np.frombuffer(bytes(t.qe), dtype=np.int32).reshape(8, 8)
    assert np.array_equal(qe, quant.qtab_qprime(t) * exact.E)
    assert t.quality == q


def test_qtab_range_flags():
    # q >= 25 tables are exact in 16-bit lanes; coarse ones need the 32-bit kernel
    assert quant.quant_table(10).wide == 1 and quant.quant_table(25).wide == 0
    assert quant.quant_table(75).aligned == 1 and quant.quant_table(25).aligned == 0
    t = quant.quant_table(75)
    # bound: 8192 + max_ij sum_uv |T_ui T_vj| E_uv Q'_uv / 2
    qe = quant.qtab_qprime(t) * exact.E
    absT = np.abs(exact.T)
    b = 8192 + max((absT[:, i][:, None] * absT[:, j][None, :] * qe).sum() / 2 for i in range(8) for j in range(8))
    assert t.max_abs_v == int(np.ceil(b))


def test_qtab_quantiser_constants_are_exact():
    """Replay the device formulas in numpy over every reachable coefficient."""
    for q in (25, 50, 75, 90, 100):
        t = quant.quant_table(q)
        Qp = quant.qtab_qprime(t).reshape(64)
        Z = np.arange(-8192, 8193, dtype=np.int64)
        want = np.sign(Z)[None, :] * ((2 * np.abs(Z)[None, :] + Qp[:, None]) // (2 * Qp[:, None]))
        mag = np.frombuffer(bytes(t.magic), dtype=np.uint32).astype(np.uint64)
        bias = np.frombuffer(bytes(t.bias), dtype=np.int32).astype(np.int64)
        mult = np.frombuffer(bytes(t.mult), dtype=np.int32).astype(np.int64)
        kq = np.frombuffer(bytes(t.kq), dtype=np.int32).astype(np.int64)
        U = (Z[None, :] + bias[:, None]) * mult[:, None] + (Z >= 0)[None, :]
        assert U.min() >= 0 and U.max() <= 0xFFFF
        got = ((U.astype(np.uint64) * mag[:, None]) >> np.uint64(32)).astype(np.int64) - kq[:, None]
        assert np.array_equal(got, want), q


def test_qtab_scalar_quantiser_constants_are_exact():
    """The wide (one block per thread) quantiser's constants over the whole
    supported Q' range (1 .. 2^20): multiply-high alone, no post-shift."""
    rng = np.random.default_rng(3)
    tables = [quant.quant_table(q) for q in (1, 10, 24)]
    tables.append(quant.quant_table(qprime_unrounded=rng.choice(
        [1.0, 3.0, 40000.0, 65536.0, 300001.0, 1048576.0], size=(8, 8))))
    # Q' across the whole supported range, incl. near powers of two
    grid = np.unique(np.concatenate([np.geomspace(1, 2**20, 40).round(), 2.0 ** np.arange(21),
                                     2.0 ** np.arange(1, 21) - 1, 2.0 ** np.arange(1, 21) + 1]))
    grid = grid[grid <= 2**20]
    for k in range(0, len(grid), 64):
        chunk = np.resize(grid[k:k + 64], 64)
        tables.append(quant.quant_table(qprime_unrounded=chunk.reshape(8, 8)))
    Z = np.arange(-8192, 8193, dtype=np.int64)
    for t in tables:
        Qp = quant.qtab_qprime(t).reshape(64)
        want = np.sign(Z)[None, :] * ((2 * np.abs(Z)[None, :] + Qp[:, None]) // (2 * Qp[:, None]))
        mag = np.frombuffer(bytes(t.magic_w), dtype=np.uint32).astype(np.uint64)
        cadd = np.frombuffer(bytes(t.cadd_w), dtype=np.int32).astype(np.int64)
        kw = np.frombuffer(bytes(t.kw), dtype=np.int32).astype(np.int64)
        assert not np.frombuffer(bytes(t.shift_w), dtype=np.int32).any()
        U = (2 * Z - (Z < 0))[None, :] + cadd[:, None]
        assert U.min() >= 0 and U.max() < 2**32
        got = ((U.astype(np.uint64) * mag[:, None]) >> np.uint64(32)).astype(np.int64) - kw[:, None]
        assert np.array_equal(got, want)


def _float_quantiser_replay(t):
    """RN(M + Z r) - M for every |Z| <= 8192 and position, in exact integer
    arithmetic (what the device FFMA2 computes: exact product, one rounding to
    the ulp-1 grid of [2^23, 2^24), ties to even; M = 1.5 * 2^23 is even)."""
    bits = np.frombuffer(bytes(t.recip_f), dtype=np.uint32)
    r = bits.view(np.float32).astype(np.float64)
    mant, e = np.frexp(r)  # r = mant * 2^e, mant in [0.5, 1)
    m24 = np.ldexp(mant, 24).astype(np.int64)  # exact 24-bit integer
    sh = (24 - e).astype(np.int64)
    Z = np.arange(-8192, 8193, dtype=np.int64)
    num = Z[None, :] * m24[:, None]
    fl = num >> sh[:, None]
    rem = num - (fl << sh[:, None])
    half = np.left_shift(np.int64(1), sh - 1)[:, None]
    return fl + ((rem > half) | ((rem == half) & (fl & 1 == 1))), Z


def test_qtab_float_quantiser_is_exact():
    """The float quantiser constants (recip_f, the default device path) give
    round-half-away-from-zero of Z / Q' for every reachable Z, across quality
    tables and explicit Q' over the whole supported range."""
    rng = np.random.default_rng(5)
    tables = [quant.quant_table(q) for q in (1, 5, 10, 25, 50, 75, 90, 100)]
    grid = np.unique(np.concatenate([np.arange(1, 600), np.geomspace(600, 2**20, 60).round(),
                                     2.0 ** np.arange(21), 2.0 ** np.arange(1, 21) + 1, 3 * 2.0 ** np.arange(19),
                                     rng.integers(1, 20000, 256)]))
    grid = grid[grid <= 2**20]
    for k in range(0, len(grid), 64):
        chunk = np.resize(grid[k:k + 64], 64).astype(np.float64)
        tables.append(quant.quant_table(qprime_unrounded=chunk.reshape(8, 8)))
    for t in tables:
        got, Z = _float_quantiser_replay(t)
        Qp = quant.qtab_qprime(t).reshape(64)
        want = np.sign(Z)[None, :] * ((2 * np.abs(Z)[None, :] + Qp[:, None]) // (2 * Qp[:, None]))
        assert np.array_equal(got, want)
        # r is within 2^-13 relative of 1/Q' (the exhaustive replay above is the property)
        r = np.frombuffer(bytes(t.recip_f), dtype=np.uint32).view(np.float32).astype(np.float64)
        assert np.all(np.abs(r * Qp - 1.0) < 2.0 ** -13)


def test_qtab_build_from_fold_and_errors():
    from paper_1702_00817_b200 import transforms

    tr = transforms.proposed_transform()
    qpu = quant.fold_scaling_into_quantization(tr, quant.q50_luma() * 0.5)
    t = quant.quant_table(qprime_unrounded=qpu)
    assert np.array_equal(quant.qtab_qprime(t), quant.qtab_qprime(quant.quant_table(75)))
    assert t.quality == -1
    bad = qpu.copy()
    bad[3, 3] = 0.0
    with pytest.raises(errors.NonPositiveQuantizer):
        quant.quant_table(qprime_unrounded=bad)
    with pytest.raises(errors.NonPositiveQuantizer):
        quant.fold_scaling_into_quantization(tr, -np.ones((8, 8)))
    with pytest.raises(errors.BadDimensions):
        quant.fold_scaling_into_quantization(tr, np.ones((4, 4)))
    with pytest.raises(ValueError):
        quant.quant_table(0)


def test_entry_points_validate_before_any_cuda_call():
    """Contract errors come back before anything touches the device, so they
    work on a CPU-only box with null pointers."""
    L = _lib.lib()
    n = ctypes.c_void_p(0)
    assert L.adct_compress_retain(n, n, 1, 64, 64, 4096, 4096, 0, n, n, n) == 2  # InvalidRetention
    assert L.adct_compress_retain(n, n, 1, 64, 64, 4096, 4096, 65, n, n, n) == 2
    assert L.adct_compress_retain(n, n, 1, 60, 64, 4096, 4096, 10, n, n, n) == 1  # BadDimensions
    assert L.adct_compress_retain(n, n, -1, 64, 64, 4096, 4096, 10, n, n, n) == 5
    assert L.adct_forward_int32(n, 1, 64, 63, 4096, 0, n, n) == 1
    assert L.adct_sweep_retain_sse(n, 1, 64, 64, 4096, 5, 4, n, n, n) == 2
    cm = (ctypes.c_double * 64)()
    assert L.adct_sweep_dense(n, 0, 1, 64, 64, cm, 0, 5, n, n) == 2
    assert L.adct_forward_dense(n, 0, 1, 64, 60, cm, n, n) == 1
    assert L.adct_inverse_f64(n, 1, 64, 64, 0, 1, n, n) == 2
    # zero images: nothing to do, no device access
    assert L.adct_compress_retain(n, n, 0, 64, 64, 4096, 4096, 10, n, n, n) == 0
    qt = quant.quant_table(50)
    assert L.adct_compress_quant(n, n, 1, 64, 12, 768, 768, ctypes.byref(qt), n, n) == 1
    bad = _lib.QTab()
    assert L.adct_compress_quant(n, n, 1, 64, 64, 4096, 4096, ctypes.byref(bad), n, n) == 3
    planes = (_lib.Plane * 4)()
    assert L.adct_compress_quant_planes(planes, 4, 1, ctypes.byref(qt), n, n) == 5
    # fused SSE exchange: missing accumulator / peers / counters, bad peer count or offset
    p8 = ctypes.c_void_p(0x1000)
    X = L.adct_compress_retain_exchange
    assert X(n, n, 1, 64, 64, 4096, 4096, 10, n, p8, 1, 0, p8, n) == 5
    assert X(n, n, 1, 64, 64, 4096, 4096, 10, p8, n, 1, 0, p8, n) == 5
    assert X(n, n, 1, 64, 64, 4096, 4096, 10, p8, p8, 1, 0, n, n) == 5
    assert X(n, n, 1, 64, 64, 4096, 4096, 10, p8, p8, 0, 0, p8, n) == 5
    assert X(n, n, 1, 64, 64, 4096, 4096, 10, p8, p8, 1, -1, p8, n) == 5
    assert X(n, n, 1, 64, 64, 4096, 4096, 10, ctypes.c_void_p(0x1004), p8, 1, 0, p8, n) == 6
    assert X(n, n, 1, 64, 64, 4096, 4096, 0, p8, p8, 1, 0, p8, n) == 2
    assert X(n, n, 0, 64, 64, 4096, 4096, 10, p8, p8, 1, 0, p8, n) == 0
    assert X(n, n, 0, 64, 64, 4096, 4096, 10, n, n, 1, 0, n, n) == 0  # empty call: nothing touched
    assert L.adct_compress_retain(n, n, 2**31, 8, 8, 64, 64, 10, n, n, n) == 5  # > 2^31 frames


def test_error_mapping():
    with pytest.raises(errors.InvalidRetention):
        _lib.check(2)
    with pytest.raises(errors.BadDimensions):
        _lib.check(1)
    with pytest.raises(errors.NonPositiveQuantizer):
        _lib.check(3)
    with pytest.raises(RuntimeError):
        _lib.check(7)


def test_qtab_random_tables_replay_exactly():
    """Seeded random Q' tables over the supported range (1 .. 2^20, halves
    included to exercise the rounding): the builder either reports the table
    as packed-capable and the two-lane constants replay exactly, or marks it
    wide; the scalar constants always replay exactly."""
    rng = np.random.default_rng(7)
    Z = np.arange(-8192, 8193, dtype=np.int64)
    for _ in range(12):
        scale = 10.0 ** rng.uniform(0, 6.3, size=(8, 8))
        qpu = np.where(rng.random((8, 8)) < 0.2, np.floor(scale) + 0.5, scale)
        qpu = np.minimum(qpu, 2.0**20)
        t = quant.quant_table(qprime_unrounded=qpu)
        Qp = quant.qtab_qprime(t).reshape(64)
        assert (Qp == np.maximum(1, np.floor(qpu.reshape(64) + 0.5))).all()
        want = np.sign(Z)[None, :] * ((2 * np.abs(Z)[None, :] + Qp[:, None]) // (2 * Qp[:, None]))
        mag_w = np.frombuffer(bytes(t.magic_w), dtype=np.uint32).astype(np.uint64)
        cadd = np.frombuffer(bytes(t.cadd_w), dtype=np.int32).astype(np.int64)
        kw = np.frombuffer(bytes(t.kw), dtype=np.int32).astype(np.int64)
        U = (2 * Z - (Z < 0))[None, :] + cadd[:, None]
        got = ((U.astype(np.uint64) * mag_w[:, None]) >> np.uint64(32)).astype(np.int64) - kw[:, None]
        assert np.array_equal(got, want)
        mult = np.frombuffer(bytes(t.mult), dtype=np.int32).astype(np.int64)
        packed = mult != 0
        if packed.any():
            mag = np.frombuffer(bytes(t.magic), dtype=np.uint32).astype(np.uint64)[packed]
            bias = np.frombuffer(bytes(t.bias), dtype=np.int32).astype(np.int64)[packed]
            kq = np.frombuffer(bytes(t.kq), dtype=np.int32).astype(np.int64)[packed]
            Up = (Z[None, :] + bias[:, None]) * mult[packed][:, None] + (Z >= 0)[None, :]
            assert Up.min() >= 0 and Up.max() <= 0xFFFF
            gotp = ((Up.astype(np.uint64) * mag[:, None]) >> np.uint64(32)).astype(np.int64) - kq[:, None]
            assert np.array_equal(gotp, want[packed])
        if not packed.all():
            assert t.wide == 1
