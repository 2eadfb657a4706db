"""Pin the CPU oracle (oracle/exact.py, oracle/refport.py) to the reference.

1. Against tests/golden/golden.json — results of the reference itself
   (tests/golden/make_golden.py), so this runs anywhere (GPU box included).
2. Against the live reference package when /root/reference is present.
3. The dyadic identities the exact oracle relies on.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import exact, refport

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
IMAGES = dict(np.load(os.path.join(HERE, "golden", "images.npz")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- known answers (SPEC.md examples, evaluated by the reference) -------------

def test_kernel_matrix_and_stages():
    k = GOLDEN["kat"]
    assert exact.T.tolist() == k["T"]
    assert (exact.T @ exact.T.T).tolist() == k["gram"]
    assert [m.tolist() for m in (exact.A1, exact.A2, exact.A3, exact.P)] == k["stages"]
    assert np.array_equal(exact.P @ exact.A3 @ exact.A2 @ exact.A1, exact.T)
    assert np.array_equal(np.diag(exact.T @ exact.T.T), [8, 2, 4, 2, 8, 2, 4, 2])
    assert np.count_nonzero(exact.T) == 32  # SPEC.md:59 says 24; the reference matrix has 32


def test_flow_graph_kats():
    k = GOLDEN["kat"]
    assert (exact.T @ np.arange(1, 9)).tolist() == k["fast_forward_1to8"] == [36, -7, 0, 3, 0, 5, 0, 1]
    assert (exact.T @ np.ones(8, dtype=np.int64)).tolist() == k["fast_forward_ones"]
    assert k["op_count"] == [14, 0, 0]


def test_scaling_and_zigzag():
    k = GOLDEN["kat"]
    assert np.allclose(exact.D, k["scaling_diag"], rtol=0, atol=0)
    assert list(exact.zigzag_indices()) == k["zigzag"]
    assert sorted(exact.zigzag_indices()) == list(range(64))
    assert exact.zigzag_indices()[:6] == (0, 1, 8, 16, 9, 2)
    assert np.array_equal(np.argwhere(exact.retention_mask(3)).tolist(), [[0, 0], [0, 1], [1, 0]])


def test_dyadic_identities():
    # N2: E = 64 d^2 d^2^T is an integer in {1,2,4,8,16} and E * n_u * n_v = 64
    assert set(np.unique(exact.E).tolist()) == {1, 2, 4, 8, 16}
    assert np.all(exact.E * np.outer(exact.N_ROW, exact.N_ROW) == 64)
    # N3: T^T diag(e) T = 8 I  (so 64 X = T^T (E o Z) T exactly)
    assert np.array_equal(exact.T.T @ np.diag(exact.E_VEC) @ exact.T, 8 * np.eye(8, dtype=np.int64))
    # N10: T^T e0 e0^T T = all ones
    e0 = np.zeros((8, 8), dtype=np.int64)
    e0[0, 0] = 1
    assert np.all(exact.T.T @ e0 @ exact.T == 1)


def test_compression_ratio_and_fold_kats():
    k = GOLDEN["kat"]
    assert k["compression_ratio"]["2"] == 96.875 and k["compression_ratio"]["45"] == 29.6875
    assert k["compression_ratio"]["25"] == 60.9375
    assert k["fold_ones_00"] == pytest.approx(8.0, abs=1e-12)
    assert k["fold_ones_11"] == pytest.approx(2.0, abs=1e-12)
    qpu = np.ones((8, 8)) / np.outer(exact.D, exact.D)
    assert qpu[0, 0] == pytest.approx(8.0) and qpu[1, 1] == pytest.approx(2.0)


def test_psnr_kats():
    k = GOLDEN["kat"]
    assert refport.psnr(1.0) == pytest.approx(k["psnr"]["1"], abs=1e-12) == pytest.approx(48.1308036, abs=1e-6)
    assert refport.psnr(255.0**2) == 0.0 == k["psnr"]["65025"]
    assert math.isinf(refport.psnr(0.0)) and k["psnr"]["0"] == "inf"
    assert float(exact.psnr(1, 1)) == pytest.approx(k["psnr"]["1"], abs=1e-12)
    assert refport.mse(np.array([[0, 1], [2, 3]]), np.array([[1, 2], [3, 4]])) == k["mse_2x2"] == 1.0


def test_const_and_dc_blocks():
    k = GOLDEN["kat"]
    assert k["forward_const128_dc"] == pytest.approx(1024.0, abs=1e-9)
    assert np.allclose(k["inverse_dc1024"], 128.0, atol=1e-9)
    Z = exact.forward_unscaled(np.full((8, 8), 128))
    assert Z[0, 0, 0] == 8192 and np.count_nonzero(Z) == 1
    rec, sse, ssef = exact.compress_retain(np.full((16, 16), 128, np.uint8), 1)
    assert sse == 0 and ssef == 0 and np.all(rec == 128)


# --- config 0: exact integer forward -------------------------------------------

def test_config0_coefficients_bit_exact():
    g = GOLDEN["config0"]
    img = IMAGES["c0_seed0_512"]
    Z = exact.forward_unscaled(img).reshape(-1, 8, 8).astype(np.int64)
    assert sha(Z) == g["coef_sha256_int64"]
    assert int(Z.sum()) == g["coef_sum"] and int(np.abs(Z).max()) == g["coef_abs_max"]
    assert Z[:4].tolist() == g["coef_blocks_0_3"] and Z[-1].tolist() == g["coef_block_last"]
    assert np.abs(Z).max() <= 16320  # int16-safe
    assert g["roundtrip_max_err"] < 1e-9


def test_config0_roundtrip_refport():
    img = IMAGES["c0_seed0_512"].astype(np.float64)
    c = refport.coefficient_blocks(img)
    back = exact.untile(refport.C.T @ c @ refport.C, 512, 512)
    assert np.abs(back - img).max() < 1e-9


# --- config 1: retain-r ----------------------------------------------------------

@pytest.mark.parametrize("name", ["c0_seed0_512", "c1_seed1_128", "c1_seed2_128", "ragged_40x24", "noise_64", "saturated_32x48"])
def test_config1_retain_matches_reference(name):
    img = IMAGES[name]
    n_px = img.size
    for r_s, g in GOLDEN["config1"][name].items():
        r = int(r_s)
        rec, sse, ssef = exact.compress_retain(img, r)
        assert sse == g["sse_rounded"], (name, r)
        assert sha(rec) == g["rec_sha256"], (name, r)
        # the reference's own (unrounded, clamped) convention, exactly: ssef / 4096
        mse_f = ssef / (4096.0 * n_px)
        assert mse_f == pytest.approx(g["mse_ref"], rel=1e-9, abs=1e-12)
        assert refport.psnr(mse_f) == pytest.approx(g["psnr_ref"], abs=1e-9)


def test_config1_mse_monotone_in_r():
    img = IMAGES["c1_seed1_128"]
    ssef = [exact.compress_retain(img, r)[2] for r in range(2, 46)]
    assert all(a >= b for a, b in zip(ssef, ssef[1:]))


def test_config1_sweep_equals_single_r():
    img = np.stack([IMAGES["c1_seed1_128"], IMAGES["c1_seed2_128"]])
    s = exact.sweep_sse(img, 1, 45)
    for r in (1, 10, 45):
        assert np.array_equal(s[:, r - 1], exact.compress_retain(img, r)[1])


def test_full_retention_is_lossless():
    img = IMAGES["noise_64"]
    rec, sse, ssef = exact.compress_retain(img, 64)
    assert sse == 0 and ssef == 0 and np.array_equal(rec, img)


# --- configs 2/4: quantised pipeline -------------------------------------------------

@pytest.mark.parametrize("name", ["c2_seed3_128", "noise_64", "saturated_32x48", "ragged_40x24"])
@pytest.mark.parametrize("q", [10, 50, 75, 90])
def test_quant_matches_reference_composition(name, q):
    from paper_1702_00817_b200.quant import q50_luma

    g = GOLDEN["quant"][name][str(q)]
    Qp = exact.qprime(q50_luma(), q)
    assert Qp.tolist() == g["qprime"]
    rec, sse = exact.compress_quant(IMAGES[name], Qp)
    assert sse == g["sse"] and sha(rec) == g["rec_sha256"]


def test_quantize_round_half_away():
    Qp = np.full((8, 8), 4, dtype=np.int64)
    Z = np.array([-6, -5, -2, -1, 0, 1, 2, 5, 6, 10])
    q = exact.quantize(Z[:, None, None] * np.ones((1, 8, 8), np.int64), Qp)[:, 0, 0]
    assert q.tolist() == [-2, -1, -1, 0, 0, 0, 1, 1, 2, 3]  # -1.5 -> -2, 0.5 -> 1, 2.5 -> 3


def test_folding_property():
    """dividing unscaled coefficients by Q' equals dividing scaled by Q."""
    rng = np.random.default_rng(0)
    blocks = rng.integers(0, 256, (50, 8, 8))
    Q = rng.uniform(1, 50, (8, 8))
    Z = exact.T @ blocks @ exact.T.T
    Y = np.outer(exact.D, exact.D) * Z
    Qp = Q / np.outer(exact.D, exact.D)
    assert np.allclose(Z / Qp, Y / Q, rtol=1e-12, atol=1e-12)


# --- live reference (build container only) ---------------------------------------------

def test_refport_equals_live_reference(reference):
    t = reference.proposed_transform()
    img = IMAGES["c1_seed1_128"].astype(np.float64)
    for r in (1, 10, 25, 45):
        ref = reference.compress_image(t, img, r)
        ours = refport.compress_image(img, r)
        assert np.abs(ref - ours).max() < 1e-12


def test_exact_vs_live_reference_differs_only_at_ties(reference):
    t = reference.proposed_transform()
    img = IMAGES["c0_seed0_512"]
    for r in (3, 10, 25):
        ref = reference.compress_image(t, img.astype(np.float64), r)
        V = exact.inverse64(exact.E * exact.retention_mask(r) * exact.forward_unscaled(img))
        v64 = exact.untile(V, 512, 512)
        assert np.abs(np.clip(v64, 0, 16320) / 64.0 - ref).max() < 1e-9  # N4
        naive = np.clip(np.rint(ref), 0, 255)
        exact_rec = exact.compress_retain(img, r)[0]
        diff = naive != exact_rec
        on_tie = (v64 % 64) == 32
        assert np.all(on_tie[diff])  # N5: every disagreement is an exact .5 tie


def test_zigzag_matches_reference(reference):
    from paper_1702_00817_b200 import codec

    assert tuple(reference.codec.ZIGZAG_INDICES) == codec.ZIGZAG_INDICES == exact.zigzag_indices()


# --- the plain-C oracle (oracle/exact_c.c via oracle/fast.py): pinned to the
# --- reference-made golden vectors and to the numpy oracle --------------------------

def test_c_oracle_config0_golden():
    from oracle import fast

    g = GOLDEN["config0"]
    Z = fast.forward(IMAGES["c0_seed0_512"])[0].astype(np.int64)
    assert sha(Z) == g["coef_sha256_int64"]
    assert np.array_equal(fast.forward(IMAGES["noise_64"], level_shift=True),
                          exact.forward_unscaled(IMAGES["noise_64"], level_shift=True)[None])


@pytest.mark.parametrize("name", ["c0_seed0_512", "c1_seed1_128", "c1_seed2_128", "ragged_40x24", "noise_64", "saturated_32x48"])
def test_c_oracle_retain_golden(name):
    from oracle import fast

    img = IMAGES[name]
    for r_s, g in GOLDEN["config1"][name].items():
        rec, sse, ssef = fast.compress_retain(img, int(r_s), threads=3)
        assert int(sse[0]) == g["sse_rounded"] and sha(rec[0]) == g["rec_sha256"], (name, r_s)
        assert ssef[0] / (4096.0 * img.size) == pytest.approx(g["mse_ref"], rel=1e-9, abs=1e-12)


def test_c_oracle_sweep_golden_and_numpy():
    from oracle import fast

    name = "c1_seed1_128"
    s, sf = fast.sweep_sse(IMAGES[name], 1, 45, threads=2)
    assert [int(v) for v in s[0]] == [GOLDEN["config1"][name][str(r)]["sse_rounded"] for r in range(1, 46)]
    img = np.stack([IMAGES["c1_seed1_128"], IMAGES["c1_seed2_128"]])
    s, sf = fast.sweep_sse(img, 3, 17)
    assert np.array_equal(s, exact.sweep_sse(img, 3, 17))
    assert np.array_equal(sf[:, 10 - 3], exact.compress_retain(img, 10)[2])


@pytest.mark.parametrize("name", ["c2_seed3_128", "noise_64", "saturated_32x48", "ragged_40x24"])
@pytest.mark.parametrize("q", [10, 50, 75, 90])
def test_c_oracle_quant_golden(name, q):
    from oracle import fast
    from paper_1702_00817_b200.quant import q50_luma

    g = GOLDEN["quant"][name][str(q)]
    rec, sse = fast.compress_quant(IMAGES[name], exact.qprime(q50_luma(), q), threads=4)
    assert int(sse[0]) == g["sse"] and sha(rec[0]) == g["rec_sha256"]


def test_c_oracle_equals_numpy_oracle_random():
    """Random batches, ragged shapes, extreme tables: the two oracles agree."""
    from oracle import fast

    rng = np.random.default_rng(11)
    for shape in ((3, 64, 96), (2, 40, 24), (1, 8, 8)):
        x = rng.integers(0, 256, shape, dtype=np.uint8)
        for Qp in (np.ones((8, 8), np.int64), rng.integers(1, 3000, (8, 8)), np.full((8, 8), 2**20)):
            a, b = exact.compress_quant(x, Qp), fast.compress_quant(x, Qp, threads=3)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        for r in (1, 2, 10, 33, 64):
            a, b = exact.compress_retain(x, r), fast.compress_retain(x, r, threads=2)
            assert all(np.array_equal(u, v) for u, v in zip(a, b)), r
