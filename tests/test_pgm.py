"""PGM ingestion (row f4): header rules and errors like the reference's
corpus.read_pgm, P2/P5 round trips, and (GPU) files -> pinned -> pipeline."""

import numpy as np
import pytest

from oracle import exact
from paper_1702_00817_b200 import errors, pgm


def _write(path, data: bytes):
    path.write_bytes(data)
    return path


def test_p5_and_p2_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (16, 24), dtype=np.uint8)
    pgm.write_pgm_u8(img, tmp_path / "a.pgm")
    assert np.array_equal(pgm.read_pgm_u8(tmp_path / "a.pgm"), img)
    text = "P2\n# comment\n24 16\n255\n" + " ".join(str(int(v)) for v in img.ravel()) + "\n"
    _write(tmp_path / "b.pgm", text.encode())
    assert np.array_equal(pgm.read_pgm_u8(tmp_path / "b.pgm"), img)


def test_header_errors(tmp_path):
    with pytest.raises(errors.MalformedHeader):
        pgm.read_pgm_u8(_write(tmp_path / "e", b""))
    with pytest.raises(errors.MalformedHeader):
        pgm.read_pgm_u8(_write(tmp_path / "m", b"P6\n2 2\n255\n" + bytes(12)))
    with pytest.raises(errors.UnsupportedMaxval):
        pgm.read_pgm_u8(_write(tmp_path / "x", b"P5\n2 2\n65535\n" + bytes(8)))
    with pytest.raises(errors.TruncatedData):
        pgm.read_pgm_u8(_write(tmp_path / "t", b"P5\n4 4\n255\n" + bytes(5)))
    with pytest.raises(errors.MalformedHeader):
        pgm.read_pgm_u8(_write(tmp_path / "h", b"P5\n4 x\n255\n"))
    with pytest.raises(errors.MalformedHeader):
        pgm.read_pgm_u8(_write(tmp_path / "v", b"P2\n2 1\n7\n3 9\n"))


def test_matches_reference_reader(tmp_path, reference):
    rng = np.random.default_rng(1)
    img = rng.integers(0, 200, (8, 16), dtype=np.uint8)
    raw = b"P5 # c\n16 8\n200\n" + img.tobytes()
    p = _write(tmp_path / "r.pgm", raw)
    ref = reference.corpus.read_pgm(p)
    assert np.array_equal(ref.samples.astype(np.uint8), pgm.read_pgm_u8(p))


def test_load_batch_unpinned(tmp_path):
    imgs = [np.full((8, 8), k, np.uint8) for k in range(3)]
    paths = []
    for k, im in enumerate(imgs):
        pgm.write_pgm_u8(im, tmp_path / f"{k}.pgm")
        paths.append(tmp_path / f"{k}.pgm")
    b = pgm.load_batch(paths, pinned=False)
    assert b.shape == (3, 8, 8) and np.array_equal(b[2], imgs[2])


@pytest.mark.gpu
def test_compress_files_end_to_end(tmp_path, cuda):
    rng = np.random.default_rng(2)
    imgs = rng.integers(0, 256, (5, 64, 48), dtype=np.uint8)
    paths = []
    for k in range(5):
        pgm.write_pgm_u8(imgs[k], tmp_path / f"im{k}.pgm")
        paths.append(tmp_path / f"im{k}.pgm")
    res = pgm.compress_files(paths, 10, out_dir=tmp_path / "out")
    wr, ws, _ = exact.compress_retain(imgs, 10)
    for k, (name, m, _) in enumerate(res):
        assert name == f"im{k}" and m == ws[k] / (64 * 48)
        assert np.array_equal(pgm.read_pgm_u8(tmp_path / "out" / f"im{k}_r10.pgm"), wr[k])


def test_error_classes_match_reference_reader(tmp_path, reference):
    """Every malformed file raises the same error class as corpus.read_pgm."""
    cases = {
        "empty": b"", "magic": b"P6\n2 2\n255\n" + bytes(12), "maxval": b"P5\n2 2\n65535\n" + bytes(8),
        "maxval0": b"P5\n2 2\n0\n" + bytes(4), "trunc5": b"P5\n4 4\n255\n" + bytes(5),
        "nonint": b"P5\n4 x\n255\n", "early": b"P5\n4 4\n", "zero": b"P5\n0 4\n255\n",
        "neg": b"P2\n-2 2\n255\n1 2 3 4\n", "above": b"P2\n2 1\n7\n3 9\n",
        "trunc2": b"P2\n2 2\n255\n1 2 3\n", "badsample": b"P2\n2 1\n255\n1 q\n",
        "comments": b"P2 # a\n# b\n2 1 # c\n255\n7 # d\n 8\n", "plus": b"P5\n+2 1\n255\n\x01\x02",
        "above5": b"P5\n2 1\n100\n\x01\xff",
    }
    for name, raw in cases.items():
        p = _write(tmp_path / f"{name}.pgm", raw)
        try:
            ref = reference.corpus.read_pgm(p).samples
            ref_exc = None
        except Exception as e:  # noqa: BLE001
            ref_exc = type(e)
        try:
            ours = pgm.read_pgm_u8(p)
            our_exc = None
        except Exception as e:  # noqa: BLE001
            our_exc = type(e)
        # same class name (ours mirror the reference's errors.py) and base class
        assert (our_exc and our_exc.__name__) == (ref_exc and ref_exc.__name__), (name, our_exc, ref_exc)
        assert our_exc is None or our_exc.__mro__[1].__name__ == ref_exc.__mro__[1].__name__
        if ref_exc is None:
            assert np.array_equal(ours, ref.astype(np.uint8)), name
