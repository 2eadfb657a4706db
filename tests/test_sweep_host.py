"""Host logic of sweep.run_sweep (no GPU: the per-transform MSE matrix is
stubbed).  Its summaries are built straight from the MSE matrix and must equal
the reference-semantics metrics.summarize over the records it returns,
bit for bit, for both PSNR conventions, unique or repeated transform names
and ragged corpora.  The corpus batching must be zero-copy for consecutive
planes of one array."""

import numpy as np
import pytest

from paper_1702_00817_b200 import metrics, sweep


def _stub(monkeypatch, seed):
    rng = np.random.default_rng(seed)

    def fake(t, stack, r_min, r_max, device=None):
        m = rng.random((stack.shape[0], r_max - r_min + 1)) * 80.0
        m[:, -1] *= rng.integers(0, 2, stack.shape[0])  # some lossless (MSE 0, PSNR inf)
        return m

    monkeypatch.setattr(sweep, "sweep_mse", fake)


@pytest.mark.parametrize("names", [("proposed",), ("dct", "proposed"), ("proposed", "proposed")])
@pytest.mark.parametrize("flag", [False, True])
def test_summaries_equal_reference_summarize(monkeypatch, names, flag):
    _stub(monkeypatch, len(names) + 10 * flag)
    base = np.zeros((7, 16, 24), np.uint8)
    images = [(f"a{k}", base[k]) for k in range(7)] + [("odd", np.zeros((8, 40), np.uint8)),
                                                     ("f", np.zeros((16, 24), np.float64))]
    cfg = sweep.ExperimentConfig(transforms=names, r_min=3, r_max=17, psnr_from_avg_mse=flag)
    records, summaries, ape = sweep.run_sweep(cfg, images)
    ref = metrics.summarize(records, psnr_from_avg_mse=flag)
    key = lambda s: (s.transform_name, s.r, s.avg_mse, s.avg_psnr, s.n_images)  # noqa: E731
    assert [key(s) for s in summaries] == [key(s) for s in ref]
    assert len(records) == len(names) * len(images) * 15
    if "dct" in names:
        assert set(ape) == {(s.transform_name, s.r) for s in summaries}


def test_empty_corpus_raises_like_the_reference(monkeypatch):
    _stub(monkeypatch, 0)
    with pytest.raises(metrics.EmptyGroup if hasattr(metrics, "EmptyGroup") else Exception):
        sweep.run_sweep(sweep.ExperimentConfig(transforms=("proposed",)), [])


def test_batch_of_is_zero_copy_for_consecutive_planes():
    base = np.arange(5 * 8 * 16, dtype=np.uint8).reshape(5, 8, 16)
    images = [(str(k), base[k]) for k in range(5)]
    b = sweep._batch_of(images, [1, 2, 3])
    assert np.shares_memory(b, base) and np.array_equal(b, base[1:4])
    b2 = sweep._batch_of(images, [0, 2, 3])  # not consecutive: a copy, same values
    assert not np.shares_memory(b2, base) and np.array_equal(b2, base[[0, 2, 3]])
    loose = [(str(k), base[k].copy()) for k in range(3)]
    assert np.array_equal(sweep._batch_of(loose, [0, 1, 2]), base[:3])
