"""INTEGRATION.md's reference-side binding sample (adct/_gpu.py) runs as
written against the in-tree library and matches the oracle."""

import os
import re

import numpy as np
import pytest

from oracle import exact
from paper_1702_00817_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_sample(cuda, monkeypatch):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.findall(r"```python\n(# adct/_gpu.py.*?)```", text, re.S)[0]
    code = code.replace("from .errors import", "from paper_1702_00817_b200.errors import")
    monkeypatch.setenv("ADCT_CUDA_LIB", os.path.join(ROOT, "paper_1702_00817_b200", "libadct_cuda.so"))
    ns = {}
    exec(compile(code, "INTEGRATION.md:adct/_gpu.py", "exec"), ns)
    img = synth.images_np([3], 128, 256, 16, 8.0, 64.0)
    rec, sse = ns["compress_batch_u8"](img, 10)
    wr, ws, _ = exact.compress_retain(img, 10)
    assert np.array_equal(rec, wr) and np.array_equal(sse, ws)
    got = ns["sweep_sse"](img[0], 2, 12)
    want = np.array([exact.compress_retain(img, r)[2][0] / 4096.0 for r in range(2, 13)])
    assert np.array_equal(got, want)
