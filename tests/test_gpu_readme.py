"""The README's usage snippet runs as written (keeps the documentation honest)."""

import os
import re

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_usage_snippet_runs(cuda):
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.findall(r"Use:\n\n```python\n(.*?)```", text, re.S)[0]
    ns: dict = {}
    exec(compile(code, "README.md", "exec"), ns)
    assert ns["rec"].shape == ns["imgs"].shape and ns["out"].shape == ns["host"].shape
    assert ns["x"].shape == (512, 512)
