"""Regenerate ``paper_1702_00817_b200/data/q50_luma.txt``.

The quantised pipeline (BASELINE configs 2 and 4) needs the standard JPEG
luminance base table Q50 (ITU-T T.81 Annex K, Table K.1).  It is not present
anywhere in the reference package, and it must not be typed from memory, so it
is read back from libjpeg through Pillow: a JPEG written at ``quality=50`` uses
Q50 itself (IJG scale factor 100 %), and ``Image.quantization[0]`` returns the
table in natural row-major order (u*8+v) in Pillow >= 9.

Run: ``python tools/gen_q50.py``.  The output is committed; nothing reads
Pillow at run time.
"""

from __future__ import annotations

import io
from pathlib import Path

import numpy as np
from PIL import Image

OUT = Path(__file__).resolve().parents[1] / "paper_1702_00817_b200" / "data" / "q50_luma.txt"


def main() -> None:
    buf = io.BytesIO()
    # A textured image so the encoder cannot take any shortcut; the table
    # written to the DQT segment depends only on the quality setting.
    rng = np.random.default_rng(0)
    Image.fromarray(rng.integers(0, 256, (64, 64), dtype=np.uint8)).save(buf, "JPEG", quality=50)
    buf.seek(0)
    table = np.asarray(Image.open(buf).quantization[0], dtype=np.int64).reshape(8, 8)
    # Sanity: a luminance table grows towards high frequencies (roughness test).
    assert table[0, 0] < table[7, 7] and table.min() >= 1 and table.max() <= 255
    lines = [
        "# JPEG luminance base quantisation table Q50 (ITU-T T.81 Annex K, Table K.1),",
        "# natural row-major order, read back from libjpeg via Pillow by tools/gen_q50.py",
    ]
    lines += [" ".join(f"{int(x):3d}" for x in row) for row in table]
    OUT.write_text("\n".join(lines) + "\n")
    print(OUT.read_text())


if __name__ == "__main__":
    main()
