"""Prove the 16-bit lane bounds used by the fused kernels.

For the retain-r pipeline with level-shifted pixels X' = X - 128 in
[-128, 127], every intermediate of the inverse flow graph (column pass, row
pass) and every output V = 64 (x_hat - 128) is a linear functional of X';
its maximum magnitude is 128 * sum |coefficients|.  The script evaluates
that for every mask r = 1..64 and prints the worst case, which must stay
below 32767 - 32 (rounding bias) for the output fields to be unambiguous.
Run: python tools/range_bounds.py
"""

import numpy as np

import sys, os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.exact import A1, A2, A3, E, P, T, zigzag_indices  # noqa: E402

# inverse 1-D flow graph x = A1 A2 A3 P^T y; new values: b0, b1 (A3), a0..a3 (A2), outputs
M = P.T
b = A3 @ M
a = A2 @ b
x = A1 @ a
assert (x == T.T).all()
STEPS = np.vstack([b[:2], a[:4], x])  # 14 linear functionals of the 8 inputs


def worst(r: int) -> int:
    mask = np.zeros(64, dtype=np.int64)
    mask[list(zigzag_indices()[:r])] = 1
    K = np.einsum("ui,vj->uvij", T, T).reshape(64, 64) * (E.reshape(64) * mask)[:, None]  # W = K @ x'
    W = K.reshape(8, 8, 64)
    col = np.einsum("ku,uvx->kvx", STEPS, W)  # column pass: (14, v, x)
    row = np.einsum("kv,ivx->ikx", STEPS, col[6:])  # row pass on column outputs
    return int(max(np.abs(col).sum(-1).max(), np.abs(row).sum(-1).max()) * 128)


if __name__ == "__main__":
    w = {r: worst(r) for r in range(1, 65)}
    print("worst |intermediate| per r:", w)
    print("max over r:", max(w.values()), "(limit 32735)")
    assert max(w.values()) + 32 <= 32767
