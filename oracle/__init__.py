"""CPU oracle for the 8x8 approximate-DCT hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference's algorithm (arxiv 1702.00817, package
`adct`, /root/reference/pkg/src/adct) on the CPU so the CUDA path can be
checked against it.  Only tests/, __graft_entry__.smoke() and bench.py's
`cpu_baseline` / `--impl reference` legs may import it, and only as the
checker or the timed CPU baseline — never as a product code path.

* exact.py   — exact integer restatement (int64 numpy): forward T X T^T,
               dyadic inverse 64 X = T^T (E o Z) T, retain-r, round-half-away
               quantiser, SSE.  Bit-exact target for every config.
* exact_c.c / fast.py — the same exact results from plain C (straight
               matrix products with T, int64), built by oracle/Makefile into
               oracle/_build/ and driven over a thread pool: fast enough to
               check every BASELINE config at its full size
               (tests/test_gpu_fullsize.py).  Pinned to exact.py and the
               golden vectors in tests/test_oracle.py.
* refport.py — float64 restatement of the reference's own dense-matrix code
               path (codec.py:68-155, metrics.py:49-65), used to cross-check
               exact.py (differences only at exact .5 ties) and as the CPU
               baseline ("port") timed by bench.py.

Pinning: exact.py and refport.py are checked (tests/test_oracle.py) against
the SPEC.md known-answer examples, against golden vectors produced by
importing the reference itself (tests/golden/make_golden.py), and — when
/root/reference is present — against the live reference.
"""
