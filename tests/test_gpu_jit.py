"""Run-time specialisation of the quantised kernels (csrc/quant_jit.cu):
with ADCT_QUANT_JIT_AFTER=1 every table is rebuilt with NVRTC on first use;
all four k_quant_p variants and the hybrid coarse-table kernel must stay
bit-exact, and the counters must show specialised launches.  Child processes:
the threshold is read once per process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import ctypes, numpy as np, torch
from oracle import exact
from paper_1702_00817_b200 import batch, quant, synth, _lib
dev = torch.device("cuda", 0)
def stats():
    c, l, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.lib().adct_quant_jit_stats(ctypes.byref(c), ctypes.byref(l), ctypes.byref(f))
    return c.value, l.value, f.value
xp = synth.config_images_device(2, [3, 4], device=dev)[:, :128, :512].contiguous()
xs = xp[:, :, :504].contiguous()
rng = np.random.default_rng(5)
custom = quant.quant_table(qprime_unrounded=rng.choice([1.0, 3.0, 6.0, 16.5, 255.0, 4000.0], size=(8, 8)))
cases = [(xp, quant.quant_table(75)), (xp, quant.quant_table(30)), (xs, quant.quant_table(75)),
         (xs, quant.quant_table(30)), (xp, quant.quant_table(10)), (xp, custom)]
for x, qt in cases:
    for rep in range(2):
        rec, sse = batch.compress_quant(x, qt)
        torch.cuda.synchronize()
        wr, ws = exact.compress_quant(x.cpu().numpy(), quant.qtab_qprime(qt))
        assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws)
planes = [xp, xp[:, :64, :256].contiguous(), xp[:, 64:, 256:].contiguous()]
qt = quant.quant_table(75)
recs, sse = batch.compress_quant_planes(planes, qt)
torch.cuda.synchronize()
for k, p in enumerate(planes):
    wr, ws = exact.compress_quant(p.cpu().numpy(), quant.qtab_qprime(qt))
    assert np.array_equal(recs[k].cpu().numpy(), wr) and np.array_equal(sse[:, k].cpu().numpy(), ws)
print("STATS", *stats())
'''


def _run(after):
    env = dict(os.environ, PYTHONPATH=ROOT, ADCT_QUANT_JIT_AFTER=str(after), ADCT_QUANT_JIT_LOG="1")
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("STATS")][-1]
    return tuple(int(v) for v in line.split()[1:])


def test_specialised_kernels_are_exact():
    compiled, launches, failures = _run(1)
    assert failures == 0
    assert compiled >= 4  # pair/single x aligned/flip (coarse tables run k_quant_fi, never specialised)
    assert launches >= 9  # 4 tables x 2 calls + the planes call


def test_specialisation_off():
    assert _run(0) == (0, 0, 0)


def test_first_use_inside_graph_capture():
    """A table first seen while the stream is being captured keeps the generic
    kernel in the graph (no module load during capture); the replay is exact
    and the next uncaptured call specialises."""
    code = r'''
import ctypes, numpy as np, torch
from oracle import exact
from paper_1702_00817_b200 import batch, quant, synth, _lib
dev = torch.device("cuda", 0)
x = synth.config_images_device(2, [5], device=dev)[:, :128, :256].contiguous()
qt = quant.quant_table(75)
rec = torch.empty_like(x); sse = torch.empty(1, dtype=torch.int64, device=dev)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        batch.compress_quant(x, qt, out=rec, sse_out=sse)
g.replay(); torch.cuda.synchronize()
wr, ws = exact.compress_quant(x.cpu().numpy(), quant.qtab_qprime(qt))
assert np.array_equal(rec.cpu().numpy(), wr) and np.array_equal(sse.cpu().numpy(), ws)
batch.compress_quant(x, qt, out=rec, sse_out=sse); torch.cuda.synchronize()
assert np.array_equal(rec.cpu().numpy(), wr)
c, l, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
_lib.lib().adct_quant_jit_stats(ctypes.byref(c), ctypes.byref(l), ctypes.byref(f))
print("STATS", c.value, l.value, f.value)
'''
    env = dict(os.environ, PYTHONPATH=ROOT, ADCT_QUANT_JIT_AFTER="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    compiled, launches, failures = (int(v) for v in r.stdout.split("STATS")[1].split())
    assert failures == 0 and compiled == 1 and launches == 1
