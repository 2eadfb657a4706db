"""bench.py's driver contract on CPU: the reference arm (which needs no GPU)
prints one JSON line with the required keys; --help works."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_help():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "--impl" in r.stdout and "--exchange" in r.stdout


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, RANK="0"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    ref_installed = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "adct"))
    assert d["cpu_baseline"]["kind"] == ("reference" if ref_installed else "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["units_per_gpu"] == 1 and d["config"]["pixels_per_step"] == 512 * 512


def test_reference_arm_nonzero_rank_is_silent():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, RANK="1"))
    assert r.returncode == 0 and r.stdout.strip() == ""


def _plan(nproc, *extra):
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(nproc), "--plan", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=dict(os.environ, ADCT_DIST_BACKEND="gloo"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_two_rank_plan_is_strong_scaling_of_config3():
    """torchrun --nproc-per-node 2 bench.py --gpus 2: BASELINE config 3's 4096
    images split over the ranks (not 4096 per rank)."""
    d = _plan(2)
    assert d["config"]["units_per_gpu"] == 2048
    assert d["config"]["pixels_per_step"] == 17179869184  # 4096 x 2048^2, the whole config once
    assert d["config"]["scaling"] == "strong" and d["units_all_ranks"] == 4096
    assert d["first_unit_per_rank"] == [0, 2048]


def test_two_rank_plan_config4_frames_and_weak_option():
    d = _plan(2, "--config", "4")
    assert d["config"]["units_per_gpu"] == 256 and d["units_all_ranks"] == 512
    assert d["config"]["pixels_per_step"] == 512 * (3840 * 2160 + 2 * 1920 * 1080)
    w = _plan(2, "--scaling", "weak")
    assert w["config"]["units_per_gpu"] == 4096 and w["config"]["pixels_per_step"] == 2 * 17179869184


def test_clock_sampler_parses_nvidia_smi_lines():
    """The clocks record of the bench line: median SM clock under load, max,
    and every throttle reason seen, from nvidia-smi's CSV samples."""
    sys.path.insert(0, ROOT)
    import bench

    cs = bench.ClockSampler(0)
    cs.proc = type("P", (), {"terminate": lambda self: None, "wait": lambda self, timeout=None: 0,
                             "kill": lambda self: None})()
    cs.t = type("T", (), {"join": lambda self, timeout=None: None})()
    cs.lines = [
        "0, 1965, 1965, 900.1, 0x0, Not Active, Not Active, Not Active, Not Active",
        "0, 1800, 1965, 1000.3, 0x4, Not Active, Not Active, Not Active, Active",
        "0, 1965, 1965, 950.0, 0x0, Not Active, Not Active, Not Active, Not Active",
        "garbage line",
    ]
    rec = cs.stop()
    assert rec["sm_mhz"] == 1965.0 and rec["sm_max_mhz"] == 1965.0 and rec["samples"] == 3
    assert rec["reasons"] == ["sw_power_cap"]


def test_hbm_peak_source(tmp_path, monkeypatch):
    sys.path.insert(0, ROOT)
    import bench

    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    peak, src = bench.measured_hbm_peak()
    assert peak == bench.FALLBACK_HBM_GBS and "fallback" in src
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_gbs": 6462.7}))
    peak, src = bench.measured_hbm_peak()
    assert peak == 6462.7 and "MEASURED_PEAKS" in src
