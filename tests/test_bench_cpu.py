"""bench.py host-side pieces: the flop model and the reference arm (the oracle) JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_flop_model_matches_survey():
    f = bench.flops_per_instance(50, chunk=1)
    # ~16.8 n^3 per full combine, 2(L-1) - floor(log2 L) combines for L = 52
    assert 2.5e6 < f["k_scan_bwd"] < 4.5e6
    g = bench.flops_per_instance(50, chunk=52)
    assert abs(g["k_scan_bwd"] - 51 * (8.67 * 12 ** 3 + 4 * 144)) < 1
    assert g["k_srbd_bwd_fold"] > g["k_scan_bwd"]


def test_fp32_peak():
    assert abs(bench.fp32_peak_tflops(1965.0) - 74.45) < 0.01


def test_reference_arm_json():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--ref-sample", "16", "--N", "10"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "solves/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
