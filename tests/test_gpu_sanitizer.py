"""compute-sanitizer memcheck / racecheck / synccheck / initcheck over small runs of every kernel family
(fused fold path, cooperative grid scans, single-CTA scans, padded and large-dimension paths)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_smoke.py")], capture_output=True, text=True, timeout=900)
    if r.returncode == 86 or "closed on this pool" in (r.stdout + r.stderr):
        pytest.skip("compute-sanitizer is disabled on this GPU pool (the wrapper refuses to run); "
                    "the committed logs under profiles/ (r2_initcheck.log) are the evidence")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize smoke done" in r.stdout
