"""Host-only (nvcc, no GPU): the FAST selector's reflection form (k_down.cuh bucket32_fast, the
form every down kernel runs) against the rotation form it replaced, on random Gram-matrix window
sums and on tensors placed within 1e-5 rad of every orientation edge: no pixel certified by both
forms may get a different orientation bin ("The FAST bucket decision")."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="needs nvcc")
def test_reflection_form_matches_rotation_form(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "bfc"
    subprocess.check_call([nvcc, "-std=c++17", "-O2", "-arch=sm_100a", "-I", str(ROOT / "paper_1802_06130_b200/csrc"),
                           str(ROOT / "scripts/probes/bucket_fast_check.cu"), "-o", str(exe)],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    r = subprocess.run([str(exe), "2000000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "orient mismatches among both-certified: 0" in r.stdout, r.stdout
