"""Soundness of the float32 cone filter (hp_cone.cuh) on the CPU: the same
__host__ __device__ code the kernels run, stressed with adversarial
(ray, point) pairs near the t-range and cone boundaries.  A sure-accept must
be an fp64 accept and a sure-reject an fp64 reject (zero violations)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_filter_never_contradicts_fp64(tmp_path):
    exe = tmp_path / "cone_check"
    subprocess.run(["nvcc", "-O2", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-ffp-contract=off",
                    "-o", str(exe), os.path.join(ROOT, "tests", "native", "cone_filter_check.cu")],
                   check=True)
    out = subprocess.run([str(exe), "3000000"], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout
    fields = dict(kv.split("=") for kv in out.stdout.split())
    assert int(fields["violations"]) == 0
    assert int(fields["sure_accept"]) > 0 and int(fields["sure_reject"]) > 0


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_footprint_contains_every_accepted_point(tmp_path):
    exe = tmp_path / "fp_check"
    subprocess.run(["nvcc", "-O2", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-ffp-contract=off",
                    "-o", str(exe), os.path.join(ROOT, "tests", "native", "footprint_check.cu")],
                   check=True)
    out = subprocess.run([str(exe), "60"], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout
    assert "violations=0" in out.stdout
