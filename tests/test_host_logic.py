"""Host-side logic of the exact kernel's work partition, on the CPU: the
__host__ __device__ helpers of bl_kernel.cuh (bl_geom, bl_units,
bl_guided_start) compiled by nvcc into a host program (tests/cpp/) and run
here -- no GPU needed.  They decide which resident source slots each work
unit sweeps and whether the dirty slots (sources being updated in the same
phase) get their own sub-range; a gap or overlap would drop or double-count
pairs of Alg. 2's repulsion sum."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_work_partition_helpers(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "test_units"
    subprocess.run([nvcc, "-std=c++17", "-O1",
                    "-I", os.path.join(ROOT, "paper_2002_08233_b200", "csrc"),
                    "-I", os.path.join(ROOT, "include"),
                    "-o", str(exe), os.path.join(ROOT, "tests", "cpp", "test_units.cu")],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "OK (0 failures)" in r.stdout
