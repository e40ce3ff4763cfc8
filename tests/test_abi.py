"""C-ABI checks that need no GPU: libbl.so loads, exports every symbol
include/bl.h declares, rejects invalid CSR / params with BL_EINVAL, and the
binding has no CPU fallback path."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "bl.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bl_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    import paper_2002_08233_b200 as bl
    names = _header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(bl.lib, name), name
    assert sorted(bl.EXPORTS) == names


def test_library_is_sm100a():
    """The in-tree .so carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    so = os.path.join(ROOT, "paper_2002_08233_b200", "libbl.so")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_params_default_are_the_papers():
    import paper_2002_08233_b200 as bl
    p = bl.bl_params_default()
    assert (p.iters, p.batch) == (600, 256)
    assert (p.K, p.C, p.step0) == (1.0, 1.0, 1.0)
    assert p.cooling == 0.999
    assert (p.tol, p.max_batches, p.flags) == (0.0, 0, 0)


def test_status_strings():
    import paper_2002_08233_b200 as bl
    for s in (0, -1, -2, -3, -4):
        assert bl.lib.bl_status_string(s).startswith(b"BL_")


@pytest.mark.parametrize("case", [
    ("n0", 0, [0], []),
    ("rowptr0", 2, [1, 1, 2], [1, 0]),
    ("decreasing", 3, [0, 2, 1, 2], [1, 2]),
    ("range", 2, [0, 1, 2], [5, 0]),
    ("selfloop", 2, [0, 1, 1], [0]),
    ("unsorted", 3, [0, 2, 3, 4], [2, 1, 0, 0]),
    ("duplicate", 2, [0, 2, 4], [1, 1, 0, 0]),
    ("asymmetric", 3, [0, 1, 1, 1], [1]),
])
def test_create_rejects_invalid_csr(case):
    import paper_2002_08233_b200 as bl
    _, n, rp, ci = case
    with pytest.raises(bl.BLError) as ei:
        bl.bl_create(n, np.array(rp, np.int32), np.array(ci, np.int32))
    assert ei.value.status == bl.BL_EINVAL


def test_create_without_gpu_is_a_cuda_error_not_a_fallback():
    import torch
    import paper_2002_08233_b200 as bl
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bl.BLError) as ei:
        bl.bl_create(3, np.array([0, 1, 2, 2], np.int32), np.array([1, 0], np.int32))
    assert ei.value.status == bl.BL_ECUDA


def test_null_args():
    import paper_2002_08233_b200 as bl
    assert bl.lib.bl_create(3, None, None, None) == bl.BL_EINVAL
    assert bl.lib.bl_layout(None, None, None, None) == bl.BL_EINVAL
    assert bl.lib.bl_energy(None, None, None, 0, None, None) == bl.BL_EINVAL
    bl.lib.bl_destroy(None)  # no-op


def test_product_package_does_not_import_oracle():
    """The product path never touches oracle/ (DESIGN.md §2)."""
    pkg = os.path.join(ROOT, "paper_2002_08233_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("no CPU fallback", ""), f


@pytest.mark.parametrize("case", [
    ("rowptr_short", 3, [0, 1, 2], [1, 0]),          # n + 1 = 4 entries expected
    ("rowptr_long", 2, [0, 1, 2, 2], [1, 0]),
    ("colidx_short", 2, [0, 1, 2], [1]),             # rowptr[n] = 2 entries expected
    ("colidx_long", 2, [0, 1, 2], [1, 0, 1]),
])
def test_binding_rejects_missized_csr_before_the_c_call(case):
    """The C side reads rowptr[0..n] and colidx[0..rowptr[n]) unconditionally;
    the binding checks the array sizes first (no out-of-bounds host read)."""
    import paper_2002_08233_b200 as bl
    _, n, rp, ci = case
    with pytest.raises(bl.BLError) as ei:
        bl.bl_create(n, np.array(rp, np.int32), np.array(ci, np.int32))
    assert ei.value.status == bl.BL_EINVAL
    assert "entries" in str(ei.value)
