"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol include/helmsweep.h declares, and fails loudly (no CPU fallback)
when there is no CUDA device."""
import ctypes
import os
import re

import pytest

from paper_2408_11929_b200 import build as build_mod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    hdr = open(os.path.join(ROOT, "include", "helmsweep.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = re.findall(r"^\s*(?:int|void|long|const char\*)\s+(\w+)\s*\(", hdr, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    path = build_mod.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ["helm_assemble", "sweep_setup", "sweep_apply", "mpgmres_solve", "helm_spmv",
                     "helm_load_vector"]:
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_lists_every_export():
    import paper_2408_11929_b200 as pkg
    assert sorted(pkg.EXPORTS) == declared_functions()


def test_sass_is_sm100a():
    """The fat binary holds sm_100a SASS and the sweep kernel uses the TMA
    bulk-copy engine (UBLKCP) with mbarriers (SYNCS)."""
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump not available")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", build_mod.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sweep = out[out.find("k_sweep_apply"):]
    assert "UBLKCP" in sweep


def test_no_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2408_11929_b200 as pkg
    with pytest.raises(pkg.HelmError) as ei:
        pkg.Problem(8, 8, 1.0 / 8, 5.0)
    assert ei.value.code == 4   # HELM_ECUDA


def test_missing_library_fails_loudly(tmp_path):
    """Without the built CUDA library the product path raises at the first call
    (there is no CPU fallback to land on)."""
    import subprocess
    import sys
    code = ("import paper_2408_11929_b200 as hs\n"
            "try:\n"
            "    hs.Problem(8, 8, 1.0 / 8, 5.0)\n"
            "except ImportError as e:\n"
            "    print('IMPORTERROR', e)\n")
    env = dict(os.environ, HELM_LIB=str(tmp_path / "libhelmsweep.so"), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "IMPORTERROR" in out.stdout and "not built" in out.stdout


def test_knobs_are_explicit_calls(lib):
    """Kernel / path choices are explicit helm_set_knob calls (no environment
    variable is read by the library); unknown names and values are rejected."""
    import paper_2408_11929_b200 as pkg
    pkg.set_knob("sweep_kernel", 3)
    pkg.set_knob("sweep_kernel", 0)
    with pytest.raises(pkg.HelmError) as ei:
        pkg.set_knob("sweep_kernel", 1)
    assert ei.value.code == 1
    with pytest.raises(pkg.HelmError):
        pkg.set_knob("no_such_knob", 1)
    so = open(build_mod.LIB, "rb").read()
    assert b"getenv" not in so


def test_binding_rejects_wrong_buffers():
    """The binding checks dtype, contiguity and size before handing a pointer to
    the C ABI (a complex64 or short tensor would be read / written out of bounds)."""
    import numpy as np
    import torch
    import paper_2408_11929_b200 as pkg
    with pytest.raises(ValueError):
        pkg._ptr(torch.zeros(8, dtype=torch.complex64), np.complex128, 8)
    with pytest.raises(ValueError):
        pkg._ptr(torch.zeros(7, dtype=torch.complex128), np.complex128, 8)
    with pytest.raises(ValueError):
        pkg._ptr(torch.zeros(16, dtype=torch.complex128)[::2], np.complex128, 8)
    with pytest.raises(ValueError):
        pkg._ptr(np.zeros(8, dtype=np.complex64), np.complex128, 8, out=True)
    p, keep = pkg._ptr(np.zeros(8, dtype=np.float32), np.complex128, 8)   # inputs are converted
    assert keep.dtype == np.complex128
