"""CPU-side checks of the boundary: the library builds, loads, and exports every
symbol include/setbwte.h declares (no compute calls -- no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "setbwte.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(setbwte_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1410_0562_b200 import _build
    _build.build()
    return ctypes.CDLL(_build.LIB)


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["setbwte_create", "setbwte_append", "setbwte_bwt", "setbwte_rank",
              "setbwte_destroy"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_covers_every_declared_symbol():
    from paper_1410_0562_b200 import binding
    assert sorted(binding.EXPORTS) == _declared()


def test_binding_loads_and_strerror(lib):
    from paper_1410_0562_b200 import binding
    L = binding.load_library()
    assert L.setbwte_strerror(0) == b"ok"
    assert L.setbwte_strerror(2) == b"invalid character"
    assert b"NCCL" in L.setbwte_strerror(8)


def test_set_comm_argument_checks_without_gpu(lib):
    """setbwte_set_comm rejects a NULL handle before touching NCCL or CUDA."""
    from paper_1410_0562_b200 import binding
    L = binding.load_library()
    assert L.setbwte_set_comm(None, None, 0, 1) == 1


def test_create_without_gpu_fails_loudly(lib):
    """No CPU fallback: without a device, create returns a CUDA error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1410_0562_b200 import SetBWTE, SetBWTEError
    with pytest.raises(SetBWTEError):
        SetBWTE("ACGT")


def test_create_rejects_bad_alphabets(lib):
    from paper_1410_0562_b200 import binding
    L = binding.load_library()
    h = ctypes.c_void_p()
    assert L.setbwte_create(b"ACGTNX", ctypes.byref(h)) == 6  # sigma > 5: unsupported
    assert L.setbwte_create(b"", ctypes.byref(h)) == 1
    assert L.setbwte_create(b"AA", ctypes.byref(h)) == 1
    assert L.setbwte_create(b"A$", ctypes.byref(h)) == 1
    assert L.setbwte_create(b"Aa", ctypes.byref(h)) == 1      # case-insensitive duplicate


def test_sm100a_cubin_present(lib):
    import subprocess
    from paper_1410_0562_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
