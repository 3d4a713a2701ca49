"""C-ABI boundary checks that run without a GPU: the library loads, exports
every function include/milo_b200.h declares, validates descriptors in the
reference's categories before touching the device, and the C++ host header
(include/milo_b200.hpp) compiles against it."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "milo_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2504_02658_b200 import LIB_PATH
    from paper_2504_02658_b200 import build as b
    if not os.path.exists(LIB_PATH):
        b.build()
    return ctypes.CDLL(LIB_PATH)


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(milo_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib.milo_device_check.restype = ctypes.c_int
    assert lib.milo_device_check() == 100  # MILO_ERR_CUDA, no CPU fallback
    lib.milo_last_error.restype = ctypes.c_char_p
    assert b"device" in lib.milo_last_error()


def test_cpp_header_compiles_and_validates(lib, tmp_path):
    from paper_2504_02658_b200 import LIB_PATH
    exe = str(tmp_path / "abi_check")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "abi_check.cpp"), LIB_PATH,
                           "-Wl,-rpath," + os.path.dirname(LIB_PATH), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "abi_check ok" in out.stdout
