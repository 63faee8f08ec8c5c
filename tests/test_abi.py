"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/surrogate.h declares, and its host-only entry points validate."""

import ctypes
import os
import re

import pytest

import paper_2306_14011_b200 as pk
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    pk.build_library()
    return pk.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "surrogate.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(surrogate_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["surrogate_load_weights", "surrogate_predict", "surrogate_sweep"]:  # north star
        assert must in names
    assert set(names) == set(pk.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_sm100a_code_in_library(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", pk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_space_size_exact_and_overflow(lib):
    assert pk.space_size(workloads.space("paper")) == 10 ** 7 * 12 ** 7
    assert pk.space_size(workloads.space("cfg5")) == 28 ** 7
    with pytest.raises(pk.SurrogateError, match="64 bits"):
        pk.space_size([list(range(1, 17))] * 17)   # 16^17 = 2^68 > 2^64


def test_create_without_gpu_reports_no_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = lib.surrogate_create(0, ctypes.byref(h))
    assert rc == 3  # SURR_E_NO_DEVICE: there is no CPU fallback
    assert b"device" in lib.surrogate_last_error(None)


def test_binding_refuses_without_library(monkeypatch):
    monkeypatch.setattr(pk, "LIB_PATH", "/nonexistent/libsurrogate.so")
    monkeypatch.setattr(pk, "_LIB", None)
    with pytest.raises(pk.SurrogateError, match="no CPU fallback"):
        pk.lib()


def test_key_mapping_roundtrip():
    import numpy as np
    t = np.array([-2.5, -0.0, 0.0, 0.75, 1.5, np.inf], np.float32)
    # order-preserving keys as the kernels compute them (f2key), inverted by the binding
    u = t.view(np.uint32)
    keys = np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint32)
    assert np.all(np.diff(keys.astype(np.int64)) > 0)
    assert np.array_equal(pk.key_to_float(keys), t)
