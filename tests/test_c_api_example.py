"""The C ABI used from plain C (examples/c_api_example.c): compiled with gcc
against include/surrogate.h and linked with libsurrogate.so.  On a machine
without an sm_100 device it must exit 2 with SURR_E_NO_DEVICE's message; on a
B200 (-m gpu) its top-3 must match the oracle's for the same seeded net."""

import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "c_api_example.c")
PKG = os.path.join(ROOT, "paper_2306_14011_b200")


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    import paper_2306_14011_b200 as pk
    pk.build_library()
    exe = str(tmp_path / "c_api_example")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-L", PKG, "-lsurrogate",
                    f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_c_api_example_builds_and_reports_device(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode in (0, 2), res.stdout + res.stderr
    if res.returncode == 2:
        assert "no sm_100 device" in res.stdout


def _splitmix_net():
    """The example's seeded weights, regenerated (same SplitMix64 stream)."""
    state = [0x2306014011]
    M = (1 << 64) - 1

    def urand():
        state[0] = (state[0] + 0x9E3779B97F4A7C15) & M
        z = state[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        return (z >> 11) * (1.0 / 9007199254740992.0)

    widths = [14, 32, 32, 1]
    bounds = [0.38, 0.3, 0.42]
    W, b = [], []
    for l in range(3):
        W.append(np.array([(2.0 * urand() - 1.0) * bounds[l] for _ in range(widths[l] * widths[l + 1])])
                 .reshape(widths[l], widths[l + 1]))
        b.append(np.array([(2.0 * urand() - 1.0) * bounds[l] for _ in range(widths[l + 1])]))
    vl = [[100.0, 1000.0] if j % 2 == 0 else [32.0, 384.0] for j in range(14)]
    shift = np.array([0.5 * (v[0] + v[1]) for v in vl])
    scale = np.array([0.5 * (v[1] - v[0]) for v in vl])
    model = dict(widths=widths, members=[dict(W=W, b=b)], x_shift=shift, x_scale=scale, y_mean=1.4,
                 y_scale=0.3, const_features=np.zeros(0), x_scaler="custom")
    return model, vl


@pytest.mark.gpu
def test_c_api_example_matches_oracle(tmp_path):
    from oracle import sweep as osweep
    from tests.helpers import TOL, check_topk, need_gpu
    need_gpu()
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    lines = res.stdout.strip().splitlines()[1:]
    idx = np.array([int(l.split()[0]) for l in lines], np.uint64)
    t = np.array([float(l.split()[1]) for l in lines])
    model, vl = _splitmix_net()
    ri, rt = osweep.topk(model, vl, 3)
    check_topk(idx, t, ri, rt, lambda i: osweep.times_at(model, vl, i), TOL["fp32"], model["y_scale"])
