"""The end-to-end example (examples/autotune_end_to_end.py) on the GPU: train,
save / load the model file, sweep, and the returned configurations are the
oracle's best under the trained model (re-evaluated in float64)."""

import importlib.util
import os

import numpy as np
import pytest

from oracle import sweep as osweep
from tests.helpers import TOL, need_gpu, rel_err

pytestmark = pytest.mark.gpu


def test_example_end_to_end():
    need_gpu()
    path = os.path.join(os.path.dirname(os.path.dirname(__file__)), "examples", "autotune_end_to_end.py")
    spec = importlib.util.spec_from_file_location("example", path)
    ex = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ex)
    out = ex.main(["--n", "4000", "--epochs", "60", "--k", "5"])
    assert out["r2"] > 0.9
    tr = osweep.times_at(out["model"], out["vl"], out["idx"])
    assert rel_err(out["t"], tr, out["model"]["y_scale"]).max() <= TOL["fp32"]
    assert np.all(np.diff(out["t"]) >= 0)
