"""Model / space files (paper_2306_14011_b200.modelfile): versioned JSON model
round trip, error paths, and the paper's space from the range
shorthand (Table "Tuning Parameters")."""

import json
import os

import numpy as np
import pytest

import workloads
from oracle import mlp
from oracle import space as ospace
from paper_2306_14011_b200 import modelfile as mf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")


@pytest.mark.parametrize("stem", ["cfg2_14-128-128-1", "cfg4_17-128-128-1_x8", "tiny_14-32-32-1"])
def test_model_round_trip_is_bit_exact(stem, tmp_path):
    m = workloads.load_model(stem)
    p = str(tmp_path / "m.json")
    mf.save_model(m, p, extra={"source": stem})
    r = mf.load_model(p)
    assert r["widths"] == m["widths"] and len(r["members"]) == len(m["members"])
    for a, c in zip(m["members"], r["members"]):
        assert all(np.array_equal(x, y) for x, y in zip(a["W"] + a["b"], c["W"] + c["b"]))
    for key in ("x_shift", "x_scale", "const_features"):
        assert np.array_equal(np.asarray(m[key], np.float64), r[key])
    assert (r["y_mean"], r["y_scale"]) == (m["y_mean"], m["y_scale"])
    X = workloads.predict_rows(workloads.space("cfg2"), 500, seed=1)
    if m["widths"][0] == 14:  # save -> load -> predict equals the original bitwise (SPEC S:258 example)
        assert np.array_equal(mlp.predict(m, X), mlp.predict(r, X))


def test_model_file_errors(tmp_path):
    m = workloads.load_model("tiny_14-32-32-1")
    text = mf.model_to_json(m)
    with pytest.raises(mf.ModelFileError, match="corrupt"):
        mf.model_from_json(text[: len(text) // 2])          # truncated
    doc = json.loads(text)
    doc["format_version"] = 2
    with pytest.raises(mf.ModelFileError, match="version"):
        mf.model_from_json(json.dumps(doc))
    doc = json.loads(text)
    doc["members"][0]["W"][1] = doc["members"][0]["W"][1][:-1]
    with pytest.raises(mf.ModelFileError, match="shape"):
        mf.model_from_json(json.dumps(doc))
    with pytest.raises(mf.ModelFileError):
        mf.model_from_json(json.dumps({"format": "something else"}))


def test_paper_space_from_range_shorthand():
    names, vl = mf.space_from_json(mf.PAPER_SPACE_JSON)
    assert len(names) == 14 and names[0] == "xi_limiter_gang" and names[1] == "xi_limiter_vector"
    assert vl == [[float(v) for v in l] for l in workloads.space("paper")]
    paper = json.load(open(GOLDEN))
    assert vl[0] == [float(v) for v in paper["gang_values"]["value"]]
    assert vl[1] == [float(v) for v in paper["vector_values"]["value"]]
    assert ospace.cardinality([len(v) for v in vl]) == paper["search_space_size"]["value"]


def test_space_file_validation():
    bad = {"parameters": [{"name": "g", "values": [4, 2]}]}
    with pytest.raises(mf.ModelFileError, match="increasing"):
        mf.space_from_json(json.dumps(bad))
    with pytest.raises(mf.ModelFileError):
        mf.space_from_json(json.dumps({"parameters": [{"name": "g", "range": {"start": 5, "stop": 1, "step": 1}}]}))
    names, vl = mf.space_from_json(json.dumps({"parameters": [{"name": "v", "range": {"start": 32, "stop": 384,
                                                                                       "step": 32}}]}))
    assert vl == [[32.0 * i for i in range(1, 13)]]
