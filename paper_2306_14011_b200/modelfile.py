"""Model and search-space files (host-side plumbing around the C ABI).

Model file: versioned JSON ("Model file: versioned JSON —
{format_version, layer_sizes, row-major weight arrays, biases, x_scaler
{means, stds}, y_scaler, ...}"), extended with ensemble members and constant
device features.  Doubles are written with 17 significant
digits, so a save -> load round trip is bit-exact and the loaded model predicts
bitwise-identically.  Weights are row-major fan_in x fan_out.

Space file: a list of {name, values | range: {start, stop, step}} (SPEC
"Space definition file", the range shorthand expanding at parse time; the
canonical example reproduces the paper's Table "Tuning Parameters",
PAPER.md:253-266).  Values must be strictly increasing and positive.
"""

from __future__ import annotations

import json
import math

import numpy as np

FORMAT = "paper_2306_14011_b200.model"
FORMAT_VERSION = 1


class ModelFileError(ValueError):
    """Corrupt, truncated or wrong-version model / space file."""


def _f(x) -> float:
    return float(x)


def model_to_json(model: dict, extra: dict | None = None) -> str:
    """The model record (see workloads.load_model) as versioned JSON."""
    members = [{"W": [np.asarray(w, np.float64).tolist() for w in m["W"]],
                "b": [np.asarray(v, np.float64).reshape(-1).tolist() for v in m["b"]]} for m in model["members"]]
    doc = {
        "format": FORMAT, "format_version": FORMAT_VERSION,
        "layer_sizes": [int(w) for w in model["widths"]],
        "members": members,
        "x_scaler": {"kind": model.get("x_scaler", "standard"),
                     "shift": np.asarray(model["x_shift"], np.float64).tolist(),
                     "scale": np.asarray(model["x_scale"], np.float64).tolist()},
        "y_scaler": {"mean": _f(model["y_mean"]), "scale": _f(model["y_scale"])},
        "const_features": np.asarray(model.get("const_features", []), np.float64).reshape(-1).tolist(),
    }
    if extra:
        doc["meta"] = extra
    # repr of a Python float is the shortest string that round-trips exactly
    return json.dumps(doc, allow_nan=True)


def model_from_json(text: str) -> dict:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ModelFileError(f"corrupt model file: {e}") from None
    if not isinstance(doc, dict) or doc.get("format") != FORMAT:
        raise ModelFileError("not a paper_2306_14011_b200 model file")
    if doc.get("format_version") != FORMAT_VERSION:
        raise ModelFileError(f"model format version {doc.get('format_version')} (this build reads {FORMAT_VERSION})")
    try:
        widths = [int(w) for w in doc["layer_sizes"]]
        members = []
        for m in doc["members"]:
            W = [np.asarray(w, np.float64) for w in m["W"]]
            b = [np.asarray(v, np.float64) for v in m["b"]]
            if len(W) != len(widths) - 1 or len(b) != len(W):
                raise ModelFileError("layer count does not match layer_sizes")
            for l, (w, v) in enumerate(zip(W, b)):
                if w.shape != (widths[l], widths[l + 1]) or v.shape != (widths[l + 1],):
                    raise ModelFileError(f"layer {l}: shape {w.shape} / {v.shape} vs layer_sizes")
            members.append(dict(W=W, b=b))
        if not members:
            raise ModelFileError("no members")
        xs = doc["x_scaler"]
        model = dict(widths=widths, members=members,
                     x_shift=np.asarray(xs["shift"], np.float64), x_scale=np.asarray(xs["scale"], np.float64),
                     y_mean=float(doc["y_scaler"]["mean"]), y_scale=float(doc["y_scaler"]["scale"]),
                     const_features=np.asarray(doc.get("const_features", []), np.float64),
                     x_scaler=str(xs.get("kind", "standard")))
    except (KeyError, TypeError, ValueError) as e:
        if isinstance(e, ModelFileError):
            raise
        raise ModelFileError(f"corrupt model file: {e!r}") from None
    if model["x_shift"].shape != (widths[0],) or model["x_scale"].shape != (widths[0],):
        raise ModelFileError("x_scaler size does not match the input width")
    return model


def save_model(model: dict, path: str, extra: dict | None = None) -> None:
    with open(path, "w") as f:
        f.write(model_to_json(model, extra))


def load_model(path: str) -> dict:
    with open(path) as f:
        return model_from_json(f.read())


def expand_values(entry: dict) -> list:
    """One parameter: explicit `values`, or `range: {start, stop, step}` with stop
    inclusive (Table "Tuning Parameters" lists e.g. 100 ... 1000 step 100)."""
    if "values" in entry:
        vals = [float(v) for v in entry["values"]]
    elif "range" in entry:
        r = entry["range"]
        start, stop, step = float(r["start"]), float(r["stop"]), float(r["step"])
        if not (step > 0 and stop >= start):
            raise ModelFileError(f"bad range {r}")
        n = int(math.floor((stop - start) / step + 1e-9)) + 1
        vals = [start + i * step for i in range(n)]
    else:
        raise ModelFileError(f"parameter {entry.get('name', '?')}: needs values or range")
    if not vals or any(v <= 0 for v in vals) or any(b <= a for a, b in zip(vals, vals[1:])):
        raise ModelFileError(f"parameter {entry.get('name', '?')}: values must be positive and strictly increasing")
    return vals


def space_from_json(text: str) -> tuple[list, list]:
    """(names, value lists) of a space file: {"parameters": [{name, values | range}, ...]}."""
    try:
        doc = json.loads(text)
        params = doc["parameters"]
    except (json.JSONDecodeError, KeyError, TypeError) as e:
        raise ModelFileError(f"corrupt space file: {e!r}") from None
    return [str(p.get("name", f"p{i}")) for i, p in enumerate(params)], [expand_values(p) for p in params]


# the paper's 14-parameter space (Table "Tuning Parameters"):
# gang counts 100 ... 1000 step 100, vector lengths 32 ... 384 step 32, per kernel
PAPER_KERNELS = ["xi_limiter", "eta_limiter", "xi_flux", "eta_flux", "source", "rhs", "update"]
PAPER_SPACE_JSON = json.dumps({"parameters": [
    p for k in PAPER_KERNELS for p in (
        {"name": f"{k}_gang", "range": {"start": 100, "stop": 1000, "step": 100}},
        {"name": f"{k}_vector", "range": {"start": 32, "stop": 384, "step": 32}})]}, indent=1)
