"""Decoded tuples of the SWEEP ITSELF, bit-exact (north star: "agree with the
oracle bit-exactly on decoded parameter tuples and config indices"; SURVEY
§8(a) a2 mixed-radix decode, a3 normalisation prologue).

The fused sweep kernel, in the launch configuration of the corresponding
sweep (its grid, slot stride and odometer), writes the layer-1 operand row it
built for every sampled config (surrogate_sweep_operands, MODE_A0).  Each row
must equal, bit for bit, the oracle's decoded tuple mapped through the
documented rounding points (tests/operands.py).  Whole-space launches are
sampled with a prime stride; ragged ends and windows near the top of the u64
range are dumped densely.
"""

import numpy as np
import pytest

import workloads
from tests import operands as ops
from tests.helpers import need_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    return need_gpu()


CASES = [
    # name, weights, precision, begin, end (None: |S|), stride
    ("tiny", "tiny_14-32-32-1", "fp32", 0, None, 1),            # 3xFP16 kernel, every config
    ("tiny", "random32", "fp16", 0, None, 1),                   # 16-bit kernel, H = 32
    ("cfg2", "cfg2_14-128-128-1", "fp16", 0, None, 997),        # headline kernel, whole space
    ("cfg2", "cfg2_14-128-128-1", "fp16", 170859375 - 4099, None, 1),  # ragged last tiles
    ("cfg2", "cfg2_14-128-128-1", "bf16", 0, None, 4099),
    ("cfg2", "cfg2_14-128-128-1", "fp32", 0, None, 1009),       # FP32 path (3-slot 3xFP16 kernel)
    ("cfg2", "cfg2_14-128-128-1", "fp32", 98_765_431, 98_765_431 + 300_007, 1),
    ("cfg5", "cfg5_14-128-128-1", "fp16", 0, None, 100_003),     # bench launch (1.35e10)
    ("cfg5", "cfg5_14-128-128-1", "fp16", 13492928512 - 70001, None, 1),
    ("cfg3", "cfg3_14-256-256-256-1", "fp16", 0, None, 10_007),  # CTA-pair kernel, whole space
    ("paper", "paper_14-128-128-1", "fp16", 358318080000000 - 65536 - 3, None, 1),
    ("paper", "paper_14-128-128-1", "fp16", 119439360000000, 119439360000000 + (1 << 24), 61),
]


@pytest.mark.parametrize("name,weights,prec,begin,end,stride", CASES)
def test_sweep_operands_bit_exact(pk, name, weights, prec, begin, end, stride):
    vl = workloads.space(name)
    model = (workloads.random_net(vl, [32, 32], seed=4) if weights == "random32"
             else workloads.load_model(weights))
    h = pk.Surrogate(0).load(model, prec)
    N = int(np.prod([len(v) for v in vl], dtype=object))
    end = N if end is None else end
    got = h.sweep_operands(vl, begin, end, stride).cpu().numpy().view(np.uint32)
    idx = np.arange(begin, end, stride, dtype=np.uint64)
    assert got.shape == (len(idx), 16)
    exp = ops.expected_rows(model, vl, idx, prec)
    bad = np.nonzero((got != exp).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first I = {int(idx[bad[0]])}: {got[bad[0]]} vs {exp[bad[0]]}"
