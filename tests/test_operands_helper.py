"""CPU pins of the operand-row expectation used by the decoded-tuple parity test
(tests/operands.py): its fp32 / fp16 / bf16 rounding against numpy and hand
values, and the row layout on hand-decoded configs."""

from fractions import Fraction

import numpy as np

import workloads
from tests import operands as ops


def test_round_f32_matches_numpy_on_doubles():
    rng = np.random.default_rng(3)
    for x in np.concatenate([rng.normal(0, 2, 2000), rng.uniform(-1e-3, 1e-3, 500)]):
        assert ops.round_f32(Fraction(float(x))) == np.float32(x)


def test_round_f32_ties_to_even():
    one = Fraction(1)
    ulp = Fraction(1, 2 ** 23)
    assert ops.round_f32(one + ulp / 2) == np.float32(1.0)              # tie -> even (1.0)
    assert ops.round_f32(one + ulp + ulp / 2) == np.float32(1.0 + 2 * 2.0 ** -23)  # tie -> even (odd + half)
    assert ops.round_f32(-(one + ulp / 2 + Fraction(1, 2 ** 40))) == np.float32(-(1.0 + 2.0 ** -23))


def test_16bit_roundings_hand_values():
    assert ops.f16_bits(np.float32(1.0)) == 0x3C00 and ops.bf16_bits(np.float32(1.0)) == 0x3F80
    assert ops.f16_bits(np.float32(-2.0)) == 0xC000 and ops.bf16_bits(np.float32(-2.0)) == 0xC000
    assert ops.f16_bits(np.float32(65504.0)) == 0x7BFF
    assert ops.f16_bits(np.float32(1.0 + 2.0 ** -11)) == 0x3C00          # tie -> even
    assert ops.f16_bits(np.float32(1.0 + 3 * 2.0 ** -11)) == 0x3C02      # tie -> even (up)
    assert ops.bf16_bits(np.float32(1.0 + 2.0 ** -8)) == 0x3F80          # tie -> even
    assert ops.bf16_bits(np.float32(1.0 + 3 * 2.0 ** -8)) == 0x3F82
    # 3xFP16 lo: z - hi is exact and small
    z = np.float32(0.1)
    h = ops.f16_bits(z)
    lo = np.float32(z - ops.f16_value(h))
    assert float(ops.f16_value(h)) + float(lo) == float(z)


def test_expected_rows_layout_on_hand_decoded_configs():
    vl = [[1, 3], [10, 20, 30], [5, 7]]
    model = dict(x_shift=np.array([2.0, 20.0, 6.0]), x_scale=np.array([1.0, 10.0, 1.0]))
    # I = 0 -> (1, 10, 5) -> z = (-1, -1, -1); I = 11 -> digits (1, 2, 1) -> (3, 30, 7) -> (1, 1, 1)
    rows = ops.expected_rows(model, vl, [0, 11], "fp16")
    m1, p1, one = 0xBC00, 0x3C00, 0x3C00
    assert rows[0, 0] == m1 | (m1 << 16) and rows[0, 1] == m1 | (one << 16)   # slot 3 = 1.0 (bias)
    assert rows[1, 0] == p1 | (p1 << 16) and rows[1, 1] == p1 | (one << 16)
    assert not rows[:, 2:].any()
    # I = 4 -> digits (0, 2, 0): z = (-1, 1, -1)
    r = ops.expected_rows(model, vl, [4], "bf16")[0]
    assert r[0] == 0xBF80 | (0x3F80 << 16) and r[1] == 0xBF80 | (0x3F80 << 16)


def test_expected_rows_3xfp16_reconstructs_z():
    vl = workloads.space("cfg5")
    model = workloads.load_model("cfg5_14-128-128-1")
    rows = ops.expected_rows(model, vl, np.arange(0, 13492928512, 987654321, dtype=np.uint64), "fp32")
    hi = np.stack([rows[:, :8] & 0xFFFF, rows[:, :8] >> 16], axis=2).reshape(-1, 16)[:, :14]
    lo = np.stack([rows[:, 8:] & 0xFFFF, rows[:, 8:] >> 16], axis=2).reshape(-1, 16)[:, :14]
    z = hi.astype(np.uint16).view(np.float16).astype(np.float64) + lo.astype(np.uint16).view(np.float16).astype(np.float64)
    from oracle import space
    d = space.decode(np.arange(0, 13492928512, 987654321, dtype=np.uint64), workloads.radices("cfg5"))
    x = space.values_of(d, vl)
    zt = (x - model["x_shift"][:14]) / model["x_scale"][:14]
    assert np.max(np.abs(z - zt)) < 1e-6 * np.max(np.abs(zt))
