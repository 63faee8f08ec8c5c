"""Expected layer-1 operand rows of the sweep (parity of decoded tuples, a2 + a3).

The decoded tuple of config I comes from the ORACLE (``oracle.space.decode``,
parameter 0 most significant, G10); it is mapped to the operand the
tensor core reads through the rounding points DESIGN.md section 5 documents
(they are not the method's arithmetic: the method is z = (x - shift) / scale,
P:273, which the oracle evaluates in float64):

    z   = fp32 FMA of (fp32(x), fp32(1/scale), fp32(-shift/scale))   (one rounding)
    fp16 / bf16 operand = RNE(z);  3xFP16: hi = fp16(z), lo = fp16(z - hi)
    slot P = 1.0 (carries b_1), slots > P = 0; word w = slot 2w | slot 2w+1 << 16

The FMA is evaluated exactly with rationals and rounded once to fp32, so the
expectation does not depend on the host's or the GPU's FMA.  Nothing here
imports the CUDA path.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from oracle import space as ospace


def round_f32(q: Fraction) -> np.float32:
    """Round a rational to the nearest IEEE binary32 (ties to even), normal range."""
    if q == 0:
        return np.float32(0.0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    # 2^23 <= a / 2^(e - 23) < 2^24 after the adjustment
    while a >= Fraction(2) ** (e + 1):
        e += 1
    while a < Fraction(2) ** e:
        e -= 1
    if e < -126:
        raise ValueError("subnormal fp32 not expected for a normalised parameter")
    scaled = a / (Fraction(2) ** (e - 23))
    m = scaled.numerator // scaled.denominator
    r = scaled - m
    if r > Fraction(1, 2) or (r == Fraction(1, 2) and m % 2 == 1):
        m += 1
    return np.float32(sign * float(m) * 2.0 ** (e - 23))


def z_fp32(x: float, shift: float, scale: float) -> np.float32:
    """fp32 z of one value: fma(fp32(x), fp32(1/scale), fp32(-shift/scale)), one rounding."""
    scale = 1.0 if scale == 0.0 else scale
    xf = np.float32(x)
    zinv = np.float32(1.0 / scale)
    zc = np.float32(-shift / scale)
    return round_f32(Fraction(float(xf)) * Fraction(float(zinv)) + Fraction(float(zc)))


def f16_bits(v: np.float32) -> int:
    return int(np.array([v], np.float32).astype(np.float16).view(np.uint16)[0])  # RNE


def bf16_bits(v: np.float32) -> int:
    u = int(np.array([v], np.float32).view(np.uint32)[0])
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF


def f16_value(bits: int) -> np.float32:
    return np.float32(np.array([bits], np.uint16).view(np.float16)[0])


def slot_tables(model, value_lists, precision: str):
    """Per parameter j: (hi[r_j], lo[r_j]) 16-bit words of every value of list j."""
    P = len(value_lists)
    tabs = []
    for j in range(P):
        hi, lo = [], []
        for x in value_lists[j]:
            z = z_fp32(float(x), float(model["x_shift"][j]), float(model["x_scale"][j]))
            if precision == "bf16":
                hi.append(bf16_bits(z)); lo.append(0)
            elif precision == "fp16":
                hi.append(f16_bits(z)); lo.append(0)
            elif precision == "fp32":  # 3xFP16
                h = f16_bits(z)
                hi.append(h)
                lo.append(f16_bits(np.float32(z - f16_value(h))))  # exact in fp32
            else:
                raise ValueError(precision)
        tabs.append((np.array(hi, np.uint32), np.array(lo, np.uint32)))
    return tabs


def expected_rows(model, value_lists, idx, precision: str) -> np.ndarray:
    """uint32 [n, 16]: the operand rows the sweep must build for configs idx."""
    radices = [len(v) for v in value_lists]
    digits = ospace.decode(np.asarray(idx, np.uint64), radices)  # oracle decode (bit-exact target)
    P = len(value_lists)
    n = digits.shape[0]
    one = 0x3F80 if precision == "bf16" else 0x3C00
    hi = np.zeros((n, 16), np.uint32)
    lo = np.zeros((n, 16), np.uint32)
    tabs = slot_tables(model, value_lists, precision)
    for j in range(P):
        hi[:, j] = tabs[j][0][digits[:, j]]
        lo[:, j] = tabs[j][1][digits[:, j]]
    hi[:, P] = one
    out = np.zeros((n, 16), np.uint32)
    out[:, :8] = hi[:, 0::2] | (hi[:, 1::2] << 16)
    out[:, 8:] = lo[:, 0::2] | (lo[:, 1::2] << 16)
    return out
