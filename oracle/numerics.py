"""Rounding emulation for the oracle (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

bf16 round-to-nearest-even of a value held in fp32 (SPEC.md:27-32, 50-58 numeric-core
"round_to"; §IV-A BF16 AMP). Used only at the rounding points listed
in DESIGN.md reading R20; everything else in the oracle stays in fp64.
"""
import numpy as np


def fp32(x):
    """Round to the nearest fp32 value (IEEE RNE), returned as float64."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def bf16(x):
    """RNE to bfloat16 of fp32(x); returned as float64 (exactly representable).

    Bit-level definition: keep the top 16 bits of the fp32 pattern after
    adding 0x7FFF + lsb (ties to even). Inputs are finite in every use here.
    """
    x32 = np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))
    u = x32.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def fp16(x):
    """RNE to IEEE binary16 of fp32(x) (subnormals kept, +-inf on overflow); returned as float64.
    PAPER.md:164 ("FP16 (half precision)" AMP); numpy's float32 -> float16 cast rounds to nearest even."""
    x32 = np.asarray(x, dtype=np.float64).astype(np.float32)
    with np.errstate(over="ignore"):   # overflow to +-inf is the defined result, not an error
        return x32.astype(np.float16).astype(np.float64)


def identity(x):
    return np.asarray(x, dtype=np.float64)


def rounder(precision: str):
    """Operand rounding for a GEMM operand at a DESIGN.md R20 rounding point."""
    if precision == "bf16":
        return bf16
    if precision == "fp16":
        return fp16
    if precision == "fp32":
        return identity
    raise ValueError(f"unknown precision {precision!r}")
