"""Host-side hi/lo operand splits for the three-pass tensor-core expansion.

TF32: hi = x rounded to a 10-bit mantissa (kept in a float32 container, the
tensor core reads only the TF32 bits), lo = x - hi in float32.
F16:  hi = half(x), lo = half(x - hi); callers scale rows/columns by powers of
two so |x| <= 1 (subnormal lo parts keep ~2^-25 absolute accuracy).
"""
from __future__ import annotations


def _tf32_round(x32):
    import torch
    bits = x32.view(torch.int32)
    # round to nearest (ties away) at mantissa bit 13, then clear the low 13 bits
    r = (bits + 0x1000) & ~0x1FFF
    return r.view(torch.float32)


def split_tf32(x):
    import torch
    x64 = x.double()
    x32 = x64.float()
    hi = _tf32_round(x32.clone())
    lo = (x64 - hi.double()).float()
    return hi.contiguous(), lo.contiguous()


def split_f16(x):
    import torch
    x64 = x.double()
    hi = x64.half()
    lo = (x64 - hi.double()).half()
    return hi.contiguous(), lo.contiguous()
