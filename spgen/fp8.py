"""FP8 (OCP e4m3) inputs for SURVEY 8(f) row f4 -- test/bench infrastructure.

Input preparation only (no method arithmetic): the generator's bf16 values,
multiplied by a power-of-two inverse scale (exact), are rounded to e4m3 codes
by torch's float8_e4m3fn conversion (round to nearest even).  The oracle
decodes the codes itself (oracle.ref.e4m3_to_f64); the CUDA path takes the
codes and the dequantisation scale 1/inv_scale.
"""
from __future__ import annotations

import torch

Q_INV_SCALE = 8.0      # q_scale = 1/8:  |Q| <= ~1.6 -> codes <= ~13
K_INV_SCALE = 16.0     # k_scale = 1/16: |K| <= ~5.6 -> codes <= ~90 (e4m3 max 448)


def to_e4m3_codes(x_bf16: torch.Tensor, inv_scale: float) -> torch.Tensor:
    """uint8 e4m3 codes of x * inv_scale (same device, same shape, contiguous)."""
    y = (x_bf16.float() * inv_scale).to(torch.float8_e4m3fn)
    return y.view(torch.uint8).contiguous()
