"""Synthetic misaligned exposure stacks, generated on the GPU.

Mirrors mtbalign.synth (pkg/src/mtbalign/synth.py:17-103): the base image is
displaced by the negated cumulative offset (fill 0) and passed through a
gain/gamma tone curve.  The random draws (offsets, gains, gammas) use the
same numpy Generator sequence as the reference, so a given seed yields the
same manifest and byte-identical images.  Used to feed parity tests and the
benchmark with inputs resident in HBM; not part of the alignment path.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .image import ShiftOffset, shift_rgb_device, validate_rgb

MIN_OVERLAP = 0.75
GAIN_RANGE = (0.5, 2.0)
GAMMA_RANGE = (0.7, 1.4)
MIN_BASE_SIZE = 64


def tone_lut(gain: float, gamma: float) -> np.ndarray:
    """256-entry curve clamp(round(255 * (gain * v / 255) ** (1 / gamma))) (synth.py:25-29)."""
    v = np.arange(256, dtype=np.float64) / 255.0
    return np.clip(np.round(255.0 * np.power(gain * v, 1.0 / gamma)), 0, 255).astype(np.uint8)


def apply_lut_device(img_dev, lut: np.ndarray, out=None):
    torch = _dev.torch_mod()
    lut_dev = torch.from_numpy(np.ascontiguousarray(lut, dtype=np.uint8)).to("cuda")
    if out is None:
        out = torch.empty_like(img_dev)
    _lib.call("mtb_apply_lut", _dev.ptr(img_dev), _dev.ptr(lut_dev), int(img_dev.numel()), _dev.ptr(out),
              _dev.stream())
    return out


def _check_overlap(off: ShiftOffset, w: int, h: int) -> None:
    left = (w - abs(off.dx)) * (h - abs(off.dy))
    if abs(off.dx) >= w or abs(off.dy) >= h or left < MIN_OVERLAP * w * h:
        raise ValueError(f"offset ({off.dx}, {off.dy}) keeps less than {MIN_OVERLAP:.0%} of a {w}x{h} base")


def draw_manifest(count: int, pairwise=None, seed: int = 0, max_shift: int = 16, gains=None, gammas=None):
    """The reference's draw order (synth.py:65-81): offsets, then gains, then gammas."""
    rng = np.random.default_rng(seed)
    if pairwise is None:
        pairwise = [ShiftOffset(int(rng.integers(-max_shift, max_shift + 1)),
                                int(rng.integers(-max_shift, max_shift + 1))) for _ in range(count - 1)]
    else:
        pairwise = [ShiftOffset(int(o[0]), int(o[1])) for o in pairwise]
        if len(pairwise) != count - 1:
            raise ValueError(f"need {count - 1} pairwise offsets, got {len(pairwise)}")
    if gains is None:
        gains = [float(rng.uniform(*GAIN_RANGE)) for _ in range(count)]
    if gammas is None:
        gammas = [float(rng.uniform(*GAMMA_RANGE)) for _ in range(count)]
    if len(gains) != count or len(gammas) != count:
        raise ValueError("one gain and one gamma per image are required")
    cumulative = [ShiftOffset(0, 0)]
    for off in pairwise:
        cumulative.append(cumulative[-1] + off)
    return pairwise, cumulative, list(gains), list(gammas)


def generate_stack(base, count: int, pairwise=None, seed: int = 0, max_shift: int = 16, gains=None, gammas=None):
    """`count` exposures of one base with known offsets (synth.py:45-103)."""
    validate_rgb(base)
    h, w = _dev.shape_of(base)[:2]
    if w < MIN_BASE_SIZE or h < MIN_BASE_SIZE:
        raise ValueError(f"base must be at least {MIN_BASE_SIZE}x{MIN_BASE_SIZE}; got {w}x{h}")
    if count < 2:
        raise ValueError("count must be >= 2")
    pairwise, cumulative, gains, gammas = draw_manifest(count, pairwise, seed, max_shift, gains, gammas)
    for cum in cumulative:
        _check_overlap(cum, w, h)
    torch = _dev.torch_mod()
    src = _dev.to_device(base)
    batch = src.unsqueeze(0).expand(count, h, w, 3).contiguous()
    displaced = shift_rgb_device(batch, [(-c.dx, -c.dy) for c in cumulative])
    out = torch.empty_like(displaced)
    for i in range(count):
        apply_lut_device(displaced[i], tone_lut(gains[i], gammas[i]), out=out[i])
    as_numpy = isinstance(base, np.ndarray)
    host = out.cpu().numpy() if as_numpy else out
    images = [host[i] for i in range(count)]
    manifest = {
        "count": count, "seed": seed, "max_shift": max_shift,
        "pairwise": [[o.dx, o.dy] for o in pairwise],
        "cumulative": [[o.dx, o.dy] for o in cumulative],
        "gains": gains, "gammas": gammas,
    }
    return images, manifest


def synthetic_gray_device(seed: int, width: int, height: int, cells: int = 12, noise: float = 10.0):
    """The engine_bench.py:22-35 field (coarse uniform grid, bilinear upsample,
    N(0, noise), round, clip) generated on the device.  Statistically the
    reference recipe; not bit-identical to its numpy draws."""
    torch = _dev.torch_mod()
    g = torch.Generator(device="cuda")
    g.manual_seed(int(seed))
    coarse = torch.rand((1, 1, cells, cells), generator=g, device="cuda", dtype=torch.float32) * 255.0
    up = torch.nn.functional.interpolate(coarse, size=(height, width), mode="bilinear", align_corners=True)[0, 0]
    up += torch.randn((height, width), generator=g, device="cuda", dtype=torch.float32) * noise
    return up.round_().clamp_(0, 255).to(torch.uint8)


def synthetic_rgb_device(seed: int, width: int, height: int):
    """(H, W, 3) base with three independent synthetic channels."""
    torch = _dev.torch_mod()
    return torch.stack([synthetic_gray_device(seed * 3 + c, width, height) for c in range(3)], dim=-1).contiguous()
