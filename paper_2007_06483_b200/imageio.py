"""Image ingest: binary PPM (P6) and 8-bit PNG decode/encode (mirror of
mtbalign.imageio, imageio.py:1-116), plus the B200 ingest path of SURVEY
8(f)3: files decoded by a thread pool straight into one pinned host batch,
then uploaded image by image on a copy stream while the fused pipeline
already runs (K1 of image i starts when its copy lands; see
MtbEngine.align_fused_host and mtb_align_fused_ex).

Errors follow the reference: FileNotFoundError for a missing file,
ImageFormatError (a ValueError) for unsupported or malformed data, OSError
on write failures.  PPM is parsed here (the raster is read with one
`readinto` into its pinned slot, no intermediate copy); PNG goes through
Pillow and must be 8-bit RGB or RGBA (alpha dropped).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import _dev
from .image import validate_rgb

_PNG_MAGIC = b"\x89PNG\r\n\x1a\n"
_WS = b" \t\n\r\v\f"


class ImageFormatError(ValueError):
    """Unsupported or malformed image data."""


def _ppm_header(data: bytes, path) -> tuple[int, int, int]:
    """(width, height, raster offset) of a binary P6 header (imageio.py:22-65).

    Header integers are whitespace separated; '#' starts a comment that runs
    to the end of the line; exactly one whitespace byte ends the header.
    """
    vals = []
    i, n = 2, len(data)
    while len(vals) < 3:
        while i < n and data[i] in _WS:
            i += 1
        if i < n and data[i] == 0x23:   # '#'
            j = data.find(b"\n", i)
            i = n if j < 0 else j + 1
            continue
        j = i
        while j < n and data[j] not in _WS:
            j += 1
        tok = data[i:j]
        if not tok.isdigit():
            raise ImageFormatError(f"{path}: malformed PPM header token {tok!r}")
        vals.append(int(tok))
        i = j
    if i >= n or data[i] not in _WS:
        raise ImageFormatError(f"{path}: PPM header not terminated by whitespace")
    w, h, maxval = vals
    if maxval != 255:
        raise ImageFormatError(f"{path}: unsupported PPM maxval {maxval}; only 8-bit (255) is supported")
    if w < 1 or h < 1:
        raise ImageFormatError(f"{path}: invalid PPM dimensions {w}x{h}")
    return w, h, i + 1


def _sniff(path: Path) -> tuple[str, bytes]:
    if not path.is_file():
        raise FileNotFoundError(f"input image not found: {path}")
    with open(path, "rb") as f:
        head = f.read(4096)
    if head[:2] == b"P6":
        return "ppm", head
    if head[:8] == _PNG_MAGIC:
        return "png", head
    if head[:2] in (b"P1", b"P2", b"P3", b"P4", b"P5"):
        raise ImageFormatError(f"{path}: unsupported PNM variant; only binary P6 is supported")
    raise ImageFormatError(f"{path}: unrecognized image format")


def _ppm_geometry(path: Path, head: bytes) -> tuple[int, int, int]:
    try:
        return _ppm_header(head, path)
    except ImageFormatError:
        if len(head) < 4096:
            raise
    return _ppm_header(path.read_bytes(), path)   # header longer than the sniffed block


def _png_array(path: Path) -> np.ndarray:
    from PIL import Image, UnidentifiedImageError

    try:
        with Image.open(path) as img:
            if img.mode not in ("RGB", "RGBA"):
                raise ImageFormatError(f"{path}: unsupported PNG mode {img.mode!r}; only 8-bit RGB/RGBA is supported")
            arr = np.asarray(img, dtype=np.uint8)
    except UnidentifiedImageError as exc:
        raise ImageFormatError(f"{path}: not a decodable PNG file") from exc
    except OSError as exc:   # Pillow reports truncated / corrupt streams as OSError
        raise ImageFormatError(f"{path}: corrupt PNG data ({exc})") from exc
    return arr[:, :, :3]


def image_size(path) -> tuple[int, int]:
    """(width, height) of a PPM or PNG file without decoding the raster."""
    path = Path(path)
    kind, head = _sniff(path)
    if kind == "ppm":
        w, h, _ = _ppm_geometry(path, head)
        return w, h
    from PIL import Image, UnidentifiedImageError

    try:
        with Image.open(path) as img:
            return img.size
    except (UnidentifiedImageError, OSError) as exc:
        raise ImageFormatError(f"{path}: not a decodable PNG file") from exc


def decode_into(path, out: np.ndarray) -> np.ndarray:
    """Decode `path` into the preallocated (H, W, 3) uint8 array `out` (e.g.
    one image slot of a pinned batch); its shape must match the file."""
    path = Path(path)
    kind, head = _sniff(path)
    if kind == "ppm":
        w, h, start = _ppm_geometry(path, head)
        if out.shape != (h, w, 3):
            raise ValueError(f"{path}: image is {w}x{h}, slot is {out.shape[1]}x{out.shape[0]}")
        want = w * h * 3
        with open(path, "rb") as f:
            f.seek(start)
            got = f.readinto(memoryview(out.reshape(-1)))
        if got < want:
            raise ImageFormatError(f"{path}: truncated PPM data, expected {want} bytes, got {got}")
        return out
    arr = _png_array(path)
    if arr.shape != out.shape:
        raise ValueError(f"{path}: image is {arr.shape[1]}x{arr.shape[0]}, slot is {out.shape[1]}x{out.shape[0]}")
    out[...] = arr
    return out


def decode_image(path) -> np.ndarray:
    """Decode a PPM (binary P6, maxval 255) or PNG (8-bit RGB/RGBA) file (imageio.py:82-94)."""
    path = Path(path)
    kind, head = _sniff(path)
    if kind == "ppm":
        w, h, _ = _ppm_geometry(path, head)
        return decode_into(path, np.empty((h, w, 3), dtype=np.uint8))
    return np.ascontiguousarray(_png_array(path))


def encode_image(img: np.ndarray, path) -> None:
    """Write an RGB raster; the extension (.ppm / .png) selects the format (imageio.py:97-116)."""
    validate_rgb(img)
    path = Path(path)
    suffix = path.suffix.lower()
    if suffix == ".ppm":
        header = b"P6\n%d %d\n255\n" % (img.shape[1], img.shape[0])
        try:
            with open(path, "wb") as f:
                f.write(header)
                f.write(np.ascontiguousarray(img).data)
        except OSError as exc:
            raise OSError(f"failed to write {path}: {exc}") from exc
    elif suffix == ".png":
        from PIL import Image

        try:
            Image.fromarray(np.ascontiguousarray(img), mode="RGB").save(path, format="PNG")
        except OSError as exc:
            raise OSError(f"failed to write {path}: {exc}") from exc
    else:
        raise ImageFormatError(f"{path}: unsupported output extension {suffix!r}; use .ppm or .png")


def load_stack(paths, workers: int | None = None, pinned: bool = True):
    """Decode every file into ONE (N, H, W, 3) uint8 host batch (pinned when
    `pinned`, so its H2D copies run at full PCIe rate and asynchronously),
    `workers` files at a time.  All files must have the same size."""
    paths = [Path(p) for p in paths]
    if not paths:
        raise ValueError("no input images")
    w, h = image_size(paths[0])
    for p in paths[1:]:
        wp, hp = image_size(p)
        if (wp, hp) != (w, h):
            raise ValueError(f"{p} is {wp}x{hp} but {paths[0]} is {w}x{h}")
    if pinned:
        torch = _dev.torch_mod()
        batch = torch.empty((len(paths), h, w, 3), dtype=torch.uint8, pin_memory=True)
        view = batch.numpy()
    else:
        batch = view = np.empty((len(paths), h, w, 3), dtype=np.uint8)
    nw = workers or min(len(paths), os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=max(1, nw)) as ex:
        list(ex.map(lambda i: decode_into(paths[i], view[i]), range(len(paths))))
    return batch
