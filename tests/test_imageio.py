"""Ingest API on CPU (imageio.py:1-116 behaviour: the reference's test_imageio.py
cases as known answers) plus the pinned-batch loader's host side."""

import numpy as np
import pytest

from paper_2007_06483_b200 import ImageFormatError, decode_image, encode_image, load_stack
from paper_2007_06483_b200.imageio import decode_into, image_size


def _rgb(seed, w, h):
    return np.random.RandomState(seed).randint(0, 256, size=(h, w, 3), dtype=np.uint8)


def test_minimal_p6(tmp_path):
    p = tmp_path / "t.ppm"
    p.write_bytes(b"P6\n2 1\n255\n" + bytes([1, 2, 3, 4, 5, 6]))
    img = decode_image(p)
    assert img.shape == (1, 2, 3) and img.tobytes() == bytes([1, 2, 3, 4, 5, 6])


def test_header_comments_and_trailing_bytes(tmp_path):
    p = tmp_path / "c.ppm"
    p.write_bytes(b"P6\n# hand made\n2 1 # dims\n255\n" + bytes(range(6)) + b"extra")
    assert decode_image(p).tobytes() == bytes(range(6))


def test_long_header_past_sniff_block(tmp_path):
    p = tmp_path / "long.ppm"
    p.write_bytes(b"P6\n#" + b"x" * 5000 + b"\n3 2\n255\n" + bytes(18))
    assert decode_image(p).shape == (2, 3, 3)


@pytest.mark.parametrize("payload,match", [
    (b"P6\n2 1\n65535\n" + bytes(12), "maxval"),
    (b"P6\n4 4\n255\n" + bytes(10), "truncated"),
    (b"P5\n2 2\n255\n" + bytes(4), "P6"),
    (b"\x01\x02junkjunkjunk", "unrecognized"),
    (b"P6\n2 x\n255\n" + bytes(6), "malformed"),
    (b"P6\n0 1\n255\n", "dimensions"),
    (b"P6\n2 1\n255", "terminated|malformed"),
])
def test_bad_ppm(tmp_path, payload, match):
    p = tmp_path / "bad.ppm"
    p.write_bytes(payload)
    with pytest.raises(ImageFormatError, match=match):
        decode_image(p)
    assert issubclass(ImageFormatError, ValueError)


def test_missing_file(tmp_path):
    with pytest.raises(FileNotFoundError):
        decode_image(tmp_path / "nope.ppm")


def test_ppm_round_trip_and_size(tmp_path):
    img = _rgb(100, 17, 9)
    p = tmp_path / "rt.ppm"
    encode_image(img, p)
    assert p.stat().st_size == len(b"P6\n17 9\n255\n") + 17 * 9 * 3
    np.testing.assert_array_equal(decode_image(p), img)
    encode_image(decode_image(p), p)
    np.testing.assert_array_equal(decode_image(p), img)
    assert image_size(p) == (17, 9)


def test_png_round_trip_alpha_and_mode(tmp_path):
    from PIL import Image

    img = _rgb(101, 12, 15)
    p = tmp_path / "rt.png"
    encode_image(img, p)
    np.testing.assert_array_equal(decode_image(p), img)
    rgba = np.random.RandomState(102).randint(0, 256, size=(6, 6, 4), dtype=np.uint8)
    Image.fromarray(rgba, mode="RGBA").save(tmp_path / "a.png")
    np.testing.assert_array_equal(decode_image(tmp_path / "a.png"), rgba[:, :, :3])
    Image.fromarray(np.zeros((4, 4), np.uint8), mode="L").save(tmp_path / "g.png")
    with pytest.raises(ImageFormatError, match="mode"):
        decode_image(tmp_path / "g.png")
    (tmp_path / "bad.png").write_bytes(b"\x89PNG\r\n\x1a\n" + b"corrupted")
    with pytest.raises(ImageFormatError):
        decode_image(tmp_path / "bad.png")


def test_unknown_extension(tmp_path):
    with pytest.raises(ImageFormatError, match="extension"):
        encode_image(np.zeros((2, 2, 3), np.uint8), tmp_path / "img.bmp")


def test_decode_into_slot_and_load_stack(tmp_path):
    imgs = [_rgb(7 + i, 33, 20) for i in range(5)]
    paths = []
    for i, im in enumerate(imgs):
        p = tmp_path / (f"{i}.ppm" if i % 2 == 0 else f"{i}.png")
        encode_image(im, p)
        paths.append(p)
    slot = np.empty((20, 33, 3), np.uint8)
    np.testing.assert_array_equal(decode_into(paths[0], slot), imgs[0])
    with pytest.raises(ValueError, match="slot"):
        decode_into(paths[0], np.empty((20, 32, 3), np.uint8))
    batch = load_stack(paths, workers=3, pinned=False)
    assert batch.shape == (5, 20, 33, 3)
    for i in range(5):
        np.testing.assert_array_equal(batch[i], imgs[i])
    encode_image(_rgb(1, 32, 20), tmp_path / "odd.ppm")
    with pytest.raises(ValueError, match="is 32x20"):
        load_stack(paths + [tmp_path / "odd.ppm"], pinned=False)
