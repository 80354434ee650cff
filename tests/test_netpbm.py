"""Netpbm ingestion (API parity with the reference's load_image / write_pgm, imaging.py:78-194)."""

import numpy as np
import pytest

import paper_2510_14982_b200 as pz


def test_round_trips_and_luminance():
    rnd = np.random.default_rng(0)
    img = pz.GrayImage(rnd.integers(0, 256, (7, 5), dtype=np.uint8))
    for binary in (True, False):
        assert np.array_equal(pz.load_image(pz.write_pgm(img, binary)).pixels, img.pixels)
    assert pz.write_pgm(img).startswith(b"P5\n5 7\n255\n")
    rgb = np.array([[[255, 0, 0], [0, 255, 0], [0, 0, 255], [10, 20, 30]]], dtype=np.uint8)
    want = np.floor(0.299 * rgb[..., 0] + 0.587 * rgb[..., 1] + 0.114 * rgb[..., 2] + 0.5).astype(np.uint8)
    p6 = b"P6\n# colour\n4 1\n255\n" + rgb.tobytes()
    p3 = ("P3 4 1 255 " + " ".join(map(str, rgb.ravel().tolist()))).encode()
    assert np.array_equal(pz.load_image(p6).pixels, want) and np.array_equal(pz.load_image(p3).pixels, want)


@pytest.mark.parametrize("data,offset", [(b"P7 1 1 255 0", 0), (b"P5 0 1 255 \x00", 3), (b"P5 2 2 254 \x00", 7),
                                         (b"P5 2 2 255 \x00", 12), (b"P2 1 1 255 300", 11), (b"P2 2", 4)])
def test_errors_carry_offsets(data, offset):
    with pytest.raises(pz.ImageFormatError) as err:
        pz.load_image(data)
    assert err.value.offset == offset
