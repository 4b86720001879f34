"""png_io (proj/src/png_io.cpp:30-144): PNG ingest/egress of the device path.

CPU tests pin the label colour hash against the restated reference; GPU tests
decode fixtures written with every filter type, colour type, both bit depths
and Adam7, save every image kind and read the files back with PIL, and check
the reference's error texts.
"""
import io

import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import (DeviceImage, ImageBuffer, PixelKind, RunError, decodePng,
                                   labelColor, loadPng, savePng)
from paper_2010_07284_b200.executor import RunOptions, run_text


def test_label_color_matches_reference_hash():
    for packed in [0, 1, 2, 3, 255, 65536, 123456, 0xFFFFFFFD, 0x7FFFFFFF] + list(range(5, 400, 7)):
        assert labelColor(packed) == O.label_color(packed), packed


CASES = [(16, 0, (0,)), (16, 0, (1,)), (16, 0, (2,)), (16, 0, (3,)), (16, 0, (4,)),
         (16, 0, (0, 1, 2, 3, 4)), (8, 0, (4, 2, 1)), (8, 2, (0, 1, 2, 3, 4)),
         (16, 2, (4, 3)), (8, 4, (1, 4)), (16, 4, (2,)), (8, 6, (3, 4, 0)), (16, 6, (1, 2))]


@pytest.mark.gpu
@pytest.mark.parametrize("interlace", [False, True])
@pytest.mark.parametrize("depth,color,filters", CASES)
def test_decode_matches_first_channel(dev, depth, color, filters, interlace):
    ch = {0: 1, 2: 3, 4: 2, 6: 4}[color]
    rng = np.random.default_rng(depth * 10 + color + len(filters))
    for h, w in ((1, 1), (7, 13), (37, 29), (64, 100)):
        a = rng.integers(0, 1 << depth, size=(h, w, ch), dtype=np.uint32)
        a = a.astype(np.uint16 if depth == 16 else np.uint8)
        data = O.png_encode(a, depth, color, filters, interlace, chunk_split=97)
        got = decodePng(data, dev).numpy()
        assert got.dtype == np.uint16 and got.shape == (h, w)
        assert np.array_equal(got, O.png_first_channel_u16(a, depth))


@pytest.mark.gpu
def test_decode_pil_written_files(dev, tmp_path):
    from PIL import Image
    rng = np.random.default_rng(5)
    g8 = rng.integers(0, 256, (50, 70), dtype=np.uint8)
    g16 = rng.integers(0, 65536, (50, 70), dtype=np.uint16)
    rgb = rng.integers(0, 256, (50, 70, 3), dtype=np.uint8)
    for arr, mode, want in ((g8, "L", g8.astype(np.uint16) * 257),
                            (g16, "I;16", g16),
                            (rgb, "RGB", rgb[..., 0].astype(np.uint16) * 257)):
        p = tmp_path / f"{mode.replace(';', '')}.png"
        Image.fromarray(arr).save(p)  # dtype/shape select L, I;16, RGB
        assert np.array_equal(loadPng(str(p), dev).numpy(), want), mode


@pytest.mark.gpu
def test_save_kinds_round_trip_through_pil(dev, tmp_path):
    from PIL import Image
    rng = np.random.default_rng(9)
    b = (rng.random((33, 65)) < 0.4).astype(np.uint8)
    u = rng.integers(0, 65536, (33, 65), dtype=np.uint16)
    lab = np.where(b > 0, rng.integers(1, 33 * 65, (33, 65)), 0).astype(np.uint32)
    savePng(str(tmp_path / "b.png"), ImageBuffer(65, 33, PixelKind.Bool, b), dev)
    savePng(str(tmp_path / "u.png"), ImageBuffer(65, 33, PixelKind.U16, u), dev)
    savePng(str(tmp_path / "l.png"), DeviceImage.upload(lab, PixelKind.LabelPair, dev), dev)
    ib = np.array(Image.open(tmp_path / "b.png"))
    assert np.array_equal(ib.astype(np.uint32), b.astype(np.uint32) * 65535)
    assert np.array_equal(np.array(Image.open(tmp_path / "u.png")).astype(np.uint16), u)
    il = np.array(Image.open(tmp_path / "l.png").convert("RGB"))
    want = np.array([[O.label_color(int(x)) for x in row] for row in lab], np.uint8)
    assert np.array_equal(il, want)
    # our own reader round-trips the u16 and bool files
    assert np.array_equal(loadPng(str(tmp_path / "u.png"), dev).numpy(), u)
    assert np.array_equal(loadPng(str(tmp_path / "b.png"), dev).numpy(), b.astype(np.uint16) * 65535)


@pytest.mark.gpu
def test_png_errors_match_reference_texts(dev, tmp_path):
    from PIL import Image
    pal = tmp_path / "pal.png"
    Image.fromarray(np.zeros((4, 4), np.uint8), "L").convert("P").save(pal)
    with pytest.raises(RunError, match=r"unsupported PNG: palette images are not supported \(.*pal.png\)"):
        loadPng(str(pal), dev)
    bw = tmp_path / "bw.png"
    Image.fromarray(np.zeros((4, 4), np.uint8), "L").convert("1").save(bw)
    with pytest.raises(RunError, match=r"unsupported PNG bit depth 1 \(.*bw.png\)"):
        loadPng(str(bw), dev)
    with pytest.raises(RunError, match="cannot open file for reading: "):
        loadPng(str(tmp_path / "missing.png"), dev)
    data = bytearray(O.png_encode(np.zeros((3, 3), np.uint16), 16, 0))
    data[20] ^= 0xFF  # inside IHDR -> CRC mismatch
    with pytest.raises(RunError, match="libpng: IHDR: CRC error"):
        decodePng(bytes(data), dev)
    with pytest.raises(RunError, match="libpng: Not a PNG file"):
        decodePng(b"GIF89a" + bytes(20), dev)


@pytest.mark.gpu
def test_spec_run_reads_and_writes_files(dev, tmp_path):
    # the reference's spec flow: load a PNG, evaluate, save a PNG (executor.cpp:78-86)
    from PIL import Image
    img = O.blob_noise(96, 80, 3)
    Image.fromarray(img).save(tmp_path / "input.png")  # uint16 -> 16-bit grey
    spec = ('load img = "input.png"\nlet a = img >. 30000\n'
            'save "out.png" grow(a, img >. 20000)\n')
    rep = run_text(spec, {}, RunOptions(baseDir=str(tmp_path)))
    assert rep.savedFiles == ["out.png"]
    a, b = O.threshold(0, img, 30000), O.threshold(0, img, 20000)
    want = O.grow(a, b).astype(np.uint32) * 65535
    assert np.array_equal(np.array(Image.open(tmp_path / "out.png")).astype(np.uint32), want)
