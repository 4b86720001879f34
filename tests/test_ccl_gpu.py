"""GPU parity of union-find CCL against the reference's canonical labels.

Mirrors the observable contract of proj/tests/test_ccl.cpp: labels equal
ccl::floodFillLabel (component max index + 1, ccl.hpp:52-60) bit-exactly,
plus the fixed known answers.  (initLabels / mainIteration / reconnect are
internals of the pointer-jumping algorithm that the union-find kernel does
not have -- DESIGN.md.)
"""
import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import (DeviceImage, ImageBuffer, PixelKind, RunError, ccl, mask,
                                   packLabel, maxvol)

pytestmark = pytest.mark.gpu


def B(a):
    a = np.asarray(a, np.uint8)
    return ImageBuffer(a.shape[1], a.shape[0], PixelKind.Bool, a)


def labels(a):
    return ccl.label(B(a)).data


def test_all_true_3x3_converges_to_the_max_coordinate(dev):
    l = labels(np.ones((3, 3), np.uint8))
    assert (l == packLabel(2, 2, 3)).all()


def test_concave_corner_l(dev):
    start = mask("xxxxx/x..../x..../x..../x....")
    l = ccl.label(start).data
    expect = packLabel(4, 0, 5)
    assert all(l[r, c] == expect for r in range(5) for c in range(5) if start.boolAt(r, c))
    assert l[1, 1] == 0


def test_label_equals_flood_fill_on_random_masks(dev):
    rng = O.Rng(36)
    for i in range(60):
        density = 0.1 + rng.unit() * 0.8
        start = O.random_mask(64, 64, density, rng)
        assert np.array_equal(labels(start), O.flood_fill_label(start)), (i, density)


def test_flood_fill_canonical_form_and_checkerboard(dev):
    l = ccl.label(mask("x.x/.../x.x")).data
    assert l[0, 0] == packLabel(0, 0, 3) and l[2, 2] == packLabel(2, 2, 3) and l[1, 1] == 0
    chk = np.fromfunction(lambda r, c: (r + c) % 2 == 0, (8, 8)).astype(np.uint8)
    cl = labels(chk)
    assert (cl[chk == 1] == packLabel(7, 7, 8)).all()


def test_rejects_non_boolean(dev):
    with pytest.raises(RunError, match="expects a boolean image"):
        ccl.label(ImageBuffer(4, 4, PixelKind.U16))


SIZES = [(1, 1), (1, 9), (9, 1), (2, 2), (3, 5), (33, 17), (63, 65), (64, 64), (65, 63),
         (127, 129), (240, 240), (256, 256), (257, 256), (256, 257), (300, 200), (513, 129),
         (1000, 1000), (4096, 70), (70, 4096), (2048, 2048)]


@pytest.mark.parametrize("w,h", SIZES)
@pytest.mark.parametrize("density", [0.2, 0.41, 0.5, 0.7, 0.97])
def test_label_sweep_vs_flood_fill(dev, w, h, density):
    rng = O.Rng(w * 7 + h * 13 + int(density * 100))
    a = O.random_mask(w, h, density, rng)
    assert np.array_equal(labels(a), O.flood_fill_label(a))


def test_concave_corner_fixture_128_and_1024(dev):
    R = O.Reference() if O.ref_available() else None
    for n in (128, 1024):
        img = (R.concave_corner(n, n) if R else None)
        if img is None:
            pytest.skip("reference fixture generator unavailable")
        a = (img > 0).astype(np.uint8)
        assert np.array_equal(labels(a), O.flood_fill_label(a))


def spiral_mask(n, spacing=6):
    """One long connected curve (a corrected spiral; synth.cpp:83-124 hangs)."""
    a = np.zeros((n, n), np.uint8)
    top, left, bot, right = 0, 0, n - 1, n - 1
    r, c = 0, 0
    while top <= bot and left <= right:
        a[top, left:right + 1] = 1
        a[top:bot + 1, right] = 1
        if bot - top < spacing or right - left < spacing:
            break
        a[bot, left + spacing:right + 1] = 1
        a[top + spacing:bot + 1, left + spacing] = 1
        top += spacing
        left += spacing
        bot -= spacing
        right -= spacing
        a[top, left - spacing:left + 1] = 1
    return a


@pytest.mark.parametrize("n", [64, 257, 1024, 2048])
def test_spiral_single_long_component(dev, n):
    a = spiral_mask(n)
    assert np.array_equal(labels(a), O.flood_fill_label(a))


def test_batched_labels(dev):
    rng = O.Rng(77)
    a = np.stack([O.random_mask(240, 240, 0.45, rng) for _ in range(4)])
    got = ccl.label(DeviceImage.upload(a, PixelKind.Bool, dev)).numpy()
    for i in range(4):
        assert np.array_equal(got[i], O.flood_fill_label(a[i]))


def test_batched_labels_large_path(dev):
    rng = O.Rng(78)
    a = np.stack([O.random_mask(300, 290, 0.45, rng) for _ in range(3)])
    got = ccl.label(DeviceImage.upload(a, PixelKind.Bool, dev)).numpy()
    for i in range(3):
        assert np.array_equal(got[i], O.flood_fill_label(a[i]))


# ---- maxvol (new opcode; oracle = floodFillLabel + size histogram) ---------------
@pytest.mark.parametrize("w,h", [(8, 8), (64, 64), (240, 240), (256, 256), (300, 301),
                                 (1024, 1024)])
@pytest.mark.parametrize("density", [0.0, 0.3, 0.45, 0.6])
def test_maxvol_vs_oracle(dev, w, h, density):
    rng = O.Rng(w + h + int(density * 10))
    a = O.random_mask(w, h, density, rng)
    assert np.array_equal(maxvol(B(a)).data, O.maxvol(a))


def test_maxvol_ties_keep_all_maxima(dev):
    m = mask("xx...xx/xx...xx/......./x......")
    got = maxvol(m).data
    assert np.array_equal(got, mask("xx...xx/xx...xx/......./.......").data)
    big = np.zeros((300, 300), np.uint8)
    big[10:20, 10:20] = 1
    big[100:110, 200:210] = 1
    big[250, 250] = 1
    assert np.array_equal(maxvol(B(big)).data, O.maxvol(big))


@pytest.mark.parametrize("w,h,n", [(256, 256, 60), (240, 240, 60), (600, 520, 25)])
def test_race_stress_many_masks(dev, w, h, n):
    """Union-find races show up as rare single-pixel errors: hammer them."""
    rng = O.Rng(9000 + w)
    for i in range(n):
        d = 0.35 + 0.3 * rng.unit()
        a = O.random_mask(w, h, d, rng)
        t = O.random_mask(w, h, 0.01, rng)
        da = DeviceImage.upload(a, PixelKind.Bool, dev)
        assert np.array_equal(ccl.label(da).numpy(), O.flood_fill_label(a)), (i, d)
        if i % 5 == 0:
            from paper_2010_07284_b200 import reach
            got = reach(DeviceImage.upload(t, PixelKind.Bool, dev), da).numpy()
            assert np.array_equal(got, O.reach(t, a)), (i, d)


@pytest.mark.parametrize("n,seed", [(512, 1), (2048, 3), (4096, 7)])
def test_generated_spirals_vs_flood_fill(dev, n, seed):
    # synth.spiral (corrected synth.cpp:83-124): one thin curve across every tile
    from paper_2010_07284_b200 import synth as S
    a = (S.spiral(n, n, seed) > 0).astype(np.uint8)
    assert np.array_equal(labels(a), O.flood_fill_label(a))
