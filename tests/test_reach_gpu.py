"""GPU parity of reach and the stdlib derived operators.

Mirrors proj/tests/test_reach.cpp (same seeds/shapes; BFS path oracle and the
touch/grow/surrounded oracles), then sweeps the large-image tiled path.
"""
import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import (DeviceImage, ImageBuffer, PixelKind, RunError, grow, interior,
                                   kernels, mask, reach, surrounded, touch)

pytestmark = pytest.mark.gpu


def B(a):
    a = np.asarray(a, np.uint8)
    return ImageBuffer(a.shape[1], a.shape[0], PixelKind.Bool, a)


def all_true(w, h):
    return B(np.ones((h, w), np.uint8))


def empty(w, h):
    return B(np.zeros((h, w), np.uint8))


def test_reach_includes_the_target(dev):
    rng = O.Rng(41)
    for _ in range(20):
        t = B(O.random_mask(10, 10, 0.3, rng))
        u = B(O.random_mask(10, 10, 0.3, rng))
        r = reach(t, u)
        assert kernels.logicalOr(t, r) == r


def test_1x5_row(dev):
    t, u = mask("....x"), mask("..xx.")
    r = reach(t, u)
    assert not r.boolAt(0, 0)
    assert all(r.boolAt(0, c) for c in range(1, 5))
    assert np.array_equal(r.data, O.reach_bfs(t.data, u.data))


def test_reach_all_true_empty(dev):
    assert reach(all_true(6, 4), empty(6, 4)) == all_true(6, 4)


def test_reach_empty_anything(dev):
    rng = O.Rng(42)
    u = B(O.random_mask(8, 8, 0.6, rng))
    assert reach(empty(8, 8), u) == empty(8, 8)


def test_reach_equals_bfs_oracle_on_random_pairs(dev):
    rng = O.Rng(43)
    for i in range(60):
        t = O.random_mask(32, 32, 0.05 + rng.unit() * 0.3, rng)
        u = O.random_mask(32, 32, 0.2 + rng.unit() * 0.6, rng)
        assert np.array_equal(reach(B(t), B(u)).data, O.reach_bfs(t, u)), i


def test_reach_monotone(dev):
    rng = O.Rng(44)
    for _ in range(25):
        t1 = O.random_mask(12, 12, 0.2, rng)
        t2 = t1 | O.random_mask(12, 12, 0.2, rng)
        u1 = O.random_mask(12, 12, 0.3, rng)
        u2 = u1 | O.random_mask(12, 12, 0.3, rng)
        r11, r21, r12 = (reach(B(t1), B(u1)).data, reach(B(t2), B(u1)).data,
                         reach(B(t1), B(u2)).data)
        assert ((r11 | r21) == r21).all() and ((r11 | r12) == r12).all()


def test_reach_rejects_mismatch_and_kinds(dev):
    with pytest.raises(RunError):
        reach(empty(4, 4), empty(5, 4))
    with pytest.raises(RunError, match="reach expects boolean images"):
        reach(ImageBuffer(4, 4, PixelKind.U16), empty(4, 4))


def test_interior_examples(dev):
    assert interior(all_true(5, 5)) == all_true(5, 5)
    assert interior(mask("...../..x../.....")) == empty(5, 3)
    sq = np.zeros((8, 8), np.uint8)
    sq[2:6, 2:6] = 1
    core = np.zeros((8, 8), np.uint8)
    core[3:5, 3:5] = 1
    assert np.array_equal(interior(B(sq)).data, core)


def test_interior_matches_erosion_oracle(dev):
    rng = O.Rng(45)
    for _ in range(50):
        a = O.random_mask(10, 10, rng.unit(), rng)
        assert np.array_equal(interior(B(a)).data, O.erode(a))


def test_touch_grow_surrounded_vs_oracles(dev):
    rng = O.Rng(46)
    for _ in range(10):
        a = O.random_mask(9, 9, 0.4, rng)
        assert np.array_equal(touch(B(a), B(a)).data, a)
    for _ in range(50):
        a = O.random_mask(14, 14, 0.35, rng)
        b = O.random_mask(14, 14, 0.2, rng)
        assert np.array_equal(touch(B(a), B(b)).data, O.touch(a, b))
    rng = O.Rng(47)
    for _ in range(50):
        a = O.random_mask(14, 14, 0.3, rng)
        b = O.random_mask(14, 14, 0.3, rng)
        assert np.array_equal(grow(B(a), B(b)).data, O.grow(a, b))
    rng = O.Rng(49)
    for _ in range(60):
        a = O.random_mask(12, 12, 0.3, rng)
        b = O.random_mask(12, 12, 0.3, rng)
        assert np.array_equal(surrounded(B(a), B(b)).data, O.surrounded(a, b))


def test_surrounded_ring(dev):
    a = mask("......./......./...x.../..xxx../...x.../......./.......")
    b = mask("......./..xxx../.xx.xx./.xx.xx./.xx.xx./..xxx../.......")
    ring = kernels.logicalAnd(b, kernels.logicalNot(a))
    assert surrounded(a, ring) == a
    assert surrounded(all_true(4, 4), empty(4, 4)) == all_true(4, 4)


SIZES = [(3, 3), (33, 31), (64, 64), (100, 257), (240, 240), (256, 256), (257, 257),
         (300, 200), (129, 513), (1000, 1000), (2048, 2048), (4096, 64)]


@pytest.mark.parametrize("w,h", SIZES)
@pytest.mark.parametrize("td,ud", [(0.01, 0.41), (0.05, 0.5), (0.002, 0.7), (0.2, 0.2)])
def test_reach_sweep_vs_oracle(dev, w, h, td, ud):
    rng = O.Rng(w * 3 + h * 5 + int(ud * 100))
    t = O.random_mask(w, h, td, rng)
    u = O.random_mask(w, h, ud, rng)
    assert np.array_equal(reach(B(t), B(u)).data, O.reach(t, u))


def test_reach_blob_noise_segmentation(dev):
    for n, seed in ((240, 100), (512, 1), (1024, 3)):
        img = O.blob_noise(n, n, seed)
        hI = (img > 62258).astype(np.uint8)
        vI = (img > 56360).astype(np.uint8)
        assert np.array_equal(grow(B(hI), B(vI)).data, O.grow(hI, vI))
        assert np.array_equal(surrounded(B(hI), B(vI)).data, O.surrounded(hI, vI))


def test_batched_reach(dev):
    rng = O.Rng(91)
    for w, h in ((240, 240), (300, 300)):
        t = np.stack([O.random_mask(w, h, 0.01, rng) for _ in range(3)])
        u = np.stack([O.random_mask(w, h, 0.45, rng) for _ in range(3)])
        got = reach(DeviceImage.upload(t, PixelKind.Bool, dev),
                    DeviceImage.upload(u, PixelKind.Bool, dev)).numpy()
        for i in range(3):
            assert np.array_equal(got[i], O.reach(t[i], u[i]))


def test_reach_beyond_fused_capacity_uses_tiled_kernels(dev):
    # 6144 x 4096 = 768 fused tiles (> 2 x 148 x 2 co-resident 512-thread CTAs):
    # the multi-kernel tiled path; 4096 x 4096 = 512 tiles stays fused
    for w, h in ((6144, 4096), (4096, 4096)):
        rng = O.Rng(w + h)
        t = O.random_mask(w, h, 0.002, rng)
        u = O.random_mask(w, h, 0.45, rng)
        assert np.array_equal(reach(B(t), B(u)).data, O.reach(t, u))
