"""GPU parity of the elementwise / stencil primitives against the oracle.

Mirrors proj/tests/test_kernels.cpp (same seeds and shapes, same splitmix64
streams) and adds size sweeps over word-boundary widths.  Every comparison is
bit-exact.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import (CmpOp, DeviceImage, ImageBuffer, PixelKind, RunError, kernels,
                                   mask)

pytestmark = pytest.mark.gpu


def B(a):
    a = np.asarray(a, np.uint8)
    return ImageBuffer(a.shape[1], a.shape[0], PixelKind.Bool, a)


def U(a):
    a = np.asarray(a, np.uint16)
    return ImageBuffer(a.shape[1], a.shape[0], PixelKind.U16, a)


def all_of(w, h, v):
    return B(np.full((h, w), 1 if v else 0, np.uint8))


def rm(w, h, d, rng):
    return O.random_mask(w, h, d, rng)


# ---- test_kernels.cpp:26-41 -------------------------------------------------
def test_logical_not_basics(dev):
    assert kernels.logicalNot(all_of(4, 4, True)) == all_of(4, 4, False)
    checker = mask("x.x./.x.x/x.x./.x.x")
    inv = mask(".x.x/x.x./.x.x/x.x.")
    assert kernels.logicalNot(checker) == inv
    rng = O.Rng(5)
    for _ in range(50):
        a = B(rm(9, 7, rng.unit(), rng))
        assert kernels.logicalNot(kernels.logicalNot(a)) == a


# ---- test_kernels.cpp:43-58 -------------------------------------------------
def test_and_or_basics_and_oracle(dev):
    rng = O.Rng(6)
    a = rm(8, 8, 0.5, rng)
    assert kernels.logicalAnd(B(a), all_of(8, 8, True)) == B(a)
    assert kernels.logicalOr(B(a), kernels.logicalNot(B(a))) == all_of(8, 8, True)
    b = rm(8, 8, 0.5, rng)
    assert np.array_equal(kernels.logicalAnd(B(a), B(b)).data, a & b)
    assert np.array_equal(kernels.logicalOr(B(a), B(b)).data, a | b)


def test_binary_kernels_reject_mismatched_dimensions(dev):
    a, b = ImageBuffer(4, 4, PixelKind.Bool), ImageBuffer(5, 4, PixelKind.Bool)
    with pytest.raises(RunError, match="dimension mismatch"):
        kernels.logicalAnd(a, b)
    with pytest.raises(RunError):
        kernels.logicalOr(a, b)


# ---- test_kernels.cpp:69-97 -------------------------------------------------
def test_threshold_comparisons(dev):
    img = U([[62257, 62258, 62259]])
    gt = kernels.threshold(CmpOp.Gt, img, 62258)
    assert not gt.boolAt(0, 0) and not gt.boolAt(0, 1) and gt.boolAt(0, 2)
    assert kernels.threshold(CmpOp.Ge, img, 0) == all_of(3, 1, True)
    lt = kernels.threshold(CmpOp.Lt, img, 62258)
    assert lt.boolAt(0, 0) and not lt.boolAt(0, 1)
    le = kernels.threshold(CmpOp.Le, img, 62258)
    assert le.boolAt(0, 1) and not le.boolAt(0, 2)
    assert kernels.threshold(CmpOp.Lt, img, 70000) == all_of(3, 1, True)
    assert kernels.threshold(CmpOp.Gt, img, 70000) == all_of(3, 1, False)


def test_threshold_equality_on_a_ramp(dev):
    ramp = np.array([[c * 1000 + r for c in range(64)] for r in range(4)], np.uint16)
    eq = kernels.threshold(CmpOp.Eq, U(ramp), 56360)
    assert np.array_equal(eq.data, (ramp == 56360).astype(np.uint8))
    assert kernels.threshold(CmpOp.Eq, U(ramp), 56360.5) == all_of(64, 4, False)
    with pytest.raises(RunError):
        kernels.threshold(CmpOp.Gt, all_of(2, 2, True), 1)


@pytest.mark.parametrize("n", [0, 1, 0.5, -0.5, 62258, 62258.25, 56360.5, 65535, 65535.5,
                               70000, -1e300, 1e300, math.inf, -math.inf, math.nan, -0.0])
def test_threshold_every_op_matches_oracle(dev, n):
    rng = np.random.default_rng(7)
    img = rng.integers(0, 65536, (37, 101), dtype=np.uint16)
    img[0, :6] = [0, 1, 65535, 62258, 62259, 56360]
    for op in range(5):
        got = kernels.threshold(CmpOp(op), U(img), n).data
        assert np.array_equal(got, O.threshold(op, img, n)), (op, n)


# ---- test_kernels.cpp:99-113 ------------------------------------------------
def test_dilate_examples(dev):
    assert kernels.dilate(all_of(5, 5, False)) == all_of(5, 5, False)
    assert kernels.dilate(mask(".../.x./...")) == all_of(3, 3, True)
    corner = mask("x..../...../...../...../.....")
    expect = mask("xx.../xx.../...../...../.....")
    assert kernels.dilate(corner) == expect


def test_dilate_matches_window_scan_oracle(dev):
    rng = O.Rng(7)
    for _ in range(100):
        a = rm(11, 9, rng.unit(), rng)
        assert np.array_equal(kernels.dilate(B(a)).data, O.dilate(a))


def test_dilate_algebra(dev):
    rng = O.Rng(8)
    for _ in range(100):
        a = B(rm(10, 10, rng.unit() * 0.8, rng))
        b = B(rm(10, 10, rng.unit() * 0.8, rng))
        da, db = kernels.dilate(a), kernels.dilate(b)
        ab = kernels.logicalOr(a, b)
        assert kernels.logicalOr(a, da) == da
        dab = kernels.dilate(ab)
        assert kernels.logicalOr(da, dab) == dab
        assert dab == kernels.logicalOr(da, db)


def test_de_morgan(dev):
    rng = O.Rng(9)
    for _ in range(100):
        a = B(rm(9, 9, rng.unit(), rng))
        b = B(rm(9, 9, rng.unit(), rng))
        lhs = kernels.logicalNot(kernels.logicalAnd(a, b))
        rhs = kernels.logicalOr(kernels.logicalNot(a), kernels.logicalNot(b))
        assert lhs == rhs


def test_count_true(dev):
    assert kernels.countTrue(all_of(4, 5, False)) == 0
    assert kernels.countTrue(all_of(4, 5, True)) == 20
    rng = O.Rng(10)
    a = rm(31, 17, 0.3, rng)
    assert kernels.countTrue(B(a)) == int(a.sum())


# ---- size sweeps: word boundaries, thin shapes, the config widths ------------
SHAPES = [(1, 1), (1, 7), (7, 1), (31, 3), (32, 5), (33, 5), (63, 2), (64, 3), (65, 4),
          (100, 9), (127, 13), (128, 128), (129, 3), (240, 240), (255, 17), (256, 256),
          (257, 9), (1000, 3), (3, 700), (2049, 5), (4096, 4)]


@pytest.mark.parametrize("w,h", SHAPES)
def test_elementwise_and_stencils_sweep(dev, w, h):
    rng = O.Rng(w * 1000 + h)
    for d in (0.05, 0.5, 0.95):
        a = rm(w, h, d, rng)
        b = rm(w, h, 0.5, rng)
        A, Bb = B(a), B(b)
        assert np.array_equal(kernels.logicalNot(A).data, O.logical_not(a))
        assert np.array_equal(kernels.logicalAnd(A, Bb).data, O.logical_and(a, b))
        assert np.array_equal(kernels.logicalOr(A, Bb).data, O.logical_or(a, b))
        assert np.array_equal(kernels.dilate(A).data, O.dilate(a))
        assert np.array_equal(kernels.erode(A).data, O.erode(a))
        assert kernels.countTrue(A) == O.count_true(a)
        img = (rng.next() % 65536 + np.arange(w * h, dtype=np.uint64).reshape(h, w) * 7919
               ) % 65536
        img = img.astype(np.uint16)
        n = float(rng.below(65536))
        for op in range(5):
            assert np.array_equal(kernels.threshold(CmpOp(op), U(img), n).data,
                                  O.threshold(op, img, n))


@pytest.mark.parametrize("w,h", [(11, 9), (64, 64), (100, 37), (240, 240), (1031, 77)])
@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 11])
def test_near_k_and_interior_k_equal_repeated_application(dev, w, h, k):
    rng = O.Rng(w + h + k)
    a = rm(w, h, 0.03 if k > 2 else 0.2, rng)
    exp_d, exp_e = a, rm(w, h, 0.97, rng)
    e_in = exp_e.copy()
    for _ in range(k):
        exp_d = O.dilate(exp_d)
        exp_e = O.erode(exp_e)
    assert np.array_equal(kernels.dilateK(B(a), k).data, exp_d)
    assert np.array_equal(kernels.erodeK(B(e_in), k).data, exp_e)


def test_interior_border_is_inside(dev):
    # interior(all-true) = all-true (tests/test_reach.cpp:120)
    assert kernels.erode(all_of(5, 5, True)) == all_of(5, 5, True)
    assert kernels.erode(all_of(70, 3, True)) == all_of(70, 3, True)


def test_device_images_stay_on_device(dev):
    rng = O.Rng(99)
    a = rm(300, 200, 0.4, rng)
    da = DeviceImage.upload(a, PixelKind.Bool, dev)
    r = kernels.dilate(kernels.logicalNot(da))
    assert isinstance(r, DeviceImage)
    assert np.array_equal(r.numpy(), O.dilate(O.logical_not(a)))


def test_batched_slices(dev):
    rng = O.Rng(123)
    a = np.stack([rm(240, 240, 0.3 + 0.01 * i, rng) for i in range(5)])
    da = DeviceImage.upload(a, PixelKind.Bool, dev)
    got = kernels.dilate(da).numpy()
    for i in range(5):
        assert np.array_equal(got[i], O.dilate(a[i]))
    assert kernels.countTrue(da) == [int(x.sum()) for x in a]


def test_u16_coerces_to_mask_where_booleans_are_expected(dev):
    # executor.cpp:43-50 / test_executor.cpp:204-218 -- coercion is the evalTask
    # contract, exposed by the C ABI; the kernels:: mirror keeps requireBool.
    import ctypes as C
    from paper_2010_07284_b200 import _lib
    img = np.array([[0, 1, 40000, 0]], np.uint16)
    du = DeviceImage.upload(img, PixelKind.U16, dev)
    out = (C.c_int64 * 1)()
    assert _lib.load().slcs_volume(dev.handle, du.handle, out) == 0
    assert out[0] == 2
    with pytest.raises(RunError, match="expects a boolean image, got u16"):
        kernels.logicalNot(du)


def test_device_random_mask_matches_reference_stream(dev):
    from paper_2010_07284_b200.pixlog import random_mask_device
    for (w, h, d, seed) in [(37, 19, 0.5, 7), (300, 200, 0.41, 1), (64, 64, 0.05, 2)]:
        full = O.random_mask(w, h, d, O.Rng(seed))
        assert np.array_equal(random_mask_device(w, h, d, seed, 0, dev).numpy(), full)
        # a band starting mid-image continues the same stream
        band = random_mask_device(w, 7, d, seed, 5, dev).numpy()
        assert np.array_equal(band, full[5:12])


def test_volume_async_writes_device_counts(dev):
    # slcs_volume_async: counts land in device memory in stream order, and the
    # self-resetting accumulators give the same count on every call
    import ctypes as C

    import torch

    from paper_2010_07284_b200 import _lib
    rng = O.Rng(77)
    a = np.stack([O.random_mask(333, 211, d, rng) for d in (0.1, 0.5, 0.9)])
    img = DeviceImage.upload(a, PixelKind.Bool, dev)
    out = torch.zeros(3, dtype=torch.int64, device="cuda:0")
    lib = _lib.load()
    for _ in range(3):
        assert lib.slcs_volume_async(dev.handle, img.handle, C.c_void_p(out.data_ptr())) == 0
        dev.synchronize()
        assert out.cpu().tolist() == [int(x.sum()) for x in a]


@pytest.mark.parametrize("w,h,batch", [(4096, 515, 1), (4129, 600, 1), (8192 + 7, 257, 1),
                                       (4096, 130, 4), (16384, 64, 9)])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_wide_images_bulk_slab_near(dev, w, h, batch, k):
    # rows >= 4096 px take the bulk-async slab kernel (one cp.async.bulk per slab,
    # identity rows at the image edges, slabs crossing slice boundaries in a batch)
    rng = O.Rng(w * 7 + h + k + batch)
    a = np.stack([rm(w, h, 0.02, rng) for _ in range(batch)])
    e = np.stack([rm(w, h, 0.98, rng) for _ in range(batch)])
    got_d = kernels.dilateK(DeviceImage.upload(a, PixelKind.Bool, dev), k).numpy().reshape(a.shape)
    got_e = kernels.erodeK(DeviceImage.upload(e, PixelKind.Bool, dev), k).numpy().reshape(e.shape)
    for i in range(batch):
        ed, ee = a[i], e[i]
        for _ in range(k):
            ed, ee = O.dilate(ed), O.erode(ee)
        assert np.array_equal(got_d[i], ed)
        assert np.array_equal(got_e[i], ee)


@pytest.mark.parametrize("shape", [(1, 128, 1), (3, 17, 256), (2, 5, 1024), (1, 9, 4096),
                                   (1, 8, 160), (2, 3, 100)])
def test_bool_upload_pack_round_trip(dev, shape):
    # 1 B/px -> bit-packed upload: the vectorised 16-byte path (rows of a multiple of
    # 128 px) and the generic path must agree with the bytes (any nonzero is true)
    b, h, w = shape
    rng = np.random.default_rng(b * 1000 + h * 10 + w)
    a = rng.integers(0, 4, size=(b, h, w), dtype=np.uint8) * rng.integers(0, 2, size=(b, h, w),
                                                                          dtype=np.uint8)
    arr = a[0] if b == 1 else a
    img = DeviceImage.upload(arr, PixelKind.Bool)
    got = img.numpy()
    assert np.array_equal(got, (arr != 0).astype(np.uint8))
    want = [int((s_ != 0).sum()) for s_ in a]
    assert kernels.countTrue(img) == (want[0] if b == 1 else want)
