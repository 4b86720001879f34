"""GPU: the row-band path (bands.py) equals the single-image path bit-exactly.

N bands run on one GPU through LocalGroup (the same protocol a torch.distributed
job runs across GPUs: halo rows, border-row export, cross-band union-find,
flag hand-back, halo-exchanged closing near)."""
import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import DeviceImage, PixelKind, kernels, reach
from paper_2010_07284_b200.bands import (LocalGroup, band_rows, near_banded, reach_banded,
                                         volume_banded)

pytestmark = pytest.mark.gpu


def split(dev, a, world):
    h = a.shape[0]
    return [DeviceImage.upload(a[slice(*band_rows(h, world, r))], PixelKind.Bool, dev)
            for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("w,h,ud", [(600, 517, 0.5), (1000, 1000, 0.41), (300, 257, 0.7)])
def test_banded_reach_near_volume(dev, world, w, h, ud):
    rng = O.Rng(w + h + world)
    t = O.random_mask(w, h, 0.01, rng)
    u = O.random_mask(w, h, ud, rng)
    tb, ub = split(dev, t, world), split(dev, u, world)
    grp = LocalGroup(world)
    out = grp.run(lambda c, b: reach_banded(c, b[0], b[1]).numpy(), list(zip(tb, ub)))
    assert np.array_equal(np.concatenate(out), O.reach(t, u))
    near = grp.run(lambda c, b: near_banded(c, b, 2).numpy(), ub)
    assert np.array_equal(np.concatenate(near), O.dilate(O.dilate(u)))
    inter = grp.run(lambda c, b: near_banded(c, b, 1, erode=True).numpy(), ub)
    assert np.array_equal(np.concatenate(inter), O.erode(u))
    vol = grp.run(lambda c, b: volume_banded(c, b), ub)
    assert all(v == int(u.sum()) for v in vol)


def test_banded_reach_blob_giant_component(dev):
    img = O.blob_noise(1024, 1024, 1)
    t = O.threshold(0, img, 62258)
    u = O.threshold(0, img, 56360)
    for world in (2, 5):
        tb, ub = split(dev, t, world), split(dev, u, world)
        out = LocalGroup(world).run(lambda c, b: reach_banded(c, b[0], b[1]).numpy(),
                                    list(zip(tb, ub)))
        assert np.array_equal(np.concatenate(out), O.reach(t, u))


@pytest.mark.parametrize("world,h", [(2, 300), (4, 10), (3, 7)])
@pytest.mark.parametrize("k", [3, 4])
def test_banded_near_k_halo_exchange(dev, world, h, k):
    # k halo rows per neighbour and one fused near^k / interior^k launch; bands
    # thinner than k (h=10 over 4 bands) fall back to single steps
    rng = O.Rng(world * 100 + h + k)
    u = O.random_mask(257, h, 0.3, rng)
    ub = split(dev, u, world)
    grp = LocalGroup(world)
    ref_n, ref_e = u, u
    for _ in range(k):
        ref_n, ref_e = O.dilate(ref_n), O.erode(ref_e)
    got = grp.run(lambda c, b: near_banded(c, b, k).numpy(), ub)
    assert np.array_equal(np.concatenate(got), ref_n)
    got = grp.run(lambda c, b: near_banded(c, b, k, erode=True).numpy(), ub)
    assert np.array_equal(np.concatenate(got), ref_e)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("w,h,ud", [(1000, 1000, 0.41), (600, 517, 0.5)])
def test_banded_ccl_equals_single_image_labels(dev, world, w, h, ud):
    from paper_2010_07284_b200 import ccl
    from paper_2010_07284_b200.bands import ccl_banded
    u = O.random_mask(w, h, ud, O.Rng(w + h + 7 * world))
    ub = split(dev, u, world)
    got = LocalGroup(world).run(lambda c, b: ccl_banded(c, b).cpu().numpy(), ub)
    want = ccl.label(DeviceImage.upload(u, PixelKind.Bool, dev)).numpy().astype(np.int64)
    assert np.array_equal(np.concatenate(got), want)


@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("w,h", [(200, 150), (256, 256), (257, 90), (1000, 64)])
@pytest.mark.parametrize("given_labels", [False, True])
def test_banded_ccl_both_paths(dev, world, w, h, given_labels):
    """ccl_banded without labels (slcs_ccl_band_begin/finish: 64-bit labels
    straight from the union-find; bands the one-CTA path takes keep u32 labels)
    and with band labels given (slcs_band_ccl_relabel) agree with the whole image."""
    from paper_2010_07284_b200 import ccl
    from paper_2010_07284_b200.bands import ccl_banded
    u = O.random_mask(w, h, 0.45, O.Rng(w * 3 + h + world))
    ub = split(dev, u, world)

    def one(c, b):
        local = ccl.label(b, dev) if given_labels else None
        return ccl_banded(c, b, local).cpu().numpy()
    got = LocalGroup(world).run(one, ub)
    assert np.array_equal(np.concatenate(got), O.flood_fill_label(u).astype(np.int64))


def test_banded_ccl_blob_and_64bit_offsets(dev):
    # a giant blob component crossing every band; labels of the lower bands exceed
    # the band-local range, exercising the 64-bit global offsets
    from paper_2010_07284_b200.bands import ccl_banded
    img = O.blob_noise(1024, 1024, 1)
    u = O.threshold(0, img, 56360)
    got = LocalGroup(6).run(lambda c, b: ccl_banded(c, b).cpu().numpy(), split(dev, u, 6))
    assert np.array_equal(np.concatenate(got), O.flood_fill_label(u).astype(np.int64))


def _storage_bytes(img):
    from paper_2010_07284_b200.bands import device_bytes
    ptr, pitch, _ = img.storage()
    return device_bytes(ptr, pitch * img.height, img.device.device)


@pytest.mark.parametrize("world", [2, 8])
def test_banded_c5_scale_equals_whole_image(dev, world):
    """Config 5's banded path at the largest size a single image still labels in
    32 bits (65535^2, image.cpp:26-28): banded near^4 / volume / reach / ccl equal
    the whole-image kernels bit for bit (compared on the device)."""
    import torch
    from paper_2010_07284_b200 import ccl
    from paper_2010_07284_b200.bands import ccl_banded, device_bytes
    from paper_2010_07284_b200.pixlog import random_mask_device
    n = 65535
    spans = [band_rows(n, world, r) for r in range(world)]
    masks = [random_mask_device(n, r1 - r0, 0.5, 1, r0, dev) for r0, r1 in spans]
    tgts = [random_mask_device(n, r1 - r0, 0.05, 2, r0, dev) for r0, r1 in spans]
    whole_m = random_mask_device(n, n, 0.5, 1, 0, dev)
    whole_t = random_mask_device(n, n, 0.05, 2, 0, dev)
    grp = LocalGroup(world)

    def same_rows(parts, whole):
        dev.synchronize()  # the library's stream -> torch's
        w_all = _storage_bytes(whole)
        _, pitch, _ = whole.storage()
        for (r0, r1), p in zip(spans, parts):
            assert torch.equal(_storage_bytes(p), w_all[r0 * pitch:r1 * pitch]), (r0, r1)

    # near^4 and volume
    got = grp.run(lambda c, b: near_banded(c, b, 4), masks)
    same_rows(got, kernels.dilateK(whole_m, 4, dev))
    del got
    vols = grp.run(lambda c, b: volume_banded(c, b), masks)
    assert all(v == kernels.countTrue(whole_m, dev) for v in vols)
    # reach
    got = grp.run(lambda c, b: reach_banded(c, b[0], b[1]), list(zip(tgts, masks)))
    same_rows(got, reach(whole_t, whole_m, dev))
    del got
    # ccl: 64-bit band labels vs the whole image's 32-bit canonical labels
    whole_lab = ccl.label(whole_m, dev)
    dev.synchronize()
    ptr, _, _ = whole_lab.storage()
    lab = device_bytes(ptr, n * n * 4, dev.device).view(torch.int32)
    labs = grp.run(lambda c, b: ccl_banded(c, b), masks)
    for (r0, r1), l64 in zip(spans, labs):
        want = lab[r0 * n:r1 * n].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(l64.view(-1), want), (r0, r1)
    del labs
    # reach + ccl from one labelling (the C5 bench step)
    from paper_2010_07284_b200.bands import reach_ccl_banded
    both = grp.run(lambda c, b: reach_ccl_banded(c, b[0], b[1]), list(zip(tgts, masks)))
    same_rows([x[0] for x in both], reach(whole_t, whole_m, dev))
    for (r0, r1), (_, l64) in zip(spans, both):
        want = lab[r0 * n:r1 * n].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(l64.view(-1), want), (r0, r1)


def test_ccl_band_job_errors_and_early_destroy(dev):
    """A job can be destroyed without finishing; bad finish arguments are a
    status code, and the job stays destroyable."""
    import ctypes as C
    from paper_2010_07284_b200 import _lib
    from paper_2010_07284_b200.bands import _zeros
    L = _lib.load()
    u = O.random_mask(700, 300, 0.5, O.Rng(5))
    img = DeviceImage.upload(u, PixelKind.Bool, dev)
    rec = _zeros(L.slcs_band_record_bytes(1, 700), dev)
    for finish in (False, True):
        job = C.c_void_p()
        assert L.slcs_ccl_band_begin(dev.handle, img.handle, C.c_void_p(rec.data_ptr()),
                                     C.byref(job)) == 0
        if finish:
            hs = (C.c_longlong * 1)(300)
            rc = L.slcs_ccl_band_finish(job, 1, 3, C.c_void_p(rec.data_ptr()), hs,
                                        C.c_void_p(rec.data_ptr()))
            assert rc != 0 and "band" in L.slcs_last_error().decode()
        assert L.slcs_ccl_job_destroy(job) == 0
    lab = DeviceImage.upload(u, PixelKind.Bool, dev)
    job = C.c_void_p()
    from paper_2010_07284_b200 import ccl
    labels = ccl.label(lab, dev)
    rc = L.slcs_ccl_band_begin(dev.handle, labels.handle, C.c_void_p(rec.data_ptr()),
                               C.byref(job))
    assert rc != 0 and "expects a boolean image" in L.slcs_last_error().decode()


@pytest.mark.parametrize("use_job", [False, True])
def test_band_labels_to_unaligned_output(dev, use_job):
    """64-bit label output that is 8- but not 16-byte aligned takes the scalar
    store path of k_relabel_hash / k_tile_labels<u64>; the labels are the same."""
    import ctypes as C
    import torch
    from paper_2010_07284_b200 import _lib, ccl
    from paper_2010_07284_b200.bands import _zeros
    L = _lib.load()
    w, h = 777, 300
    u = O.random_mask(w, h, 0.5, O.Rng(9))
    img = DeviceImage.upload(u, PixelKind.Bool, dev)
    rec = _zeros(L.slcs_band_record_bytes(1, w), dev)
    buf = torch.zeros(w * h + 1, dtype=torch.int64, device=torch.device("cuda", dev.device))
    out_ptr = C.c_void_p(buf.data_ptr() + 8)
    hs = (C.c_longlong * 1)(h)
    if use_job:
        job = C.c_void_p()
        assert L.slcs_ccl_band_begin(dev.handle, img.handle, C.c_void_p(rec.data_ptr()),
                                     C.byref(job)) == 0
        assert L.slcs_ccl_band_finish(job, 1, 0, C.c_void_p(rec.data_ptr()), hs, out_ptr) == 0
        assert L.slcs_ccl_job_destroy(job) == 0
    else:
        lab = ccl.label(img, dev)
        assert L.slcs_band_ccl_relabel(dev.handle, lab.handle, 1, 0, None, hs, out_ptr) == 0
    dev.synchronize()
    got = buf[1:].cpu().numpy().reshape(h, w)
    assert np.array_equal(got, O.flood_fill_label(u).astype(np.int64))


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("w,h,ud", [(600, 517, 0.5), (1000, 700, 0.41), (200, 150, 0.45)])
def test_reach_ccl_banded_shares_one_labelling(dev, world, w, h, ud):
    """reach_ccl_banded: reach and 64-bit ccl::label of the same band from one
    union-find equal the whole-image reach and the reference labels."""
    from paper_2010_07284_b200.bands import reach_ccl_banded
    rng = O.Rng(w + 11 * world)
    u = O.random_mask(w, h, ud, rng)
    t = O.random_mask(w, h, 0.03, rng)
    ub, tb = split(dev, u, world), split(dev, t, world)
    got = LocalGroup(world).run(
        lambda c, b: tuple(x.numpy() if hasattr(x, "numpy") and not hasattr(x, "cpu")
                           else x.cpu().numpy() for x in reach_ccl_banded(c, b[0], b[1])),
        list(zip(tb, ub)))
    assert np.array_equal(np.concatenate([g[0] for g in got]), O.reach(t, u))
    assert np.array_equal(np.concatenate([g[1] for g in got]),
                          O.flood_fill_label(u).astype(np.int64))


def test_ccl_job_keeps_reach_labelling_alive(dev):
    """A ccl job borrowed from a reach state stays valid after the reach state is
    destroyed first (the job holds a reference); labels are still exact."""
    import ctypes as C
    import torch
    from paper_2010_07284_b200 import _lib
    from paper_2010_07284_b200.bands import _zeros
    L = _lib.load()
    w, h = 640, 300
    rng = O.Rng(21)
    u, t = O.random_mask(w, h, 0.5, rng), O.random_mask(w, h, 0.03, rng)
    du, dt = (DeviceImage.upload(x, PixelKind.Bool, dev) for x in (u, t))
    st, job = C.c_void_p(), C.c_void_p()
    assert L.slcs_reach_prepare(dev.handle, dt.handle, du.handle, C.byref(st)) == 0
    rec = _zeros(L.slcs_band_record_bytes(1, w), dev)
    rc = L.slcs_ccl_band_begin_reach(st, C.c_void_p(rec.data_ptr()), C.byref(job))
    assert rc != 0 and "max keys" in L.slcs_last_error().decode()
    assert L.slcs_reach_state_destroy(st) == 0
    assert L.slcs_reach_prepare_labels(dev.handle, dt.handle, du.handle, C.byref(st)) == 0
    assert L.slcs_ccl_band_begin_reach(st, C.c_void_p(rec.data_ptr()), C.byref(job)) == 0
    assert L.slcs_reach_state_destroy(st) == 0  # before the job: the job keeps it alive
    out = torch.zeros((h, w), dtype=torch.int64, device=torch.device("cuda", dev.device))
    hs = (C.c_longlong * 1)(h)
    assert L.slcs_ccl_band_finish(job, 1, 0, C.c_void_p(rec.data_ptr()), hs,
                                  C.c_void_p(out.data_ptr())) == 0
    assert L.slcs_ccl_job_destroy(job) == 0
    dev.synchronize()
    assert np.array_equal(out.cpu().numpy(), O.flood_fill_label(u).astype(np.int64))
