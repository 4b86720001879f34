"""Host-in/host-out C ABI with page-locked host buffers.

Pinned buffers (a torch pin_memory() tensor, cudaHostAlloc / cudaHostRegister)
are copied to and from directly, without the staging memcpy the pageable
(std::vector-backed, reference ImageBuffer) buffers go through.  Results must be
the same either way, and a pinned upload source must be free for reuse once the
call returns (the DMA read it already)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    from paper_2010_07284_b200 import Device, _lib
    from paper_2010_07284_b200.pixlog import _check
    return Device(0), _lib.load(), _check


def _pinned(a: np.ndarray) -> torch.Tensor:
    t = torch.empty(a.shape, dtype={np.uint8: torch.uint8, np.int32: torch.int32,
                                     np.uint32: torch.int32}[a.dtype.type]).pin_memory()
    t.numpy()[...] = a.view(t.numpy().dtype)
    return t


def _ptr(x):
    return C.c_void_p(x.data_ptr() if isinstance(x, torch.Tensor) else x.ctypes.data)


@pytest.mark.parametrize("pin_in,pin_out", [(True, True), (True, False), (False, True)])
def test_ccl_and_reach_pinned(env, pin_in, pin_out):
    dev, L, check = env
    rng = O.Rng(11)
    w, h = 1000, 700
    u = O.random_mask(w, h, 0.5, rng)
    t = O.random_mask(w, h, 0.02, rng)
    ui = _pinned(u) if pin_in else np.ascontiguousarray(u)
    ti = _pinned(t) if pin_in else np.ascontiguousarray(t)
    lab = _pinned(np.zeros((h, w), np.int32)) if pin_out else np.zeros((h, w), np.uint32)
    rch = _pinned(np.zeros((h, w), np.uint8)) if pin_out else np.zeros((h, w), np.uint8)
    check(L.slcs_h_ccl_label(dev.handle, _ptr(ui), w, h, _ptr(lab)))
    check(L.slcs_h_reach(dev.handle, _ptr(ti), _ptr(ui), w, h, _ptr(rch)))
    got_lab = (lab.numpy() if pin_out else lab).view(np.uint32)
    got_r = rch.numpy() if pin_out else rch
    assert np.array_equal(got_lab, O.flood_fill_label(u))
    assert np.array_equal(got_r, O.reach(t, u))


def test_pinned_upload_source_reusable_on_return(env):
    from paper_2010_07284_b200 import PixelKind
    dev, L, check = env
    rng = O.Rng(5)
    w, h = 4096, 2048  # large enough that an unfinished DMA would be caught
    a = O.random_mask(w, h, 0.5, rng)
    src = _pinned(a)
    img = C.c_void_p()
    check(L.slcs_image_upload(dev.handle, int(PixelKind.Bool), w, h, 1, _ptr(src),
                              C.byref(img)))
    src.numpy()[...] = 1 - src.numpy()  # the caller reuses its buffer at once
    out = _pinned(np.zeros((h, w), np.uint8))
    try:
        check(L.slcs_image_download(dev.handle, img, _ptr(out), w * h))
    finally:
        L.slcs_image_release(img)
    assert np.array_equal(out.numpy(), a)
