"""Concurrent entry-point calls from several host threads (SURVEY §8(b) "Threading").

The reference's executor runs independent DAG nodes concurrently on its WorkerPool
(proj/src/executor.cpp:220, 259), so `evalTask` -- and with it every primitive --
is called from several threads at once.  Here eight Python threads drive the C ABI
concurrently (ctypes releases the GIL around each call), sharing one context and
passing device images between threads; every result must equal the oracle
bit-exactly.
"""
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import (CmpOp, DeviceImage, PixelKind, ccl, kernels, maxvol, reach)

pytestmark = pytest.mark.gpu


def _work(seed, size):
    rng = O.Rng(seed)
    w, h = size + seed % 7, size - seed % 5
    img = O.blob_noise(w, h, seed)
    t = O.random_mask(w, h, 0.02, rng)
    u16 = DeviceImage.upload(img, PixelKind.U16)
    tgt = DeviceImage.upload(t, PixelKind.Bool)
    through = kernels.threshold(CmpOp.Gt, u16, 56360)
    r = reach(kernels.dilate(tgt), through)
    lab = ccl.label(through)
    mv = maxvol(through)
    vol = kernels.countTrue(r)
    return seed, img, t, through, r, lab, mv, vol


def _check(seed, img, t, through, r, lab, mv, vol):
    th = O.threshold(0, img, 56360)
    assert np.array_equal(through.numpy(), th), seed
    ref = O.reach(O.dilate(t), th)
    assert np.array_equal(r.numpy(), ref), seed
    assert vol == int(ref.sum()), seed
    assert np.array_equal(lab.numpy(), O.flood_fill_label(th)), seed
    assert np.array_equal(mv.numpy(), O.maxvol(th)), seed


@pytest.mark.parametrize("size", [200, 700])
def test_concurrent_primitives_match_the_oracle(dev, size):
    with ThreadPoolExecutor(max_workers=8) as ex:
        results = list(ex.map(lambda s: _work(s, size), range(1, 17)))
    for res in results:
        _check(*res)


def test_images_shared_across_threads(dev):
    """One thread's output is another thread's input (the executor hands Values
    between worker threads); producers and consumers race on one context."""
    size = 512
    img = O.blob_noise(size, size, 3)
    u16 = DeviceImage.upload(img, PixelKind.U16)
    base = kernels.threshold(CmpOp.Gt, u16, 56360)
    th = O.threshold(0, img, 56360)
    outs, lock = {}, threading.Lock()

    def chain(k):
        x = base
        for _ in range(k):
            x = kernels.dilate(x)
        y = reach(x, base)
        with lock:
            outs[k] = y

    threads = [threading.Thread(target=chain, args=(k,)) for k in range(1, 9)]
    for th_ in threads:
        th_.start()
    for th_ in threads:
        th_.join()
    for k in range(1, 9):
        x = th
        for _ in range(k):
            x = O.dilate(x)
        assert np.array_equal(outs[k].numpy(), O.reach(x, th)), k
