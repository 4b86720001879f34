"""Row-band decomposition of very large images across GPUs.

A W x H image is split into contiguous row bands, one per rank (one process
per GPU, ``torch.distributed`` over NCCL; gloo in the CPU tests).  The
reference cannot process these images at all (its labels throw at
W*H >= 0xFFFFFFFE, image.cpp:26-28); the banded path computes the same
results as a single-device run:

* elementwise ops / thresholds: local, no communication;
* ``near`` / ``interior``: exchange one halo row with each neighbour, run the
  stencil on [halo; band; halo], crop (out-of-image halo = 0 for dilation, 1
  for erosion -- the reference's clipping, kernels.cpp:106-121);
* ``volume``: local popcount + all-reduce SUM;
* ``reach(t, u)``: each band labels its own ``u`` with the tiled union-find
  (target halo rows supply near(t) at the band edges), exports the root node
  and seed class of every pixel of its first and last row, all ranks
  all-gather those border rows, resolve the components that cross band
  borders with one small union-find (``resolve_border_flags``, pure numpy),
  push the newly seeded roots back, select, and close with a halo-exchanged
  ``near``.

``Comm`` abstracts the exchange so the same code runs under torch.distributed
(``TorchComm``) or as N bands on one GPU (``LocalGroup``, used to check the
banded path bit-exactly against the single-image path on one device).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .pixlog import Device, DeviceImage, PixelKind, RunError, _check, kernels, reach


def band_rows(h: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row ranges; every band gets at least one row."""
    if world > h:
        raise RunError(f"cannot split {h} rows into {world} bands", 2)
    base, extra = divmod(h, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


# ---------------------------------------------------------------- cross-band merge
def border_edges(last_roots: np.ndarray, last_cls: np.ndarray, first_roots: np.ndarray,
                 first_cls: np.ndarray) -> np.ndarray:
    """Pixel adjacency between the last row of band r and the first row of band
    r+1 (8-connectivity: column offsets -1, 0, +1) as unique (root_a, root_b)."""
    a = last_cls > 0
    b = first_cls > 0
    w = a.size
    pairs = []
    for d in (-1, 0, 1):
        lo, hi = max(0, -d), min(w, w - d)
        m = a[lo:hi] & b[lo + d:hi + d]
        if m.any():
            pairs.append(np.stack([last_roots[lo:hi][m], first_roots[lo + d:hi + d][m]], 1))
    if not pairs:
        return np.zeros((0, 2), np.uint32)
    return np.unique(np.concatenate(pairs).astype(np.uint32), axis=0)


def resolve_border_flags(rows: list) -> list:
    """rows[r] = (first_roots, first_cls, last_roots, last_cls) of band r.

    Returns, per band, the root nodes that must become seeded because their
    component crosses a band border into a seeded component (cls 2 = seeded,
    1 = unseeded, 0 = background).  Nodes are (band, root) pairs; the result is
    identical on every rank (deterministic)."""
    nb = len(rows)
    keys = []   # (band, root) -> node ids via unique over a structured key
    seeded = []
    for r, (fr, fc, lr, lc) in enumerate(rows):
        for roots, cls in ((fr, fc), (lr, lc)):
            m = cls > 0
            keys.append(np.stack([np.full(m.sum(), r, np.uint64), roots[m].astype(np.uint64)], 1))
            seeded.append(cls[m] == 2)
    if not keys:
        return [np.zeros(0, np.uint32) for _ in range(nb)]
    allk = np.concatenate(keys)
    if allk.size == 0:
        return [np.zeros(0, np.uint32) for _ in range(nb)]
    packed = (allk[:, 0] << np.uint64(32)) | allk[:, 1]
    uniq, inv = np.unique(packed, return_inverse=True)
    seed_node = np.zeros(uniq.size, bool)
    np.logical_or.at(seed_node, inv, np.concatenate(seeded))
    src, dst = [], []
    for r in range(nb - 1):
        e = border_edges(rows[r][2], rows[r][3], rows[r + 1][0], rows[r + 1][1])
        if len(e):
            src.append(np.searchsorted(uniq, (np.uint64(r) << np.uint64(32)) | e[:, 0].astype(np.uint64)))
            dst.append(np.searchsorted(uniq, (np.uint64(r + 1) << np.uint64(32)) | e[:, 1].astype(np.uint64)))
    comp = _components(uniq.size, np.concatenate(src) if src else np.zeros(0, np.int64),
                       np.concatenate(dst) if dst else np.zeros(0, np.int64))
    comp_seeded = np.zeros(comp.max() + 1 if comp.size else 0, bool)
    np.logical_or.at(comp_seeded, comp, seed_node)
    newly = comp_seeded[comp] & ~seed_node
    band = (uniq >> np.uint64(32)).astype(np.int64)
    root = (uniq & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return [root[newly & (band == r)] for r in range(nb)]


def merge_band_labels(rows: list, width: int) -> list:
    """Cross-band CCL label merge.  rows[r] = (first_row_labels,
    last_row_labels, height) of band r, labels band-local (local max index + 1,
    0 = background).  Band r's global labels are local + row0_r * W.  Components
    that touch across a band border (8-connectivity: column offsets -1, 0, +1)
    are united and take the largest global label of the union -- the canonical
    label of the whole-image ccl::label (max index + 1, ccl.hpp:52-60).  Returns,
    per band, (keys: sorted local labels (uint32), vals: new global labels
    (uint64)) for the labels whose global value changes."""
    nb = len(rows)
    row0 = np.cumsum([0] + [int(r[2]) for r in rows[:-1]]).astype(np.uint64)
    W = np.uint64(width)
    src, dst = [], []
    for r in range(nb - 1):
        a = np.asarray(rows[r][1], np.uint64)
        b = np.asarray(rows[r + 1][0], np.uint64)
        for d in (-1, 0, 1):
            lo, hi = max(0, -d), min(width, width - d)
            m = (a[lo:hi] > 0) & (b[lo + d:hi + d] > 0)
            if m.any():
                src.append(a[lo:hi][m] + row0[r] * W)
                dst.append(b[lo + d:hi + d][m] + row0[r + 1] * W)
    if not src:
        return [(np.zeros(0, np.uint32), np.zeros(0, np.uint64)) for _ in range(nb)]
    src, dst = np.concatenate(src), np.concatenate(dst)
    ids, inv = np.unique(np.concatenate([src, dst]), return_inverse=True)
    comp = _components(ids.size, inv[:src.size], inv[src.size:])
    cmax = np.zeros(comp.max() + 1, np.uint64)
    np.maximum.at(cmax, comp, ids)
    new = cmax[comp]
    changed = new != ids
    out = []
    for r in range(nb):
        lo_id = row0[r] * W
        hi_id = lo_id + np.uint64(int(rows[r][2])) * W
        mine = changed & (ids > lo_id) & (ids <= hi_id)
        keys = (ids[mine] - lo_id).astype(np.uint32)
        order = np.argsort(keys)
        out.append((keys[order], new[mine][order]))
    return out


def _components(n: int, src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """Connected components of the undirected border graph (scipy csgraph)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    if n == 0:
        return np.zeros(0, np.int64)
    g = coo_matrix((np.ones(src.size, np.int8), (src, dst)), shape=(n, n))
    return connected_components(g, directed=False)[1].astype(np.int64)


# ---------------------------------------------------------------- communication
class Comm:
    """Exchange primitives a banded computation needs."""

    rank: int
    world: int

    def neighbours(self, first: np.ndarray, last: np.ndarray):
        """Send my first row up and my last row down; return (row above, row below)
        (None at the image edges)."""
        raise NotImplementedError

    def allgather(self, obj) -> list:
        raise NotImplementedError

    def allreduce_sum(self, x: int) -> int:
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed (NCCL between GPUs, gloo on CPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def neighbours(self, first, last):
        rows = self.allgather((first, last))
        above = rows[self.rank - 1][1] if self.rank > 0 else None
        below = rows[self.rank + 1][0] if self.rank + 1 < self.world else None
        return above, below

    def allgather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def allreduce_sum(self, x):
        out = [None] * self.world
        self.dist.all_gather_object(out, int(x))
        return sum(out)


class LocalGroup:
    """N bands in one process -- the same protocol, exchanges are list lookups.
    Runs the banded algorithm on a single GPU for bit-exact checks."""

    def __init__(self, world: int):
        self.world = world

    def run(self, fn, bands: list):
        """fn(comm, band) for every band, stepping all bands through each exchange."""
        import threading
        results = [None] * self.world
        errors = []
        barrier = threading.Barrier(self.world)
        shared = {}

        class _C(Comm):
            def __init__(s, r):
                s.rank, s.world = r, self.world

            def _exchange(s, obj):
                shared[s.rank] = obj
                barrier.wait()
                out = [shared[i] for i in range(self.world)]
                barrier.wait()
                return out

            def neighbours(s, first, last):
                rows = s._exchange((first, last))
                above = rows[s.rank - 1][1] if s.rank > 0 else None
                below = rows[s.rank + 1][0] if s.rank + 1 < s.world else None
                return above, below

            def allgather(s, obj):
                return s._exchange(obj)

            def allreduce_sum(s, x):
                return sum(s._exchange(int(x)))

        def body(r):
            try:
                results[r] = fn(_C(r), bands[r])
            except BaseException as e:  # surfaced below
                errors.append(e)
                barrier.abort()

        threads = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return results


# ---------------------------------------------------------------- banded ops (device)
def _rows(img: DeviceImage, r0: int, n: int) -> DeviceImage:
    out = C.c_void_p()
    _check(_lib.load().slcs_image_rows(img.device.handle, img.handle, r0, n, C.byref(out)))
    return DeviceImage(out, img.device)


def _vstack(imgs: list) -> DeviceImage:
    arr = (C.c_void_p * len(imgs))(*[i.handle for i in imgs])
    out = C.c_void_p()
    _check(_lib.load().slcs_image_vstack(imgs[0].device.handle, len(imgs), arr, C.byref(out)))
    return DeviceImage(out, imgs[0].device)


def _row_bytes(img: DeviceImage, r: int) -> np.ndarray:
    return _rows(img, r, 1).numpy().reshape(-1)


def _halo(row: Optional[np.ndarray], w: int, fill: int, dev: Device) -> DeviceImage:
    a = np.full((1, w), fill, np.uint8) if row is None else row.reshape(1, w).astype(np.uint8)
    return DeviceImage.upload(a, PixelKind.Bool, dev)


def _extend(cur: DeviceImage, above, below, fill: int):
    """[above; cur; below] with halo rows only where a neighbour exists (at the
    image edges the kernels clip exactly like the reference)."""
    dev, w = cur.device, cur.width
    parts, off = [], 0
    if above is not None:
        parts.append(_halo(above, w, fill, dev))
        off = 1
    parts.append(cur)
    if below is not None:
        parts.append(_halo(below, w, fill, dev))
    return (_vstack(parts) if len(parts) > 1 else cur), off


def _rows_bytes(img: DeviceImage, r0: int, n: int) -> np.ndarray:
    return _rows(img, r0, n).numpy().reshape(n, -1)


def near_banded(comm: Comm, band: DeviceImage, k: int = 1, erode: bool = False) -> DeviceImage:
    """near^k (or interior^k) of the full image, restricted to this band: one exchange
    of k halo rows with each neighbour, then one fused near^k launch (csrc k_near*).
    Every branch is taken uniformly by all ranks (each exchange is a collective)."""
    dev, h = band.device, band.height
    op = kernels.erodeK if erode else kernels.dilateK
    if comm.world == 1:  # the band is the whole image: no halo
        return op(band, k, dev)
    if k > 1 and min(comm.allgather(h)) < k:
        # some band is thinner than the halo: every rank takes k single steps
        # (the decision must be uniform -- each step is a collective exchange)
        cur = band
        for _ in range(k):
            cur = near_banded(comm, cur, 1, erode)
        return cur
    above, below = comm.neighbours(_rows_bytes(band, 0, k), _rows_bytes(band, h - k, k))
    parts, off = [], 0
    if above is not None:
        parts.append(DeviceImage.upload(above, PixelKind.Bool, dev))
        off = above.shape[0]
    parts.append(band)
    if below is not None:
        parts.append(DeviceImage.upload(below, PixelKind.Bool, dev))
    ext = _vstack(parts) if len(parts) > 1 else band
    out = op(ext, k, dev)
    return _rows(out, off, h) if out.height != h else out


def volume_banded(comm: Comm, band: DeviceImage) -> int:
    return comm.allreduce_sum(kernels.countTrue(band, band.device))


def reach_banded(comm: Comm, target: DeviceImage, through: DeviceImage) -> DeviceImage:
    """reach(target, through) of the full image, restricted to this band."""
    L = _lib.load()
    dev, w, h = target.device, target.width, target.height
    if comm.world == 1:  # the band is the whole image
        return reach(target, through, dev)
    above, below = comm.neighbours(_row_bytes(target, 0), _row_bytes(target, h - 1))
    t_ext, off = _extend(target, above, below, 0)
    zero = np.zeros((1, w), np.uint8)
    u_ext, _ = _extend(through, None if above is None else zero,
                       None if below is None else zero, 0)
    st = C.c_void_p()
    _check(L.slcs_reach_prepare(dev.handle, t_ext.handle, u_ext.handle, C.byref(st)))
    try:
        def row(r):
            roots = np.zeros(w, np.uint32)
            cls = np.zeros(w, np.uint8)
            _check(L.slcs_reach_row(st, r, roots.ctypes.data, cls.ctypes.data))
            return roots, cls

        fr, fc = row(off)
        lr, lc = row(off + h - 1)
        rows = comm.allgather((fr, fc, lr, lc))
        newly = np.ascontiguousarray(resolve_border_flags(rows)[comm.rank], np.uint32)
        if newly.size:
            _check(L.slcs_reach_set_flags(st, int(newly.size), newly.ctypes.data))
        sel = C.c_void_p()
        _check(L.slcs_reach_finish(st, 0, C.byref(sel)))
        sel_ext = DeviceImage(sel, dev)
    finally:
        L.slcs_reach_state_destroy(st)
    sel_band = _rows(sel_ext, off, h) if sel_ext.height != h else sel_ext
    return near_banded(comm, sel_band, 1)


def ccl_banded(comm: Comm, band: DeviceImage):
    """ccl::label of the full image, restricted to this band, as global 64-bit labels
    (a torch.int64 tensor on the band's device): band-local union-find labels, one
    exchange of the first/last label rows, the cross-band merge above, and a device
    relabel (slcs_ccl_band_relabel).  Equal to the single-image labels where those
    fit in 32 bits; 65536^2 (config 5) needs the 64-bit form."""
    import torch

    from .pixlog import ccl
    dev, w, h = band.device, band.width, band.height
    local = ccl.label(band, dev)
    first = _rows(local, 0, 1).numpy().reshape(-1)
    last = _rows(local, h - 1, 1).numpy().reshape(-1)
    rows = comm.allgather((first, last, h))
    keys, vals = merge_band_labels(rows, w)[comm.rank]
    row0 = sum(int(r[2]) for r in rows[:comm.rank])
    tdev = torch.device("cuda", dev.device)
    out = torch.empty((h, w), dtype=torch.int64, device=tdev)
    k = torch.from_numpy(keys.astype(np.int32)).to(tdev) if keys.size else None
    v = torch.from_numpy(vals.astype(np.int64)).to(tdev) if vals.size else None
    torch.cuda.synchronize(tdev)  # the uploads are on torch's stream
    _check(_lib.load().slcs_ccl_band_relabel(
        dev.handle, local.handle, row0, None if k is None else k.data_ptr(),
        None if v is None else v.data_ptr(), int(keys.size), out.data_ptr()))
    dev.synchronize()
    return out
