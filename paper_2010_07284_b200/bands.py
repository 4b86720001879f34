"""Row-band decomposition of very large images across GPUs.

A W x H image is split into contiguous row bands, one per rank (one process per
GPU, ``torch.distributed`` over NCCL).  The reference cannot process these
images at all (its labels throw at W*H >= 0xFFFFFFFE, image.cpp:26-28); the
banded path computes the same results as a single-device run, and every byte it
exchanges stays in device memory:

* elementwise ops / thresholds: local, no communication;
* ``near^k`` / ``interior^k``: each rank sends its first k packed rows up and its
  last k rows down (point-to-point NCCL send/recv, neighbours only) into halo
  buffers, and one ``slcs_near_k_halo`` launch reads them in place -- no band
  copies (out-of-image rows stay absent: 0 for near, 1 for interior, the
  reference's clipping, kernels.cpp:106-121);
* ``volume``: device popcount into an int64 + NCCL all-reduce SUM;
* ``reach(t, u)``: each band labels its own ``u`` (``slcs_reach_prepare``),
  writes a small border record (roots / seed classes of its first and last row
  and its first and last target row), the records are all-gathered (NCCL), and
  every rank resolves the components that cross band borders with one small
  device union-find (``slcs_band_reach_merge``, csrc/bands.cu), flags its newly
  seeded roots, selects ``t | S`` and closes with a halo ``near``;
* ``ccl::label``: the band's union-find and its label border record
  (``slcs_ccl_band_begin``: the u32 labels of its first and last row, no label
  image), all-gather, then a device merge and the global 64-bit labels written
  straight from the union-find (``slcs_ccl_band_finish``).  With band labels
  already at hand, ``slcs_ccl_border_record`` + ``slcs_band_ccl_relabel``;
  with a reach on the same image, ``reach_ccl_banded`` labels the band once for
  both.

Per step and rank the communication is: near^k 2*k packed rows (k * W/8 bytes
each way), reach 2 * (5 W + W/4) bytes all-gathered per band plus the closing
near's halo, ccl 8 W bytes per band, volume 8 bytes.

``Comm`` abstracts the exchanges: ``TorchComm`` (torch.distributed; NCCL on
device tensors, or gloo, which stages through host memory, in the CPU tests and
the one-GPU test mode) and ``LocalGroup`` (N bands on one GPU, threads -- the
bit-exact check against the single-image path).  Collectives raise
``RunError(..., SLCS_ERR_NCCL)`` on failure.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Optional

from . import _lib
from .pixlog import Device, DeviceImage, PixelKind, RunError, _check, kernels, reach

SLCS_ERR_NCCL = 6


def band_rows(h: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row ranges; every band gets at least one row."""
    if world > h:
        raise RunError(f"cannot split {h} rows into {world} bands", 2)
    base, extra = divmod(h, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


# ---------------------------------------------------------------- device memory views
class _CudaArray:
    """__cuda_array_interface__ of raw library memory (zero-copy torch views)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 2, "strides": None}


def device_bytes(ptr: int, nbytes: int, device: int):
    """A uint8 torch tensor aliasing `nbytes` of device memory at `ptr` (no copy; the
    owner -- e.g. a DeviceImage -- must outlive it)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, nbytes), device=torch.device("cuda", device))


def _rows_view(img: DeviceImage, r0: int, n: int):
    """Packed rows [r0, r0 + n) of a Bool band, zero-copy."""
    ptr, pitch, _ = img.storage()
    return device_bytes(ptr + r0 * pitch, n * pitch, img.device.device)


# ---------------------------------------------------------------- communication
class Comm:
    """Exchange primitives of a banded computation, on device tensors (uint8 /
    int64).  Every call is a collective: all ranks make it in the same order."""

    rank: int
    world: int

    def halo(self, send_up, send_down, recv_up, recv_down, dev: Device) -> None:
        """send_up -> rank-1, send_down -> rank+1; recv_up <- rank-1, recv_down
        <- rank+1 (None where there is no neighbour)."""
        raise NotImplementedError

    def allgather(self, src, out, dev: Device) -> None:
        """out = concatenation of every rank's src, in rank order."""
        raise NotImplementedError

    def allreduce_sum(self, t, dev: Device) -> None:
        """In-place SUM over ranks."""
        raise NotImplementedError

    def allgather_object(self, obj) -> list:
        """Small host metadata (band heights)."""
        raise NotImplementedError

    _heights: Optional[tuple] = None

    def band_heights(self, h: int) -> list:
        """Every rank's band height (cached while this rank's height is unchanged)."""
        if self._heights is None or self._heights[0] != h:
            self._heights = (h, [int(x) for x in self.allgather_object(int(h))])
        return self._heights[1]


def _streams_differ(dev: Device) -> bool:
    import torch
    return dev.stream != torch.cuda.current_stream(dev.device).cuda_stream


class TorchComm(Comm):
    """torch.distributed.  NCCL works on the device tensors directly; its
    collectives are ordered after the work on torch's current stream, so a
    Device built on that stream (``Device(i, stream=torch.cuda.current_stream(i)
    .cuda_stream)``) needs no host synchronisation.  gloo stages through host
    memory (CPU tests, the one-GPU test mode)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.staged = dist.get_backend() != "nccl"

    def _before(self, dev: Optional[Device]):
        if dev is not None and (self.staged or _streams_differ(dev)):
            dev.synchronize()

    def _after(self, dev: Optional[Device]):
        if dev is not None and (self.staged or _streams_differ(dev)):
            import torch
            torch.cuda.current_stream(dev.device).synchronize()

    def _guard(self, fn):
        try:
            return fn()
        except RunError:
            raise
        except Exception as e:  # NCCL / gloo failures surface as SLCS_ERR_NCCL
            raise RunError(f"collective failed: {e}", SLCS_ERR_NCCL) from e

    def halo(self, send_up, send_down, recv_up, recv_down, dev=None):
        d = self.dist
        self._before(dev)

        def go():
            stage = self.staged and any(
                x is not None and x.is_cuda for x in (send_up, send_down, recv_up, recv_down))
            host = (lambda x: None if x is None else x.cpu()) if stage else (lambda x: x)
            su, sd = host(send_up), host(send_down)
            ru, rd = host(recv_up), host(recv_down)
            ops = []
            if self.rank > 0:
                ops += [d.P2POp(d.isend, su, self.rank - 1), d.P2POp(d.irecv, ru, self.rank - 1)]
            if self.rank + 1 < self.world:
                ops += [d.P2POp(d.isend, sd, self.rank + 1), d.P2POp(d.irecv, rd, self.rank + 1)]
            if ops:
                for w in d.batch_isend_irecv(ops):
                    w.wait()
            if stage:
                if recv_up is not None and self.rank > 0:
                    recv_up.copy_(ru)
                if recv_down is not None and self.rank + 1 < self.world:
                    recv_down.copy_(rd)
        self._guard(go)
        self._after(dev)

    def allgather(self, src, out, dev=None):
        self._before(dev)

        def go():
            if self.staged and src.is_cuda:
                o = out.cpu()
                self.dist.all_gather_into_tensor(o, src.cpu())
                out.copy_(o)
            else:
                self.dist.all_gather_into_tensor(out, src)
        self._guard(go)
        self._after(dev)

    def allreduce_sum(self, t, dev=None):
        self._before(dev)

        def go():
            if self.staged and t.is_cuda:
                h = t.cpu()
                self.dist.all_reduce(h)
                t.copy_(h)
            else:
                self.dist.all_reduce(t)
        self._guard(go)
        self._after(dev)

    def allgather_object(self, obj):
        out = [None] * self.world
        self._guard(lambda: self.dist.all_gather_object(out, obj))
        return out


class SoloComm(Comm):
    """World size 1: the band is the whole image."""

    rank, world = 0, 1

    def halo(self, send_up, send_down, recv_up, recv_down, dev=None):
        pass

    def allgather(self, src, out, dev=None):
        out.copy_(src)

    def allreduce_sum(self, t, dev=None):
        pass

    def allgather_object(self, obj):
        return [obj]


class LocalGroup:
    """N bands in one process on one GPU (threads): the same protocol, with
    device-to-device copies for the exchanges.  Runs the banded algorithm for
    bit-exact checks against the single-image kernels."""

    def __init__(self, world: int):
        self.world = world

    def run(self, fn, bands: list):
        """fn(comm, band) for every band, stepping all bands through each exchange."""
        import torch
        results = [None] * self.world
        errors = []
        barrier = threading.Barrier(self.world)
        shared = {}
        world = self.world

        class _C(Comm):
            def __init__(s, r):
                s.rank, s.world = r, world

            def _publish(s, obj, dev):
                if dev is not None:
                    dev.synchronize()
                shared[s.rank] = obj
                barrier.wait()
                return [shared[i] for i in range(world)]

            def _done(s):
                torch.cuda.synchronize()
                barrier.wait()

            def halo(s, send_up, send_down, recv_up, recv_down, dev=None):
                peers = s._publish((send_up, send_down), dev)
                if s.rank > 0 and recv_up is not None:
                    recv_up.copy_(peers[s.rank - 1][1])
                if s.rank + 1 < world and recv_down is not None:
                    recv_down.copy_(peers[s.rank + 1][0])
                s._done()

            def allgather(s, src, out, dev=None):
                peers = s._publish(src, dev)
                n = src.numel()
                for i, p in enumerate(peers):
                    out[i * n:(i + 1) * n].copy_(p)
                s._done()

            def allreduce_sum(s, t, dev=None):
                if dev is not None:
                    dev.synchronize()  # t is written on the library's stream
                peers = s._publish(t.clone(), None)
                total = peers[0].clone()
                for p in peers[1:]:
                    total += p
                s._done()
                t.copy_(total)
                torch.cuda.synchronize()

            def allgather_object(s, obj):
                out = s._publish(obj, None)
                barrier.wait()
                return out

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
def _empty(nbytes: int, dev: Device):
    import torch
    return torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", dev.device))


def _zeros(nbytes: int, dev: Device):
    """Border records: alignment gaps are sent too, so they are zero (initcheck-clean)."""
    import torch
    return torch.zeros(nbytes, dtype=torch.uint8, device=torch.device("cuda", dev.device))


def near_banded(comm: Comm, band: DeviceImage, k: int = 1, erode: bool = False) -> DeviceImage:
    """near^k (or interior^k) of the full image, restricted to this band: k halo
    rows from each neighbour, then one fused near^k launch that reads them in
    place (csrc/bitops.cu, Halo).  Every branch is taken uniformly by all ranks."""
    dev, h = band.device, band.height
    if comm.world == 1:  # the band is the whole image: no halo
        return (kernels.erodeK if erode else kernels.dilateK)(band, k, dev)
    if band.kind != PixelKind.Bool:
        band = kernels.threshold(0, band, 0.0, dev)  # boolArg: p > 0 (executor.cpp:43-50)
    if k > 1 and min(comm.band_heights(h)) < k:
        # some band is thinner than the halo: every rank takes k single steps
        cur = band
        for _ in range(k):
            cur = near_banded(comm, cur, 1, erode)
        return cur
    _, pitch, _ = band.storage()
    up = comm.rank > 0
    down = comm.rank + 1 < comm.world
    top = _empty(k * pitch, dev) if up else None
    bot = _empty(k * pitch, dev) if down else None
    comm.halo(_rows_view(band, 0, k) if up else None,
              _rows_view(band, h - k, k) if down else None, top, bot, dev)
    out = C.c_void_p()
    _check(_lib.load().slcs_near_k_halo(
        dev.handle, band.handle, int(k), int(erode), None if top is None else top.data_ptr(),
        k if up else 0, None if bot is None else bot.data_ptr(), k if down else 0, C.byref(out)))
    if _streams_differ(dev):  # the halo buffers belong to torch's stream
        dev.synchronize()
    return DeviceImage(out, dev)


def volume_banded(comm: Comm, band: DeviceImage) -> int:
    """volume of the full image: device popcount + all-reduce SUM (8 bytes)."""
    import torch
    dev = band.device
    t = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", dev.device))
    if comm.world == 1:
        return kernels.countTrue(band, dev)
    _check(_lib.load().slcs_volume_async(dev.handle, band.handle, C.c_void_p(t.data_ptr())))
    comm.allreduce_sum(t, dev)
    return int(t.item())


def reach_banded(comm: Comm, target: DeviceImage, through: DeviceImage) -> DeviceImage:
    """reach(target, through) of the full image, restricted to this band."""
    L = _lib.load()
    dev, w = target.device, target.width
    if comm.world == 1:  # the band is the whole image
        return reach(target, through, dev)
    st = C.c_void_p()
    _check(L.slcs_reach_prepare(dev.handle, target.handle, through.handle, C.byref(st)))
    try:
        nrec = L.slcs_band_record_bytes(0, w)
        mine = _zeros(nrec, dev)
        _check(L.slcs_reach_border_record(st, C.c_void_p(mine.data_ptr())))
        allrec = _empty(nrec * comm.world, dev)
        comm.allgather(mine, allrec, dev)
        _check(L.slcs_band_reach_merge(st, comm.world, comm.rank, C.c_void_p(allrec.data_ptr())))
        sel = C.c_void_p()
        _check(L.slcs_reach_finish(st, 0, C.byref(sel)))
        sel_band = DeviceImage(sel, dev)
        # the merge reads `allrec` in stream order before it is freed (torch's
        # caching allocator may recycle it on its own stream)
        if _streams_differ(dev):
            dev.synchronize()
    finally:
        L.slcs_reach_state_destroy(st)
    return near_banded(comm, sel_band, 1)  # reach = near(t | S)


def reach_ccl_banded(comm: Comm, target: DeviceImage, through: DeviceImage):
    """(reach(target, through), ccl::label(through)) of the full image,
    restricted to this band, from ONE labelling of the band's `through`
    (slcs_reach_prepare_labels + slcs_ccl_band_begin_reach): the reach's
    border-record merge and the labels' merge run as in reach_banded and
    ccl_banded, the band union-find only once."""
    import torch
    L = _lib.load()
    dev, w, h = target.device, target.width, target.height
    heights = comm.band_heights(h)
    hs = (C.c_longlong * comm.world)(*heights)
    st = C.c_void_p()
    _check(L.slcs_reach_prepare_labels(dev.handle, target.handle, through.handle, C.byref(st)))
    try:
        nrec_l = L.slcs_band_record_bytes(1, w)
        lrec = _zeros(nrec_l, dev)
        job = C.c_void_p()
        _check(L.slcs_ccl_band_begin_reach(st, C.c_void_p(lrec.data_ptr()), C.byref(job)))
        try:
            lall = lrec
            if comm.world > 1:
                nrec = L.slcs_band_record_bytes(0, w)
                mine = _zeros(nrec, dev)
                _check(L.slcs_reach_border_record(st, C.c_void_p(mine.data_ptr())))
                allrec = _empty(nrec * comm.world, dev)
                comm.allgather(mine, allrec, dev)
                _check(L.slcs_band_reach_merge(st, comm.world, comm.rank,
                                               C.c_void_p(allrec.data_ptr())))
                lall = _empty(nrec_l * comm.world, dev)
                comm.allgather(lrec, lall, dev)
            sel = C.c_void_p()
            _check(L.slcs_reach_finish(st, 0, C.byref(sel)))
            sel_band = DeviceImage(sel, dev)
            out = torch.empty((h, w), dtype=torch.int64, device=torch.device("cuda", dev.device))
            _check(L.slcs_ccl_band_finish(job, comm.world, comm.rank,
                                          C.c_void_p(lall.data_ptr()), hs,
                                          C.c_void_p(out.data_ptr())))
            if _streams_differ(dev):
                dev.synchronize()
        finally:
            _check(L.slcs_ccl_job_destroy(job))
    finally:
        L.slcs_reach_state_destroy(st)
    return near_banded(comm, sel_band, 1), out


def ccl_banded(comm: Comm, band: DeviceImage, local=None):
    """ccl::label of the full image, restricted to this band, as global 64-bit
    labels (a torch.int64 tensor on the band's device): band-local union-find
    labels, a label border record all-gathered, and the device merge + relabel.
    Equal to the single-image labels where those fit in 32 bits; 65536^2
    (config 5) needs the 64-bit form.  `local`: the band's labels if already
    computed."""
    import torch

    from .pixlog import ccl
    L = _lib.load()
    dev, w, h = band.device, band.width, band.height
    heights = comm.band_heights(h)
    nrec = L.slcs_band_record_bytes(1, w)
    out = torch.empty((h, w), dtype=torch.int64, device=torch.device("cuda", dev.device))
    hs = (C.c_longlong * comm.world)(*heights)
    mine = _zeros(nrec, dev)
    if local is None:
        # no u32 label image: the band's union-find -> record -> 64-bit labels
        job = C.c_void_p()
        _check(L.slcs_ccl_band_begin(dev.handle, band.handle, C.c_void_p(mine.data_ptr()),
                                     C.byref(job)))
        try:
            allrec = mine
            if comm.world > 1:
                allrec = _empty(nrec * comm.world, dev)
                comm.allgather(mine, allrec, dev)
            _check(L.slcs_ccl_band_finish(job, comm.world, comm.rank,
                                          C.c_void_p(allrec.data_ptr()), hs,
                                          C.c_void_p(out.data_ptr())))
        finally:
            _check(L.slcs_ccl_job_destroy(job))
    else:
        allrec = None
        if comm.world > 1:
            _check(L.slcs_ccl_border_record(dev.handle, local.handle,
                                            C.c_void_p(mine.data_ptr())))
            allrec = _empty(nrec * comm.world, dev)
            comm.allgather(mine, allrec, dev)
        _check(L.slcs_band_ccl_relabel(dev.handle, local.handle, comm.world, comm.rank,
                                       None if allrec is None else C.c_void_p(allrec.data_ptr()),
                                       hs, C.c_void_p(out.data_ptr())))
    if _streams_differ(dev):
        dev.synchronize()
    return out
