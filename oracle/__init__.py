"""CPU oracles for the SLCS hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both loaded with ctypes:

* ``liboracle.so`` -- the plain-C restatement in ``slcs_oracle.c`` (each
  function cites the reference file:line it restates);
* ``_ref/libpixlog_ref.so`` -- the unmodified reference sources compiled in
  place from ``/root/reference/proj/src`` by ``oracle/Makefile`` (present in
  this container, and on a GPU box only when the prebuilt .so travelled).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline.  The product package
(``paper_2010_07284_b200``) never imports it.

Every function takes/returns numpy arrays in the reference ImageBuffer layout
(row-major; Bool as uint8 0/1, U16 as uint16, labels as uint32 idx+1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libpixlog_ref.so")
REFERENCE_SRC = "/root/reference/proj/src"

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Build liboracle.so (always) and oracle/_ref (when the reference is here)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE):
            build(ref=False)
        L = C.CDLL(_ORACLE)
        L.or_rng_next.restype = C.c_uint64
        L.or_rng_next.argtypes = [C.POINTER(C.c_uint64)]
        L.or_random_mask.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(C.c_uint64), _u8p]
        L.or_blob_noise.argtypes = [C.c_int, C.c_int, C.c_uint64, _u16p]
        L.or_checksum.restype = C.c_uint64
        L.or_checksum.argtypes = [C.c_void_p, C.c_size_t]
        L.or_threshold.argtypes = [C.c_int, _u16p, C.c_int, C.c_int, C.c_double, _u8p]
        L.or_not.argtypes = [_u8p, C.c_size_t, _u8p]
        L.or_and.argtypes = [_u8p, _u8p, C.c_size_t, _u8p]
        L.or_or.argtypes = [_u8p, _u8p, C.c_size_t, _u8p]
        L.or_dilate.argtypes = [_u8p, C.c_int, C.c_int, _u8p]
        L.or_erode.argtypes = [_u8p, C.c_int, C.c_int, _u8p]
        L.or_count_true.restype = C.c_int64
        L.or_count_true.argtypes = [_u8p, C.c_size_t]
        L.or_flood_fill_label.argtypes = [_u8p, C.c_int, C.c_int, _u32p]
        L.or_reach.argtypes = [_u8p, _u8p, C.c_int, C.c_int, _u8p]
        L.or_reach_bfs.argtypes = [_u8p, _u8p, C.c_int, C.c_int, _u8p]
        L.or_maxvol.argtypes = [_u8p, C.c_int, C.c_int, _u8p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF) or os.path.isdir(REFERENCE_SRC)


def ref() -> C.CDLL:
    """The reference's own code (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            build(ref=True)
        R = C.CDLL(_REF)
        R.pxref_last_error.restype = C.c_char_p
        R.pxref_threshold.argtypes = [C.c_int, _u16p, C.c_int, C.c_int, C.c_double, _u8p, C.c_int]
        R.pxref_bool_op.argtypes = [C.c_int, _u8p, C.c_void_p, C.c_int, C.c_int, _u8p, C.c_int]
        R.pxref_count_true.argtypes = [_u8p, C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_int]
        R.pxref_ccl_label.argtypes = [_u8p, C.c_int, C.c_int, _u32p, C.c_int, C.c_int,
                                      C.POINTER(C.c_int)]
        R.pxref_flood_fill_label.argtypes = [_u8p, C.c_int, C.c_int, _u32p]
        R.pxref_reach.argtypes = [_u8p, _u8p, C.c_int, C.c_int, _u8p, C.c_int]
        R.pxref_blob_noise.argtypes = [C.c_int, C.c_int, C.c_uint64, _u16p]
        R.pxref_concave_corner.argtypes = [C.c_int, C.c_int, _u16p]
        R.pxref_set_stdlib.argtypes = [C.c_char_p]
        R.pxref_put_u16.argtypes = [C.c_char_p, _u16p, C.c_int, C.c_int]
        R.pxref_put_bool.argtypes = [C.c_char_p, _u8p, C.c_int, C.c_int]
        R.pxref_get.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_int), C.c_void_p]
        R.pxref_run.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int),
                                C.c_char_p, C.c_int]
        R.pxref_dump.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        _ref = R
    return _ref


class OracleError(RuntimeError):
    pass


def _check(rc: int, which: str = "oracle") -> None:
    if rc != 0:
        msg = ref().pxref_last_error().decode() if which == "ref" else "oracle failure"
        raise OracleError(msg)


# --- splitmix64 fixtures (proj/include/pixlog/rng.hpp, tests/oracles.cpp:44-49) ---

class Rng:
    """splitmix64 (proj/include/pixlog/rng.hpp:10-35), stepped in C."""

    def __init__(self, seed: int):
        self.state = C.c_uint64(seed)

    def next(self) -> int:
        return lib().or_rng_next(C.byref(self.state))

    def unit(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        return self.next() % n


def random_mask(w: int, h: int, density: float, rng: Rng) -> np.ndarray:
    out = np.zeros((h, w), np.uint8)
    lib().or_random_mask(w, h, density, C.byref(rng.state), out)
    return out


def blob_noise(w: int, h: int, seed: int) -> np.ndarray:
    out = np.zeros((h, w), np.uint16)
    lib().or_blob_noise(w, h, seed, out)
    return out


def checksum(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return lib().or_checksum(a.ctypes.data, a.nbytes)


# --- primitives (C restatement) ---

def threshold(op: int, img: np.ndarray, n: float) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint16)
    h, w = img.shape
    out = np.zeros((h, w), np.uint8)
    lib().or_threshold(op, img, w, h, float(n), out)
    return out


def logical_not(a):
    a = np.ascontiguousarray(a, np.uint8)
    out = np.zeros_like(a)
    lib().or_not(a, a.size, out)
    return out


def logical_and(a, b):
    a = np.ascontiguousarray(a, np.uint8); b = np.ascontiguousarray(b, np.uint8)
    out = np.zeros_like(a)
    lib().or_and(a, b, a.size, out)
    return out


def logical_or(a, b):
    a = np.ascontiguousarray(a, np.uint8); b = np.ascontiguousarray(b, np.uint8)
    out = np.zeros_like(a)
    lib().or_or(a, b, a.size, out)
    return out


def dilate(a):
    a = np.ascontiguousarray(a, np.uint8)
    h, w = a.shape
    out = np.zeros_like(a)
    lib().or_dilate(a, w, h, out)
    return out


def erode(a):
    a = np.ascontiguousarray(a, np.uint8)
    h, w = a.shape
    out = np.zeros_like(a)
    lib().or_erode(a, w, h, out)
    return out


def count_true(a) -> int:
    a = np.ascontiguousarray(a, np.uint8)
    return int(lib().or_count_true(a, a.size))


def flood_fill_label(a) -> np.ndarray:
    a = np.ascontiguousarray(a, np.uint8)
    h, w = a.shape
    out = np.zeros((h, w), np.uint32)
    if lib().or_flood_fill_label(a, w, h, out) != 0:
        raise OracleError("image too large for packed coordinate labels")
    return out


def reach(t, u) -> np.ndarray:
    t = np.ascontiguousarray(t, np.uint8); u = np.ascontiguousarray(u, np.uint8)
    h, w = t.shape
    out = np.zeros((h, w), np.uint8)
    _check(lib().or_reach(t, u, w, h, out))
    return out


def reach_bfs(t, u) -> np.ndarray:
    t = np.ascontiguousarray(t, np.uint8); u = np.ascontiguousarray(u, np.uint8)
    h, w = t.shape
    out = np.zeros((h, w), np.uint8)
    _check(lib().or_reach_bfs(t, u, w, h, out))
    return out


def maxvol(a) -> np.ndarray:
    a = np.ascontiguousarray(a, np.uint8)
    h, w = a.shape
    out = np.zeros((h, w), np.uint8)
    _check(lib().or_maxvol(a, w, h, out))
    return out


# stdlib compositions (proj/stdlib/stdlib.imgql:5-14), over the primitives.
def interior(a):
    return logical_not(dilate(logical_not(a)))


def touch(a, b):
    return logical_and(a, reach(b, a))


def grow(a, b):
    return logical_or(a, touch(b, a))


def surrounded(a, b):
    return logical_and(a, logical_not(reach(logical_not(logical_or(a, b)), logical_not(b))))


# --- png_io (proj/src/png_io.cpp) -- restated; libpng is absent here ---

def label_color(packed: int) -> tuple[int, int, int]:
    """labelColor (png_io.cpp:75-90): lowbias32 hash, null -> black, black reserved."""
    if packed == 0:
        return 0, 0, 0
    h = packed & 0xFFFFFFFF
    h ^= h >> 16
    h = (h * 0x7FEB352D) & 0xFFFFFFFF
    h ^= h >> 15
    h = (h * 0x846CA68B) & 0xFFFFFFFF
    h ^= h >> 16
    rgb = ((h >> 16) & 255, (h >> 8) & 255, h & 255)
    return (rgb[0], rgb[1], 1) if rgb == (0, 0, 0) else rgb


def png_first_channel_u16(samples: np.ndarray, depth: int) -> np.ndarray:
    """loadPng's sample mapping (png_io.cpp:60-72): first channel; 8-bit -> v*257."""
    ch = samples[..., 0] if samples.ndim == 3 else samples
    return ch.astype(np.uint16) if depth == 16 else (ch.astype(np.uint16) * 257).astype(np.uint16)


_ADAM7 = ((0, 0, 8, 8), (0, 4, 8, 8), (4, 0, 8, 4), (0, 2, 4, 4), (2, 0, 4, 2), (0, 1, 2, 2),
          (1, 0, 2, 1))


def png_encode(samples: np.ndarray, depth: int, color: int, filters=(0,), interlace: bool = False,
               chunk_split: int = 0) -> bytes:
    """A plain PNG writer for fixtures (ISO 15948): `samples` (H, W[, C]) of uint8/uint16,
    row filters cycled from `filters` (0 None .. 4 Paeth), optional Adam7, optional
    IDAT split every `chunk_split` bytes.  Test infrastructure only."""
    import struct
    import zlib
    a = samples if samples.ndim == 3 else samples[..., None]
    h, w, ch = a.shape
    bps = depth // 8
    if depth == 16:
        raw = a.astype(">u2").view(np.uint8).reshape(h, w * ch * 2)
    else:
        raw = a.astype(np.uint8).reshape(h, w * ch)
    bpp = ch * bps

    def filt(rows):
        out, prev, k = bytearray(), None, 0
        for r in rows:
            r = r.astype(np.int32)
            p = np.zeros_like(r) if prev is None else prev
            ft = filters[k % len(filters)]
            k += 1
            a_ = np.concatenate([np.zeros(bpp, np.int32), r[:-bpp]]) if len(r) > bpp else np.zeros_like(r)
            c_ = np.concatenate([np.zeros(bpp, np.int32), p[:-bpp]]) if len(p) > bpp else np.zeros_like(p)
            if ft == 0:
                f = r
            elif ft == 1:
                f = r - a_
            elif ft == 2:
                f = r - p
            elif ft == 3:
                f = r - ((a_ + p) >> 1)
            else:
                pp = a_ + p - c_
                pa, pb, pc = np.abs(pp - a_), np.abs(pp - p), np.abs(pp - c_)
                pred = np.where((pa <= pb) & (pa <= pc), a_, np.where(pb <= pc, p, c_))
                f = r - pred
            out.append(ft)
            out += (f & 255).astype(np.uint8).tobytes()
            prev = r
        return bytes(out)

    if not interlace:
        data = filt(list(raw))
    else:
        data = b""
        for y0, x0, dy, dx in _ADAM7:
            sub = a[y0::dy, x0::dx]
            if sub.size == 0:
                continue
            sr = (sub.astype(">u2").view(np.uint8) if depth == 16 else sub.astype(np.uint8))
            data += filt(list(sr.reshape(sub.shape[0], -1)))
    z = zlib.compress(data, 6)

    def chunk(t, body):
        return struct.pack(">I", len(body)) + t + body + struct.pack(">I", zlib.crc32(t + body))

    out = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, color, 0,
                                                                0, 1 if interlace else 0))
    if chunk_split:
        for i in range(0, len(z), chunk_split):
            out += chunk(b"IDAT", z[i:i + chunk_split])
    else:
        out += chunk(b"IDAT", z)
    return out + chunk(b"IEND", b"")


# --- the reference itself (oracle/_ref) ---

class Reference:
    """Direct calls into the unmodified reference (kernels::*, ccl::label, reach)."""

    def __init__(self, workers: int = 1):
        self.workers = workers
        self.R = ref()

    def threshold(self, op, img, n):
        img = np.ascontiguousarray(img, np.uint16)
        h, w = img.shape
        out = np.zeros((h, w), np.uint8)
        _check(self.R.pxref_threshold(op, img, w, h, float(n), out, self.workers), "ref")
        return out

    def _bool(self, op, a, b=None):
        a = np.ascontiguousarray(a, np.uint8)
        h, w = a.shape
        out = np.zeros((h, w), np.uint8)
        bp = None if b is None else np.ascontiguousarray(b, np.uint8)
        _check(self.R.pxref_bool_op(op, a, None if bp is None else bp.ctypes.data, w, h, out,
                                    self.workers), "ref")
        return out

    def logical_not(self, a):
        return self._bool(0, a)

    def logical_and(self, a, b):
        return self._bool(1, a, b)

    def logical_or(self, a, b):
        return self._bool(2, a, b)

    def dilate(self, a):
        return self._bool(3, a)

    def count_true(self, a):
        a = np.ascontiguousarray(a, np.uint8)
        h, w = a.shape
        v = C.c_int64()
        _check(self.R.pxref_count_true(a, w, h, C.byref(v), self.workers), "ref")
        return int(v.value)

    def ccl_label(self, a, reconnect_interval=0):
        a = np.ascontiguousarray(a, np.uint8)
        h, w = a.shape
        out = np.zeros((h, w), np.uint32)
        it = C.c_int()
        _check(self.R.pxref_ccl_label(a, w, h, out, self.workers, reconnect_interval,
                                      C.byref(it)), "ref")
        return out

    def flood_fill_label(self, a):
        a = np.ascontiguousarray(a, np.uint8)
        h, w = a.shape
        out = np.zeros((h, w), np.uint32)
        _check(self.R.pxref_flood_fill_label(a, w, h, out), "ref")
        return out

    def reach(self, t, u):
        t = np.ascontiguousarray(t, np.uint8); u = np.ascontiguousarray(u, np.uint8)
        h, w = t.shape
        out = np.zeros((h, w), np.uint8)
        _check(self.R.pxref_reach(t, u, w, h, out, self.workers), "ref")
        return out

    def blob_noise(self, w, h, seed):
        out = np.zeros((h, w), np.uint16)
        _check(self.R.pxref_blob_noise(w, h, seed, out), "ref")
        return out

    def concave_corner(self, w, h):
        out = np.zeros((h, w), np.uint16)
        _check(self.R.pxref_concave_corner(w, h, out), "ref")
        return out

    # whole formulas through the reference executor (executor.cpp:231-282)
    def run(self, spec: str, images: dict, stdlib: str, outputs=()):
        R = self.R
        R.pxref_clear()
        R.pxref_set_stdlib(stdlib.encode())
        for name, img in images.items():
            img = np.ascontiguousarray(img)
            h, w = img.shape
            if img.dtype == np.uint16:
                _check(R.pxref_put_u16(name.encode(), img, w, h), "ref")
            else:
                _check(R.pxref_put_bool(name.encode(), img.astype(np.uint8), w, h), "ref")
        ms = C.c_double()
        tasks = C.c_int()
        buf = C.create_string_buffer(1 << 16)
        _check(R.pxref_run(spec.encode(), self.workers, C.byref(ms), C.byref(tasks), buf,
                           1 << 16), "ref")
        res = {}
        for name in outputs:
            k, w, h = C.c_int(), C.c_int(), C.c_int()
            _check(R.pxref_get(name.encode(), C.byref(k), C.byref(w), C.byref(h), None), "ref")
            dt = {0: np.uint8, 1: np.uint16, 2: np.uint32}[k.value]
            out = np.zeros((h.value, w.value), dt)
            _check(R.pxref_get(name.encode(), C.byref(k), C.byref(w), C.byref(h),
                               out.ctypes.data), "ref")
            res[name] = out
        prints = [l for l in buf.value.decode().split("\n") if l]
        return {"computation_ms": ms.value, "tasks": tasks.value, "prints": prints,
                "outputs": res}

    def dump(self, spec: str, stdlib: str) -> str:
        self.R.pxref_set_stdlib(stdlib.encode())
        buf = C.create_string_buffer(1 << 20)
        n = self.R.pxref_dump(spec.encode(), buf, 1 << 20)
        if n < 0:
            raise OracleError(self.R.pxref_last_error().decode())
        return buf.value.decode()
