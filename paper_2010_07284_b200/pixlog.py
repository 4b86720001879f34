"""Host-side mirror of the reference's primitive API, backed by the sm_100a
library through the C ABI.

Names, argument meaning and error behaviour follow the reference so the
parity tests read like its own suites:

=============================  ==============================================
reference (proj/)              here
=============================  ==============================================
``PixelKind`` image.hpp:16      ``PixelKind``
``ImageBuffer`` image.hpp:38    ``ImageBuffer`` (host, numpy-backed)
``packLabel`` image.hpp:25      ``packLabel`` / ``unpackLabel`` / ``kNullLabel``
``RunError`` errors.hpp:52      ``RunError``
``kernels::*`` kernels.hpp      ``kernels.threshold/logicalNot/logicalAnd/
                                logicalOr/dilate/countTrue/arith``
``ccl::label`` ccl.hpp:55       ``ccl.label`` (``ccl.floodFillLabel`` is the
                                oracle and lives in ``oracle/``, not here)
``reach`` reach.hpp:15          ``reach``
=============================  ==============================================

Every function accepts a host ``ImageBuffer`` (host in -> host out, like the
reference) or a ``DeviceImage`` (device in -> device out, no copies).  There
is no CPU fallback: without the CUDA library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from typing import Optional, Union

import numpy as np

from . import _lib


class RunError(RuntimeError):
    """Evaluation error (proj/include/pixlog/errors.hpp:52-76)."""

    def __init__(self, message: str, code: int = 8):
        super().__init__(message)
        self.code = code


class PixelKind(enum.IntEnum):
    Bool = 0
    U16 = 1
    LabelPair = 2


_KIND_NAME = {PixelKind.Bool: "bool", PixelKind.U16: "u16", PixelKind.LabelPair: "label"}
_DTYPE = {PixelKind.Bool: np.uint8, PixelKind.U16: np.uint16, PixelKind.LabelPair: np.uint32}

kNullLabel = 0


def pixelKindName(k: PixelKind) -> str:
    return _KIND_NAME[PixelKind(k)]


def packLabel(row: int, col: int, width: int) -> int:
    return row * width + col + 1


def unpackLabel(label: int, width: int) -> tuple[int, int]:
    assert label != kNullLabel
    v = label - 1
    return v // width, v % width


class CmpOp(enum.IntEnum):
    Gt = 0
    Ge = 1
    Lt = 2
    Le = 3
    Eq = 4


_CMP_SYMBOL = {CmpOp.Gt: ">.", CmpOp.Ge: ">=.", CmpOp.Lt: "<.", CmpOp.Le: "<=.", CmpOp.Eq: "=."}


def cmpOpSymbol(op: CmpOp) -> str:
    return _CMP_SYMBOL[CmpOp(op)]


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.load().slcs_last_error().decode()
        raise RunError(msg, rc)


# --------------------------------------------------------------------------
class Device:
    """A context on one GPU (slcs_ctx): stream + stream-ordered memory pool."""

    _defaults: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        L = _lib.load()
        h = C.c_void_p()
        _check(L.slcs_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.handle = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Device":
        with cls._lock:
            d = cls._defaults.get(device)
            if d is None:
                d = cls._defaults[device] = Device(device)
            return d

    def synchronize(self) -> None:
        _check(_lib.load().slcs_ctx_synchronize(self.handle))

    @property
    def stream(self) -> int:
        return _lib.load().slcs_ctx_stream(self.handle) or 0

    @property
    def launches(self) -> int:
        return int(_lib.load().slcs_ctx_launch_count(self.handle))

    def close(self) -> None:
        if self.handle:
            _lib.load().slcs_ctx_destroy(self.handle)
            self.handle = None


class DeviceImage:
    """Refcounted device image handle (mirrors shared_ptr<const ImageBuffer>)."""

    __slots__ = ("handle", "device", "kind", "width", "height", "batch", "__weakref__")

    def __init__(self, handle: C.c_void_p, device: Device):
        self.handle = handle
        self.device = device
        k, w, h, b = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_lib.load().slcs_image_info(handle, C.byref(k), C.byref(w), C.byref(h),
                                           C.byref(b)))
        self.kind = PixelKind(k.value)
        self.width, self.height, self.batch = w.value, h.value, b.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib._lib is not None:
            _lib._lib.slcs_image_release(h)
            self.handle = None

    def pixelCount(self) -> int:
        return self.width * self.height

    def numpy(self) -> np.ndarray:
        dt = _DTYPE[self.kind]
        shape = (self.height, self.width) if self.batch == 1 else (self.batch, self.height,
                                                                  self.width)
        out = np.empty(shape, dt)
        _check(_lib.load().slcs_image_download(self.device.handle, self.handle,
                                               out.ctypes.data, out.nbytes))
        return out

    def download(self) -> "ImageBuffer":
        return ImageBuffer.from_array(self.numpy(), self.kind)

    def storage(self) -> tuple[int, int, int]:
        p, rp, sp = C.c_void_p(), C.c_size_t(), C.c_size_t()
        _check(_lib.load().slcs_image_storage(self.handle, C.byref(p), C.byref(rp), C.byref(sp)))
        return p.value, rp.value, sp.value

    @staticmethod
    def upload(arr: np.ndarray, kind: PixelKind, device: Optional[Device] = None
               ) -> "DeviceImage":
        device = device or Device.default()
        a = np.ascontiguousarray(arr, _DTYPE[PixelKind(kind)])
        if a.ndim == 2:
            b, (h, w) = 1, a.shape
        elif a.ndim == 3:
            b, h, w = a.shape
        else:
            raise RunError("image arrays must be 2-D (H, W) or 3-D (batch, H, W)", 7)
        hd = C.c_void_p()
        _check(_lib.load().slcs_image_upload(device.handle, int(kind), w, h, b, a.ctypes.data,
                                             C.byref(hd)))
        return DeviceImage(hd, device)

    @staticmethod
    def from_device(ptr: int, kind: PixelKind, width: int, height: int, batch: int = 1,
                    device: Optional[Device] = None) -> "DeviceImage":
        """Copy from device memory in the reference dense layout (e.g. a torch tensor's
        data_ptr()), packing on the device; no host round trip."""
        device = device or Device.default()
        hd = C.c_void_p()
        _check(_lib.load().slcs_image_from_device(device.handle, int(kind), width, height, batch,
                                                  C.c_void_p(ptr), C.byref(hd)))
        return DeviceImage(hd, device)

    def __repr__(self):
        return f"DeviceImage({self.width}x{self.height},{pixelKindName(self.kind)},batch={self.batch})"


class ImageBuffer:
    """Dense row-major host image (proj/include/pixlog/image.hpp:36-75)."""

    def __init__(self, width: int, height: int, kind: PixelKind, data: Optional[np.ndarray] = None):
        if width < 1 or height < 1:
            raise RunError(f"image dimensions must be at least 1x1, got {width}x{height}", 2)
        kind = PixelKind(kind)
        if kind == PixelKind.LabelPair and width * height >= 0xFFFFFFFE:
            raise RunError("image too large for packed coordinate labels", 3)
        self._w, self._h, self._kind = width, height, kind
        if data is None:
            data = np.zeros((height, width), _DTYPE[kind])
        self.data = np.ascontiguousarray(data, _DTYPE[kind]).reshape(height, width)

    @staticmethod
    def from_array(a: np.ndarray, kind: PixelKind) -> "ImageBuffer":
        a = np.asarray(a)
        if a.ndim == 3 and a.shape[0] == 1:
            a = a[0]
        h, w = a.shape
        return ImageBuffer(w, h, kind, a)

    def width(self) -> int:
        return self._w

    def height(self) -> int:
        return self._h

    def kind(self) -> PixelKind:
        return self._kind

    def pixelCount(self) -> int:
        return self._w * self._h

    def idx(self, row: int, col: int) -> int:
        return row * self._w + col

    def inBounds(self, row: int, col: int) -> bool:
        return 0 <= row < self._h and 0 <= col < self._w

    def sameShape(self, o: "ImageBuffer") -> bool:
        return self._w == o._w and self._h == o._h

    def boolAt(self, r: int, c: int) -> bool:
        return bool(self.data[r, c])

    def u16At(self, r: int, c: int) -> int:
        return int(self.data[r, c])

    def labelAt(self, r: int, c: int) -> int:
        return int(self.data[r, c])

    def __eq__(self, o: object) -> bool:
        return (isinstance(o, ImageBuffer) and self._w == o._w and self._h == o._h
                and self._kind == o._kind and np.array_equal(self.data, o.data))

    def to_device(self, device: Optional[Device] = None) -> DeviceImage:
        return DeviceImage.upload(self.data, self._kind, device)

    def __repr__(self):
        return f"ImageBuffer({self._w}x{self._h},{pixelKindName(self._kind)})"


Image = Union[ImageBuffer, DeviceImage]


def _dev(img: Image, device: Optional[Device]) -> tuple[DeviceImage, bool]:
    if isinstance(img, DeviceImage):
        return img, False
    if isinstance(img, ImageBuffer):
        return img.to_device(device), True
    raise RunError("expected an ImageBuffer or DeviceImage", 7)


def _kind(img: Image) -> PixelKind:
    return img.kind() if isinstance(img, ImageBuffer) else img.kind


def _shape(img: Image) -> tuple[int, int]:
    if isinstance(img, ImageBuffer):
        return img.width(), img.height()
    return img.width, img.height


def _wrap(h: C.c_void_p, device: Device) -> DeviceImage:
    return DeviceImage(h, device)


def _require_bool(a: Image, kernel: str) -> None:
    # kernels.cpp:10-14 -- the kernel level does not coerce (evalTask does)
    if _kind(a) != PixelKind.Bool:
        raise RunError(f"{kernel} expects a boolean image, got {pixelKindName(_kind(a))}", 1)


def _require_same_shape(a: Image, b: Image, kernel: str) -> None:
    (aw, ah), (bw, bh) = _shape(a), _shape(b)
    if (aw, ah) != (bw, bh):
        raise RunError(f"{kernel}: dimension mismatch ({aw}x{ah} vs {bw}x{bh})", 2)


def _call(fn_name: str, args: list, inputs: list, device: Optional[Device]):
    """Runs a primitive; host inputs give a host result, device inputs a device one."""
    host = any(isinstance(x, ImageBuffer) for x in inputs)
    dev_inputs = []
    for x in inputs:
        d, _ = _dev(x, device or (x.device if isinstance(x, DeviceImage) else None))
        dev_inputs.append(d)
    ctx = device or dev_inputs[0].device
    out = C.c_void_p()
    fn = getattr(_lib.load(), fn_name)
    call_args = [ctx.handle]
    it = iter(dev_inputs)
    for a in args:
        call_args.append(next(it).handle if a is _IMG else a)
    _check(fn(*call_args, C.byref(out)))
    res = _wrap(out, ctx)
    return res.download() if host else res


_IMG = object()  # placeholder for an image argument in _call


class kernels:
    """kernels:: namespace (proj/include/pixlog/kernels.hpp:14-29)."""

    CmpOp = CmpOp

    @staticmethod
    def threshold(op: CmpOp, img: Image, n: float, device: Optional[Device] = None):
        if _kind(img) != PixelKind.U16:
            raise RunError(f"{cmpOpSymbol(op)} expects a numeric image, got "
                           f"{pixelKindName(_kind(img))}", 1)
        return _call("slcs_threshold", [int(op), _IMG, float(n)], [img], device)

    @staticmethod
    def logicalNot(a: Image, device: Optional[Device] = None):
        _require_bool(a, "!")
        return _call("slcs_not", [_IMG], [a], device)

    @staticmethod
    def logicalAnd(a: Image, b: Image, device: Optional[Device] = None):
        _require_bool(a, "&"); _require_bool(b, "&"); _require_same_shape(a, b, "&")
        return _call("slcs_and", [_IMG, _IMG], [a, b], device)

    @staticmethod
    def logicalOr(a: Image, b: Image, device: Optional[Device] = None):
        _require_bool(a, "|"); _require_bool(b, "|"); _require_same_shape(a, b, "|")
        return _call("slcs_or", [_IMG, _IMG], [a, b], device)

    @staticmethod
    def dilate(a: Image, device: Optional[Device] = None):
        _require_bool(a, "near")
        return _call("slcs_near", [_IMG], [a], device)

    @staticmethod
    def dilateK(a: Image, k: int, device: Optional[Device] = None):
        _require_bool(a, "near")
        return _call("slcs_near_k", [_IMG, int(k)], [a], device)

    @staticmethod
    def erode(a: Image, device: Optional[Device] = None):
        """stdlib interior(a) = !near(!a) (stdlib.imgql:5), one launch."""
        _require_bool(a, "interior")
        return _call("slcs_interior", [_IMG], [a], device)

    @staticmethod
    def erodeK(a: Image, k: int, device: Optional[Device] = None):
        _require_bool(a, "interior")
        return _call("slcs_interior_k", [_IMG, int(k)], [a], device)

    @staticmethod
    def countTrue(a: Image, device: Optional[Device] = None) -> int:
        _require_bool(a, "volume")
        d, _ = _dev(a, device)
        n = max(1, getattr(d, "batch", 1))
        out = (C.c_int64 * n)()
        _check(_lib.load().slcs_volume((device or d.device).handle, d.handle, out))
        return int(out[0]) if n == 1 else [int(x) for x in out]

    @staticmethod
    def arith(op: str, x: float, y: float) -> float:
        # kernels.cpp:138-148 -- scalar arithmetic stays on the host
        if op == "+":
            return x + y
        if op == "-":
            return x - y
        if op == "*":
            return x * y
        if op == "/":
            if y == 0.0:
                raise RunError("division by zero")
            return x / y
        raise RunError(f"unknown arithmetic operator '{op}'")


class ccl:
    """ccl:: namespace (proj/include/pixlog/ccl.hpp:33-60)."""

    @staticmethod
    def label(start: Image, device: Optional[Device] = None):
        if _kind(start) != PixelKind.Bool:
            raise RunError("component labelling expects a boolean image, got "
                           f"{pixelKindName(_kind(start))}", 1)
        return _call("slcs_ccl", [_IMG], [start], device)


def reach(target: Image, through: Image, device: Optional[Device] = None):
    """reach(target, through) (proj/include/pixlog/reach.hpp:15-17)."""
    if _kind(target) != PixelKind.Bool or _kind(through) != PixelKind.Bool:
        raise RunError("reach expects boolean images", 1)
    (aw, ah), (bw, bh) = _shape(target), _shape(through)
    if (aw, ah) != (bw, bh):
        raise RunError(f"reach: dimension mismatch ({aw}x{ah} vs {bw}x{bh})", 2)
    return _call("slcs_reach", [_IMG, _IMG], [target, through], device)


def maxvol(a: Image, device: Optional[Device] = None):
    """NEW opcode: union of the maximal-volume 8-connected components."""
    _require_bool(a, "maxvol")
    return _call("slcs_maxvol", [_IMG], [a], device)


# stdlib macros composed over the primitives (proj/stdlib/stdlib.imgql:5-14)
def interior(a: Image, device: Optional[Device] = None):
    return kernels.erode(a, device)


def touch(a: Image, b: Image, device: Optional[Device] = None):
    return kernels.logicalAnd(a, reach(b, a, device), device)


def grow(a: Image, b: Image, device: Optional[Device] = None):
    return kernels.logicalOr(a, touch(b, a, device), device)


def surrounded(a: Image, b: Image, device: Optional[Device] = None):
    notAB = kernels.logicalNot(kernels.logicalOr(a, b, device), device)
    notB = kernels.logicalNot(b, device)
    return kernels.logicalAnd(a, kernels.logicalNot(reach(notAB, notB, device), device), device)


def random_mask_device(w: int, h: int, density: float, seed: int, row0: int = 0,
                       device: Optional[Device] = None) -> DeviceImage:
    """Rows [row0, row0+h) of randomMask(w, H, density, Rng(seed)), generated on the GPU
    (bit-identical to the reference fixture, tests/oracles.cpp:44-49)."""
    device = device or Device.default()
    out = C.c_void_p()
    _check(_lib.load().slcs_random_mask(device.handle, w, h, row0, seed, float(density),
                                        C.byref(out)))
    return DeviceImage(out, device)


def random_u16_device(w: int, h: int, seed: int, row0: int = 0,
                      device: Optional[Device] = None) -> DeviceImage:
    """Rows [row0, row0+h) of the uniform u16 fixture (pixel i = draw i of
    splitmix64(seed) % 65536, Rng::below(65536) per pixel), generated on the GPU."""
    device = device or Device.default()
    out = C.c_void_p()
    _check(_lib.load().slcs_random_u16(device.handle, w, h, row0, seed, C.byref(out)))
    return DeviceImage(out, device)


def loadPng(path: str, device: Optional[Device] = None) -> DeviceImage:
    """png_io loadPng (proj/src/png_io.cpp:30-73): a U16 device image (first channel,
    8-bit samples widened by v*257)."""
    device = device or Device.default()
    out = C.c_void_p()
    _check(_lib.load().slcs_png_load(device.handle, os.fsencode(path), C.byref(out)))
    return DeviceImage(out, device)


def decodePng(data: bytes, device: Optional[Device] = None) -> DeviceImage:
    """loadPng from an in-memory PNG byte stream."""
    device = device or Device.default()
    out = C.c_void_p()
    buf = C.create_string_buffer(data, len(data))
    _check(_lib.load().slcs_png_decode(device.handle, buf, len(data), C.byref(out)))
    return DeviceImage(out, device)


def savePng(path: str, img: Image, device: Optional[Device] = None) -> None:
    """png_io savePng (png_io.cpp:95-143): Bool -> 16-bit grey 0/65535, U16 verbatim,
    labels -> 8-bit RGB via labelColor."""
    d, _ = _dev(img, device)
    _check(_lib.load().slcs_png_save(d.device.handle, d.handle, os.fsencode(path)))


def labelColor(packed: int) -> tuple[int, int, int]:
    """labelColor (png_io.cpp:75-90): lowbias32 colour of a packed label, null -> black."""
    rgb = (C.c_uint8 * 3)()
    _lib.load().slcs_label_color(packed & 0xFFFFFFFF, rgb)
    return rgb[0], rgb[1], rgb[2]


def mask(pattern: str) -> ImageBuffer:
    """ASCII mask helper of tests/oracles.cpp:20-42 ('x', '#', '1' set; '/' rows)."""
    rows = [r for r in pattern.replace("\n", "/").split("/") if r != ""]
    h, w = len(rows), len(rows[0])
    a = np.zeros((h, w), np.uint8)
    for r, row in enumerate(rows):
        for c, ch in enumerate(row):
            a[r, c] = 1 if ch in "x#1" else 0
    return ImageBuffer(w, h, PixelKind.Bool, a)
