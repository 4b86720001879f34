"""paper_2010_07284_b200 -- B200-native SLCS/ImgQL primitive layer.

The hot path of VoxLogicA-GPU (arXiv 2010.07284): bit-packed boolean image
primitives, union-find connected components, reach and maxvol as
hand-written sm_100a CUDA (``csrc/``), behind the C ABI in ``include/slcs.h``.
``pixlog`` mirrors the reference's primitive API; ``imgql`` + ``executor``
are the host layer that turns ImgQL text into a device-resident program.
"""
from . import _lib  # noqa: F401
from .pixlog import (CmpOp, Device, DeviceImage, ImageBuffer, PixelKind, RunError,  # noqa: F401
                     ccl, decodePng, grow, interior, kernels, kNullLabel, labelColor, loadPng,
                     mask, maxvol, packLabel, reach, savePng, surrounded, touch, unpackLabel)

__all__ = ["CmpOp", "Device", "DeviceImage", "ImageBuffer", "PixelKind", "RunError", "ccl",
           "decodePng", "grow", "interior", "kernels", "kNullLabel", "labelColor", "loadPng",
           "mask", "maxvol", "packLabel", "reach", "savePng", "surrounded", "touch", "unpackLabel"]
