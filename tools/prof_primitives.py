"""Profiling driver: a few launches of each primitive on config-shaped inputs
(run under ncu; numbers printed here are NOT bench values)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_07284_b200 import Device, DeviceImage, PixelKind, ccl, kernels, maxvol, reach  # noqa: E402
from paper_2010_07284_b200 import synth as S  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--size", type=int, default=4096)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--ops", default="reach,ccl,near,threshold,maxvol")
p.add_argument("--random", type=float, default=0.0, help="random mask density instead of blob")
a = p.parse_args()
dev = Device(0)
n = a.size
if a.random:
    u = S.random_mask(n, n, a.random, S.Rng(1))
    t = S.random_mask(n, n, 0.05, S.Rng(2))
    du = DeviceImage.upload(u, PixelKind.Bool, dev)
    dt = DeviceImage.upload(t, PixelKind.Bool, dev)
    dimg = None
else:
    img = S.blob_noise(n, n, 1)
    dimg = DeviceImage.upload(img, PixelKind.U16, dev)
    du = kernels.threshold(kernels.CmpOp.Gt, dimg, 56360, dev)
    dt = kernels.dilate(kernels.threshold(kernels.CmpOp.Gt, dimg, 62258, dev), dev)
ops = a.ops.split(",")
for _ in range(a.reps):
    if "reach" in ops:
        r = reach(dt, du, dev)
    if "ccl" in ops:
        l = ccl.label(du, dev)
    if "near" in ops:
        x = kernels.dilate(du, dev)
    if "threshold" in ops and dimg is not None:
        y = kernels.threshold(kernels.CmpOp.Gt, dimg, 56360, dev)
    if "maxvol" in ops:
        m = maxvol(du, dev)
dev.synchronize()
print("done")
