"""Diagnostic: banded vs whole-image reach at growing sizes (mismatch rows)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2010_07284_b200 import Device, reach, kernels
from paper_2010_07284_b200.bands import LocalGroup, band_rows, reach_banded, device_bytes
from paper_2010_07284_b200.pixlog import random_mask_device

dev = Device(0)


def sb(img):
    p, pitch, _ = img.storage()
    return device_bytes(p, pitch * img.height, 0), pitch


for n, world in [(16384, 2), (32768, 2), (40000, 2), (50000, 2), (65535, 2)]:
    spans = [band_rows(n, world, r) for r in range(world)]
    masks = [random_mask_device(n, b - a, 0.5, 1, a, dev) for a, b in spans]
    tgts = [random_mask_device(n, b - a, 0.05, 2, a, dev) for a, b in spans]
    wm = random_mask_device(n, n, 0.5, 1, 0, dev)
    wt = random_mask_device(n, n, 0.05, 2, 0, dev)
    got = LocalGroup(world).run(lambda c, b: reach_banded(c, b[0], b[1]), list(zip(tgts, masks)))
    whole = reach(wt, wm, dev)
    dev.synchronize()
    W, pitch = sb(whole)
    bad = []
    for (a, b), g in zip(spans, got):
        G, _ = sb(g)
        d = (G != W[a * pitch:b * pitch]).view(b - a, pitch).any(1)
        rows = torch.nonzero(d).flatten()
        if rows.numel():
            bad.append((a, b, rows.numel(), int(rows[0]) + a, int(rows[-1]) + a))
    print(n, world, "mismatch bands:", bad, "vol whole", kernels.countTrue(whole, dev),
          "vol bands", sum(kernels.countTrue(g, dev) for g in got), flush=True)
    del got, whole, masks, tgts, wm, wt
    torch.cuda.empty_cache()
