import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2010_07284_b200 import Device, DeviceImage, PixelKind, ccl, maxvol, reach
dev = Device(0)
fails = 0
for (w, h) in [(240, 240), (127, 129), (256, 256), (64, 64), (300, 200), (1000, 1000)]:
    for d in (0.2, 0.41, 0.5, 0.7, 0.97):
        for rep in range(3):
            rng = O.Rng(w * 7 + h * 13 + int(d * 100) + 1000 * rep)
            a = O.random_mask(w, h, d, rng)
            got = ccl.label(DeviceImage.upload(a, PixelKind.Bool, dev)).numpy()
            ref = O.flood_fill_label(a)
            nb = int((got != ref).sum())
            if nb:
                fails += 1
                print(f"FAIL {w}x{h} d={d} rep={rep}: {nb} px differ; first {np.argwhere(got != ref)[:3].tolist()}")
                if fails == 1:
                    np.savez_compressed("gpurun_out/fail_case.npz", a=a, got=got, ref=ref)
print("fails", fails)
