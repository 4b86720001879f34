"""Generates tests/golden/reference_vectors.npz from the REFERENCE itself.

Every array here is an output of the unmodified reference hot path
(/root/reference/proj/src compiled by oracle/Makefile into
oracle/_ref/libpixlog_ref.so): kernels::threshold/logicalNot/And/Or/dilate/
countTrue, ccl::label (pointer jumping), reach, synth::generate, and the
TaskGraph dumps of the ImgQL front end.  Inputs are splitmix64 masks with
the reference's own Rng seeds (rng.hpp, tests/oracles.cpp:44-49).

Run (in the container that has /root/reference):
    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2010_07284_b200.imgql import STDLIB  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")
SPECS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_dags.json")

SPEC_TEXTS = {
    "segmentation": 'load img = "input.png"\nlet hI = intensity(img) >. 62258\n'
                    'let vI = intensity(img) >. 56360\nlet gtv = grow(hI,vI)\n'
                    'save "segmentation.png" gtv\n',
    "c1": 'load img = "img.png"\nlet a = img >. 62258\nlet b = img >. 56360\n'
          'save "out.png" reach(near(near(near(near(a & !b)))), b)\n',
    "contradiction": 'load x = "m.png"\nsave "out.png" near(x) & !near(x)\n',
    "surrounded": 'load a = "a.png"\nload b = "b.png"\nsave "o.png" surrounded(a,b)\n'
                  'print "v" volume(a) / 3\n',
    "prints": 'load x = "m.png"\nprint "vol" volume(x)\nprint "ratio" 1 / 3\n'
              'print "img" near(x)\n',
    "interior": 'load x = "m.png"\nsave "o.png" near(x) | interior(x)\n',
}


def main():
    R = O.Reference(workers=2)
    g = {}
    # kernels (test_kernels.cpp shapes)
    rng = O.Rng(2024)
    for i, (w, h) in enumerate([(11, 9), (33, 17), (64, 64), (100, 37), (240, 240)]):
        a = O.random_mask(w, h, 0.3 + 0.1 * i, rng)
        b = O.random_mask(w, h, 0.5, rng)
        img = np.array([rng.below(65536) for _ in range(w * h)], np.uint16).reshape(h, w)
        g[f"k{i}_a"], g[f"k{i}_b"], g[f"k{i}_img"] = a, b, img
        g[f"k{i}_not"] = R.logical_not(a)
        g[f"k{i}_and"] = R.logical_and(a, b)
        g[f"k{i}_or"] = R.logical_or(a, b)
        g[f"k{i}_dilate"] = R.dilate(a)
        g[f"k{i}_count"] = np.array([R.count_true(a)], np.int64)
        for op in range(5):
            for n in (62258.0, 56360.5, 0.0, 70000.0):
                g[f"k{i}_thr{op}_{int(n * 2)}"] = R.threshold(op, img, n)
    # ccl::label (pointer jumping, k = 8) -- canonical max+1 labels
    rng = O.Rng(36)
    for i in range(8):
        d = 0.1 + rng.unit() * 0.8
        m = O.random_mask(64, 64, d, rng)
        g[f"ccl{i}_in"], g[f"ccl{i}_out"] = m, R.ccl_label(m)
    for i, d in enumerate((0.41, 0.5, 0.7)):
        m = O.random_mask(128, 96, d, O.Rng(500 + i))
        g[f"cclb{i}_in"], g[f"cclb{i}_out"] = m, R.ccl_label(m)
    cc = (R.concave_corner(128, 128) > 0).astype(np.uint8)
    g["concave_in"], g["concave_out"] = cc, R.ccl_label(cc)
    # reach
    rng = O.Rng(43)
    for i in range(8):
        t = O.random_mask(32, 32, 0.05 + rng.unit() * 0.3, rng)
        u = O.random_mask(32, 32, 0.2 + rng.unit() * 0.6, rng)
        g[f"reach{i}_t"], g[f"reach{i}_u"], g[f"reach{i}_out"] = t, u, R.reach(t, u)
    # synth fixtures (checksums + a small image)
    checks = {}
    for (w, h, s) in [(512, 512, 1), (240, 240, 100), (240, 240, 254), (256, 256, 1),
                      (4096, 4096, 1)]:
        checks[f"blob_{w}x{h}_{s}"] = O.checksum(R.blob_noise(w, h, s))
    checks["concave_128"] = O.checksum(R.concave_corner(128, 128))
    g["blob_64_7"] = R.blob_noise(64, 64, 7)
    # whole-formula runs through the reference executor
    img = R.blob_noise(96, 96, 3)
    res = R.run(SPEC_TEXTS["segmentation"], {"input.png": img}, STDLIB, ["segmentation.png"])
    g["seg_in"], g["seg_out"] = img, res["outputs"]["segmentation.png"]
    res = R.run(SPEC_TEXTS["c1"], {"img.png": img}, STDLIB, ["out.png"])
    g["c1_out"] = res["outputs"]["out.png"]
    np.savez_compressed(OUT, **g)
    dags = {k: R.dump(v, STDLIB) for k, v in SPEC_TEXTS.items()}
    with open(SPECS, "w") as f:
        json.dump({"specs": SPEC_TEXTS, "dumps": dags, "checksums": {k: f"{v:016x}" for k, v in
                                                                     checks.items()}},
                  f, indent=1, sort_keys=True)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} B) and {SPECS}")


if __name__ == "__main__":
    main()
