"""Reference-pinned checksums at the BASELINE sizes (tests/golden/large_checksums.json).

TEST INFRASTRUCTURE.  Every number written here is an output of the UNMODIFIED
reference hot path (/root/reference/proj/src compiled in place by
oracle/Makefile into oracle/_ref/libpixlog_ref.so, Release flags), hashed with
the reference's FNV-1a (proj/src/synth.cpp:162-184, restated in
oracle/slcs_oracle.c) over the reference's host layout: Bool = one 0/1 byte per
pixel, labels = little-endian uint32 (image.hpp:20-34).  Inputs are the
reference's own fixtures:

  c2  4096^2 blob-noise seed 1 (synth.cpp:43-81) through the BASELINE config-2
      near/reach chain (synth.near_reach_chain), run by executor::run
      (executor.cpp:231-282); checksums of x2, x20, x100, x500 and x1000.
  c4  randomMask(16384, 16384, d, Rng(1)) for d in 0.41/0.5/0.7
      (tests/oracles.cpp:44-49) -> ccl::label (ccl.cpp:127-165) and
      reach(randomMask(.., 0.05, Rng(2)), mask) (reach.cpp:10-50).
  c3  155 blob-noise 240^2 slices, seeds 100..254, through executor::run of
      grow(hI, vI) and surrounded(hI, vI) (stdlib.imgql:11,14); maxvol (a NEW
      opcode, no reference) is derived from the reference's own ccl::label
      of grow (largest components by pixel count, ties kept).
  c5  65536^2: randomMask(.., 0.5, Rng(1)) -> dilate^4 (kernels.cpp:99-124)
      and countTrue (kernels.cpp:126-136); a uniform u16 image (pixel i =
      Rng(3) draw i % 65536, i.e. Rng::below(65536) per pixel) thresholded
      `>. 32768` (kernels.cpp:75-97).  Labels/reach cannot run here: the
      reference cannot allocate a 65536^2 label image (image.cpp:26-28).
  fig3 the paper's Fig. 3 workload: specs/segmentation.imgql
      (grow(hI, vI)) on a 7680^2 blob-noise image, seed 1.

Run in the container that has /root/reference (each section is independent):
    python tests/golden/make_golden_large.py c3 c4 c5 fig3 c2
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2010_07284_b200 import synth as S  # noqa: E402
from paper_2010_07284_b200.imgql import STDLIB  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large_checksums.json")
WORKERS = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 8))


def hx(a) -> str:
    return f"{O.checksum(np.ascontiguousarray(a)):016x}"


def sha(a) -> str:
    """sha256 of the same bytes: bench.py checks its timed output with this (the
    stdlib hashes 16 MiB in milliseconds; bench.py may not call the oracle)."""
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save(section: str, data: dict) -> None:
    cur = json.load(open(OUT)) if os.path.exists(OUT) else {}
    cur[section] = data
    with open(OUT + ".tmp", "w") as f:
        json.dump(cur, f, indent=1, sort_keys=True)
    os.replace(OUT + ".tmp", OUT)
    print(f"[{section}] written", flush=True)


def random_u16(w: int, h: int, seed: int) -> np.ndarray:
    """Pixel i = (i-th splitmix64(seed) draw) % 65536 (Rng::below, rng.hpp:21-23)."""
    out = np.empty(w * h, np.uint16)
    step = 1 << 26
    for s in range(0, w * h, step):
        n = min(step, w * h - s)
        out[s:s + n] = (S.stream(seed, s, n) & np.uint64(0xFFFF)).astype(np.uint16)
    return out.reshape(h, w)


def c2(R):
    img = R.blob_noise(4096, 4096, 1)
    depth = 1000
    spec = S.near_reach_chain(depth)
    keep = [2, 20, 100, 500, 1000]
    extra = "".join(f'save "d{k}.png" x{k}\n' for k in keep if k != depth)
    t0 = time.time()
    res = R.run(spec + extra, {"img.png": img}, STDLIB, ["out.png"] + [f"d{k}.png" for k in keep
                                                                         if k != depth])
    dt = time.time() - t0
    outs = {k: res["outputs"]["out.png" if k == depth else f"d{k}.png"] for k in keep}
    sums = {f"x{k}": hx(v) for k, v in outs.items()}
    shas = {f"x{k}": sha(v) for k, v in outs.items()}
    save("c2", {"image": "4096x4096 blob-noise seed 1", "depth": depth, "checksums": sums,
                "sha256": shas,
                "volume_x1000": int(res["outputs"]["out.png"].sum()),
                "reference_seconds": round(dt, 1), "workers": WORKERS})


def c4(R):
    n = 16384
    t = O.random_mask(n, n, 0.05, O.Rng(2))
    out = {"image": f"{n}x{n}", "target": "randomMask density 0.05 Rng(2)",
           "target_checksum": hx(t), "workers": WORKERS}
    for d in (0.41, 0.5, 0.7):
        m = O.random_mask(n, n, d, O.Rng(1))
        t0 = time.time()
        lab = R.ccl_label(m)
        t1 = time.time()
        rc = R.reach(t, m)
        t2 = time.time()
        out[f"d{d}"] = {"mask": hx(m), "ccl": hx(lab), "reach": hx(rc),
                        "ccl_sha256": sha(lab), "reach_sha256": sha(rc),
                        "components": int(np.unique(lab).size - (1 if (lab == 0).any() else 0)),
                        "reach_volume": int(rc.sum()),
                        "ccl_seconds": round(t1 - t0, 1), "reach_seconds": round(t2 - t1, 1)}
        print(f"[c4] d={d}: ccl {t1 - t0:.1f}s reach {t2 - t1:.1f}s", flush=True)
        del lab, rc, m
    save("c4", out)


def maxvol_from_labels(lab: np.ndarray) -> np.ndarray:
    flat = lab.ravel()
    if not flat.any():
        return np.zeros(lab.shape, np.uint8)
    uniq, cnt = np.unique(flat[flat != 0], return_counts=True)
    best = uniq[cnt == cnt.max()]
    return np.isin(lab, best).astype(np.uint8)


def c3(R):
    spec = ('load img = "slice.png"\nlet hI = intensity(img) >. 62258\n'
            'let vI = intensity(img) >. 56360\n'
            'save "grow.png" grow(hI, vI)\nsave "sur.png" surrounded(hI, vI)\n')
    per = []
    allout = []
    t0 = time.time()
    for seed in range(100, 255):
        img = R.blob_noise(240, 240, seed)
        res = R.run(spec, {"slice.png": img}, STDLIB, ["grow.png", "sur.png"])
        g, su = res["outputs"]["grow.png"], res["outputs"]["sur.png"]
        mv = maxvol_from_labels(R.ccl_label(g))
        seg = (mv | su).astype(np.uint8)
        allout.append(seg)
        per.append({"seed": seed, "grow": hx(g), "surrounded": hx(su), "maxvol": hx(mv),
                    "segmentation": hx(seg)})
    batch = np.stack(allout)
    save("c3", {"spec": S.SEGMENTATION_SPEC, "slices": per, "batch_checksum": hx(batch),
                "batch_sha256": sha(batch),
                "note": "maxvol derived from the reference's ccl::label of grow (new opcode)",
                "reference_seconds": round(time.time() - t0, 1)})


def c5(R):
    n = 65536
    m = O.random_mask(n, n, 0.5, O.Rng(1))
    out = {"image": f"{n}x{n}", "mask": "randomMask density 0.5 Rng(1)", "mask_checksum": hx(m),
           "workers": WORKERS}
    t0 = time.time()
    out["volume"] = int(R.count_true(m))
    x = m
    for k in range(1, 5):
        x = R.dilate(x)
        if k in (1, 4):
            out[f"near{k}"] = hx(x)
            out[f"near{k}_sha256"] = sha(x)
    del x
    out["near_seconds"] = round(time.time() - t0, 1)
    del m
    img = random_u16(n, n, 3)
    out["u16"] = "pixel i = Rng(3) draw i % 65536"
    out["u16_checksum"] = hx(img)
    thr = R.threshold(0, img, 32768.0)
    out["threshold_gt_32768"] = hx(thr)
    out["threshold_gt_32768_sha256"] = sha(thr)
    out["threshold_volume"] = int(thr.sum(dtype=np.int64))
    save("c5", out)


def fig3(R):
    n = 7680
    img = R.blob_noise(n, n, 1)
    spec = open("/root/reference/proj/specs/segmentation.imgql").read()
    t0 = time.time()
    res = R.run(spec, {"input.png": img}, STDLIB, ["segmentation.png"])
    seg = res["outputs"]["segmentation.png"]
    save("fig3", {"image": f"{n}x{n} blob-noise seed 1", "spec": "specs/segmentation.imgql",
                  "input_checksum": hx(img), "segmentation": hx(seg),
                  "segmentation_sha256": sha(seg),
                  "volume": int(seg.sum(dtype=np.int64)),
                  "reference_computation_ms": round(res["computation_ms"], 1),
                  "reference_seconds": round(time.time() - t0, 1), "workers": WORKERS})


def main():
    R = O.Reference(workers=WORKERS)
    for sec in sys.argv[1:] or ["c3", "c4", "c5", "fig3", "c2"]:
        print(f"[{sec}] start", flush=True)
        globals()[sec](R)


if __name__ == "__main__":
    main()
