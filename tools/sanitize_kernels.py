"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs the union-find kernels on the paths they take at small sizes -- k_small
(<= 256^2), the cooperative fused reach (k_reach_fused, <= 592 tiles) and the
tiled path (k_tile_local -> k_tile_merge -> k_root_flatten -> labels / select,
forced with SLCS_NO_FUSED_REACH=1 or by size) -- plus maxvol, the stencils with
halo rows and the cross-band merges, and checks every result against the
oracle, so a sanitizer run also shows the results stayed exact.

  compute-sanitizer --tool racecheck python tools/sanitize_kernels.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (checker)
from paper_2010_07284_b200 import (DeviceImage, Device, PixelKind, ccl, kernels, maxvol,  # noqa
                                   reach)
from paper_2010_07284_b200.bands import (LocalGroup, band_rows, ccl_banded, near_banded,  # noqa
                                         reach_banded)

dev = Device(0)
n_ok = 0
for (w, h, d) in [(256, 256, 0.5), (1024, 1024, 0.41), (1000, 700, 0.5), (2100, 1300, 0.45)]:
    rng = O.Rng(w + h)
    u = O.random_mask(w, h, d, rng)
    t = O.random_mask(w, h, 0.02, rng)
    du = DeviceImage.upload(u, PixelKind.Bool, dev)
    dt = DeviceImage.upload(t, PixelKind.Bool, dev)
    assert np.array_equal(ccl.label(du, dev).numpy(), O.flood_fill_label(u)), (w, h, "ccl")
    assert np.array_equal(reach(dt, du, dev).numpy(), O.reach(t, u)), (w, h, "reach")
    assert np.array_equal(maxvol(du, dev).numpy(), O.maxvol(u)), (w, h, "maxvol")
    assert np.array_equal(kernels.dilateK(du, 3, dev).numpy(),
                          O.dilate(O.dilate(O.dilate(u)))), (w, h, "near^3")
    n_ok += 4
    if w >= 1000:
        bands = [DeviceImage.upload(u[slice(*band_rows(h, 3, r))], PixelKind.Bool, dev)
                 for r in range(3)]
        tb = [DeviceImage.upload(t[slice(*band_rows(h, 3, r))], PixelKind.Bool, dev)
              for r in range(3)]
        g = LocalGroup(3)
        got = g.run(lambda c, b: reach_banded(c, b[0], b[1]).numpy(), list(zip(tb, bands)))
        assert np.array_equal(np.concatenate(got), O.reach(t, u)), (w, h, "banded reach")
        got = g.run(lambda c, b: near_banded(c, b, 2).numpy(), bands)
        assert np.array_equal(np.concatenate(got), O.dilate(O.dilate(u))), (w, h, "banded near")
        got = g.run(lambda c, b: ccl_banded(c, b).cpu().numpy(), bands)
        assert np.array_equal(np.concatenate(got), O.flood_fill_label(u).astype(np.int64)), \
            (w, h, "banded ccl")
        n_ok += 3
# the persistent reach chain (k_reach_chain: halo records, arrivals, flag stamps)
# and a program's adjacent volumes (k_volume_multi)
from paper_2010_07284_b200 import synth as S  # noqa: E402
from paper_2010_07284_b200.executor import Program  # noqa: E402
from paper_2010_07284_b200.imgql import compile_text  # noqa: E402
w, h, depth = 900, 700, 12
img = O.blob_noise(w, h, 5)
graph = compile_text(S.near_reach_chain(depth) + 'print "v1" volume(b)\nprint "v2" volume(x0)\n')
out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
prog = Program(graph, dev)
prog.set_input_host("img.png", img, PixelKind.U16)
prog.run()
assert "chain of" in prog.plan, prog.plan
out = np.zeros((h, w), np.uint8)
prog.download(out_task, out)
b, x = O.threshold(0, img, 56360), O.threshold(0, img, 62258)
xs = [x]
for k in range(depth):
    x = O.dilate(x) if k % 2 == 0 else O.reach(x, b)
    xs.append(x)
assert np.array_equal(out, x), "reach chain"
vols = [prog.download(i) for i, t in enumerate(graph.nodes) if t.opcode == "volume"]
assert sorted(vols) == sorted([float(b.sum()), float(xs[0].sum())]), "volumes"
n_ok += 2
dev.synchronize()
print(f"sanitize workload ok: {n_ok} checks, {dev.launches} launches")
