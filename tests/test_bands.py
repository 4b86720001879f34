"""CPU: the row-band protocol of paper_2010_07284_b200/bands.py.

The device work of each band (band-local components, seed classes) is
emulated with the oracle, so the host protocol -- border edges, the cross-band
union-find, flag hand-back -- is checked against the full-image reach on CPU,
in-process and across 2 processes with torch.distributed gloo.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from band_oracle import border_edges, merge_band_labels, resolve_border_flags
from paper_2010_07284_b200.bands import band_rows


def test_band_rows_partition():
    for h in (1, 2, 7, 100, 65536):
        for world in (1, 2, 3, 8):
            if world > h:
                continue
            spans = [band_rows(h, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def emulate_band(t_full, u_full, r0, r1):
    """What the device exports for one band: per-pixel (root, class) rows + labels."""
    u = u_full[r0:r1]
    lab = O.flood_fill_label(u)                 # band-local components
    nt = O.dilate(t_full[r0:r1])                # near(t) from the band's own target rows
    seeded = np.zeros(lab.max() + 1, bool)
    seeded[lab[(u > 0) & (nt > 0)]] = True
    seeded[0] = False
    cls = np.where(lab > 0, np.where(seeded[lab], 2, 1), 0).astype(np.uint8)
    roots = (lab * 2654435761).astype(np.uint32)  # any per-band unique ids
    return lab, roots, cls, seeded


def finish_band(lab, roots, seeded, newly):
    extra = np.isin(roots, newly) & (lab > 0)
    return (seeded[lab] & (lab > 0)) | extra


def banded_reach_cpu(t, u, world):
    h = t.shape[0]
    parts = []
    for r in range(world):
        r0, r1 = band_rows(h, world, r)
        lab, roots, cls, seeded = emulate_band(t, u, r0, r1)
        parts.append((r0, r1, lab, roots, cls, seeded))
    rows = [(p[3][0], p[4][0], p[3][-1], p[4][-1], t[p[0]], t[p[1] - 1]) for p in parts]
    newly = resolve_border_flags(rows)
    S = np.zeros_like(u)
    for (r0, r1, lab, roots, cls, seeded), nw in zip(parts, newly):
        S[r0:r1] = finish_band(lab, roots, seeded, nw)
    return O.dilate(O.logical_or(t, S.astype(np.uint8)))


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("w,h,ud", [(40, 37, 0.5), (64, 64, 0.41), (33, 90, 0.6)])
def test_banded_reach_protocol_matches_full_image(world, w, h, ud):
    rng = O.Rng(w * h + world)
    t = O.random_mask(w, h, 0.02, rng)
    u = O.random_mask(w, h, ud, rng)
    assert np.array_equal(banded_reach_cpu(t, u, world), O.reach(t, u))


def test_border_edges_use_8_connectivity():
    last_cls = np.array([0, 1, 0, 0], np.uint8)
    first_cls = np.array([0, 0, 1, 0], np.uint8)   # diagonal neighbour
    e = border_edges(np.array([0, 7, 0, 0], np.uint32), last_cls,
                     np.array([0, 0, 9, 0], np.uint32), first_cls)
    assert e.tolist() == [[7, 9]]
    first_cls = np.array([0, 0, 0, 1], np.uint8)   # two columns away: no edge
    assert len(border_edges(np.array([0, 7, 0, 0], np.uint32), last_cls,
                            np.array([0, 0, 0, 9], np.uint32), first_cls)) == 0


def test_long_component_crossing_many_bands():
    # a vertical line through every band, seeded only in the last band
    h, w = 40, 9
    u = np.zeros((h, w), np.uint8)
    u[:, 4] = 1
    t = np.zeros((h, w), np.uint8)
    t[h - 1, 0] = 0
    t[h - 1, 3] = 1
    assert np.array_equal(banded_reach_cpu(t, u, 8), O.reach(t, u))


def _gloo_worker(rank, world, port, t, u, out):
    """The banded reach protocol through TorchComm (gloo, CPU tensors): border
    records all-gathered as bytes, the merge rule resolved on every rank, halo
    rows exchanged with the neighbours, volume all-reduced."""
    import torch
    import torch.distributed as dist
    from paper_2010_07284_b200.bands import TorchComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    comm = TorchComm()
    h, w = t.shape
    r0, r1 = band_rows(h, world, rank)
    lab, roots, cls, seeded = emulate_band(t, u, r0, r1)
    assert comm.band_heights(r1 - r0) == [b - a for a, b in (band_rows(h, world, r)
                                                              for r in range(world))]
    # border record: roots (u32) + classes + target rows, as one byte tensor
    rec = np.concatenate([roots[0].view(np.uint8), roots[-1].view(np.uint8), cls[0], cls[-1],
                          t[r0], t[r1 - 1]]).astype(np.uint8)
    allrec = torch.empty(world * rec.size, dtype=torch.uint8)
    comm.allgather(torch.from_numpy(rec), allrec)
    recs = allrec.numpy().reshape(world, -1)
    rows = []
    for x in recs:
        rows.append((x[:4 * w].view(np.uint32), x[8 * w:9 * w], x[4 * w:8 * w].view(np.uint32),
                     x[9 * w:10 * w], x[10 * w:11 * w], x[11 * w:12 * w]))
    newly = resolve_border_flags(rows)[rank]
    S = finish_band(lab, roots, seeded, newly).astype(np.uint8)
    band = np.logical_or(t[r0:r1], S).astype(np.uint8)
    # halo: one row up / down, then the closing near of the band
    up = torch.zeros(w, dtype=torch.uint8)
    down = torch.zeros(w, dtype=torch.uint8)
    comm.halo(torch.from_numpy(band[0].copy()), torch.from_numpy(band[-1].copy()), up, down)
    ext = np.concatenate([up.numpy()[None], band, down.numpy()[None]])
    closed = O.dilate(ext)[1:-1]
    vol = torch.tensor([int(closed.sum())], dtype=torch.int64)
    comm.allreduce_sum(vol)
    parts = comm.allgather_object(closed)
    if rank == 0:
        out.put((np.concatenate(parts), int(vol.item())))
    dist.destroy_process_group()


def test_two_process_gloo_banded_reach():
    import torch.multiprocessing as mp
    rng = O.Rng(2024)
    t = O.random_mask(48, 50, 0.03, rng)
    u = O.random_mask(48, 50, 0.5, rng)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, t, u, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, vol = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = O.reach(t, u)
    assert np.array_equal(got, want)
    assert vol == int(want.sum())


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("w,h,d", [(97, 61, 0.41), (64, 200, 0.55), (33, 17, 0.7)])
def test_cross_band_label_merge_matches_whole_image(world, w, h, d):
    # band-local oracle labels + merge_band_labels + the relabel rule must give the
    # whole-image ccl::label labels (canonical max index + 1)
    a = O.random_mask(w, h, d, O.Rng(w * h + world))
    bands = [a[slice(*band_rows(h, world, r))] for r in range(world)]
    local = [O.flood_fill_label(b).astype(np.uint64) for b in bands]
    rows = [(l[0], l[-1], l.shape[0]) for l in local]
    maps = merge_band_labels(rows, w)
    row0 = 0
    out = []
    for l, (keys, vals) in zip(local, maps):
        g = np.where(l > 0, l + np.uint64(row0 * w), 0).astype(np.uint64)
        if keys.size:
            idx = np.searchsorted(keys, l.astype(np.uint32))
            hit = (idx < keys.size) & (keys[np.minimum(idx, keys.size - 1)] == l)
            g = np.where(hit, vals[np.minimum(idx, keys.size - 1)], g)
        out.append(g)
        row0 += l.shape[0]
    assert np.array_equal(np.concatenate(out), O.flood_fill_label(a).astype(np.uint64))
