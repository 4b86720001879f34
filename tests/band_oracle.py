"""CPU restatement of the cross-band merge rules (TEST INFRASTRUCTURE).

The product resolves components that cross row-band borders on the device
(paper_2010_07284_b200/csrc/bands.cu).  This numpy version states the same rules
-- 8-connected border edges, a union-find over (band, component) nodes, seeded
sets for reach, max global label for ccl -- so tests/test_bands.py can check the
RULES against the whole-image oracle on CPU, independently of the kernels.
"""
import numpy as np

from paper_2010_07284_b200.bands import band_rows  # noqa: F401  (re-exported for tests)


def border_edges(last_roots: np.ndarray, last_cls: np.ndarray, first_roots: np.ndarray,
                 first_cls: np.ndarray) -> np.ndarray:
    """Pixel adjacency between the last row of band r and the first row of band
    r+1 (8-connectivity: column offsets -1, 0, +1) as unique (root_a, root_b)."""
    a = last_cls > 0
    b = first_cls > 0
    w = a.size
    pairs = []
    for d in (-1, 0, 1):
        lo, hi = max(0, -d), min(w, w - d)
        m = a[lo:hi] & b[lo + d:hi + d]
        if m.any():
            pairs.append(np.stack([last_roots[lo:hi][m], first_roots[lo + d:hi + d][m]], 1))
    if not pairs:
        return np.zeros((0, 2), np.uint32)
    return np.unique(np.concatenate(pairs).astype(np.uint32), axis=0)


def resolve_border_flags(rows: list) -> list:
    """rows[r] = (first_roots, first_cls, last_roots, last_cls, first_t, last_t) of
    band r: the through-component root and class (2 = seeded in the band,
    1 = unseeded, 0 = background) of every pixel of the band's first and last
    row, and the band's first and last TARGET row (0/1).

    A band seeds only from its own target rows; a component is seeded across a
    border if one of its border pixels touches a target pixel of the
    neighbouring band (near(t) reaches one row into it).  Returns, per band, the
    roots that must become seeded: those in a cross-band component that holds a
    seed.  Nodes are (band, root) pairs; the result is identical on every rank."""
    nb = len(rows)
    keys = []
    seeded = []
    for r, (fr, fc, lr, lc, ft, lt) in enumerate(rows):
        for side, (roots, cls) in enumerate(((fr, fc), (lr, lc))):
            m = cls > 0
            keys.append(np.stack([np.full(m.sum(), r, np.uint64), roots[m].astype(np.uint64)], 1))
            s = cls == 2
            nbr = r - 1 if side == 0 else r + 1
            if 0 <= nbr < nb:
                t = np.asarray(rows[nbr][5 if side == 0 else 4], bool)
                near_t = t.copy()
                near_t[1:] |= t[:-1]
                near_t[:-1] |= t[1:]
                s = s | near_t
            seeded.append(s[m])
    if not keys:
        return [np.zeros(0, np.uint32) for _ in range(nb)]
    allk = np.concatenate(keys)
    if allk.size == 0:
        return [np.zeros(0, np.uint32) for _ in range(nb)]
    packed = (allk[:, 0] << np.uint64(32)) | allk[:, 1]
    uniq, inv = np.unique(packed, return_inverse=True)
    seed_node = np.zeros(uniq.size, bool)
    np.logical_or.at(seed_node, inv, np.concatenate(seeded))
    local_seed = np.zeros(uniq.size, bool)
    np.logical_or.at(local_seed, inv, np.concatenate(
        [(c[c > 0] == 2) for (fr, fc, lr, lc, ft, lt) in rows for c in (fc, lc)]))
    src, dst = [], []
    for r in range(nb - 1):
        e = border_edges(rows[r][2], rows[r][3], rows[r + 1][0], rows[r + 1][1])
        if len(e):
            src.append(np.searchsorted(uniq, (np.uint64(r) << np.uint64(32)) | e[:, 0].astype(np.uint64)))
            dst.append(np.searchsorted(uniq, (np.uint64(r + 1) << np.uint64(32)) | e[:, 1].astype(np.uint64)))
    comp = _components(uniq.size, np.concatenate(src) if src else np.zeros(0, np.int64),
                       np.concatenate(dst) if dst else np.zeros(0, np.int64))
    comp_seeded = np.zeros(comp.max() + 1 if comp.size else 0, bool)
    np.logical_or.at(comp_seeded, comp, seed_node)
    newly = comp_seeded[comp] & ~local_seed
    band = (uniq >> np.uint64(32)).astype(np.int64)
    root = (uniq & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return [root[newly & (band == r)] for r in range(nb)]


def merge_band_labels(rows: list, width: int) -> list:
    """Cross-band CCL label merge.  rows[r] = (first_row_labels,
    last_row_labels, height) of band r, labels band-local (local max index + 1,
    0 = background).  Band r's global labels are local + row0_r * W.  Components
    that touch across a band border (8-connectivity: column offsets -1, 0, +1)
    are united and take the largest global label of the union -- the canonical
    label of the whole-image ccl::label (max index + 1, ccl.hpp:52-60).  Returns,
    per band, (keys: sorted local labels (uint32), vals: new global labels
    (uint64)) for the labels whose global value changes."""
    nb = len(rows)
    row0 = np.cumsum([0] + [int(r[2]) for r in rows[:-1]]).astype(np.uint64)
    W = np.uint64(width)
    src, dst = [], []
    for r in range(nb - 1):
        a = np.asarray(rows[r][1], np.uint64)
        b = np.asarray(rows[r + 1][0], np.uint64)
        for d in (-1, 0, 1):
            lo, hi = max(0, -d), min(width, width - d)
            m = (a[lo:hi] > 0) & (b[lo + d:hi + d] > 0)
            if m.any():
                src.append(a[lo:hi][m] + row0[r] * W)
                dst.append(b[lo + d:hi + d][m] + row0[r + 1] * W)
    if not src:
        return [(np.zeros(0, np.uint32), np.zeros(0, np.uint64)) for _ in range(nb)]
    src, dst = np.concatenate(src), np.concatenate(dst)
    ids, inv = np.unique(np.concatenate([src, dst]), return_inverse=True)
    comp = _components(ids.size, inv[:src.size], inv[src.size:])
    cmax = np.zeros(comp.max() + 1, np.uint64)
    np.maximum.at(cmax, comp, ids)
    new = cmax[comp]
    changed = new != ids
    out = []
    for r in range(nb):
        lo_id = row0[r] * W
        hi_id = lo_id + np.uint64(int(rows[r][2])) * W
        mine = changed & (ids > lo_id) & (ids <= hi_id)
        keys = (ids[mine] - lo_id).astype(np.uint32)
        order = np.argsort(keys)
        out.append((keys[order], new[mine][order]))
    return out


def _components(n: int, src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """Connected components of the undirected border graph (scipy csgraph)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    if n == 0:
        return np.zeros(0, np.int64)
    g = coo_matrix((np.ones(src.size, np.int8), (src, dst)), shape=(n, n))
    return connected_components(g, directed=False)[1].astype(np.int64)
