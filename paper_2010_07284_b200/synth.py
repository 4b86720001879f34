"""Deterministic synthetic inputs, bit-identical to the reference fixtures.

* ``Rng`` / ``random_mask`` -- splitmix64 (proj/include/pixlog/rng.hpp:14-33)
  and randomMask (proj/tests/oracles.cpp:44-49).  The i-th draw depends only
  on seed + (i+1)*gamma, so whole masks are generated vectorised.
* ``blob_noise`` -- synth::generate(BlobNoise) (proj/src/synth.cpp:43-81).
* ``near_reach_chain`` -- the BASELINE config-2 formula:
  x0 = img >. 62258, x(2k+1) = near(x(2k)), x(2k+2) = reach(x(2k+1), b),
  b = img >. 56360.
* ``segmentation_spec`` -- the frozen config-3 spec.
* ``spiral`` -- synth::generate(Spiral) (proj/src/synth.cpp:83-124) with the
  Bresenham step conditions corrected (the reference's drawSegment never
  terminates).

Tests check every generator against the C oracle / reference checksums.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
MASK64 = (1 << 64) - 1


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def stream(seed: int, start: int, n: int) -> np.ndarray:
    """Draws start .. start+n-1 of splitmix64(seed), vectorised."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        return _mix(np.uint64(seed) + idx * GAMMA)


class Rng:
    """Scalar splitmix64 with the reference's next/below/unit/chance."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        return self.next() % n

    def unit(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def chance(self, p: float) -> bool:
        return self.unit() < p

    def draws(self, n: int) -> np.ndarray:
        out = stream(self.state, 0, n)
        self.state = (self.state + n * 0x9E3779B97F4A7C15) & MASK64
        return out


def random_mask(w: int, h: int, density: float, rng: Rng) -> np.ndarray:
    z = rng.draws(w * h)
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (u < density).astype(np.uint8).reshape(h, w)


def blob_noise(w: int, h: int, seed: int) -> np.ndarray:
    n = w * h
    z = stream(seed, 0, n)
    r = np.arange(h, dtype=np.float64)[:, None]
    c = np.arange(w, dtype=np.float64)[None, :]
    cr, cc = h / 2.0, w / 2.0
    d = np.hypot(r - cr, c - cc).reshape(-1)
    disc_r = max(2.0, min(w, h) / 6.0)
    halo_r = disc_r * 2.0
    bright = np.uint64(63000) + z % np.uint64(65535 - 63000 + 1)
    mid = np.uint64(57500) + z % np.uint64(61000 - 57500 + 1)
    dark = np.uint64(5000) + z % np.uint64(30000 - 5000 + 1)
    px = np.where(d <= disc_r, bright, np.where(d <= halo_r, mid, dark)).astype(np.uint16)
    # salt specks: sequential draws continuing the stream (synth.cpp:68-80)
    want = max(3, n // 400)
    budget = want * 20
    chunk_len = 4 * want + 1024
    buf, buf_start = stream(seed, n, chunk_len), n
    nxt = n  # absolute index of the next draw

    def draw() -> int:
        nonlocal buf, buf_start, nxt
        if nxt - buf_start >= len(buf):
            buf, buf_start = stream(seed, nxt, chunk_len), nxt
        v = int(buf[nxt - buf_start])
        nxt += 1
        return v

    placed, attempt = 0, 0
    limit = halo_r + 4.0
    while attempt < budget and placed < want:
        rr = draw() % h
        c2 = draw() % w
        attempt += 1
        if np.hypot(rr - cr, c2 - cc) <= limit:
            continue
        px[rr * w + c2] = 57500 + draw() % 3501
        placed += 1
    return px.reshape(h, w)


def _draw_segment(px: np.ndarray, r0: int, c0: int, r1: int, c1: int) -> None:
    """drawSegment (synth.cpp:83-101) with the error terms tested against the
    right axes (`e2 > -dr` -> step c, `e2 < dc` -> step r), i.e. standard Bresenham."""
    h, w = px.shape
    dr, dc = abs(r1 - r0), abs(c1 - c0)
    sr, sc = (1 if r0 < r1 else -1), (1 if c0 < c1 else -1)
    err = dc - dr
    while True:
        if 0 <= r0 < h and 0 <= c0 < w:
            px[r0, c0] = 65535
        if r0 == r1 and c0 == c1:
            return
        e2 = 2 * err
        if e2 > -dr:
            err -= dr
            c0 += sc
        if e2 < dc:
            err += dc
            r0 += sr


def _lround(x: float) -> int:
    """std::lround: halves away from zero."""
    import math
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


def spiral(w: int, h: int, seed: int) -> np.ndarray:
    """synth::generate(Spiral) (synth.cpp:103-124): an Archimedean spiral of
    16-px spacing with a seeded phase, drawn as one connected 8-connected curve."""
    import math
    px = np.zeros((h, w), np.uint16)
    rng = Rng(seed)
    spacing = 16.0
    a = spacing / (2.0 * math.pi)
    cr, cc = h / 2.0, w / 2.0
    max_r = min(w, h) / 2.0 - 4.0
    phase = rng.unit() * 2.0 * math.pi
    theta = 0.0
    pr, pc = int(round(cr)), int(round(cc))
    while a * theta < max_r:
        r = a * theta
        qr = _lround(cr + r * math.sin(theta + phase))
        qc = _lround(cc + r * math.cos(theta + phase))
        _draw_segment(px, pr, pc, qr, qc)
        pr, pc = qr, qc
        theta += 0.5 / max(r, 1.0)
    return px


def near_reach_chain(depth: int, through_thr: float = 56360, target_thr: float = 62258,
                     path: str = "img.png") -> str:
    """BASELINE config 2: `depth` alternating near / reach steps."""
    lines = [f'load img = "{path}"', f"let b = img >. {through_thr:g}",
             f"let x0 = img >. {target_thr:g}"]
    for k in range(depth):
        src = f"x{k}"
        if k % 2 == 0:
            lines.append(f"let x{k + 1} = near({src})")
        else:
            lines.append(f"let x{k + 1} = reach({src}, b)")
    lines.append(f'save "out.png" x{depth}')
    return "\n".join(lines) + "\n"


def sequential_formula(depth: int, path: str = "x.png") -> str:
    """gen::sequentialFormula (proj/src/formula_gen.cpp:8-17): near / ! chain."""
    expr = "x"
    for i in range(depth):
        expr = f"near({expr})" if i % 2 == 0 else f"!({expr})"
    return f'load x = "{path}"\nsave "sequential-out.png" {expr}\n'


# SURVEY.md §8d config 3, frozen here (BASELINE names only the ops)
SEGMENTATION_SPEC = ('load img = "slices.png"\n'
                     'let hI = intensity(img) >. 62258\n'
                     'let vI = intensity(img) >. 56360\n'
                     'let gtv = grow(hI, vI)\n'
                     'save "segmentation.png" maxvol(gtv) | surrounded(hI, vI)\n')
