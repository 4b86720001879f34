/*
 * slcs_oracle.c -- CPU restatement of the reference's hot-path algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2010_07284_b200/) may link, load or call this file.  It is
 * imported by tests/, by __graft_entry__.smoke() as the checker, and by
 * bench.py's cpu_baseline / --impl reference legs when oracle/_ref is absent.
 *
 * Parity pin: every function below is checked against golden vectors that
 * were produced by the reference itself (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile) -- see tests/golden/ and
 * tests/test_oracle.py.  maxvol has no reference implementation (it is a new
 * opcode); its definition is stated in DESIGN.md and pinned only by
 * hand-computed known answers ("parity unpinned" for maxvol).
 *
 * Layout follows the reference ImageBuffer (proj/include/pixlog/image.hpp:36-75):
 * row-major, origin top-left, Bool = 1 byte per pixel (0/1), U16 = 2 bytes,
 * labels = uint32 packed row*W+col+1 with 0 = null (image.hpp:20-29).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- splitmix64, proj/include/pixlog/rng.hpp:14-33 ---------------------- */

uint64_t or_rng_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static double rng_unit(uint64_t* s) { return (double)(or_rng_next(s) >> 11) * 0x1.0p-53; }
static uint64_t rng_below(uint64_t* s, uint64_t n) { return or_rng_next(s) % n; }

/* randomMask, proj/tests/oracles.cpp:44-49: one chance(density) per pixel in
 * row-major order. */
void or_random_mask(int w, int h, double density, uint64_t* state, uint8_t* out) {
  size_t n = (size_t)w * (size_t)h;
  for (size_t i = 0; i < n; ++i) out[i] = rng_unit(state) < density ? 1 : 0;
}

/* synth::blobNoise, proj/src/synth.cpp:43-81 (bands at synth.cpp:36-39). */
static uint16_t pick(uint64_t* s, uint16_t lo, uint16_t hi) {
  return (uint16_t)(lo + rng_below(s, (uint64_t)(hi - lo + 1)));
}

void or_blob_noise(int w, int h, uint64_t seed, uint16_t* px) {
  uint64_t s = seed;
  const double cr = h / 2.0, cc = w / 2.0;
  double m = (w < h ? w : h) / 6.0;
  const double discR = m > 2.0 ? m : 2.0;
  const double haloR = discR * 2.0;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      size_t i = (size_t)r * w + c;
      double d = hypot(r - cr, c - cc);
      if (d <= discR)
        px[i] = pick(&s, 63000, 65535);
      else if (d <= haloR)
        px[i] = pick(&s, 57500, 61000);
      else
        px[i] = pick(&s, 5000, 30000);
    }
  int want = w * h / 400;
  if (want < 3) want = 3;
  int placed = 0;
  for (int attempt = 0; attempt < want * 20 && placed < want; ++attempt) {
    int r = (int)rng_below(&s, (uint64_t)h);
    int c = (int)rng_below(&s, (uint64_t)w);
    if (hypot(r - cr, c - cc) <= haloR + 4.0) continue;
    px[(size_t)r * w + c] = pick(&s, 57500, 61000);
    ++placed;
  }
}

/* synth::checksum, proj/src/synth.cpp:162-184 (FNV-1a over LE bytes). */
uint64_t or_checksum(const void* data, size_t nbytes) {
  const uint8_t* b = (const uint8_t*)data;
  uint64_t hsh = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < nbytes; ++i) {
    hsh ^= b[i];
    hsh *= 0x100000001b3ull;
  }
  return hsh;
}

/* ---- kernels, proj/src/kernels.cpp ------------------------------------- */

/* kernels::threshold, kernels.cpp:75-97: double(p) op n.  op: 0 >, 1 >=, 2 <,
 * 3 <=, 4 = (CmpOp order, kernels.hpp:10). */
void or_threshold(int op, const uint16_t* src, int w, int h, double n, uint8_t* dst) {
  size_t cnt = (size_t)w * (size_t)h;
  for (size_t i = 0; i < cnt; ++i) {
    double p = (double)src[i];
    int r = 0;
    switch (op) {
      case 0: r = p > n; break;
      case 1: r = p >= n; break;
      case 2: r = p < n; break;
      case 3: r = p <= n; break;
      case 4: r = p == n; break;
    }
    dst[i] = r ? 1 : 0;
  }
}

/* kernels::logicalNot/And/Or, kernels.cpp:36-73. */
void or_not(const uint8_t* a, size_t n, uint8_t* dst) {
  for (size_t i = 0; i < n; ++i) dst[i] = a[i] ? 0 : 1;
}
void or_and(const uint8_t* a, const uint8_t* b, size_t n, uint8_t* dst) {
  for (size_t i = 0; i < n; ++i) dst[i] = (a[i] && b[i]) ? 1 : 0;
}
void or_or(const uint8_t* a, const uint8_t* b, size_t n, uint8_t* dst) {
  for (size_t i = 0; i < n; ++i) dst[i] = (a[i] || b[i]) ? 1 : 0;
}

/* kernels::dilate (= near), kernels.cpp:99-124: clipped 3x3 window, centre
 * included, out-of-image cells absent (false). */
void or_dilate(const uint8_t* a, int w, int h, uint8_t* dst) {
  for (int r = 0; r < h; ++r) {
    int r0 = r > 0 ? r - 1 : 0, r1 = r < h - 1 ? r + 1 : h - 1;
    for (int c = 0; c < w; ++c) {
      int c0 = c > 0 ? c - 1 : 0, c1 = c < w - 1 ? c + 1 : w - 1;
      uint8_t any = 0;
      for (int rr = r0; rr <= r1 && !any; ++rr)
        for (int cc = c0; cc <= c1; ++cc)
          if (a[(size_t)rr * w + cc]) { any = 1; break; }
      dst[(size_t)r * w + c] = any;
    }
  }
}

/* interior = !near(!a) (proj/stdlib/stdlib.imgql:5); equivalently the
 * clipped erosion of tests/oracles.cpp:97-105 (out-of-image absent = true). */
void or_erode(const uint8_t* a, int w, int h, uint8_t* dst) {
  for (int r = 0; r < h; ++r) {
    int r0 = r > 0 ? r - 1 : 0, r1 = r < h - 1 ? r + 1 : h - 1;
    for (int c = 0; c < w; ++c) {
      int c0 = c > 0 ? c - 1 : 0, c1 = c < w - 1 ? c + 1 : w - 1;
      uint8_t all = 1;
      for (int rr = r0; rr <= r1 && all; ++rr)
        for (int cc = c0; cc <= c1; ++cc)
          if (!a[(size_t)rr * w + cc]) { all = 0; break; }
      dst[(size_t)r * w + c] = all;
    }
  }
}

/* kernels::countTrue (= volume), kernels.cpp:126-136. */
int64_t or_count_true(const uint8_t* a, size_t n) {
  int64_t t = 0;
  for (size_t i = 0; i < n; ++i) t += a[i] ? 1 : 0;
  return t;
}

/* ---- component labelling ------------------------------------------------ */

/* ccl::floodFillLabel, proj/src/ccl.cpp:167-202: 8-connected components, each
 * labelled with its lexicographic-max coordinate packed as idx+1.  Returns 0,
 * or -1 when W*H >= 0xFFFFFFFE (image.cpp:26-28) or on allocation failure. */
int or_flood_fill_label(const uint8_t* on, int w, int h, uint32_t* dst) {
  size_t n = (size_t)w * (size_t)h;
  if (n >= 0xfffffffeull) return -1;
  uint8_t* seen = (uint8_t*)calloc(n, 1);
  size_t* stack = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
  size_t* comp = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
  if (!seen || !stack || !comp) {
    free(seen); free(stack); free(comp);
    return -1;
  }
  memset(dst, 0, n * sizeof(uint32_t));
  for (size_t seed = 0; seed < n; ++seed) {
    if (!on[seed] || seen[seed]) continue;
    size_t sp = 0, cn = 0;
    stack[sp++] = seed;
    seen[seed] = 1;
    uint32_t best = 0;
    while (sp) {
      size_t i = stack[--sp];
      comp[cn++] = i;
      int r = (int)(i / (size_t)w), c = (int)(i % (size_t)w);
      uint32_t lab = (uint32_t)i + 1u;
      if (lab > best) best = lab;
      int r0 = r > 0 ? r - 1 : 0, r1 = r < h - 1 ? r + 1 : h - 1;
      int c0 = c > 0 ? c - 1 : 0, c1 = c < w - 1 ? c + 1 : w - 1;
      for (int rr = r0; rr <= r1; ++rr)
        for (int cc = c0; cc <= c1; ++cc) {
          size_t j = (size_t)rr * w + cc;
          if (on[j] && !seen[j]) {
            seen[j] = 1;
            stack[sp++] = j;
          }
        }
    }
    for (size_t k = 0; k < cn; ++k) dst[comp[k]] = best;
  }
  free(seen); free(stack); free(comp);
  return 0;
}

/* reach, proj/src/reach.cpp:10-50: near(t) | near(S) where S is the union of
 * through-components holding a pixel of near(t). */
int or_reach(const uint8_t* t, const uint8_t* u, int w, int h, uint8_t* dst) {
  size_t n = (size_t)w * (size_t)h;
  uint8_t* nt = (uint8_t*)malloc(n ? n : 1);
  uint8_t* sel = (uint8_t*)calloc(n ? n : 1, 1);
  uint8_t* nsel = (uint8_t*)malloc(n ? n : 1);
  uint32_t* lab = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint8_t* flagged = (uint8_t*)calloc(n + 1, 1);
  int rc = -1;
  if (!nt || !sel || !nsel || !lab || !flagged) goto out;
  if (or_flood_fill_label(u, w, h, lab) != 0) goto out;
  or_dilate(t, w, h, nt);
  for (size_t i = 0; i < n; ++i)
    if (lab[i] && nt[i]) flagged[lab[i]] = 1;
  for (size_t i = 0; i < n; ++i) sel[i] = (lab[i] && flagged[lab[i]]) ? 1 : 0;
  or_dilate(sel, w, h, nsel);
  or_or(nt, nsel, n, dst);
  rc = 0;
out:
  free(nt); free(sel); free(nsel); free(lab); free(flagged);
  return rc;
}

/* reachOracle, proj/tests/oracles.cpp:107-150: BFS over the path definition
 * (independent of labelling; used to cross-check or_reach). */
int or_reach_bfs(const uint8_t* t, const uint8_t* u, int w, int h, uint8_t* dst) {
  size_t n = (size_t)w * (size_t)h;
  uint8_t* reached = (uint8_t*)calloc(n ? n : 1, 1);
  size_t* queue = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
  if (!reached || !queue) {
    free(reached); free(queue);
    return -1;
  }
  or_dilate(t, w, h, dst);
  size_t qh = 0, qt = 0;
  for (size_t i = 0; i < n; ++i)
    if (u[i] && dst[i] && !reached[i]) {
      reached[i] = 1;
      queue[qt++] = i;
    }
  while (qh < qt) {
    size_t i = queue[qh++];
    int r = (int)(i / (size_t)w), c = (int)(i % (size_t)w);
    int r0 = r > 0 ? r - 1 : 0, r1 = r < h - 1 ? r + 1 : h - 1;
    int c0 = c > 0 ? c - 1 : 0, c1 = c < w - 1 ? c + 1 : w - 1;
    for (int rr = r0; rr <= r1; ++rr)
      for (int cc = c0; cc <= c1; ++cc) {
        size_t j = (size_t)rr * w + cc;
        if (u[j] && !reached[j]) {
          reached[j] = 1;
          queue[qt++] = j;
        }
      }
  }
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      size_t i = (size_t)r * w + c;
      if (dst[i]) continue;
      int r0 = r > 0 ? r - 1 : 0, r1 = r < h - 1 ? r + 1 : h - 1;
      int c0 = c > 0 ? c - 1 : 0, c1 = c < w - 1 ? c + 1 : w - 1;
      for (int rr = r0; rr <= r1 && !dst[i]; ++rr)
        for (int cc = c0; cc <= c1; ++cc)
          if (reached[(size_t)rr * w + cc]) { dst[i] = 1; break; }
    }
  free(reached); free(queue);
  return 0;
}

/* maxvol (NEW opcode, no reference implementation):
 * the union of the 8-connected components of `a` whose pixel count equals the
 * maximum component pixel count (ties keep every maximal component; an empty
 * input gives an empty output).  Built on the floodFillLabel labelling
 * (ccl.cpp:167-202) plus a size histogram. */
int or_maxvol(const uint8_t* a, int w, int h, uint8_t* dst) {
  size_t n = (size_t)w * (size_t)h;
  uint32_t* lab = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* size = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
  if (!lab || !size) {
    free(lab); free(size);
    return -1;
  }
  if (or_flood_fill_label(a, w, h, lab) != 0) {
    free(lab); free(size);
    return -1;
  }
  uint32_t best = 0;
  for (size_t i = 0; i < n; ++i)
    if (lab[i]) {
      uint32_t s = ++size[lab[i]];
      if (s > best) best = s;
    }
  for (size_t i = 0; i < n; ++i) dst[i] = (lab[i] && size[lab[i]] == best) ? 1 : 0;
  free(lab); free(size);
  return 0;
}
