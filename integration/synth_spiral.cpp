// synth_spiral.cpp -- synth::generate with a terminating Spiral fixture (TEST FIXTURE).
//
// The reference's drawSegment (proj/src/synth.cpp:83-101) tests its Bresenham
// error terms against the wrong axes and never terminates, so
// synth::generate(Spiral, ...) hangs and acceptance criterion 3
// (tests/acceptance_main.cpp:91-108) cannot run.  integration/Makefile renames
// the reference's generate to synth::ref::generate (objcopy --redefine-sym);
// this generate draws the Spiral with the corrected segment walk and forwards
// every other kind to the reference's own code.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "pixlog/rng.hpp"
#include "pixlog/synth.hpp"

namespace pixlog {

// ---- synth: corrected Spiral, everything else the reference's ------------------
namespace synth {
namespace ref {
// the reference's generate (synth.cpp), renamed by objcopy in integration/Makefile
ImageBuffer generate(ImageKind kind, int width, int height, uint64_t seed, BlobNoiseInfo* info);
}  // namespace ref

namespace {
// drawSegment (synth.cpp:83-101) with each error test on its own axis
void drawSegment(ImageBuffer& img, int r0, int c0, int r1, int c1) {
  auto px = img.u16Data();
  const int dr = std::abs(r1 - r0), dc = std::abs(c1 - c0);
  const int sr = r0 < r1 ? 1 : -1, sc = c0 < c1 ? 1 : -1;
  int err = dc - dr;
  for (;;) {
    if (img.inBounds(r0, c0)) px[img.idx(r0, c0)] = 65535;
    if (r0 == r1 && c0 == c1) break;
    const int e2 = 2 * err;
    if (e2 > -dr) {
      err -= dr;
      c0 += sc;
    }
    if (e2 < dc) {
      err += dc;
      r0 += sr;
    }
  }
}

// spiral (synth.cpp:103-124): same curve parameters and seeded phase
ImageBuffer spiral(int w, int h, uint64_t seed) {
  ImageBuffer img(w, h, PixelKind::U16);
  Rng rng(seed);
  const double spacing = 16.0;
  const double a = spacing / (2.0 * M_PI);
  const double cr = h / 2.0, cc = w / 2.0;
  const double maxR = std::min(w, h) / 2.0 - 4.0;
  const double phase = rng.unit() * 2.0 * M_PI;
  double theta = 0.0;
  int pr = int(std::lround(cr)), pc = int(std::lround(cc));
  while (a * theta < maxR) {
    const double r = a * theta;
    const int qr = int(std::lround(cr + r * std::sin(theta + phase)));
    const int qc = int(std::lround(cc + r * std::cos(theta + phase)));
    drawSegment(img, pr, pc, qr, qc);
    pr = qr;
    pc = qc;
    theta += 0.5 / std::max(r, 1.0);
  }
  return img;
}
}  // namespace

ImageBuffer generate(ImageKind kind, int width, int height, uint64_t seed, BlobNoiseInfo* info) {
  if (kind == ImageKind::Spiral) return spiral(width, height, seed);
  return ref::generate(kind, width, height, seed, info);
}
}  // namespace synth

}  // namespace pixlog
