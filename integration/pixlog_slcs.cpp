// pixlog_slcs.cpp -- the reference's hot-path API served by the B200 library.
//
// This is the C++ a reference maintainer links INSTEAD of the CPU bodies of
// proj/src/kernels.cpp, ccl.cpp and reach.cpp ("Level 1"): the
// same declarations (proj/include/pixlog/kernels.hpp:14-29, ccl.hpp:55-56,
// reach.hpp:15-17), the same argument contracts and RunError texts, with the
// pixel work done by libslcs.so through its C ABI (include/slcs.h).  The
// reference's executor (executor.cpp:74-115, evalTask) and everything above it
// are linked unmodified and call these functions as before.
//
// Also provided, because the reference's own version cannot be built here
// (libpng is absent): png_io (png_io.hpp:12-20) on the library's
// PNG codec (slcs_png_*).  cli_main.cpp and synth_spiral.cpp complete the
// link.
//
// integration/Makefile links this file with the reference objects whose
// replaced symbols were made weak (objcopy -W), so the strong definitions
// here win while e.g. ccl::floodFillLabel, the test oracle, stays the
// reference's own.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "pixlog/ccl.hpp"
#include "pixlog/executor.hpp"
#include "pixlog/kernels.hpp"
#include "pixlog/png_io.hpp"
#include "pixlog/reach.hpp"
#include "slcs.h"

namespace pixlog {
namespace slcs_bridge {

// One process-wide context (device: $SLCS_DEVICE, default 0).  Every entry
// point of the library is thread-safe, so WorkerPool threads share it.
slcs_ctx* ctx() {
  static std::once_flag once;
  static slcs_ctx* c = nullptr;
  static std::string err;
  std::call_once(once, [] {
    const char* d = std::getenv("SLCS_DEVICE");
    if (slcs_ctx_create(d ? std::atoi(d) : 0, nullptr, &c) != SLCS_OK) {
      err = slcs_last_error();
      c = nullptr;
    }
  });
  if (!c) throw RunError("GPU context unavailable: " + err);
  return c;
}

void check(int rc) {
  if (rc != SLCS_OK) throw RunError(slcs_last_error());
}

// RAII device image handle
struct Img {
  slcs_image* p = nullptr;
  Img() = default;
  Img(const Img&) = delete;
  ~Img() {
    if (p) slcs_image_release(p);
  }
};

slcs_kind kindOf(PixelKind k) {
  switch (k) {
    case PixelKind::Bool: return SLCS_BOOL;
    case PixelKind::U16: return SLCS_U16;
    case PixelKind::LabelPair: return SLCS_LABEL;
  }
  return SLCS_BOOL;
}

const void* hostData(const ImageBuffer& img) {
  switch (img.kind()) {
    case PixelKind::Bool: return img.boolData().data();
    case PixelKind::U16: return img.u16Data().data();
    case PixelKind::LabelPair: return img.labelData().data();
  }
  return nullptr;
}

void upload(const ImageBuffer& img, Img& out) {
  check(slcs_image_upload(ctx(), kindOf(img.kind()), img.width(), img.height(), 1, hostData(img),
                          &out.p));
}

}  // namespace slcs_bridge

using slcs_bridge::check;
using slcs_bridge::ctx;

// ---- kernels (kernels.hpp:14-29) -----------------------------------------------
namespace kernels {
namespace {

void requireBool(const ImageBuffer& a, const char* kernel) {  // kernels.cpp:10-14
  if (a.kind() != PixelKind::Bool)
    throw RunError(std::string(kernel) + " expects a boolean image, got " +
                   pixelKindName(a.kind()));
}

void requireSameShape(const ImageBuffer& a, const ImageBuffer& b, const char* kernel) {
  if (!a.sameShape(b))  // kernels.cpp:16-21
    throw RunError(std::string(kernel) + ": dimension mismatch (" + std::to_string(a.width()) +
                   "x" + std::to_string(a.height()) + " vs " + std::to_string(b.width()) + "x" +
                   std::to_string(b.height()) + ")");
}

}  // namespace

ImageBuffer logicalNot(const ImageBuffer& a, WorkerPool&) {
  requireBool(a, "!");
  ImageBuffer out(a.width(), a.height(), PixelKind::Bool);
  check(slcs_h_not(ctx(), a.boolData().data(), a.width(), a.height(), out.boolData().data()));
  return out;
}

ImageBuffer logicalAnd(const ImageBuffer& a, const ImageBuffer& b, WorkerPool&) {
  requireBool(a, "&");
  requireBool(b, "&");
  requireSameShape(a, b, "&");
  ImageBuffer out(a.width(), a.height(), PixelKind::Bool);
  check(slcs_h_and(ctx(), a.boolData().data(), b.boolData().data(), a.width(), a.height(),
                   out.boolData().data()));
  return out;
}

ImageBuffer logicalOr(const ImageBuffer& a, const ImageBuffer& b, WorkerPool&) {
  requireBool(a, "|");
  requireBool(b, "|");
  requireSameShape(a, b, "|");
  ImageBuffer out(a.width(), a.height(), PixelKind::Bool);
  check(slcs_h_or(ctx(), a.boolData().data(), b.boolData().data(), a.width(), a.height(),
                  out.boolData().data()));
  return out;
}

ImageBuffer threshold(CmpOp op, const ImageBuffer& img, double n, WorkerPool&) {
  if (img.kind() != PixelKind::U16)  // kernels.cpp:75-79
    throw RunError(std::string(cmpOpSymbol(op)) + " expects a numeric image, got " +
                   pixelKindName(img.kind()));
  ImageBuffer out(img.width(), img.height(), PixelKind::Bool);
  check(slcs_h_threshold(ctx(), slcs_cmp(int(op)), img.u16Data().data(), img.width(),
                         img.height(), n, out.boolData().data()));
  return out;
}

ImageBuffer dilate(const ImageBuffer& a, WorkerPool&) {
  requireBool(a, "near");
  ImageBuffer out(a.width(), a.height(), PixelKind::Bool);
  check(slcs_h_dilate(ctx(), a.boolData().data(), a.width(), a.height(), out.boolData().data()));
  return out;
}

int64_t countTrue(const ImageBuffer& a, WorkerPool&) {
  requireBool(a, "volume");
  int64_t n = 0;
  check(slcs_h_count_true(ctx(), a.boolData().data(), a.width(), a.height(), &n));
  return n;
}

}  // namespace kernels

// ---- ccl::label (ccl.hpp:55-56) ------------------------------------------------
namespace ccl {
namespace {

void validate(const ImageBuffer& start, const CclConfig& cfg) {
  if (start.kind() != PixelKind::Bool)  // ccl.cpp:13-16
    throw RunError(std::string("component labelling expects a boolean image, got ") +
                   pixelKindName(start.kind()));
  if (cfg.reconnectInterval < 1)  // ccl.cpp:130-132
    throw RunError("reconnect interval must be at least 1, got " +
                   std::to_string(cfg.reconnectInterval));
}

// CclStats of the union-find labelling.  It has no pointer-jumping rounds: one
// labelling pass that always converges.  reconnectWrites -- "label cells
// actually raised" by the reference's atomic repair pass -- is reported as the
// number of merges a union-find over the image's row runs needs: every
// successful union joins two sets, so that is (row runs - components).
void fillStats(const ImageBuffer& start, const ImageBuffer& labels, CclStats* stats) {
  if (!stats) return;
  auto s = start.boolData();
  auto l = labels.labelData();
  const int w = start.width(), h = start.height();
  int64_t runs = 0, comps = 0;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      const size_t i = size_t(r) * w + c;
      if (s[i] && (c == 0 || !s[i - 1])) ++runs;
      if (l[i] == uint32_t(i + 1)) ++comps;  // canonical label = max index + 1
    }
  *stats = CclStats{};
  stats->mainIterations = 1;
  stats->reconnectPasses = 0;
  stats->reconnectWrites = runs - comps;
  stats->totalIterations = 1;
  stats->converged = true;
}

}  // namespace

// cfg.maxRounds bounds the pointer-jumping rounds; the union-find has none and
// always converges, so it cannot trip that guard.  The iteration hook (the
// --debug-ccl PNG dump, executor.cpp:61-70) sees the one final labelling.
ImageBuffer label(const ImageBuffer& start, const CclConfig& cfg, WorkerPool&, CclStats* stats,
                  const IterationHook& hook) {
  validate(start, cfg);
  ImageBuffer out(start.width(), start.height(), PixelKind::LabelPair);
  check(slcs_h_ccl_label(ctx(), start.boolData().data(), start.width(), start.height(),
                         out.labelData().data()));
  fillStats(start, out, stats);
  if (hook) hook(1, out);
  return out;
}

}  // namespace ccl

// ---- reach (reach.hpp:15-17) ---------------------------------------------------
ImageBuffer reach(const ImageBuffer& target, const ImageBuffer& through, WorkerPool& pool,
                  const ccl::CclConfig& cfg, ccl::CclStats* stats,
                  const ccl::IterationHook& hook) {
  if (target.kind() != PixelKind::Bool || through.kind() != PixelKind::Bool)
    throw RunError("reach expects boolean images");  // reach.cpp:13-14
  if (!target.sameShape(through))
    throw RunError("reach: dimension mismatch (" + std::to_string(target.width()) + "x" +
                   std::to_string(target.height()) + " vs " + std::to_string(through.width()) +
                   "x" + std::to_string(through.height()) + ")");
  if (cfg.reconnectInterval < 1)
    throw RunError("reconnect interval must be at least 1, got " +
                   std::to_string(cfg.reconnectInterval));
  // the reference labels `through` (reach.cpp:21) and reports that labelling's
  // stats/hook; the fused reach never materialises labels, so they are produced
  // only when a caller asks for them
  if (stats || hook) ccl::label(through, cfg, pool, stats, hook);
  ImageBuffer out(target.width(), target.height(), PixelKind::Bool);
  check(slcs_h_reach(ctx(), target.boolData().data(), through.boolData().data(), target.width(),
                     target.height(), out.boolData().data()));
  return out;
}

// ---- png_io (png_io.hpp:12-20) on the library's codec ----------------------------
Value loadPng(const std::filesystem::path& path) {
  slcs_bridge::Img img;
  check(slcs_png_load(ctx(), path.string().c_str(), &img.p));
  int kind = 0, w = 0, h = 0, batch = 0;
  check(slcs_image_info(img.p, &kind, &w, &h, &batch));
  ImageBuffer out(w, h, PixelKind::U16);
  check(slcs_image_download(ctx(), img.p, out.u16Data().data(), out.pixelCount() * 2));
  return Value::image(std::move(out));
}

void savePng(const std::filesystem::path& path, const Value& v) {
  if (!v.isImage())  // png_io.cpp:96-97
    throw RunError("cannot save a number as an image (use print): " + path.string());
  slcs_bridge::Img img;
  slcs_bridge::upload(v.img(), img);
  check(slcs_png_save(ctx(), img.p, path.string().c_str()));
}

void labelColor(uint32_t packed, uint8_t rgb[3]) { slcs_label_color(packed, rgb); }

}  // namespace pixlog
