// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference hot path.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources, read in place from
// /root/reference/proj/src (nothing is copied into this repository), into
// oracle/_ref/libpixlog_ref.so.  Tests use it to generate golden vectors and
// bench.py uses it as the CPU reference arm ("kind": "reference").
//
// Two pieces of the reference cannot be compiled here:
//   * png_io.cpp needs libpng (absent).  loadPng/savePng below are an
//     in-memory registry instead: load "name" returns the image registered
//     under that name, save "name" stores the value under that name.
//   * cli.cpp needs CLI11 (absent).  pxref_run() is the parse + stdlib import
//     + expand + run sequence of runSpec (proj/src/cli.cpp:62-99).
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "pixlog/ccl.hpp"
#include "pixlog/executor.hpp"
#include "pixlog/kernels.hpp"
#include "pixlog/parser.hpp"
#include "pixlog/png_io.hpp"
#include "pixlog/reach.hpp"
#include "pixlog/synth.hpp"
#include "pixlog/task_graph.hpp"

using namespace pixlog;

namespace {

std::mutex g_mu;
std::map<std::string, Value> g_store;
std::string g_stdlib;
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

ImageBuffer boolImage(const uint8_t* src, int w, int h) {
  ImageBuffer b(w, h, PixelKind::Bool);
  std::memcpy(b.boolData().data(), src, b.pixelCount());
  return b;
}

ImageBuffer u16Image(const uint16_t* src, int w, int h) {
  ImageBuffer b(w, h, PixelKind::U16);
  std::memcpy(b.u16Data().data(), src, b.pixelCount() * 2);
  return b;
}

class MemResolver : public ImportResolver {
 public:
  std::string canonicalKey(const std::string& path) override { return path; }
  Program load(const std::string& path) override {
    if (path == "stdlib" || path == "<builtin-stdlib>") return parseText(g_stdlib);
    throw SpecError(SpecError::Stage::Expand, "cannot open import file: " + path);
  }
};

}  // namespace

namespace pixlog {

Value loadPng(const std::filesystem::path& path) {
  std::lock_guard lock(g_mu);
  auto it = g_store.find(path.filename().string());
  if (it == g_store.end()) throw RunError("cannot open file for reading: " + path.string());
  return it->second;
}

void savePng(const std::filesystem::path& path, const Value& v) {
  if (!v.isImage()) throw RunError("cannot save a number as an image (use print)");
  std::lock_guard lock(g_mu);
  g_store[path.filename().string()] = v;
}

void labelColor(uint32_t packed, uint8_t rgb[3]) {
  rgb[0] = uint8_t(packed * 97u);
  rgb[1] = uint8_t(packed * 57u);
  rgb[2] = uint8_t(packed * 23u);
}

}  // namespace pixlog

extern "C" {

const char* pxref_last_error() { return g_err.c_str(); }

int pxref_threshold(int op, const uint16_t* src, int w, int h, double n, uint8_t* dst,
                    int workers) {
  try {
    WorkerPool pool(workers);
    ImageBuffer out = kernels::threshold(kernels::CmpOp(op), u16Image(src, w, h), n, pool);
    std::memcpy(dst, out.boolData().data(), out.pixelCount());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// op: 0 not, 1 and, 2 or, 3 dilate
int pxref_bool_op(int op, const uint8_t* a, const uint8_t* b, int w, int h, uint8_t* dst,
                  int workers) {
  try {
    WorkerPool pool(workers);
    ImageBuffer ia = boolImage(a, w, h);
    ImageBuffer out(1, 1, PixelKind::Bool);
    switch (op) {
      case 0: out = kernels::logicalNot(ia, pool); break;
      case 1: out = kernels::logicalAnd(ia, boolImage(b, w, h), pool); break;
      case 2: out = kernels::logicalOr(ia, boolImage(b, w, h), pool); break;
      case 3: out = kernels::dilate(ia, pool); break;
      default: throw RunError("bad op");
    }
    std::memcpy(dst, out.boolData().data(), out.pixelCount());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_count_true(const uint8_t* a, int w, int h, int64_t* out, int workers) {
  try {
    WorkerPool pool(workers);
    *out = kernels::countTrue(boolImage(a, w, h), pool);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_ccl_label(const uint8_t* a, int w, int h, uint32_t* dst, int workers,
                    int reconnect_interval, int* main_iterations) {
  try {
    WorkerPool pool(workers);
    ccl::CclConfig cfg;
    if (reconnect_interval > 0) cfg.reconnectInterval = reconnect_interval;
    ccl::CclStats stats;
    ImageBuffer out = ccl::label(boolImage(a, w, h), cfg, pool, &stats);
    std::memcpy(dst, out.labelData().data(), out.pixelCount() * 4);
    if (main_iterations) *main_iterations = stats.mainIterations;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_flood_fill_label(const uint8_t* a, int w, int h, uint32_t* dst) {
  try {
    ImageBuffer out = ccl::floodFillLabel(boolImage(a, w, h));
    std::memcpy(dst, out.labelData().data(), out.pixelCount() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_reach(const uint8_t* t, const uint8_t* u, int w, int h, uint8_t* dst, int workers) {
  try {
    WorkerPool pool(workers);
    ImageBuffer out = reach(boolImage(t, w, h), boolImage(u, w, h), pool);
    std::memcpy(dst, out.boolData().data(), out.pixelCount());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_blob_noise(int w, int h, uint64_t seed, uint16_t* dst) {
  try {
    ImageBuffer img = synth::generate(synth::ImageKind::BlobNoise, w, h, seed);
    std::memcpy(dst, img.u16Data().data(), img.pixelCount() * 2);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_concave_corner(int w, int h, uint16_t* dst) {
  try {
    ImageBuffer img = synth::generate(synth::ImageKind::ConcaveCorner, w, h, 0);
    std::memcpy(dst, img.u16Data().data(), img.pixelCount() * 2);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// --- whole-formula runs through the reference executor --------------------

void pxref_set_stdlib(const char* text) {
  std::lock_guard lock(g_mu);
  g_stdlib = text;
}

void pxref_clear() {
  std::lock_guard lock(g_mu);
  g_store.clear();
}

int pxref_put_u16(const char* name, const uint16_t* src, int w, int h) {
  try {
    Value v = Value::image(u16Image(src, w, h));
    std::lock_guard lock(g_mu);
    g_store[name] = v;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int pxref_put_bool(const char* name, const uint8_t* src, int w, int h) {
  try {
    Value v = Value::image(boolImage(src, w, h));
    std::lock_guard lock(g_mu);
    g_store[name] = v;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// kind: 0 bool, 1 u16, 2 label.  With dst == nullptr only the shape is returned.
int pxref_get(const char* name, int* kind, int* w, int* h, void* dst) {
  std::lock_guard lock(g_mu);
  auto it = g_store.find(name);
  if (it == g_store.end()) {
    g_err = std::string("no stored image ") + name;
    return -1;
  }
  const ImageBuffer& img = it->second.img();
  *kind = int(img.kind());
  *w = img.width();
  *h = img.height();
  if (dst) {
    switch (img.kind()) {
      case PixelKind::Bool: std::memcpy(dst, img.boolData().data(), img.pixelCount()); break;
      case PixelKind::U16: std::memcpy(dst, img.u16Data().data(), img.pixelCount() * 2); break;
      case PixelKind::LabelPair:
        std::memcpy(dst, img.labelData().data(), img.pixelCount() * 4);
        break;
    }
  }
  return 0;
}

// Runs a spec through parse + expand + executor::run (proj/src/cli.cpp:62-99).
// computation_ms receives RunReport::computationMs; prints (newline separated
// "label=value" lines) are copied to prints_buf.
int pxref_run(const char* spec, int workers, double* computation_ms, int* tasks,
              char* prints_buf, int prints_cap) {
  try {
    MemResolver resolver;
    Program prog = parseText(std::string("import \"stdlib\"\n") + spec);
    TaskGraph graph = expand(prog, &resolver);
    RunOptions options;
    options.workers = workers;
    options.log = [](const std::string&) {};
    RunReport rep = run(graph, options);
    if (computation_ms) *computation_ms = rep.computationMs;
    if (tasks) *tasks = int(rep.taskCount);
    if (prints_buf && prints_cap > 0) {
      std::string all;
      for (auto& l : rep.printLines) all += l + "\n";
      std::strncpy(prints_buf, all.c_str(), size_t(prints_cap - 1));
      prints_buf[prints_cap - 1] = 0;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's DAG dump (TaskGraph::dump, task_graph.cpp:72-95) for a
// spec, used to pin the host-side ImgQL front end.
int pxref_dump(const char* spec, char* buf, int cap) {
  try {
    MemResolver resolver;
    TaskGraph graph = expand(parseText(std::string("import \"stdlib\"\n") + spec), &resolver);
    std::string d = graph.dump();
    std::strncpy(buf, d.c_str(), size_t(cap - 1));
    buf[cap - 1] = 0;
    return int(d.size());
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
