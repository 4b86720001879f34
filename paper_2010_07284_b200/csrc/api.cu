// api.cu -- the C ABI (include/slcs.h): contexts, refcounted device images,
// primitive entry points with the reference's argument checks and error
// texts, and host-in/host-out wrappers with the kernels::/ccl::/reach
// signatures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>

#include "slcs_internal.h"

#include <memory>

namespace slcs {
int launch_pack_u16_mask(const uint16_t* dense, uint32_t* bits, const Geo& g, cudaStream_t st);
}

using namespace slcs;

namespace {

thread_local std::string g_err;

// Every entry point runs under guard: exceptions become status codes plus the
// thread-local message, and a launch error left by the call (CUDA error state
// is per host thread) fails the call instead of returning SLCS_OK with an
// unwritten output.
template <class F>
int guard(F&& f) {
  try {
    f();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      g_err = std::string("CUDA error: ") + cudaGetErrorString(e);
      return e == cudaErrorMemoryAllocation ? SLCS_ERR_OOM : SLCS_ERR_CUDA;
    }
    return SLCS_OK;
  } catch (const Error& e) {
    g_err = e.what();
    cudaGetLastError();  // reported: do not blame the next call
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SLCS_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SLCS_ERR_RUN;
  }
}

// ---- per-thread pinned staging ------------------------------------------------
// Host<->device copies go through pinned per-thread buffers, so the context
// lock covers only ENQUEUEING: the host memcpy into staging happens before the
// lock is taken and the wait for a result after it is released.  Concurrent
// callers (the reference evaluates independent nodes on WorkerPool threads,
// executor.cpp:220,259) therefore never block each other on a stream
// synchronisation.  Slots: 0/1 inputs, 2/3 outputs.  A slot is reused only
// after the copy that last used it has completed (its event).  Buffers larger
// than kStageMax fall back to pageable copies under the lock.
constexpr size_t kStageMax = size_t(256) << 20;
struct StageSlot {
  void* p = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  int ev_dev = -1;
  bool pending = false;
};
struct ThreadStage {
  StageSlot s[4];
  ~ThreadStage() {
    for (auto& x : s) {
      if (x.p) cudaFreeHost(x.p);
      if (x.ev) cudaEventDestroy(x.ev);
    }
  }
};
thread_local ThreadStage t_stage;

void stage_wait(int i) {
  StageSlot& x = t_stage.s[i];
  if (x.pending) {
    x.pending = false;
    cuda_check(cudaEventSynchronize(x.ev), "staging wait");
  }
}
// the slot, grown to n bytes, once its previous copy is done (nullptr: too big)
void* stage_slot(int i, size_t n) {
  if (n > kStageMax) return nullptr;
  StageSlot& x = t_stage.s[i];
  stage_wait(i);
  if (x.cap < n) {
    if (x.p) cudaFreeHost(x.p);
    x.p = nullptr;
    x.cap = 0;
    cuda_check(cudaMallocHost(&x.p, n), "cudaMallocHost");
    x.cap = n;
  }
  return x.p;
}
// the slot stays busy until the work enqueued so far on `st` has completed
void stage_fence(int i, int dev, cudaStream_t st) {
  StageSlot& x = t_stage.s[i];
  if (x.ev && x.ev_dev != dev) {
    cudaEventDestroy(x.ev);
    x.ev = nullptr;
  }
  if (!x.ev) {
    cuda_check(cudaEventCreateWithFlags(&x.ev, cudaEventDisableTiming), "event");
    x.ev_dev = dev;
  }
  cuda_check(cudaEventRecord(x.ev, st), "event");
  x.pending = true;
}
// Page-locked host memory (cudaHostAlloc / cudaHostRegister, e.g. a torch
// pin_memory() tensor) is a DMA source/target already: copies go straight to and
// from it at full link speed instead of through a staging memcpy.  Pageable
// memory (the reference's std::vector-backed ImageBuffer) keeps the staging path.
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // an unregistered pointer is not an error here
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// host source -> pinned staging copy (or the source itself when it is pinned
// already or too big to stage)
const void* stage_in(int i, const void* src, size_t n) {
  if (host_pinned(src)) return src;
  void* p = stage_slot(i, n);
  if (!p) return src;
  std::memcpy(p, src, n);
  return p;
}

// a device->host copy enqueued under the lock, completed after it
struct HostOut {
  int slot = -1;
  bool staged = false;  // bytes land in the slot's pinned buffer (else in place)
  void* dst = nullptr;
  size_t n = 0;
  // enqueue the D2H of `bytes` at dev_src for host memory `host` on st
  void enqueue(int i, void* host, const void* dev_src, size_t bytes, int dev, cudaStream_t st,
               const char* what) {
    stage_wait(i);
    slot = i;
    dst = host;
    n = bytes;
    void* p = host_pinned(host) ? nullptr : stage_slot(i, bytes);
    staged = p != nullptr;
    cuda_check(cudaMemcpyAsync(staged ? p : host, dev_src, bytes, cudaMemcpyDeviceToHost, st),
               what);
    stage_fence(i, dev, st);
  }
  // wait (no lock held) and deliver
  void finish() {
    if (slot < 0) return;
    stage_wait(slot);
    if (staged) std::memcpy(dst, t_stage.s[slot].p, n);
    slot = -1;
  }
};

const char* kind_name(int k) {
  switch (k) {
    case SLCS_BOOL: return "bool";
    case SLCS_U16: return "u16";
    case SLCS_LABEL: return "label";
  }
  return "?";
}

size_t unit_bytes(int kind) { return kind == SLCS_U16 ? 2 : 4; }
// bytes of a host image in the reference layout (Bool 1 B/px)
size_t host_bytes(int kind, int w, int h, int batch) {
  const size_t px = size_t(w) * size_t(h) * size_t(batch);
  return px * (kind == SLCS_BOOL ? 1 : (kind == SLCS_U16 ? 2 : 4));
}

Geo geo_for(int kind, int w, int h, int batch) {
  switch (kind) {
    case SLCS_BOOL: return bool_geo(w, h, batch);
    case SLCS_U16: return u16_geo(w, h, batch);
    case SLCS_LABEL: return label_geo(w, h, batch);
  }
  fail(SLCS_ERR_ARG, "unknown pixel kind");
}

void check_dims(int w, int h, int batch) {
  if (w < 1 || h < 1)
    fail(SLCS_ERR_SHAPE, "image dimensions must be at least 1x1, got " + std::to_string(w) +
                             "x" + std::to_string(h));
  if (batch < 1) fail(SLCS_ERR_SHAPE, "batch must be at least 1");
  if (batch > 65535) fail(SLCS_ERR_SHAPE, "batch must be at most 65535 slices");
}

struct DeviceGuard {
  explicit DeviceGuard(int dev) { cuda_check(cudaSetDevice(dev), "cudaSetDevice"); }
};

}  // namespace

void slcs::set_last_error(const std::string& msg) { g_err = msg; }

bool slcs::pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SLCS_NO_PDL");
    return !(e && e[0] && e[0] != '0');
  }();
  return on;
}

bool slcs::fault_launch() {
  static const long long at = [] {
    const char* e = std::getenv("SLCS_FAULT_LAUNCH");
    return e ? std::atoll(e) : 0ll;
  }();
  if (at <= 0) return false;
  static std::atomic<long long> n{0};
  return ++n == at;
}

void* slcs_ctx::alloc(size_t bytes) {
  void* p = nullptr;
  cuda_check(cudaMallocAsync(&p, bytes ? bytes : 16, stream), "cudaMallocAsync");
  return p;
}

void slcs_ctx::release(void* p) {
  if (p) cudaFreeAsync(p, stream);
}

namespace slcs {

slcs_image* new_image(slcs_ctx* ctx, int kind, int w, int h, int batch) {
  check_dims(w, h, batch);
  auto* img = new slcs_image;
  img->ctx = ctx;
  img->kind = kind;
  img->geo = geo_for(kind, w, h, batch);
  img->bytes = img->geo.slice * size_t(batch) * unit_bytes(kind);
  try {
    img->data = ctx->alloc(img->bytes);
  } catch (...) {
    delete img;
    throw;
  }
  return img;
}

void drop_image(slcs_image* img) {
  if (img && img->refs.fetch_sub(1) == 1) {
    DeviceGuard dg(img->ctx->device);
    img->ctx->release(img->data);
    delete img;
  }
}

// RAII holder for intermediate images
struct Ref {
  slcs_image* p = nullptr;
  Ref() = default;
  explicit Ref(slcs_image* q) : p(q) {}
  Ref(const Ref&) = delete;
  ~Ref() { drop_image(p); }
  slcs_image* release() {
    slcs_image* q = p;
    p = nullptr;
    return q;
  }
};

const uint32_t* words(const slcs_image* img) { return static_cast<const uint32_t*>(img->data); }
uint32_t* words(slcs_image* img) { return static_cast<uint32_t*>(img->data); }

void need_ctx(slcs_ctx* ctx) {
  if (!ctx) fail(SLCS_ERR_ARG, "null context");
}
void need_img(const slcs_image* img) {
  if (!img) fail(SLCS_ERR_ARG, "null image");
}

// boolArg (executor.cpp:43-50): Bool passes through, U16 coerces by p > 0,
// anything else is a type error.  Returns a NEW reference.
slcs_image* bool_arg(slcs_ctx* ctx, const slcs_image* v, const char* op) {
  need_img(v);
  if (v->kind == SLCS_BOOL) {
    const_cast<slcs_image*>(v)->refs.fetch_add(1);
    return const_cast<slcs_image*>(v);
  }
  if (v->kind == SLCS_U16) {
    Ref out(new_image(ctx, SLCS_BOOL, v->geo.w, v->geo.h, v->geo.batch));
    ctx->launches += launch_threshold(static_cast<const uint16_t*>(v->data), words(out.p),
                                      v->geo, out.p->geo, 1, 65535, ctx->stream);
    return out.release();
  }
  fail(SLCS_ERR_KIND, std::string("'") + op + "' expects a boolean image, got " +
                          kind_name(v->kind));
}

void same_shape(const slcs_image* a, const slcs_image* b, const char* op) {
  if (a->geo.w != b->geo.w || a->geo.h != b->geo.h || a->geo.batch != b->geo.batch)
    fail(SLCS_ERR_SHAPE, std::string(op) + ": dimension mismatch (" + std::to_string(a->geo.w) +
                             "x" + std::to_string(a->geo.h) + " vs " + std::to_string(b->geo.w) +
                             "x" + std::to_string(b->geo.h) + ")");
}

// threshold interval of SURVEY.md Appendix A #5 (host side)
void threshold_interval(int op, double n, int& lo, int& hi) {
  lo = 1;
  hi = 0;
  if (std::isnan(n)) return;
  double l = 0.0, u = 65535.0;
  switch (op) {
    case SLCS_GT: l = std::floor(n) + 1.0; break;
    case SLCS_GE: l = std::ceil(n); break;
    case SLCS_LT: u = std::ceil(n) - 1.0; break;
    case SLCS_LE: u = std::floor(n); break;
    case SLCS_EQ:
      if (std::floor(n) != n) return;
      l = u = n;
      break;
    default: fail(SLCS_ERR_ARG, "unknown comparison operator");
  }
  if (l < 0.0) l = 0.0;
  if (u > 65535.0) u = 65535.0;
  if (l > u) return;
  lo = int(l);
  hi = int(u);
}

const char* cmp_symbol(int op) {
  switch (op) {
    case SLCS_GT: return ">.";
    case SLCS_GE: return ">=.";
    case SLCS_LT: return "<.";
    case SLCS_LE: return "<=.";
    case SLCS_EQ: return "=.";
  }
  return "?";
}

slcs_image* op_threshold(slcs_ctx* ctx, int op, const slcs_image* img, double n) {
  need_img(img);
  if (op < 0 || op > 4) fail(SLCS_ERR_ARG, "unknown comparison operator");
  if (img->kind != SLCS_U16)
    fail(SLCS_ERR_KIND, std::string(cmp_symbol(op)) + " expects a numeric image, got " +
                            kind_name(img->kind));
  int lo, hi;
  threshold_interval(op, n, lo, hi);
  Ref out(new_image(ctx, SLCS_BOOL, img->geo.w, img->geo.h, img->geo.batch));
  ctx->launches += launch_threshold(static_cast<const uint16_t*>(img->data), words(out.p),
                                    img->geo, out.p->geo, lo, hi, ctx->stream);
  return out.release();
}

slcs_image* op_not(slcs_ctx* ctx, const slcs_image* a0) {
  Ref a(bool_arg(ctx, a0, "!"));
  Ref out(new_image(ctx, SLCS_BOOL, a.p->geo.w, a.p->geo.h, a.p->geo.batch));
  ctx->launches += launch_not(words(a.p), words(out.p), a.p->geo, ctx->stream);
  return out.release();
}

slcs_image* op_binary(slcs_ctx* ctx, const slcs_image* a0, const slcs_image* b0, bool is_and) {
  const char* name = is_and ? "&" : "|";
  Ref a(bool_arg(ctx, a0, name));
  Ref b(bool_arg(ctx, b0, name));
  same_shape(a.p, b.p, name);
  Ref out(new_image(ctx, SLCS_BOOL, a.p->geo.w, a.p->geo.h, a.p->geo.batch));
  if (is_and)
    ctx->launches += launch_and(words(a.p), words(b.p), words(out.p), a.p->geo, ctx->stream);
  else
    ctx->launches += launch_or(words(a.p), words(b.p), words(out.p), a.p->geo, ctx->stream);
  return out.release();
}

slcs_image* op_near(slcs_ctx* ctx, const slcs_image* a0, int k, bool erode) {
  if (k < 1) fail(SLCS_ERR_ARG, "near/interior: k must be >= 1");
  Ref a(bool_arg(ctx, a0, erode ? "interior" : "near"));
  const Geo& g = a.p->geo;
  Ref cur;
  const slcs_image* src = a.p;
  while (k > 0) {
    int step = k > 8 ? 8 : k;
    Ref out(new_image(ctx, SLCS_BOOL, g.w, g.h, g.batch));
    ctx->launches += launch_near(words(src), words(out.p), g, step, erode, ctx->stream);
    k -= step;
    drop_image(cur.p);
    cur.p = out.release();
    src = cur.p;
  }
  return cur.release();
}

void ensure_counts(slcs_ctx* ctx, int b) {
  if (ctx->counts_cap >= b) return;
  if (ctx->d_counts) cudaFree(ctx->d_counts);
  if (ctx->d_vscratch) cudaFree(ctx->d_vscratch);
  ctx->d_counts = nullptr;
  ctx->d_vscratch = nullptr;
  ctx->counts_cap = 0;
  cuda_check(cudaMalloc(&ctx->d_counts, sizeof(unsigned long long) * b), "cudaMalloc");
  cuda_check(cudaMalloc(&ctx->d_vscratch, sizeof(unsigned long long) * 2 * b), "cudaMalloc");
  cuda_check(cudaMemsetAsync(ctx->d_vscratch, 0, sizeof(unsigned long long) * 2 * b, ctx->stream),
             "cudaMemsetAsync");
  ctx->counts_cap = b;
}

// counts (u64, identical bits to int64 below 2^63) land in `out` at ho->finish()
void op_volume(slcs_ctx* ctx, const slcs_image* a0, int64_t* out, HostOut* ho) {
  Ref a(bool_arg(ctx, a0, "volume"));
  int b = a.p->geo.batch;
  ensure_counts(ctx, b);
  ctx->launches += launch_volume(words(a.p), ctx->d_counts, nullptr, ctx->d_vscratch, a.p->geo,
                                 ctx->stream);
  ho->enqueue(3, out, ctx->d_counts, sizeof(unsigned long long) * b, ctx->device, ctx->stream,
              "volume readback");
}

// device-side volume: counts land in device memory, no synchronisation
void op_volume_async(slcs_ctx* ctx, const slcs_image* a0, int64_t* dev_counts) {
  Ref a(bool_arg(ctx, a0, "volume"));
  ensure_counts(ctx, a.p->geo.batch);
  ctx->launches += launch_volume(words(a.p), reinterpret_cast<unsigned long long*>(dev_counts),
                                 nullptr, ctx->d_vscratch, a.p->geo, ctx->stream);
}

struct Scratch {
  slcs_ctx* ctx;
  void* p = nullptr;
  Scratch(slcs_ctx* c, size_t bytes) : ctx(c) {
    if (bytes) p = ctx->alloc(bytes);
  }
  ~Scratch() { ctx->release(p); }
};

slcs_image* op_ccl(slcs_ctx* ctx, const slcs_image* a0) {
  need_img(a0);
  if (a0->kind == SLCS_LABEL)
    fail(SLCS_ERR_KIND, "component labelling expects a boolean image, got label");
  Ref a(bool_arg(ctx, a0, "ccl"));
  const Geo& g = a.p->geo;
  if ((unsigned long long)g.w * (unsigned long long)g.h >= 0xfffffffeull)
    fail(SLCS_ERR_TOO_LARGE, "image too large for packed coordinate labels");
  Ref out(new_image(ctx, SLCS_LABEL, g.w, g.h, g.batch));
  Scratch s(ctx, ccl_scratch_bytes(g.w, g.h, g.batch, false, true));  // sizes hold max keys
  CclScratch cs;
  ccl_scratch_carve(s.p, g.w, g.h, g.batch, false, true, &cs);
  ctx->launches += launch_ccl(words(a.p), words(out.p), g, cs, ctx->stream);
  return out.release();
}

slcs_image* op_reach(slcs_ctx* ctx, const slcs_image* t0, const slcs_image* u0) {
  need_img(t0);
  need_img(u0);
  if (t0->kind == SLCS_LABEL || u0->kind == SLCS_LABEL)
    fail(SLCS_ERR_KIND, "reach expects boolean images");
  Ref t(bool_arg(ctx, t0, "reach"));
  Ref u(bool_arg(ctx, u0, "reach"));
  if (t.p->geo.w != u.p->geo.w || t.p->geo.h != u.p->geo.h || t.p->geo.batch != u.p->geo.batch)
    fail(SLCS_ERR_SHAPE, "reach: dimension mismatch (" + std::to_string(t.p->geo.w) + "x" +
                             std::to_string(t.p->geo.h) + " vs " + std::to_string(u.p->geo.w) +
                             "x" + std::to_string(u.p->geo.h) + ")");
  const Geo& g = t.p->geo;
  Ref out(new_image(ctx, SLCS_BOOL, g.w, g.h, g.batch));
  bool small = ccl_small_path(g.w, g.h);
  size_t sb = ccl_scratch_bytes(g.w, g.h, g.batch, true, false);
  size_t tb = small ? 0 : g.slice * size_t(g.batch) * 4;
  Scratch s(ctx, sb + tb);
  CclScratch cs;
  ccl_scratch_carve(s.p, g.w, g.h, g.batch, true, false, &cs);
  uint32_t* tmp = small ? nullptr : reinterpret_cast<uint32_t*>(static_cast<char*>(s.p) + sb);
  ctx->launches +=
      launch_reach(words(t.p), words(u.p), words(out.p), tmp, g, cs, ctx->stream);
  return out.release();
}

slcs_image* op_maxvol(slcs_ctx* ctx, const slcs_image* a0) {
  Ref a(bool_arg(ctx, a0, "maxvol"));
  const Geo& g = a.p->geo;
  Ref out(new_image(ctx, SLCS_BOOL, g.w, g.h, g.batch));
  Scratch s(ctx, ccl_scratch_bytes(g.w, g.h, g.batch, false, true));
  CclScratch cs;
  ccl_scratch_carve(s.p, g.w, g.h, g.batch, false, true, &cs);
  ctx->launches += launch_maxvol(words(a.p), words(out.p), g, cs, ctx->stream);
  return out.release();
}

slcs_image* upload(slcs_ctx* ctx, int kind, int w, int h, int batch, const void* src,
                   bool from_device) {
  need_ctx(ctx);
  check_dims(w, h, batch);
  if (!src) fail(SLCS_ERR_ARG, "null source buffer");
  Ref img(new_image(ctx, kind, w, h, batch));
  size_t npx = size_t(w) * size_t(h) * size_t(batch);
  cudaMemcpyKind dir = from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (kind == SLCS_LABEL) {
    cuda_check(cudaMemcpyAsync(img.p->data, src, npx * 4, dir, ctx->stream), "upload labels");
  } else if (kind == SLCS_U16) {
    if (!from_device && img.p->geo.pitch != size_t(w)) {
      // dense H2D, then a device-side repitch (short pitched host rows are slow)
      void* staging = ctx->alloc(npx * 2);
      cuda_check(cudaMemcpyAsync(staging, src, npx * 2, cudaMemcpyHostToDevice, ctx->stream),
                 "upload u16");
      ctx->launches += launch_repitch_u16(static_cast<const uint16_t*>(staging), size_t(w),
                                          static_cast<uint16_t*>(img.p->data), img.p->geo.pitch,
                                          w, size_t(h) * size_t(batch), ctx->stream);
      ctx->release(staging);
    } else if (img.p->geo.pitch != size_t(w)) {  // device source: repitch in place
      ctx->launches += launch_repitch_u16(static_cast<const uint16_t*>(src), size_t(w),
                                          static_cast<uint16_t*>(img.p->data), img.p->geo.pitch,
                                          w, size_t(h) * size_t(batch), ctx->stream);
    } else {
      cuda_check(cudaMemcpyAsync(img.p->data, src, npx * 2, dir, ctx->stream), "upload u16");
    }
  } else {
    const void* dev = src;
    void* staging = nullptr;
    if (!from_device) {
      staging = ctx->alloc(npx);
      cuda_check(cudaMemcpyAsync(staging, src, npx, cudaMemcpyHostToDevice, ctx->stream),
                 "upload bool");
      dev = staging;
    }
    ctx->launches += launch_pack_u8(static_cast<const uint8_t*>(dev), words(img.p), img.p->geo,
                                    true, ctx->stream);
    ctx->release(staging);
  }
  return img.release();
}

// to_device: dense copy into device memory `dst`.  Otherwise the D2H copy into
// host memory `dst` is enqueued on `ho` and completes in ho->finish() (call it
// after releasing the context lock).
void download(slcs_ctx* ctx, const slcs_image* img, void* dst, size_t bytes, bool to_device,
              HostOut* ho = nullptr) {
  need_ctx(ctx);
  need_img(img);
  if (!dst) fail(SLCS_ERR_ARG, "null destination buffer");
  if (!to_device && !ho) fail(SLCS_ERR_ARG, "host download without a completion");
  const Geo& g = img->geo;
  size_t npx = size_t(g.w) * size_t(g.h) * size_t(g.batch);
  size_t need = npx * (img->kind == SLCS_BOOL ? 1 : unit_bytes(img->kind));
  if (bytes < need) fail(SLCS_ERR_ARG, "destination buffer too small");
  // the dense reference layout on the device: in place, or a staging buffer
  const void* dense = img->data;
  void* staging = nullptr;
  void* target = to_device ? dst : nullptr;
  const bool dense_already =
      img->kind == SLCS_LABEL || (img->kind == SLCS_U16 && g.pitch == size_t(g.w));
  if (dense_already) {
    if (to_device)
      cuda_check(cudaMemcpyAsync(dst, img->data, need, cudaMemcpyDeviceToDevice, ctx->stream),
                 "download");
  } else {
    if (!to_device) target = staging = ctx->alloc(need);
    if (img->kind == SLCS_U16)
      ctx->launches += launch_repitch_u16(static_cast<const uint16_t*>(img->data), g.pitch,
                                          static_cast<uint16_t*>(target), size_t(g.w), g.w,
                                          size_t(g.h) * size_t(g.batch), ctx->stream);
    else
      ctx->launches += launch_unpack(words(img), static_cast<uint8_t*>(target), g, ctx->stream);
    dense = target;
  }
  if (!to_device) ho->enqueue(2, dst, dense, need, ctx->device, ctx->stream, "download");
  ctx->release(staging);  // stream-ordered: after the copy
}

}  // namespace slcs

// ============================================================================
extern "C" {

int slcs_abi_version(void) { return SLCS_ABI_VERSION; }
const char* slcs_last_error(void) { return g_err.c_str(); }

int slcs_ctx_create(int device, void* cuda_stream, slcs_ctx** out) {
  return guard([&] {
    if (!out) fail(SLCS_ERR_ARG, "null output pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      fail(SLCS_ERR_NOGPU, "no CUDA device available (the SLCS library has no CPU fallback)");
    if (device < 0 || device >= n) fail(SLCS_ERR_ARG, "device index out of range");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new slcs_ctx;
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cuda_stream) {
      c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
      cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
      c->own_stream = true;
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
  });
}

int slcs_ctx_destroy(slcs_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->d_counts) cudaFree(ctx->d_counts);
      if (ctx->d_vscratch) cudaFree(ctx->d_vscratch);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int slcs_ctx_synchronize(slcs_ctx* ctx) {
  return guard([&] {
    need_ctx(ctx);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    cuda_check(cudaGetLastError(), "kernel launch");
  });
}

void* slcs_ctx_stream(slcs_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int64_t slcs_ctx_launch_count(slcs_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

#define LOCKED(ctx) \
  need_ctx(ctx);    \
  std::lock_guard<std::mutex> lock_((ctx)->mu); \
  DeviceGuard dg_((ctx)->device)

int slcs_image_upload(slcs_ctx* ctx, slcs_kind kind, int w, int h, int batch, const void* host,
                      slcs_image** out) {
  return guard([&] {
    need_ctx(ctx);
    if (!out) fail(SLCS_ERR_ARG, "null output pointer");
    if (!host) fail(SLCS_ERR_ARG, "null source buffer");
    check_dims(w, h, batch);
    const void* src = stage_in(0, host, host_bytes(kind, w, h, batch));
    cudaEvent_t done = nullptr;
    {
      LOCKED(ctx);
      *out = upload(ctx, kind, w, h, batch, src, false);
      if (src != host) {
        stage_fence(0, ctx->device, ctx->stream);
      } else if (host_pinned(host)) {
        // a pinned source is read by the DMA after this call would return: the
        // caller may reuse its buffer only once the copy is done
        cuda_check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(done, ctx->stream), "event");
      }
    }
    if (done) {
      const cudaError_t e = cudaEventSynchronize(done);
      cudaEventDestroy(done);
      cuda_check(e, "upload wait");
    }
  });
}

int slcs_image_from_device(slcs_ctx* ctx, slcs_kind kind, int w, int h, int batch,
                           const void* dev, slcs_image** out) {
  return guard([&] {
    LOCKED(ctx);
    if (!out) fail(SLCS_ERR_ARG, "null output pointer");
    *out = upload(ctx, kind, w, h, batch, dev, true);
  });
}

int slcs_image_download(slcs_ctx* ctx, const slcs_image* img, void* host, size_t bytes) {
  return guard([&] {
    HostOut ho;
    {
      LOCKED(ctx);
      download(ctx, img, host, bytes, false, &ho);
    }
    ho.finish();
  });
}

int slcs_image_to_device(slcs_ctx* ctx, const slcs_image* img, void* dev, size_t bytes) {
  return guard([&] {
    LOCKED(ctx);
    download(ctx, img, dev, bytes, true);
  });
}

int slcs_random_mask(slcs_ctx* ctx, int w, int h, long long row0, uint64_t seed, double density,
                     slcs_image** out) {
  return guard([&] {
    LOCKED(ctx);
    if (!out) fail(SLCS_ERR_ARG, "null output");
    if (row0 < 0) fail(SLCS_ERR_ARG, "row0 must be >= 0");
    Ref img(new_image(ctx, SLCS_BOOL, w, h, 1));
    ctx->launches += launch_random_mask(words(img.p), img.p->geo, row0, seed, density, ctx->stream);
    *out = img.release();
  });
}

int slcs_random_u16(slcs_ctx* ctx, int w, int h, long long row0, uint64_t seed,
                    slcs_image** out) {
  return guard([&] {
    LOCKED(ctx);
    if (!out) fail(SLCS_ERR_ARG, "null output");
    if (row0 < 0) fail(SLCS_ERR_ARG, "row0 must be >= 0");
    Ref img(new_image(ctx, SLCS_U16, w, h, 1));
    ctx->launches += launch_random_u16(static_cast<uint16_t*>(img.p->data), img.p->geo, row0, seed,
                                       ctx->stream);
    *out = img.release();
  });
}

int slcs_image_retain(slcs_image* img) {
  return guard([&] {
    need_img(img);
    img->refs.fetch_add(1);
  });
}

int slcs_image_release(slcs_image* img) {
  return guard([&] {
    if (!img) return;
    std::lock_guard<std::mutex> lock(img->ctx->mu);
    drop_image(img);
  });
}

int slcs_image_info(const slcs_image* img, int* kind, int* w, int* h, int* batch) {
  return guard([&] {
    need_img(img);
    if (kind) *kind = img->kind;
    if (w) *w = img->geo.w;
    if (h) *h = img->geo.h;
    if (batch) *batch = img->geo.batch;
  });
}

int slcs_image_storage(const slcs_image* img, void** dev, size_t* row_pitch_bytes,
                       size_t* slice_bytes) {
  return guard([&] {
    need_img(img);
    size_t u = unit_bytes(img->kind);
    if (dev) *dev = img->data;
    if (row_pitch_bytes) *row_pitch_bytes = img->geo.pitch * u;
    if (slice_bytes) *slice_bytes = img->geo.slice * u;
  });
}

#define PRIM(body)                               \
  return guard([&] {                             \
    LOCKED(ctx);                                 \
    if (!out) fail(SLCS_ERR_ARG, "null output"); \
    body;                                        \
  })

int slcs_threshold(slcs_ctx* ctx, slcs_cmp op, const slcs_image* img, double n,
                   slcs_image** out) {
  PRIM(*out = op_threshold(ctx, op, img, n));
}
int slcs_not(slcs_ctx* ctx, const slcs_image* a, slcs_image** out) { PRIM(*out = op_not(ctx, a)); }
int slcs_and(slcs_ctx* ctx, const slcs_image* a, const slcs_image* b, slcs_image** out) {
  PRIM(*out = op_binary(ctx, a, b, true));
}
int slcs_or(slcs_ctx* ctx, const slcs_image* a, const slcs_image* b, slcs_image** out) {
  PRIM(*out = op_binary(ctx, a, b, false));
}
int slcs_near(slcs_ctx* ctx, const slcs_image* a, slcs_image** out) {
  PRIM(*out = op_near(ctx, a, 1, false));
}
int slcs_near_k(slcs_ctx* ctx, const slcs_image* a, int k, slcs_image** out) {
  PRIM(*out = op_near(ctx, a, k, false));
}
int slcs_interior(slcs_ctx* ctx, const slcs_image* a, slcs_image** out) {
  PRIM(*out = op_near(ctx, a, 1, true));
}
int slcs_interior_k(slcs_ctx* ctx, const slcs_image* a, int k, slcs_image** out) {
  PRIM(*out = op_near(ctx, a, k, true));
}
int slcs_volume(slcs_ctx* ctx, const slcs_image* a, int64_t* out) {
  return guard([&] {
    HostOut ho;
    {
      LOCKED(ctx);
      if (!out) fail(SLCS_ERR_ARG, "null output");
      op_volume(ctx, a, out, &ho);
    }
    ho.finish();
  });
}
int slcs_volume_async(slcs_ctx* ctx, const slcs_image* a, int64_t* dev_counts) {
  return guard([&] {
    LOCKED(ctx);
    if (!dev_counts) fail(SLCS_ERR_ARG, "null output");
    op_volume_async(ctx, a, dev_counts);
  });
}
int slcs_ccl(slcs_ctx* ctx, const slcs_image* a, slcs_image** out) { PRIM(*out = op_ccl(ctx, a)); }
int slcs_reach(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
               slcs_image** out) {
  PRIM(*out = op_reach(ctx, target, through));
}
int slcs_maxvol(slcs_ctx* ctx, const slcs_image* a, slcs_image** out) {
  PRIM(*out = op_maxvol(ctx, a));
}

// ---- row bands ------------------------------------------------------------------
int slcs_image_rows(slcs_ctx* ctx, const slcs_image* img, int row0, int nrows, slcs_image** out) {
  return guard([&] {
    LOCKED(ctx);
    need_img(img);
    if (!out) fail(SLCS_ERR_ARG, "null output");
    const Geo& g = img->geo;
    if (g.batch != 1) fail(SLCS_ERR_ARG, "row crop needs a single image");
    if (row0 < 0 || nrows < 1 || row0 + nrows > g.h) fail(SLCS_ERR_SHAPE, "row range out of image");
    Ref o(new_image(ctx, img->kind, g.w, nrows, 1));
    size_t rowb = g.pitch * unit_bytes(img->kind);
    cuda_check(cudaMemcpyAsync(o.p->data, static_cast<char*>(img->data) + size_t(row0) * rowb,
                               rowb * size_t(nrows), cudaMemcpyDeviceToDevice, ctx->stream),
               "row crop");
    *out = o.release();
  });
}

int slcs_image_vstack(slcs_ctx* ctx, int n, const slcs_image* const* imgs, slcs_image** out) {
  return guard([&] {
    LOCKED(ctx);
    if (!out || n < 1 || !imgs) fail(SLCS_ERR_ARG, "bad vstack arguments");
    int h = 0;
    for (int i = 0; i < n; ++i) {
      need_img(imgs[i]);
      if (imgs[i]->kind != imgs[0]->kind || imgs[i]->geo.w != imgs[0]->geo.w ||
          imgs[i]->geo.batch != 1)
        fail(SLCS_ERR_SHAPE, "vstack: images must share kind and width");
      h += imgs[i]->geo.h;
    }
    Ref o(new_image(ctx, imgs[0]->kind, imgs[0]->geo.w, h, 1));
    size_t rowb = imgs[0]->geo.pitch * unit_bytes(imgs[0]->kind), off = 0;
    for (int i = 0; i < n; ++i) {
      size_t b = rowb * size_t(imgs[i]->geo.h);
      cuda_check(cudaMemcpyAsync(static_cast<char*>(o.p->data) + off, imgs[i]->data, b,
                                 cudaMemcpyDeviceToDevice, ctx->stream),
                 "vstack");
      off += b;
    }
    *out = o.release();
  });
}

}  // extern "C"

struct slcs_reach_state {
  slcs_ctx* ctx = nullptr;
  std::atomic<int> refs{1};  // the caller's + one per ccl job borrowing the labelling
  bool max_keys = false;  // the labelling also holds max keys (slcs_reach_prepare_labels)
  slcs_image* t = nullptr;
  slcs_image* u = nullptr;
  void* scratch = nullptr;
  CclScratch cs;
  uint32_t* tmp = nullptr;
  uint32_t* d_roots = nullptr;
  uint8_t* d_cls = nullptr;
  int d_cap = 0;
  void* merge = nullptr;  // cross-band merge scratch (bands.cu)
  size_t merge_bytes = 0;
};

extern "C" {

static int reach_prepare(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
                         slcs_reach_state** out, bool max_keys) {
  return guard([&] {
    LOCKED(ctx);
    if (!out) fail(SLCS_ERR_ARG, "null output");
    Ref t(bool_arg(ctx, target, "reach"));
    Ref u(bool_arg(ctx, through, "reach"));
    same_shape(t.p, u.p, "reach");
    if (t.p->geo.batch != 1) fail(SLCS_ERR_ARG, "banded reach takes single images");
    const Geo& g = t.p->geo;
    std::unique_ptr<slcs_reach_state> st(new slcs_reach_state);
    st->ctx = ctx;
    st->max_keys = max_keys;
    size_t sb = ccl_scratch_bytes_large(g.w, g.h, 1, true, max_keys);
    st->scratch = ctx->alloc(sb + g.slice * 4);
    ccl_scratch_carve_large(st->scratch, g.w, g.h, 1, true, max_keys, &st->cs);
    st->tmp = reinterpret_cast<uint32_t*>(static_cast<char*>(st->scratch) + sb);
    try {
      ctx->launches += launch_reach_prepare(words(t.p), words(u.p), g, st->cs, ctx->stream,
                                            max_keys);
    } catch (...) {
      ctx->release(st->scratch);
      throw;
    }
    st->t = t.release();
    st->u = u.release();
    *out = st.release();
  });
}

int slcs_reach_prepare(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
                       slcs_reach_state** out) {
  return reach_prepare(ctx, target, through, out, false);
}

int slcs_reach_prepare_labels(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
                              slcs_reach_state** out) {
  return reach_prepare(ctx, target, through, out, true);
}

int slcs_reach_row(slcs_reach_state* st, int row, uint32_t* roots, uint8_t* cls) {
  return guard([&] {
    if (!st || !roots || !cls) fail(SLCS_ERR_ARG, "null argument");
    slcs_ctx* ctx = st->ctx;
    HostOut o1, o2;
    {
    LOCKED(ctx);
    const Geo& g = st->u->geo;
    if (row < 0 || row >= g.h) fail(SLCS_ERR_SHAPE, "row out of image");
    if (st->d_cap < g.w) {
      ctx->release(st->d_roots);
      ctx->release(st->d_cls);
      st->d_roots = static_cast<uint32_t*>(ctx->alloc(size_t(g.w) * 4));
      st->d_cls = static_cast<uint8_t*>(ctx->alloc(size_t(g.w)));
      st->d_cap = g.w;
    }
    ctx->launches += launch_reach_row(words(st->u), st->cs, g, row, st->d_roots, st->d_cls,
                                      ctx->stream);
    o1.enqueue(2, roots, st->d_roots, size_t(g.w) * 4, ctx->device, ctx->stream, "row roots");
    o2.enqueue(3, cls, st->d_cls, size_t(g.w), ctx->device, ctx->stream, "row classes");
    }
    o1.finish();
    o2.finish();
  });
}

int slcs_reach_set_flags(slcs_reach_state* st, int n, const uint32_t* roots) {
  return guard([&] {
    if (!st || (n > 0 && !roots)) fail(SLCS_ERR_ARG, "null argument");
    if (n <= 0) return;
    slcs_ctx* ctx = st->ctx;
    LOCKED(ctx);
    uint32_t* d = static_cast<uint32_t*>(ctx->alloc(size_t(n) * 4));
    cuda_check(cudaMemcpyAsync(d, roots, size_t(n) * 4, cudaMemcpyHostToDevice, ctx->stream),
               "flags upload");
    ctx->launches += launch_reach_set_flags(st->cs, st->u->geo, d, n, ctx->stream);
    ctx->release(d);
  });
}

int slcs_reach_border_record(slcs_reach_state* st, void* record_dev) {
  return guard([&] {
    if (!st || !record_dev) fail(SLCS_ERR_ARG, "null argument");
    slcs_ctx* ctx = st->ctx;
    LOCKED(ctx);
    const Geo& g = st->u->geo;
    size_t roots[2], cls[2], tgt[2];
    band_reach_record_offsets(g.w, g.pitch, roots, cls, tgt);
    char* rec = static_cast<char*>(record_dev);
    const int rows[2] = {0, g.h - 1};
    for (int side = 0; side < 2; ++side) {
      ctx->launches += launch_reach_row(words(st->u), st->cs, g, rows[side],
                                        reinterpret_cast<uint32_t*>(rec + roots[side]),
                                        reinterpret_cast<uint8_t*>(rec + cls[side]), ctx->stream);
      cuda_check(cudaMemcpyAsync(rec + tgt[side], words(st->t) + size_t(rows[side]) * g.pitch,
                                 g.pitch * 4, cudaMemcpyDeviceToDevice, ctx->stream),
                 "border record");
    }
  });
}

int slcs_band_reach_merge(slcs_reach_state* st, int nb, int me, const void* records_dev) {
  return guard([&] {
    if (!st || !records_dev) fail(SLCS_ERR_ARG, "null argument");
    if (nb < 1 || me < 0 || me >= nb) fail(SLCS_ERR_ARG, "bad band index");
    slcs_ctx* ctx = st->ctx;
    LOCKED(ctx);
    const Geo& g = st->u->geo;
    const size_t need = band_merge_scratch_bytes(nb, g.w);
    if (st->merge_bytes < need) {
      ctx->release(st->merge);
      st->merge = ctx->alloc(need);
      st->merge_bytes = need;
    }
    uint32_t* roots = nullptr;
    int* count = nullptr;
    ctx->launches += launch_band_reach_merge(nb, g.w, g.pitch, me, records_dev, st->merge, &roots,
                                             &count, ctx->stream);
    ctx->launches += launch_reach_set_flags_dev(st->cs, g, roots, count, 2 * g.w, ctx->stream);
  });
}

int slcs_reach_finish(slcs_reach_state* st, int k_out, slcs_image** out) {
  return guard([&] {
    if (!st || !out) fail(SLCS_ERR_ARG, "null argument");
    if (k_out < 0 || k_out > 8) fail(SLCS_ERR_ARG, "closing radius must be in 0..8");
    slcs_ctx* ctx = st->ctx;
    LOCKED(ctx);
    const Geo& g = st->u->geo;
    Ref o(new_image(ctx, SLCS_BOOL, g.w, g.h, 1));
    ctx->launches += launch_reach_finish(words(st->t), words(st->u), st->cs, words(o.p), st->tmp,
                                         g, k_out, ctx->stream);
    *out = o.release();
  });
}

// the state is freed when its last holder lets go (the caller's destroy, or the
// last ccl job that borrows its labelling)
static void reach_state_unref(slcs_reach_state* st) {
  if (st->refs.fetch_sub(1) != 1) return;
  slcs_ctx* ctx = st->ctx;
  {
    LOCKED(ctx);
    ctx->release(st->scratch);
    ctx->release(st->d_roots);
    ctx->release(st->d_cls);
    ctx->release(st->merge);
  }
  slcs_image_release(st->t);
  slcs_image_release(st->u);
  delete st;
}

int slcs_reach_state_destroy(slcs_reach_state* st) {
  return guard([&] {
    if (!st) return;
    reach_state_unref(st);
  });
}

// ---- host-in / host-out wrappers ------------------------------------------------
}  // extern "C"

namespace {
// host-in/host-out: stage the inputs (no lock), enqueue upload + op + download
// under the lock, wait for the result after it
template <class F>
int host_unary(slcs_ctx* ctx, int kind, const void* a, int w, int h, void* out, size_t out_bytes,
               F&& op) {
  return guard([&] {
    need_ctx(ctx);
    if (!out || !a) fail(SLCS_ERR_ARG, "null argument");
    check_dims(w, h, 1);
    const void* sa = stage_in(0, a, host_bytes(kind, w, h, 1));
    HostOut ho;
    {
      LOCKED(ctx);
      Ref ia(upload(ctx, kind, w, h, 1, sa, false));
      if (sa != a) stage_fence(0, ctx->device, ctx->stream);
      Ref r(op(ia.p));
      download(ctx, r.p, out, out_bytes, false, &ho);
    }
    ho.finish();
  });
}
template <class F>
int host_binary(slcs_ctx* ctx, const void* a, const void* b, int w, int h, void* out, F&& op) {
  return guard([&] {
    need_ctx(ctx);
    if (!out || !a || !b) fail(SLCS_ERR_ARG, "null argument");
    check_dims(w, h, 1);
    const size_t n = host_bytes(SLCS_BOOL, w, h, 1);
    const void* sa = stage_in(0, a, n);
    const void* sb = stage_in(1, b, n);
    HostOut ho;
    {
      LOCKED(ctx);
      Ref ia(upload(ctx, SLCS_BOOL, w, h, 1, sa, false));
      Ref ib(upload(ctx, SLCS_BOOL, w, h, 1, sb, false));
      if (sa != a) stage_fence(0, ctx->device, ctx->stream);
      if (sb != b) stage_fence(1, ctx->device, ctx->stream);
      Ref r(op(ia.p, ib.p));
      download(ctx, r.p, out, n, false, &ho);
    }
    ho.finish();
  });
}
}  // namespace

extern "C" {

int slcs_h_threshold(slcs_ctx* ctx, slcs_cmp op, const uint16_t* img, int w, int h, double n,
                     uint8_t* out) {
  return host_unary(ctx, SLCS_U16, img, w, h, out, size_t(w) * size_t(h),
                    [&](slcs_image* a) { return op_threshold(ctx, op, a, n); });
}
int slcs_h_not(slcs_ctx* ctx, const uint8_t* a, int w, int h, uint8_t* out) {
  return host_unary(ctx, SLCS_BOOL, a, w, h, out, size_t(w) * size_t(h),
                    [&](slcs_image* x) { return op_not(ctx, x); });
}
int slcs_h_and(slcs_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, uint8_t* out) {
  return host_binary(ctx, a, b, w, h, out,
                     [&](slcs_image* x, slcs_image* y) { return op_binary(ctx, x, y, true); });
}
int slcs_h_or(slcs_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, uint8_t* out) {
  return host_binary(ctx, a, b, w, h, out,
                     [&](slcs_image* x, slcs_image* y) { return op_binary(ctx, x, y, false); });
}
int slcs_h_dilate(slcs_ctx* ctx, const uint8_t* a, int w, int h, uint8_t* out) {
  return host_unary(ctx, SLCS_BOOL, a, w, h, out, size_t(w) * size_t(h),
                    [&](slcs_image* x) { return op_near(ctx, x, 1, false); });
}
int slcs_h_count_true(slcs_ctx* ctx, const uint8_t* a, int w, int h, int64_t* out) {
  return guard([&] {
    need_ctx(ctx);
    if (!out || !a) fail(SLCS_ERR_ARG, "null argument");
    check_dims(w, h, 1);
    const void* sa = stage_in(0, a, host_bytes(SLCS_BOOL, w, h, 1));
    HostOut ho;
    {
      LOCKED(ctx);
      Ref ia(upload(ctx, SLCS_BOOL, w, h, 1, sa, false));
      if (sa != a) stage_fence(0, ctx->device, ctx->stream);
      op_volume(ctx, ia.p, out, &ho);
    }
    ho.finish();
  });
}
int slcs_h_ccl_label(slcs_ctx* ctx, const uint8_t* a, int w, int h, uint32_t* out) {
  return host_unary(ctx, SLCS_BOOL, a, w, h, out, size_t(w) * size_t(h) * 4,
                    [&](slcs_image* x) { return op_ccl(ctx, x); });
}
int slcs_h_reach(slcs_ctx* ctx, const uint8_t* target, const uint8_t* through, int w, int h,
                 uint8_t* out) {
  return host_binary(ctx, target, through, w, h, out,
                     [&](slcs_image* x, slcs_image* y) { return op_reach(ctx, x, y); });
}

}  // extern "C"

// ---- png_io (proj/src/png_io.cpp:30-144) ---------------------------------------
namespace {

// decode on the host (no lock), then upload + per-pixel conversion on the device
slcs_image* png_to_image(slcs_ctx* ctx, const uint8_t* bytes, size_t n) {
  need_ctx(ctx);
  PngInfo info;
  const std::vector<uint8_t> raw = png_decode(bytes, n, info);
  // pageable H2D copies return once the source is consumed, so `raw` may be
  // freed right after the enqueue either way
  const void* src = stage_in(0, raw.data(), raw.size());
  LOCKED(ctx);
  Ref img(new_image(ctx, SLCS_U16, info.w, info.h, 1));
  void* staging = ctx->alloc(raw.size());
  cuda_check(cudaMemcpyAsync(staging, src, raw.size(), cudaMemcpyHostToDevice, ctx->stream),
             "png upload");
  if (src != raw.data()) stage_fence(0, ctx->device, ctx->stream);
  ctx->launches += launch_png_to_u16(static_cast<const uint8_t*>(staging), info,
                                     static_cast<uint16_t*>(img.p->data), img.p->geo, ctx->stream);
  ctx->release(staging);
  return img.release();
}

}  // namespace

int slcs_png_decode(slcs_ctx* ctx, const void* bytes, size_t n, slcs_image** out) {
  return guard([&] {
    if (!out || !bytes) fail(SLCS_ERR_ARG, "null argument");
    *out = png_to_image(ctx, static_cast<const uint8_t*>(bytes), n);
  });
}

int slcs_png_load(slcs_ctx* ctx, const char* path, slcs_image** out) {
  return guard([&] {
    need_ctx(ctx);
    if (!out || !path) fail(SLCS_ERR_ARG, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(SLCS_ERR_RUN, std::string("cannot open file for reading: ") + path);
    std::vector<uint8_t> bytes;
    uint8_t buf[1 << 16];
    for (size_t k; (k = std::fread(buf, 1, sizeof buf, f)) > 0;) bytes.insert(bytes.end(), buf, buf + k);
    std::fclose(f);
    try {
      *out = png_to_image(ctx, bytes.data(), bytes.size());
    } catch (const Error& e) {
      const std::string m = e.what();
      if (m.rfind("unsupported PNG", 0) == 0) fail(e.code, m + " (" + path + ")");
      throw;
    }
  });
}

int slcs_png_save(slcs_ctx* ctx, const slcs_image* img, const char* path) {
  return guard([&] {
    need_ctx(ctx);
    need_img(img);
    if (!path) fail(SLCS_ERR_ARG, "null path");
    if (img->geo.batch != 1) fail(SLCS_ERR_SHAPE, "savePng: one image per file (batch must be 1)");
    const Geo& g = img->geo;
    const int bytes_px = img->kind == SLCS_LABEL ? 3 : 2;
    const size_t n = size_t(g.h) * (size_t(g.w) * bytes_px + 1);
    std::vector<uint8_t> host(n);
    HostOut ho;
    {
      LOCKED(ctx);
      void* rows = ctx->alloc(n);
      ctx->launches += launch_png_rows(img->data, img->kind, g, static_cast<uint8_t*>(rows),
                                       ctx->stream);
      ho.enqueue(2, host.data(), rows, n, ctx->device, ctx->stream, "png rows");
      ctx->release(rows);
    }
    ho.finish();  // filtering + zlib below run without the context lock
    const std::vector<uint8_t> file =
        png_encode(host.data(), g.w, g.h, img->kind == SLCS_LABEL ? 8 : 16,
                   img->kind == SLCS_LABEL ? 2 : 0);
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(SLCS_ERR_RUN, std::string("cannot open file for writing: ") + path);
    const size_t wrote = std::fwrite(file.data(), 1, file.size(), f);
    std::fclose(f);
    if (wrote != file.size()) fail(SLCS_ERR_RUN, std::string("short write: ") + path);
  });
}

void slcs_label_color(uint32_t packed, uint8_t rgb[3]) { png_label_color(packed, rgb); }

size_t slcs_band_record_bytes(int kind, int w) {
  if (w < 1 || (kind != 0 && kind != 1)) return 0;
  return band_record_bytes(kind, w, bool_geo(w, 1, 1).pitch);
}

int slcs_ccl_border_record(slcs_ctx* ctx, const slcs_image* labels, void* record_dev) {
  return guard([&] {
    LOCKED(ctx);
    need_img(labels);
    if (labels->kind != SLCS_LABEL) fail(SLCS_ERR_KIND, "border record expects a label image");
    if (labels->geo.batch != 1) fail(SLCS_ERR_ARG, "row bands take single images");
    if (!record_dev) fail(SLCS_ERR_ARG, "null record");
    const Geo& g = labels->geo;
    size_t off[2];
    band_label_record_offsets(g.w, off);
    const size_t rowb = size_t(g.w) * 4;
    const char* base = static_cast<const char*>(labels->data);
    char* rec = static_cast<char*>(record_dev);
    cuda_check(cudaMemcpyAsync(rec + off[0], base, rowb, cudaMemcpyDeviceToDevice, ctx->stream),
               "border record");
    cuda_check(cudaMemcpyAsync(rec + off[1], base + size_t(g.h - 1) * rowb, rowb,
                               cudaMemcpyDeviceToDevice, ctx->stream),
               "border record");
  });
}

int slcs_band_ccl_relabel(slcs_ctx* ctx, const slcs_image* labels, int nb, int me,
                          const void* records_dev, const long long* band_heights,
                          uint64_t* out_dev) {
  return guard([&] {
    LOCKED(ctx);
    need_img(labels);
    if (labels->kind != SLCS_LABEL) fail(SLCS_ERR_KIND, "band relabel expects a label image");
    if (nb < 1 || me < 0 || me >= nb || !band_heights || !out_dev || (nb > 1 && !records_dev))
      fail(SLCS_ERR_ARG, "bad band relabel arguments");
    const Geo& g = labels->geo;
    if (band_heights[me] != g.h) fail(SLCS_ERR_SHAPE, "band height does not match the labels");
    std::vector<unsigned long long> row0w(static_cast<size_t>(nb));
    unsigned long long r0 = 0;
    for (int b = 0; b < nb; ++b) {
      row0w[size_t(b)] = r0 * (unsigned long long)g.w;
      r0 += (unsigned long long)band_heights[b];
    }
    void* scratch = ctx->alloc(band_merge_scratch_bytes(nb, g.w));
    ctx->launches += launch_band_ccl_merge_relabel(
        nb, g.w, me, records_dev, row0w.data(), scratch, static_cast<const uint32_t*>(labels->data),
        size_t(g.w) * size_t(g.h), reinterpret_cast<unsigned long long*>(out_dev), ctx->stream);
    ctx->release(scratch);  // stream-ordered; row0w (pageable) was consumed by the enqueue
  });
}

// a band's CCL between its border record and its 64-bit labels: the band's
// union-find (large images), or its u32 labels (images the one-CTA path takes)
struct slcs_ccl_job {
  slcs_ctx* ctx = nullptr;
  slcs_image* band = nullptr;    // bool view of the band (retained)
  slcs_image* labels = nullptr;  // small path only: the u32 labels
  void* scratch = nullptr;       // owned (null when the labelling is a reach state's)
  slcs_reach_state* reach = nullptr;  // the reach state whose labelling this borrows (ref)
  CclScratch cs;
};

int slcs_ccl_band_begin(slcs_ctx* ctx, const slcs_image* band, void* record_dev,
                        slcs_ccl_job** out) {
  return guard([&] {
    LOCKED(ctx);
    if (!out || !record_dev) fail(SLCS_ERR_ARG, "null argument");
    need_img(band);
    if (band->kind == SLCS_LABEL)
      fail(SLCS_ERR_KIND, "component labelling expects a boolean image, got label");
    Ref b(bool_arg(ctx, band, "ccl"));
    const Geo& g = b.p->geo;
    if (g.batch != 1) fail(SLCS_ERR_ARG, "row bands take single images");
    std::unique_ptr<slcs_ccl_job> job(new slcs_ccl_job);
    job->ctx = ctx;
    size_t off[2];
    band_label_record_offsets(g.w, off);
    char* rec = static_cast<char*>(record_dev);
    if (ccl_small_path(g.w, g.h)) {
      job->labels = op_ccl(ctx, b.p);
      const size_t rowb = size_t(g.w) * 4;
      const char* lab = static_cast<const char*>(job->labels->data);
      cuda_check(cudaMemcpyAsync(rec + off[0], lab, rowb, cudaMemcpyDeviceToDevice, ctx->stream),
                 "border record");
      cuda_check(cudaMemcpyAsync(rec + off[1], lab + size_t(g.h - 1) * rowb, rowb,
                                 cudaMemcpyDeviceToDevice, ctx->stream),
                 "border record");
    } else {
      job->scratch = ctx->alloc(ccl_scratch_bytes_large(g.w, g.h, 1, false, true));
      ccl_scratch_carve_large(job->scratch, g.w, g.h, 1, false, true, &job->cs);
      ctx->launches += launch_ccl_prepare(words(b.p), g, job->cs, ctx->stream);
      ctx->launches += launch_ccl_row_labels(words(b.p), g, job->cs, 0,
                                             reinterpret_cast<uint32_t*>(rec + off[0]), ctx->stream);
      ctx->launches += launch_ccl_row_labels(words(b.p), g, job->cs, g.h - 1,
                                             reinterpret_cast<uint32_t*>(rec + off[1]), ctx->stream);
    }
    job->band = b.release();
    *out = job.release();
  });
}

int slcs_ccl_band_begin_reach(slcs_reach_state* rs, void* record_dev, slcs_ccl_job** out) {
  return guard([&] {
    if (!rs || !out || !record_dev) fail(SLCS_ERR_ARG, "null argument");
    if (!rs->max_keys)
      fail(SLCS_ERR_ARG, "the reach state carries no max keys (use slcs_reach_prepare_labels)");
    slcs_ctx* ctx = rs->ctx;
    LOCKED(ctx);
    const Geo& g = rs->u->geo;
    std::unique_ptr<slcs_ccl_job> job(new slcs_ccl_job);
    job->ctx = ctx;
    job->cs = rs->cs;  // borrowed: the job holds a reference to the reach state
    size_t off[2];
    band_label_record_offsets(g.w, off);
    char* rec = static_cast<char*>(record_dev);
    ctx->launches += launch_ccl_row_labels(words(rs->u), g, job->cs, 0,
                                           reinterpret_cast<uint32_t*>(rec + off[0]), ctx->stream);
    ctx->launches += launch_ccl_row_labels(words(rs->u), g, job->cs, g.h - 1,
                                           reinterpret_cast<uint32_t*>(rec + off[1]), ctx->stream);
    rs->u->refs.fetch_add(1);
    job->band = rs->u;
    rs->refs.fetch_add(1);
    job->reach = rs;
    *out = job.release();
  });
}

int slcs_ccl_band_finish(slcs_ccl_job* job, int nb, int me, const void* records_dev,
                         const long long* band_heights, uint64_t* out_dev) {
  return guard([&] {
    if (!job) fail(SLCS_ERR_ARG, "null job");
    slcs_ctx* ctx = job->ctx;
    LOCKED(ctx);
    if (nb < 1 || me < 0 || me >= nb || !band_heights || !out_dev || (nb > 1 && !records_dev))
      fail(SLCS_ERR_ARG, "bad band relabel arguments");
    const Geo& g = job->band->geo;
    if (band_heights[me] != g.h) fail(SLCS_ERR_SHAPE, "band height does not match the labels");
    std::vector<unsigned long long> row0w(static_cast<size_t>(nb));
    unsigned long long r0 = 0;
    for (int b = 0; b < nb; ++b) {
      row0w[size_t(b)] = r0 * (unsigned long long)g.w;
      r0 += (unsigned long long)band_heights[b];
    }
    void* scratch = ctx->alloc(band_merge_scratch_bytes(nb, g.w));
    auto* out = reinterpret_cast<unsigned long long*>(out_dev);
    if (job->labels) {
      ctx->launches += launch_band_ccl_merge_relabel(
          nb, g.w, me, records_dev, row0w.data(), scratch,
          static_cast<const uint32_t*>(job->labels->data), size_t(g.w) * size_t(g.h), out,
          ctx->stream);
    } else {
      LabelMap64 map;
      ctx->launches += launch_band_ccl_merge(nb, g.w, me, records_dev, row0w.data(), scratch,
                                             &map, ctx->stream);
      ctx->launches += launch_ccl_labels64(words(job->band), g, job->cs, map, out, ctx->stream);
    }
    ctx->release(scratch);  // stream-ordered; row0w (pageable) was consumed by the enqueue
  });
}

int slcs_ccl_job_destroy(slcs_ccl_job* job) {
  return guard([&] {
    if (!job) return;
    slcs_ctx* ctx = job->ctx;
    {
      LOCKED(ctx);
      ctx->release(job->scratch);
    }
    if (job->labels) slcs_image_release(job->labels);
    slcs_image_release(job->band);
    if (job->reach) reach_state_unref(job->reach);
    delete job;
  });
}

int slcs_near_k_halo(slcs_ctx* ctx, const slcs_image* a, int k, int erode, const void* top_dev,
                     int top_rows, const void* bot_dev, int bot_rows, slcs_image** out) {
  return guard([&] {
    LOCKED(ctx);
    if (!out) fail(SLCS_ERR_ARG, "null output");
    if (k < 1 || k > 8) fail(SLCS_ERR_ARG, "near with halo rows: k must be in 1..8");
    if (top_rows < 0 || bot_rows < 0) fail(SLCS_ERR_ARG, "negative halo row count");
    Ref x(bool_arg(ctx, a, erode ? "interior" : "near"));
    const Geo& g = x.p->geo;
    if (g.batch != 1) fail(SLCS_ERR_ARG, "halo rows need a single image");
    Ref o(new_image(ctx, SLCS_BOOL, g.w, g.h, 1));
    ctx->launches += launch_near_halo(words(x.p), words(o.p), g, k, erode != 0,
                                      static_cast<const uint32_t*>(top_dev), top_rows,
                                      static_cast<const uint32_t*>(bot_dev), bot_rows,
                                      ctx->stream);
    *out = o.release();
  });
}
