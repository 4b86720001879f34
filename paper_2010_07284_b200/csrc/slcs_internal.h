// slcs_internal.h -- shared declarations of the sm_100a primitive library.
//
// Device data layout:
//   Bool  : bit-packed, 32 px per uint32 word, bit b of word j of row r is
//           pixel (r, 32j+b) (LSB = lowest column).  Row pitch P words,
//           P = round_up(ceil(W/32), 4) so every row starts 16 B aligned and
//           uint4 accesses never straddle rows.  Padding bits (cols >= W) and
//           padding words are ZERO -- every kernel preserves this invariant.
//   U16   : row pitch round_up(W, 32) pixels, so a 32-px word maps to 64
//           aligned bytes (4 x uint4).  Padding pixels are don't-care.
//   Label : dense uint32, pitch W (the reference layout, image.hpp:20-29).
//   Batch : `batch` slices of identical shape, slice stride = P*H units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <utility>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/slcs.h"

namespace slcs {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// thread-local message returned by slcs_last_error (api.cu)
void set_last_error(const std::string& msg);

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation)
    fail(SLCS_ERR_OOM, std::string("device allocation failed in ") + what);
  fail(SLCS_ERR_CUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

inline size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }

// ---- programmatic dependent launch (sm_90+) ----------------------------------
// Every kernel starts with slcs_pdl_wait() and is launched with the
// programmatic-stream-serialization attribute.  The wait (griddepcontrol.wait)
// returns only once the predecessor grid has COMPLETED and its memory is
// visible.  Kernels do not signal launch_dependents early: an early trigger
// right after the wait measured slower on B200 (config-2 chain 25.6 -> 27.0
// ms, threshold 0.82 -> 0.68 of HBM peak).  Set SLCS_NO_PDL=1 to launch
// plainly.
__device__ __forceinline__ void slcs_pdl_wait() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  cudaGridDependencySynchronize();
#endif
}

bool pdl_enabled();
// Fault injection for tests: with SLCS_FAULT_LAUNCH=n in the
// environment, the n-th kernel launch of the process is issued with an
// impossible shared-memory request, so it fails like a real launch error.
bool fault_launch();

template <typename... KArgs, typename... Args>
inline void pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  if (fault_launch()) cfg.dynamicSmemBytes = size_t(1) << 30;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), "kernel launch");
}

// ---- per-device one-time initialisation ----------------------------------------
// Kernel attributes (the dynamic shared-memory opt-in) and occupancy are per
// device, and a process may hold contexts on several devices, so one-time
// set-up is keyed by the calling thread's current device (every entry point
// selects its context's device first).
constexpr int kMaxDevices = 64;
template <typename T>
struct PerDevice {
  std::once_flag once[kMaxDevices];
  T val[kMaxDevices] = {};
  template <typename F>
  T get(F&& init) {
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    if (d < 0 || d >= kMaxDevices) fail(SLCS_ERR_ARG, "device index out of range");
    std::call_once(once[d], [&] { val[d] = init(d); });
    return val[d];
  }
};
// opt a kernel into `bytes` of dynamic shared memory on the current device
template <typename K>
inline void smem_opt_in(PerDevice<int>& pd, K kern, size_t bytes) {
  int rc = pd.get([&](int) {
    return int(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  });
  if (rc != cudaSuccess)
    fail(SLCS_ERR_CUDA, std::string("cudaFuncSetAttribute(MaxDynamicSharedMemorySize): ") +
                            cudaGetErrorString(cudaError_t(rc)));
}
inline int device_sm_count() {
  static PerDevice<int> pd;
  return pd.get([](int d) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n > 0 ? n : 148;
  });
}

// Row geometry of one image kind.
struct Geo {
  int w = 0, h = 0, batch = 1;
  int wpr = 0;        // Bool: valid words per row = ceil(w/32)
  size_t pitch = 0;   // row pitch in storage units (words / u16 / u32)
  size_t slice = 0;   // units per slice = pitch * h
  uint32_t lastmask = 0;  // Bool: valid-bit mask of word wpr-1
};

Geo bool_geo(int w, int h, int batch);
// valid-bit mask of Bool word j of a row (padding bits/words are zero)
__device__ __forceinline__ uint32_t valid_mask(int j, int wpr, uint32_t lastmask) {
  return j < wpr - 1 ? 0xffffffffu : (j == wpr - 1 ? lastmask : 0u);
}
Geo u16_geo(int w, int h, int batch);
Geo label_geo(int w, int h, int batch);

// Packed CCL keys: a pixel (r, c) is keyed (r << s) | c with s = bits(W-1),
// which preserves the reference's row-first lexicographic order
// (image.hpp:20-29) while making key -> 2x2 block a pair of shifts.
struct KeyGeo {
  int s = 1;
  uint32_t cmask = 1;
  int bw = 0, bh = 0;      // 2x2 block grid
  size_t slice_blocks = 0;
};
KeyGeo key_geo(int w, int h);

// ---- kernel launchers (stream-ordered, no sync) ----------------------------
// All return the number of kernel launches issued.
int launch_pack_u8(const uint8_t* dense, uint32_t* bits, const Geo& g, bool nonzero_is_true,
                   cudaStream_t st);
int launch_unpack(const uint32_t* bits, uint8_t* dense, const Geo& g, cudaStream_t st);
// u16 rows from pitch spitch to pitch dpitch (pixels), columns >= w of dst zeroed
int launch_repitch_u16(const uint16_t* src, size_t spitch, uint16_t* dst, size_t dpitch, int w,
                       size_t rows, cudaStream_t st);
// interval threshold: bit = lo <= p <= hi (empty interval when lo > hi)
int launch_threshold(const uint16_t* px, uint32_t* bits, const Geo& gu, const Geo& gb, int lo,
                     int hi, cudaStream_t st);
// device-scalar threshold: comparand read from *n_dev (a double) on device
int launch_threshold_dev(const uint16_t* px, uint32_t* bits, const Geo& gu, const Geo& gb,
                         int op, const double* n_dev, cudaStream_t st);
int launch_not(const uint32_t* a, uint32_t* out, const Geo& g, cudaStream_t st);
int launch_and(const uint32_t* a, const uint32_t* b, uint32_t* out, const Geo& g,
               cudaStream_t st);
int launch_or(const uint32_t* a, const uint32_t* b, uint32_t* out, const Geo& g,
              cudaStream_t st);
// k-fold near (dilate) or interior (erode), 1 <= k <= 31 per launch
int launch_near(const uint32_t* a, uint32_t* out, const Geo& g, int k, bool erode,
                cudaStream_t st);
// the same with halo rows from neighbouring row bands: ntop packed rows (pitch of
// g) directly above row 0 at `top`, nbot rows directly below row h-1 at `bot`;
// rows beyond them are absent (0 for near, 1 for interior)
int launch_near_halo(const uint32_t* a, uint32_t* out, const Geo& g, int k, bool erode,
                     const uint32_t* top, int ntop, const uint32_t* bot, int nbot,
                     cudaStream_t st);
// counts (u64) and/or dbl (double) per slice; vscratch = batch zeroed u64
// accumulators (left zeroed by the launch)
// (accumulators + done counters), left zeroed by the kernel
int launch_volume(const uint32_t* a, unsigned long long* counts, double* dbl,
                  unsigned long long* vscratch, const Geo& g, cudaStream_t st);
// several independent volumes in one launch: image words (a multiple of 4, the
// slice), a zeroed u64 accumulator each (left zeroed), counts and/or dbl out
constexpr int kVolumeJobsMax = 8;
struct VolumeJob {
  const uint32_t* a;
  size_t words;
  unsigned long long* acc;
  unsigned long long* counts;
  double* dbl;
};
struct VolumeJobs {
  VolumeJob job[kVolumeJobsMax];
  int n;
};
int launch_volume_multi(const VolumeJobs& jobs, cudaStream_t st);
// rows [row0, row0 + g.h) of randomMask(g.w x H, density, Rng(seed)) as bits
int launch_random_mask(uint32_t* bits, const Geo& g, long long row0, unsigned long long seed,
                       double density, cudaStream_t st);

// rows [row0, row0 + g.h) of the uniform u16 fixture (pixel i = draw i % 65536)
int launch_random_u16(uint16_t* px, const Geo& g, long long row0, unsigned long long seed,
                      cudaStream_t st);

// Fused elementwise program over bit-packed words (see fused.cu).
struct FusedOp {
  uint8_t op;    // FOP_*
  uint8_t dst;   // register
  uint8_t a, b;  // registers / input index
  int32_t lo, hi;
};
enum : uint8_t {
  FOP_LOADB = 0,   // r[dst] = bool input a
  FOP_THRESH = 1,  // r[dst] = (lo <= u16 input a <= hi)
  FOP_NOT = 2,
  FOP_AND = 3,
  FOP_OR = 4,
  FOP_ANDNOT = 5,  // r[a] & ~r[b]
  FOP_STORE = 6,   // output a = r[dst]
  FOP_PRESET = 7,  // r[dst] = the host kernel's own result word (epilogues inside k_small)
};
constexpr int kFusedMaxOps = 24;
constexpr int kFusedMaxIn = 8;
constexpr int kFusedMaxOut = 4;
constexpr int kFusedRegs = 8;
struct FusedProgram {
  int n_ops = 0;
  int n_bin = 0;  // bool inputs in use (bin[0..n_bin))
  FusedOp ops[kFusedMaxOps];
  const uint32_t* bin[kFusedMaxIn];
  const uint16_t* uin[kFusedMaxIn];
  uint32_t* out[kFusedMaxOut];
};
int launch_fused(const FusedProgram& p, const Geo& gb, const Geo& gu, cudaStream_t st);

// ---- connected components (ccl.cu) -------------------------------------------
struct CclScratch {
  uint32_t* parent = nullptr;  // per 2x2 block, packed key + 1 (0 = empty)
  uint32_t* lists = nullptr;   // per tile: count + ring-touching local roots
  uint8_t* flag = nullptr;     // per block
  uint32_t* size = nullptr;    // per block (maxvol)
  unsigned int* maxv = nullptr;  // per slice (maxvol)
};
size_t ccl_scratch_bytes(int w, int h, int batch, bool flags, bool sizes);
void ccl_scratch_carve(void* base, int w, int h, int batch, bool flags, bool sizes,
                       CclScratch* s);
bool ccl_small_path(int w, int h);
// small-image maxvol with an elementwise prologue (its operand computed from a
// bool-only listing, `bits` unused) and/or epilogue (a listing over the maxvol
// result, read as FOP_PRESET); either may be null
int launch_maxvol_small_listing(const FusedProgram* pro, const FusedProgram* epi,
                                const uint32_t* bits, uint32_t* out, const Geo& gb,
                                cudaStream_t st);
// n <= 4 independent reaches of one small shape (k_out 1, tk 0) in one launch
int launch_reach_small_multi(const uint32_t* const* target, const uint32_t* const* through,
                             uint32_t* const* out, int n, const Geo& gb, cudaStream_t st);
// the tiled path's scratch regardless of size (row bands always use it)
size_t ccl_scratch_bytes_large(int w, int h, int batch, bool flags, bool sizes);
void ccl_scratch_carve_large(void* base, int w, int h, int batch, bool flags, bool sizes,
                             CclScratch* s);
int launch_ccl(const uint32_t* bits, uint32_t* labels, const Geo& gb, CclScratch& s,
               cudaStream_t st);
// k_out: radius of the closing near (1 = reach; > 1 absorbs following nears;
// 0 = emit the selection t | S, its consumer folds the closing near as its tk).
// tk: the target operand is near^tk(target) (nears folded into the reach).
int launch_reach(const uint32_t* target, const uint32_t* through, uint32_t* out,
                 uint32_t* tmp_bits, const Geo& gb, CclScratch& s, cudaStream_t st,
                 int k_out = 1, int tk = 0, bool early_through = false);
// early_through: `through` was not written by the launch just before this one
// (the fused kernel may then read it before its programmatic-launch wait)
int launch_maxvol(const uint32_t* bits, uint32_t* out, const Geo& gb, CclScratch& s,
                  cudaStream_t st);
// row bands: reach in phases (large path always); max_keys: the labelling also
// carries each component's max key (s.size), so ccl::label can reuse it
int launch_reach_prepare(const uint32_t* target, const uint32_t* through, const Geo& gb,
                         CclScratch& s, cudaStream_t st, bool max_keys = false);
int launch_reach_row(const uint32_t* through, const CclScratch& s, const Geo& gb, int row,
                     uint32_t* roots, uint8_t* cls, cudaStream_t st);
int launch_reach_set_flags(const CclScratch& s, const Geo& gb, const uint32_t* roots, int n,
                           cudaStream_t st);
int launch_reach_finish(const uint32_t* target, const uint32_t* through, const CclScratch& s,
                        uint32_t* out, uint32_t* tmp_bits, const Geo& gb, int k_out,
                        cudaStream_t st);
// label CSE: one labelling of `through` (large path only), reused by many reaches
size_t ccl_labels_bytes(int w, int h, int batch);
int launch_labels(const uint32_t* through, void* labels, const Geo& gb, cudaStream_t st);
// flags32: one uint32 per 2x2 block, zeroed by the labelling step once per run;
// reach number idx (< 4096) of that labelling stamps idx + 1
int launch_reach_labeled(const uint32_t* target, const uint32_t* through, const void* labels,
                         uint32_t* flags32, uint32_t idx, uint32_t* out,
                         uint32_t* tmp_bits, const Geo& gb, cudaStream_t st, int k_out = 1);

// a chain of `steps` reaches on one labelling (label CSE) in ONE cooperative
// launch: reach s (idx0 + s) targets near^kmid of the previous selection (the
// first targets x), the last closes with near^klast; tmp2 = two bool images
bool reach_chain_fits(const Geo& gb, int steps, int kmid, int klast);
size_t reach_chain_scratch_bytes(const Geo& gb, int steps);
int launch_reach_chain(const uint32_t* x, const uint32_t* through, const void* labels,
                       uint32_t* flags32, uint32_t idx0, int steps, int kmid, int klast,
                       uint32_t* out, uint32_t* tmp2, const Geo& gb, cudaStream_t st);
int launch_reach_set_flags_dev(const CclScratch& s, const Geo& gb, const uint32_t* roots,
                               const int* n_dev, int max_n, cudaStream_t st);

// ---- row bands: cross-band merges (bands.cu) ---------------------------------
// border record bytes: kind 0 = reach (roots/classes/target of the first and last
// row), 1 = labels (band-local labels of the first and last row)
size_t band_record_bytes(int kind, int w, size_t pitch_words);
void band_reach_record_offsets(int w, size_t pitch_words, size_t* roots, size_t* cls,
                               size_t* tgt);
void band_label_record_offsets(int w, size_t* lab);
size_t band_merge_scratch_bytes(int nb, int w);
// union-find over all bands' reach records; this band's newly seeded roots and
// their count land in scratch (*roots_out, *count_out)
int launch_band_reach_merge(int nb, int w, size_t pitch_words, int me, const void* records,
                            void* scratch, uint32_t** roots_out, int** count_out,
                            cudaStream_t st);
// union-find over all bands' label records + relabel of this band's labels to
// global 64-bit labels (row0w_host[b] = first row of band b times W)
int launch_band_ccl_merge_relabel(int nb, int w, int me, const void* records,
                                  const unsigned long long* row0w_host, void* scratch,
                                  const uint32_t* labels, size_t npx, unsigned long long* out,
                                  cudaStream_t st);
// A band's u32 label -> its global 64-bit label: offset (first row of the band
// times W) + l, or the merged value of a component that crosses a band border
// (open-addressed hash rkeys -> rvals, EMPTY = ~0; any = 0: a single band)
struct LabelMap64 {
  unsigned long long offset = 0;
  const unsigned long long* rkeys = nullptr;
  const unsigned long long* rvals = nullptr;
  uint32_t rmask = 0;
  int any = 0;
};
__device__ __forceinline__ uint32_t band_hash_slot(unsigned long long key, uint32_t mask) {
  key ^= key >> 33;
  key *= 0xff51afd7ed558ccdull;
  key ^= key >> 33;
  return uint32_t(key) & mask;
}
__device__ __forceinline__ unsigned long long map_label64(uint32_t l, const LabelMap64& m) {
  if (!l) return 0ull;
  if (m.any) {
    for (uint32_t h = band_hash_slot(l, m.rmask);; h = (h + 1) & m.rmask) {
      const unsigned long long k = __ldg(m.rkeys + h);
      if (k == l) return __ldg(m.rvals + h);
      if (k == ~0ull) break;
    }
  }
  return m.offset + l;
}
// the cross-band merge alone: fills *map (tables in scratch) for this band
int launch_band_ccl_merge(int nb, int w, int me, const void* records,
                          const unsigned long long* row0w_host, void* scratch, LabelMap64* map,
                          cudaStream_t st);
// band CCL without a u32 label image: local union-find (P / max keys in s),
// the u32 labels of rows r0 and r1 (the border record), then the global 64-bit
// labels written straight from the union-find through `map`
int launch_ccl_prepare(const uint32_t* bits, const Geo& gb, CclScratch& s, cudaStream_t st);
int launch_ccl_row_labels(const uint32_t* bits, const Geo& gb, const CclScratch& s, int row,
                          uint32_t* out, cudaStream_t st);
int launch_ccl_labels64(const uint32_t* bits, const Geo& gb, const CclScratch& s,
                        const LabelMap64& map, unsigned long long* out, cudaStream_t st);

// ---- PNG ingest/egress (png.cu) --------------------------------------------------
struct PngInfo {
  int w = 0, h = 0, depth = 8, channels = 1;
};
// container + inflate + unfilter (+ Adam7) on the host: raw samples, rows of w*channels
std::vector<uint8_t> png_decode(const uint8_t* data, size_t n, PngInfo& info);
// rows: h x (1 + w*channels*depth/8) filtered bytes; color 0 (grey) or 2 (RGB)
std::vector<uint8_t> png_encode(const uint8_t* rows, int w, int h, int depth, int color);
int launch_png_to_u16(const uint8_t* raw, const PngInfo& info, uint16_t* out, const Geo& gu,
                      cudaStream_t st);
int launch_png_rows(const void* img, int kind, const Geo& g, uint8_t* rows, cudaStream_t st);
void png_label_color(uint32_t packed, uint8_t rgb[3]);

}  // namespace slcs

// ---- opaque handle definitions -------------------------------------------------

struct slcs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 0;
  std::mutex mu;
  std::atomic<int64_t> launches{0};
  // small pinned/device scratch for reductions
  unsigned long long* d_counts = nullptr;
  unsigned long long* d_vscratch = nullptr;  // 2 * counts_cap, zeroed (launch_volume)
  int counts_cap = 0;

  void* alloc(size_t bytes);
  void release(void* p);
};

struct slcs_image {
  std::atomic<int> refs{1};
  slcs_ctx* ctx = nullptr;
  int kind = SLCS_BOOL;
  slcs::Geo geo;
  void* data = nullptr;
  size_t bytes = 0;
};
