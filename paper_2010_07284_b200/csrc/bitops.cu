// bitops.cu -- bit-packed Bool primitives for sm_100a.
//
// Every primitive here is HBM-bound integer work (no tensor cores): the
// kernels move 32 pixels per uint32 word, use 16 B vector accesses where the
// row layout allows, and keep the zero-padding invariant of slcs_internal.h.
//
//   threshold  kernels.cpp:75-97   u16 -> bits, integer interval compare
//   ! & |      kernels.cpp:36-73   word NOT/AND/OR (uint4)
//   near       kernels.cpp:99-124  funnel-shift 3x3 (k-fold: (2k+1)^2) OR
//   interior   stdlib.imgql:5      same stencil with AND, out-of-image = 1
//   volume     kernels.cpp:126-136 popcount + warp/block reduce + 1 atomic
#include <type_traits>
#include "slcs_internal.h"

namespace slcs {

Geo bool_geo(int w, int h, int batch) {
  Geo g;
  g.w = w;
  g.h = h;
  g.batch = batch;
  g.wpr = (w + 31) / 32;
  g.pitch = round_up(size_t(g.wpr), 4);
  g.slice = g.pitch * size_t(h);
  int rem = w % 32;
  g.lastmask = rem ? ((1u << rem) - 1u) : 0xffffffffu;
  return g;
}

Geo u16_geo(int w, int h, int batch) {
  Geo g;
  g.w = w;
  g.h = h;
  g.batch = batch;
  g.wpr = (w + 31) / 32;
  g.pitch = round_up(size_t(w), 32);
  g.slice = g.pitch * size_t(h);
  return g;
}

Geo label_geo(int w, int h, int batch) {
  Geo g;
  g.w = w;
  g.h = h;
  g.batch = batch;
  g.wpr = (w + 31) / 32;
  g.pitch = size_t(w);
  g.slice = g.pitch * size_t(h);
  return g;
}

namespace {

constexpr int kThreads = 256;

inline int grid_for(size_t n, int threads, int cap = 148 * 16) {
  size_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > size_t(cap)) b = cap;
  return int(b);
}


// dense bytes (reference Bool / U16-as-mask layout) -> bit-packed rows
__global__ void k_pack_u8(const uint8_t* __restrict__ dense, uint32_t* __restrict__ bits, int w,
                          int h, int wpr, size_t pitch, size_t nwords_total) {
  slcs_pdl_wait();
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords_total;
       q += size_t(gridDim.x) * blockDim.x) {
    size_t row = q / pitch;  // global row over the batch
    int j = int(q - row * pitch);
    uint32_t word = 0;
    if (j < wpr) {
      const uint8_t* src = dense + row * size_t(w) + size_t(j) * 32;
      int n = min(32, w - j * 32);
      for (int b = 0; b < n; ++b) word |= (src[b] != 0 ? 1u : 0u) << b;
    }
    bits[q] = word;
  }
}

// 1 B/px -> bits for rows of a multiple of 128 px (no padding words): a thread
// packs 16 bytes from one coalesced 16 B load (4 bytes -> 4 bits by one
// multiply), and an even lane joins its odd neighbour's half into a word.
__device__ __forceinline__ uint32_t nz4(uint32_t v) {
  const uint32_t x = __vcmpne4(v, 0u) & 0x01010101u;
  return (x * 0x01020408u) >> 24;
}
__global__ void k_pack_u8_vec(const uint4* __restrict__ dense, uint32_t* __restrict__ bits,
                              size_t halves) {
  slcs_pdl_wait();
  // warp-uniform trip count (blockDim is a multiple of 32), so the whole warp
  // takes part in every shuffle; lanes past the end load nothing
  const unsigned lane = threadIdx.x & 31u;
  for (size_t base = size_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); base < halves;
       base += size_t(gridDim.x) * blockDim.x) {
    const size_t i = base + lane;
    const bool ok = i < halves;
    const uint4 v = ok ? __ldg(dense + i) : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t h = nz4(v.x) | (nz4(v.y) << 4) | (nz4(v.z) << 8) | (nz4(v.w) << 12);
    const uint32_t hi = __shfl_down_sync(0xffffffffu, h, 1);
    if (ok && !(i & 1)) bits[i >> 1] = h | (hi << 16);
  }
}

// bits -> 1 B/px for rows of a multiple of 128 px: 16 pixels per thread, a
// nibble spread to four 0/1 bytes by one multiply, one 16 B store
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }
__global__ void k_unpack_vec(const uint32_t* __restrict__ bits, uint4* __restrict__ dense,
                             size_t halves) {
  slcs_pdl_wait();
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < halves;
       i += size_t(gridDim.x) * blockDim.x) {
    const uint32_t h = (__ldg(bits + (i >> 1)) >> ((i & 1) * 16)) & 0xffffu;
    dense[i] = make_uint4(spread4(h & 15u), spread4((h >> 4) & 15u), spread4((h >> 8) & 15u),
                          spread4(h >> 12));
  }
}

__global__ void k_pack_u16(const uint16_t* __restrict__ dense, uint32_t* __restrict__ bits, int w,
                           int wpr, size_t pitch, size_t nwords_total) {
  slcs_pdl_wait();
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords_total;
       q += size_t(gridDim.x) * blockDim.x) {
    size_t row = q / pitch;
    int j = int(q - row * pitch);
    uint32_t word = 0;
    if (j < wpr) {
      const uint16_t* src = dense + row * size_t(w) + size_t(j) * 32;
      int n = min(32, w - j * 32);
      for (int b = 0; b < n; ++b) word |= (src[b] != 0 ? 1u : 0u) << b;
    }
    bits[q] = word;
  }
}

// bits -> dense bytes: one thread per output byte group of 4 pixels
__global__ void k_unpack(const uint32_t* __restrict__ bits, uint8_t* __restrict__ dense, int w,
                         size_t pitch, size_t npix_total) {
  slcs_pdl_wait();
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < npix_total;
       i += size_t(gridDim.x) * blockDim.x) {
    size_t row = i / size_t(w);
    int c = int(i - row * size_t(w));
    uint32_t word = __ldg(bits + row * pitch + (c >> 5));
    dense[i] = uint8_t((word >> (c & 31)) & 1u);
  }
}

// u16 rows between two pitches (dense host layout <-> the padded device
// layout), padding columns zeroed.  Replaces cudaMemcpy2D for short rows
// (C3's 240-px slices: 37,200 rows of 480 B), which the copy engine moves
// row by row.
__global__ void k_repitch_u16(const uint16_t* __restrict__ src, size_t spitch,
                              uint16_t* __restrict__ dst, size_t dpitch, int w, size_t total) {
  slcs_pdl_wait();
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const size_t row = i / dpitch;
    const int c = int(i - row * dpitch);
    dst[i] = c < w ? __ldg(src + row * spitch + c) : uint16_t(0);
  }
}

// threshold: one thread per output word; 4 x 16 B loads of u16 pixels.
__global__ void k_threshold(const uint16_t* __restrict__ px, uint32_t* __restrict__ bits,
                            int wpr, uint32_t lastmask, size_t bpitch, size_t upitch,
                            size_t nwords_total, int lo, int hi) {
  slcs_pdl_wait();
  const unsigned span = unsigned(hi - lo);  // valid only when lo <= hi
  const bool empty = lo > hi;
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords_total;
       q += size_t(gridDim.x) * blockDim.x) {
    size_t row = q / bpitch;
    int j = int(q - row * bpitch);
    uint32_t word = 0;
    if (j < wpr && !empty) {
      const uint4* src = reinterpret_cast<const uint4*>(px + row * upitch + size_t(j) * 32);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 x = __ldg(src + v);
        uint32_t comp[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          unsigned p0 = comp[e] & 0xffffu, p1 = comp[e] >> 16;
          word |= (unsigned(p0 - unsigned(lo)) <= span ? 1u : 0u) << (v * 8 + e * 2);
          word |= (unsigned(p1 - unsigned(lo)) <= span ? 1u : 0u) << (v * 8 + e * 2 + 1);
        }
      }
      word &= valid_mask(j, wpr, lastmask);
    }
    bits[q] = word;
  }
}

__device__ __forceinline__ void interval_of(int op, double n, int& lo, int& hi) {
  // Appendix A #5 of SURVEY.md: double(p) op n on integer p in [0, 65535]
  double l = 0.0, u = 65535.0;
  if (n != n) {
    lo = 1;
    hi = 0;
    return;
  }
  switch (op) {
    case SLCS_GT: l = floor(n) + 1.0; break;
    case SLCS_GE: l = ceil(n); break;
    case SLCS_LT: u = ceil(n) - 1.0; break;
    case SLCS_LE: u = floor(n); break;
    default:
      if (floor(n) != n) {
        lo = 1;
        hi = 0;
        return;
      }
      l = u = n;
  }
  if (l < 0.0) l = 0.0;
  if (u > 65535.0) u = 65535.0;
  if (l > u) {
    lo = 1;
    hi = 0;
    return;
  }
  lo = int(l);
  hi = int(u);
}

__global__ void k_threshold_dev(const uint16_t* __restrict__ px, uint32_t* __restrict__ bits,
                                int wpr, uint32_t lastmask, size_t bpitch, size_t upitch,
                                size_t nwords_total, int op, const double* n_dev) {
  slcs_pdl_wait();
  int lo, hi;
  interval_of(op, *n_dev, lo, hi);
  const unsigned span = unsigned(hi - lo);
  const bool empty = lo > hi;
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords_total;
       q += size_t(gridDim.x) * blockDim.x) {
    size_t row = q / bpitch;
    int j = int(q - row * bpitch);
    uint32_t word = 0;
    if (j < wpr && !empty) {
      const uint16_t* src = px + row * upitch + size_t(j) * 32;
      for (int b = 0; b < 32; ++b) word |= (unsigned(src[b] - unsigned(lo)) <= span ? 1u : 0u) << b;
      word &= valid_mask(j, wpr, lastmask);
    }
    bits[q] = word;
  }
}

// NOT / AND / OR over uint4 groups (the row pitch is a multiple of 4 words).
// Grid-stride with UNR independent 16 B loads per operand in flight per
// thread; NOT re-masks the padding bits/words of every row.
constexpr int kUnr = 4;

__device__ __forceinline__ uint4 not_group(uint4 x, size_t q, size_t pitch4, int wpr,
                                           uint32_t lastmask) {
  const int j0 = int(q % pitch4) * 4;
  x.x = ~x.x & valid_mask(j0 + 0, wpr, lastmask);
  x.y = ~x.y & valid_mask(j0 + 1, wpr, lastmask);
  x.z = ~x.z & valid_mask(j0 + 2, wpr, lastmask);
  x.w = ~x.w & valid_mask(j0 + 3, wpr, lastmask);
  return x;
}

__global__ void k_not(const uint4* __restrict__ a, uint4* __restrict__ out, int wpr,
                      uint32_t lastmask, size_t pitch4, size_t n4) {
  slcs_pdl_wait();
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; q + (kUnr - 1) * stride < n4; q += kUnr * stride) {
    uint4 x[kUnr];
#pragma unroll
    for (int u = 0; u < kUnr; ++u) x[u] = __ldg(a + q + u * stride);
#pragma unroll
    for (int u = 0; u < kUnr; ++u) out[q + u * stride] = not_group(x[u], q + u * stride, pitch4, wpr, lastmask);
  }
  for (; q < n4; q += stride) out[q] = not_group(__ldg(a + q), q, pitch4, wpr, lastmask);
}

template <int OP>
__device__ __forceinline__ uint4 bin_group(uint4 x, const uint4 y) {
  if (OP == 0) {
    x.x &= y.x; x.y &= y.y; x.z &= y.z; x.w &= y.w;
  } else {
    x.x |= y.x; x.y |= y.y; x.z |= y.z; x.w |= y.w;
  }
  return x;
}

template <int OP>
__global__ void k_binop(const uint4* __restrict__ a, const uint4* __restrict__ b,
                        uint4* __restrict__ out, size_t n4) {
  slcs_pdl_wait();
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; q + (kUnr - 1) * stride < n4; q += kUnr * stride) {
    uint4 x[kUnr], y[kUnr];
#pragma unroll
    for (int u = 0; u < kUnr; ++u) {
      x[u] = __ldg(a + q + u * stride);
      y[u] = __ldg(b + q + u * stride);
    }
#pragma unroll
    for (int u = 0; u < kUnr; ++u) out[q + u * stride] = bin_group<OP>(x[u], y[u]);
  }
  for (; q < n4; q += stride) out[q] = bin_group<OP>(__ldg(a + q), __ldg(b + q));
}

// Rows above / below the image supplied by a neighbouring row band:
// image row r < 0 is top[(r + ntop) * pitch], r >= h is bot[(r - h) * pitch];
// rows beyond the halo are absent (the clipping identity).  An empty Halo (the
// default) is a whole image.  Single images only (batch 1).
struct Halo {
  const uint32_t* top = nullptr;
  const uint32_t* bot = nullptr;
  int ntop = 0, nbot = 0;
};
__device__ __forceinline__ const uint32_t* row_at(const uint32_t* src, int r, int h, size_t pitch,
                                                  const Halo& hl) {
  if (r >= 0 && r < h) return src + size_t(r) * pitch;
  if (r < 0 && r >= -hl.ntop) return hl.top + size_t(r + hl.ntop) * pitch;
  if (r >= h && r < h + hl.nbot) return hl.bot + size_t(r - h) * pitch;
  return nullptr;
}

// k-fold near / interior.  Thread = (16 B column group q of 4 words, strip of
// S rows).  All S + 2K input rows are loaded up front (one uint4 plus the two
// neighbouring words per row, independent loads -> deep memory-level
// parallelism), each row is dilated (eroded) horizontally with funnel shifts,
// then the (2K+1)-row window is OR-ed (AND-ed) vertically and S uint4 rows are
// stored.  Rows/columns outside the image are absent: 0 for dilation
// (kernels.cpp:106-121), 1 for erosion (interior(all) = all,
// tests/test_reach.cpp:120); padding bits/words of the output stay zero.
template <int K, bool ERODE, int S>
__global__ void __launch_bounds__(128) k_near(const uint32_t* __restrict__ in,
                                              uint32_t* __restrict__ out, int h, int wpr,
                                              uint32_t lastmask, int pitch4, size_t slice,
                                              int nstrips, Halo hl) {
  slcs_pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = t / pitch4, q = t - s * pitch4;
  if (s >= nstrips) return;
  const uint32_t* src = in + size_t(blockIdx.y) * slice;
  uint4* dst = reinterpret_cast<uint4*>(out + size_t(blockIdx.y) * slice);
  const int r0 = s * S, j0 = 4 * q;
  const int rows = min(S, h - r0);
  const size_t pitch = size_t(pitch4) * 4;
  if (j0 >= wpr) {  // a group of padding words: stays zero
    for (int i = 0; i < rows; ++i) dst[size_t(r0 + i) * pitch4 + q] = make_uint4(0, 0, 0, 0);
    return;
  }
  constexpr uint32_t ID = ERODE ? 0xffffffffu : 0u;
  uint32_t pad[5];  // erosion: out-of-image bits of words j0..j0+4 act as 1
#pragma unroll
  for (int e = 0; e < 5; ++e) pad[e] = ERODE ? ~valid_mask(j0 + e, wpr, lastmask) : 0u;
  const bool has_l = j0 > 0, has_r = j0 + 4 < wpr;

  uint32_t hr[S + 2 * K][4];
#pragma unroll
  for (int i = 0; i < S + 2 * K; ++i) {
    const int r = r0 - K + i;
    uint32_t w[6];
    const uint32_t* row = row_at(src, r, h, pitch, hl);
    if (!row) {
#pragma unroll
      for (int e = 0; e < 6; ++e) w[e] = ID;
    } else {
      const uint4 c = __ldg(reinterpret_cast<const uint4*>(row + j0));
      w[0] = has_l ? __ldg(row + j0 - 1) : ID;
      w[1] = c.x | pad[0];
      w[2] = c.y | pad[1];
      w[3] = c.z | pad[2];
      w[4] = c.w | pad[3];
      w[5] = has_r ? (__ldg(row + j0 + 4) | pad[4]) : ID;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t acc = w[e + 1];
#pragma unroll
      for (int d = 1; d <= K; ++d) {
        const uint32_t lft = __funnelshift_l(w[e], w[e + 1], d);
        const uint32_t rgt = __funnelshift_r(w[e + 1], w[e + 2], d);
        acc = ERODE ? (acc & lft & rgt) : (acc | lft | rgt);
      }
      hr[i][e] = acc;
    }
  }
  uint32_t vm[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) vm[e] = valid_mask(j0 + e, wpr, lastmask);
#pragma unroll
  for (int i = 0; i < S; ++i) {
    if (i < rows) {
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t acc = hr[i][e];
#pragma unroll
        for (int d = 1; d <= 2 * K; ++d) acc = ERODE ? (acc & hr[i + d][e]) : (acc | hr[i + d][e]);
        o[e] = acc & vm[e];
      }
      dst[size_t(r0 + i) * pitch4 + q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// k >= 2: a strip of S rows streamed through a (2K+1)-row register ring; P new
// rows are loaded per step (independent loads in flight) so the 2K halo rows
// are amortised over a long strip instead of being re-read per short strip.
// A thread owns W consecutive words of the strip (W = 4: one uint4 per row);
// smaller images use W = 2 or 1 so that the grid still fills the GPU.
template <int W>
struct WordVec;
template <>
struct WordVec<4> {
  using V = uint4;
  __device__ static void load(const uint32_t* p, uint32_t (&o)[4]) {
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(p));
    o[0] = c.x, o[1] = c.y, o[2] = c.z, o[3] = c.w;
  }
  __device__ static void store(uint32_t* p, const uint32_t (&o)[4]) {
    *reinterpret_cast<uint4*>(p) = make_uint4(o[0], o[1], o[2], o[3]);
  }
};
template <>
struct WordVec<2> {
  __device__ static void load(const uint32_t* p, uint32_t (&o)[2]) {
    const uint2 c = __ldg(reinterpret_cast<const uint2*>(p));
    o[0] = c.x, o[1] = c.y;
  }
  __device__ static void store(uint32_t* p, const uint32_t (&o)[2]) {
    *reinterpret_cast<uint2*>(p) = make_uint2(o[0], o[1]);
  }
};
template <>
struct WordVec<1> {
  __device__ static void load(const uint32_t* p, uint32_t (&o)[1]) { o[0] = __ldg(p); }
  __device__ static void store(uint32_t* p, const uint32_t (&o)[1]) { *p = o[0]; }
};

template <int K, bool ERODE, int S, int P, int W>
__global__ void __launch_bounds__(128) k_near_stream(const uint32_t* __restrict__ in,
                                                     uint32_t* __restrict__ out, int h, int wpr,
                                                     uint32_t lastmask, int groups, size_t slice,
                                                     int nstrips, Halo hl) {
  slcs_pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = t / groups, q = t - s * groups;
  if (s >= nstrips) return;
  const uint32_t* src = in + size_t(blockIdx.y) * slice;
  uint32_t* dst = out + size_t(blockIdx.y) * slice;
  const int r0 = s * S, j0 = W * q;
  const int rows = min(S, h - r0);
  const size_t pitch = size_t(groups) * W;
  if (j0 >= wpr) {
    const uint32_t z[W] = {};
    for (int i = 0; i < rows; ++i) WordVec<W>::store(dst + size_t(r0 + i) * pitch + j0, z);
    return;
  }
  constexpr uint32_t ID = ERODE ? 0xffffffffu : 0u;
  uint32_t pad[W + 1];
#pragma unroll
  for (int e = 0; e < W + 1; ++e) pad[e] = ERODE ? ~valid_mask(j0 + e, wpr, lastmask) : 0u;
  const bool has_l = j0 > 0, has_r = j0 + W < wpr;
  uint32_t vm[W];
#pragma unroll
  for (int e = 0; e < W; ++e) vm[e] = valid_mask(j0 + e, wpr, lastmask);

  // one input row -> its horizontal dilation (erosion) by K bits
  auto hdil = [&](const uint32_t* row, uint32_t (&o)[W]) {
    uint32_t w[W + 2];
    if (!row) {
#pragma unroll
      for (int e = 0; e < W + 2; ++e) w[e] = ID;
    } else {
      uint32_t c[W];
      WordVec<W>::load(row + j0, c);
      w[0] = has_l ? __ldg(row + j0 - 1) : ID;
#pragma unroll
      for (int e = 0; e < W; ++e) w[e + 1] = c[e] | pad[e];
      w[W + 1] = has_r ? (__ldg(row + j0 + W) | pad[W]) : ID;
    }
#pragma unroll
    for (int e = 0; e < W; ++e) {
      uint32_t acc = w[e + 1];
#pragma unroll
      for (int d = 1; d <= K; ++d) {
        const uint32_t lft = __funnelshift_l(w[e], w[e + 1], d);
        const uint32_t rgt = __funnelshift_r(w[e + 1], w[e + 2], d);
        acc = ERODE ? (acc & lft & rgt) : (acc | lft | rgt);
      }
      o[e] = acc;
    }
  };
  // the strip through a (2K + P)-row register ring; FULL: every input row is an
  // image row and every output row exists, so rows are a pointer walk with no
  // per-row bounds or halo logic (all strips but the first and last)
  auto run = [&](auto full) {
    constexpr bool FULL = decltype(full)::value;
    const uint32_t* rp = src + size_t(r0 - K) * pitch;
    uint32_t* dp = dst + size_t(r0) * pitch + j0;
    auto fetch = [&](int r, uint32_t (&o)[W]) {
      if (FULL) {
        hdil(rp, o);
        rp += pitch;
      } else {
        hdil(row_at(src, r, h, pitch, hl), o);
      }
    };
    uint32_t ring[2 * K + P][W];
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) fetch(r0 - K + i, ring[i]);
#pragma unroll
    for (int c = 0; c < S; c += P) {
#pragma unroll
      for (int p = 0; p < P; ++p) fetch(r0 + c + K + p, ring[2 * K + p]);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (FULL || c + p < rows) {
          uint32_t o[W];
#pragma unroll
          for (int e = 0; e < W; ++e) {
            uint32_t acc = ring[p][e];
#pragma unroll
            for (int d = 1; d <= 2 * K; ++d)
              acc = ERODE ? (acc & ring[p + d][e]) : (acc | ring[p + d][e]);
            o[e] = acc & vm[e];
          }
          WordVec<W>::store(dp, o);
        }
        dp += pitch;
      }
#pragma unroll
      for (int i = 0; i < 2 * K; ++i)
#pragma unroll
        for (int e = 0; e < W; ++e) ring[i][e] = ring[i + P][e];
    }
  };
  if (r0 - K >= 0 && r0 + S + K <= h)
    run(std::true_type{});
  else
    run(std::false_type{});
}

// ---- near / interior for wide images: bulk-async (TMA engine) slabs -----------
// A persistent CTA walks slabs of R output rows x the full row.  Rows are
// contiguous in HBM, so a slab's R + 2K input rows are ONE cp.async.bulk copy
// into shared memory, completed on an mbarrier; the next slab's copy is in
// flight while this one is computed (two stages).  Threads then stream their
// 16 B column groups down 4-row chunks from shared memory (register ring, one
// horizontal pass per row) and store uint4 words to HBM.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kBulkRC = 4;  // output rows per thread work item

template <int K, bool ERODE>
__global__ void __launch_bounds__(256) k_near_bulk(const uint32_t* __restrict__ in,
                                                   uint32_t* __restrict__ out, int h, int wpr,
                                                   uint32_t lastmask, int pitch4, size_t slice,
                                                   int R, int slabs_per_slice, int total, Halo hl) {
  slcs_pdl_wait();
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t pitch = size_t(pitch4) * 4;
  const int rows_in = R + 2 * K;
  const size_t stage_words = size_t(rows_in) * pitch;
  uint32_t* buf0 = reinterpret_cast<uint32_t*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * stage_words * 4);
  constexpr uint32_t ID = ERODE ? 0xffffffffu : 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // slab rows [r0 - K, r0 + R + K): up to three contiguous pieces -- the top
  // halo, the image, the bottom halo -- copied on one mbarrier
  auto issue = [&](int slab, int st) {  // thread 0
    const int sl = slab / slabs_per_slice, r0 = (slab % slabs_per_slice) * R;
    const int want_lo = r0 - K, want_hi = r0 + R + K;
    uint32_t* base = buf0 + st * stage_words;
    const int lo = max(0, want_lo), hi = min(h, want_hi);
    const int tlo = max(want_lo, -hl.ntop), thi = min(want_hi, 0);
    const int blo = max(want_lo, h), bhi = min(want_hi, h + hl.nbot);
    const size_t rowb = pitch * 4;
    unsigned bytes = unsigned(size_t(hi - lo) * rowb);
    if (thi > tlo) bytes += unsigned(size_t(thi - tlo) * rowb);
    if (bhi > blo) bytes += unsigned(size_t(bhi - blo) * rowb);
    mbar_expect_tx(&bar[st], bytes);
    bulk_g2s(base + size_t(lo - want_lo) * pitch, in + size_t(sl) * slice + size_t(lo) * pitch,
             unsigned(size_t(hi - lo) * rowb), &bar[st]);
    if (thi > tlo)
      bulk_g2s(base + size_t(tlo - want_lo) * pitch, hl.top + size_t(tlo + hl.ntop) * pitch,
               unsigned(size_t(thi - tlo) * rowb), &bar[st]);
    if (bhi > blo)
      bulk_g2s(base + size_t(blo - want_lo) * pitch, hl.bot + size_t(blo - h) * pitch,
               unsigned(size_t(bhi - blo) * rowb), &bar[st]);
  };
  if (threadIdx.x == 0 && int(blockIdx.x) < total) issue(blockIdx.x, 0);
  int it = 0;
  for (int slab = blockIdx.x; slab < total; slab += gridDim.x, ++it) {
    const int st = it & 1;
    if (threadIdx.x == 0 && slab + int(gridDim.x) < total) issue(slab + gridDim.x, st ^ 1);
    const int sl = slab / slabs_per_slice, r0 = (slab % slabs_per_slice) * R;
    uint32_t* b = buf0 + st * stage_words;
    // rows outside the image and its halo (not part of the copy) read as the identity
    const int top = max(0, K - r0 - hl.ntop), bot = max(0, r0 + R + K - h - hl.nbot);
    for (size_t q = threadIdx.x; q < size_t(top) * pitch; q += blockDim.x) b[q] = ID;
    for (size_t q = threadIdx.x; q < size_t(bot) * pitch; q += blockDim.x)
      b[size_t(rows_in - bot) * pitch + q] = ID;
    mbar_wait(&bar[st], unsigned(it >> 1) & 1u);
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(out + size_t(sl) * slice);
    const int items = pitch4 * (R / kBulkRC);
    for (int item = threadIdx.x; item < items; item += blockDim.x) {
      const int q = item % pitch4, c = item / pitch4;
      const int j0 = 4 * q;
      const int rr0 = c * kBulkRC;  // first output row of the chunk, slab-relative
      if (r0 + rr0 >= h) continue;
      if (j0 >= wpr) {
        for (int i = 0; i < kBulkRC && r0 + rr0 + i < h; ++i)
          dst[size_t(r0 + rr0 + i) * pitch4 + q] = make_uint4(0, 0, 0, 0);
        continue;
      }
      uint32_t pad[5], vm[4];
#pragma unroll
      for (int e = 0; e < 5; ++e) pad[e] = ERODE ? ~valid_mask(j0 + e, wpr, lastmask) : 0u;
#pragma unroll
      for (int e = 0; e < 4; ++e) vm[e] = valid_mask(j0 + e, wpr, lastmask);
      const bool has_l = j0 > 0, has_r = j0 + 4 < wpr;
      uint32_t hr[kBulkRC + 2 * K][4];
#pragma unroll
      for (int i = 0; i < kBulkRC + 2 * K; ++i) {
        const uint32_t* row = b + size_t(rr0 + i) * pitch;  // buffer row = slab row - K
        const uint4 cw = *reinterpret_cast<const uint4*>(row + j0);
        uint32_t w[6];
        w[0] = has_l ? row[j0 - 1] : ID;
        w[1] = cw.x | pad[0];
        w[2] = cw.y | pad[1];
        w[3] = cw.z | pad[2];
        w[4] = cw.w | pad[3];
        w[5] = has_r ? (row[j0 + 4] | pad[4]) : ID;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t acc = w[e + 1];
#pragma unroll
          for (int d = 1; d <= K; ++d) {
            const uint32_t lft = __funnelshift_l(w[e], w[e + 1], d);
            const uint32_t rgt = __funnelshift_r(w[e + 1], w[e + 2], d);
            acc = ERODE ? (acc & lft & rgt) : (acc | lft | rgt);
          }
          hr[i][e] = acc;
        }
      }
#pragma unroll
      for (int i = 0; i < kBulkRC; ++i) {
        if (r0 + rr0 + i < h) {
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t acc = hr[i][e];
#pragma unroll
            for (int d = 1; d <= 2 * K; ++d) acc = ERODE ? (acc & hr[i + d][e]) : (acc | hr[i + d][e]);
            o[e] = acc & vm[e];
          }
          dst[size_t(r0 + rr0 + i) * pitch4 + q] = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
    }
    __syncthreads();  // stage st is reused by the copy issued two slabs later
  }
}

// slab height for the bulk path: R + 2K input rows in <= 52 KB per stage (two
// stages, two CTAs per SM), R a multiple of the 4-row chunk; 0 when rows are too
// wide or the image too small.  Used for K = 1 (near / interior): for K >= 2 the
// 2K halo rows per slab cost more than the streaming kernel's long strips
// (measured: near^4 at 16384^2 0.39 -> 0.32 of peak on the bulk path).
inline int bulk_slab_rows(const Geo& g, int k) {
  const size_t rowbytes = g.pitch * 4;
  if (k != 1 || g.pitch < 128 || size_t(g.h) * size_t(g.batch) < 512) return 0;
  int R = int(53248 / rowbytes) - 2 * k;
  R = std::min(R, 32) / kBulkRC * kBulkRC;
  return R >= kBulkRC ? R : 0;
}

template <int K, bool ERODE>
bool near_bulk_launch(const uint32_t* a, uint32_t* out, const Geo& g, cudaStream_t st,
                      const Halo& hl) {
  static const bool off = [] {
    const char* e = std::getenv("SLCS_NO_BULK_NEAR");
    return e && *e && *e != '0';
  }();
  const int R = bulk_slab_rows(g, K);
  if (off || R == 0) return false;
  const size_t smem = 2 * size_t(R + 2 * K) * g.pitch * 4 + 16;
  static PerDevice<int> attr;
  smem_opt_in(attr, k_near_bulk<K, ERODE>, 112 * 1024);
  const int per_slice = (g.h + R - 1) / R;
  const int total = per_slice * g.batch;
  const int ctas = std::min(total, device_sm_count() * 2);
  pdl(k_near_bulk<K, ERODE>, ctas, 256, smem, st, a, out, g.h, g.wpr, g.lastmask,
      int(g.pitch / 4), g.slice, R, per_slice, total, hl);
  return true;
}

template <int K, bool ERODE>
void near_launch(const uint32_t* a, uint32_t* out, const Geo& g, cudaStream_t st,
                 const Halo& hl) {
  if (near_bulk_launch<K, ERODE>(a, out, g, st, hl)) return;
  const int pitch4 = int(g.pitch / 4);
  const int block = 128;
  if (K == 1) {
    constexpr int S = 4;
    const int nstrips = (g.h + S - 1) / S;
    const size_t threads = size_t(pitch4) * size_t(nstrips);
    dim3 grid(unsigned((threads + block - 1) / block), unsigned(g.batch));
    pdl(k_near<K, ERODE, S>, grid, block, 0, st, a, out, g.h, g.wpr, g.lastmask, pitch4, g.slice,
        nstrips, hl);
  } else {
    // long strips amortise the 2K halo rows (32 rows, a uint4 of words per
    // thread); images too small to fill the GPU that way use 16-row strips of
    // two words per thread (measured at 16384^2: 16 x 2 = 27 us, 16 x 4 = 27,
    // 16 x 1 = 29, 32 x 2 = 32, 32 x 4 = 36)
#ifndef SLCS_NS_P
#define SLCS_NS_P 4
#endif
    constexpr int P = SLCS_NS_P;
    const bool big = size_t(g.pitch / 4) * size_t((g.h + 31) / 32) * size_t(g.batch) >= 148u * 2048u;
    const int S = big ? 32 : 16, W = big ? 4 : 2;
    const int nstrips = (g.h + S - 1) / S;
    const int groups = int(g.pitch / W);
    const size_t threads = size_t(groups) * size_t(nstrips);
    dim3 grid(unsigned((threads + block - 1) / block), unsigned(g.batch));
    auto go = [&](auto kern) {
      pdl(kern, grid, block, 0, st, a, out, g.h, g.wpr, g.lastmask, groups, g.slice, nstrips, hl);
    };
    if (big) go(k_near_stream<K, ERODE, 32, P, 4>);
    else go(k_near_stream<K, ERODE, 16, P, 2>);
  }
}

template <bool ERODE>
void near_dispatch(const uint32_t* a, uint32_t* out, const Geo& g, int k, cudaStream_t st,
                   const Halo& hl) {
  switch (k) {
    case 1: near_launch<1, ERODE>(a, out, g, st, hl); break;
    case 2: near_launch<2, ERODE>(a, out, g, st, hl); break;
    case 3: near_launch<3, ERODE>(a, out, g, st, hl); break;
    case 4: near_launch<4, ERODE>(a, out, g, st, hl); break;
    case 5: near_launch<5, ERODE>(a, out, g, st, hl); break;
    case 6: near_launch<6, ERODE>(a, out, g, st, hl); break;
    case 7: near_launch<7, ERODE>(a, out, g, st, hl); break;
    case 8: near_launch<8, ERODE>(a, out, g, st, hl); break;
    default: fail(SLCS_ERR_ARG, "near: k out of range");
  }
}

// volume: one launch.  8 independent uint4 loads in flight per thread,
// popcount, warp + block reduction, then ONE returning 64-bit atomic per CTA on
// the slice's accumulator, which packs (count << 20) | CTAs-arrived: the CTA
// that sees CTAs-arrived == gridDim.x - 1 is the last, and the value it got
// back already holds every other CTA's count (one location, so the atomic's
// total order is the synchronisation -- no fences, no second counter).  That
// CTA publishes the count (u64 and/or double) and resets the accumulator to
// zero, so no memset launch is needed (acc must be zero before the first use).
// Counts up to 2^44 px, grids up to 2^20 CTAs per slice.
__device__ __forceinline__ void vol_body(const uint4* __restrict__ src, size_t n4,
                                         unsigned long long* acc,
                                         unsigned long long* __restrict__ counts,
                                         double* __restrict__ dbl) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long local = 0;
  for (; q + 7 * stride < n4; q += 8 * stride) {
    uint4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(src + q + u * stride);
    unsigned c = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) c += __popc(x[u].x) + __popc(x[u].y) + __popc(x[u].z) + __popc(x[u].w);
    local += c;
  }
  for (; q < n4; q += stride) {
    const uint4 x = __ldg(src + q);
    local += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
  }
  // the reads are done: let the next kernel's CTAs launch during the reduction
  // tail (they still wait for this grid to complete before reading anything)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ unsigned long long part[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) part[wid] = local;
  __syncthreads();
  if (wid == 0) {
    local = lane < int(blockDim.x >> 5) ? part[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if (lane == 0) {
      const unsigned long long old = atomicAdd(acc, (local << 20) | 1ull);
      if ((old & 0xfffffull) == gridDim.x - 1) {
        const unsigned long long total = (old >> 20) + local;
        *acc = 0ull;
        if (counts) *counts = total;
        if (dbl) *dbl = double(total);
      }
    }
  }
}

// one slice per blockIdx.y
__global__ void k_volume(const uint4* __restrict__ a, size_t slice4, unsigned long long* acc,
                         unsigned long long* __restrict__ counts, double* __restrict__ dbl) {
  slcs_pdl_wait();
  const int s = blockIdx.y;
  vol_body(a + size_t(s) * slice4, slice4, acc + s, counts ? counts + s : nullptr,
           dbl ? dbl + s : nullptr);
}

// independent volumes of different images in one launch, one per blockIdx.y
// (a device program's adjacent volume steps: one launch instead of n)
__global__ void k_volume_multi(VolumeJobs jobs) {
  slcs_pdl_wait();
  const VolumeJob& j = jobs.job[blockIdx.y];
  vol_body(reinterpret_cast<const uint4*>(j.a), j.words / 4, j.acc, j.counts, j.dbl);
}

// randomMask (tests/oracles.cpp:44-49) on device: pixel i of the full image
// consumes draw i of splitmix64(seed) (rng.hpp:14-19), so any row band is
// generated independently and bit-identically to the CPU fixture.
__global__ void k_random_mask(uint32_t* __restrict__ bits, int w, int h, long long row0,
                              int wpr, size_t pitch, unsigned long long seed, double density) {
  slcs_pdl_wait();
  const size_t n = pitch * size_t(h);
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += size_t(gridDim.x) * blockDim.x) {
    const size_t r = q / pitch;
    const int j = int(q - r * pitch);
    uint32_t word = 0;
    if (j < wpr) {
      const unsigned long long base =
          (unsigned long long)(row0 + (long long)r) * (unsigned long long)w + 32ull * j;
      const int nb = min(32, w - 32 * j);
      for (int b = 0; b < nb; ++b) {
        unsigned long long z = seed + (base + b + 1ull) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        const double u = double(z >> 11) * 0x1.0p-53;
        word |= (u < density ? 1u : 0u) << b;
      }
    }
    bits[q] = word;
  }
}

// uniform u16 fixture: pixel i = (draw i of splitmix64(seed)) % 65536, the
// reference's Rng::below(65536) per pixel (rng.hpp:21-23) -- the C5 threshold
// input.  Rows [row0, row0 + h) of a w-wide image; u16 rows use pitch `pitch`.
__global__ void k_random_u16(uint16_t* __restrict__ px, int w, int h, long long row0,
                             size_t pitch, unsigned long long seed) {
  slcs_pdl_wait();
  const size_t n = pitch * size_t(h);
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += size_t(gridDim.x) * blockDim.x) {
    const size_t r = q / pitch;
    const int c = int(q - r * pitch);
    uint16_t v = 0;
    if (c < w) {
      const unsigned long long i =
          (unsigned long long)(row0 + (long long)r) * (unsigned long long)w + (unsigned long long)c;
      unsigned long long z = seed + (i + 1ull) * 0x9e3779b97f4a7c15ull;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      z ^= z >> 31;
      v = uint16_t(z & 0xffffu);
    }
    px[q] = v;
  }
}

}  // namespace

int launch_random_u16(uint16_t* px, const Geo& g, long long row0, unsigned long long seed,
                      cudaStream_t st) {
  size_t n = g.slice;
  pdl(k_random_u16, grid_for(n, kThreads, 148 * 32), kThreads, 0, st, px, g.w, g.h, row0,
      g.pitch, seed);
  return 1;
}

int launch_pack_u8(const uint8_t* dense, uint32_t* bits, const Geo& g, bool, cudaStream_t st) {
  if (g.w % 128 == 0 && g.pitch == size_t(g.wpr) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0) {
    const size_t halves = size_t(g.w) / 16 * size_t(g.h) * size_t(g.batch);
    pdl(k_pack_u8_vec, grid_for(halves, kThreads, 148 * 16), kThreads, 0, st,
        reinterpret_cast<const uint4*>(dense), bits, halves);
    return 1;
  }
  size_t n = g.slice * size_t(g.batch);
  pdl(k_pack_u8, grid_for(n, kThreads), kThreads, 0, st, dense, bits, g.w, g.h, g.wpr, g.pitch,
                                                        n);
  return 1;
}

int launch_pack_u16_mask(const uint16_t* dense, uint32_t* bits, const Geo& g, cudaStream_t st) {
  size_t n = g.slice * size_t(g.batch);
  pdl(k_pack_u16, grid_for(n, kThreads), kThreads, 0, st, dense, bits, g.w, g.wpr, g.pitch, n);
  return 1;
}

int launch_repitch_u16(const uint16_t* src, size_t spitch, uint16_t* dst, size_t dpitch, int w,
                       size_t rows, cudaStream_t st) {
  const size_t total = dpitch * rows;
  pdl(k_repitch_u16, grid_for(total, kThreads, 148 * 32), kThreads, 0, st, src, spitch, dst,
      dpitch, w, total);
  return 1;
}

int launch_unpack(const uint32_t* bits, uint8_t* dense, const Geo& g, cudaStream_t st) {
  if (g.w % 128 == 0 && g.pitch == size_t(g.wpr) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0) {
    const size_t halves = size_t(g.w) / 16 * size_t(g.h) * size_t(g.batch);
    pdl(k_unpack_vec, grid_for(halves, kThreads, 148 * 16), kThreads, 0, st, bits,
        reinterpret_cast<uint4*>(dense), halves);
    return 1;
  }
  size_t n = size_t(g.w) * size_t(g.h) * size_t(g.batch);
  pdl(k_unpack, grid_for(n, kThreads, 148 * 32), kThreads, 0, st, bits, dense, g.w, g.pitch, n);
  return 1;
}

int launch_threshold(const uint16_t* px, uint32_t* bits, const Geo& gu, const Geo& gb, int lo,
                     int hi, cudaStream_t st) {
  size_t n = gb.slice * size_t(gb.batch);
  pdl(k_threshold, grid_for(n, kThreads, 148 * 32), kThreads, 0, st, 
      px, bits, gb.wpr, gb.lastmask, gb.pitch, gu.pitch, n, lo, hi);
  return 1;
}

int launch_threshold_dev(const uint16_t* px, uint32_t* bits, const Geo& gu, const Geo& gb,
                         int op, const double* n_dev, cudaStream_t st) {
  size_t n = gb.slice * size_t(gb.batch);
  pdl(k_threshold_dev, grid_for(n, kThreads, 148 * 32), kThreads, 0, st, 
      px, bits, gb.wpr, gb.lastmask, gb.pitch, gu.pitch, n, op, n_dev);
  return 1;
}

int launch_not(const uint32_t* a, uint32_t* out, const Geo& g, cudaStream_t st) {
  size_t n4 = g.slice * size_t(g.batch) / 4;
  pdl(k_not, grid_for(n4, kThreads * kUnr, 148 * 8), kThreads, 0, st, 
      reinterpret_cast<const uint4*>(a), reinterpret_cast<uint4*>(out), g.wpr, g.lastmask,
      g.pitch / 4, n4);
  return 1;
}

int launch_and(const uint32_t* a, const uint32_t* b, uint32_t* out, const Geo& g,
               cudaStream_t st) {
  size_t n4 = g.slice * size_t(g.batch) / 4;
  pdl(k_binop<0>, grid_for(n4, kThreads * kUnr, 148 * 8), kThreads, 0, st, 
      reinterpret_cast<const uint4*>(a), reinterpret_cast<const uint4*>(b),
      reinterpret_cast<uint4*>(out), n4);
  return 1;
}

int launch_or(const uint32_t* a, const uint32_t* b, uint32_t* out, const Geo& g,
              cudaStream_t st) {
  size_t n4 = g.slice * size_t(g.batch) / 4;
  pdl(k_binop<1>, grid_for(n4, kThreads * kUnr, 148 * 8), kThreads, 0, st, 
      reinterpret_cast<const uint4*>(a), reinterpret_cast<const uint4*>(b),
      reinterpret_cast<uint4*>(out), n4);
  return 1;
}

int launch_near(const uint32_t* a, uint32_t* out, const Geo& g, int k, bool erode,
                cudaStream_t st) {
  return launch_near_halo(a, out, g, k, erode, nullptr, 0, nullptr, 0, st);
}

int launch_near_halo(const uint32_t* a, uint32_t* out, const Geo& g, int k, bool erode,
                     const uint32_t* top, int ntop, const uint32_t* bot, int nbot,
                     cudaStream_t st) {
  if (k < 1 || k > 8) fail(SLCS_ERR_ARG, "near: k must be in 1..8 per launch");
  if ((ntop > 0 || nbot > 0) && g.batch != 1) fail(SLCS_ERR_ARG, "halo rows need a single image");
  Halo hl;
  hl.top = top;
  hl.ntop = top ? ntop : 0;
  hl.bot = bot;
  hl.nbot = bot ? nbot : 0;
  if (erode)
    near_dispatch<true>(a, out, g, k, st, hl);
  else
    near_dispatch<false>(a, out, g, k, st, hl);
  return 1;
}

int launch_volume(const uint32_t* a, unsigned long long* counts, double* dbl,
                  unsigned long long* vscratch, const Geo& g, cudaStream_t st) {
  size_t n4 = g.slice / 4;
  int gx = grid_for(n4, kThreads * 8, 148 * 8);
  if (g.batch > 1) gx = std::max(1, std::min(gx, (148 * 8 + g.batch - 1) / g.batch));
  dim3 grid(unsigned(gx), unsigned(g.batch));
  pdl(k_volume, grid, kThreads, 0, st, reinterpret_cast<const uint4*>(a), n4, vscratch, counts,
      dbl);
  return 1;
}

int launch_volume_multi(const VolumeJobs& jobs, cudaStream_t st) {
  if (jobs.n < 1 || jobs.n > kVolumeJobsMax) fail(SLCS_ERR_ARG, "volume: bad job count");
  size_t n4 = 0;
  for (int i = 0; i < jobs.n; ++i) n4 = std::max(n4, jobs.job[i].words / 4);
  int gx = grid_for(n4, kThreads * 8, 148 * 8);
  gx = std::max(1, std::min(gx, (148 * 8 + jobs.n - 1) / jobs.n));
  pdl(k_volume_multi, dim3(unsigned(gx), unsigned(jobs.n)), kThreads, 0, st, jobs);
  return 1;
}

int launch_random_mask(uint32_t* bits, const Geo& g, long long row0, unsigned long long seed,
                       double density, cudaStream_t st) {
  size_t n = g.slice;
  pdl(k_random_mask, grid_for(n, kThreads, 148 * 32), kThreads, 0, st, bits, g.w, g.h, row0, g.wpr,
                                                                      g.pitch, seed, density);
  return 1;
}


}  // namespace slcs
