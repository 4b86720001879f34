// png.cu -- image ingest/egress for the device path: the
// reference's png_io (proj/src/png_io.cpp:30-144, libpng) restated on zlib.
//
//   load  PNG -> U16: 8/16-bit grey, grey+alpha, RGB, RGBA, Adam7 or not; the
//         first channel is kept and 8-bit samples widen by v * 257
//         (png_io.cpp:60-72); palette images and bit depths other than 8/16
//         are rejected with the reference's messages (png_io.cpp:52-58).
//   save  Bool -> 16-bit grey (true = 65535), U16 verbatim, labels -> 8-bit RGB
//         via the lowbias32 colour hash (png_io.cpp:75-143).
//
// The container parse, CRC checks, inflate/deflate and the row unfiltering
// are byte-serial and stay on the host (zlib); the per-pixel work -- channel
// selection, byte order, widening, the bit-image expansion and the label
// colouring -- runs on the device next to the image, so only the PNG byte
// stream crosses PCIe.
#include <zlib.h>

#include <cstring>
#include <string>
#include <vector>

#include "slcs_internal.h"

namespace slcs {
namespace {

[[noreturn]] void png_fail(const std::string& msg) { fail(SLCS_ERR_RUN, "libpng: " + msg); }

uint32_t be32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}
void put32(std::vector<uint8_t>& v, uint32_t x) {
  v.push_back(uint8_t(x >> 24));
  v.push_back(uint8_t(x >> 16));
  v.push_back(uint8_t(x >> 8));
  v.push_back(uint8_t(x));
}

const uint8_t kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

// PNG filter reconstruction of one scanline (ISO 15948 §9.2)
void unfilter(uint8_t* cur, const uint8_t* prev, size_t n, int bpp, int type) {
  switch (type) {
    case 0: break;
    case 1:
      for (size_t i = size_t(bpp); i < n; ++i) cur[i] = uint8_t(cur[i] + cur[i - bpp]);
      break;
    case 2:
      if (prev)
        for (size_t i = 0; i < n; ++i) cur[i] = uint8_t(cur[i] + prev[i]);
      break;
    case 3:
      for (size_t i = 0; i < n; ++i) {
        const int a = i >= size_t(bpp) ? cur[i - bpp] : 0, b = prev ? prev[i] : 0;
        cur[i] = uint8_t(cur[i] + ((a + b) >> 1));
      }
      break;
    case 4:
      for (size_t i = 0; i < n; ++i) {
        const int a = i >= size_t(bpp) ? cur[i - bpp] : 0, b = prev ? prev[i] : 0;
        const int c = (prev && i >= size_t(bpp)) ? prev[i - bpp] : 0;
        const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
        cur[i] = uint8_t(cur[i] + ((pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c)));
      }
      break;
    default: png_fail("bad adaptive filter value");
  }
}

// the `sub` image (w x h, rows of 1 + rowbytes filtered bytes) -> raw rows
void unfilter_image(const uint8_t* src, uint8_t* dst, int w, int h, int bpp) {
  const size_t rb = size_t(w) * size_t(bpp);
  for (int r = 0; r < h; ++r) {
    const uint8_t* in = src + size_t(r) * (rb + 1);
    uint8_t* out = dst + size_t(r) * rb;
    std::memcpy(out, in + 1, rb);
    unfilter(out, r ? out - rb : nullptr, rb, bpp, in[0]);
  }
}

}  // namespace

std::vector<uint8_t> png_decode(const uint8_t* data, size_t n, PngInfo& info) {
  if (n < 8 || std::memcmp(data, kSig, 8) != 0) png_fail("Not a PNG file");
  size_t p = 8;
  bool have_ihdr = false, have_iend = false;
  int depth = 0, color = 0, interlace = 0;
  std::vector<uint8_t> idat;
  while (p + 12 <= n && !have_iend) {
    const uint32_t len = be32(data + p);
    if (len > n - p - 12) png_fail("chunk length exceeds the file");
    const uint8_t* type = data + p + 4;
    const uint8_t* body = data + p + 8;
    const uint32_t crc = be32(body + len);
    if (uint32_t(crc32(crc32(0L, Z_NULL, 0), type, uInt(len + 4))) != crc &&
        !(type[0] & 0x20))  // ancillary chunks with bad CRCs are skipped, as libpng does
      png_fail(std::string(reinterpret_cast<const char*>(type), 4) + ": CRC error");
    if (!std::memcmp(type, "IHDR", 4)) {
      if (len != 13) png_fail("Invalid IHDR length");
      info.w = int(be32(body));
      info.h = int(be32(body + 4));
      depth = body[8];
      color = body[9];
      if (body[10] != 0 || body[11] != 0) png_fail("Unknown compression or filter method");
      interlace = body[12];
      if (info.w <= 0 || info.h <= 0) png_fail("Invalid image size in IHDR");
      have_ihdr = true;
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), body, body + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      have_iend = true;
    } else if (!std::memcmp(type, "PLTE", 4)) {
      // only meaningful for palette images, which are rejected below
    }
    p += size_t(len) + 12;
  }
  if (!have_ihdr) png_fail("Missing IHDR before IDAT");
  if (color == 3) fail(SLCS_ERR_RUN, "unsupported PNG: palette images are not supported");
  if (depth != 8 && depth != 16) fail(SLCS_ERR_RUN, "unsupported PNG bit depth " + std::to_string(depth));
  switch (color) {
    case 0: info.channels = 1; break;
    case 2: info.channels = 3; break;
    case 4: info.channels = 2; break;
    case 6: info.channels = 4; break;
    default: png_fail("Invalid color type in IHDR");
  }
  info.depth = depth;
  const int bpp = info.channels * depth / 8;
  const size_t rb = size_t(info.w) * size_t(bpp);
  // Adam7 pass geometry (start row, start col, row step, col step)
  static const int A7[7][4] = {{0, 0, 8, 8}, {0, 4, 8, 8}, {4, 0, 8, 4}, {0, 2, 4, 4},
                               {2, 0, 4, 2}, {0, 1, 2, 2}, {1, 0, 2, 1}};
  size_t filtered = 0;
  if (!interlace) {
    filtered = size_t(info.h) * (rb + 1);
  } else {
    for (const auto& a : A7) {
      const size_t pw = info.w > a[1] ? size_t(info.w - a[1] + a[3] - 1) / a[3] : 0;
      const size_t ph = info.h > a[0] ? size_t(info.h - a[0] + a[2] - 1) / a[2] : 0;
      if (pw && ph) filtered += ph * (pw * bpp + 1);
    }
  }
  std::vector<uint8_t> flt(filtered);
  uLongf out_len = uLongf(filtered);
  const int zr = uncompress(flt.data(), &out_len, idat.data(), uLong(idat.size()));
  if (zr != Z_OK && !(zr == Z_BUF_ERROR && out_len == filtered))
    png_fail(zr == Z_DATA_ERROR ? "IDAT: invalid distance too far back / incorrect header check"
                                : "IDAT: decompression failed");
  if (out_len != filtered) png_fail("Not enough image data");
  std::vector<uint8_t> raw(rb * size_t(info.h));
  if (!interlace) {
    unfilter_image(flt.data(), raw.data(), info.w, info.h, bpp);
  } else {
    size_t off = 0;
    std::vector<uint8_t> pass;
    for (const auto& a : A7) {
      const int pw = info.w > a[1] ? (info.w - a[1] + a[3] - 1) / a[3] : 0;
      const int ph = info.h > a[0] ? (info.h - a[0] + a[2] - 1) / a[2] : 0;
      if (!pw || !ph) continue;
      pass.resize(size_t(pw) * bpp * ph);
      unfilter_image(flt.data() + off, pass.data(), pw, ph, bpp);
      off += size_t(ph) * (size_t(pw) * bpp + 1);
      for (int y = 0; y < ph; ++y)
        for (int x = 0; x < pw; ++x)
          std::memcpy(raw.data() + size_t(a[0] + y * a[2]) * rb + size_t(a[1] + x * a[3]) * bpp,
                      pass.data() + (size_t(y) * pw + x) * bpp, size_t(bpp));
    }
  }
  return raw;
}

std::vector<uint8_t> png_encode(const uint8_t* rows, int w, int h, int depth, int color) {
  const int channels = color == 2 ? 3 : 1;
  const size_t n = size_t(h) * (size_t(w) * channels * depth / 8 + 1);
  uLongf cap = compressBound(uLong(n));
  std::vector<uint8_t> z(cap);
  // level 1: the pixel content is what the reference pins; speed over ratio
  if (compress2(z.data(), &cap, rows, uLong(n), 1) != Z_OK) png_fail("deflate failed");
  std::vector<uint8_t> out(kSig, kSig + 8);
  auto chunk = [&](const char* type, const uint8_t* body, size_t len) {
    put32(out, uint32_t(len));
    const size_t at = out.size();
    out.insert(out.end(), type, type + 4);
    out.insert(out.end(), body, body + len);
    put32(out, uint32_t(crc32(crc32(0L, Z_NULL, 0), out.data() + at, uInt(len + 4))));
  };
  uint8_t ihdr[13];
  const uint32_t dims[2] = {uint32_t(w), uint32_t(h)};
  for (int i = 0; i < 2; ++i)
    for (int b = 0; b < 4; ++b) ihdr[4 * i + b] = uint8_t(dims[i] >> (24 - 8 * b));
  ihdr[8] = uint8_t(depth);
  ihdr[9] = uint8_t(color);
  ihdr[10] = ihdr[11] = ihdr[12] = 0;
  chunk("IHDR", ihdr, 13);
  chunk("IDAT", z.data(), cap);
  chunk("IEND", nullptr, 0);
  return out;
}

namespace {

// raw rows (w x channels samples of depth bits) -> U16 image, first channel
__global__ void k_png_to_u16(const uint8_t* __restrict__ raw, uint16_t* __restrict__ out, int w,
                             int h, int channels, int depth, size_t upitch) {
  slcs_pdl_wait();
  const size_t n = size_t(w) * size_t(h);
  const size_t rb = size_t(w) * channels * (depth / 8);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const size_t r = i / size_t(w), c = i - r * size_t(w);
    const uint8_t* px = raw + r * rb + c * channels * (depth / 8);
    out[r * upitch + c] = depth == 16 ? uint16_t((px[0] << 8) | px[1]) : uint16_t(px[0] * 257u);
  }
}

__device__ __forceinline__ void label_rgb(uint32_t packed, uint8_t* rgb) {
  if (packed == 0) {
    rgb[0] = rgb[1] = rgb[2] = 0;
    return;
  }
  uint32_t x = packed;  // lowbias32 (png_io.cpp:75-90)
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  rgb[0] = uint8_t(x >> 16);
  rgb[1] = uint8_t(x >> 8);
  rgb[2] = uint8_t(x);
  if (!rgb[0] && !rgb[1] && !rgb[2]) rgb[2] = 1;  // black is reserved for null
}

// image -> PNG scanlines (filter byte 0 + samples): Bool / U16 as 16-bit grey
// big-endian, labels as 8-bit RGB
__global__ void k_png_rows(const void* __restrict__ img, int kind, int w, int h, size_t pitch,
                           uint8_t* __restrict__ rows) {
  slcs_pdl_wait();
  const size_t n = size_t(w) * size_t(h);
  const size_t rb = size_t(w) * (kind == SLCS_LABEL ? 3 : 2) + 1;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const size_t r = i / size_t(w), c = i - r * size_t(w);
    uint8_t* row = rows + r * rb;
    if (c == 0) row[0] = 0;
    if (kind == SLCS_LABEL) {
      label_rgb(static_cast<const uint32_t*>(img)[r * pitch + c], row + 1 + 3 * c);
    } else {
      uint16_t v;
      if (kind == SLCS_U16) {
        v = static_cast<const uint16_t*>(img)[r * pitch + c];
      } else {
        const uint32_t word = static_cast<const uint32_t*>(img)[r * pitch + (c >> 5)];
        v = ((word >> (c & 31)) & 1u) ? 65535 : 0;
      }
      row[1 + 2 * c] = uint8_t(v >> 8);
      row[2 + 2 * c] = uint8_t(v);
    }
  }
}

}  // namespace

int launch_png_to_u16(const uint8_t* raw, const PngInfo& info, uint16_t* out, const Geo& gu,
                      cudaStream_t st) {
  const size_t n = size_t(info.w) * size_t(info.h);
  pdl(k_png_to_u16, unsigned(std::min<size_t>((n + 255) / 256, 148 * 32)), 256, 0, st, raw, out,
      info.w, info.h, info.channels, info.depth, gu.pitch);
  return 1;
}

int launch_png_rows(const void* img, int kind, const Geo& g, uint8_t* rows, cudaStream_t st) {
  const size_t n = size_t(g.w) * size_t(g.h);
  pdl(k_png_rows, unsigned(std::min<size_t>((n + 255) / 256, 148 * 32)), 256, 0, st, img, kind,
      g.w, g.h, g.pitch, rows);
  return 1;
}

void png_label_color(uint32_t packed, uint8_t rgb[3]) {
  if (packed == 0) {
    rgb[0] = rgb[1] = rgb[2] = 0;
    return;
  }
  uint32_t x = packed;
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  rgb[0] = uint8_t(x >> 16);
  rgb[1] = uint8_t(x >> 8);
  rgb[2] = uint8_t(x);
  if (!rgb[0] && !rgb[1] && !rgb[2]) rgb[2] = 1;
}

}  // namespace slcs
