// png_raw_stub.cpp -- TEST INFRASTRUCTURE for the CPU-only reference build.
//
// The reference's png_io.cpp needs libpng, which is absent.  For
// running the reference's own unit suites against its own CPU code (the
// baseline that shows the harness is sound), loadPng/savePng here write a raw
// container instead of PNG: "SLCSRAW1", int32 width, height, kind, then the
// pixels.  Semantics follow png_io.hpp:12-20: Bool saves as u16 0/65535,
// loads always yield U16, numbers are rejected.  cliMain is provided by
// pixlog_slcs.cpp's GPU build only; the CPU build never calls it.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <vector>

#include "pixlog/png_io.hpp"

namespace pixlog {

Value loadPng(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw RunError("cannot open file for reading: " + path.string());
  char magic[8];
  int32_t hdr[3];
  in.read(magic, 8);
  in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  if (!in || std::memcmp(magic, "SLCSRAW1", 8) != 0)
    throw RunError("libpng: not a raw test image: " + path.string());
  ImageBuffer out(hdr[0], hdr[1], PixelKind::U16);
  in.read(reinterpret_cast<char*>(out.u16Data().data()), std::streamsize(out.pixelCount() * 2));
  return Value::image(std::move(out));
}

void savePng(const std::filesystem::path& path, const Value& v) {
  if (!v.isImage())
    throw RunError("cannot save a number as an image (use print): " + path.string());
  const ImageBuffer& img = v.img();
  std::vector<uint16_t> px(img.pixelCount());
  for (size_t i = 0; i < px.size(); ++i) {
    switch (img.kind()) {
      case PixelKind::Bool: px[i] = img.boolData()[i] ? 65535 : 0; break;
      case PixelKind::U16: px[i] = img.u16Data()[i]; break;
      case PixelKind::LabelPair: px[i] = uint16_t(img.labelData()[i]); break;
    }
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw RunError("cannot open file for writing: " + path.string());
  const int32_t hdr[3] = {img.width(), img.height(), int32_t(img.kind())};
  out.write("SLCSRAW1", 8);
  out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  out.write(reinterpret_cast<const char*>(px.data()), std::streamsize(px.size() * 2));
}

void labelColor(uint32_t packed, uint8_t rgb[3]) {
  rgb[0] = uint8_t(packed * 97u);
  rgb[1] = uint8_t(packed * 57u);
  rgb[2] = uint8_t(packed * 23u);
}

}  // namespace pixlog
