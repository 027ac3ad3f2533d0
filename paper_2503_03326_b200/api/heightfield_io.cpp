// heightfield_io.cpp — ABHF / CSV heightfields for the drop-in API.
// Host-field writers / readers follow the byte layout of the reference's
// heightfield_io.hpp:11-16 (its heightfield_io.cpp:30-103 behaviour, same
// IoError messages); the device overloads write straight from the fp32 maps
// through the C-ABI (ocn_heightfield_write_*).
#include "ocean/heightfield_io.hpp"

#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>

#include "ocean/interactive.hpp"
#include "ocean/surface.hpp"
#include "ocean_b200.h"

namespace ocean {

void throw_on_status(int st, const char* where);  // ocean_api.cpp

namespace {

// The whole file image: 16-byte header, then the samples as fp32.
std::vector<unsigned char> abhf_image(const HeightfieldHeader& h, const RealField& field) {
  const size_t nn = field.count();
  std::vector<unsigned char> img(16 + 4 * nn);
  unsigned char* p = img.data();
  std::memcpy(p, "ABHF", 4);
  std::memcpy(p + 4, &h.resolution, 4);
  std::memcpy(p + 8, &h.cascade, 4);
  std::memcpy(p + 12, &h.time, 4);
  const double* src = field.data();
  for (size_t q = 0; q < nn; ++q) {
    const float v = static_cast<float>(src[q]);
    std::memcpy(p + 16 + 4 * q, &v, 4);
  }
  return img;
}

template <typename T>
T take(const unsigned char* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

void read_exact(std::istream& in, unsigned char* dst, size_t bytes) {
  in.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(bytes));
  if (!in) throw IoError("heightfield: truncated stream");
}

std::vector<ocn_zone*> zone_handles(const std::vector<const FdmZone*>& zones) {
  std::vector<ocn_zone*> h;
  for (const FdmZone* z : zones) h.push_back(z->device_handle());
  return h;
}

}  // namespace

void write_heightfield(std::ostream& out, const HeightfieldHeader& header, const RealField& field) {
  if (static_cast<uint32_t>(field.size()) != header.resolution)
    throw IoError("heightfield: header resolution does not match field");
  const std::vector<unsigned char> img = abhf_image(header, field);
  out.write(reinterpret_cast<const char*>(img.data()), static_cast<std::streamsize>(img.size()));
  if (!out) throw IoError("heightfield: write failed");
}

RealField read_heightfield(std::istream& in, HeightfieldHeader* header) {
  unsigned char hdr[16];
  in.read(reinterpret_cast<char*>(hdr), 4);
  if (!in || std::memcmp(hdr, "ABHF", 4) != 0)
    throw IoError("heightfield: bad magic, not an ABHF file");
  read_exact(in, hdr + 4, 12);
  HeightfieldHeader h;
  h.resolution = take<uint32_t>(hdr + 4);
  h.cascade = take<int32_t>(hdr + 8);
  h.time = take<float>(hdr + 12);
  if (h.resolution == 0 || h.resolution > (1u << 16)) throw IoError("heightfield: bad resolution");
  RealField field(static_cast<int>(h.resolution));
  std::vector<unsigned char> raw(4 * field.count());
  read_exact(in, raw.data(), raw.size());
  double* dst = field.data();
  for (size_t q = 0; q < field.count(); ++q) dst[q] = take<float>(raw.data() + 4 * q);
  if (header) *header = h;
  return field;
}

void write_heightfield_file(const std::string& path, const HeightfieldHeader& header,
                            const RealField& field) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open for writing: " + path);
  write_heightfield(out, header, field);
}

RealField read_heightfield_file(const std::string& path, HeightfieldHeader* header) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open: " + path);
  return read_heightfield(in, header);
}

void write_heightfield_csv(std::ostream& out, const RealField& field) {
  out.precision(9);
  const int n = field.size();
  for (int i = 0; i < n; ++i) {
    const double* row = field.data() + static_cast<size_t>(i) * n;
    for (int j = 0; j < n; ++j) out << (j ? "," : "") << row[j];
    out << '\n';
  }
}

void write_heightfield_csv_file(const std::string& path, const RealField& field) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open for writing: " + path);
  write_heightfield_csv(out, field);
}

void write_heightfield_file(const std::string& path, const SurfaceMaps& maps, int cascade,
                            int field, double time) {
  throw_on_status(ocn_heightfield_write_field(maps.device_handle(), cascade, field,
                                              static_cast<float>(time), path.c_str()),
                  "write_heightfield_file");
}

std::vector<double> compose_height(const SurfaceMaps& maps, const std::vector<const FdmZone*>& zones,
                                   const std::vector<Vec2>& points) {
  std::vector<ocn_zone*> zh = zone_handles(zones);
  std::vector<double> xz(2 * points.size()), out(points.size());
  for (size_t i = 0; i < points.size(); ++i) xz[2 * i] = points[i].x, xz[2 * i + 1] = points[i].z;
  throw_on_status(ocn_compose_height(maps.device_handle(), static_cast<int>(zh.size()), zh.data(),
                                     static_cast<int64_t>(points.size()), xz.data(), out.data()),
                  "compose_height");
  return out;
}

void write_composed_heightfield_file(const std::string& path, const SurfaceMaps& maps,
                                     const std::vector<const FdmZone*>& zones, int resolution,
                                     double extent, double time) {
  std::vector<ocn_zone*> zh = zone_handles(zones);
  throw_on_status(ocn_heightfield_write_composed(maps.device_handle(), static_cast<int>(zh.size()),
                                                 zh.data(), resolution, extent,
                                                 static_cast<float>(time), path.c_str()),
                  "write_composed_heightfield_file");
}

}  // namespace ocean
