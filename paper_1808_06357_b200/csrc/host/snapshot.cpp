// Snapshot write/read (include/lattdse/snapshot.hpp). Data file and sidecar
// are both written under temporary names, then renamed data first, sidecar
// last; the sidecar carries the data file's FNV-1a checksum, so a crash
// between the two renames (new data, old sidecar) is detected on read
// instead of resuming stale state under new metadata.
#include "lattdse/snapshot.hpp"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "json_min.hpp"
#include "lattdse/errors.hpp"

namespace lattdse {
namespace {

constexpr const char* kFormat = "lattdse-snapshot-1";

std::string hex64(std::uint64_t v) {
  char b[24];
  std::snprintf(b, sizeof b, "0x%016llx", static_cast<unsigned long long>(v));
  return b;
}

bool little_endian() {
  const std::uint16_t one = 1;
  unsigned char c;
  std::memcpy(&c, &one, 1);
  return c == 1;
}

// FNV-1a 64 over the data bytes, in 8-byte words (the sidecar's data_fnv1a)
std::uint64_t data_checksum(const std::complex<double>* data, std::int64_t count) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(data);
  const std::int64_t nbytes = count * static_cast<std::int64_t>(sizeof(std::complex<double>));
  std::uint64_t h = 1469598103934665603ull;
  for (std::int64_t i = 0; i < nbytes; i += 8) {
    std::uint64_t w;
    std::memcpy(&w, p + i, 8);
    h = (h ^ w) * 1099511628211ull;
  }
  return h;
}

std::string read_text(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) raise(Errc::io_error, "cannot open snapshot sidecar " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

}  // namespace

void snapshot_write(const std::string& path, const Lattice& lat, const std::complex<double>* data,
                    const SnapshotMeta& meta) {
  if (!little_endian()) raise(Errc::unsupported, "snapshots are little-endian; big-endian host");
  if (meta.members < 1) raise(Errc::invalid_argument, "snapshot members must be >= 1");
  if (meta.space != 0 && meta.space != 1) raise(Errc::invalid_argument, "snapshot space must be 0 or 1");
  const std::int64_t n = lat.n_total();
  json::Value side = json::Value::object();
  side.obj["format"] = json::Value::string(kFormat);
  side.obj["length"] = json::Value::integer(n);
  side.obj["members"] = json::Value::integer(meta.members);
  side.obj["ordering"] = json::Value::string(meta.space == 0 ? "kappa" : "chi");
  side.obj["space"] = json::Value::string(meta.space == 0 ? "samples" : "coefficients");
  side.obj["lattice"] = json::parse(lat.to_json());
  side.obj["lattice_hash"] = json::Value::string(hex64(lat.hash()));
  side.obj["step"] = json::Value::integer(meta.step);
  side.obj["time"] = json::Value::number(meta.time);
  side.obj["dt"] = json::Value::number(meta.dt);
  side.obj["data_fnv1a"] = json::Value::string(hex64(data_checksum(data, n * meta.members)));

  const std::string tmp = path + ".tmp", side_tmp = path + ".json.tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) raise(Errc::io_error, "cannot create snapshot " + tmp);
    f.write(reinterpret_cast<const char*>(data),
            static_cast<std::streamsize>(sizeof(std::complex<double>) * n * meta.members));
    if (!f) raise(Errc::io_error, "short write to snapshot " + tmp);
  }
  {
    std::ofstream f(side_tmp, std::ios::trunc);
    if (!f) raise(Errc::io_error, "cannot create snapshot sidecar " + side_tmp);
    f << side.dump() << "\n";
    if (!f) raise(Errc::io_error, "short write to snapshot sidecar");
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) raise(Errc::io_error, "cannot rename " + tmp + " to " + path);
  const std::string side_path = path + ".json";
  if (std::rename(side_tmp.c_str(), side_path.c_str()) != 0)
    raise(Errc::io_error, "cannot rename " + side_tmp + " to " + side_path);
}

SnapshotMeta snapshot_probe(const std::string& path, const Lattice& lat) {
  json::Value side;
  try {
    side = json::parse(read_text(path + ".json"));
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    raise(Errc::io_error, std::string("malformed snapshot sidecar: ") + e.what());
  }
  if (!side.has("format") || side.at("format").s != kFormat)
    raise(Errc::io_error, "not a " + std::string(kFormat) + " sidecar: " + path + ".json");
  if (side.at("lattice_hash").s != hex64(lat.hash()))
    raise(Errc::config_error, "snapshot lattice hash " + side.at("lattice_hash").s + " != " + hex64(lat.hash()));
  if (side.at("length").as_int() != lat.n_total())
    raise(Errc::config_error, "snapshot length does not match the lattice");
  SnapshotMeta m;
  m.members = side.at("members").as_int();
  const std::string& sp = side.at("space").s;
  if (sp != "samples" && sp != "coefficients") raise(Errc::io_error, "snapshot space '" + sp + "' unknown");
  m.space = sp == "samples" ? 0 : 1;
  m.step = side.at("step").as_int();
  m.time = side.at("time").as_double();
  m.dt = side.at("dt").as_double();
  return m;
}

SnapshotMeta snapshot_read(const std::string& path, const Lattice& lat, std::complex<double>* data,
                           std::int64_t capacity) {
  SnapshotMeta m = snapshot_probe(path, lat);
  const std::int64_t count = lat.n_total() * m.members;
  if (capacity < count) raise(Errc::invalid_argument, "snapshot holds more values than the buffer");
  std::ifstream f(path, std::ios::binary);
  if (!f) raise(Errc::io_error, "cannot open snapshot " + path);
  f.read(reinterpret_cast<char*>(data), static_cast<std::streamsize>(sizeof(std::complex<double>) * count));
  if (f.gcount() != static_cast<std::streamsize>(sizeof(std::complex<double>) * count))
    raise(Errc::io_error, "snapshot " + path + " is truncated");
  json::Value side = json::parse(read_text(path + ".json"));
  if (side.has("data_fnv1a") && side.at("data_fnv1a").s != hex64(data_checksum(data, count)))
    raise(Errc::io_error, "snapshot " + path + " does not match its sidecar (data_fnv1a): interrupted write?");
  return m;
}

}  // namespace lattdse
