// State snapshots (SURVEY.md §5 checkpoint/resume): the
// wave function as raw little-endian interleaved complex128 in `path`, and a
// JSON sidecar `path + ".json"` carrying what is needed to resume safely:
//   {"format":"lattdse-snapshot-1","length":L,"members":B,"ordering":"kappa"|"chi",
//    "space":"samples"|"coefficients","lattice":{...},"lattice_hash":"0x...",
//    "step":k,"time":t,"dt":dt}
// Reading checks the sidecar against the caller's lattice (hash and length)
// and raises config_error on a mismatch, io_error on missing/short files.
#pragma once

#include <complex>
#include <cstdint>
#include <string>

#include "lattice.hpp"

namespace lattdse {

struct SnapshotMeta {
  std::int64_t members = 1;
  int space = 0;  // 0 = samples (kappa order), 1 = coefficients (chi order)
  std::int64_t step = 0;
  double time = 0.0;
  double dt = 0.0;
};

void snapshot_write(const std::string& path, const Lattice& lat, const std::complex<double>* data,
                    const SnapshotMeta& meta);

/// Reads the sidecar only (no data) after checking it against `lat`.
SnapshotMeta snapshot_probe(const std::string& path, const Lattice& lat);

/// Reads members*N values into `data` (capacity `capacity` complex values).
SnapshotMeta snapshot_read(const std::string& path, const Lattice& lat, std::complex<double>* data,
                           std::int64_t capacity);

}  // namespace lattdse
