// Device builder of the anti-aliasing norm table (aaset_dev.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lattdse/lattice.hpp"

namespace lattdse::dev {

/// Fills table[chi] (N uint16 on the current device, enqueued on `st`) with
/// min ||h||^2 over z.h == chi (mod N) for a rank-1 lattice; returns the
/// largest entry. cap_radius <= 0: SPEC's default 4 N^(1/d) + 16.
std::uint32_t aaset_norms_device(const Lattice& lat, unsigned short* table, cudaStream_t st, double cap_radius = -1.0);

}  // namespace lattdse::dev
