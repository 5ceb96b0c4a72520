// Error model of the lattdse API.
//
// Mirrors the reference's lattdse::Errc / lattdse::Error / raise()
// (/root/reference/proj/src/core/errors.hpp:8-34): the first 13 codes keep the
// reference's names and ordinals so the C ABI can map them 1:1
// (C return code = ordinal + 1). Codes for the device path are appended after
// io_error and are never renumbered.
#pragma once

#include <stdexcept>
#include <string>

namespace lattdse {

enum class Errc : int {
  invalid_argument = 0,
  non_divisible_moduli,
  non_coprime_component,
  rank_deficient,
  point_count_mismatch,
  overflow_risk,
  radius_exhausted,
  spec_mismatch,
  non_normalizable,
  config_error,
  reference_too_coarse,
  numerical_invariant,
  io_error,
  // ---- appended for the B200 path (not in the reference) ----
  device_error,       // CUDA runtime / kernel failure
  unsupported,        // valid input the device path has no kernel for
  nccl_error,         // collective failure (multi-GPU paths)
};

inline const char* errc_name(Errc c) {
  switch (c) {
    case Errc::invalid_argument: return "invalid_argument";
    case Errc::non_divisible_moduli: return "non_divisible_moduli";
    case Errc::non_coprime_component: return "non_coprime_component";
    case Errc::rank_deficient: return "rank_deficient";
    case Errc::point_count_mismatch: return "point_count_mismatch";
    case Errc::overflow_risk: return "overflow_risk";
    case Errc::radius_exhausted: return "radius_exhausted";
    case Errc::spec_mismatch: return "spec_mismatch";
    case Errc::non_normalizable: return "non_normalizable";
    case Errc::config_error: return "config_error";
    case Errc::reference_too_coarse: return "reference_too_coarse";
    case Errc::numerical_invariant: return "numerical_invariant";
    case Errc::io_error: return "io_error";
    case Errc::device_error: return "device_error";
    case Errc::unsupported: return "unsupported";
    case Errc::nccl_error: return "nccl_error";
  }
  return "unknown";
}

/// Exception carrying a machine-readable code next to the message.
class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

[[noreturn]] inline void raise(Errc code, const std::string& what) { throw Error(code, what); }

}  // namespace lattdse
