// Host complex FFT of any length, used only for setup (the fast CBC
// construction's length n-1 cyclic correlation). Never on the time-stepping
// path, which is CUDA only.
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace lattdse::hostfft {

using cd = std::complex<double>;

/// In-place unnormalised DFT, sign -1 (forward) or +1 (inverse), any length.
void dft(std::vector<cd>& x, int sign);

/// Smallest 5-smooth integer >= n.
std::int64_t next_smooth(std::int64_t n);

}  // namespace lattdse::hostfft
