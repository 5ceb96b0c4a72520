// lattdse::Lattice -- fresh implementation of the reference API
// (/root/reference/proj/src/core/lattice.hpp:31-86). Validation order, error
// codes, limits (lcm <= 2^40, prod n <= 2^62, lcm*max|z| <= 2^62; reference
// lattice.cpp:16-17,202-214), point ordering, FNV-1a hash and JSON form
// follow the reference (lattice.cpp:167-364); the algorithms are our own:
// independence by modular elimination certified by an exact fraction-free
// pass, and the distinct-point count by a Hermite reduction of the generated
// subgroup of (Z_L)^d instead of the reference's Smith-style sweep.
#include "lattdse/lattice.hpp"

#include <algorithm>
#include <numeric>

#include "json_min.hpp"

namespace lattdse {

namespace {

using i128 = __int128;
using u64 = std::uint64_t;

constexpr i64 kDenomLimit = i64(1) << 40;
constexpr i64 kCountLimit = i64(1) << 62;

inline i64 modp(i128 v, i64 m) {
  i128 r = v % m;
  if (r < 0) r += m;
  return static_cast<i64>(r);
}

// Rank of the r x d matrix (rows = generator columns) modulo a prime p.
int rank_modp(const std::vector<std::vector<i64>>& rows, u64 p) {
  const size_t nr = rows.size(), nc = nr ? rows[0].size() : 0;
  std::vector<std::vector<u64>> m(nr, std::vector<u64>(nc));
  for (size_t i = 0; i < nr; ++i)
    for (size_t j = 0; j < nc; ++j) m[i][j] = static_cast<u64>(modp(rows[i][j], static_cast<i64>(p)));
  auto mulm = [p](u64 a, u64 b) { return static_cast<u64>((static_cast<unsigned __int128>(a) * b) % p); };
  auto inv = [&](u64 a) {
    u64 r = 1, e = p - 2;
    while (e) {
      if (e & 1) r = mulm(r, a);
      a = mulm(a, a);
      e >>= 1;
    }
    return r;
  };
  int rank = 0;
  for (size_t c = 0; c < nc && static_cast<size_t>(rank) < nr; ++c) {
    size_t piv = rank;
    while (piv < nr && m[piv][c] == 0) ++piv;
    if (piv == nr) continue;
    std::swap(m[piv], m[rank]);
    u64 iv = inv(m[rank][c]);
    for (size_t i = rank + 1; i < nr; ++i) {
      if (!m[i][c]) continue;
      u64 f = mulm(m[i][c], iv);
      for (size_t j = c; j < nc; ++j) m[i][j] = (m[i][j] + p - mulm(f, m[rank][j])) % p;
    }
    ++rank;
  }
  return rank;
}

// Exact rank by fraction-free elimination; nullopt if a 128-bit overflow
// would occur.
std::optional<int> rank_exact(const std::vector<std::vector<i64>>& rows) {
  const size_t nr = rows.size(), nc = nr ? rows[0].size() : 0;
  std::vector<std::vector<i128>> m(nr, std::vector<i128>(nc));
  for (size_t i = 0; i < nr; ++i)
    for (size_t j = 0; j < nc; ++j) m[i][j] = rows[i][j];
  i128 prev = 1;
  int rank = 0;
  for (size_t c = 0; c < nc && static_cast<size_t>(rank) < nr; ++c) {
    size_t piv = rank;
    while (piv < nr && m[piv][c] == 0) ++piv;
    if (piv == nr) continue;
    std::swap(m[piv], m[rank]);
    for (size_t i = rank + 1; i < nr; ++i) {
      for (size_t j = c + 1; j < nc; ++j) {
        i128 x, y, z;
        if (__builtin_mul_overflow(m[rank][c], m[i][j], &x)) return std::nullopt;
        if (__builtin_mul_overflow(m[i][c], m[rank][j], &y)) return std::nullopt;
        if (__builtin_sub_overflow(x, y, &z)) return std::nullopt;
        m[i][j] = z / prev;
      }
      m[i][c] = 0;
    }
    prev = m[rank][c];
    ++rank;
  }
  return rank;
}

bool independent_over_Q(const std::vector<std::vector<i64>>& cols) {
  const int r = static_cast<int>(cols.size());
  // A full rank modulo any prime certifies independence over Q.
  for (u64 p : {u64(2305843009213693951ULL), u64(4611686018427387847ULL), u64(1000000007ULL)})
    if (rank_modp(cols, p) == r) return true;
  // Deficient modulo all three primes: settle exactly when 128 bits suffice.
  if (auto e = rank_exact(cols)) return *e == r;
  return false;
}

// |<(L/n_i) z_i>| in (Z_L)^d: Hermite-reduce the lattice spanned by the
// scaled generators together with L*Z^d, row by row modulo L. The lattice
// determinant is prod g_t, so the subgroup order is prod (L / g_t).
i64 subgroup_order(const std::vector<std::vector<i64>>& cols, const std::vector<i64>& scale, i64 L, int d) {
  const int r = static_cast<int>(cols.size());
  std::vector<std::vector<i64>> v(r, std::vector<i64>(d));
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < d; ++j) v[i][j] = modp(static_cast<i128>(scale[i]) * cols[i][j], L);
  auto egcd = [](i64 a, i64 b, i64& x, i64& y) {
    i64 x0 = 1, y0 = 0, x1 = 0, y1 = 1;
    while (b != 0) {
      i64 q = a / b, t = a - q * b;
      a = b;
      b = t;
      t = x0 - q * x1; x0 = x1; x1 = t;
      t = y0 - q * y1; y0 = y1; y1 = t;
    }
    x = x0;
    y = y0;
    return a;
  };
  i64 count = 1;
  for (int t = 0; t < d; ++t) {
    // pivot starts as the implicit column L*e_t
    std::vector<i64> pv(d, 0);
    i64 g = L;
    for (int i = 0; i < r; ++i) {
      i64 a = v[i][t];
      if (a == 0) continue;
      i64 x, y;
      i64 h = egcd(g, a, x, y);  // x*g + y*a = h
      const i64 ga = g / h, aa = a / h;
      for (int j = t + 1; j < d; ++j) {
        i64 p_j = pv[j], c_j = v[i][j];
        pv[j] = modp(static_cast<i128>(x) * p_j + static_cast<i128>(y) * c_j, L);
        v[i][j] = modp(static_cast<i128>(aa) * p_j - static_cast<i128>(ga) * c_j, L);
      }
      v[i][t] = 0;
      g = h;
    }
    count *= L / g;
  }
  return count;
}

u64 fnv1a_i64(u64 h, i64 v) {
  const u64 x = static_cast<u64>(v);
  for (int byte = 0; byte < 8; ++byte) {
    h ^= (x >> (8 * byte)) & 0xffu;
    h *= 1099511628211ULL;
  }
  return h;
}

}  // namespace

std::vector<double> LatticePoint::coords() const {
  std::vector<double> out;
  out.reserve(num.size());
  for (i64 a : num) out.push_back(static_cast<double>(a) / static_cast<double>(denom));
  return out;
}

Lattice Lattice::create(int dim, int rank, std::vector<std::vector<i64>> gen, std::vector<i64> moduli) {
  if (dim < 1 || rank < 1 || rank > dim) raise(Errc::invalid_argument, "lattice requires 1 <= rank <= dim");
  if (static_cast<int>(gen.size()) != rank || static_cast<int>(moduli.size()) != rank)
    raise(Errc::invalid_argument, "generator must have rank columns and rank moduli");
  for (const auto& col : gen)
    if (static_cast<int>(col.size()) != dim) raise(Errc::invalid_argument, "generator column length must equal dim");
  if (std::any_of(moduli.begin(), moduli.end(), [](i64 n) { return n < 1; }))
    raise(Errc::invalid_argument, "moduli must be >= 1");

  for (int i = 1; i < rank; ++i)
    if (moduli[i - 1] % moduli[i] != 0)
      raise(Errc::non_divisible_moduli,
            "modulus " + std::to_string(moduli[i]) + " does not divide " + std::to_string(moduli[i - 1]));

  for (int i = 0; i < rank; ++i)
    for (int j = 0; j < dim; ++j) {
      const i64 c = modp(gen[i][j], moduli[i]);
      if (c != 0 && std::gcd(c, moduli[i]) != 1)
        raise(Errc::non_coprime_component, "generator column " + std::to_string(i) + ", coordinate " +
                                               std::to_string(j) + ": component " + std::to_string(gen[i][j]) +
                                               " is not coprime to modulus " + std::to_string(moduli[i]));
    }

  if (!independent_over_Q(gen)) raise(Errc::rank_deficient, "generator columns are linearly dependent over Q");

  // exact-integer range guards
  i64 L = 1, total = 1, zmax = 1;
  for (int i = 0; i < rank; ++i) {
    const i64 n = moduli[i];
    const i64 step = L / std::gcd(L, n);
    if (step > kDenomLimit / n) raise(Errc::overflow_risk, "lcm of the moduli exceeds 2^40");
    L = step * n;
    if (total > kCountLimit / n) raise(Errc::overflow_risk, "number of points exceeds 2^62");
    total *= n;
    for (i64 z : gen[i]) zmax = std::max(zmax, z < 0 ? -z : z);
  }
  if (zmax > kCountLimit / L) raise(Errc::overflow_risk, "lcm(moduli) * max|z| exceeds 2^62");

  Lattice lat;
  lat.dim_ = dim;
  lat.rank_ = rank;
  lat.gen_ = std::move(gen);
  lat.moduli_ = std::move(moduli);
  lat.denom_ = L;
  lat.n_total_ = total;
  lat.col_scale_.resize(rank);
  lat.flat_weights_.assign(rank, 1);
  for (int i = 0; i < rank; ++i) lat.col_scale_[i] = L / lat.moduli_[i];
  for (int i = rank - 2; i >= 0; --i) lat.flat_weights_[i] = lat.flat_weights_[i + 1] * lat.moduli_[i + 1];

  const i64 distinct = subgroup_order(lat.gen_, lat.col_scale_, L, dim);
  if (distinct != total)
    raise(Errc::point_count_mismatch,
          "generators give " + std::to_string(distinct) + " distinct points, expected " + std::to_string(total));

  u64 h = 14695981039346656037ULL;
  h = fnv1a_i64(h, dim);
  h = fnv1a_i64(h, rank);
  for (i64 n : lat.moduli_) h = fnv1a_i64(h, n);
  for (const auto& col : lat.gen_)
    for (i64 z : col) h = fnv1a_i64(h, z);
  lat.hash_ = h;
  return lat;
}

Lattice Lattice::rank1(std::vector<i64> z, i64 n) {
  const int d = static_cast<int>(z.size());
  std::vector<std::vector<i64>> gen;
  gen.push_back(std::move(z));
  return create(d, 1, std::move(gen), {n});
}

Lattice Lattice::grid(std::vector<i64> moduli) {
  const int d = static_cast<int>(moduli.size());
  std::vector<std::vector<i64>> gen(d, std::vector<i64>(d, 0));
  for (int i = 0; i < d; ++i) gen[i][i] = 1;
  return create(d, d, std::move(gen), std::move(moduli));
}

bool Lattice::in_dual(std::span<const i64> h) const {
  if (static_cast<int>(h.size()) != dim_) raise(Errc::invalid_argument, "in_dual: dimension mismatch");
  for (int i = 0; i < rank_; ++i) {
    i128 dot = 0;
    for (int j = 0; j < dim_; ++j) dot += static_cast<i128>(gen_[i][j]) * h[j];
    if (modp(dot, moduli_[i]) != 0) return false;
  }
  return true;
}

std::vector<i64> Lattice::residue(std::span<const i64> h) const {
  if (static_cast<int>(h.size()) != dim_) raise(Errc::invalid_argument, "residue: dimension mismatch");
  std::vector<i64> xi(rank_);
  for (int i = 0; i < rank_; ++i) {
    i128 dot = 0;
    for (int j = 0; j < dim_; ++j) dot += static_cast<i128>(gen_[i][j]) * h[j];
    xi[i] = modp(dot, moduli_[i]);
  }
  return xi;
}

i64 Lattice::flat_residue(std::span<const i64> h) const {
  if (static_cast<int>(h.size()) != dim_) raise(Errc::invalid_argument, "flat_residue: dimension mismatch");
  i64 flat = 0;
  const auto xi = residue(h);
  for (int i = 0; i < rank_; ++i) flat += xi[i] * flat_weights_[i];
  return flat;
}

std::vector<std::vector<i64>> Lattice::numerator_steps() const {
  std::vector<std::vector<i64>> step(rank_, std::vector<i64>(dim_));
  for (int i = 0; i < rank_; ++i)
    for (int j = 0; j < dim_; ++j) step[i][j] = modp(static_cast<i128>(col_scale_[i]) * gen_[i][j], denom_);
  return step;
}

LatticePoint Lattice::point(i64 flat_index) const {
  if (flat_index < 0 || flat_index >= n_total_) raise(Errc::invalid_argument, "point index out of range");
  LatticePoint p;
  p.denom = denom_;
  p.flat_index = flat_index;
  p.index.assign(rank_, 0);
  for (int i = 0; i < rank_; ++i) p.index[i] = (flat_index / flat_weights_[i]) % moduli_[i];
  const auto step = numerator_steps();
  p.num.assign(dim_, 0);
  for (int j = 0; j < dim_; ++j) {
    i128 acc = 0;
    for (int i = 0; i < rank_; ++i) acc += static_cast<i128>(step[i][j]) * p.index[i];
    p.num[j] = modp(acc, denom_);
  }
  return p;
}

std::vector<LatticePoint> Lattice::enumerate_points() const {
  std::vector<LatticePoint> pts;
  pts.reserve(static_cast<size_t>(n_total_));
  for (i64 k = 0; k < n_total_; ++k) pts.push_back(point(k));
  return pts;
}

std::vector<i64> Lattice::point_numerators() const {
  std::vector<i64> out(static_cast<size_t>(n_total_) * dim_);
  const auto step = numerator_steps();
  // Odometer over the multi-index k (last coordinate fastest); the running
  // numerator vector is updated by one column step per increment.
  std::vector<i64> k(rank_, 0), cur(dim_, 0);
  for (i64 kappa = 0; kappa < n_total_; ++kappa) {
    std::copy(cur.begin(), cur.end(), out.begin() + kappa * dim_);
    for (int i = rank_ - 1; i >= 0; --i) {
      if (++k[i] < moduli_[i]) {
        for (int j = 0; j < dim_; ++j) {
          i64 x = cur[j] + step[i][j];
          cur[j] = x >= denom_ ? x - denom_ : x;
        }
        break;
      }
      k[i] = 0;  // wrap: remove (n_i - 1) steps of column i
      for (int j = 0; j < dim_; ++j)
        cur[j] = modp(static_cast<i128>(cur[j]) - static_cast<i128>(step[i][j]) * (moduli_[i] - 1), denom_);
    }
  }
  return out;
}

std::vector<double> Lattice::point_coords() const {
  const auto num = point_numerators();
  std::vector<double> out(num.size());
  const double inv = 1.0 / static_cast<double>(denom_);
  for (size_t i = 0; i < num.size(); ++i) out[i] = static_cast<double>(num[i]) * inv;
  return out;
}

std::string Lattice::to_json() const {
  json::Value o = json::Value::object();
  json::Value Z = json::Value::array();
  for (const auto& col : gen_) {
    json::Value c = json::Value::array();
    for (i64 z : col) c.arr.push_back(json::Value::integer(z));
    Z.arr.push_back(std::move(c));
  }
  json::Value n = json::Value::array();
  for (i64 m : moduli_) n.arr.push_back(json::Value::integer(m));
  o.obj["Z"] = std::move(Z);
  o.obj["d"] = json::Value::integer(dim_);
  o.obj["n"] = std::move(n);
  o.obj["r"] = json::Value::integer(rank_);
  return o.dump();
}

Lattice Lattice::from_json(const std::string& text) {
  json::Value j;
  try {
    j = json::parse(text);
  } catch (const std::exception& e) {
    raise(Errc::io_error, std::string("lattice JSON parse failure: ") + e.what());
  }
  if (!j.has("d") || !j.has("r") || !j.has("Z") || !j.has("n"))
    raise(Errc::io_error, "lattice JSON requires fields d, r, Z, n");
  int d = 0, r = 0;
  std::vector<std::vector<i64>> Z;
  std::vector<i64> n;
  try {
    d = static_cast<int>(j.at("d").as_int());
    r = static_cast<int>(j.at("r").as_int());
    const auto& zj = j.at("Z");
    if (zj.kind != json::Value::Array) throw std::runtime_error("Z must be an array");
    for (const auto& col : zj.arr) {
      if (col.kind != json::Value::Array) throw std::runtime_error("Z columns must be arrays");
      std::vector<i64> c;
      for (const auto& x : col.arr) c.push_back(x.as_int());
      Z.push_back(std::move(c));
    }
    const auto& nj = j.at("n");
    if (nj.kind != json::Value::Array) throw std::runtime_error("n must be an array");
    for (const auto& x : nj.arr) n.push_back(x.as_int());
  } catch (const std::exception& e) {
    raise(Errc::io_error, std::string("lattice JSON field types: ") + e.what());
  }
  return create(d, r, std::move(Z), std::move(n));
}

}  // namespace lattdse
