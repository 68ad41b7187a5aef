// Initial lattice generation, bit-identical to /root/reference/proj/src/seeding.cpp
// (bounded :11-19, vehicles_per_species :21-24, init_grid :26-51). Host-side
// input generation, outside the stepped hot path. Uses 32-bit indices when
// n^2 <= 2^32 (all n <= 65536), halving the shuffle's memory (16 GiB instead
// of 32 GiB at n = 65536) without changing the permutation.
#include "bml/seeding.hpp"

#include <cmath>
#include <numeric>
#include <stdexcept>
#include <utility>
#include <vector>

namespace bml {

std::uint64_t bounded(SplitMix64& rng, std::uint64_t m) {
    if (m == 0) throw std::invalid_argument("bounded: m must be >= 1");
    // accept r < 2^64 - (2^64 mod m): the largest multiple of m
    const std::uint64_t excess = (0 - m) % m;  // == 2^64 mod m
    for (;;) {
        const std::uint64_t r = rng.next();
        if (excess == 0 || r < 0 - excess) return r % m;
    }
}

std::int64_t vehicles_per_species(int n, double rho) {
    const double nn = static_cast<double>(n);
    return static_cast<std::int64_t>(std::floor(rho * nn * nn / 2.0));
}

namespace {

template <typename Index>
void place(const SeedSpec& spec, Grid& g) {
    const std::uint64_t cells = static_cast<std::uint64_t>(spec.n) * spec.n;
    std::vector<Index> perm(cells);
    std::iota(perm.begin(), perm.end(), Index{0});
    SplitMix64 rng(spec.seed);
    for (std::uint64_t i = cells - 1; i > 0; --i) {
        const std::uint64_t j = bounded(rng, i + 1);
        std::swap(perm[i], perm[j]);
    }
    const std::int64_t k = vehicles_per_species(spec.n, spec.rho);
    for (std::int64_t i = 0; i < 2 * k; ++i) {
        const std::uint64_t c = perm[static_cast<std::size_t>(i)];
        g.interior(static_cast<int>(c / spec.n), static_cast<int>(c % spec.n)) =
            i < k ? Cell::LR : Cell::TB;
    }
}

}  // namespace

Grid init_grid(const SeedSpec& spec) {
    if (spec.n < 1) throw std::invalid_argument("init_grid: n must be >= 1");
    if (!(spec.rho >= 0.0 && spec.rho <= 1.0))
        throw std::invalid_argument("init_grid: density must be in [0, 1]");
    Grid g = Grid::with_halo(spec.n);
    const std::uint64_t cells = static_cast<std::uint64_t>(spec.n) * spec.n;
    if (cells <= (std::uint64_t{1} << 32))
        place<std::uint32_t>(spec, g);
    else
        place<std::uint64_t>(spec, g);
    return g;
}

}  // namespace bml
