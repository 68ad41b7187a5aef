// tests/ref_unit/detail_shim.cpp — see detail_shim.hpp. Test infrastructure only.
#include "detail_shim.hpp"

#include <stdexcept>

namespace bml::detail {

namespace {
Grid device_phase(const Grid& cur, Phase phase) {
    GridPair pair{cur, Grid::with_halo(cur.n())};
    if (!cur.has_halo()) pair = GridPair{cur.to_halo(), Grid::with_halo(cur.n())};
    step_phase(Backend::B200, pair, phase, 1);
    return pair.cur;
}
}  // namespace

void halo_phase_rows(const Grid& cur, Grid& next, Phase phase, int row_begin, int row_end) {
    if (next.n() != cur.n()) throw std::invalid_argument("halo_phase_rows: size mismatch");
    const Grid out = device_phase(cur, phase);
    for (int r = row_begin - 1; r < row_end; ++r)
        for (int c = 0; c < cur.n(); ++c) next.interior(r, c) = out.interior(r, c);
}

void swar_phase(const Grid& cur, Grid& next, Phase phase) { halo_phase_rows(cur, next, phase, 1, cur.n()); }

}  // namespace bml::detail
