// tests/ref_unit/detail_shim.hpp — test adapter, force-included (-include) only
// when compiling the reference's test_engine.cpp. That file calls two internal
// CPU kernels of the reference engine (proj/include/bml/engine.hpp:81-91,
// bml::detail::halo_phase_rows and swar_phase) which this library does not
// have. Both are implemented in detail_shim.cpp on the public step_phase (the
// device engine), so test_engine.cpp's other 16 cases can run; the one case
// comparing those two kernels against each other is vacuous here.
#pragma once

#include "bml/engine.hpp"
#include "bml/grid.hpp"

namespace bml::detail {
// rows are interior indices, 1-based, inclusive (reference engine.hpp:82-84)
void halo_phase_rows(const Grid& cur, Grid& next, Phase phase, int row_begin, int row_end);
void swar_phase(const Grid& cur, Grid& next, Phase phase);
}  // namespace bml::detail
