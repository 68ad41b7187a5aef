// Cross-configuration verification of the device engine; see bml/verify.hpp.
// Mirrors /root/reference/proj/src/verify.cpp:11-43 (one initial lattice, per-step
// conservation, cell-for-cell comparison of the finals, one digest per run).
#include "bml/verify.hpp"

#include <algorithm>
#include <stdexcept>

#include "bml/digest.hpp"
#include "bml/metrics.hpp"
#include "bml/seeding.hpp"

namespace bml {

std::optional<GridMismatch> first_mismatch(const std::vector<NamedGrid>& grids) {
    for (std::size_t i = 1; i < grids.size(); ++i) {
        if (const auto diff = first_interior_mismatch(grids[0].grid, grids[i].grid))
            return GridMismatch{grids[0].name, grids[i].name, diff->first, diff->second};
    }
    return std::nullopt;
}

namespace {

// Row bands for the banded path: the largest g <= 4 whose ceil(n/g) split
// (engine.cpp:131-137) leaves every band >= 16 rows (the ghost depth), else 1.
int verify_bands(int n) {
    for (int g = 4; g >= 2; --g) {
        const int band = (n + g - 1) / g;
        if (n - (g - 1) * band >= 16) return g;
    }
    return 1;
}

bool conserved_run(DeviceLattice& lat, long steps, const VehicleCounts& initial) {
    lat.set_census(true);  // the reference's per-step check, exactly (verify.cpp:27-30)
    try {
        const auto metrics = lat.step_with_metrics(steps);
        for (const StepMetrics& m : metrics)
            if (m.lr_count != initial.lr || m.tb_count != initial.tb) return false;
    } catch (const std::logic_error&) {
        return false;
    }
    return true;
}

}  // namespace

namespace {

const char* const kDevicePaths[] = {"b200", "b200-streaming", "b200-even-odd", "b200-phases", "b200-bands"};

// One device path from `initial`: the final grid and its digest go into the
// report, a census difference clears report.conserved.
void run_device_path(const std::string& name, const SimConfig& cfg, const Grid& initial,
                     const VehicleCounts& start, VerifyReport& report, std::vector<NamedGrid>& finals) {
    auto record = [&](DeviceLattice& lat) {
        report.digests.push_back(PathDigest{name, lat.digest()});
        finals.push_back(NamedGrid{name, lat.download()});
    };
    if (name == "b200-phases") {  // single-phase kernels, one phase per launch (step_phase)
        DeviceLattice lat(cfg.n);
        lat.upload(initial);
        for (long s = 0; s < cfg.steps; ++s) {
            lat.phase(Phase::Horizontal);
            lat.phase(Phase::Vertical);
            const VehicleCounts c = lat.counts();
            if (c.lr != start.lr || c.tb != start.tb) report.conserved = false;
        }
        record(lat);
        return;
    }
    if (name == "b200-bands") {  // row bands with in-kernel ghost-row exchange (block depth 1 when too small)
        const int bands = verify_bands(cfg.n);
        DeviceLattice lat(cfg.n, bands);
        if (bands == 1) lat.configure(1, 0);
        lat.upload(initial);
        if (!conserved_run(lat, cfg.steps, start)) report.conserved = false;
        record(lat);
        return;
    }
    DeviceLattice lat(cfg.n);
    if (name == "b200-streaming") {  // narrow streaming temporally blocked kernel only
        lat.set_resident(0);
        lat.set_variant(1);
    } else if (name == "b200-even-odd") {  // even/odd-layout streaming kernel
        lat.set_resident(0);
        lat.set_variant(6);
    } else if (name != "b200") {  // default path: resident cluster kernel when the lattice qualifies
        throw std::invalid_argument("verify_device: unknown path '" + name + "'");
    }
    lat.upload(initial);
    if (!conserved_run(lat, cfg.steps, start)) report.conserved = false;
    record(lat);
}

VerifyReport verify_paths(const SimConfig& cfg, const std::vector<std::string>& paths) {
    validate(cfg);
    for (const std::string& p : paths)
        if (std::find(std::begin(kDevicePaths), std::end(kDevicePaths), p) == std::end(kDevicePaths))
            throw std::invalid_argument("verify_device: unknown path '" + p + "'");
    const Grid initial = init_grid({cfg.n, cfg.rho, cfg.seed});
    const VehicleCounts start = count_vehicles(initial);
    VerifyReport report;
    std::vector<NamedGrid> finals;
    for (const std::string& p : paths) run_device_path(p, cfg, initial, start, report, finals);
    report.mismatch = first_mismatch(finals);
    return report;
}

}  // namespace

// The reference's four slots (verify.cpp:19-42), filled with four device paths.
VerifyReport verify_backends(const SimConfig& cfg) {
    return verify_paths(cfg, {"b200", "b200-streaming", "b200-phases", "b200-bands"});
}

VerifyReport verify_device(const SimConfig& cfg, const std::vector<std::string>& paths) {
    if (!paths.empty()) return verify_paths(cfg, paths);
    return verify_paths(cfg, std::vector<std::string>(std::begin(kDevicePaths), std::end(kDevicePaths)));
}

}  // namespace bml
