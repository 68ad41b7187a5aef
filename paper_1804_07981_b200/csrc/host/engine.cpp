// Engine front end for the b200 backend. Keeps the reference's validation and
// error behaviour (/root/reference/proj/src/engine.cpp:45-64 validate /
// make_grid_pair, :148-179 step_phase checks, :201-237 run) and routes all
// stepping through the C-ABI (include/bml_dev.h). There is no CPU stepping
// code in this library.
#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "bml/engine.hpp"
#include "bml/metrics.hpp"
#include "bml/seeding.hpp"
#include "bml/snapshot.hpp"
#include "bml_dev.h"

namespace bml {

namespace {

[[noreturn]] void raise(int rc, const std::string& what) {
    const std::string msg = what + ": " + bml_dev_last_error();
    if (rc == BML_EINVAL) throw std::invalid_argument(msg);
    if (rc == BML_ECONSERVE) throw std::logic_error(msg);
    throw std::runtime_error(msg);  // BML_ECUDA, BML_ENOMEM
}

inline void ok(int rc, const char* what) {
    if (rc != BML_OK) raise(rc, what);
}

}  // namespace

std::string_view backend_name(Backend b) {
    switch (b) {
        case Backend::ScalarNaive: return "naive";
        case Backend::ScalarHalo: return "halo";
        case Backend::ParallelRows: return "parallel";
        case Backend::Lanes: return "lanes";
        case Backend::B200: return "b200";
    }
    return "?";
}

std::optional<Backend> backend_from_name(std::string_view name) {
    for (Backend b : {Backend::ScalarNaive, Backend::ScalarHalo, Backend::ParallelRows,
                      Backend::Lanes, Backend::B200})
        if (backend_name(b) == name) return b;
    return std::nullopt;
}

int lane_width() { return 32; }

void validate(const SimConfig& cfg) {
    if (cfg.n < 1) throw std::invalid_argument("config: n must be >= 1");
    if (!(cfg.rho >= 0.0 && cfg.rho <= 1.0))
        throw std::invalid_argument("config: density must be in [0, 1]");
    if (cfg.steps < 0) throw std::invalid_argument("config: steps must be >= 0");
    if (cfg.threads < 1) throw std::invalid_argument("config: threads must be >= 1");
    if (cfg.snapshot_every < 0)
        throw std::invalid_argument("config: snapshot cadence must be >= 0");
    if (cfg.threads > 1 && cfg.backend != Backend::ParallelRows)
        throw std::invalid_argument("config: backend '" + std::string(backend_name(cfg.backend)) +
                                    "' does not support threads > 1");
    if (cfg.devices < 1) throw std::invalid_argument("config: devices must be >= 1");
    if (cfg.devices > 1 && cfg.backend != Backend::B200)
        throw std::invalid_argument("config: devices > 1 requires backend 'b200'");
}

GridPair make_grid_pair(Backend backend, const Grid& initial) {
    if (backend == Backend::ScalarNaive)
        return GridPair{initial.to_dense(), Grid::dense(initial.n())};
    return GridPair{initial.to_halo(), Grid::with_halo(initial.n())};
}

// ------------------------------------------------------------ DeviceLattice
DeviceLattice::DeviceLattice(int n, int devices) : n_(n) {
    if (n < 1) throw std::invalid_argument("DeviceLattice: n must be >= 1");
    if (devices < 1) throw std::invalid_argument("DeviceLattice: devices must be >= 1");
    if (devices == 1) {
        bml_dev* h = nullptr;
        ok(bml_dev_create(n, -1, &h), "bml_dev_create");
        bands_.push_back(h);
        return;
    }
    int gpus = 0;
    ok(bml_dev_device_count(&gpus), "bml_dev_device_count");
    if (gpus < 1) throw std::runtime_error("DeviceLattice: no CUDA device visible");
    const int band = (n + devices - 1) / devices;  // parallel_rows_phase's split, engine.cpp:131-137
    if (n - (devices - 1) * band < 16)
        throw std::invalid_argument("DeviceLattice: every row band needs >= 16 rows (n=" +
                                    std::to_string(n) + ", devices=" + std::to_string(devices) + ")");
    try {
        for (int g = 0; g < devices; ++g) {
            bml_dev* h = nullptr;
            const int r0 = g * band, r1 = std::min(n, r0 + band);
            ok(bml_dev_create_band(n, r0, r1, g % gpus, &h), "bml_dev_create_band");
            bands_.push_back(h);
        }
        for (int g = 0; g < devices; ++g)
            ok(bml_dev_connect_local(bands_[g], bands_[(g + devices - 1) % devices],
                                     bands_[(g + 1) % devices]),
               "bml_dev_connect_local");
    } catch (...) {
        for (bml_dev* h : bands_) bml_dev_destroy(h);
        bands_.clear();
        throw;
    }
}

DeviceLattice::~DeviceLattice() {
    for (bml_dev* h : bands_) bml_dev_destroy(h);
}

void DeviceLattice::upload(const Grid& g) {
    if (g.n() != n_) throw std::invalid_argument("DeviceLattice::upload: grid size mismatch");
    for (bml_dev* h : bands_) {
        int r0 = 0;
        ok(bml_dev_info(h, nullptr, &r0, nullptr, nullptr, nullptr, nullptr), "bml_dev_info");
        const auto* src = reinterpret_cast<const std::uint8_t*>(g.interior_data()) +
                          static_cast<std::size_t>(r0) * g.stride();
        ok(bml_dev_upload(h, src, static_cast<std::size_t>(g.stride())), "bml_dev_upload");
    }
    if (bands_.size() > 1)
        for (bml_dev* h : bands_) ok(bml_dev_exchange_halos(h), "bml_dev_exchange_halos");
}

void DeviceLattice::init_random(double rho, std::uint64_t seed) {
    for (bml_dev* h : bands_) ok(bml_dev_init_random(h, rho, seed), "bml_dev_init_random");
    if (bands_.size() > 1)
        for (bml_dev* h : bands_) ok(bml_dev_exchange_halos(h), "bml_dev_exchange_halos");
}

Grid init_grid_device(const SeedSpec& spec) {
    if (spec.n < 1) throw std::invalid_argument("init_grid: n must be >= 1");
    if (!(spec.rho >= 0.0 && spec.rho <= 1.0))
        throw std::invalid_argument("init_grid: density must be in [0, 1]");
    DeviceLattice lat(spec.n);
    lat.init_random(spec.rho, spec.seed);
    return lat.download();
}

std::vector<std::uint8_t> DeviceLattice::encode_ppm() const {
    const std::string header = ppm_header(n_);
    std::vector<std::uint8_t> out(header.size() + 3u * static_cast<std::size_t>(n_) * n_);
    std::copy(header.begin(), header.end(), out.begin());
    for (bml_dev* h : bands_) {
        int r0 = 0;
        ok(bml_dev_info(h, nullptr, &r0, nullptr, nullptr, nullptr, nullptr), "bml_dev_info");
        ok(bml_dev_encode_ppm(h, out.data() + header.size() + 3u * static_cast<std::size_t>(r0) * n_,
                              3u * static_cast<std::size_t>(n_)),
           "bml_dev_encode_ppm");
    }
    return out;
}

std::uint64_t DeviceLattice::digest() const {
    std::vector<std::uint64_t> segs(6 * bands_.size());
    for (std::size_t b = 0; b < bands_.size(); ++b)
        ok(bml_dev_digest_segment(bands_[b], segs.data() + 6 * b), "bml_dev_digest_segment");
    std::uint64_t h = 0;
    ok(bml_digest_finish(segs.data(), static_cast<int>(bands_.size()), &h), "bml_digest_finish");
    return h;
}

void DeviceLattice::download(Grid& g) const {
    if (g.n() != n_) throw std::invalid_argument("DeviceLattice::download: grid size mismatch");
    for (bml_dev* h : bands_) {
        int r0 = 0;
        ok(bml_dev_info(h, nullptr, &r0, nullptr, nullptr, nullptr, nullptr), "bml_dev_info");
        auto* dst = reinterpret_cast<std::uint8_t*>(g.interior_data()) +
                    static_cast<std::size_t>(r0) * g.stride();
        ok(bml_dev_download(h, dst, static_cast<std::size_t>(g.stride())), "bml_dev_download");
    }
}

Grid DeviceLattice::download() const {
    Grid g = Grid::with_halo(n_);
    download(g);
    return g;
}

namespace {
int block_for(long remaining, int cap) {
    int k = 16;
    while (k > 1 && (k > remaining || k > cap)) k >>= 1;
    return k;
}
}  // namespace

void DeviceLattice::step(long steps) {
    if (steps < 0) throw std::invalid_argument("step: steps must be >= 0");
    if (bands_.size() == 1) {
        ok(bml_dev_step(bands_[0], steps, nullptr, nullptr, nullptr, nullptr), "bml_dev_step");
        return;
    }
    // lockstep: one launch per band per block, all asynchronous
    for (long done = 0; done < steps;) {
        const int k = block_for(steps - done, block_steps_);
        for (bml_dev* h : bands_)
            ok(bml_dev_step(h, k, nullptr, nullptr, nullptr, nullptr), "bml_dev_step");
        done += k;
    }
}

void DeviceLattice::set_census(bool every_step) {
    for (bml_dev* h : bands_) ok(bml_dev_set_census(h, every_step ? 1 : 0), "bml_dev_set_census");
}

void DeviceLattice::debug_fault(long at_step, int row, int col) {
    if (bands_.size() != 1) throw std::invalid_argument("debug_fault: single-band lattices only");
    ok(bml_dev_debug_fault(bands_[0], at_step, row, col), "bml_dev_debug_fault");
}

std::vector<StepMetrics> DeviceLattice::step_with_metrics(long steps, long first_step,
                                                          bool throw_on_violation) {
    if (steps < 0) throw std::invalid_argument("step: steps must be >= 0");
    std::vector<StepMetrics> out(static_cast<std::size_t>(steps));
    if (steps == 0) return out;
    std::vector<std::int64_t> lm(steps, 0), tm(steps, 0), lc(steps, 0), tc(steps, 0);
    if (bands_.size() == 1) {
        // BML_ECONSERVE still fills the arrays (through the violating step)
        const int rc = bml_dev_step(bands_[0], steps, lm.data(), tm.data(), lc.data(), tc.data());
        if (rc != BML_OK && (rc != BML_ECONSERVE || throw_on_violation)) raise(rc, "bml_dev_step");
    } else {
        std::vector<std::int64_t> a(16), b(16), c(16), d(16);
        for (long done = 0; done < steps;) {
            const int k = block_for(steps - done, block_steps_);
            for (bml_dev* h : bands_) {
                const int rc = bml_dev_step(h, k, a.data(), b.data(), c.data(), d.data());
                if (rc != BML_OK) raise(rc, "bml_dev_step");
                for (int s = 0; s < k; ++s) {
                    lm[done + s] += a[s];
                    tm[done + s] += b[s];
                    lc[done + s] += c[s];
                    tc[done + s] += d[s];
                }
            }
            done += k;
        }
    }
    for (long s = 0; s < steps; ++s) {
        StepMetrics& m = out[static_cast<std::size_t>(s)];
        m.step = first_step + s;
        m.lr_moved = lm[s];
        m.tb_moved = tm[s];
        m.lr_count = lc[s];
        m.tb_count = tc[s];
        const std::int64_t total = m.lr_count + m.tb_count;
        m.mobility = total == 0 ? 1.0 : static_cast<double>(m.lr_moved + m.tb_moved) / total;
    }
    return out;
}

std::int64_t DeviceLattice::phase(Phase p) {
    if (bands_.size() != 1)
        throw std::invalid_argument("DeviceLattice::phase: single phases need one band");
    std::int64_t moved = 0;
    ok(bml_dev_phase(bands_[0], p == Phase::Horizontal ? BML_PHASE_HORIZONTAL : BML_PHASE_VERTICAL,
                     &moved),
       "bml_dev_phase");
    return moved;
}

VehicleCounts DeviceLattice::counts() const {
    VehicleCounts total;
    for (bml_dev* h : bands_) {
        std::int64_t lr = 0, tb = 0;
        ok(bml_dev_counts(h, &lr, &tb), "bml_dev_counts");
        total.lr += lr;
        total.tb += tb;
    }
    return total;
}

void DeviceLattice::configure(int block_steps, int strip_rows) {
    for (bml_dev* h : bands_) ok(bml_dev_configure(h, block_steps, strip_rows), "bml_dev_configure");
    if (block_steps) block_steps_ = block_steps;
}

void DeviceLattice::set_resident(int mode) {
    for (bml_dev* h : bands_) ok(bml_dev_set_resident(h, mode), "bml_dev_set_resident");
}

void DeviceLattice::set_variant(int variant) {
    if (bands_.size() > 1) throw std::invalid_argument("set_variant: single-band lattices only");
    ok(bml_dev_set_variant(bands_[0], variant), "bml_dev_set_variant");
}

int DeviceLattice::resident_cluster() const {
    int c = 0;
    ok(bml_dev_path(bands_[0], &c), "bml_dev_path");
    return c;
}

void DeviceLattice::set_stream(void* cuda_stream) {
    if (bands_.size() != 1) throw std::invalid_argument("set_stream: single-band lattices only");
    ok(bml_dev_set_stream(bands_[0], cuda_stream), "bml_dev_set_stream");
}

void DeviceLattice::synchronize() const {
    for (bml_dev* h : bands_) ok(bml_dev_sync(h), "bml_dev_sync");
}

// ------------------------------------------------------------ engine entry points
namespace {

// One cached device lattice per host thread, reused while (n, devices) match,
// so repeated step()/run() calls do not re-allocate device memory.
DeviceLattice& lattice_for(int n, int devices) {
    thread_local std::unique_ptr<DeviceLattice> cache;
    if (!cache || cache->n() != n || cache->bands() != devices) {
        cache.reset();
        cache = std::make_unique<DeviceLattice>(n, devices);
    }
    return *cache;
}

void check_pair(std::string_view where, const GridPair& pair, Backend backend, int threads) {
    if (pair.cur.n() != pair.next.n() || pair.cur.stride() != pair.next.stride())
        throw std::invalid_argument(std::string(where) + ": cur/next buffers differ in size");
    if (threads < 1) throw std::invalid_argument(std::string(where) + ": threads must be >= 1");
    if (threads > 1 && backend != Backend::ParallelRows)
        throw std::invalid_argument(std::string(where) + ": backend '" +
                                    std::string(backend_name(backend)) +
                                    "' does not support threads > 1");
    // The reference backend names keep the reference's layout contract
    // (engine.cpp:157-162: naive wants a dense grid, the others a halo grid);
    // the phase itself runs on the device engine, as for b200, which takes
    // either layout.
    if (backend != Backend::B200) {
        const bool want_halo = backend != Backend::ScalarNaive;
        if (pair.cur.has_halo() != want_halo)
            throw std::invalid_argument(std::string(where) + ": backend '" +
                                        std::string(backend_name(backend)) +
                                        (want_halo ? "' requires a halo grid" : "' requires a dense grid"));
    }
}

}  // namespace

void step_phase(Backend backend, GridPair& pair, Phase phase, int threads) {
    check_pair("step_phase", pair, backend, threads);
    DeviceLattice& dev = lattice_for(pair.cur.n(), 1);
    dev.upload(pair.cur);
    dev.phase(phase);
    dev.download(pair.next);
    std::swap(pair.cur, pair.next);
}

void step(Backend backend, GridPair& pair, int threads) {
    check_pair("step", pair, backend, threads);
    DeviceLattice& dev = lattice_for(pair.cur.n(), 1);
    dev.upload(pair.cur);
    dev.step(1);
    dev.download(pair.next);
    std::swap(pair.cur, pair.next);
}

Grid run(const SimConfig& cfg, GridPair& pair, const StepObserver& observer) {
    validate(cfg);
    if (pair.cur.n() != cfg.n) throw std::invalid_argument("run: grid size does not match config");
    if (cfg.steps > 0) check_pair("run", pair, cfg.backend, cfg.threads);
    DeviceLattice& dev = lattice_for(cfg.n, cfg.devices);
    dev.set_census(cfg.strict_census);
    dev.upload(pair.cur);
    if (!observer) {
        dev.step(cfg.steps);
        dev.download(pair.cur);
        return pair.cur;
    }
    const VehicleCounts initial = dev.counts();
    auto deliver = [&](const StepMetrics& m) {
        if (m.lr_count != initial.lr || m.tb_count != initial.tb)
            throw std::logic_error("conservation violated at step " + std::to_string(m.step) +
                                   ": lr " + std::to_string(m.lr_count) + "/" +
                                   std::to_string(initial.lr) + ", tb " +
                                   std::to_string(m.tb_count) + "/" + std::to_string(initial.tb));
        observer(m);
    };
    if (cfg.observer_reads_grid) {
        // reference contract: pair.cur holds the post-step grid at every call
        for (long s = 1; s <= cfg.steps; ++s) {
            const std::vector<StepMetrics> m = dev.step_with_metrics(1, s, false);
            dev.download(pair.cur);
            deliver(m[0]);
        }
    } else {
        constexpr long kChunk = 1L << 16;
        for (long s = 1; s <= cfg.steps; s += kChunk) {
            const long k = std::min(kChunk, cfg.steps - s + 1);
            for (const StepMetrics& m : dev.step_with_metrics(k, s, false)) deliver(m);
        }
        dev.download(pair.cur);
    }
    return pair.cur;
}

}  // namespace bml
