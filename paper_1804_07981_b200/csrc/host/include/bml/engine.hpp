// bml/engine.hpp — the reference engine interface
// (/root/reference/proj/include/bml/engine.hpp:15-79) with one new backend,
// Backend::B200 ("b200"), implemented on sm_100a through the C-ABI in
// include/bml_dev.h. This library ships no CPU stepping engine. The four
// reference backend names stay valid so reference call sites compile and run
// unchanged: they keep the reference's layout and thread rules (naive wants a
// dense grid, the others a halo grid; only parallel takes threads > 1) and
// their phases execute on the device engine, bit-identical by construction.
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
#include <memory>
#include <optional>
#include <string_view>
#include <vector>

#include "bml/grid.hpp"

struct bml_dev;

namespace bml {

enum class Backend {
    ScalarNaive,   // reference name: dense layout, runs on the device engine
    ScalarHalo,    // reference name: halo layout, runs on the device engine
    ParallelRows,  // reference name: halo layout, threads accepted, runs on the device
    Lanes,         // reference name: halo layout, runs on the device engine
    B200,          // device-resident bit-plane lattice on NVIDIA B200 (sm_100a)
};

enum class Phase { Horizontal, Vertical };

std::string_view backend_name(Backend b);
std::optional<Backend> backend_from_name(std::string_view name);

// Cells advanced per device word (the bit-plane width).
int lane_width();

constexpr Cell horizontal_rule(Cell left, Cell center, Cell right) {
    if (center == Cell::Empty) return left == Cell::LR ? Cell::LR : Cell::Empty;
    if (center == Cell::LR && right == Cell::Empty) return Cell::Empty;
    return center;
}

constexpr Cell vertical_rule(Cell top, Cell center, Cell bottom) {
    if (center == Cell::Empty) return top == Cell::TB ? Cell::TB : Cell::Empty;
    if (center == Cell::TB && bottom == Cell::Empty) return Cell::Empty;
    return center;
}

struct SimConfig {
    int n = 0;
    double rho = 0.0;
    long steps = 0;
    std::uint64_t seed = 0;
    Backend backend = Backend::B200;
    int threads = 1;
    long snapshot_every = 0;
    std::filesystem::path out_dir;
    // --- extensions (defaults keep reference call sites valid) ---
    int devices = 1;                  // row bands (GPUs); placed round-robin on visible GPUs
    bool observer_reads_grid = true;  // download pair.cur before every observer call
    bool strict_census = false;       // single band: vehicle census after every step, not
                                      // only at launch boundaries (bml_dev_set_census)
};

void validate(const SimConfig& cfg);

GridPair make_grid_pair(Backend backend, const Grid& initial);

void step_phase(Backend backend, GridPair& pair, Phase phase, int threads = 1);

void step(Backend backend, GridPair& pair, int threads = 1);

struct StepMetrics;
using StepObserver = std::function<void(const StepMetrics&)>;

Grid run(const SimConfig& cfg, GridPair& pair, const StepObserver& observer = {});

// ---- device-resident lattice (extension; what run()/step() use internally) ----
struct VehicleCounts;

// One n x n torus resident on the GPU(s): `devices` row bands placed
// round-robin on the visible GPUs, halo rows exchanged by the step kernel
// itself. Throws std::invalid_argument / std::runtime_error / std::bad_alloc
// mapped from the C-ABI status codes.
class DeviceLattice {
public:
    explicit DeviceLattice(int n, int devices = 1);
    ~DeviceLattice();
    DeviceLattice(const DeviceLattice&) = delete;
    DeviceLattice& operator=(const DeviceLattice&) = delete;

    int n() const { return n_; }
    int bands() const { return static_cast<int>(bands_.size()); }

    void upload(const Grid& g);
    // The reference init_grid({n, rho, seed}) lattice, generated on the device
    // (bit-identical; bml_dev_init_random). n <= 65536.
    void init_random(double rho, std::uint64_t seed);
    void download(Grid& g) const;  // writes the interior of g (any layout, size n)
    Grid download() const;         // halo-layout grid, ghosts unfilled

    void step(long steps);
    // Per-step metrics for `steps` steps; step indices start at first_step.
    // Throws std::logic_error on a conservation violation (engine.cpp:219-224)
    // unless throw_on_violation is false: then the metrics come back with the
    // measured (violating) counts and the caller decides (run() throws at the
    // first step whose counts differ, delivering the steps before it).
    std::vector<StepMetrics> step_with_metrics(long steps, long first_step = 1,
                                               bool throw_on_violation = true);
    // Vehicle-census cadence on a single band: after every step (true) or after
    // each launch's last step (false, default). See bml_dev_set_census.
    void set_census(bool every_step);
    // TEST HOOK: toggle cell (row, col) after `at_step` steps of the next
    // step()/step_with_metrics() call (bml_dev_debug_fault). Single band only.
    void debug_fault(long at_step, int row, int col);
    std::int64_t phase(Phase p);  // returns moved_in_phase
    VehicleCounts counts() const;
    // grid_digest (digest.hpp) of the device lattice, computed on the GPU(s).
    std::uint64_t digest() const;
    // encode_ppm (snapshot.hpp) of the device lattice; pixels expanded on the GPU.
    std::vector<std::uint8_t> encode_ppm() const;

    void configure(int block_steps, int strip_rows);
    // Small-lattice cluster-resident kernel: enabled by default; resident_cluster()
    // reports the cluster size the last step() used (0 = streaming kernel).
    void set_resident(int mode);  // 0 = off, 1 = ghost-zone kernel (default), 2 = p2p kernel
    // Streaming-kernel variant (bml_dev_set_variant): 0 automatic, 1 narrow, 6 even/odd layout, ...
    void set_variant(int variant);
    int resident_cluster() const;
    void set_stream(void* cuda_stream);  // single-band only
    void synchronize() const;
    bml_dev* handle(int band = 0) const { return bands_.at(static_cast<std::size_t>(band)); }

private:
    int n_;
    std::vector<bml_dev*> bands_;
    int block_steps_ = 8;
};

struct SeedSpec;
// init_grid (seeding.hpp) computed on the GPU and read back: same Grid, bit for
// bit, without the serial host shuffle (minutes at n = 65536). n <= 65536.
Grid init_grid_device(const SeedSpec& spec);

}  // namespace bml
