// pybind11 module `_bml` — the reference's Python surface
// (/root/reference/proj/bindings/py_module.cpp:38-158, re-exported by
// proj/python/bml/__init__.py) backed by the b200 engine. Differences, all
// additive: Backend.b200 (the default), a `devices=` keyword on step/simulate,
// Grid.from_bytes/to_bytes for bulk I/O, and DeviceLattice for a lattice that
// stays resident on the GPU between calls. Long device calls release the GIL.
#include <pybind11/functional.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>
#include <pybind11/stl/filesystem.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "bml/digest.hpp"
#include "bml/engine.hpp"
#include "bml/metrics.hpp"
#include "bml/seeding.hpp"
#include "bml/snapshot.hpp"
#include "bml/verify.hpp"
#include "bml_dev.h"

namespace py = pybind11;

namespace {

bml::Grid step_many(const bml::Grid& grid, long steps, bml::Backend backend, int threads,
                    int devices) {
    bml::SimConfig cfg;
    cfg.n = grid.n();
    cfg.steps = steps;
    cfg.backend = backend;
    cfg.threads = threads;
    cfg.devices = devices;
    bml::GridPair pair = bml::make_grid_pair(backend, grid);
    py::gil_scoped_release nogil;
    return bml::run(cfg, pair);
}

std::pair<bml::Grid, std::vector<bml::StepMetrics>> simulate(const bml::Grid& grid, long steps,
                                                             bml::Backend backend, int threads,
                                                             int devices, bool strict_census) {
    bml::SimConfig cfg;
    cfg.n = grid.n();
    cfg.steps = steps;
    cfg.backend = backend;
    cfg.threads = threads;
    cfg.devices = devices;
    cfg.strict_census = strict_census;
    cfg.observer_reads_grid = false;  // the collector below never reads the grid
    bml::GridPair pair = bml::make_grid_pair(backend, grid);
    std::vector<bml::StepMetrics> metrics;
    metrics.reserve(static_cast<std::size_t>(std::max(0L, steps)));
    {
        py::gil_scoped_release nogil;
        bml::run(cfg, pair, [&](const bml::StepMetrics& m) { metrics.push_back(m); });
    }
    return {pair.cur, std::move(metrics)};
}

bml::Grid grid_from_bytes(int n, const py::bytes& data) {
    const std::string s = data;
    if (n < 1) throw std::invalid_argument("from_bytes: n must be >= 1");
    if (s.size() != static_cast<std::size_t>(n) * n)
        throw std::invalid_argument("from_bytes: expected n*n bytes");
    bml::Grid g = bml::Grid::with_halo(n);
    for (int r = 0; r < n; ++r) {
        for (int c = 0; c < n; ++c) {
            const auto v = static_cast<std::uint8_t>(s[static_cast<std::size_t>(r) * n + c]);
            if (v > 2) throw std::invalid_argument("from_bytes: cell value outside {0,1,2}");
            g.interior(r, c) = static_cast<bml::Cell>(v);
        }
    }
    return g;
}

py::bytes grid_to_bytes(const bml::Grid& g) {
    std::string s(static_cast<std::size_t>(g.n()) * g.n(), '\0');
    for (int r = 0; r < g.n(); ++r)
        std::memcpy(&s[static_cast<std::size_t>(r) * g.n()],
                    g.interior_data() + static_cast<std::size_t>(r) * g.stride(),
                    static_cast<std::size_t>(g.n()));
    return py::bytes(s);
}

}  // namespace

PYBIND11_MODULE(_bml, m) {
    m.doc() = "Biham-Middleton-Levine traffic CA — B200-native (sm_100a) engine";

    py::enum_<bml::Cell>(m, "Cell")
        .value("empty", bml::Cell::Empty)
        .value("lr", bml::Cell::LR)
        .value("tb", bml::Cell::TB);

    py::enum_<bml::Backend>(m, "Backend")
        .value("naive", bml::Backend::ScalarNaive)
        .value("halo", bml::Backend::ScalarHalo)
        .value("parallel", bml::Backend::ParallelRows)
        .value("lanes", bml::Backend::Lanes)
        .value("b200", bml::Backend::B200);

    py::enum_<bml::Phase>(m, "Phase")
        .value("horizontal", bml::Phase::Horizontal)
        .value("vertical", bml::Phase::Vertical);

    py::enum_<bml::Regime>(m, "Regime")
        .value("FreeFlow", bml::Regime::FreeFlow)
        .value("Jammed", bml::Regime::Jammed)
        .value("Intermediate", bml::Regime::Intermediate);

    py::class_<bml::Grid>(m, "Grid")
        .def_static("from_text", &bml::parse_grid, py::arg("text"))
        .def_static("from_bytes", &grid_from_bytes, py::arg("n"), py::arg("data"),
                    "Dense n*n interior bytes (0/1/2), row-major.")
        .def_property_readonly("n", &bml::Grid::n)
        .def("to_text", &bml::render_grid)
        .def("to_bytes", &grid_to_bytes)
        .def("cell",
             [](const bml::Grid& g, int r, int c) {
                 if (r < 0 || r >= g.n() || c < 0 || c >= g.n())
                     throw py::index_error("cell index out of range");
                 return g.interior(r, c);
             },
             py::arg("row"), py::arg("col"))
        .def("set_cell",
             [](bml::Grid& g, int r, int c, bml::Cell cell) {
                 if (r < 0 || r >= g.n() || c < 0 || c >= g.n())
                     throw py::index_error("cell index out of range");
                 g.interior(r, c) = cell;
             },
             py::arg("row"), py::arg("col"), py::arg("cell"))
        .def("digest", &bml::grid_digest)
        .def("__eq__", [](const bml::Grid& a, const bml::Grid& b) { return a == b; },
             py::is_operator())
        .def("__repr__",
             [](const bml::Grid& g) { return "<bml.Grid n=" + std::to_string(g.n()) + ">"; });

    py::class_<bml::StepMetrics>(m, "StepMetrics")
        .def_readonly("step", &bml::StepMetrics::step)
        .def_readonly("lr_count", &bml::StepMetrics::lr_count)
        .def_readonly("tb_count", &bml::StepMetrics::tb_count)
        .def_readonly("lr_moved", &bml::StepMetrics::lr_moved)
        .def_readonly("tb_moved", &bml::StepMetrics::tb_moved)
        .def_readonly("mobility", &bml::StepMetrics::mobility)
        .def("__repr__", [](const bml::StepMetrics& s) {
            return "<bml.StepMetrics step=" + std::to_string(s.step) +
                   " mobility=" + std::to_string(s.mobility) + ">";
        });

    m.def("init_grid",
          [](int n, double rho, std::uint64_t seed, bool on_device) {
              py::gil_scoped_release nogil;
              if (on_device) return bml::init_grid_device({n, rho, seed});
              return bml::init_grid({n, rho, seed});
          },
          py::arg("n"), py::arg("rho"), py::arg("seed"), py::arg("on_device") = false,
          "The reference init_grid lattice; on_device=True computes the same lattice on the GPU.");

    py::class_<bml::VerifyReport>(m, "VerifyReport")
        .def_property_readonly("ok", &bml::VerifyReport::ok)
        .def_readonly("conserved", &bml::VerifyReport::conserved)
        .def_property_readonly("digests", [](const bml::VerifyReport& r) {
            py::dict out;
            for (const auto& d : r.digests) out[py::str(d.path)] = d.digest;
            return out;
        })
        .def_property_readonly("mismatch", [](const bml::VerifyReport& r) -> py::object {
            if (!r.mismatch) return py::none();
            return py::make_tuple(r.mismatch->a, r.mismatch->b, r.mismatch->row, r.mismatch->col);
        });

    m.def("verify_backends",
          [](int n, double rho, long steps, std::uint64_t seed, int threads) {
              bml::SimConfig cfg;
              cfg.n = n;
              cfg.rho = rho;
              cfg.steps = steps;
              cfg.seed = seed;
              cfg.threads = 1;
              (void)threads;  // reference signature; the device paths take no thread count
              cfg.backend = bml::Backend::B200;
              py::gil_scoped_release nogil;
              return bml::verify_backends(cfg);
          },
          py::arg("n"), py::arg("rho"), py::arg("steps"), py::arg("seed") = 1,
          py::arg("threads") = 1,
          "Run the four device code paths from one initial grid and compare bit-exactly.");

    m.def("verify_device",
          [](int n, double rho, long steps, std::uint64_t seed, std::vector<std::string> paths) {
              bml::SimConfig cfg;
              cfg.n = n;
              cfg.rho = rho;
              cfg.steps = steps;
              cfg.seed = seed;
              cfg.backend = bml::Backend::B200;
              py::gil_scoped_release nogil;
              return bml::verify_device(cfg, paths);
          },
          py::arg("n"), py::arg("rho"), py::arg("steps"), py::arg("seed") = 1,
          py::arg("paths") = std::vector<std::string>{},
          "Cross-check every device code path (or the named subset) from one initial grid, bit-exactly.");

    m.def("encode_ppm", [](const bml::Grid& g) {
        const auto bytes = bml::encode_ppm(g);
        return py::bytes(reinterpret_cast<const char*>(bytes.data()), bytes.size());
    }, py::arg("grid"));
    // str or os.PathLike, as in the reference binding (py_module.cpp:135)
    m.def("write_ppm", [](const bml::Grid& g, const std::filesystem::path& path) { bml::write_ppm(g, path); },
          py::arg("grid"), py::arg("path"));

    m.def("vehicles_per_species", &bml::vehicles_per_species, py::arg("n"), py::arg("rho"));

    m.def("step", &step_many, py::arg("grid"), py::arg("steps") = 1,
          py::arg("backend") = bml::Backend::B200, py::arg("threads") = 1, py::arg("devices") = 1,
          "Advance `steps` full steps on the GPU and return the resulting grid.");

    m.def("step_phase",
          [](const bml::Grid& grid, bml::Phase phase, bml::Backend backend) {
              bml::GridPair pair = bml::make_grid_pair(backend, grid);
              py::gil_scoped_release nogil;
              bml::step_phase(backend, pair, phase, 1);
              return pair.cur;
          },
          py::arg("grid"), py::arg("phase"), py::arg("backend") = bml::Backend::B200,
          "One phase (step_phase) on the GPU.");

    m.def("simulate", &simulate, py::arg("grid"), py::arg("steps"),
          py::arg("backend") = bml::Backend::B200, py::arg("threads") = 1, py::arg("devices") = 1,
          py::arg("strict_census") = false,
          "Advance and record per-step metrics; returns (grid, [StepMetrics]). strict_census: "
          "vehicle census after every step (the reference's exact per-step check) rather than "
          "at launch boundaries.");

    m.def("count_vehicles",
          [](const bml::Grid& g) {
              const auto c = bml::count_vehicles(g);
              return py::make_tuple(c.lr, c.tb);
          },
          py::arg("grid"));

    m.def("moved_in_phase", &bml::moved_in_phase, py::arg("before"), py::arg("after"),
          py::arg("phase"));

    m.def("classify", [](const std::vector<double>& w) { return bml::classify(w); },
          py::arg("mobility_window"));

    m.def("backend_from_name", &bml::backend_from_name, py::arg("name"));
    m.def("lane_width", &bml::lane_width);
    m.def("device_count", []() {
        int c = 0;
        if (bml_dev_device_count(&c) != BML_OK) return 0;
        return c;
    });
    m.def("library_version", []() { return std::string(bml_dev_version()); });

    py::class_<bml::DeviceLattice>(m, "DeviceLattice")
        .def(py::init<int, int>(), py::arg("n"), py::arg("devices") = 1)
        .def_property_readonly("n", &bml::DeviceLattice::n)
        .def_property_readonly("bands", &bml::DeviceLattice::bands)
        .def("upload", &bml::DeviceLattice::upload, py::arg("grid"),
             py::call_guard<py::gil_scoped_release>())
        .def("init_random", &bml::DeviceLattice::init_random, py::arg("rho"), py::arg("seed"),
             py::call_guard<py::gil_scoped_release>())
        .def("download", py::overload_cast<>(&bml::DeviceLattice::download, py::const_),
             py::call_guard<py::gil_scoped_release>())
        .def("step", &bml::DeviceLattice::step, py::arg("steps"),
             py::call_guard<py::gil_scoped_release>())
        .def("step_with_metrics", &bml::DeviceLattice::step_with_metrics, py::arg("steps"),
             py::arg("first_step") = 1, py::arg("throw_on_violation") = true,
             py::call_guard<py::gil_scoped_release>())
        .def("set_census", &bml::DeviceLattice::set_census, py::arg("every_step"))
        .def("debug_fault", &bml::DeviceLattice::debug_fault, py::arg("at_step"), py::arg("row"),
             py::arg("col"), "TEST HOOK: toggle a cell after at_step steps of the next step call.")
        .def("phase", &bml::DeviceLattice::phase, py::arg("phase"),
             py::call_guard<py::gil_scoped_release>())
        .def("counts",
             [](const bml::DeviceLattice& d) {
                 const auto c = d.counts();
                 return py::make_tuple(c.lr, c.tb);
             })
        .def("digest", &bml::DeviceLattice::digest, py::call_guard<py::gil_scoped_release>(),
             "grid_digest of the device lattice, computed on the GPU")
        .def("encode_ppm",
             [](const bml::DeviceLattice& d) {
                 std::vector<std::uint8_t> bytes;
                 {
                     py::gil_scoped_release nogil;
                     bytes = d.encode_ppm();
                 }
                 return py::bytes(reinterpret_cast<const char*>(bytes.data()), bytes.size());
             },
             "encode_ppm of the device lattice (pixels expanded on the GPU)")
        .def("configure", &bml::DeviceLattice::configure, py::arg("block_steps") = 0,
             py::arg("strip_rows") = 0)
        .def("set_resident", &bml::DeviceLattice::set_resident, py::arg("mode"))
        .def("set_variant", &bml::DeviceLattice::set_variant, py::arg("variant"))
        .def_property_readonly("resident_cluster", &bml::DeviceLattice::resident_cluster)
        .def("set_stream",
             [](bml::DeviceLattice& d, std::uintptr_t s) { d.set_stream(reinterpret_cast<void*>(s)); },
             py::arg("stream"))
        .def("synchronize", &bml::DeviceLattice::synchronize,
             py::call_guard<py::gil_scoped_release>())
        .def("handle",
             [](const bml::DeviceLattice& d, int band) {
                 return reinterpret_cast<std::uintptr_t>(d.handle(band));
             },
             py::arg("band") = 0);

    m.attr("__version__") = "0.1.0";
}
