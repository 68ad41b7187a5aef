// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (checker, never the product).
//
// A tiny command-line harness linked against the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/). It exposes the reference's own hot path to the parity tests
// and to bench.py's reference arm without linking the reference into the
// product (both define namespace `bml`, so they must live in separate
// processes — SURVEY.md §7 step 1).
//
// Reference entry points exercised (all file:line in /root/reference/proj):
//   bml::init_grid            src/seeding.cpp:26-51
//   bml::make_grid_pair       src/engine.cpp:59-64
//   bml::run (bare loop)      src/engine.cpp:206-208   (what `bml bench` times)
//   bml::run (observer loop)  src/engine.cpp:211-235   (per-step StepMetrics)
//   bml::step_phase           src/engine.cpp:148-179
//   bml::grid_digest          src/digest.cpp:5-14
//   bench timing method       tools/main.cpp:195-214   (steady_clock around run)
//
// Usage (key=value arguments, JSON on stdout):
//   ref_driver golden  n=N rho=R seed=S steps=T [backend=lanes] [threads=1]
//                      [metrics=0|1] [dump_init=PATH] [dump_final=PATH]
//   ref_driver file    in=PATH n=N steps=T [backend=lanes] [threads=1]
//                      [phase=h|v] [metrics=0|1] [dump_final=PATH]
//   ref_driver bench   n=N rho=R seed=S steps=T backend=B [threads=0] [reps=5]
//   ref_driver ladder  n=N rho=R seed=S plan=B:threads:steps:reps[,...]
//                      [in=PATH expect_init=0xDIGEST]   (one init, several backends)
//   ref_driver info
// Lattice files are the n*n interior bytes, row-major (values 0/1/2).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bml/digest.hpp"
#include "bml/engine.hpp"
#include "bml/metrics.hpp"
#include "bml/seeding.hpp"

namespace {

using Args = std::map<std::string, std::string>;

Args parse_args(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        auto eq = s.find('=');
        if (eq == std::string::npos) throw std::invalid_argument("expected key=value: " + s);
        a[s.substr(0, eq)] = s.substr(eq + 1);
    }
    return a;
}

std::string get(const Args& a, const std::string& k, const std::string& dflt) {
    auto it = a.find(k);
    return it == a.end() ? dflt : it->second;
}

std::string need(const Args& a, const std::string& k) {
    auto it = a.find(k);
    if (it == a.end()) throw std::invalid_argument("missing argument " + k);
    return it->second;
}

bml::Backend backend_arg(const Args& a) {
    auto b = bml::backend_from_name(get(a, "backend", "lanes"));
    if (!b) throw std::invalid_argument("unknown backend");
    return *b;
}

int threads_arg(const Args& a, bml::Backend b) {
    int t = std::stoi(get(a, "threads", "1"));
    if (t <= 0) {
        if (b != bml::Backend::ParallelRows) return 1;
        unsigned hw = std::thread::hardware_concurrency();
        return hw == 0 ? 1 : static_cast<int>(hw);
    }
    return t;
}

std::string hex(std::uint64_t v) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "\"0x%016llx\"", static_cast<unsigned long long>(v));
    return buf;
}

void dump_interior(const bml::Grid& g, const std::string& path) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error("cannot open " + path);
    std::vector<char> row(static_cast<std::size_t>(g.n()));
    for (int r = 0; r < g.n(); ++r) {
        for (int c = 0; c < g.n(); ++c) row[c] = static_cast<char>(g.interior(r, c));
        f.write(row.data(), static_cast<std::streamsize>(row.size()));
    }
}

bml::Grid load_interior(const std::string& path, int n) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    bml::Grid g = bml::Grid::with_halo(n);
    std::vector<char> row(static_cast<std::size_t>(n));
    for (int r = 0; r < n; ++r) {
        f.read(row.data(), n);
        if (!f) throw std::runtime_error("short lattice file " + path);
        for (int c = 0; c < n; ++c) g.interior(r, c) = static_cast<bml::Cell>(row[c]);
    }
    return g;
}

// Runs `steps` steps (or one phase) from `initial` through the reference and
// prints a JSON record. With metrics=1 the observer loop runs, so per-step
// conservation is asserted by the reference itself.
int simulate_and_report(const bml::Grid& initial, const Args& a, long steps, double init_s,
                        const std::string& extra) {
    const bml::Backend backend = backend_arg(a);
    const int threads = threads_arg(a, backend);
    const bool metrics = get(a, "metrics", "0") == "1";
    const std::string phase = get(a, "phase", "");

    bml::GridPair pair = bml::make_grid_pair(backend, initial);
    std::string metrics_json;
    const auto t0 = std::chrono::steady_clock::now();
    if (!phase.empty()) {
        const bml::Phase p = phase == "h" ? bml::Phase::Horizontal : bml::Phase::Vertical;
        if (backend != bml::Backend::ScalarNaive) {
            if (p == bml::Phase::Horizontal) pair.cur.fill_horizontal_halo();
            else pair.cur.fill_vertical_halo();
        }
        bml::step_phase(backend, pair, p, threads);
    } else if (metrics) {
        bml::SimConfig cfg;
        cfg.n = initial.n();
        cfg.steps = steps;
        cfg.backend = backend;
        cfg.threads = threads;
        std::int64_t sum_lr = 0, sum_tb = 0;
        std::vector<bml::StepMetrics> all;
        bml::run(cfg, pair, [&](const bml::StepMetrics& m) {
            sum_lr += m.lr_moved;
            sum_tb += m.tb_moved;
            all.push_back(m);
        });
        char buf[512];
        std::snprintf(buf, sizeof buf, ",\"sum_lr_moved\":%lld,\"sum_tb_moved\":%lld",
                      static_cast<long long>(sum_lr), static_cast<long long>(sum_tb));
        metrics_json = buf;
        if (!all.empty()) {
            const auto& m = all.back();
            std::snprintf(buf, sizeof buf,
                          ",\"last\":{\"step\":%lld,\"lr_count\":%lld,\"tb_count\":%lld,"
                          "\"lr_moved\":%lld,\"tb_moved\":%lld,\"mobility\":%.17g}",
                          static_cast<long long>(m.step), static_cast<long long>(m.lr_count),
                          static_cast<long long>(m.tb_count), static_cast<long long>(m.lr_moved),
                          static_cast<long long>(m.tb_moved), m.mobility);
            metrics_json += buf;
            // the regime the reference's CLI / acceptance program reports: classify()
            // over the last kClassifyWindow mobilities (acceptance_main.cpp:74-78)
            const std::size_t w = std::min(all.size(), static_cast<std::size_t>(bml::kClassifyWindow));
            std::vector<double> window;
            for (std::size_t i = all.size() - w; i < all.size(); ++i) window.push_back(all[i].mobility);
            std::snprintf(buf, sizeof buf, ",\"regime\":\"%s\"",
                          std::string(bml::regime_name(bml::classify(window))).c_str());
            metrics_json += buf;
        }
        const std::string per_step = get(a, "per_step", "");
        if (!per_step.empty()) {
            std::ofstream f(per_step, std::ios::trunc);
            f << "step,lr_count,tb_count,lr_moved,tb_moved\n";
            for (const auto& m : all)
                f << m.step << ',' << m.lr_count << ',' << m.tb_count << ',' << m.lr_moved << ','
                  << m.tb_moved << '\n';
        }
    } else {
        bml::SimConfig cfg;
        cfg.n = initial.n();
        cfg.steps = steps;
        cfg.backend = backend;
        cfg.threads = threads;
        bml::run(cfg, pair);
    }
    const double run_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    const auto counts = bml::count_vehicles(pair.cur);
    const std::string dump_final = get(a, "dump_final", "");
    if (!dump_final.empty()) dump_interior(pair.cur, dump_final);

    std::printf(
        "{\"n\":%d,\"steps\":%ld,\"backend\":\"%s\",\"threads\":%d,\"final_digest\":%s,"
        "\"lr_count\":%lld,\"tb_count\":%lld,\"init_s\":%.6f,\"run_s\":%.6f%s%s}\n",
        initial.n(), steps, std::string(bml::backend_name(backend)).c_str(), threads,
        hex(bml::grid_digest(pair.cur)).c_str(), static_cast<long long>(counts.lr),
        static_cast<long long>(counts.tb), init_s, run_s, extra.c_str(), metrics_json.c_str());
    return 0;
}

int cmd_golden(const Args& a) {
    const int n = std::stoi(need(a, "n"));
    const double rho = std::stod(need(a, "rho"));
    const std::uint64_t seed = std::stoull(need(a, "seed"));
    const long steps = std::stol(get(a, "steps", "0"));
    const auto t0 = std::chrono::steady_clock::now();
    const bml::Grid initial = bml::init_grid({n, rho, seed});
    const double init_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const std::string dump_init = get(a, "dump_init", "");
    if (!dump_init.empty()) dump_interior(initial, dump_init);
    char buf[256];
    std::snprintf(buf, sizeof buf, ",\"rho\":%.17g,\"seed\":%llu,\"k\":%lld,\"init_digest\":%s",
                  rho, static_cast<unsigned long long>(seed),
                  static_cast<long long>(bml::vehicles_per_species(n, rho)),
                  hex(bml::grid_digest(initial)).c_str());
    return simulate_and_report(initial, a, steps, init_s, buf);
}

int cmd_file(const Args& a) {
    const int n = std::stoi(need(a, "n"));
    const long steps = std::stol(get(a, "steps", "0"));
    const bml::Grid initial = load_interior(need(a, "in"), n);
    char buf[64];
    std::snprintf(buf, sizeof buf, ",\"init_digest\":%s", hex(bml::grid_digest(initial)).c_str());
    return simulate_and_report(initial, a, steps, 0.0, buf);
}

// The reference's own bench method (tools/main.cpp:186-214): init once, then
// per rep make_grid_pair (untimed) + steady_clock around run() without an
// observer; mean and population stddev.
std::string bench_backend(const bml::Grid& initial, double rho, std::uint64_t seed,
                          bml::Backend backend, int threads, long steps, int reps) {
    bml::SimConfig cfg;
    cfg.n = initial.n();
    cfg.rho = rho;
    cfg.steps = steps;
    cfg.seed = seed;
    cfg.backend = backend;
    cfg.threads = threads;
    bml::validate(cfg);
    std::vector<double> times;
    std::uint64_t digest = 0;
    for (int rep = 0; rep < reps; ++rep) {
        bml::GridPair pair = bml::make_grid_pair(backend, initial);
        const auto t0 = std::chrono::steady_clock::now();
        bml::run(cfg, pair);
        const auto t1 = std::chrono::steady_clock::now();
        times.push_back(std::chrono::duration<double>(t1 - t0).count());
        digest = bml::grid_digest(pair.cur);
    }
    double mean = 0.0;
    for (double t : times) mean += t;
    mean /= reps;
    double var = 0.0;
    for (double t : times) var += (t - mean) * (t - mean);
    var /= reps;
    std::string ts;
    for (std::size_t i = 0; i < times.size(); ++i) {
        char buf[32];
        std::snprintf(buf, sizeof buf, "%s%.6f", i ? "," : "", times[i]);
        ts += buf;
    }
    char head[512];
    std::snprintf(head, sizeof head,
                  "{\"backend\":\"%s\",\"n\":%d,\"threads\":%d,\"reps\":%d,\"steps\":%ld,\"mean_s\":%.6f,"
                  "\"stddev_s\":%.6f,\"times\":[",
                  std::string(bml::backend_name(backend)).c_str(), initial.n(), threads, reps, steps,
                  mean, std::sqrt(var));
    char tail[256];
    std::snprintf(tail, sizeof tail,
                  "],\"final_digest\":%s,\"lane_width\":%d,\"hardware_concurrency\":%u}",
                  hex(digest).c_str(), bml::lane_width(), std::thread::hardware_concurrency());
    return std::string(head) + ts + tail;
}

int cmd_bench(const Args& a) {
    const int n = std::stoi(need(a, "n"));
    const double rho = std::stod(need(a, "rho"));
    const std::uint64_t seed = std::stoull(get(a, "seed", "1"));
    const long steps = std::stol(need(a, "steps"));
    const int reps = std::stoi(get(a, "reps", "5"));
    const bml::Backend backend = backend_arg(a);
    const int threads = threads_arg(a, backend);
    const bml::Grid initial = bml::init_grid({n, rho, seed});
    std::printf("%s\n", bench_backend(initial, rho, seed, backend, threads, steps, reps).c_str());
    return 0;
}

// One input lattice, several backends: the reference bench method per backend
// (bench_backend) after a SINGLE init — at n = 65536 the reference init_grid
// alone takes ~8 min and ~43 GB (seeding.cpp:26-51), so the CPU arm cannot
// afford one per backend. The lattice is the reference's own init_grid, or
// (in=PATH) n*n interior bytes whose grid_digest must equal expect_init
// (the reference init digest from the committed goldens).
//   plan=backend:threads:steps:reps[,backend:threads:steps:reps...]
int cmd_ladder(const Args& a) {
    const int n = std::stoi(need(a, "n"));
    const double rho = std::stod(need(a, "rho"));
    const std::uint64_t seed = std::stoull(get(a, "seed", "1"));
    const std::string in = get(a, "in", "");
    const auto t0 = std::chrono::steady_clock::now();
    const bml::Grid initial = in.empty() ? bml::init_grid({n, rho, seed}) : load_interior(in, n);
    const double init_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const std::uint64_t init_digest = bml::grid_digest(initial);
    const std::string expect = get(a, "expect_init", "");
    if (!expect.empty() && std::stoull(expect, nullptr, 16) != init_digest)
        throw std::runtime_error("ladder: input lattice digest " + hex(init_digest) +
                                 " differs from expect_init " + expect);
    std::string results;
    std::string plan = need(a, "plan");
    std::size_t pos = 0;
    while (pos <= plan.size()) {
        const std::size_t comma = std::min(plan.find(',', pos), plan.size());
        const std::string item = plan.substr(pos, comma - pos);
        pos = comma + 1;
        if (item.empty()) continue;
        std::vector<std::string> f;
        std::size_t p = 0;
        while (p <= item.size()) {
            const std::size_t c = std::min(item.find(':', p), item.size());
            f.push_back(item.substr(p, c - p));
            p = c + 1;
        }
        if (f.size() != 4) throw std::invalid_argument("ladder: plan item must be backend:threads:steps:reps");
        auto b = bml::backend_from_name(f[0]);
        if (!b) throw std::invalid_argument("ladder: unknown backend " + f[0]);
        Args ta;
        ta["threads"] = f[1];
        const int threads = threads_arg(ta, *b);
        results += (results.empty() ? "" : ",") +
                   bench_backend(initial, rho, seed, *b, threads, std::stol(f[2]), std::stoi(f[3]));
    }
    std::printf("{\"n\":%d,\"rho\":%.17g,\"seed\":%llu,\"init_source\":\"%s\",\"init_s\":%.6f,"
                "\"init_digest\":%s,\"results\":[%s]}\n",
                n, rho, static_cast<unsigned long long>(seed), in.empty() ? "init_grid" : "file",
                init_s, hex(init_digest).c_str(), results.c_str());
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_driver golden|file|bench|info key=value...\n");
        return 1;
    }
    try {
        const std::string cmd = argv[1];
        const Args a = parse_args(argc, argv, 2);
        if (cmd == "golden") return cmd_golden(a);
        if (cmd == "file") return cmd_file(a);
        if (cmd == "bench") return cmd_bench(a);
        if (cmd == "ladder") return cmd_ladder(a);
        if (cmd == "info") {
            std::printf("{\"lane_width\":%d,\"hardware_concurrency\":%u}\n", bml::lane_width(),
                        std::thread::hardware_concurrency());
            return 0;
        }
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 1;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const std::logic_error& e) {
        std::fprintf(stderr, "logic_error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    }
}
