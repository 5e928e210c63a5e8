// plbm_gpu_run.cpp — the reference's simulation driver on the B200 engine.
//
// This is the reference side of the drop-in boundary ("C++
// side"): a GpuEngine with plbm::engine::Engine's shape wraps the C-ABI of
// include/plbm_gpu.h, and a driver cloned from the output contract of
// engine::run_scenario (proj/src/engine.cpp:580-704) runs a scenario TOML
// loaded and validated by the reference's own iobench::load_config, with the
// reference's own report writers (proj/src/report.cpp) producing
// time_series.csv, creation_log.csv and summary.json, and plbm_gpu_dump_field
// producing the snapshots (byte-identical to iobench::dump_field).
//
// Build: integration/Makefile links the reference objects compiled from
// /root/reference/proj/src (oracle/Makefile) with libplbm_gpu.so.
//   integration/_bin/plbm_gpu_run <scenario.toml> [--output DIR] [--device N] [--compare 1]
// --compare 1 is the reference's `compare` subcommand (proj/src/cli.cpp:133-157).
#include "plbm/dump.hpp"
#include "plbm/engine.hpp"
#include "plbm/geometry.hpp"
#include "plbm/report.hpp"
#include "plbm/scenario.hpp"
#include "plbm/tile.hpp"
#include "plbm/tilemap.hpp"
#include "plbm/topology.hpp"

#include "plbm_gpu.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

using namespace plbm;

namespace {

// The descriptor the C-ABI takes, filled from a validated ScenarioConfig
// (INTEGRATION.md §1).  The vectors own the storage the pointers refer to.
struct GpuDesc {
    plbm_scenario_desc d{};
    std::vector<plbm_component_desc> comps;
    std::vector<plbm_seed_desc> seeds;
    std::vector<double> coupling;
    std::vector<uint8_t> p2p;
    std::vector<uint8_t> geometry;
};

GpuDesc make_desc(const iobench::ScenarioConfig& cfg, const iobench::GeometryMask& geom,
                  const sched::DeviceTopology& topo) {
    if (!cfg.three_d()) throw std::runtime_error("plbm_gpu_run: the GPU step loop is D3Q19 only");
    GpuDesc g;
    for (const auto& c : cfg.components)  // physics.hpp:14-30
        g.comps.push_back({c.tau, c.rho_ambient, c.g_self, c.beta,
                           {c.gravity[0], c.gravity[1], c.gravity[2]},
                           c.eos.a, c.eos.b, c.eos.R, c.eos.T, c.eos.Tc, c.eos.omega});
    for (const auto& r : cfg.seeds) {  // scenario.hpp:18-30
        plbm_seed_desc s{};
        s.shape = r.shape == iobench::SeedRegion::Shape::Sphere ? PLBM_SEED_SPHERE : PLBM_SEED_BOX;
        s.component = r.component;
        for (int a = 0; a < 3; ++a) {
            s.box_min[a] = r.box_min[a];
            s.box_max[a] = r.box_max[a];
            s.center[a] = r.center[a];
            s.velocity[a] = r.velocity[a];
        }
        s.radius = r.radius;
        s.rho = r.rho;
        g.seeds.push_back(s);
    }
    g.coupling = cfg.coupling.g;
    g.p2p = topo.p2p;
    if (geom.solid_count() > 0) g.geometry = geom.solid;
    plbm_scenario_desc& d = g.d;
    for (int a = 0; a < 3; ++a) {
        d.domain[a] = cfg.domain[a];
        d.periodic[a] = cfg.boundary[a] == iobench::BoundaryKind::Periodic;
    }
    d.tile_extent = cfg.tile_extent;
    d.mode = cfg.mode == iobench::RunMode::Static ? PLBM_MODE_STATIC : PLBM_MODE_PROGRESSIVE;
    d.threshold = cfg.threshold;
    d.devices = topo.n_devices;
    d.policy = cfg.policy == sched::AssignPolicy::Simple ? PLBM_POLICY_SIMPLE : PLBM_POLICY_OPTIMIZED;
    d.weight_p2p = topo.weight_p2p;
    d.weight_staged = topo.weight_staged;
    d.p2p = g.p2p.data();
    d.n_components = int(g.comps.size());
    d.components = g.comps.data();
    d.coupling = g.coupling.empty() ? nullptr : g.coupling.data();
    d.n_seeds = int(g.seeds.size());
    d.seeds = g.seeds.data();
    d.geometry = g.geometry.empty() ? nullptr : g.geometry.data();
    return g;
}

// Engine's shape (engine.hpp:98-116) over the C-ABI.
class GpuEngine {
  public:
    GpuEngine(const iobench::ScenarioConfig& cfg, const iobench::GeometryMask& geom,
              const sched::DeviceTopology& topo, int device)
        : desc_(make_desc(cfg, geom, topo)) {
        plbm_error e{};
        h_ = plbm_gpu_create(&desc_.d, device, &e);
        if (!h_) throw std::runtime_error(std::string("plbm_gpu_create: ") + e.message);
    }
    ~GpuEngine() { plbm_gpu_destroy(h_); }
    GpuEngine(const GpuEngine&) = delete;
    GpuEngine& operator=(const GpuEngine&) = delete;

    // engine.cpp:537-563; EngineError on NaN / EOS pole, counters unchanged.
    void step() {
        plbm_error e{};
        if (plbm_gpu_step(h_, 1, &e) == 0) return;
        if (e.code != 1) throw std::runtime_error(e.message);
        std::string msg = e.message;  // "iteration ..., tile (...), phase Pk: <what>"
        const std::string key = std::string("phase ") + e.phase + ": ";
        const size_t at = msg.find(key);
        const std::string what = at == std::string::npos ? msg : msg.substr(at + key.size());
        throw engine::EngineError(long(e.iteration), mesh::TileCoord{e.tile[0], e.tile[1], e.tile[2]},
                                  e.phase, what);
    }
    plbm_counters counters() {
        plbm_counters c{};
        plbm_gpu_counters(h_, &c);
        return c;
    }
    std::vector<mesh::CreationEvent> creation_log() {
        const int n = plbm_gpu_creation_log(h_, nullptr, 0);
        std::vector<plbm_creation_event> rows(size_t(std::max(n, 1)));
        plbm_gpu_creation_log(h_, rows.data(), n);
        std::vector<mesh::CreationEvent> out;
        for (int k = 0; k < n; ++k) {
            mesh::CreationEvent e;
            e.iteration = long(rows[k].iteration);
            e.coords = {rows[k].coords[0], rows[k].coords[1], rows[k].coords[2]};
            e.trigger = rows[k].trigger < 0 ? std::string("init") : std::string(mesh::kFaceNames[rows[k].trigger]);
            e.owner_device = rows[k].owner;
            out.push_back(e);
        }
        return out;
    }
    std::vector<std::uint64_t> tiles_per_device(int devices) {
        const int n = plbm_gpu_tiles(h_, nullptr, nullptr, nullptr, 0);
        std::vector<int32_t> coords(3 * size_t(std::max(n, 1))), owners(size_t(std::max(n, 1)));
        std::vector<int64_t> births(size_t(std::max(n, 1)));
        plbm_gpu_tiles(h_, coords.data(), owners.data(), births.data(), n);
        std::vector<std::uint64_t> per(size_t(devices), 0);
        for (int k = 0; k < n; ++k)
            if (owners[k] >= 0 && owners[k] < devices) ++per[size_t(owners[k])];
        return per;
    }
    void dump_field(const std::string& field, int comp, long it, const std::string& base, bool pgm) {
        if (plbm_gpu_dump_field(h_, field.c_str(), comp, it, base.c_str(), pgm ? 1 : 0) != 0)
            throw std::runtime_error("plbm_gpu_dump_field failed for " + base);
    }
    void set_capture(bool on) { plbm_gpu_set_capture(h_, on ? 1 : 0); }

  private:
    GpuDesc desc_;
    void* h_ = nullptr;
};

std::string snapshot_base(const std::string& field, int comp, long iteration) {
    char buf[96];  // engine.cpp:570-576
    std::snprintf(buf, sizeof buf, "%s_c%d_i%07ld", field.c_str(), comp, iteration);
    return buf;
}

// engine::run_scenario's output contract (engine.cpp:580-704) on GpuEngine.
engine::RunResult run(const iobench::ScenarioConfig& cfg, int device) {
    engine::RunResult res;
    res.output_dir = cfg.output_dir;
    namespace fs = std::filesystem;
    iobench::GeometryMask geom = cfg.geometry_path.empty()
                                     ? iobench::make_empty_geometry(cfg.domain[0], cfg.domain[1], cfg.domain[2])
                                     : iobench::load_geometry(cfg.geometry_path);
    sched::DeviceTopology topo =
        cfg.topology_path.empty() ? sched::make_full_p2p(cfg.devices) : sched::load_topology(cfg.topology_path);
    topo.weight_p2p = cfg.weight_p2p;
    topo.weight_staged = cfg.weight_staged;
    sched::validate_topology(topo);
    GpuEngine eng(cfg, geom, topo, device);
    const bool snapshots = cfg.snapshot_interval > 0;
    const bool want_psi =
        std::find(cfg.snapshot_fields.begin(), cfg.snapshot_fields.end(), "psi") != cfg.snapshot_fields.end();
    if (snapshots && want_psi) eng.set_capture(true);

    fs::create_directories(cfg.output_dir);
    if (snapshots) fs::create_directories(cfg.output_dir + "/snapshots");
    auto take_snapshot = [&](long iter) {
        for (const std::string& field : cfg.snapshot_fields)
            for (int c = 0; c < cfg.n_components(); ++c) {
                const std::string base = snapshot_base(field, c, iter);
                eng.dump_field(field, c, iter, cfg.output_dir + "/snapshots/" + base, cfg.snapshot_pgm);
                res.snapshot_bases.push_back("snapshots/" + base);
            }
    };
    if (snapshots) take_snapshot(0);

    const std::uint64_t bbox_cells = std::uint64_t(cfg.domain[0]) * cfg.domain[1] * cfg.domain[2];
    std::vector<iobench::ReportRow>& rows = res.rows;
    std::uint64_t peak_bytes = eng.counters().bytes_resident;
    double total_seconds = 0.0, win_seconds = 0.0;
    std::uint64_t win_updates = 0, win_steps = 0;
    std::uint64_t last_neg = 0, last_clamp = 0, last_sup = 0;
    auto flush_row = [&](long iter) {
        const plbm_counters c = eng.counters();
        iobench::ReportRow row;
        row.iteration = iter;
        row.tiles = c.tiles;
        row.active_cells = c.active_cells;
        row.bytes = {c.bytes[0], c.bytes[1], c.bytes[2]};
        row.window_seconds = win_seconds;
        row.window_mlups = iobench::mlups(win_updates, win_seconds);
        row.window_mlups_bbox = iobench::mlups(win_steps * bbox_cells, win_seconds);
        row.window_negative_populations = c.negative_populations - last_neg;
        row.window_psi_clamps = c.psi_clamps - last_clamp;
        row.window_suppressed_expansions = c.suppressed_expansions - last_sup;
        last_neg = c.negative_populations;
        last_clamp = c.psi_clamps;
        last_sup = c.suppressed_expansions;
        rows.push_back(row);
        win_seconds = 0.0;
        win_updates = 0;
        win_steps = 0;
    };
    bool aborted = false;
    std::string abort_context;
    for (long k = 1; k <= cfg.iterations; ++k) {
        const std::uint64_t before = eng.counters().cell_updates;
        const auto t0 = std::chrono::steady_clock::now();
        try {
            eng.step();
        } catch (const engine::EngineError& e) {
            aborted = true;
            abort_context = e.what();
            break;
        }
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const plbm_counters c = eng.counters();
        total_seconds += dt;
        win_seconds += dt;
        win_updates += c.cell_updates - before;
        ++win_steps;
        peak_bytes = std::max(peak_bytes, c.bytes_resident);
        if (k % cfg.report_interval == 0 || k == cfg.iterations) flush_row(k);
        if (snapshots && (k % cfg.snapshot_interval == 0 || k == cfg.iterations)) take_snapshot(k);
    }
    const plbm_counters c = eng.counters();
    if (aborted && win_steps > 0) flush_row(long(c.iteration));

    iobench::RunSummary& sum = res.summary;
    sum.name = cfg.name;
    sum.mode = cfg.mode == iobench::RunMode::Static ? "static" : "progressive";
    sum.policy = cfg.policy == sched::AssignPolicy::Simple ? "simple" : "optimized";
    sum.stencil = "D3Q19";
    sum.devices = topo.n_devices;
    sum.workers = cfg.workers > 0 ? cfg.workers : topo.n_devices;  // Engine(n_workers <= 0) = one per device
    sum.tile_extent = cfg.tile_extent;
    sum.domain = cfg.domain;
    sum.iterations = long(c.iteration);
    sum.total_cell_updates = c.cell_updates;
    sum.compute_seconds = total_seconds;
    sum.mlups = iobench::mlups(c.cell_updates, total_seconds);
    sum.mlups_bbox = iobench::mlups(std::uint64_t(c.iteration) * bbox_cells, total_seconds);
    sum.peak_resident_bytes = peak_bytes;
    sum.footprint_formula = mesh::tile_footprint_formula();
    sum.tiles_final = c.tiles;
    sum.active_cells_final = c.active_cells;
    sum.bytes = {c.bytes[0], c.bytes[1], c.bytes[2]};
    sum.negative_populations = c.negative_populations;
    sum.psi_clamps = c.psi_clamps;
    sum.suppressed_expansions = c.suppressed_expansions;
    sum.zero_rho_forcings = c.zero_rho_forcings;
    sum.per_device_tiles = eng.tiles_per_device(topo.n_devices);
    sum.status = aborted ? "aborted: " + abort_context : "completed";
    iobench::write_time_series_csv(rows, cfg.output_dir + "/time_series.csv");
    iobench::write_creation_log_csv(eng.creation_log(), cfg.output_dir + "/creation_log.csv");
    iobench::write_summary_json(sum, cfg.output_dir + "/summary.json");
    std::printf("%s: %ld iterations, %llu cell updates, %.3f s, %.1f MLUPS -> %s\n", cfg.name.c_str(),
                sum.iterations, (unsigned long long)sum.total_cell_updates, total_seconds, sum.mlups,
                cfg.output_dir.c_str());
    res.aborted = aborted;
    res.abort_context = abort_context;
    return res;
}

// ---- compare mode (proj/src/cli.cpp:133-157) --------------------------------
// Both modes on the GPU engine under <out>/static and <out>/progressive, the
// max |a - b| of every snapshot pair, and the joined compare.csv /
// compare_summary.json in the reference's formats (cli.cpp:35-131).
struct PairDiff {
    std::string base;
    double max_abs;
};

double max_abs_diff(const std::string& a_dir, const std::string& b_dir, const std::string& base) {
    const std::vector<double> a = iobench::read_raw(a_dir + "/" + base + ".raw");
    const std::vector<double> b = iobench::read_raw(b_dir + "/" + base + ".raw");
    if (a.size() != b.size()) throw std::runtime_error("compare: snapshot size mismatch at " + base);
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

std::string fmt(const char* f, double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, f, v);
    return buf;
}

void write_compare_csv(const iobench::ScenarioConfig& cfg, const engine::RunResult& st,
                       const engine::RunResult& pr, const std::vector<PairDiff>& diffs, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + path);
    const std::uint64_t fp =
        mesh::tile_footprint_bytes(cfg.tile_extent, cfg.three_d(), cfg.n_components(), cfg.three_d() ? 19 : 9);
    std::map<long, double> at;  // snapshot iteration ("..._i<iter>") -> max over fields and components
    for (const PairDiff& d : diffs) {
        const long it = std::stol(d.base.substr(d.base.rfind("_i") + 2));
        auto [e, fresh] = at.try_emplace(it, d.max_abs);
        if (!fresh) e->second = std::max(e->second, d.max_abs);
    }
    out << "iteration";
    for (const std::string side : {"static", "progressive"})
        for (const char* col : {"_tiles", "_active_cells", "_resident_bytes", "_bytes_intra", "_bytes_p2p",
                                "_bytes_staged", "_window_mlups", "_window_mlups_bbox"})
            out << ',' << side << col;
    out << ",field_diff_max\n";
    for (size_t i = 0; i < std::min(st.rows.size(), pr.rows.size()); ++i) {
        out << st.rows[i].iteration;
        for (const iobench::ReportRow* r : {&st.rows[i], &pr.rows[i]})
            out << ',' << r->tiles << ',' << r->active_cells << ',' << r->tiles * fp << ',' << r->bytes[0] << ','
                << r->bytes[1] << ',' << r->bytes[2] << fmt(",%.6g", r->window_mlups)
                << fmt(",%.6g", r->window_mlups_bbox);
        const auto e = at.find(st.rows[i].iteration);
        out << (e == at.end() ? std::string(",") : fmt(",%.17g", e->second)) << '\n';
    }
}

void write_compare_summary(const iobench::ScenarioConfig& cfg, const engine::RunResult& st,
                           const engine::RunResult& pr, const std::vector<PairDiff>& diffs, double dmax,
                           const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + path);
    char buf[512];
    out << "{\n  \"scenario\": \"" << cfg.name << "\",\n";
    for (const auto* side : {&st, &pr}) {
        const iobench::RunSummary& s = side->summary;
        std::snprintf(buf, sizeof buf,
                      "  \"%s\": {\"status\": \"%s\", \"iterations\": %ld, \"tiles_final\": %llu, "
                      "\"peak_resident_bytes\": %llu, \"mlups\": %.6g, \"mlups_bbox\": %.6g, "
                      "\"bytes_intra\": %llu, \"bytes_p2p\": %llu, \"bytes_staged\": %llu},\n",
                      side == &st ? "static" : "progressive", s.status.c_str(), s.iterations,
                      (unsigned long long)s.tiles_final, (unsigned long long)s.peak_resident_bytes, s.mlups,
                      s.mlups_bbox, (unsigned long long)s.bytes[0], (unsigned long long)s.bytes[1],
                      (unsigned long long)s.bytes[2]);
        out << buf;
    }
    const double ratio = st.summary.peak_resident_bytes ? double(pr.summary.peak_resident_bytes) /
                                                              double(st.summary.peak_resident_bytes)
                                                        : 0.0;
    out << fmt("  \"peak_bytes_ratio\": %.6g,\n", ratio) << "  \"snapshot_diffs\": [";
    for (size_t i = 0; i < diffs.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%s{\"base\": \"%s\", \"max\": %.17g}", i ? ", " : "",
                      diffs[i].base.c_str(), diffs[i].max_abs);
        out << buf;
    }
    out << "],\n" << fmt("  \"field_diff_max\": %.17g\n", dmax) << "}\n";
}

int compare(const iobench::ScenarioConfig& cfg, int device) {
    iobench::ScenarioConfig sc = cfg, pc = cfg;
    sc.mode = iobench::RunMode::Static;
    sc.output_dir = cfg.output_dir + "/static";
    pc.mode = iobench::RunMode::Progressive;
    pc.output_dir = cfg.output_dir + "/progressive";
    const engine::RunResult st = run(sc, device);
    const engine::RunResult pr = run(pc, device);
    std::vector<PairDiff> diffs;
    double dmax = 0.0;
    for (const std::string& base : pr.snapshot_bases) {
        diffs.push_back({base, max_abs_diff(sc.output_dir, pc.output_dir, base)});
        dmax = std::max(dmax, diffs.back().max_abs);
    }
    write_compare_csv(cfg, st, pr, diffs, cfg.output_dir + "/compare.csv");
    write_compare_summary(cfg, st, pr, diffs, dmax, cfg.output_dir + "/compare_summary.json");
    std::printf("compare: max field diff over %zu snapshots %.3g -> %s\n", diffs.size(), dmax,
                cfg.output_dir.c_str());
    return (st.aborted || pr.aborted) ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <scenario.toml> [--output DIR] [--iterations N] [--device N] [--compare 1]\n",
                     argv[0]);
        return 2;
    }
    try {
        iobench::ScenarioConfig cfg = iobench::load_config(argv[1]);
        int device = 0;
        bool cmp = false;
        for (int k = 2; k + 1 < argc; k += 2) {
            const std::string opt = argv[k];
            if (opt == "--output") cfg.output_dir = argv[k + 1];
            else if (opt == "--iterations") cfg.iterations = std::atol(argv[k + 1]);
            else if (opt == "--device") device = std::atoi(argv[k + 1]);
            else if (opt == "--compare") cmp = std::atoi(argv[k + 1]) != 0;
            else throw std::runtime_error("unknown option " + opt);
        }
        iobench::validate_config(cfg);
        if (cmp) return compare(cfg, device);
        return run(cfg, device).aborted ? 1 : 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "plbm_gpu_run: %s\n", e.what());
        return 2;
    }
}
