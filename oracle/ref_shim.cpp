// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" wrapper around the UNMODIFIED reference engine
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libplbm_ref.so).  It exposes the same plain-C surface as the
// oracle restatement (oracle/plbm_oracle.c) and the B200 engine
// (include/plbm_gpu.h) so the tests can drive all three with one
// plbm_scenario_desc and compare bit for bit.
//
// Mapping onto the reference:
//   plbm_ref_create  -> iobench::ScenarioConfig + engine::make_state + Engine
//                       (proj/src/engine.cpp:91-161, 530-533)
//   plbm_ref_step    -> Engine::step() n times (proj/src/engine.cpp:537-563)
//   plbm_ref_read_tile / counters / creation_log -> the state callers read
//                       between steps (SURVEY §8b "State read by callers").
#include "plbm/cli.hpp"
#include "plbm/dump.hpp"
#include "plbm/engine.hpp"
#include "plbm/scenario.hpp"
#include "plbm/kernels.hpp"
#include "plbm/physics.hpp"
#include "plbm/geometry.hpp"
#include "plbm/topology.hpp"

#include "plbm_scenario.h"

#include <array>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <string>
#include <unistd.h>

using namespace plbm;

namespace {

struct RefHandle {
    std::unique_ptr<engine::SimulationState> st;
    std::unique_ptr<engine::Engine> eng;
    std::string tmpdir;
    std::array<int, 3> domain{};
};

void set_err(plbm_error* e, int code, const std::string& msg) {
    if (!e) return;
    std::memset(e, 0, sizeof *e);
    e->code = code;
    std::snprintf(e->message, sizeof e->message, "%s", msg.c_str());
}

iobench::ScenarioConfig to_config(const plbm_scenario_desc* d,
                                  const std::string& tmpdir) {
    iobench::ScenarioConfig cfg;
    cfg.name = "shim";
    cfg.stencil = lattice::StencilKind::D3Q19;
    cfg.domain = {d->domain[0], d->domain[1], d->domain[2]};
    cfg.tile_extent = d->tile_extent;
    cfg.mode = d->mode == PLBM_MODE_STATIC ? iobench::RunMode::Static
                                           : iobench::RunMode::Progressive;
    cfg.iterations = 1;
    cfg.threshold = d->threshold;
    cfg.devices = d->devices;
    cfg.policy = d->policy == PLBM_POLICY_SIMPLE ? sched::AssignPolicy::Simple
                                                 : sched::AssignPolicy::Optimized;
    cfg.weight_p2p = d->weight_p2p;
    cfg.weight_staged = d->weight_staged;
    for (int a = 0; a < 3; ++a)
        cfg.boundary[a] = d->periodic[a] ? iobench::BoundaryKind::Periodic
                                         : iobench::BoundaryKind::Ambient;
    const int n = d->n_components;
    for (int c = 0; c < n; ++c) {
        const plbm_component_desc& s = d->components[c];
        physics::ComponentParams p;
        p.tau = s.tau;
        p.rho_ambient = s.rho_ambient;
        p.g_self = s.g_self;
        p.beta = s.beta;
        p.gravity = {s.gravity[0], s.gravity[1], s.gravity[2]};
        p.eos.a = s.a;
        p.eos.b = s.b;
        p.eos.R = s.R;
        p.eos.T = s.T;
        p.eos.Tc = s.Tc;
        p.eos.omega = s.omega;
        cfg.components.push_back(p);
    }
    cfg.coupling.n = n;
    cfg.coupling.g.assign(std::size_t(n) * n, 0.0);
    if (d->coupling)
        for (int k = 0; k < n * n; ++k) cfg.coupling.g[k] = d->coupling[k];
    for (int k = 0; k < d->n_seeds; ++k) {
        const plbm_seed_desc& s = d->seeds[k];
        iobench::SeedRegion r;
        r.shape = s.shape == PLBM_SEED_SPHERE ? iobench::SeedRegion::Shape::Sphere
                                              : iobench::SeedRegion::Shape::Box;
        r.component = s.component;
        for (int a = 0; a < 3; ++a) {
            r.box_min[a] = s.box_min[a];
            r.box_max[a] = s.box_max[a];
            r.center[a] = s.center[a];
            r.velocity[a] = s.velocity[a];
        }
        r.radius = s.radius;
        r.rho = s.rho;
        cfg.seeds.push_back(r);
    }
    if (d->geometry) {
        iobench::GeometryMask m = iobench::make_empty_geometry(
            d->domain[0], d->domain[1], d->domain[2]);
        std::memcpy(m.solid.data(), d->geometry, m.solid.size());
        const std::string path = tmpdir + "/geometry.lbmgeo";
        iobench::save_geometry(m, path);
        cfg.geometry_path = path;
    }
    if (d->p2p) {
        const std::string path = tmpdir + "/topology.txt";
        std::ofstream out(path);
        out << d->devices << "\n";
        for (int i = 0; i < d->devices; ++i) {
            for (int j = 0; j < d->devices; ++j)
                out << int(d->p2p[i * d->devices + j]) << (j + 1 < d->devices ? " " : "");
            out << "\n";
        }
        cfg.topology_path = path;
    }
    return cfg;
}

} // namespace

extern "C" {

void* plbm_ref_create(const plbm_scenario_desc* d, int workers,
                      plbm_error* err) {
    set_err(err, 0, "");
    char tmpl[] = "/tmp/plbm_ref_XXXXXX";
    const char* dir = mkdtemp(tmpl);
    if (!dir) {
        set_err(err, 3, "mkdtemp failed");
        return nullptr;
    }
    auto h = std::make_unique<RefHandle>();
    h->tmpdir = dir;
    try {
        const auto cfg = to_config(d, h->tmpdir);
        h->domain = cfg.domain;
        h->st = engine::make_state(cfg);
        h->eng = std::make_unique<engine::Engine>(*h->st, workers);
    } catch (const std::exception& e) {
        set_err(err, 2, e.what());
        std::filesystem::remove_all(h->tmpdir);
        return nullptr;
    }
    return h.release();
}

int plbm_ref_step(void* hp, int n, plbm_error* err) {
    auto* h = static_cast<RefHandle*>(hp);
    set_err(err, 0, "");
    for (int k = 0; k < n; ++k) {
        try {
            h->eng->step();
        } catch (const engine::EngineError& e) {
            set_err(err, 1, e.what());
            if (err) {
                err->tile[0] = e.tile.x;
                err->tile[1] = e.tile.y;
                err->tile[2] = e.tile.z;
                err->iteration = e.iteration;
                std::snprintf(err->phase, sizeof err->phase, "%s",
                              e.phase.c_str());
            }
            return 1;
        } catch (const std::exception& e) {
            set_err(err, 2, e.what());
            return 2;
        }
    }
    return 0;
}

void plbm_ref_counters(void* hp, plbm_counters* out) {
    auto* h = static_cast<RefHandle*>(hp);
    const engine::SimulationState& s = *h->st;
    std::memset(out, 0, sizeof *out);
    out->iteration = s.iteration;
    out->cell_updates = s.cell_updates;
    out->negative_populations = s.diag.negative_populations.load();
    out->psi_clamps = s.diag.psi_clamps.load();
    out->zero_rho_forcings = s.diag.zero_rho_forcings.load();
    out->suppressed_expansions = s.map.suppressed_expansions();
    const auto b = s.topo.byte_totals();
    for (int k = 0; k < 3; ++k) out->bytes[k] = b[k];
    const auto rep = s.map.active_report();
    out->tiles = rep.tiles;
    out->active_cells = rep.active_cells;
    out->bytes_resident = rep.bytes_resident;
}

// Tiles in map (coordinate) order.
int plbm_ref_tiles(void* hp, int32_t* coords, int32_t* owners,
                   int64_t* births, int max) {
    auto* h = static_cast<RefHandle*>(hp);
    int k = 0;
    for (const auto& [c, tp] : h->st->map.tiles()) {
        if (k < max) {
            if (coords) {
                coords[3 * k] = c.x;
                coords[3 * k + 1] = c.y;
                coords[3 * k + 2] = c.z;
            }
            if (owners) owners[k] = tp->owner_device;
            if (births) births[k] = tp->birth_iteration;
        }
        ++k;
    }
    return k;
}

int plbm_ref_read_tile(void* hp, const int32_t* coords, int comp, int field,
                       double* out) {
    auto* h = static_cast<RefHandle*>(hp);
    const mesh::Tile* t = h->st->map.at({coords[0], coords[1], coords[2]});
    if (!t) return -1;
    if (comp < 0 || comp >= int(t->comp.size())) return -2;
    const mesh::ComponentState& cs = t->comp[std::size_t(comp)];
    const int e = t->extent;
    const std::size_t n = std::size_t(e) * e * e;
    auto gather = [&](const double* src, double* dst) {
        for (int z = 0; z < e; ++z)
            for (int y = 0; y < e; ++y)
                for (int x = 0; x < e; ++x)
                    dst[std::size_t(x) + std::size_t(e) * (y + std::size_t(e) * z)] =
                        src[t->gidx(x, y, z)];
    };
    switch (field) {
    case PLBM_FIELD_F:
        for (int i = 0; i < 19; ++i)
            gather(t->f_read(comp) + std::size_t(i) * t->gcells, out + i * n);
        return 0;
    case PLBM_FIELD_RHO: gather(cs.rho.data(), out); return 0;
    case PLBM_FIELD_UX: gather(cs.ux.data(), out); return 0;
    case PLBM_FIELD_UY: gather(cs.uy.data(), out); return 0;
    case PLBM_FIELD_UZ: gather(cs.uz.data(), out); return 0;
    case PLBM_FIELD_PUX: gather(cs.pux.data(), out); return 0;
    case PLBM_FIELD_PUY: gather(cs.puy.data(), out); return 0;
    case PLBM_FIELD_PUZ: gather(cs.puz.data(), out); return 0;
    case PLBM_FIELD_PSI: gather(cs.psi.data(), out); return 0;
    default: return -3;
    }
}

int plbm_ref_creation_log(void* hp, plbm_creation_event* out, int max) {
    auto* h = static_cast<RefHandle*>(hp);
    const auto& log = h->st->map.creation_log();
    for (int k = 0; k < int(log.size()) && k < max; ++k) {
        const auto& ev = log[std::size_t(k)];
        out[k].iteration = ev.iteration;
        out[k].coords[0] = ev.coords.x;
        out[k].coords[1] = ev.coords.y;
        out[k].coords[2] = ev.coords.z;
        out[k].trigger = -1;
        for (int f = 0; f < 6; ++f)
            if (ev.trigger == mesh::kFaceNames[f]) out[k].trigger = f;
        out[k].owner = ev.owner_device;
        out[k].pad = 0;
    }
    return int(log.size());
}

// Overwrites one post-stream population (tests: NaN poisoning,
// proj/tests/test_engine.cpp:284-310).
int plbm_ref_poke_f(void* hp, const int32_t* coords, int comp, int i,
                    const int32_t* local, double v) {
    auto* h = static_cast<RefHandle*>(hp);
    mesh::Tile* t = h->st->map.at({coords[0], coords[1], coords[2]});
    if (!t) return -1;
    t->f_read(comp)[std::size_t(i) * t->gcells +
                    t->gidx(local[0], local[1], local[2])] = v;
    return 0;
}

void plbm_ref_destroy(void* hp) {
    auto* h = static_cast<RefHandle*>(hp);
    if (!h) return;
    h->eng.reset();
    h->st.reset();
    std::filesystem::remove_all(h->tmpdir);
    delete h;
}


// ---- known-answer entry points straight into the reference's functions
namespace {
physics::ComponentParams to_params(const plbm_component_desc* c) {
    physics::ComponentParams p;
    p.tau = c->tau;
    p.rho_ambient = c->rho_ambient;
    p.g_self = c->g_self;
    p.beta = c->beta;
    p.gravity = {c->gravity[0], c->gravity[1], c->gravity[2]};
    p.eos.a = c->a;
    p.eos.b = c->b;
    p.eos.R = c->R;
    p.eos.T = c->T;
    p.eos.Tc = c->Tc;
    p.eos.omega = c->omega;
    return p;
}
const lattice::Stencil& st3() {
    static const lattice::Stencil s = lattice::make_stencil(lattice::StencilKind::D3Q19);
    return s;
}
}  // namespace

double plbm_ref_kat_pr_pressure(double rho, const plbm_component_desc* c, int* pole) {
    *pole = 0;
    try {
        return physics::pr_pressure(rho, to_params(c));
    } catch (const std::domain_error&) {
        *pole = 1;
        return 0.0;
    }
}
double plbm_ref_kat_psi(double rho, double press, double g_self, int* clamped) {
    std::uint64_t n = 0;
    const double v = physics::pseudo_potential(rho, press, g_self, st3().cs2, &n);
    *clamped = int(n);
    return v;
}
void plbm_ref_kat_equilibrium(double rho, const double* u, double* out) {
    lattice::equilibrium(rho, u, st3(), out);
}
void plbm_ref_kat_moments(const double* f, double* rho, double* u) {
    lattice::moments(f, st3(), *rho, u);
}
void plbm_ref_kat_intra_force(const double* psi, long cell, const long* stride,
                              const plbm_component_desc* c, double* F) {
    const auto r = physics::intra_force(psi, cell, stride, to_params(c), st3());
    F[0] = r[0]; F[1] = r[1]; F[2] = r[2];
}
void plbm_ref_kat_inter_force(double psi_self, const double* psi_other, long cell,
                              const long* stride, double g, double* F) {
    const auto r = physics::inter_force(psi_self, psi_other, cell, stride, g, st3());
    F[0] = r[0]; F[1] = r[1]; F[2] = r[2];
}
void plbm_ref_kat_stencil(int* e, double* w, int* opp) {
    const auto& s = st3();
    for (int i = 0; i < 19; ++i) {
        for (int a = 0; a < 3; ++a) e[3 * i + a] = s.e[i][a];
        w[i] = s.w[i];
        opp[i] = s.opp[i];
    }
}

// iobench::dump_field on the reference state (proj/src/dump.cpp:59-125).
int plbm_ref_dump_field(void* hp, const char* field, int comp, long iteration,
                        const char* base_path, int with_pgm) {
    auto* h = static_cast<RefHandle*>(hp);
    try {
        iobench::dump_field(h->st->map, h->domain, field, comp, iteration,
                            base_path, with_pgm != 0);
    } catch (const std::exception&) {
        return -5;
    }
    return 0;
}

// The reference driver itself, engine::run_scenario (proj/src/engine.cpp:
// 580-704): time_series.csv, creation_log.csv, summary.json and snapshots
// under output_dir.  fields: comma-separated snapshot field names.
int plbm_ref_run_scenario(const plbm_scenario_desc* d, int workers,
                          long iterations, int report_interval,
                          int snapshot_interval, const char* fields,
                          int with_pgm, const char* name,
                          const char* output_dir) {
    char tmpl[] = "/tmp/plbm_refrun_XXXXXX";
    const char* dir = mkdtemp(tmpl);
    if (!dir) return -3;
    int rc = 0;
    try {
        auto cfg = to_config(d, dir);
        cfg.name = name;
        cfg.workers = workers;
        cfg.iterations = iterations;
        cfg.report_interval = report_interval;
        cfg.snapshot_interval = snapshot_interval;
        cfg.snapshot_pgm = with_pgm != 0;
        cfg.output_dir = output_dir;
        cfg.snapshot_fields.clear();
        std::string f = fields ? fields : "";
        size_t p = 0;
        while (p < f.size()) {
            const size_t q = f.find(',', p);
            cfg.snapshot_fields.push_back(f.substr(p, q == std::string::npos ? std::string::npos : q - p));
            if (q == std::string::npos) break;
            p = q + 1;
        }
        engine::run_scenario(cfg);
    } catch (const std::exception&) {
        rc = -2;
    }
    std::filesystem::remove_all(dir);
    return rc;
}

// The reference's CLI `run` path without CLI11: iobench::load_config on a
// scenario TOML, the output directory overridden, engine::run_scenario.
int plbm_ref_run_toml(const char* path, const char* output_dir) {
    try {
        auto cfg = iobench::load_config(path);
        cfg.output_dir = output_dir;
        engine::run_scenario(cfg);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "plbm_ref_run_toml: %s\n", e.what());
        return -2;
    }
    return 0;
}

// The reference's compare mode (proj/src/cli.cpp:133-157): the scenario in
// both modes under <output_dir>/{static,progressive}, every snapshot pair
// diffed, compare.csv and compare_summary.json written.
int plbm_ref_run_compare_toml(const char* path, const char* output_dir) {
    try {
        auto cfg = iobench::load_config(path);
        cfg.output_dir = output_dir;
        iobench::run_compare(cfg);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "plbm_ref_run_compare_toml: %s\n", e.what());
        return -2;
    }
    return 0;
}

} // extern "C"
