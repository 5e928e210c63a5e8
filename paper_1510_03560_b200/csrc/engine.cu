// engine.cu — host side of the B200 step loop behind the C-ABI (plbm_gpu.h).
//
// The host keeps only METADATA (the reference's TileMap / AssignmentState /
// DeviceTopology counters without any field buffer): tile coordinates, owners,
// creation log, per-device counts, byte classes.  All field state lives in
// device block pools (kernels.cuh).  Expansion (proj/src/tilemap.cpp:220-266)
// and placement (proj/src/assign.cpp:8-38, engine.cpp:30-41) run on this
// mirror from the per-face trigger bits the device criterion produced.
//
// Multi-GPU (one process per GPU): every rank runs the same deterministic
// mirror, so global slot ids, owners and per-rank local pool indices agree on
// all ranks without communication.  Tile owner `o` (assign_device) lives on
// rank `o % world` (the reference's worker mapping, engine.cpp:214-218).  Each
// rank allocates a pool only for its own tiles; the per-slot pointer tables
// point remote slots at the owner's pool (CUDA IPC, read over NVLink inside
// the fused kernel).  Between step_begin and step_end the caller merges the
// trigger bits of all ranks (one small all-reduce), which also orders the
// ranks' double-buffered reads and writes.
#include "kernels.cuh"
#include "dispatch.cuh"
#include "expand.cuh"
#include "plbm_gpu.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <chrono>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <string>
#include <type_traits>
#include <vector>

namespace plbm {

namespace {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

// ---- host restatements used to build the device constants (same IEEE ops,
// compiled with -ffp-contract=off) -------------------------------------------

// proj/include/plbm/kernels.hpp:17-28 (literal loop form)
void host_equilibrium(double rho, const double u[3], double* out) {
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double inv_cs2 = 1.0 / PLBM_CS2;
    for (int i = 0; i < Q; ++i) {
        const double eu = double(ex_(i)) * u[0] + double(ey_(i)) * u[1] + double(ez_(i)) * u[2];
        out[i] = w_(i) * rho *
                 (1.0 + eu * inv_cs2 + 0.5 * eu * eu * inv_cs2 * inv_cs2 - 0.5 * uu * inv_cs2);
    }
}

// theta(T) of proj/src/physics.cpp:16-21
double host_theta(const plbm_component_desc& e) {
    double theta = 1.0;
    if (e.Tc > 0.0) {
        const double kappa = 0.37464 + 1.54226 * e.omega - 0.26992 * e.omega * e.omega;
        const double root = 1.0 + kappa * (1.0 - std::sqrt(e.T / e.Tc));
        theta = root * root;
    }
    return theta;
}

// proj/src/physics.cpp:12-27
double host_pr_pressure(double rho, const plbm_component_desc& e) {
    if (e.b * rho >= 1.0) throw std::domain_error("pr_pressure: b*rho >= 1 (EOS pole)");
    const double theta = host_theta(e);
    const double ideal = rho * e.R * e.T / (1.0 - e.b * rho);
    const double attr = e.a * theta * rho * rho / (1.0 + 2.0 * e.b * rho - e.b * e.b * rho * rho);
    return ideal - attr;
}

// proj/src/physics.cpp:34-42
double host_psi(double rho, double press, double g_self) {
    const double radicand = 2.0 * (press - PLBM_CS2 * rho) / (PLBM_CS2 * g_self);
    if (radicand < 0.0) return 0.0;
    return std::sqrt(radicand);
}

template <class T>
T* dmalloc(size_t n) {
    T* p = nullptr;
    if (n) CK(cudaMalloc(&p, n * sizeof(T)));
    return p;
}

// Test hook (ordering stress of the multi-rank protocol):
// PLBM_TEST_RANK_DELAY_US="<rank>:<us>" makes that rank spin on the device
// before every step's fused kernel, so it trails its peers.
__global__ void k_spin(unsigned long long ns) {
    const unsigned long long t0 = global_ns();
    while (global_ns() - t0 < ns) __nanosleep(1000);
}

Kernels pick_kernels(int E, int C, bool nopsi) {
#ifdef PLBM_ONLY_E32C2  // experiment builds link inst_e32.cu only
    if (E == 32) return pick_kernels_e32(C, nopsi);
    throw std::invalid_argument("PLBM_ONLY_E32C2 build: E = 32, C = 2 only");
#else
    switch (E) {
    case 8: return pick_kernels_e8(C, nopsi);
    case 16: return pick_kernels_e16(C, nopsi);
    case 32: return pick_kernels_e32(C, nopsi);
    case 64: return pick_kernels_e64(C, nopsi);
    default: throw std::invalid_argument("tile_extent must be 8, 16, 32 or 64 on the GPU path");
    }
#endif
}

struct Coord {
    int x, y, z;
    bool operator<(const Coord& o) const {
        if (x != o.x) return x < o.x;
        if (y != o.y) return y < o.y;
        return z < o.z;
    }
    bool operator==(const Coord& o) const { return x == o.x && y == o.y && z == o.z; }
    bool operator!=(const Coord& o) const { return !(*this == o); }
};

struct SlotInfo {
    Coord c{};
    int owner = -1;  // assign_device result (simulated device)
    int rank = -1;   // GPU rank holding the fields (owner % world)
    int local = -1;  // index in the owner rank's pool
    long birth = 0;
    size_t log_index = 0;
    int fluid = 0;
    bool has_solid = false;
    bool device_sliced = false;  // mask written by k_slice, not uploaded from h_solid_
};

struct LogRow {
    long iteration;
    Coord c;
    int trigger;
    int owner;
};

}  // namespace

class Engine {
  public:
    Engine(const plbm_scenario_desc& d, int device, int rank, int world, int storage = PLBM_STORAGE_AB) {
        aa_ = storage == PLBM_STORAGE_AA;
        init(d, device, rank, world);
    }
    ~Engine() { release(); }

    int prepare();
    int step(int n, plbm_error* err);
    int step_begin(plbm_error* err);
    int step_main(plbm_error* err);
    int step_face();
    int step_end(const uint8_t* merged, plbm_error* err);
    int step_speculative(int n, plbm_error* err);
    void enqueue_step(long it);
    void host_expand(const uint8_t* merged, long it);
    void counters(plbm_counters* out);
    int tiles(int32_t* coords, int32_t* owners, int64_t* births, int max) const;
    int read_tile(const int32_t* coords, int comp, int field, double* out);
    int gather_field(const char* field, int comp, double* grid);
    int dump_field(const char* field, int comp, long iteration, const char* base, int with_pgm);
    int creation_log(plbm_creation_event* out, int max) const;
    int set_capture(bool on);
    int poke_f(const int32_t* coords, int comp, int i, const int32_t* local, double v);
    void set_profiling(bool on) { profiling_ = on; }
    int set_variant(int v) {
        if (aa_) {  // A-A storage: the cluster split (0 default, 20 / 26 / 27); +200 = no xcol side buffers
            const int b = v % 100;
            if (!(v >= 0 && v < 300 && v / 100 != 1 && (b == 0 || b == 20 || b == 26 || b == 27))) return -1;
            if (b == 20 && !K_.main_aa[0]) return -1;  // no whole-tile cluster at this shape
            no_xcol_ = v >= 200;
            variant_ = b;
            return 0;
        }
        const int base = v % 100;
        const bool ok = v >= 0 && v < 400 && (base == 0 || base == 1 || base == 20 || base == 21 || base == 22 ||
                                              base == 26 || base == 27
#ifdef PLBM_PROBES
                                              || base == 24
#endif
                                              );
        if (!ok) return -1;  // unknown (or probe-only) variant: keep the current one
        variant_ = base;
        fuse_ = (v / 100) & 1;     // +100: face pass in the fused kernel's tail (A/B)
        no_xcol_ = (v / 200) & 1;  // +200: face pass reads x faces from the SoA block
        return 0;
    }
    plbm_kernel_stats stats();
    void reset_stats() {
        resolve_events();
        stats_ = plbm_kernel_stats{};
    }
    cudaStream_t stream() const { return stream_; }
    int trig_bytes() const { return int(trig_bytes_); }
    uint8_t* trig_device() const { return d_trig_; }
    int local_triggers(uint8_t* out, int n);
    void pool_pointers(void** f, void** pf) const {
        *f = d_pool_f_;
        *pf = d_pool_pf_;
    }
    int ipc_handles(void* out) const;
    int open_peer(int rank, const void* handles);
    int set_peer(int rank, void* pool_f, void* pool_pf);
    int set_peer_sync(int rank, void* sync);
    void* sync_block() const { return d_sync_; }
    int rank_of(const int32_t* coords) const;
    void exchange_bytes(uint64_t* out) const;
    int probe(uint64_t* out, int max) {
        if (!d_.probe) return 0;
        const int n = std::min(max, 3 * (cap_ + 1) * 16);
        CK(cudaMemcpy(out, d_.probe, size_t(n) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        return n / 3;
    }
    int sync() {
        CK(cudaStreamSynchronize(stream_));
        return 0;
    }

  private:
    // configuration
    int dev_ = 0, rank_ = 0, world_ = 1;
    int E_ = 0, C_ = 0, E3_ = 0, E2_ = 0;
    int dom_[3]{}, grid_[3]{}, periodic_[3]{};
    int mode_ = 0, devices_ = 1, policy_ = 1;
    double threshold_ = 0.0, w_p2p_ = 0.5, w_staged_ = 1.0;
    std::vector<uint8_t> p2p_;
    std::vector<plbm_component_desc> comps_;
    std::vector<double> coupling_;
    std::vector<plbm_seed_desc> seeds_;
    std::vector<uint8_t> geom_;
    uint64_t face_xfer_ = 0;
    bool nopsi_ = false;
    Kernels K_{};
    Params params_{};

    // host mirror (replicated on every rank)
    std::vector<int> grid_slot_;  // lin -> global slot or -1
    std::vector<SlotInfo> slots_;
    std::vector<int> free_slots_;
    std::vector<int> all_active_;   // global slots in coordinate order
    std::vector<int> active_;       // this rank's slots in coordinate order
    std::vector<int> next_local_;   // per rank: next pool index
    std::vector<LogRow> log_;
    std::vector<uint64_t> per_dev_;
    uint64_t suppressed_ = 0, active_cells_ = 0, local_cells_ = 0;
    uint64_t bytes_[3]{};
    uint64_t step_bytes_[3]{};
    long iteration_ = 0;
    uint64_t cell_updates_ = 0;
    bool any_gen_ = true;
    bool routes_differ_ = false;
    bool prepared_ = false;
    int phase_ = 0;  // 0 idle, 1 main queued, 2 face queued
    std::vector<uint8_t> h_mode_;
    std::vector<uint8_t> h_has_solid_;
    std::vector<int> h_coords_;
    std::vector<uint32_t> h_solid_;
    std::vector<int> h_lidx_;
    int cap_ = 0, amb_ = 0, lcap_ = 0;
    size_t per_slot_ = 0, per_pf_ = 0;
    size_t trig_bytes_ = 0;

    // device
    cudaStream_t stream_ = nullptr;
    Dev d_{};
    double* d_pool_f_ = nullptr;   // [2][lcap+1][per_slot]  (local index lcap = ambient)
    // One rank: the population pool is a reserved virtual address range whose
    // physical memory is mapped in granules only for the pool indices the
    // launches can reach (tiles + expansion headroom) and the ambient slot,
    // so the progressive mesh's footprint follows its active tiles (the
    // reference allocates a tile at creation, tilemap.cpp:83-175).
    bool vm_pool_ = false;
    CUdeviceptr vm_base_ = 0;
    size_t vm_size_ = 0, vm_gran_ = 0;
    std::vector<CUmemGenericAllocationHandle> vm_handles_;  // per granule (0 = unmapped)
    std::atomic<uint64_t> vm_mapped_{0}, vm_map_us_{0}, vm_wait_us_{0};
    // A mapper thread backs the pool ahead of the launches (target = the
    // slots asked for + a quarter), overlapping the driver's mapping work with
    // the steps; the launching thread waits only when it outruns the mapper.
    std::thread vm_thread_;
    mutable std::mutex vm_mu_;
    std::condition_variable vm_cv_;
    int vm_want_ = 0, vm_ready_ = 0;  // pool indices [0, n) asked for / backed
    bool vm_stop_ = false;
    std::string vm_err_;
    void vm_reserve(size_t bytes);
    void vm_map_range(size_t off, size_t len);
    void vm_mapper();
    void ensure_pool(int n_slots);  // pool indices [0, n_slots) backed (waits for the mapper)
    void vm_release();

  public:
    void memory(uint64_t* out) const {
        const uint64_t full = uint64_t(nbuf_) * per_slot_ * uint64_t(lcap_ + 1) * sizeof(double);
        out[0] = vm_pool_ ? vm_size_ : full;
        out[1] = vm_pool_ ? vm_mapped_.load() : full;
        out[2] = vm_pool_ ? vm_gran_ : 0;
        out[3] = vm_map_us_.load();   // mapper thread, microseconds
        out[4] = vm_wait_us_.load();  // launching thread waiting for it
    }

  private:
    double* d_pool_pf_ = nullptr;  // [2][lcap+1][per_pf]
    std::vector<double*> peer_f_, peer_pf_;  // pool bases per rank (self = own)
    std::vector<bool> peer_opened_;
    double** d_slot_f_[2]{};
    double** d_slot_pf_[2]{};
    int* d_route_[3]{};
    bool aa_ = false;  // A-A in-place population storage (one buffer)
    int nbuf_ = 2;
    int* d_lidx_ = nullptr;
    uint32_t* d_solid_ = nullptr;
    uint8_t* d_has_solid_ = nullptr;
    uint8_t* d_no_fluid_ = nullptr;  // [slot] the tile has no fluid cell (Dev::no_fluid)
    uint8_t* d_mode_ = nullptr;
    int* d_coords_ = nullptr;
    double* d_u_face_ = nullptr;
    uint8_t* d_trig_ = nullptr;   // [parity][trig_bytes_] inside d_sync_ (one parity on one rank)
    // Sync block (IPC-exported next to the pools): [0..7] barrier flag words
    // (slot r = the last epoch rank r reached), [8] error key, [9] merged
    // error key, [16..23] this rank's diagnostic counters by step parity
    // (snapshot at the step's second barrier), [24..] trigger bytes of both
    // step parities.
    static constexpr int SYNC_SNAP = 16, SYNC_TRIG = 24;
    unsigned long long* d_sync_ = nullptr;
    unsigned long long* d_gcnt_ = nullptr;  // job-wide diagnostics of the last device-checked step
    bool gcnt_valid_ = false;
    std::vector<unsigned long long*> peer_sync_;
    unsigned long long epoch_ = 0;  // rank barriers queued so far (identical on every rank)
    uint8_t* d_merged_ = nullptr;   // world > 1: merged trigger bytes of the last check
    int* d_all_active_ = nullptr;   // world > 1: every rank's slots (the expansion's map)
    int* d_nall_ = nullptr;
    void rank_barrier(long it, bool snapshot = false);
    void reset_err();
    unsigned long long* err_word() const { return world_ > 1 ? d_sync_ + 9 : d_err_; }
    // device-side expansion (one rank progressive, or any multi-rank run; expand.cuh)
    bool dev_expand_ = false;
    int* d_gslot_ = nullptr;
    unsigned long long* d_cand_ = nullptr;
    int* d_nactive_ = nullptr;
    int* d_next_slot_ = nullptr;
    int* d_next_local_ = nullptr;
    int* d_owner_ = nullptr;
    uint8_t* d_geomdev_ = nullptr;
    uint8_t* d_p2p_ = nullptr;
    unsigned long long* d_per_dev_ = nullptr;
    unsigned long long* d_acc_ = nullptr;  // cell_updates, bytes[3], active_cells, step_bytes[3]
    BirthRec* d_births_ = nullptr;
    int* d_nbirths_ = nullptr;
    int* d_post_flags_ = nullptr;
    int synced_births_ = 0;
    int launch_tiles_ = 0;
    void sync_births();
    // tiles the launches leave room for beyond the current map (births past
    // it go to the host); PLBM_EXPAND_HEADROOM overrides (tests)
    int expand_headroom() const {
        if (const char* h = std::getenv("PLBM_EXPAND_HEADROOM")) return std::max(0, std::atoi(h));
        return std::max(64, int(all_active_.size()) / 4);
    }
    void upload_expand_state(bool initial);
    ExpandDev expand_dev() const;
    void launch_check_expand(long it);
    uint8_t* d_bmask_ = nullptr;  // [slot] faces whose trigger would be a birth
    uint8_t* d_omask_ = nullptr;  // [slot] faces whose trigger is out of bounds (suppressed)
    int* d_halt_ = nullptr;       // sticky halt flag of the speculative step queue
    unsigned long long* h_cnt_ = nullptr;  // pinned landing area of counters(): CNT_N x 2 + 4
    int* h_flags_ = nullptr;      // pinned copies of the halt flag, one per queued step (+ birth
                                  // count at h_flags_[8 + k]: sync_births needs no round trip
                                  // when the retired steps had no births)
    int births_seen_ = -1;        // birth count of the last retired queued step (-1: unknown)
    cudaEvent_t flag_ev_[8] = {};
    int spec_depth_ = 3;          // steps queued ahead (1 = a host round trip every step)
    bool in_spec_ = false;        // a speculative queue is open (profiling events stay unresolved)
    bool post_pending_ = false;   // upload_expand_state left a k_post_main to the next step_main
    Poke* d_pokes_ = nullptr;     // test hook: f_in overrides for the next step
    std::vector<Poke> pokes_;
    int* d_dep_cnt_ = nullptr;   // fused face pass: per-slot completion counts
    int* d_dep_need_ = nullptr;  // 1 + active geometric neighbours
    int* d_geo_ = nullptr;       // [slot][18] active geometric neighbour or -1
    bool face_fused_ = false;    // the last k_main ran the face pass itself
    double* d_capture_ = nullptr;
    uint8_t* d_suspect_ = nullptr;  // [slot] P5 screen marks (k_main* -> k_p5)
    unsigned* d_susp_any_ = nullptr;  // [2] per step parity: a tile was marked
    unsigned long long* d_cnt_ = nullptr;
    unsigned long long* d_err_ = nullptr;
    int* d_active_ = nullptr;
    int* d_scratch_slots_ = nullptr;
    double* d_readback_ = nullptr;
    int cur_ = 0;  // buffer holding the latest f_post (or unused before step 1)
    int solid_words_ = 0;
    bool profiling_ = false;
    int variant_ = 0;
    int mid_faces_ = 0;
    int split_ = 1;  // clusters per tile of the default k_main_pc (PLBM_SPLIT, 1 / 2 / 4)
    bool fuse_ = false, no_xcol_ = false;
    plbm_kernel_stats stats_{};
    struct EvPair {
        cudaEvent_t a = nullptr, b = nullptr;
        int kind = 0;
        uint64_t cells = 0;
    };
    std::vector<EvPair> ev_pool_;
    size_t ev_used_ = 0;

    void init(const plbm_scenario_desc& d, int device, int rank, int world);
    void release();
    size_t lin(const Coord& c) const { return (size_t(c.x) * grid_[1] + c.y) * grid_[2] + c.z; }
    int slot_at(const Coord& c) const { return grid_slot_[lin(c)]; }
    bool neighbor_coords(const Coord& from, int face, Coord& out) const;
    int create_tile(const Coord& c, long iteration, int trigger, bool slice = true);
    void slice_on_device(const std::vector<int>& slots);
    void assign_owner(int slot);
    int classify(int a, int b) const {
        if (a == b) return 0;
        return p2p_[size_t(a) * devices_ + b] ? 1 : 2;
    }
    void compute_routes(int slot, int* out) const;
    void upload_map(const std::vector<int>& new_slots, bool initial);
    void upload_pointers();
    void recompute_step_bytes();
    void launch_face(int src, int flags, long iter);
    void launch_p5(long iter);
    void launch_main(long iter);
    void expand(const std::vector<std::pair<Coord, int>>& triggers, long iteration,
                std::vector<int>& created);
    void check_error(plbm_error* err, bool& failed);
    long err_it_ = 0;     // iteration of the last error check_error decoded
    bool err_p5_ = false; // ... and whether it was a P5 error (that step's exchange bytes count)
    EvPair& next_event(int kind, uint64_t cells);
    void resolve_events();
    bool peers_ready() const {
        for (int r = 0; r < world_; ++r)
            if (!peer_f_[r] || !peer_sync_[r]) return false;
        return true;
    }
    int launch_bound() const;
};

// ---------------------------------------------------------------------------

void Engine::init(const plbm_scenario_desc& d, int device, int rank, int world) {
    dev_ = device;
    rank_ = rank;
    world_ = world;
    if (world_ < 1 || rank_ < 0 || rank_ >= world_) throw std::invalid_argument("bad rank/world");
    E_ = d.tile_extent;
    C_ = d.n_components;
    E2_ = E_ * E_;
    E3_ = E_ * E_ * E_;
    if (C_ < 1 || C_ > 3) throw std::invalid_argument("n_components must be 1..3");
    if (d.n_seeds < 0 || d.n_seeds > MAX_SEEDS) throw std::invalid_argument("too many seeds");
    for (int a = 0; a < 3; ++a) {
        dom_[a] = d.domain[a];
        periodic_[a] = d.periodic[a] ? 1 : 0;
        if (E_ < 4 || dom_[a] < 1 || dom_[a] % E_)
            throw std::invalid_argument("domain axis not divisible by tile_extent");
        grid_[a] = dom_[a] / E_;
    }
    mode_ = d.mode;
    threshold_ = d.threshold;
    devices_ = d.devices;
    policy_ = d.policy;
    w_p2p_ = d.weight_p2p;
    w_staged_ = d.weight_staged;
    if (devices_ < 1) throw std::invalid_argument("devices must be >= 1");
    p2p_.assign(size_t(devices_) * devices_, 1);
    if (d.p2p) std::memcpy(p2p_.data(), d.p2p, p2p_.size());
    comps_.assign(d.components, d.components + C_);
    coupling_.assign(size_t(C_) * C_, 0.0);
    if (d.coupling) std::memcpy(coupling_.data(), d.coupling, coupling_.size() * sizeof(double));
    seeds_.assign(d.seeds, d.seeds + d.n_seeds);
    const size_t ncell = size_t(dom_[0]) * dom_[1] * dom_[2];
    if (d.geometry) geom_.assign(d.geometry, d.geometry + ncell);
    if (mode_ == PLBM_MODE_PROGRESSIVE && seeds_.empty())
        throw std::invalid_argument("config: progressive mode requires at least one seed region");
    for (const auto& c : comps_) {
        if (!(c.tau > 0.5)) throw std::invalid_argument("tau must be > 0.5");
        if (c.b * c.rho_ambient >= 1.0) throw std::invalid_argument("rho_ambient beyond the EOS pole");
    }
    // proj/src/engine.cpp:128-132, proj/src/topology.cpp:85-89
    face_xfer_ = uint64_t(E_) * E_ * uint64_t(C_) * (5 + 1) * 8;

    // ---- device constants
    Params& p = params_;
    std::memset(&p, 0, sizeof p);
    p.C = C_;
    p.n_seeds = int(seeds_.size());
    for (int a = 0; a < 3; ++a) p.grid[a] = grid_[a];
    p.progressive = mode_ == PLBM_MODE_PROGRESSIVE;
    p.s2 = threshold_ * threshold_;
    nopsi_ = true;
    for (int c = 0; c < C_; ++c) {
        const plbm_component_desc& s = comps_[c];
        CompConst& k = p.comp[c];
        k.omega = 1.0 / s.tau;
        for (int a = 0; a < 3; ++a) k.gravity[a] = s.gravity[a];
        k.has_gravity = s.gravity[0] != 0.0 || s.gravity[1] != 0.0 || s.gravity[2] != 0.0;
        k.ideal = s.a == 0.0 && s.b == 0.0;
        k.psi_free = k.ideal && s.R == 1.0 && s.T == PLBM_CS2;
        if (!k.psi_free) nopsi_ = false;
        k.R = s.R;
        k.T = s.T;
        k.b = s.b;
        k.a_theta = s.a * host_theta(s);
        k.two_b = 2.0 * s.b;
        k.b_b = s.b * s.b;
        k.cs2_g = PLBM_CS2 * s.g_self;
        k.c1f = -s.beta * s.g_self;
        k.c2 = -0.5 * (1.0 - s.beta) * s.g_self;
        // make_ambient, proj/src/tilemap.cpp:13-28
        k.rho_amb = s.rho_ambient;
        k.psi_amb = host_psi(s.rho_ambient, host_pr_pressure(s.rho_ambient, s), s.g_self);
        const double u0[3] = {0, 0, 0};
        host_equilibrium(s.rho_ambient, u0, k.feq_amb);
        double rnb = 0.0;  // P1 density of a fresh ambient cell (sequential sum)
        for (int i = 0; i < Q; ++i) rnb += k.feq_amb[i];
        k.psi_nb = host_psi(rnb, host_pr_pressure(rnb, s), s.g_self);
    }
    for (int k = 0; k < C_ * C_; ++k) p.coupling[k] = coupling_[k];
    for (size_t s = 0; s < seeds_.size(); ++s) {
        const plbm_seed_desc& sd = seeds_[s];
        SeedConst& sc = p.seeds[s];
        sc.shape = sd.shape == PLBM_SEED_SPHERE ? 1 : 0;
        sc.comp = sd.component;
        for (int a = 0; a < 3; ++a) {
            sc.lo[a] = sd.box_min[a];
            sc.hi[a] = sd.box_max[a];
            sc.center[a] = sd.center[a];
            sc.u[a] = sd.velocity[a];
        }
        sc.r2 = sd.radius * sd.radius;
        sc.rho = sd.rho;
        host_equilibrium(sd.rho, sd.velocity, sc.feq);
    }

    // ---- capacities: global slots (all tiles) + per-rank local pools
    const size_t n_tiles = size_t(grid_[0]) * grid_[1] * grid_[2];
    cap_ = int(n_tiles);
    amb_ = cap_;
    p.amb_slot = amb_;
    // owners are balanced over `devices` (spread <= 1, assign.cpp:8-15) and
    // owner o lives on rank o % world: the busiest rank holds at most
    // ceil(devices/world) owners x ceil(tiles/devices) tiles.
    {
        const int owners_per_rank = (devices_ + world_ - 1) / world_;
        const int tiles_per_owner = int((n_tiles + devices_ - 1) / devices_);
        lcap_ = std::min(int(n_tiles), owners_per_rank * tiles_per_owner);
        if (world_ == 1) lcap_ = int(n_tiles);
    }
    // f block + xcol side buffer (A-B); A-A keeps one f block and no xcol
    per_slot_ = size_t(C_) * Q * E3_ + size_t(C_) * XN * E2_;
    nbuf_ = aa_ ? 1 : 2;
    per_pf_ = size_t(C_) * 6 * E2_;
    const int nslot = cap_ + 1;
    const int G = E_ + 2;
    solid_words_ = (G * G * G + 31) / 32;
    trig_bytes_ = (size_t(nslot) + 3) / 4 * 4;

    CK(cudaSetDevice(dev_));
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    K_ = pick_kernels(E_, C_, nopsi_);
    if (const char* sp = std::getenv("PLBM_SPLIT")) split_ = std::atoi(sp);
    else split_ = 4;
    mid_faces_ = 2 * (K_.nhmax - 1);                   // boundary rows of split-tile clusters
    params_.mid_sp = K_.nhmax > 1 ? E_ / K_.nhmax : 0;  // (Dev::mid_faces, face_xyz)
    per_pf_ = size_t(C_) * (6 + mid_faces_) * E2_;
    if (aa_ && !K_.main_aa[0] && !K_.main_aa_split[0][0])
        throw std::invalid_argument("A-A storage needs the fused cluster kernels or one CTA per tile "
                                    "(a psi-free scenario at tile_extent 64 has neither)");
    K_.preload();
    {   // this unit's kernels too (lazy loading, see dispatch.cuh preload)
        cudaFuncAttributes a;
        const void* fs[] = {(const void*)k_post_main, (const void*)k_rank_barrier, (const void*)k_check,
                            (const void*)k_err_halt, (const void*)k_fill, (const void*)k_spin};
        for (const void* f : fs) CK(cudaFuncGetAttributes(&a, f));
        switch (E_) {
        case 8: CK(cudaFuncGetAttributes(&a, (const void*)k_check_expand<8>)); break;
        case 16: CK(cudaFuncGetAttributes(&a, (const void*)k_check_expand<16>)); break;
        case 32: CK(cudaFuncGetAttributes(&a, (const void*)k_check_expand<32>)); break;
        default: CK(cudaFuncGetAttributes(&a, (const void*)k_check_expand<64>)); break;
        }
    }
    {
        const size_t bytes = size_t(nbuf_) * per_slot_ * size_t(lcap_ + 1) * sizeof(double);
        const char* lz = std::getenv("PLBM_LAZY_POOL");
        vm_pool_ = world_ == 1 && !(lz && lz[0] == '0');
        if (vm_pool_) {
            vm_reserve(bytes);
            d_pool_f_ = reinterpret_cast<double*>(vm_base_);
            const size_t slot_b = per_slot_ * sizeof(double);
            for (int b = 0; b < nbuf_; ++b)  // the ambient slot of each buffer, now
                vm_map_range((size_t(b) * (lcap_ + 1) + lcap_) * slot_b, slot_b);
        } else {
            d_pool_f_ = dmalloc<double>(bytes / sizeof(double));
        }
    }
    d_pool_pf_ = dmalloc<double>(2 * per_pf_ * size_t(lcap_ + 1));
    for (int b = 0; b < 2; ++b) {
        d_slot_f_[b] = dmalloc<double*>(nslot);
        d_slot_pf_[b] = dmalloc<double*>(nslot);
    }
    for (int r = 0; r < 3; ++r) d_route_[r] = dmalloc<int>(size_t(nslot) * 18);
    d_lidx_ = dmalloc<int>(nslot);
    d_solid_ = dmalloc<uint32_t>(size_t(nslot) * solid_words_);
    d_has_solid_ = dmalloc<uint8_t>(nslot);
    d_no_fluid_ = dmalloc<uint8_t>(nslot);
    CK(cudaMemsetAsync(d_no_fluid_, 0, nslot, stream_));
    d_mode_ = dmalloc<uint8_t>(nslot);
    d_coords_ = dmalloc<int>(size_t(nslot) * 3);
    d_u_face_ = dmalloc<double>(size_t(lcap_ + 1) * C_ * 6 * 3 * E2_);
    {
        const size_t sync_words = SYNC_TRIG + (2 * trig_bytes_ + 7) / 8;
        d_sync_ = dmalloc<unsigned long long>(sync_words);
        CK(cudaMemsetAsync(d_sync_, 0, sync_words * sizeof(unsigned long long), stream_));
        d_err_ = d_sync_ + 8;
        d_trig_ = reinterpret_cast<uint8_t*>(d_sync_ + SYNC_TRIG);
        d_gcnt_ = dmalloc<unsigned long long>(CNT_N);
        CK(cudaMemsetAsync(d_gcnt_, 0, CNT_N * sizeof(unsigned long long), stream_));
    }
    d_bmask_ = dmalloc<uint8_t>(nslot);
    d_omask_ = dmalloc<uint8_t>(nslot);
    d_halt_ = dmalloc<int>(1);
    CK(cudaMemsetAsync(d_halt_, 0, sizeof(int), stream_));
    CK(cudaMallocHost(&h_flags_, 16 * sizeof(int)));
    CK(cudaMallocHost(&h_cnt_, (2 * CNT_N + 4) * sizeof(unsigned long long)));
    // (environment overrides first: device expansion depends on the queue depth)
    if (const char* sd = std::getenv("PLBM_SPEC_DEPTH")) spec_depth_ = std::max(1, std::min(8, std::atoi(sd)));
    if (const char* fv = std::getenv("PLBM_FACE_VARIANT")) K_.face = K_.face_v[std::atoi(fv) == 1 ? 1 : 0];
    {
        const char* de = std::getenv("PLBM_DEVICE_EXPAND");
        // several ranks always expand on the device (the same merged inputs
        // on every rank); one rank does for progressive runs with a queue
        dev_expand_ = world_ > 1 ||
                      (mode_ == PLBM_MODE_PROGRESSIVE && spec_depth_ > 1 && !(de && de[0] == '0'));
        if (world_ > 8) throw std::invalid_argument("at most 8 ranks (one node)");
    }
    if (dev_expand_) {
        const size_t ngrid = size_t(grid_[0]) * grid_[1] * grid_[2];
        d_gslot_ = dmalloc<int>(ngrid);
        d_cand_ = dmalloc<unsigned long long>(ngrid);
        CK(cudaMemsetAsync(d_cand_, 0xff, ngrid * sizeof(unsigned long long), stream_));
        d_nactive_ = dmalloc<int>(1);
        d_next_slot_ = dmalloc<int>(1);
        d_next_local_ = dmalloc<int>(size_t(world_));
        if (world_ > 1) {
            d_all_active_ = dmalloc<int>(nslot);
            d_nall_ = dmalloc<int>(1);
            d_merged_ = dmalloc<uint8_t>(nslot);
        }
        d_owner_ = dmalloc<int>(nslot);
        d_p2p_ = dmalloc<uint8_t>(size_t(devices_) * devices_);
        CK(cudaMemcpyAsync(d_p2p_, p2p_.data(), p2p_.size(), cudaMemcpyHostToDevice, stream_));
        d_per_dev_ = dmalloc<unsigned long long>(size_t(devices_));
        d_acc_ = dmalloc<unsigned long long>(8);
        CK(cudaMemsetAsync(d_acc_, 0, 8 * sizeof(unsigned long long), stream_));
        d_births_ = dmalloc<BirthRec>(size_t(cap_) + 1);
        d_nbirths_ = dmalloc<int>(1);
        CK(cudaMemsetAsync(d_nbirths_, 0, sizeof(int), stream_));
        d_post_flags_ = dmalloc<int>(1);
        CK(cudaMemsetAsync(d_post_flags_, 0, sizeof(int), stream_));
        CK(cudaStreamSynchronize(stream_));
    }
    if (!geom_.empty()) {  // initial slicing (k_slice) and device expansion
        d_geomdev_ = dmalloc<uint8_t>(geom_.size());
        CK(cudaMemcpyAsync(d_geomdev_, geom_.data(), geom_.size(), cudaMemcpyHostToDevice, stream_));
    }
    for (auto& e : flag_ev_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    d_pokes_ = dmalloc<Poke>(64);
    d_dep_cnt_ = dmalloc<int>(nslot);
    d_dep_need_ = dmalloc<int>(nslot);
    d_geo_ = dmalloc<int>(size_t(nslot) * 18);
    CK(cudaMemsetAsync(d_dep_cnt_, 0, nslot * sizeof(int), stream_));
    d_cnt_ = dmalloc<unsigned long long>(CNT_N);
    d_suspect_ = dmalloc<uint8_t>(nslot);
    CK(cudaMemsetAsync(d_suspect_, 0, nslot, stream_));
    d_susp_any_ = dmalloc<unsigned>(2);
    CK(cudaMemsetAsync(d_susp_any_, 0, 2 * sizeof(unsigned), stream_));
    d_active_ = dmalloc<int>(nslot);
    d_scratch_slots_ = dmalloc<int>(nslot);
    d_readback_ = dmalloc<double>(size_t(23) * E3_);
    CK(cudaMemsetAsync(d_u_face_, 0, size_t(lcap_ + 1) * C_ * 6 * 3 * E2_ * sizeof(double), stream_));
    CK(cudaMemsetAsync(d_cnt_, 0, CNT_N * sizeof(unsigned long long), stream_));
    reset_err();
    CK(cudaMemcpyToSymbolAsync(P, &params_, sizeof(Params), 0, cudaMemcpyHostToDevice, stream_));
    K_.set_params(params_, stream_);  // the kernel unit's own copy
    // this rank's ambient slot (local index lcap): feq_amb in both buffers and
    // psi_amb on its faces for both parities
    {
        std::vector<double> amb(per_slot_);
        for (int c = 0; c < C_; ++c)
            for (int i = 0; i < Q; ++i) {
                std::fill_n(amb.begin() + (size_t(c) * Q + i) * E3_, E3_, p.comp[c].feq_amb[i]);
                for (int cls = 0; cls < 4; ++cls)
                    if (xslot_(cls, i) >= 0)
                        std::fill_n(amb.begin() + size_t(C_) * Q * E3_ + (size_t(c) * XN + xslot_(cls, i)) * E2_,
                                    E2_, p.comp[c].feq_amb[i]);
            }
        std::vector<double> pf(per_pf_);
        for (int c = 0; c < C_; ++c)
            std::fill_n(pf.begin() + size_t(c) * 6 * E2_, 6 * E2_, p.comp[c].psi_amb);
        for (int b = 0; b < 2; ++b) {
            if (b < nbuf_)
                CK(cudaMemcpy(d_pool_f_ + (size_t(b) * (lcap_ + 1) + lcap_) * per_slot_, amb.data(),
                              per_slot_ * sizeof(double), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(d_pool_pf_ + (size_t(b) * (lcap_ + 1) + lcap_) * per_pf_, pf.data(),
                          per_pf_ * sizeof(double), cudaMemcpyHostToDevice));
        }
    }
    peer_f_.assign(world_, nullptr);
    peer_pf_.assign(world_, nullptr);
    peer_opened_.assign(world_, false);
    peer_f_[rank_] = d_pool_f_;
    peer_pf_[rank_] = d_pool_pf_;
    peer_sync_.assign(world_, nullptr);
    peer_sync_[rank_] = d_sync_;
    for (int b = 0; b < 2; ++b) {
        d_.slot_f[b] = d_slot_f_[b];
        d_.slot_pf[b] = d_slot_pf_[b];
    }
    for (int r = 0; r < 3; ++r) d_.route[r] = d_route_[r];
    d_.aa = aa_ ? 1 : 0;
    d_.mid_faces = mid_faces_;
    d_.lidx = d_lidx_;
    d_.solid = d_solid_;
    d_.has_solid = d_has_solid_;
    d_.no_fluid = d_no_fluid_;
    d_.mode = d_mode_;
    d_.coords = d_coords_;
    d_.u_face = d_u_face_;
    d_.trig = d_trig_;
    d_.capture = nullptr;
    d_.cnt = d_cnt_;
    d_.err = d_err_;
    d_.solid_words = solid_words_;
    d_.dep_cnt = d_dep_cnt_;
    d_.dep_need = d_dep_need_;
    d_.geo = d_geo_;
    d_.face_flags = 0;
    d_.xcol_ok = 0;
    d_.halt = nullptr;
    d_.pokes = nullptr;
    d_.npoke = 0;
    d_.nactive = nullptr;
    d_.probe = nullptr;
    d_.tile_base = 0;
    d_.suspect = d_suspect_;
    // the P5 screen's argument needs every pulled ambient population in range
    d_.screen_all = 0;
    for (int c = 0; c < C_; ++c)
        for (int i = 0; i < Q; ++i)
            if (!screen_ok(p.comp[c].feq_amb[i])) d_.screen_all = 1;
    if (std::getenv("PLBM_P5_ALL")) d_.screen_all = 1;  // test hook: exact check of every tile
    // integer negative-population count (k_main_pc): every f_in value must be
    // nonzero-or-+0, finite and not -0; the constants a step can pull are
    // checked here, the stored populations by the previous step's screen
    // (whose marks are per rank: multi-rank runs keep the FP compares)
    d_.susp_any = world_ == 1 ? d_susp_any_ : nullptr;
    d_.neg_exact = d_.screen_all;
    auto sign_ok = [](double v) { return std::isfinite(v) && !(v == 0.0 && std::signbit(v)); };
    for (int c = 0; c < C_; ++c)
        for (int i = 0; i < Q; ++i)
            if (!sign_ok(p.comp[c].feq_amb[i])) d_.neg_exact = 1;
    for (size_t sd = 0; sd < seeds_.size(); ++sd)
        for (int i = 0; i < Q; ++i)
            if (!sign_ok(p.seeds[sd].feq[i])) d_.neg_exact = 1;
    if (std::getenv("PLBM_PROBE")) d_.probe = dmalloc<unsigned long long>(3 * size_t(cap_ + 1) * 16);

    // ---- host mirror + initial tiles (make_state, engine.cpp:134-159)
    grid_slot_.assign(n_tiles, -1);
    slots_.assign(nslot, SlotInfo{});
    free_slots_.clear();
    for (int s = cap_ - 1; s >= 0; --s) free_slots_.push_back(s);
    next_local_.assign(world_, 0);
    per_dev_.assign(devices_, 0);
    h_mode_.assign(nslot, MODE_PULL);
    h_has_solid_.assign(nslot, 0);
    h_coords_.assign(size_t(nslot) * 3, -1000000);
    h_solid_.assign(size_t(nslot) * solid_words_, 0u);
    h_lidx_.assign(nslot, -1);
    h_lidx_[amb_] = lcap_;
    std::vector<uint8_t> initial(n_tiles, 0);
    if (mode_ == PLBM_MODE_STATIC) {
        std::fill(initial.begin(), initial.end(), 1);
    } else {
        // A tile holds a seeded cell centre iff every axis has one: the box
        // test is separable, and for a sphere each squared offset is minimised
        // independently (monotone FP ops) — identical to the reference's
        // per-cell loop (engine.cpp:147-154) without touching every cell.
        for (const auto& s : seeds_)
            for (int tx = 0; tx < grid_[0]; ++tx)
                for (int ty = 0; ty < grid_[1]; ++ty)
                    for (int tz = 0; tz < grid_[2]; ++tz) {
                        const int t[3] = {tx, ty, tz};
                        bool hit;
                        if (s.shape == PLBM_SEED_BOX) {
                            hit = true;
                            for (int a = 0; a < 3 && hit; ++a) {
                                bool any = false;
                                for (int v = t[a] * E_; v < t[a] * E_ + E_ && !any; ++v) {
                                    const double cc = v + 0.5;
                                    any = cc >= s.box_min[a] && cc < s.box_max[a];
                                }
                                hit = any;
                            }
                        } else {
                            double m[3];
                            for (int a = 0; a < 3; ++a) {
                                m[a] = INFINITY;
                                for (int v = t[a] * E_; v < t[a] * E_ + E_; ++v) {
                                    const double dd = (v + 0.5) - s.center[a];
                                    m[a] = std::min(m[a], dd * dd);
                                }
                            }
                            hit = m[0] + m[1] + m[2] <= s.radius * s.radius;
                        }
                        if (hit) initial[(size_t(tx) * grid_[1] + ty) * grid_[2] + tz] = 1;
                    }
    }
    // with a geometry the initial tiles are sliced on the device (k_slice);
    // owners are assigned after the fluid counts are known, in creation order
    // (a later tile has owner -1 until then, which assign_device skips)
    const bool dev_slice = d_geomdev_ != nullptr;
    std::vector<int> created;
    for (size_t k = 0; k < n_tiles; ++k) {
        if (!initial[k]) continue;
        const Coord c{int(k / (size_t(grid_[1]) * grid_[2])), int((k / grid_[2]) % grid_[1]),
                      int(k % grid_[2])};
        const int s = create_tile(c, 0, -1, !dev_slice);
        if (!dev_slice) assign_owner(s);
        created.push_back(s);
    }
    if (dev_slice) {
        slice_on_device(created);
        for (int s : created) assign_owner(s);
    }
    for (int s : created) h_mode_[s] = MODE_GEN_SEEDED;
    upload_map(created, true);
    if (world_ == 1) prepare();
    CK(cudaStreamSynchronize(stream_));
}

// psi faces of the initial (generated) state for step 1.  Multi-rank callers
// run this on every rank after attaching peers and synchronise before step 1.
int Engine::prepare() {
    if (prepared_) return 0;
    if (!peers_ready()) return -8;
    launch_face(0, 0, 0);
    CK(cudaStreamSynchronize(stream_));
    prepared_ = true;
    return 0;
}

void Engine::release() {
    if (stream_) cudaStreamSynchronize(stream_);
    for (int r = 0; r < world_ && r < int(peer_opened_.size()); ++r)
        if (peer_opened_[r]) {
            cudaIpcCloseMemHandle(peer_f_[r]);
            cudaIpcCloseMemHandle(peer_pf_[r]);
            cudaIpcCloseMemHandle(peer_sync_[r]);
        }
    vm_release();
    if (vm_pool_) d_pool_f_ = nullptr;
    void* ptrs[] = {d_pool_f_, d_pool_pf_, d_slot_f_[0], d_slot_f_[1], d_slot_pf_[0], d_slot_pf_[1],
                    d_route_[0], d_route_[1], d_route_[2], d_lidx_, d_solid_, d_has_solid_, d_no_fluid_, d_mode_,
                    d_coords_,
                    d_u_face_, d_sync_, d_gcnt_, d_capture_, d_cnt_, d_all_active_, d_nall_, d_merged_, d_active_,
                    d_scratch_slots_,
                    d_readback_, d_dep_cnt_, d_dep_need_, d_geo_, d_bmask_, d_omask_, d_halt_, d_pokes_,
                    d_gslot_, d_cand_, d_nactive_, d_next_slot_, d_next_local_, d_owner_, d_geomdev_, d_p2p_,
                    d_per_dev_, d_acc_, d_births_, d_nbirths_, d_post_flags_, d_suspect_, d_susp_any_};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (h_flags_) cudaFreeHost(h_flags_);
    if (h_cnt_) cudaFreeHost(h_cnt_);
    for (auto& e : flag_ev_)
        if (e) cudaEventDestroy(e);
    for (auto& e : ev_pool_) {
        if (e.a) cudaEventDestroy(e.a);
        if (e.b) cudaEventDestroy(e.b);
    }
    if (stream_) cudaStreamDestroy(stream_);
    stream_ = nullptr;
}

// ---- lazily mapped population pool (one rank) ------------------------------
// driver-API entry points through the runtime (no link-time libcuda
// dependency: the library still loads on a host without a driver)
struct VmApi {
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) access = nullptr;
};
static const VmApi& vm_api() {
    static VmApi a = [] {
        VmApi v;
        auto get = [](const char* name, auto& fn) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q;
            CK(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
            if (!p || q != cudaDriverEntryPointSuccess)
                throw CudaError(std::string("driver entry point missing: ") + name);
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
        };
        get("cuMemGetAllocationGranularity", v.granularity);
        get("cuMemAddressReserve", v.reserve);
        get("cuMemAddressFree", v.free);
        get("cuMemCreate", v.create);
        get("cuMemRelease", v.release);
        get("cuMemMap", v.map);
        get("cuMemUnmap", v.unmap);
        get("cuMemSetAccess", v.access);
        return v;
    }();
    return a;
}
#define CU(x)                                                                                   \
    do {                                                                                        \
        CUresult r_ = (x);                                                                      \
        if (r_ != CUDA_SUCCESS) throw CudaError(std::string(#x) + ": CUresult " + std::to_string(int(r_))); \
    } while (0)

void Engine::vm_reserve(size_t bytes) {
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev_;
    CU(vm_api().granularity(&vm_gran_, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    // A mapping costs ~0.25 ms of host time whatever its size (tools/vm_probe.py,
    // profiles/r02q_vm_probe.jsonl), paid while the stream waits for the new
    // tiles: the pool is cut into at most ~64 granules (<= 2 GiB each, a
    // multiple of the device's granularity), so a run maps at most ~64 times.
    const char* gm = std::getenv("PLBM_POOL_GRANULE_MB");
    const size_t want = gm ? size_t(std::max(2, std::atoi(gm))) << 20
                           : std::min<size_t>(bytes / 64, size_t(2) << 30);
    vm_gran_ = std::max<size_t>(1, (want + vm_gran_ - 1) / vm_gran_) * vm_gran_;
    vm_size_ = (bytes + vm_gran_ - 1) / vm_gran_ * vm_gran_;
    CU(vm_api().reserve(&vm_base_, vm_size_, 0, 0, 0));  // device-granularity aligned
    vm_handles_.assign(vm_size_ / vm_gran_, 0);
}

void Engine::vm_map_range(size_t off, size_t len) {
    if (len == 0) return;
    const auto t0 = std::chrono::steady_clock::now();
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev_;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (size_t g = off / vm_gran_; g <= (off + len - 1) / vm_gran_ && g < vm_handles_.size(); ++g) {
        if (vm_handles_[g]) continue;
        CUmemGenericAllocationHandle h;
        CU(vm_api().create(&h, vm_gran_, &prop, 0));
        CU(vm_api().map(vm_base_ + g * vm_gran_, vm_gran_, 0, h, 0));
        CU(vm_api().access(vm_base_ + g * vm_gran_, vm_gran_, &acc, 1));
        vm_handles_[g] = h;
        vm_mapped_ += vm_gran_;
    }
    vm_map_us_ += uint64_t(
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
}

void Engine::vm_mapper() {
    const size_t slot_b = per_slot_ * sizeof(double);
    const size_t buf_b = size_t(lcap_ + 1) * slot_b;
    const int step = std::max(1, int(vm_gran_ / slot_b));
    std::unique_lock<std::mutex> lk(vm_mu_);
    try {
        CK(cudaSetDevice(dev_));
        for (;;) {
            vm_cv_.wait(lk, [&] { return vm_stop_ || vm_want_ > vm_ready_; });
            if (vm_stop_) return;
            const int want = vm_want_;
            while (vm_ready_ < want && !vm_stop_) {
                const int s0 = vm_ready_, s1 = std::min(want, s0 + step);
                lk.unlock();
                for (int b = 0; b < nbuf_; ++b)
                    vm_map_range(size_t(b) * buf_b + size_t(s0) * slot_b, size_t(s1 - s0) * slot_b);
                lk.lock();
                vm_ready_ = s1;
                vm_cv_.notify_all();
            }
        }
    } catch (const std::exception& e) {
        if (!lk.owns_lock()) lk.lock();
        vm_err_ = e.what();
        vm_cv_.notify_all();
    }
}

void Engine::ensure_pool(int n_slots) {
    if (!vm_pool_) return;
    n_slots = std::min(n_slots, lcap_);
    const int ahead = std::max(n_slots / 4, std::max(1, int(vm_gran_ / (per_slot_ * sizeof(double)))));
    std::unique_lock<std::mutex> lk(vm_mu_);
    if (!vm_thread_.joinable()) vm_thread_ = std::thread([this] { vm_mapper(); });
    const int target = std::min(lcap_, n_slots + ahead);
    if (target > vm_want_) {
        vm_want_ = target;
        vm_cv_.notify_all();
    }
    if (vm_ready_ < n_slots && vm_err_.empty()) {
        const auto t0 = std::chrono::steady_clock::now();
        vm_cv_.wait(lk, [&] { return vm_ready_ >= n_slots || !vm_err_.empty(); });
        vm_wait_us_ += uint64_t(
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    if (!vm_err_.empty()) throw CudaError("population pool mapping: " + vm_err_);
}

void Engine::vm_release() {
    if (vm_thread_.joinable()) {
        {
            std::lock_guard<std::mutex> lk(vm_mu_);
            vm_stop_ = true;
        }
        vm_cv_.notify_all();
        vm_thread_.join();
    }
    if (!vm_base_) return;
    for (size_t g = 0; g < vm_handles_.size(); ++g)
        if (vm_handles_[g]) {
            vm_api().unmap(vm_base_ + g * vm_gran_, vm_gran_);
            vm_api().release(vm_handles_[g]);
        }
    vm_api().free(vm_base_, vm_size_);
    vm_base_ = 0;
    vm_handles_.clear();
}

// proj/src/tilemap.cpp:56-67
bool Engine::neighbor_coords(const Coord& from, int face, Coord& out) const {
    int c[3] = {from.x, from.y, from.z};
    const int axis = face / 2;
    c[axis] += (face % 2) ? 1 : -1;
    if (c[axis] < 0 || c[axis] >= grid_[axis]) {
        if (!periodic_[axis]) return false;
        c[axis] = (c[axis] + grid_[axis]) % grid_[axis];
    }
    out = {c[0], c[1], c[2]};
    return true;
}

// proj/src/tilemap.cpp:83-175 (metadata + solid slicing; fields live on the device)
int Engine::create_tile(const Coord& c, long iteration, int trigger, bool slice) {
    if (free_slots_.empty()) throw std::runtime_error("block pool exhausted");
    const int s = free_slots_.back();
    free_slots_.pop_back();
    SlotInfo& si = slots_[s];
    si = SlotInfo{};
    si.c = c;
    si.birth = iteration;
    const int G = E_ + 2;
    uint32_t* bits = &h_solid_[size_t(s) * solid_words_];
    std::fill_n(bits, solid_words_, 0u);
    int fluid = 0;
    bool any = false;
    for (int lz = -1; slice && lz <= E_; ++lz)
        for (int ly = -1; ly <= E_; ++ly)
            for (int lx = -1; lx <= E_; ++lx) {
                int g[3] = {c.x * E_ + lx, c.y * E_ + ly, c.z * E_ + lz};
                bool outside = false;
                for (int a = 0; a < 3; ++a)
                    if (g[a] < 0 || g[a] >= dom_[a]) {
                        if (periodic_[a]) g[a] = (g[a] + dom_[a]) % dom_[a];
                        else outside = true;
                    }
                bool sol = false;
                if (!outside && !geom_.empty())
                    sol = geom_[size_t(g[0]) + size_t(dom_[0]) * (size_t(g[1]) + size_t(dom_[1]) * g[2])] != 0;
                const bool interior = lx >= 0 && lx < E_ && ly >= 0 && ly < E_ && lz >= 0 && lz < E_;
                if (sol) {
                    const int idx = (lx + 1) + G * ((ly + 1) + G * (lz + 1));
                    bits[idx >> 5] |= 1u << (idx & 31);
                    any = true;
                } else if (interior) {
                    ++fluid;
                }
            }
    si.fluid = fluid;
    si.has_solid = any;
    active_cells_ += uint64_t(fluid);
    si.log_index = log_.size();
    log_.push_back({iteration, c, trigger, -1});
    grid_slot_[lin(c)] = s;
    h_mode_[s] = MODE_GEN_AMBIENT;
    h_has_solid_[s] = any ? 1 : 0;
    h_coords_[3 * size_t(s)] = c.x;
    h_coords_[3 * size_t(s) + 1] = c.y;
    h_coords_[3 * size_t(s) + 2] = c.z;
    return s;
}

// create_tile's solid slicing for a batch of new tiles on the device; the
// host mirror keeps the fluid count and has_solid (the mask stays on the GPU:
// upload_map skips the slots marked device_sliced).
void Engine::slice_on_device(const std::vector<int>& slots) {
    if (slots.empty()) return;
    const int n = int(slots.size());
    std::vector<int> coords(size_t(3) * n);
    for (int k = 0; k < n; ++k) {
        const Coord& c = slots_[slots[k]].c;
        coords[3 * k] = c.x;
        coords[3 * k + 1] = c.y;
        coords[3 * k + 2] = c.z;
    }
    int* d_buf = dmalloc<int>(size_t(5) * n);  // slots, coords, fluid; has_solid bytes after
    int *d_slots = d_buf, *d_coords = d_buf + n, *d_fluid = d_buf + 4 * n;
    uint8_t* d_hs = dmalloc<uint8_t>(n);
    CK(cudaMemcpyAsync(d_slots, slots.data(), n * sizeof(int), cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_coords, coords.data(), coords.size() * sizeof(int), cudaMemcpyHostToDevice, stream_));
    auto go = [&](auto kern) {
        kern<<<n, 256, 0, stream_>>>(d_slots, d_coords, n, d_geomdev_, dom_[0], dom_[1], dom_[2], periodic_[0],
                                     periodic_[1], periodic_[2], d_solid_, solid_words_, d_hs, d_fluid);
    };
    switch (E_) {
    case 8: go(k_slice<8>); break;
    case 16: go(k_slice<16>); break;
    case 32: go(k_slice<32>); break;
    default: go(k_slice<64>); break;
    }
    CK(cudaGetLastError());
    std::vector<int> fluid(n);
    std::vector<uint8_t> hs(n);
    CK(cudaMemcpyAsync(fluid.data(), d_fluid, n * sizeof(int), cudaMemcpyDeviceToHost, stream_));
    CK(cudaMemcpyAsync(hs.data(), d_hs, n, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
    CK(cudaFree(d_buf));
    CK(cudaFree(d_hs));
    for (int k = 0; k < n; ++k) {
        SlotInfo& si = slots_[slots[k]];
        si.fluid = fluid[k];
        si.has_solid = hs[k] != 0;
        si.device_sliced = true;
        h_has_solid_[slots[k]] = hs[k];
        active_cells_ += uint64_t(fluid[k]);
    }
}

// proj/src/engine.cpp:30-41 -> proj/src/assign.cpp:8-38; then the GPU rank
// (owner % world) and its next pool index.
void Engine::assign_owner(int slot) {
    SlotInfo& t = slots_[slot];
    std::vector<int> owners;
    for (int f = 0; f < 6; ++f) {
        Coord nc;
        if (!neighbor_coords(t.c, f, nc)) continue;
        const int ns = slot_at(nc);
        if (ns >= 0 && slots_[ns].owner >= 0 && ns != slot) owners.push_back(slots_[ns].owner);
    }
    const uint64_t lo = *std::min_element(per_dev_.begin(), per_dev_.end());
    std::vector<int> eligible;
    for (int dv = 0; dv < devices_; ++dv)
        if (per_dev_[dv] == lo) eligible.push_back(dv);
    auto f_cost = [&](int cand) {
        double sum = 0.0;
        for (int o : owners) {
            const int cls = classify(cand, o);
            sum += cls == 0 ? 0.0 : (cls == 1 ? w_p2p_ * double(face_xfer_) : w_staged_ * double(face_xfer_));
        }
        return sum;
    };
    int chosen = eligible.front();
    if (policy_ == PLBM_POLICY_OPTIMIZED) {
        double best = f_cost(chosen);
        for (size_t k = 1; k < eligible.size(); ++k) {
            const double c = f_cost(eligible[k]);
            if (c < best) {
                best = c;
                chosen = eligible[k];
            }
        }
    }
    ++per_dev_[chosen];
    t.owner = chosen;
    log_[t.log_index].owner = chosen;
    t.rank = chosen % world_;
    t.local = next_local_[t.rank]++;
    if (t.local >= lcap_) throw std::runtime_error("local block pool exhausted");
    h_lidx_[slot] = t.rank == rank_ ? t.local : -1;
    if (t.rank == rank_) local_cells_ += uint64_t(t.fluid);
}

// Ghost routing (proj/src/engine.cpp:266-296): a face ghost reads the face
// neighbour; an edge ghost on axes a<b hops along b first, then a — an absent
// hop yields the ambient slot even when the diagonal tile exists.
// Real cross-GPU data volume of one step on this rank, from
// the routing tables: what this rank's kernels read from peer pools.  Per
// face route to a tile on another rank: the fused kernel pulls the 5
// crossing populations of E^2 cells and reads E^2 psi ghosts, the face pass
// pulls the 5 crossing populations of its E^2 face cells; per edge route: one
// crossing population and one psi ghost of E cells for each, and the face
// passes' edge pulls.  out = {bytes, remote face routes, remote edge routes}.
void Engine::exchange_bytes(uint64_t* out) const {
    out[0] = out[1] = out[2] = 0;
    std::vector<int> r(18);
    for (int s : active_) {
        compute_routes(s, r.data());
        for (int k = 0; k < 18; ++k) {
            const int n = r[size_t(k)];
            if (n == amb_ || slots_[n].rank == rank_) continue;
            if (k < 6) {
                ++out[1];
                out[0] += uint64_t(5 + 1 + 5) * E2_ * C_ * sizeof(double);
            } else {
                ++out[2];
                out[0] += uint64_t(1 + 1 + 2) * E_ * C_ * sizeof(double);
            }
        }
    }
}

void Engine::compute_routes(int slot, int* out) const {
    const Coord c = slots_[slot].c;
    auto nb = [&](const Coord& from, int axis, int dir, Coord& o) {
        return neighbor_coords(from, 2 * axis + (dir > 0 ? 1 : 0), o);
    };
    for (int f = 0; f < 6; ++f) {
        Coord n;
        out[f] = (nb(c, f / 2, (f % 2) ? 1 : -1, n) && slot_at(n) >= 0) ? slot_at(n) : amb_;
    }
    const int pairs[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int p = 0; p < 3; ++p)
        for (int da = -1; da <= 1; da += 2)
            for (int db = -1; db <= 1; db += 2) {
                const int a = pairs[p][0], b = pairs[p][1];
                int r = amb_;
                Coord n1, n2;
                if (nb(c, b, db, n1) && slot_at(n1) >= 0 && nb(n1, a, da, n2) && slot_at(n2) >= 0)
                    r = slot_at(n2);
                out[edge_class(a, b, da, db)] = r;
            }
}

void Engine::recompute_step_bytes() {
    // Closed form of record_exchange over one step: P2 and P4 each record one
    // transfer per (tile, face) with an existing neighbour (engine.cpp:305-309).
    step_bytes_[0] = step_bytes_[1] = step_bytes_[2] = 0;
    for (int s : all_active_) {
        for (int f = 0; f < 6; ++f) {
            Coord n;
            if (!neighbor_coords(slots_[s].c, f, n)) continue;
            const int ns = slot_at(n);
            if (ns < 0) continue;
            step_bytes_[classify(slots_[s].owner, slots_[ns].owner)] += 2 * face_xfer_;
        }
    }
}

// Per-slot device pointers: own slots and the ambient slot into this rank's
// pool, remote slots into the owner rank's pool (IPC-mapped peer memory).
void Engine::upload_pointers() {
    const size_t nslot = size_t(cap_ + 1);
    std::vector<double*> f[2], pf[2];
    for (int b = 0; b < 2; ++b) {
        f[b].assign(nslot, nullptr);
        pf[b].assign(nslot, nullptr);
    }
    auto fill = [&](int s, int r, int local) {
        for (int b = 0; b < 2; ++b) {
            if (!peer_f_[r]) continue;
            f[b][s] = peer_f_[r] + (size_t(b % nbuf_) * (lcap_ + 1) + local) * per_slot_;
            pf[b][s] = peer_pf_[r] + (size_t(b) * (lcap_ + 1) + local) * per_pf_;
        }
    };
    for (int s : all_active_) fill(s, slots_[s].rank, slots_[s].local);
    fill(amb_, rank_, lcap_);
    for (int b = 0; b < 2; ++b) {
        CK(cudaMemcpyAsync(d_slot_f_[b], f[b].data(), nslot * sizeof(double*), cudaMemcpyHostToDevice,
                           stream_));
        CK(cudaMemcpyAsync(d_slot_pf_[b], pf[b].data(), nslot * sizeof(double*), cudaMemcpyHostToDevice,
                           stream_));
    }
    stats_.h2d_bytes += 4 * nslot * sizeof(double*);
    CK(cudaStreamSynchronize(stream_));  // host vectors die here
}

void Engine::upload_map(const std::vector<int>& new_slots, bool initial) {
    // active lists in coordinate order (all tiles / this rank's tiles)
    all_active_.clear();
    active_.clear();
    for (size_t k = 0; k < grid_slot_.size(); ++k)
        if (grid_slot_[k] >= 0) {
            all_active_.push_back(grid_slot_[k]);
            if (slots_[grid_slot_[k]].rank == rank_) active_.push_back(grid_slot_[k]);
        }
    ensure_pool(std::max(next_local_[size_t(rank_)],
                         std::min(cap_, int(all_active_.size()) + expand_headroom())));
    const size_t nslot = size_t(cap_ + 1);
    CK(cudaMemcpyAsync(d_active_, active_.data(), active_.size() * sizeof(int),
                       cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_coords_, h_coords_.data(), nslot * 3 * sizeof(int), cudaMemcpyHostToDevice,
                       stream_));
    CK(cudaMemcpyAsync(d_has_solid_, h_has_solid_.data(), nslot, cudaMemcpyHostToDevice, stream_));
    {   // tiles without a fluid cell (from the mirror's fluid counts)
        std::vector<uint8_t> nf(nslot, 0);
        for (int s : all_active_) nf[size_t(s)] = slots_[s].fluid == 0 ? 1 : 0;
        CK(cudaMemcpyAsync(d_no_fluid_, nf.data(), nslot, cudaMemcpyHostToDevice, stream_));
        CK(cudaStreamSynchronize(stream_));
    }
    CK(cudaMemcpyAsync(d_mode_, h_mode_.data(), nslot, cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_lidx_, h_lidx_.data(), nslot * sizeof(int), cudaMemcpyHostToDevice, stream_));
    std::vector<int> mine;
    for (int s : new_slots) {
        if (slots_[s].rank != rank_) continue;
        mine.push_back(s);
        if (h_has_solid_[s] && !slots_[s].device_sliced)
            CK(cudaMemcpyAsync(d_solid_ + size_t(s) * solid_words_, &h_solid_[size_t(s) * solid_words_],
                               solid_words_ * sizeof(uint32_t), cudaMemcpyHostToDevice, stream_));
        if (d_capture_)
            CK(cudaMemsetAsync(d_capture_ + size_t(slots_[s].local) * C_ * 4 * E3_, 0,
                               size_t(C_) * 4 * E3_ * sizeof(double), stream_));
    }
    if (peers_ready()) upload_pointers();
    // newborns' psi faces need no write: readers see the GEN_AMBIENT mode and
    // use psi of a fresh ambient cell (kernels.cuh psi_ghost); initial tiles
    // get theirs from k_face over the generated state (prepare())
    // routes: pull table = map of the step that just ran, psi table = new map
    // geometric neighbour table + dependency counts of the fused face pass
    {
        static const int off[18][3] = {{-1, 0, 0}, {1, 0, 0},  {0, -1, 0},  {0, 1, 0},  {0, 0, -1},
                                       {0, 0, 1},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0},  {1, 1, 0},
                                       {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1}, {1, 0, 1},  {0, -1, -1},
                                       {0, 1, -1}, {0, -1, 1}, {0, 1, 1}};
        std::vector<int> geo(nslot * 18, -1), need(nslot, 0);
        for (int s : all_active_) {
            int n = 1;
            for (int k = 0; k < 18; ++k) {
                int q[3];
                bool ok = true;
                for (int a = 0; a < 3; ++a) {
                    q[a] = (a == 0 ? slots_[s].c.x : a == 1 ? slots_[s].c.y : slots_[s].c.z) + off[k][a];
                    if (q[a] < 0 || q[a] >= grid_[a]) {
                        if (!periodic_[a]) ok = false;
                        q[a] = (q[a] + grid_[a]) % grid_[a];
                    }
                }
                if (!ok) continue;
                const int m = grid_slot_[(size_t(q[0]) * grid_[1] + q[1]) * grid_[2] + q[2]];
                if (m < 0) continue;
                geo[size_t(s) * 18 + k] = m;
                ++n;
            }
            need[s] = n;
        }
        CK(cudaMemcpyAsync(d_geo_, geo.data(), geo.size() * sizeof(int), cudaMemcpyHostToDevice, stream_));
        // ROUTE_W (A-A stores): the geometric neighbour in the new map, or ambient
        std::vector<int> rw(geo);
        for (int& v : rw)
            if (v < 0) v = amb_;
        CK(cudaMemcpyAsync(d_route_[ROUTE_W], rw.data(), rw.size() * sizeof(int), cudaMemcpyHostToDevice,
                           stream_));
        CK(cudaStreamSynchronize(stream_));
        // speculative queue: which trigger bits need the host (births) and
        // which only count as suppressed expansions (out of bounds)
        std::vector<uint8_t> bm(nslot, 0), om(nslot, 0);
        for (int s : all_active_)
            for (int f = 0; f < 6; ++f) {
                Coord n;
                if (!neighbor_coords(slots_[s].c, f, n)) om[s] |= uint8_t(1u << f);
                else if (slot_at(n) < 0) bm[s] |= uint8_t(1u << f);
            }
        CK(cudaMemcpyAsync(d_bmask_, bm.data(), nslot, cudaMemcpyHostToDevice, stream_));
        CK(cudaMemcpyAsync(d_omask_, om.data(), nslot, cudaMemcpyHostToDevice, stream_));
        CK(cudaStreamSynchronize(stream_));  // host vectors die here
        CK(cudaMemcpyAsync(d_dep_need_, need.data(), need.size() * sizeof(int), cudaMemcpyHostToDevice,
                           stream_));
        stats_.h2d_bytes += (geo.size() + need.size()) * sizeof(int);
    }
    std::vector<int> routes(nslot * 18, amb_);
    for (int s : all_active_) compute_routes(s, &routes[size_t(s) * 18]);
    if (!initial)
        CK(cudaMemcpyAsync(d_route_[ROUTE_PULL], d_route_[ROUTE_PSI], routes.size() * sizeof(int),
                           cudaMemcpyDeviceToDevice, stream_));
    else
        CK(cudaMemcpyAsync(d_route_[ROUTE_PULL], routes.data(), routes.size() * sizeof(int),
                           cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_route_[ROUTE_PSI], routes.data(), routes.size() * sizeof(int),
                       cudaMemcpyHostToDevice, stream_));
    routes_differ_ = !initial;
    any_gen_ = true;
    stats_.h2d_bytes += active_.size() * sizeof(int) + nslot * (4 * sizeof(int) + 2) +
                        routes.size() * sizeof(int) * (initial ? 2 : 1);
    for (int s : mine)
        if (h_has_solid_[s]) stats_.h2d_bytes += solid_words_ * sizeof(uint32_t);
    recompute_step_bytes();
    if (dev_expand_) upload_expand_state(initial);
    // the host vectors must outlive the async copies
    CK(cudaStreamSynchronize(stream_));
}

// The host mirror is authoritative after a host-side expansion (initial tiles
// or a halt): the device-side expansion state follows it.
void Engine::upload_expand_state(bool initial) {
    const size_t nslot = size_t(cap_ + 1);
    std::vector<int> owner(nslot, -1);
    for (int s : all_active_) owner[size_t(s)] = slots_[s].owner;
    CK(cudaMemcpyAsync(d_gslot_, grid_slot_.data(), grid_slot_.size() * sizeof(int), cudaMemcpyHostToDevice,
                       stream_));
    CK(cudaMemcpyAsync(d_owner_, owner.data(), nslot * sizeof(int), cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_per_dev_, per_dev_.data(), per_dev_.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                       stream_));
    const int ints[3] = {int(all_active_.size()), cap_ - int(free_slots_.size()), int(active_.size())};
    CK(cudaMemcpyAsync(d_next_slot_, &ints[1], sizeof(int), cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_next_local_, next_local_.data(), size_t(world_) * sizeof(int), cudaMemcpyHostToDevice,
                       stream_));
    if (world_ > 1) {  // the expansion's map (all ranks) + this rank's launch list
        CK(cudaMemcpyAsync(d_nall_, &ints[0], sizeof(int), cudaMemcpyHostToDevice, stream_));
        CK(cudaMemcpyAsync(d_all_active_, all_active_.data(), all_active_.size() * sizeof(int),
                           cudaMemcpyHostToDevice, stream_));
        CK(cudaMemcpyAsync(d_nactive_, &ints[2], sizeof(int), cudaMemcpyHostToDevice, stream_));
    } else {
        CK(cudaMemcpyAsync(d_nactive_, &ints[0], sizeof(int), cudaMemcpyHostToDevice, stream_));
    }
    const unsigned long long map_acc[4] = {active_cells_, step_bytes_[0], step_bytes_[1], step_bytes_[2]};
    CK(cudaMemcpyAsync(d_acc_ + 4, map_acc, sizeof map_acc, cudaMemcpyHostToDevice, stream_));
    const int flags = initial ? 1 : 3;  // GEN modes to reset; pull routes to catch up
    CK(cudaMemcpyAsync(d_post_flags_, &flags, sizeof(int), cudaMemcpyHostToDevice, stream_));
    CK(cudaStreamSynchronize(stream_));
    any_gen_ = routes_differ_ = false;  // k_post_main does them
    post_pending_ = true;               // (the host-merge protocol's step_main launches it)
    launch_tiles_ = std::min(cap_, int(all_active_.size()) + expand_headroom());
}

// CTAs (tiles) this rank's launches cover while the global map holds at most
// launch_tiles_ tiles: every owner has <= ceil(n / devices) tiles (fairness
// spread <= 1, assign.cpp:8-15) and a rank holds ceil(devices / world) owners.
int Engine::launch_bound() const {
    if (world_ == 1) return launch_tiles_;
    const int per_owner = (launch_tiles_ + devices_ - 1) / devices_;
    const int owners = (devices_ + world_ - 1) / world_;
    return std::min(lcap_, per_owner * owners);
}

// Replays the device's births into the host mirror (slots, log, owners,
// counts), so counters, tiles, creation log and read-back see the device map.
void Engine::sync_births() {
    if (!dev_expand_) return;
    // tiles that have stepped are in PULL mode on the device (k_post_main)
    for (size_t s = 0; s < h_mode_.size(); ++s)
        if (h_mode_[s] != MODE_PULL && slots_[s].birth < iteration_) h_mode_[s] = MODE_PULL;
    int nb = 0;
    if (births_seen_ >= 0 && !in_spec_) {
        nb = births_seen_;  // (the queue is drained: the last retired step's count is final)
    } else {
        CK(cudaMemcpyAsync(&nb, d_nbirths_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }
    if (nb <= synced_births_) return;
    std::vector<BirthRec> recs(size_t(nb - synced_births_));
    CK(cudaMemcpyAsync(recs.data(), d_births_ + synced_births_, recs.size() * sizeof(BirthRec),
                       cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
    stats_.d2h_bytes += sizeof(int) + recs.size() * sizeof(BirthRec);
    for (const BirthRec& r : recs) {
        const int s = r.slot;
        if (free_slots_.empty() || free_slots_.back() != s)
            throw std::runtime_error("device expansion: slot order diverged from the host mirror");
        free_slots_.pop_back();
        SlotInfo& si = slots_[s];
        si = SlotInfo{};
        si.c = {r.x, r.y, r.z};
        si.birth = long(r.it);
        si.fluid = r.fluid;
        si.has_solid = r.has_solid != 0;
        si.owner = r.owner;
        si.rank = r.owner % world_;
        si.local = r.local;
        si.log_index = log_.size();
        log_.push_back({long(r.it), si.c, r.trigger, r.owner});
        grid_slot_[lin(si.c)] = s;
        ++per_dev_[size_t(r.owner)];
        next_local_[size_t(si.rank)] = r.local + 1;
        h_mode_[s] = long(r.it) >= iteration_ ? MODE_GEN_AMBIENT : MODE_PULL;
        h_has_solid_[s] = uint8_t(r.has_solid);
        h_coords_[3 * size_t(s)] = r.x;
        h_coords_[3 * size_t(s) + 1] = r.y;
        h_coords_[3 * size_t(s) + 2] = r.z;
        h_lidx_[s] = si.rank == rank_ ? r.local : -1;
        active_cells_ += uint64_t(r.fluid);
        if (si.rank == rank_) local_cells_ += uint64_t(r.fluid);
    }
    all_active_.clear();
    active_.clear();
    for (size_t k = 0; k < grid_slot_.size(); ++k)
        if (grid_slot_[k] >= 0) {
            all_active_.push_back(grid_slot_[k]);
            if (slots_[grid_slot_[k]].rank == rank_) active_.push_back(grid_slot_[k]);
        }
    recompute_step_bytes();
    synced_births_ = nb;
    launch_tiles_ = std::min(cap_, int(all_active_.size()) + expand_headroom());
    ensure_pool(launch_tiles_);
}

void Engine::launch_check_expand(long it) {
    ExpandDev x = expand_dev();
    if (world_ > 1) {  // this step's parity of every rank's trigger bytes
        const size_t par = size_t(it & 1);
        for (int r = 0; r < world_; ++r) {
            x.ptrig[r] = reinterpret_cast<const uint8_t*>(peer_sync_[r] + SYNC_TRIG) + par * trig_bytes_;
            x.perr[r] = peer_sync_[r] + 8;
            x.psnap[r] = peer_sync_[r] + SYNC_SNAP + par * CNT_N;
        }
        x.trig_clear = d_trig_ + (par ^ 1) * trig_bytes_;
    }
    switch (E_) {
    case 8: k_check_expand<8><<<1, 1024, 0, stream_>>>(d_, x, it, d_halt_); break;
    case 16: k_check_expand<16><<<1, 1024, 0, stream_>>>(d_, x, it, d_halt_); break;
    case 32: k_check_expand<32><<<1, 1024, 0, stream_>>>(d_, x, it, d_halt_); break;
    default: k_check_expand<64><<<1, 1024, 0, stream_>>>(d_, x, it, d_halt_); break;
    }
}

ExpandDev Engine::expand_dev() const {
    ExpandDev x{};
    x.gslot = d_gslot_;
    x.cand = d_cand_;
    x.active = world_ > 1 ? d_all_active_ : d_active_;
    x.nactive = world_ > 1 ? d_nall_ : d_nactive_;
    x.lactive = d_active_;
    x.nlactive = d_nactive_;
    x.world = world_;
    x.rank = rank_;
    x.merged = d_merged_;
    x.merr = d_sync_ + 9;
    x.gcnt = d_gcnt_;
    for (int r = 0; r < world_; ++r) {
        x.peer_f[r] = peer_f_[r];
        x.peer_pf[r] = peer_pf_[r];
    }
    x.next_slot = d_next_slot_;
    x.next_local = d_next_local_;
    x.owner = d_owner_;
    x.coords = d_coords_;
    x.mode = d_mode_;
    x.has_solid = d_has_solid_;
    x.no_fluid = d_no_fluid_;
    x.solid = d_solid_;
    x.lidx = d_lidx_;
    x.route_psi = d_route_[ROUTE_PSI];
    x.route_w = d_route_[ROUTE_W];
    x.nbuf = nbuf_;
    x.bmask = d_bmask_;
    x.omask = d_omask_;
    for (int b = 0; b < 2; ++b) {
        x.slot_f[b] = d_slot_f_[b];
        x.slot_pf[b] = d_slot_pf_[b];
    }
    x.pool_f = d_pool_f_;
    x.pool_pf = d_pool_pf_;
    x.per_slot = per_slot_;
    x.per_pf = per_pf_;
    x.lcap = lcap_;
    x.geom = d_geomdev_;
    x.p2p = d_p2p_;
    x.per_dev = d_per_dev_;
    x.acc = d_acc_;
    x.births = d_births_;
    x.nbirths = d_nbirths_;
    x.post_flags = d_post_flags_;
    x.capture = d_capture_;
    x.cap = cap_;
    x.amb = amb_;
    x.devices = devices_;
    x.policy = policy_;
    x.max_active = launch_tiles_;
    x.solid_words = solid_words_;
    for (int a = 0; a < 3; ++a) {
        x.periodic[a] = periodic_[a];
        x.dom[a] = dom_[a];
    }
    x.w_p2p = w_p2p_;
    x.w_staged = w_staged_;
    x.face_xfer = face_xfer_;
    return x;
}

void Engine::launch_face(int src, int flags, long iter) {
    if (active_.empty()) return;
    EvPair* ev = profiling_ ? &next_event(1, 0) : nullptr;
    if (ev) CK(cudaEventRecord(ev->a, stream_));
    K_.face(d_, d_active_, src, flags, iter, unsigned(dev_expand_ && d_.nactive ? launch_bound() : int(active_.size())),
            stream_);
    CK(cudaGetLastError());
    ++stats_.kernels_launched;
    if (ev) CK(cudaEventRecord(ev->b, stream_));
}

// P5 of step `iter` (k_p5): exact moments check of the tiles the fused
// kernel's screen marked, on the post-stream state in buffer cur_.
void Engine::launch_p5(long iter) {
    if (active_.empty()) return;
    K_.p5(d_, d_active_, cur_, iter, unsigned(dev_expand_ && d_.nactive ? launch_bound() : int(active_.size())),
          stream_);
    CK(cudaGetLastError());
    ++stats_.kernels_launched;
}

void Engine::launch_main(long iter) {
    if (active_.empty()) return;
    EvPair* ev = profiling_ ? &next_event(0, local_cells_) : nullptr;
    if (ev) CK(cudaEventRecord(ev->a, stream_));
    const int wu = mode_ == PLBM_MODE_PROGRESSIVE ? 1 : 0;
    MainFn fn = K_.main_plain;
    // single rank: the pc kernels run the face pass themselves (no k_face)
    const auto fusable = [&](MainFn f) { return world_ == 1 && f && (f == K_.main_pc || f == K_.main_pc2 || f == K_.main_pc_late) && !dev_expand_; };
    // clusters per tile: variant 20 = 1 (whole tiles), 26 = 2, 27 = the finest (E / 8), 0 = the default split_
    const int split = variant_ == 20 ? 1 : variant_ == 26 ? 2 : variant_ == 27 ? 4 : split_;
    const int sj = split == 2 ? 0 : split == 4 ? 1 : -1;
    if (variant_ == 0 || variant_ == 20 || variant_ == 26 || variant_ == 27) {
        if (sj >= 0 && K_.main_pc_split[sj] && !fuse_) fn = K_.main_pc_split[sj];
        else if (K_.main_pc) fn = K_.main_pc;
    }
    if (K_.main_pc_late && variant_ == 21) fn = K_.main_pc_late;
    if (K_.main_pc_mem && variant_ == 24) fn = K_.main_pc_mem;  // probe: not a correct step
    if (K_.main_pc2 && variant_ == 22) fn = K_.main_pc2;
    if (aa_) fn = (sj >= 0 && K_.main_aa_split[sj][0] ? K_.main_aa_split[sj]
                   : K_.main_aa[0] ? K_.main_aa : K_.main_aa_split[1])[aa_kind(1, iter) - 1];
    face_fused_ = fusable(fn) && fuse_;
    // the pc kernels write the xcol side buffers the face pass reads
    d_.xcol_ok = (fn == K_.main_pc || fn == K_.main_pc_split[0] || fn == K_.main_pc_split[1] ||
                  fn == K_.main_pc2 || fn == K_.main_pc_late || fn == K_.main_pc_mem ||
                  (aa_ && K_.aa_xcol)) && !no_xcol_;
    d_.face_flags = face_fused_ ? (FACE_FUSED | FACE_NAN | (mode_ == PLBM_MODE_PROGRESSIVE ? FACE_CRITERION : 0))
                                : 0;
    const int ntiles = dev_expand_ && d_.nactive ? launch_bound() : int(active_.size());
    fn(d_, d_active_, cur_, wu, iter, unsigned(ntiles), stream_);
    CK(cudaGetLastError());
    if (d_.npoke) {  // pokes apply to one step's f_in
        d_.npoke = 0;
        pokes_.clear();
    }
    ++stats_.kernels_launched;
    if (ev) CK(cudaEventRecord(ev->b, stream_));
}

Engine::EvPair& Engine::next_event(int kind, uint64_t cells) {
    if (ev_used_ == ev_pool_.size()) {
        if (ev_pool_.size() >= 8192 && !in_spec_) resolve_events();
        if (ev_used_ == ev_pool_.size()) {
            EvPair p;
            CK(cudaEventCreate(&p.a));
            CK(cudaEventCreate(&p.b));
            ev_pool_.push_back(p);
        }
    }
    EvPair& e = ev_pool_[ev_used_++];
    e.kind = kind;
    e.cells = cells;
    return e;
}

void Engine::resolve_events() {
    if (!ev_used_) return;
    CK(cudaStreamSynchronize(stream_));
    for (size_t k = 0; k < ev_used_; ++k) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_pool_[k].a, ev_pool_[k].b));
        if (ev_pool_[k].kind < 0) continue;  // a discarded speculative step (no-op launch)
        if (ev_pool_[k].kind == 0) {
            stats_.main_ms += ms;
            ++stats_.main_launches;
            stats_.main_cell_updates += ev_pool_[k].cells;
        } else {
            stats_.face_ms += ms;
            ++stats_.face_launches;
        }
    }
    ev_used_ = 0;
}

plbm_kernel_stats Engine::stats() {
    resolve_events();
    return stats_;
}

void Engine::check_error(plbm_error* err, bool& failed) {
    unsigned long long h_err = ERR_NONE_KEY;
    // several ranks: the merged key of the last device check (identical on
    // every rank, so every rank raises the same EngineError)
    CK(cudaMemcpyAsync(&h_err, world_ > 1 && in_spec_ ? err_word() : d_err_, sizeof h_err, cudaMemcpyDeviceToHost,
                       stream_));
    stats_.d2h_bytes += sizeof h_err;
    CK(cudaStreamSynchronize(stream_));
    if (world_ > 1 && !in_spec_ && peers_ready()) {
        // host-merge protocol (step_end after the trigger all-reduce: every
        // rank's face pass of this step is complete): the lowest key of all
        // ranks, read from the peers' sync blocks; a peer may already have
        // recorded a key of the next step, which does not count yet
        const unsigned long long lim = (unsigned long long)(iteration_ + 2) << 37;
        for (int r = 0; r < world_; ++r) {
            if (r == rank_) continue;
            unsigned long long k = ERR_NONE_KEY;
            CK(cudaMemcpy(&k, peer_sync_[r] + 8, sizeof k, cudaMemcpyDefault));
            if (k < lim && k < h_err) h_err = k;
        }
    }
    failed = h_err != ERR_NONE_KEY;
    if (!failed) return;
    const int code = int(h_err & 0xf);
    const long tl = long((h_err >> 4) & 0xffffffffull);
    const long it = long(h_err >> 37);
    err_it_ = it;
    err_p5_ = code == ERR_P5_NAN;
    const int tx = int(tl / (long(grid_[1]) * grid_[2]));
    const int ty = int((tl / grid_[2]) % grid_[1]);
    const int tz = int(tl % grid_[2]);
    const char* phase = code == ERR_P5_NAN ? "P5" : code == ERR_PEER_TIMEOUT ? "sync" : "P1";
    const char* what = code == ERR_P1_NAN         ? "NaN in density"
                       : code == ERR_P1_POLE      ? "pr_pressure: b*rho >= 1 (EOS pole)"
                       : code == ERR_PEER_TIMEOUT ? "a peer rank did not reach the step barrier"
                                                  : "NaN in moments";
    if (err) {
        std::memset(err, 0, sizeof *err);
        err->code = 1;
        err->tile[0] = tx;
        err->tile[1] = ty;
        err->tile[2] = tz;
        err->iteration = it;
        std::snprintf(err->phase, sizeof err->phase, "%s", phase);
        std::snprintf(err->message, sizeof err->message, "iteration %ld, tile (%d,%d,%d), phase %s: %s",
                      it, tx, ty, tz, phase, what);
    }
    // One rank: clear the key so the engine can go on.  Several ranks: a peer
    // may still have to read this rank's key (its device check or step_end
    // can run after this host saw the error), so the key stays; it carries
    // its iteration and every reader filters by iteration, and a multi-rank
    // engine that raised an EngineError stays failed (the reference's state
    // after an EngineError is not stepped further either).
    if (world_ == 1) reset_err();
    CK(cudaStreamSynchronize(stream_));
}

// Error key words to "no error" (ERR_NONE_KEY: 0x7fff..ff, little endian).
void Engine::reset_err() {
    CK(cudaMemsetAsync(d_sync_ + 8, 0xff, 2 * sizeof(unsigned long long), stream_));
    CK(cudaMemsetAsync(reinterpret_cast<uint8_t*>(d_sync_ + 8) + 7, 0x7f, 1, stream_));
    CK(cudaMemsetAsync(reinterpret_cast<uint8_t*>(d_sync_ + 9) + 7, 0x7f, 1, stream_));
}

void Engine::rank_barrier(long it, bool snapshot) {
    PeerFlags pf{};
    for (int r = 0; r < world_; ++r) pf.p[r] = peer_sync_[r];
    unsigned long long* snap = snapshot ? d_sync_ + SYNC_SNAP + size_t(it & 1) * CNT_N : nullptr;
    static const unsigned long long timeout_ns = [] {
        const char* t = std::getenv("PLBM_BARRIER_TIMEOUT_S");
        return (unsigned long long)((t ? std::atof(t) : 120.0) * 1e9);
    }();
    k_rank_barrier<<<1, 32, 0, stream_>>>(d_sync_, pf, world_, rank_, ++epoch_, d_err_, it, timeout_ns, d_cnt_,
                                          snap);
    CK(cudaGetLastError());
    ++stats_.kernels_launched;
}

// proj/src/tilemap.cpp:220-266 + proj/src/engine.cpp:554-560
void Engine::expand(const std::vector<std::pair<Coord, int>>& triggers, long iteration,
                    std::vector<int>& created) {
    struct Resolved {
        Coord target, source;
        int face;
        bool in_bounds;
    };
    std::vector<Resolved> rs;
    rs.reserve(triggers.size());
    for (const auto& [src, face] : triggers) {
        Coord t{};
        const bool ok = neighbor_coords(src, face, t);
        rs.push_back({ok ? t : Coord{}, src, face, ok});
    }
    std::sort(rs.begin(), rs.end(), [](const Resolved& a, const Resolved& b) {
        if (a.in_bounds != b.in_bounds) return a.in_bounds > b.in_bounds;
        if (a.target != b.target) return a.target < b.target;
        if (a.source != b.source) return a.source < b.source;
        return a.face < b.face;
    });
    const Coord* last = nullptr;
    for (const auto& r : rs) {
        if (!r.in_bounds) {
            ++suppressed_;
            continue;
        }
        if (last && r.target == *last) continue;
        last = &r.target;
        if (slot_at(r.target) >= 0) continue;
        created.push_back(create_tile(r.target, iteration, r.face));
    }
    std::sort(created.begin(), created.end(),
              [&](int a, int b) { return slots_[a].c < slots_[b].c; });
}

// Engine::step() in three parts so ranks can synchronise between them:
//   step_main  the fused kernel of this rank's tiles (reads peers' f_post^(k-1)
//              and psi faces of step k, all complete before the previous
//              step's trigger all-reduce)
//   -- cross-rank barrier: k_face pulls peers' f_post^(k) --
//   step_face  face pre-pass: psi faces for k+1, criterion, local trigger bits
//   -- trigger all-reduce --
//   step_end   expansion on the merged bits (touches nothing peers read)
int Engine::step_main(plbm_error* err) {
    if (!prepared_) {
        if (err) {
            std::memset(err, 0, sizeof *err);
            err->code = 2;
            std::snprintf(err->message, sizeof err->message,
                          "engine not prepared (attach peers, then plbm_gpu_prepare on every rank)");
        }
        return 2;
    }
    if (phase_ != 0) return 0;
    const long it = iteration_ + 1;
    launch_main(it);
    cur_ ^= 1;
    if (post_pending_) {  // the mode / route catch-up upload_expand_state left to the device
        const int nslot = cap_ + 1;
        k_post_main<<<std::max(1, std::min(256, (nslot * 18 + 255) / 256)), 256, 0, stream_>>>(
            d_mode_, d_route_[ROUTE_PULL], d_route_[ROUTE_PSI], nslot, d_post_flags_, d_halt_);
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(d_post_flags_, 0, sizeof(int), stream_));
        ++stats_.kernels_launched;
        post_pending_ = false;
        std::fill(h_mode_.begin(), h_mode_.end(), uint8_t(MODE_PULL));  // the mirror of its mode reset
    }
    if (any_gen_) {
        CK(cudaMemsetAsync(d_mode_, MODE_PULL, size_t(cap_ + 1), stream_));
        std::fill(h_mode_.begin(), h_mode_.end(), uint8_t(MODE_PULL));
        any_gen_ = false;
    }
    if (routes_differ_) {
        CK(cudaMemcpyAsync(d_route_[ROUTE_PULL], d_route_[ROUTE_PSI], size_t(cap_ + 1) * 18 * sizeof(int),
                           cudaMemcpyDeviceToDevice, stream_));
        routes_differ_ = false;
    }
    phase_ = 1;
    return 0;
}

int Engine::step_face() {
    if (phase_ != 1) return 0;
    if (!face_fused_) launch_face(cur_, mode_ == PLBM_MODE_PROGRESSIVE ? 3 : 2, iteration_ + 1);
    launch_p5(iteration_ + 1);
    phase_ = 2;
    return 0;
}

int Engine::step_begin(plbm_error* err) {
    const int rc = step_main(err);
    if (rc) return rc;
    return step_face();
}

// Second half: error check, then (progressive) expansion on the merged
// trigger bits of all ranks.  `merged` = host copy of the all-reduced trigger
// array, or NULL to read it from this engine's device array (single rank, or a
// caller that all-reduced d_trig_ in place).
int Engine::step_end(const uint8_t* merged, plbm_error* err) {
    if (phase_ != 2) return 0;
    phase_ = 0;
    const long it = iteration_ + 1;
    bool failed = false;
    check_error(err, failed);
    if (failed) {
        // P2 and P4 recorded this step's exchanges before P5 threw
        if (err_p5_)
            for (int a = 0; a < 3; ++a) bytes_[a] += step_bytes_[a];
        return 1;
    }
    const uint64_t updates = active_cells_;
    for (int a = 0; a < 3; ++a) bytes_[a] += step_bytes_[a];
    if (mode_ == PLBM_MODE_PROGRESSIVE) {
        std::vector<uint8_t> trig;
        if (!merged) {
            trig.resize(trig_bytes_);
            CK(cudaMemcpyAsync(trig.data(), d_trig_, trig_bytes_, cudaMemcpyDeviceToHost, stream_));
            stats_.d2h_bytes += trig_bytes_;
            CK(cudaStreamSynchronize(stream_));
            merged = trig.data();
        }
        host_expand(merged, it);
    }
    ++iteration_;
    cell_updates_ += updates;
    return 0;
}

// expand + assign_owner on the host mirror from a (merged) trigger array,
// then clear the device triggers (tilemap.cpp:220-266, engine.cpp:30-41).
void Engine::host_expand(const uint8_t* merged, long it) {
    std::vector<std::pair<Coord, int>> triggers;
    for (int s : all_active_)
        for (int f = 0; f < 6; ++f)
            if (merged[s] & (1u << f)) triggers.push_back({slots_[s].c, f});
    if (world_ > 1 && in_spec_) {
        // device protocol, host fallback after a halt at step `it`: a slower
        // peer's k_check_expand may still read this rank's bytes of step it,
        // so only the next step's parity is cleared here (step it's bytes are
        // cleared by this rank's check of step it + 1, after its barrier)
        CK(cudaMemsetAsync(d_trig_ + size_t((it + 1) & 1) * trig_bytes_, 0, trig_bytes_, stream_));
    } else {
        CK(cudaMemsetAsync(d_trig_, 0, (world_ > 1 ? 2 : 1) * trig_bytes_, stream_));
    }
    if (!triggers.empty()) {
        std::vector<int> created;
        expand(triggers, it, created);
        for (int s : created) assign_owner(s);
        if (!created.empty()) upload_map(created, false);
    }
}

// One step's launches (= step_main + step_face of a single rank).
void Engine::enqueue_step(long it) {
    if (world_ > 1) {
        const std::pair<int, long> delay = [] {
            const char* v = std::getenv("PLBM_TEST_RANK_DELAY_US");
            if (!v) return std::pair<int, long>(-1, 0);
            const char* c = std::strchr(v, ':');
            return std::pair<int, long>(std::atoi(v), c ? std::atol(c + 1) : 0);
        }();
        if (delay.first == rank_ && delay.second > 0) {
            k_spin<<<1, 1, 0, stream_>>>((unsigned long long)delay.second * 1000ull);
            CK(cudaGetLastError());
        }
    }
    launch_main(it);
    cur_ ^= 1;
    if (dev_expand_) {
        const int nslot = cap_ + 1;
        k_post_main<<<std::max(1, std::min(256, (nslot * 18 + 255) / 256)), 256, 0, stream_>>>(
            d_mode_, d_route_[ROUTE_PULL], d_route_[ROUTE_PSI], nslot, d_post_flags_, d_halt_);
        CK(cudaGetLastError());
        ++stats_.kernels_launched;
    }
    if (any_gen_) {
        CK(cudaMemsetAsync(d_mode_, MODE_PULL, size_t(cap_ + 1), stream_));
        std::fill(h_mode_.begin(), h_mode_.end(), uint8_t(MODE_PULL));
        any_gen_ = false;
    }
    if (routes_differ_) {
        CK(cudaMemcpyAsync(d_route_[ROUTE_PULL], d_route_[ROUTE_PSI], size_t(cap_ + 1) * 18 * sizeof(int),
                           cudaMemcpyDeviceToDevice, stream_));
        routes_differ_ = false;
    }
    const int fflags = mode_ == PLBM_MODE_PROGRESSIVE ? 3 : 2;
    if (world_ > 1) {
        rank_barrier(it);  // every rank's f_post^(it) is complete (k_face pulls across ranks)
        d_.trig = d_trig_ + size_t(it & 1) * trig_bytes_;
        launch_face(cur_, fflags, it);
        launch_p5(it);
        d_.trig = d_trig_;
        // every rank's triggers, error key, psi faces and diagnostics of it are final
        rank_barrier(it, true);
        gcnt_valid_ = true;
        return;
    }
    if (!face_fused_) launch_face(cur_, fflags, it);
    launch_p5(it);
}

// Progressive single-rank stepping without a host round trip per step: up to
// spec_depth_ steps are queued ahead.  After each step's face pass k_check
// decides on the device whether its triggers need the host (a birth, or an
// error); if so it sets a sticky halt flag that turns every step queued after
// it into a no-op, and the host — which retires steps in order from pinned
// copies of the flag — runs the expansion and resumes from the next step.
// Steps without births count their out-of-bounds triggers as suppressed
// expansions on the device.  Results are identical to stepping one at a time.
int Engine::step_speculative(int n, plbm_error* err) {
    struct Queued {
        long it;
        int cur_after;
        uint64_t updates;
        int flag;
        size_t ev_after;  // profiling events recorded up to and including this step
    };
    std::deque<Queued> q;
    d_.halt = d_halt_;
    if (dev_expand_) d_.nactive = d_nactive_;
    in_spec_ = true;
    int done = 0, enqueued = 0, flag_ctr = 0;
    int rc = 0;
    while (done < n) {
        while (int(q.size()) < spec_depth_ && enqueued < n) {
            Queued e{iteration_ + 1 + long(q.size()), 0, active_cells_, flag_ctr++ % 8, 0};
            enqueue_step(e.it);
            e.cur_after = cur_;
            e.ev_after = ev_used_;
            if (dev_expand_) launch_check_expand(e.it);
            else k_check<<<1, 256, 0, stream_>>>(d_, d_bmask_, d_omask_, cap_ + 1, d_halt_);
            CK(cudaGetLastError());
            ++stats_.kernels_launched;
            CK(cudaMemcpyAsync(&h_flags_[e.flag], d_halt_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
            if (dev_expand_)
                CK(cudaMemcpyAsync(&h_flags_[8 + e.flag], d_nbirths_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
            CK(cudaEventRecord(flag_ev_[e.flag], stream_));
            stats_.d2h_bytes += sizeof(int);
            q.push_back(e);
            ++enqueued;
        }
        const Queued e = q.front();
        q.pop_front();
        CK(cudaEventSynchronize(flag_ev_[e.flag]));
        if (dev_expand_) births_seen_ = h_flags_[8 + e.flag];
        if (h_flags_[e.flag] == 0) {  // final (births, if any, done on the device)
            iteration_ = e.it;
            if (!dev_expand_) {  // else counted by k_check_expand
                cell_updates_ += e.updates;
                for (int a = 0; a < 3; ++a) bytes_[a] += step_bytes_[a];
            }
            ++done;
            continue;
        }
        // halted at e: the steps queued after it did nothing
        enqueued -= int(q.size());
        q.clear();
        for (size_t k = e.ev_after; k < ev_used_; ++k) ev_pool_[k].kind = -1;
        cur_ = e.cur_after;
        bool failed = false;
        check_error(err, failed);  // synchronises the stream
        if (failed) {
            rc = 1;
            if (err_p5_) {  // P2 and P4 recorded this step's exchanges before P5 threw
                sync_births();
                for (int a = 0; a < 3; ++a) bytes_[a] += step_bytes_[a];
            }
            break;
        }
        iteration_ = e.it;
        if (!dev_expand_) {
            cell_updates_ += e.updates;
            for (int a = 0; a < 3; ++a) bytes_[a] += step_bytes_[a];
        }
        ++done;
        sync_births();  // the mirror catches up with the device's earlier births
        std::vector<uint8_t> trig(trig_bytes_);
        CK(cudaMemcpyAsync(trig.data(), world_ > 1 ? d_merged_ : d_trig_, world_ > 1 ? size_t(cap_ + 1) : trig_bytes_,
                           cudaMemcpyDeviceToHost, stream_));
        stats_.d2h_bytes += trig_bytes_;
        CK(cudaStreamSynchronize(stream_));
        host_expand(trig.data(), e.it);
        CK(cudaMemsetAsync(d_halt_, 0, sizeof(int), stream_));
    }
    if (!q.empty() || rc) CK(cudaStreamSynchronize(stream_));
    CK(cudaMemsetAsync(d_halt_, 0, sizeof(int), stream_));
    d_.halt = nullptr;
    d_.nactive = nullptr;
    in_spec_ = false;
    sync_births();
    return rc;
}

int Engine::step(int n, plbm_error* err) {
    if (world_ != 1 && !prepared_) {
        if (err) {
            std::memset(err, 0, sizeof *err);
            err->code = 2;
            std::snprintf(err->message, sizeof err->message,
                          "engine not prepared (attach peers, then plbm_gpu_prepare on every rank)");
        }
        return 2;
    }
    // several ranks: device-side barriers and expansion, steps queued ahead
    // (every rank must call plbm_gpu_step with the same n)
    if (world_ != 1 || (mode_ == PLBM_MODE_PROGRESSIVE && spec_depth_ > 1)) return step_speculative(n, err);
    if (mode_ == PLBM_MODE_PROGRESSIVE) {
        for (int k = 0; k < n; ++k) {
            int rc = step_begin(err);
            if (rc) return rc;
            rc = step_end(nullptr, err);
            if (rc) return rc;
        }
        return 0;
    }
    // Static meshes never change: the whole batch is queued without a host
    // round trip and the error flag (earliest iteration wins) is read once; a
    // recorded error halts the steps queued behind it (k_err_halt).
    const long it0 = iteration_;
    std::vector<int> cur_after;
    cur_after.reserve(size_t(n));
    d_.halt = d_halt_;
    int rc = 0;
    for (int k = 0; k < n; ++k) {
        rc = step_begin(err);
        if (rc) break;
        phase_ = 0;
        ++iteration_;  // (the next step's kernels run as iteration + 1)
        cur_after.push_back(cur_);
        k_err_halt<<<1, 1, 0, stream_>>>(d_err_, d_halt_);
        CK(cudaGetLastError());
        ++stats_.kernels_launched;
    }
    d_.halt = nullptr;
    if (rc) {
        iteration_ = it0;
        return rc;
    }
    if (n > 0) {
        bool failed = false;
        check_error(err, failed);
        CK(cudaMemsetAsync(d_halt_, 0, sizeof(int), stream_));
        const long bad = failed ? err_it_ : it0 + n + 1;
        const long done = std::max(0L, std::min(long(n), bad - 1 - it0));
        iteration_ = it0 + done;
        cell_updates_ += uint64_t(done) * active_cells_;
        for (int a = 0; a < 3; ++a) bytes_[a] += uint64_t(done + (failed && err_p5_ ? 1 : 0)) * step_bytes_[a];
        if (failed) {
            cur_ = cur_after[size_t(std::min(long(n), done + 1)) - 1];  // the failing step's output
            return 1;
        }
    }
    return 0;
}

int Engine::local_triggers(uint8_t* out, int n) {
    if (n < int(trig_bytes_)) return -1;
    CK(cudaMemcpyAsync(out, d_trig_, trig_bytes_, cudaMemcpyDeviceToHost, stream_));
    stats_.d2h_bytes += trig_bytes_;
    CK(cudaStreamSynchronize(stream_));
    return int(trig_bytes_);
}

int Engine::ipc_handles(void* out) const {
    cudaIpcMemHandle_t h[3];
    CK(cudaIpcGetMemHandle(&h[0], d_pool_f_));
    CK(cudaIpcGetMemHandle(&h[1], d_pool_pf_));
    CK(cudaIpcGetMemHandle(&h[2], d_sync_));
    std::memcpy(out, h, sizeof h);
    return int(sizeof h);
}

int Engine::open_peer(int rank, const void* handles) {
    if (rank < 0 || rank >= world_ || rank == rank_) return -1;
    cudaIpcMemHandle_t h[3];
    std::memcpy(h, handles, sizeof h);
    void* f = nullptr;
    void* pf = nullptr;
    void* sy = nullptr;
    CK(cudaIpcOpenMemHandle(&f, h[0], cudaIpcMemLazyEnablePeerAccess));
    CK(cudaIpcOpenMemHandle(&pf, h[1], cudaIpcMemLazyEnablePeerAccess));
    CK(cudaIpcOpenMemHandle(&sy, h[2], cudaIpcMemLazyEnablePeerAccess));
    peer_f_[rank] = static_cast<double*>(f);
    peer_pf_[rank] = static_cast<double*>(pf);
    peer_sync_[rank] = static_cast<unsigned long long*>(sy);
    peer_opened_[rank] = true;
    if (peers_ready()) upload_pointers();
    return 0;
}

int Engine::set_peer(int rank, void* pool_f, void* pool_pf) {
    if (rank < 0 || rank >= world_ || rank == rank_) return -1;
    peer_f_[rank] = static_cast<double*>(pool_f);
    peer_pf_[rank] = static_cast<double*>(pool_pf);
    if (peers_ready()) upload_pointers();
    return 0;
}

int Engine::set_peer_sync(int rank, void* sync) {
    if (rank < 0 || rank >= world_ || rank == rank_) return -1;
    peer_sync_[rank] = static_cast<unsigned long long*>(sync);
    if (peers_ready()) upload_pointers();
    return 0;
}

int Engine::rank_of(const int32_t* cc) const {
    const Coord c{cc[0], cc[1], cc[2]};
    if (c.x < 0 || c.y < 0 || c.z < 0 || c.x >= grid_[0] || c.y >= grid_[1] || c.z >= grid_[2])
        return -1;
    const int s = slot_at(c);
    return s < 0 ? -1 : slots_[s].rank;
}

void Engine::counters(plbm_counters* out) {
    std::memset(out, 0, sizeof *out);
    // every device word in one round trip: this rank's counters, the
    // job-wide diagnostics (several ranks), the device-side accumulators
    // (into pinned memory: true async copies, one synchronisation)
    unsigned long long* c = h_cnt_;
    unsigned long long* g = h_cnt_ + CNT_N;
    unsigned long long* acc = h_cnt_ + 2 * CNT_N;
    std::memset(h_cnt_, 0, (2 * CNT_N + 4) * sizeof(unsigned long long));
    const bool use_g = world_ > 1 && gcnt_valid_;
    CK(cudaMemcpyAsync(c, d_cnt_, CNT_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
    if (use_g) CK(cudaMemcpyAsync(g, d_gcnt_, CNT_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
    if (dev_expand_) CK(cudaMemcpyAsync(acc, d_acc_, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
    stats_.d2h_bytes += (CNT_N + (use_g ? CNT_N : 0) + (dev_expand_ ? 4 : 0)) * sizeof(unsigned long long);
    out->iteration = iteration_;
    out->cell_updates = cell_updates_;
    out->negative_populations = c[CNT_NEG];  // this rank's tiles (one rank: all)
    out->psi_clamps = c[CNT_CLAMP];
    out->zero_rho_forcings = c[CNT_ZERO_RHO];
    if (use_g) {  // job-wide sums of the last step (k_check_expand)
        out->negative_populations = g[CNT_NEG];
        out->psi_clamps = g[CNT_CLAMP];
        out->zero_rho_forcings = g[CNT_ZERO_RHO];
    }
    out->suppressed_expansions = suppressed_ + c[CNT_SUPP];  // host expand + device k_check
    for (int a = 0; a < 3; ++a) out->bytes[a] = bytes_[a];
    if (dev_expand_) {  // accumulated by k_check_expand
        out->cell_updates += acc[0];
        for (int a = 0; a < 3; ++a) out->bytes[a] += acc[1 + a];
    }
    out->tiles = all_active_.size();
    out->active_cells = active_cells_;
    const uint64_t gc = uint64_t(E_ + 2) * (E_ + 2) * (E_ + 2);
    out->bytes_resident = out->tiles * gc * (uint64_t(C_) * (2 * Q + 8) * 8 + 1);  // tile.cpp:7-13
}

int Engine::tiles(int32_t* coords, int32_t* owners, int64_t* births, int max) const {
    int k = 0;
    for (int s : all_active_) {
        if (k < max) {
            if (coords) {
                coords[3 * k] = slots_[s].c.x;
                coords[3 * k + 1] = slots_[s].c.y;
                coords[3 * k + 2] = slots_[s].c.z;
            }
            if (owners) owners[k] = slots_[s].owner;
            if (births) births[k] = slots_[s].birth;
        }
        ++k;
    }
    return k;
}

int Engine::read_tile(const int32_t* cc, int comp, int field, double* out) {
    const Coord c{cc[0], cc[1], cc[2]};
    if (c.x < 0 || c.y < 0 || c.z < 0 || c.x >= grid_[0] || c.y >= grid_[1] || c.z >= grid_[2])
        return -1;
    const int s = slot_at(c);
    if (s < 0) return -1;
    if (comp < 0 || comp >= C_) return -2;
    if (field < 0 || field > PLBM_FIELD_PSI) return -3;
    if (slots_[s].rank != rank_) return -7;  // fields live on the owner rank
    if (!peers_ready()) return -8;
    if (field == PLBM_FIELD_PSI || field >= PLBM_FIELD_PUX) {
        if (!d_capture_) return -4;
        const int which = field == PLBM_FIELD_PSI ? 0 : 1 + (field - PLBM_FIELD_PUX);
        CK(cudaMemcpyAsync(out,
                           d_capture_ + (size_t(slots_[s].local) * C_ + comp) * 4 * E3_ + size_t(which) * E3_,
                           size_t(E3_) * sizeof(double), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        return 0;
    }
    K_.readback(d_, s, comp, cur_, d_readback_, aa_kind(d_.aa, iteration_ + 1), stream_);
    CK(cudaGetLastError());
    ++stats_.kernels_launched;
    if (field == PLBM_FIELD_F) {
        CK(cudaMemcpyAsync(out, d_readback_, size_t(19) * E3_ * sizeof(double), cudaMemcpyDeviceToHost,
                           stream_));
    } else {
        const int which = field == PLBM_FIELD_RHO ? 19 : 20 + (field - PLBM_FIELD_UX);
        CK(cudaMemcpyAsync(out, d_readback_ + size_t(which) * E3_, size_t(E3_) * sizeof(double),
                           cudaMemcpyDeviceToHost, stream_));
    }
    CK(cudaStreamSynchronize(stream_));
    return 0;
}

// gather_field (dump.cpp:21-57): the whole domain, x fastest, ambient fill.
int Engine::gather_field(const char* field, int comp, double* grid) {
    const std::string f = field ? field : "";
    const int kind = f == "rho" ? 0 : f == "u_magnitude" ? 1 : f == "psi" ? 2 : -1;
    if (kind < 0) return -3;
    if (comp < 0 || comp >= C_) return -2;
    if (world_ != 1) return -7;
    if (kind == 2 && !d_capture_) return -4;
    // dump.cpp:15-20 ambient_fill: rho_ambient / psi_ambient / 0
    const double fill = kind == 0 ? params_.comp[comp].rho_amb : kind == 2 ? params_.comp[comp].psi_amb : 0.0;
    const size_t n = size_t(dom_[0]) * dom_[1] * dom_[2];
    double* d_grid = nullptr;
    CK(cudaMallocAsync(&d_grid, n * sizeof(double), stream_));
    k_fill<<<148 * 8, 256, 0, stream_>>>(d_grid, n, fill);
    if (!active_.empty())
        K_.gather(d_, d_active_, int(active_.size()), kind, comp, cur_, d_grid, dom_[0], dom_[1],
                  aa_kind(d_.aa, iteration_ + 1), stream_);
    CK(cudaGetLastError());
    stats_.kernels_launched += 2;
    CK(cudaMemcpyAsync(grid, d_grid, n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    CK(cudaFreeAsync(d_grid, stream_));
    CK(cudaStreamSynchronize(stream_));
    stats_.d2h_bytes += n * sizeof(double);
    return 0;
}

// dump_field (dump.cpp:59-125): <base>.raw (float64 grid), <base>.meta and,
// with_pgm, <base>.pgm (mid-z slice, min-max normalised to 8 bits), byte for
// byte the files the reference writes.
int Engine::dump_field(const char* field, int comp, long iteration, const char* base, int with_pgm) {
    std::vector<double> grid(size_t(dom_[0]) * dom_[1] * dom_[2]);
    const int rc = gather_field(field, comp, grid.data());
    if (rc) return rc;
    const std::string b = base;
    {
        FILE* fp = std::fopen((b + ".raw").c_str(), "wb");
        if (!fp) return -5;
        const size_t w = std::fwrite(grid.data(), sizeof(double), grid.size(), fp);
        std::fclose(fp);
        if (w != grid.size()) return -5;
    }
    double lo = grid[0], hi = grid[0];
    if (with_pgm)
        for (double v : grid) {
            lo = std::min(lo, v);
            hi = std::max(hi, v);
        }
    const std::string fs = field;
    const double fill = fs == "rho" ? params_.comp[comp].rho_amb : fs == "psi" ? params_.comp[comp].psi_amb : 0.0;
    {
        FILE* fp = std::fopen((b + ".meta").c_str(), "w");
        if (!fp) return -5;
        // std::ostream with precision(17), default float field == %.17g
        std::fprintf(fp, "dims %d %d %d\nfield %s\ncomponent %d\niteration %ld\nfill %.17g\n"
                         "layout x-fastest float64 little-endian\n",
                     dom_[0], dom_[1], dom_[2], field, comp, iteration, fill);
        if (with_pgm) std::fprintf(fp, "pgm_min %.17g\npgm_max %.17g\n", lo, hi);
        std::fclose(fp);
    }
    if (with_pgm) {
        FILE* fp = std::fopen((b + ".pgm").c_str(), "wb");
        if (!fp) return -5;
        std::fprintf(fp, "P5\n%d %d\n255\n", dom_[0], dom_[1]);
        const size_t z = size_t(dom_[2] / 2);
        const double scale = hi > lo ? 255.0 / (hi - lo) : 0.0;
        std::vector<uint8_t> row(static_cast<size_t>(dom_[0]));
        for (int y = 0; y < dom_[1]; ++y) {
            for (int x = 0; x < dom_[0]; ++x) {
                const double v = grid[size_t(x) + size_t(dom_[0]) * (size_t(y) + size_t(dom_[1]) * z)];
                row[size_t(x)] = uint8_t(std::lround((v - lo) * scale));
            }
            std::fwrite(row.data(), 1, row.size(), fp);
        }
        std::fclose(fp);
    }
    return 0;
}

int Engine::creation_log(plbm_creation_event* out, int max) const {
    for (size_t k = 0; k < log_.size() && int(k) < max; ++k) {
        out[k].iteration = log_[k].iteration;
        out[k].coords[0] = log_[k].c.x;
        out[k].coords[1] = log_[k].c.y;
        out[k].coords[2] = log_[k].c.z;
        out[k].trigger = log_[k].trigger;
        out[k].owner = log_[k].owner;
        out[k].pad = 0;
    }
    return int(log_.size());
}

int Engine::set_capture(bool on) {
    if (on && !d_capture_) {
        const size_t n = size_t(lcap_ + 1) * C_ * 4 * E3_;
        d_capture_ = dmalloc<double>(n);
        CK(cudaMemsetAsync(d_capture_, 0, n * sizeof(double), stream_));
        CK(cudaStreamSynchronize(stream_));
    } else if (!on && d_capture_) {
        CK(cudaStreamSynchronize(stream_));
        cudaFree(d_capture_);
        d_capture_ = nullptr;
    }
    d_.capture = d_capture_;
    return 0;
}

// proj/tests/test_engine.cpp:284-310: overwrite one population of f_read
// (the pulled f_in of the next step) at an interior cell of a tile.
int Engine::poke_f(const int32_t* cc, int comp, int i, const int32_t* local, double v) {
    const Coord c{cc[0], cc[1], cc[2]};
    if (c.x < 0 || c.y < 0 || c.z < 0 || c.x >= grid_[0] || c.y >= grid_[1] || c.z >= grid_[2]) return -1;
    const int s = slot_at(c);
    if (s < 0) return -1;
    if (comp < 0 || comp >= C_ || i < 0 || i >= Q) return -2;
    for (int a = 0; a < 3; ++a)
        if (local[a] < 0 || local[a] >= E_) return -3;
    if (pokes_.size() >= 64) return -4;
    pokes_.push_back({s, comp, i, (local[2] * E_ + local[1]) * E_ + local[0], v});
    CK(cudaMemcpyAsync(d_pokes_, pokes_.data(), pokes_.size() * sizeof(Poke), cudaMemcpyHostToDevice, stream_));
    CK(cudaStreamSynchronize(stream_));
    d_.pokes = d_pokes_;
    d_.npoke = int(pokes_.size());
    return 0;
}

}  // namespace plbm

// ---------------------------------------------------------------------------
// C-ABI

namespace {
void fill_err(plbm_error* e, int code, const char* msg) {
    if (!e) return;
    std::memset(e, 0, sizeof *e);
    e->code = code;
    std::snprintf(e->message, sizeof e->message, "%s", msg);
}
plbm::Engine* EG(void* h) { return static_cast<plbm::Engine*>(h); }
}  // namespace

extern "C" {

void* plbm_gpu_create_ex(const plbm_scenario_desc* desc, int device, int rank, int world,
                         const plbm_gpu_options* opt, plbm_error* err) {
    fill_err(err, 0, "");
    try {
        const int storage = opt ? opt->storage : PLBM_STORAGE_AB;
        if (storage != PLBM_STORAGE_AB && storage != PLBM_STORAGE_AA)
            throw std::invalid_argument("unknown storage kind");
        return new plbm::Engine(*desc, device, rank, world, storage);
    } catch (const plbm::CudaError& e) {
        fill_err(err, 3, e.what());
    } catch (const std::exception& e) {
        fill_err(err, 2, e.what());
    }
    return nullptr;
}

void* plbm_gpu_create_dist(const plbm_scenario_desc* desc, int device, int rank, int world,
                           plbm_error* err) {
    fill_err(err, 0, "");
    try {
        return new plbm::Engine(*desc, device, rank, world);
    } catch (const plbm::CudaError& e) {
        fill_err(err, 3, e.what());
    } catch (const std::exception& e) {
        fill_err(err, 2, e.what());
    }
    return nullptr;
}

void* plbm_gpu_create(const plbm_scenario_desc* desc, int device, plbm_error* err) {
    return plbm_gpu_create_dist(desc, device, 0, 1, err);
}

int plbm_gpu_prepare(void* h) {
    try {
        return EG(h)->prepare();
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_step(void* h, int n, plbm_error* err) {
    fill_err(err, 0, "");
    try {
        return EG(h)->step(n, err);
    } catch (const std::exception& e) {
        fill_err(err, 3, e.what());
        return 3;
    }
}

int plbm_gpu_step_begin(void* h, plbm_error* err) {
    fill_err(err, 0, "");
    try {
        return EG(h)->step_begin(err);
    } catch (const std::exception& e) {
        fill_err(err, 3, e.what());
        return 3;
    }
}

int plbm_gpu_step_main(void* h, plbm_error* err) {
    fill_err(err, 0, "");
    try {
        return EG(h)->step_main(err);
    } catch (const std::exception& e) {
        fill_err(err, 3, e.what());
        return 3;
    }
}

int plbm_gpu_step_face(void* h) {
    try {
        return EG(h)->step_face();
    } catch (const std::exception&) {
        return 3;
    }
}

int plbm_gpu_step_end(void* h, const uint8_t* merged, plbm_error* err) {
    fill_err(err, 0, "");
    try {
        return EG(h)->step_end(merged, err);
    } catch (const std::exception& e) {
        fill_err(err, 3, e.what());
        return 3;
    }
}

int plbm_gpu_trigger_bytes(void* h) { return EG(h)->trig_bytes(); }
void* plbm_gpu_triggers_device(void* h) { return EG(h)->trig_device(); }

int plbm_gpu_local_triggers(void* h, uint8_t* out, int n) {
    try {
        return EG(h)->local_triggers(out, n);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_ipc_handles(void* h, void* out) {
    try {
        return EG(h)->ipc_handles(out);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_open_peer(void* h, int rank, const void* handles) {
    try {
        return EG(h)->open_peer(rank, handles);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_set_peer_pools(void* h, int rank, void* pool_f, void* pool_pf) {
    try {
        return EG(h)->set_peer(rank, pool_f, pool_pf);
    } catch (const std::exception&) {
        return -6;
    }
}

void plbm_gpu_pool_pointers(void* h, void** pool_f, void** pool_pf) { EG(h)->pool_pointers(pool_f, pool_pf); }
void* plbm_gpu_sync_block(void* h) { return EG(h)->sync_block(); }
int plbm_gpu_set_peer_sync(void* h, int rank, void* sync_block) {
    try {
        return EG(h)->set_peer_sync(rank, sync_block);
    } catch (const std::exception&) {
        return -6;
    }
}

void plbm_gpu_exchange_bytes(void* h, uint64_t* out) { EG(h)->exchange_bytes(out); }

// measurement hook (PLBM_PROBE set at create): per-CTA {smid, start ns, end ns}
// of the last fused-kernel launch; returns the number of CTAs recorded.
int plbm_gpu_probe(void* h, uint64_t* out, int max) { return EG(h)->probe(out, max); }

int plbm_gpu_gather_field(void* h, const char* field, int comp, double* grid) {
    try {
        return EG(h)->gather_field(field, comp, grid);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_dump_field(void* h, const char* field, int comp, int64_t iteration, const char* base_path,
                        int with_pgm) {
    try {
        return EG(h)->dump_field(field, comp, iteration, base_path, with_pgm);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_tile_rank(void* h, const int32_t* coords) { return EG(h)->rank_of(coords); }

int plbm_gpu_sync(void* h) {
    try {
        return EG(h)->sync();
    } catch (const std::exception&) {
        return -6;
    }
}

void plbm_gpu_counters(void* h, plbm_counters* out) {
    try {
        EG(h)->counters(out);
    } catch (const std::exception&) {
        std::memset(out, 0, sizeof *out);
    }
}

int plbm_gpu_tiles(void* h, int32_t* coords, int32_t* owners, int64_t* births, int max) {
    return EG(h)->tiles(coords, owners, births, max);
}

int plbm_gpu_read_tile(void* h, const int32_t* coords, int comp, int field, double* out) {
    try {
        return EG(h)->read_tile(coords, comp, field, out);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_creation_log(void* h, plbm_creation_event* out, int max) {
    return EG(h)->creation_log(out, max);
}

int plbm_gpu_poke_f(void* h, const int32_t* coords, int comp, int i, const int32_t* local, double v) {
    return EG(h)->poke_f(coords, comp, i, local, v);
}

int plbm_gpu_set_capture(void* h, int on) {
    try {
        return EG(h)->set_capture(on != 0);
    } catch (const std::exception&) {
        return -6;
    }
}

int plbm_gpu_set_profiling(void* h, int on) {
    EG(h)->set_profiling(on != 0);
    return 0;
}

void plbm_gpu_kernel_stats(void* h, plbm_kernel_stats* out) {
    try {
        *out = EG(h)->stats();
    } catch (const std::exception&) {
        std::memset(out, 0, sizeof *out);
    }
}

void plbm_gpu_reset_kernel_stats(void* h) {
    try {
        EG(h)->reset_stats();
    } catch (const std::exception&) {
    }
}

void* plbm_gpu_stream(void* h) { return EG(h)->stream(); }

void plbm_gpu_memory(void* h, uint64_t* out) { EG(h)->memory(out); }

int plbm_gpu_set_kernel_variant(void* h, int variant) { return EG(h)->set_variant(variant); }

void plbm_gpu_destroy(void* h) { delete EG(h); }

}  // extern "C"
