/*
 * plbm_gpu.h — C-ABI of the B200 progressive-mesh MPMC D3Q19 step loop.
 *
 * This is the drop-in boundary for the reference's step loop.  The reference
 * has no plugin or FFI seam: its step path is the in-process C++ class
 *
 *     plbm::engine::Engine(SimulationState&, int n_workers)   engine.hpp:98-116
 *     void Engine::step()                                      engine.cpp:537-563
 *
 * plus the state callers read between steps (SimulationState fields,
 * engine.hpp:76-91; TileMap::creation_log / active_report, tilemap.hpp:39-117;
 * DeviceTopology::byte_totals, topology.hpp:48-52).  Each entry point below
 * names the reference interface it replaces.  Exceptions never cross the ABI:
 * every call returns a status and fills a plbm_error record.
 *
 * Threading: one host thread per handle.  The handle owns all device memory
 * and one CUDA stream on the device it was created on.
 */
#ifndef PLBM_GPU_H
#define PLBM_GPU_H

#include "plbm_scenario.h"

#ifdef __cplusplus
extern "C" {
#endif

/* make_state(cfg) + Engine(state, workers)   (engine.cpp:91-161, 530-533).
 * Builds the initial tile set, owners, seeds and ambient state ON THE DEVICE
 * (no host field buffers).  `device` is the CUDA ordinal.  NULL on failure. */
void* plbm_gpu_create(const plbm_scenario_desc* desc, int device, plbm_error* err);

/* Creation options (zero-initialise; unknown fields must stay 0).
 *   storage: PLBM_STORAGE_AB — two population buffers, pull from one, store
 *            the next state into the other (the reference's f[2] double
 *            buffer + swap, tile.hpp:39, engine.cpp:482-490);
 *            PLBM_STORAGE_AA — one buffer updated in place with the A-A
 *            pattern (kernels.cuh AA_*): half the population
 *            footprint, bit-identical results; tile_extent <= 32.  After an
 *            EngineError the fields of an A-A engine are not rolled back.   */
enum { PLBM_STORAGE_AB = 0, PLBM_STORAGE_AA = 1 };
typedef struct plbm_gpu_options {
    int32_t storage;
    int32_t reserved[7];
} plbm_gpu_options;
/* plbm_gpu_create / plbm_gpu_create_dist with options (opt may be NULL).    */
void* plbm_gpu_create_ex(const plbm_scenario_desc* desc, int device, int rank, int world,
                         const plbm_gpu_options* opt, plbm_error* err);

/* Engine::step() n times (engine.cpp:537-563).  Returns 0, or err->code on an
 * EngineError (NaN / EOS pole: iteration and cell_updates do not advance).  */
int plbm_gpu_step(void* h, int n, plbm_error* err);

/* SimulationState counters: iteration, cell_updates, Diagnostics,
 * suppressed_expansions, byte_totals, active_report (engine.hpp:34-38,84-88). */
void plbm_gpu_counters(void* h, plbm_counters* out);

/* TileMap::tiles() in coordinate order: coords[3n], owner_device[n],
 * birth_iteration[n].  Returns the tile count (call with max = 0 to size). */
int plbm_gpu_tiles(void* h, int32_t* coords, int32_t* owners, int64_t* births, int max);

/* Reads one field of one tile as the reference holds it between steps
 * (Tile / ComponentState, tile.hpp:38-82): interior cells, x-fastest.
 * PLBM_FIELD_PSI / PUX..PUZ need plbm_gpu_set_capture(h, 1) before the step.
 * 0 ok, -1 no such tile, -2 bad component, -3 bad field, -4 not captured,
 * -7 tile owned by another rank.                                             */
int plbm_gpu_read_tile(void* h, const int32_t* coords, int comp, int field, double* out);

/* TileMap::creation_log() (tilemap.hpp:94-96).  Returns the row count.      */
int plbm_gpu_creation_log(void* h, plbm_creation_event* out, int max);

/* Test hook: overwrite one post-stream population before the first step
 * (NaN poisoning, proj/tests/test_engine.cpp:284-310).                       */
int plbm_gpu_poke_f(void* h, const int32_t* coords, int comp, int i, const int32_t* local,
                    double value);

/* Keep psi and u_prev per cell (extra 32 B/cell/comp per step) so that
 * read_tile can serve PLBM_FIELD_PSI / PLBM_FIELD_PU*.                      */
int plbm_gpu_set_capture(void* h, int on);

/* Kernel timing for the roofline: when on, every launch of the fused kernel
 * and of the face pre-pass is bracketed by CUDA events recorded on the
 * engine's stream (no host synchronisation; resolved by kernel_stats).      */
int plbm_gpu_set_profiling(void* h, int on);
typedef struct plbm_kernel_stats {
    int64_t main_launches;
    double main_ms;            /* summed CUDA-event time of k_main          */
    int64_t face_launches;
    double face_ms;            /* summed CUDA-event time of k_face          */
    int64_t kernels_launched;  /* all kernels launched by the engine        */
    uint64_t main_cell_updates;/* cell updates covered by the timed k_main  */
    uint64_t h2d_bytes;        /* host->device bytes the engine copied      */
    uint64_t d2h_bytes;        /* device->host bytes the engine copied      */
} plbm_kernel_stats;
void plbm_gpu_kernel_stats(void* h, plbm_kernel_stats* out);
void plbm_gpu_reset_kernel_stats(void* h);

/* Fused-kernel variant (A/B measurement; all are bit-identical):
 *   0  = default: k_main_pc where it applies (E in {16,32}, a psi stencil;
 *        C = 3 at E = 32 uses a 12-CTA non-portable cluster), else the plain
 *        kernel
 *   1  = plain kernel that pulls every population twice (always used for
 *        E = 8, C = 3 and psi-free scenarios)
 *   21 = k_main_pc with the collision head (TMEM load, u) after the cluster
 *        wait (the default runs it before the wait)
 *   22 = k_main_pc with psi computed two planes ahead (three TMEM slots)
 *   20 / 26 / 27 = k_main_pc with 1 / 2 / E/8 clusters per tile (E >= 32: a
 *        cluster covers all / half / one of the tile's 8-row y-blocks; the
 *        psi rows across a cluster boundary come from the face pass's
 *        mid-face buffers).  Variant 0 uses the measured default split
 *        (PLBM_SPLIT overrides it).  A-A storage accepts 0, 20, 26, 27.
 * Modifiers (added to the variant): +100 = run the face pass in the k_main_pc
 * tail ("last arriver" dependency counting, single rank) instead of a k_face
 * launch; +200 = face pass reads the x faces from the SoA block instead of the
 * xcol side buffers.  Returns 0, or -1 for an unknown variant (the current
 * one is kept).  The memory-only roofline probe (24, NOT a valid step) exists
 * only in builds compiled with -DPLBM_PROBES.                                 */
int plbm_gpu_set_kernel_variant(void* h, int variant);

/* The engine's CUDA stream (cudaStream_t) for callers that time with events. */
void* plbm_gpu_stream(void* h);

/* Population pool footprint: out[0] = bytes of the pool's address range
 * (nbuf x (tile capacity + 1) x slot), out[1] = bytes physically backed,
 * out[2] = mapping granule (0: allocated up front), out[3] = microseconds the
 * engine's mapper thread spent mapping, out[4] = microseconds the stepping
 * thread waited for it (out has 5 elements).
 * One-rank engines reserve the range and map device memory in granules (about
 * 1/64 of the pool, at most 2 GiB) only for the tiles the launches can reach (tiles + expansion headroom), so
 * a progressive mesh occupies HBM in proportion to its active tiles
 * (PLBM_POOL_GRANULE_MB overrides the granule; PLBM_LAZY_POOL=0: allocate the whole pool up front, as multi-rank engines
 * do for their IPC-exported pools). */
void plbm_gpu_memory(void* h, uint64_t* out);

/* ---- multi-GPU (one process per GPU) -----------------------
 * Every rank builds the same deterministic host mirror from the same
 * descriptor; tile owner o (assign_device) lives on rank o % world.  Each
 * rank's block pool, psi-face pool and sync block (barrier flags, error key,
 * trigger bytes) are exported as CUDA IPC handles; peers map them and the
 * fused kernel reads remote neighbour tiles over NVLink in place.
 *
 *   h = plbm_gpu_create_dist(desc, local_device, rank, world, &err)
 *   plbm_gpu_ipc_handles(h, buf)           -> exchange (all_gather) ->
 *   plbm_gpu_open_peer(h, r, handles_r)    for every other rank r
 *   plbm_gpu_prepare(h)                    then a barrier across ranks
 *   plbm_gpu_step(h, n, &err)              on every rank with the same n
 *
 * plbm_gpu_step on several ranks needs no host collective: per step the
 * fused kernel, a device-side rank barrier (flag words in the peers' sync
 * blocks, NVLink stores), the face pass, a second barrier, then the
 * expansion kernel on EVERY rank over the merged trigger bytes and the
 * lowest error key of all ranks (read from the peers' sync blocks) — so the
 * map, placement and any EngineError are identical on every rank, and steps
 * are queued ahead without a host round trip (Engine::step_speculative).
 * After an EngineError a multi-rank engine stays failed (every later step
 * reports the same error): create the engines again to start over.
 *
 * The host-merge protocol of round 1 remains for callers that merge the
 * triggers themselves: step_main, a barrier across ranks, step_face, an
 * all-reduce(MAX) of the plbm_gpu_trigger_bytes(h) bytes at
 * plbm_gpu_triggers_device(h), then step_end(h, merged).                     */
void* plbm_gpu_create_dist(const plbm_scenario_desc* desc, int device, int rank, int world,
                           plbm_error* err);
int plbm_gpu_prepare(void* h);
int plbm_gpu_step_begin(void* h, plbm_error* err);
int plbm_gpu_step_main(void* h, plbm_error* err);
int plbm_gpu_step_face(void* h);
int plbm_gpu_step_end(void* h, const uint8_t* merged_triggers, plbm_error* err);
int plbm_gpu_trigger_bytes(void* h);
void* plbm_gpu_triggers_device(void* h);
int plbm_gpu_local_triggers(void* h, uint8_t* out, int n);   /* D2H copy, syncs */
int plbm_gpu_ipc_handles(void* h, void* out);                /* 3 x cudaIpcMemHandle_t */
int plbm_gpu_open_peer(void* h, int rank, const void* handles);
/* Same-process peers (several ranks' engines in one process on one GPU):
 * attach another engine's pools directly.                                    */
int plbm_gpu_set_peer_pools(void* h, int rank, void* pool_f, void* pool_pf);
void plbm_gpu_pool_pointers(void* h, void** pool_f, void** pool_pf);
void* plbm_gpu_sync_block(void* h);                          /* same-process peers */
int plbm_gpu_set_peer_sync(void* h, int rank, void* sync_block);
int plbm_gpu_tile_rank(void* h, const int32_t* coords);      /* -1 if absent */
int plbm_gpu_sync(void* h);
/* Real byte accounting: bytes this rank's kernels read from
 * peer pools per step on the current map (NVLink traffic), next to the
 * reference's modeled record_exchange classes (plbm_counters.bytes).
 * out[0] = bytes, out[1] = remote face routes, out[2] = remote edge routes. */
void plbm_gpu_exchange_bytes(void* h, uint64_t* out);
/* Measurement hook (env PLBM_PROBE at create): per-CTA {SM id, start ns, end
 * ns} of the last fused-kernel launch, 3 words per CTA; returns the CTAs.    */
int plbm_gpu_probe(void* h, uint64_t* out, int max);

/* ---- output path -----------------------------------------
 * iobench::gather_field (dump.cpp:21-57): one field ("rho", "u_magnitude",
 * "psi") of one component over the whole domain, x fastest, absent cells at
 * the ambient fill, values as the reference holds them between steps ("psi"
 * needs plbm_gpu_set_capture(h, 1) before the step).  grid holds
 * domain[0]*domain[1]*domain[2] doubles.  0 ok, -2 bad component, -3 bad
 * field, -4 not captured, -7 multi-rank handle.                              */
int plbm_gpu_gather_field(void* h, const char* field, int comp, double* grid);
/* iobench::dump_field (dump.cpp:59-125): <base>.raw / .meta / .pgm, byte for
 * byte the reference's files.  -5 on a file error.                           */
int plbm_gpu_dump_field(void* h, const char* field, int comp, int64_t iteration, const char* base_path,
                        int with_pgm);

/* Engine::~Engine + SimulationState release.                                 */
void plbm_gpu_destroy(void* h);

#ifdef __cplusplus
}
#endif
#endif /* PLBM_GPU_H */
