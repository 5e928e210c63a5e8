/*
 * plbm_scenario.h — plain-C description of one progressive-mesh MPMC
 * D3Q19 scenario, shared by every engine behind the step-loop boundary:
 *
 *   - the B200 engine            (include/plbm_gpu.h, libplbm_gpu.so)
 *   - the CPU oracle restatement (oracle/plbm_oracle.c, test infrastructure)
 *   - the reference shim         (oracle/ref_shim.cpp → oracle/_ref/, test
 *                                 infrastructure, built from /root/reference)
 *
 * Field-for-field this is the subset of the reference's
 * `plbm::iobench::ScenarioConfig` (proj/include/plbm/scenario.hpp:32-70)
 * that `make_state` + `Engine::step` consume (proj/src/engine.cpp:91-161,
 * 537-563).  TOML parsing, output paths and report intervals stay on the
 * reference side of the boundary; a reference driver fills this struct from
 * its already-validated ScenarioConfig.
 *
 * No torch types, no C++ types: plain pointers and sizes only.
 */
#ifndef PLBM_SCENARIO_H
#define PLBM_SCENARIO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLBM_Q 19          /* D3Q19 only on this path        */
#define PLBM_MAX_COMP 4    /* components per scenario                       */
#define PLBM_MAX_SEEDS 64  /* seed regions per scenario                     */

/* proj/include/plbm/physics.hpp:14-30 (EosParams + ComponentParams). */
typedef struct plbm_component_desc {
    double tau;          /* BGK relaxation time, > 0.5                      */
    double rho_ambient;  /* density of fresh tiles and frontier ghosts      */
    double g_self;       /* self coupling, nonzero                          */
    double beta;         /* psi / psi^2 force split, in [1, 1.5]            */
    double gravity[3];   /* body acceleration                               */
    double a, b, R, T, Tc, omega; /* Peng-Robinson EOS                      */
} plbm_component_desc;

/* proj/include/plbm/scenario.hpp:18-30 (SeedRegion). */
enum { PLBM_SEED_BOX = 0, PLBM_SEED_SPHERE = 1 };
typedef struct plbm_seed_desc {
    int32_t shape;       /* PLBM_SEED_BOX | PLBM_SEED_SPHERE                */
    int32_t component;
    double box_min[3];   /* box: [min, max) on cell centres                 */
    double box_max[3];
    double center[3];    /* sphere: |c - center|^2 <= radius^2              */
    double radius;
    double rho;
    double velocity[3];
} plbm_seed_desc;

enum { PLBM_MODE_STATIC = 0, PLBM_MODE_PROGRESSIVE = 1 };
enum { PLBM_POLICY_SIMPLE = 0, PLBM_POLICY_OPTIMIZED = 1 };

typedef struct plbm_scenario_desc {
    int32_t domain[3];         /* cells; each divisible by tile_extent      */
    int32_t tile_extent;       /* E (subdomain edge), >= 4                  */
    int32_t mode;              /* PLBM_MODE_*                               */
    double threshold;          /* S of the activation criterion             */
    int32_t devices;           /* owner count for placement                 */
    int32_t policy;            /* PLBM_POLICY_*                             */
    double weight_p2p;         /* gamma weights (topology.hpp:21-22)        */
    double weight_staged;
    const uint8_t* p2p;        /* devices x devices 0/1, NULL = all P2P     */
    int32_t periodic[3];       /* 1 = periodic axis, 0 = ambient            */
    int32_t n_components;      /* 1..PLBM_MAX_COMP                          */
    const plbm_component_desc* components;
    const double* coupling;    /* n x n symmetric, zero diagonal; NULL = 0  */
    int32_t n_seeds;
    const plbm_seed_desc* seeds;
    const uint8_t* geometry;   /* nx*ny*nz bytes x-fastest (1 = solid), or
                                  NULL for an all-fluid domain (LBMGEO v1
                                  payload, proj/include/plbm/geometry.hpp)  */
} plbm_scenario_desc;

/* Per-tile read-back fields (interior cells only, x-fastest, E^3 each;
 * PLBM_FIELD_F returns 19 direction-major planes).  The values are the
 * reference's view of the state between steps (proj/include/plbm/tile.hpp:38-82):
 * f = post-stream populations, rho/u = P5 moments (or seed / ambient values
 * before the first step), u_prev = the velocity used by the last collision,
 * psi = the P1 pseudo-potential of the last step.                          */
enum {
    PLBM_FIELD_F = 0,
    PLBM_FIELD_RHO = 1,
    PLBM_FIELD_UX = 2, PLBM_FIELD_UY = 3, PLBM_FIELD_UZ = 4,
    PLBM_FIELD_PUX = 5, PLBM_FIELD_PUY = 6, PLBM_FIELD_PUZ = 7,
    PLBM_FIELD_PSI = 8
};

/* One row of the creation log (proj/include/plbm/tilemap.hpp:27-32).
 * trigger: -1 = "init", else the face index 0..5 = -x,+x,-y,+y,-z,+z.   */
typedef struct plbm_creation_event {
    int64_t iteration;
    int32_t coords[3];
    int32_t trigger;
    int32_t owner;
    int32_t pad;
} plbm_creation_event;

/* Counters read between steps (proj/include/plbm/engine.hpp:34-38,84-88;
 * proj/include/plbm/topology.hpp:24).                                     */
typedef struct plbm_counters {
    int64_t iteration;
    uint64_t cell_updates;
    uint64_t negative_populations;
    uint64_t psi_clamps;
    uint64_t zero_rho_forcings;
    uint64_t suppressed_expansions;
    uint64_t bytes[3];          /* intra / P2P / staged modeled bytes      */
    uint64_t tiles;             /* active_report().tiles                   */
    uint64_t active_cells;      /* active_report().active_cells            */
    uint64_t bytes_resident;    /* active_report().bytes_resident          */
} plbm_counters;

/* Error record filled when a step aborts (EngineError,
 * proj/include/plbm/engine.hpp:64-74).  code 0 = ok.                      */
typedef struct plbm_error {
    int32_t code;               /* 0 ok, 1 engine error (NaN / EOS pole),
                                   2 invalid argument, 3 CUDA / resource   */
    int32_t tile[3];
    int64_t iteration;
    char phase[8];              /* "P1", "P5", ...                          */
    char message[240];
} plbm_error;

#ifdef __cplusplus
}
#endif
#endif /* PLBM_SCENARIO_H */
