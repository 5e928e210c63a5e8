// expand.cuh — the progressive mesh's expansion on the device (single rank).
//
// k_check_expand runs after every step's face pass in the speculative step
// queue.  It does what the host mirror's expand + create_tile + assign_owner
// + upload_map do (proj/src/tilemap.cpp:83-266, proj/src/engine.cpp:30-41,
// proj/src/assign.cpp:8-38), without a host round trip:
//   1. trigger resolution: every set (slot, face) bit -> target tile; out of
//      bounds -> suppressed expansion; existing target -> nothing; otherwise a
//      candidate keyed by (source tile, face) — atomicMin keeps the first in
//      the reference's sort order (target, source, face);
//   2. births in coordinate order (a scan of the tile grid in linear =
//      coordinate order): slots allocated in that order, solid mask sliced
//      from the device geometry (periodic wrap, ambient outside), fluid count;
//   3. assign_device for the newborns in coordinate order (owners of existing
//      face neighbours incl. earlier newborns, least-loaded eligible devices,
//      argmin gamma cost with strict <);
//   4. the derived tables for the new map: active list, ghost routes (hop
//      along the higher axis first), trigger masks, modeled step bytes, slot
//      pointers, and a birth record for the host mirror (replayed lazily).
// Steps also accumulate cell_updates and the modeled bytes here (with the
// pre-expansion map, as the reference counts them).  Anything the kernel
// cannot take (an error, more births than the launched grid has room for)
// sets the halt flag and leaves the triggers to the host path.
//
// Multi-rank (world > 1, one process per GPU): every rank runs this kernel
// on the SAME merged inputs — the trigger bytes of every rank (each slot's
// bits are set only by its owner rank, so OR over ranks is the merge) and
// the lowest error key of every rank, read from the peers' sync blocks over
// NVLink after a device-side rank barrier (k_rank_barrier) — so every rank's
// map, placement, halts and EngineError stay identical without a host round
// trip.  Newborn tile o lives on rank o % world (its pool index from that
// rank's counter); this rank's launch list (lactive) is rebuilt alongside the
// global one.
#pragma once

#include "kernels.cuh"

namespace plbm {

struct BirthRec {
    long long it;
    int x, y, z;
    int trigger;
    int owner;
    int slot;
    int local;
    int fluid;
    int has_solid;
    int pad;
};

struct ExpandDev {
    int* gslot;                   // [gx*gy*gz] tile grid -> slot or -1
    unsigned long long* cand;     // [gx*gy*gz] candidate keys (all ~0 between steps)
    int* active;                  // [cap] active slots in coordinate order
    int* nactive;                 // active count
    int* next_slot;               // slots are allocated 0, 1, 2, ... (never freed)
    int* next_local;              // [world] next pool index per rank
    int* owner;                   // [slot]
    int* coords;                  // [slot][3]
    uint8_t* mode;                // [slot]
    uint8_t* has_solid;           // [slot]
    uint8_t* no_fluid;            // [slot] (Dev::no_fluid)
    uint32_t* solid;              // [slot][solid_words]
    int* lidx;                    // [slot]
    int* route_psi;               // [slot][18]
    int* lactive;                 // [cap] this rank's active slots (== active when world == 1)
    int* nlactive;                // this rank's active count (== nactive when world == 1)
    int world, rank;
    const uint8_t* ptrig[8];      // per rank: this step's trigger bytes (world > 1)
    const unsigned long long* perr[8];  // per rank: error key word (world > 1)
    uint8_t* merged;              // [cap + 1] merged trigger bytes (world > 1; read by the host on a halt)
    unsigned long long* merr;     // merged error key (world > 1; read by the host on a halt)
    uint8_t* trig_clear;          // this rank's trigger bytes of the next step's parity (world > 1)
    const unsigned long long* psnap[8];  // per rank: diagnostic counters at this step's barrier
    unsigned long long* gcnt;     // job-wide diagnostics (sum over ranks; world > 1)
    double* peer_f[8];            // per rank: population pool base
    double* peer_pf[8];           // per rank: psi-face pool base
    int* route_w;                 // [slot][18] geometric neighbours (A-A stores)
    int nbuf;                     // population buffers (2 = A-B, 1 = A-A)
    uint8_t* bmask;               // [slot]
    uint8_t* omask;               // [slot]
    double** slot_f[2];           // pointer tables (local pool)
    double** slot_pf[2];
    double* pool_f;
    double* pool_pf;
    size_t per_slot, per_pf;
    int lcap;
    const uint8_t* geom;          // [nz][ny][nx] or nullptr
    const uint8_t* p2p;           // [devices][devices]
    unsigned long long* per_dev;  // [devices]
    unsigned long long* acc;      // [0] cell_updates, [1..3] bytes, [4] active_cells, [5..7] step bytes
    BirthRec* births;
    int* nbirths;
    int* post_flags;              // bit0: newborns in GEN mode, bit1: pull routes lag the psi routes
    double* capture;              // nullptr unless capture is on
    int cap, amb, devices, policy, max_active, solid_words;
    int periodic[3], dom[3];
    double w_p2p, w_staged;
    unsigned long long face_xfer;
};

template <int E>
__global__ void __launch_bounds__(1024) k_check_expand(Dev d, ExpandDev x, long iter, int* halt) {
    if (*(volatile int*)halt != 0) return;
    constexpr int G = E + 2;
    const int tid = threadIdx.x;
    constexpr int NT = 1024;
    const int gx = P.grid[0], gy = P.grid[1], gz = P.grid[2];
    const int ngrid = gx * gy * gz;
    __shared__ int s_err, s_nb, s_chunk, s_solid_any, s_any;
    __shared__ unsigned long long s_supp;
    __shared__ int s_wsum[32];
    auto wrap = [&](int* q) {  // periodic wrap; false if out of bounds
        for (int a = 0; a < 3; ++a)
            if (q[a] < 0 || q[a] >= P.grid[a]) {
                if (!x.periodic[a]) return false;
                q[a] = (q[a] + P.grid[a]) % P.grid[a];
            }
        return true;
    };
    auto lin = [&](const int* q) { return (q[0] * gy + q[1]) * gz + q[2]; };
    // block-wide exclusive prefix of `hit` over one chunk of NT items;
    // returns this thread's offset, s_chunk holds the chunk total
    auto block_scan = [&](int hit) {
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        const int lane = tid & 31, w = tid >> 5;
        if (lane == 0) s_wsum[w] = __popc(m);
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int k = 0; k < NT / 32; ++k) {
                const int c = s_wsum[k];
                s_wsum[k] = run;
                run += c;
            }
            s_chunk = run;
        }
        __syncthreads();
        return s_wsum[w] + __popc(m & ((1u << lane) - 1));
    };
    // this step's trigger bytes: own (one rank) or merged over every rank
    const uint8_t* trig = d.trig;
    if (x.world > 1) {
        for (int s = tid; s < x.cap + 1; s += NT) {
            uint8_t v = 0;
            for (int r = 0; r < x.world; ++r) v |= x.ptrig[r][s];
            x.merged[s] = v;
        }
        trig = x.merged;
    }
    if (tid == 0) {
        unsigned long long e = *(volatile const unsigned long long*)d.err;
        if (x.world > 1) {
            // a peer may already be a step ahead: only keys of this step or earlier
            const unsigned long long lim = ((unsigned long long)(iter + 1)) << 37;
            e = ERR_NONE_KEY;
            for (int r = 0; r < x.world; ++r) {
                const unsigned long long k = *(volatile const unsigned long long*)x.perr[r];
                if (k < lim && k < e) e = k;
            }
            *x.merr = e;
            // job-wide diagnostics: every rank's counters as of this step
            for (int k = 0; k < CNT_SUPP; ++k) {
                unsigned long long sum = 0;
                for (int r = 0; r < x.world; ++r) sum += *(volatile const unsigned long long*)(x.psnap[r] + k);
                x.gcnt[k] = sum;
            }
        }
        s_err = (e != ERR_NONE_KEY) ? 1 : 0;
        s_supp = 0;
        s_nb = 0;
        s_any = 0;
        *x.post_flags = 0;  // consumed by this step's k_post_main
    }
    __syncthreads();
    if (s_err) {  // the step failed: nothing is final, the host reports it
        if (tid == 0) *halt = 1;
        return;
    }
    if (tid == 0) {  // the step is final: cell updates and modeled bytes of its map
        x.acc[0] += x.acc[4];
        x.acc[1] += x.acc[5];
        x.acc[2] += x.acc[6];
        x.acc[3] += x.acc[7];
    }
    const int na = *x.nactive;
    // ---- 1. trigger resolution --------------------------------------------
    unsigned supp = 0;
    for (int k = tid; k < na * 6; k += NT) {
        const int s = x.active[k / 6], f = k % 6;
        if (!(trig[s] & (1u << f))) continue;
        int q[3] = {x.coords[3 * s], x.coords[3 * s + 1], x.coords[3 * s + 2]};
        q[f >> 1] += (f & 1) ? 1 : -1;
        if (!wrap(q)) {
            ++supp;
            continue;
        }
        const int t = lin(q);
        if (x.gslot[t] >= 0) continue;
        atomicMin(&x.cand[t], (unsigned long long)lin(&x.coords[3 * s]) * 8ull + (unsigned long long)f);
        s_any = 1;
    }
    supp = __reduce_add_sync(0xffffffffu, supp);
    if ((tid & 31) == 0 && supp) atomicAdd(&s_supp, (unsigned long long)supp);
    __syncthreads();
    // ---- 2. births in coordinate order (grid scan = coordinate order) -------
    int nb = 0;  // no candidate written (the usual step): cand is all ~0, nb = 0
    for (int base = 0; s_any && base < ngrid; base += NT) {
        const int t = base + tid;
        block_scan(t < ngrid && x.cand[t] != ~0ull);
        nb += s_chunk;
        __syncthreads();
    }
    if (nb > 0 && (na + nb > x.max_active || *x.next_slot + nb > x.cap)) {
        // more births than the launched grid has room for: the host takes
        // this expansion (triggers and suppressed count left untouched)
        for (int t = tid; t < ngrid; t += NT) x.cand[t] = ~0ull;
        if (tid == 0) *halt = 1;
        return;
    }
    if (tid == 0) d.cnt[CNT_SUPP] += s_supp;
    // consumed: one rank clears its (only) trigger array; several ranks clear
    // their array of the NEXT step's parity (every peer finished reading it
    // before the rank barrier this step's face pass waited on)
    uint8_t* clr = x.world > 1 ? x.trig_clear : d.trig;
    for (int s = tid; s < x.cap + 1; s += NT) clr[s] = 0;
    if (nb == 0) return;
    const int first_slot = *x.next_slot;
    const int b0 = *x.nbirths;
    for (int base = 0; base < ngrid; base += NT) {
        const int t = base + tid;
        const int hit = t < ngrid && x.cand[t] != ~0ull;
        const int pos = s_nb + block_scan(hit);
        if (hit) {
            const unsigned long long key = x.cand[t];
            x.cand[t] = ~0ull;
            const int slot = first_slot + pos;
            const int tx = t / (gy * gz), ty = (t / gz) % gy, tz = t % gz;
            x.gslot[t] = slot;
            x.coords[3 * slot] = tx;
            x.coords[3 * slot + 1] = ty;
            x.coords[3 * slot + 2] = tz;
            x.mode[slot] = MODE_GEN_AMBIENT;
            x.owner[slot] = -1;
            BirthRec& b = x.births[b0 + pos];
            b.it = iter;
            b.x = tx;
            b.y = ty;
            b.z = tz;
            b.trigger = int(key & 7ull);
            b.slot = slot;
        }
        __syncthreads();
        if (tid == 0) s_nb += s_chunk;
        __syncthreads();
    }
    // solid slicing + fluid count of every newborn (create_tile, tilemap.cpp:94-127)
    for (int k = 0; k < nb; ++k) {
        BirthRec& b = x.births[b0 + k];
        const int slot = b.slot;
        if (tid == 0) s_solid_any = 0;
        uint32_t* bits = x.solid + size_t(slot) * x.solid_words;
        for (int w = tid; w < x.solid_words; w += NT) bits[w] = 0u;
        __syncthreads();
        int fluid = 0, sol_any = 0;
        if (x.geom) {
            for (int c = tid; c < G * G * G; c += NT) {
                const int lx = c % G - 1, ly = (c / G) % G - 1, lz = c / (G * G) - 1;
                int g[3] = {b.x * E + lx, b.y * E + ly, b.z * E + lz};
                bool outside = false;
                for (int a = 0; a < 3; ++a)
                    if (g[a] < 0 || g[a] >= x.dom[a]) {
                        if (x.periodic[a]) g[a] = (g[a] + x.dom[a]) % x.dom[a];
                        else outside = true;
                    }
                const bool sol = !outside &&
                                 x.geom[size_t(g[0]) + size_t(x.dom[0]) * (size_t(g[1]) + size_t(x.dom[1]) * g[2])];
                const bool interior = lx >= 0 && lx < E && ly >= 0 && ly < E && lz >= 0 && lz < E;
                if (sol) {
                    atomicOr(&bits[c >> 5], 1u << (c & 31));
                    sol_any = 1;
                } else if (interior) {
                    ++fluid;
                }
            }
        } else if (tid == 0) {
            fluid = E * E * E;
        }
        fluid = __reduce_add_sync(0xffffffffu, fluid);
        sol_any = __any_sync(0xffffffffu, sol_any);
        if ((tid & 31) == 0) {
            s_wsum[tid >> 5] = fluid;
            if (sol_any) s_solid_any = 1;
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < NT / 32; ++w) tot += s_wsum[w];
            b.fluid = tot;
            b.has_solid = s_solid_any;
            x.has_solid[slot] = uint8_t(s_solid_any);
            x.no_fluid[slot] = uint8_t(tot == 0);
        }
        __syncthreads();
    }
    // ---- 3. assign_device in coordinate order (assign.cpp:17-38) ---------------
    if (tid == 0) {
        unsigned long long add_cells = 0;
        for (int k = 0; k < nb; ++k) {
            BirthRec& b = x.births[b0 + k];
            const int c[3] = {b.x, b.y, b.z};
            int owners[6], no = 0;
            for (int f = 0; f < 6; ++f) {
                int q[3] = {c[0], c[1], c[2]};
                q[f >> 1] += (f & 1) ? 1 : -1;
                if (!wrap(q)) continue;
                const int ns = x.gslot[lin(q)];
                if (ns >= 0 && ns != b.slot && x.owner[ns] >= 0) owners[no++] = x.owner[ns];
            }
            unsigned long long lo = x.per_dev[0];
            for (int dv = 1; dv < x.devices; ++dv) lo = x.per_dev[dv] < lo ? x.per_dev[dv] : lo;
            int chosen = -1;
            double best = 0.0;
            for (int dv = 0; dv < x.devices; ++dv) {
                if (x.per_dev[dv] != lo) continue;
                if (chosen < 0) {
                    chosen = dv;
                    if (x.policy != 1) break;  // simple: the first eligible
                    best = 0.0;
                    for (int o = 0; o < no; ++o) {
                        const int cls = dv == owners[o] ? 0 : (x.p2p[dv * x.devices + owners[o]] ? 1 : 2);
                        best += cls == 0 ? 0.0 : (cls == 1 ? x.w_p2p * double(x.face_xfer) : x.w_staged * double(x.face_xfer));
                    }
                    continue;
                }
                double cost = 0.0;
                for (int o = 0; o < no; ++o) {
                    const int cls = dv == owners[o] ? 0 : (x.p2p[dv * x.devices + owners[o]] ? 1 : 2);
                    cost += cls == 0 ? 0.0 : (cls == 1 ? x.w_p2p * double(x.face_xfer) : x.w_staged * double(x.face_xfer));
                }
                if (cost < best) {
                    best = cost;
                    chosen = dv;
                }
            }
            ++x.per_dev[chosen];
            x.owner[b.slot] = chosen;
            b.owner = chosen;
            // GPU rank owner % world and its next pool index (engine.cu
            // assign_owner; the fairness spread <= 1 bounds every rank's count
            // by the pool it allocated, lcap)
            const int rk = chosen % x.world;
            const int local = x.next_local[rk]++;
            x.lidx[b.slot] = rk == x.rank ? local : -1;
            b.local = local;
            for (int bb = 0; bb < 2; ++bb) {
                x.slot_f[bb][b.slot] = x.peer_f[rk] + (size_t(bb % x.nbuf) * (x.lcap + 1) + local) * x.per_slot;
                x.slot_pf[bb][b.slot] = x.peer_pf[rk] + (size_t(bb) * (x.lcap + 1) + local) * x.per_pf;
            }
            add_cells += (unsigned long long)b.fluid;
        }
        *x.next_slot += nb;
        *x.nbirths += nb;
        x.acc[4] += add_cells;
        *x.post_flags = 3;
    }
    __syncthreads();
    // capture buffer of the newborns starts at zero (engine.cu upload_map)
    if (x.capture)
        for (int k = 0; k < nb; ++k) {
            const int slot = first_slot + k;
            if (x.lidx[slot] < 0) continue;  // another rank's tile
            double* cp = x.capture + size_t(x.lidx[slot]) * P.C * 4 * (E * E * E);
            for (int c = tid; c < P.C * 4 * E * E * E; c += NT) cp[c] = 0.0;
        }
    // ---- 4. tables of the new map ----------------------------------------------
    // active list in coordinate order
    if (tid == 0) s_nb = 0;
    __syncthreads();
    for (int base = 0; base < ngrid; base += NT) {
        const int t = base + tid;
        const int sl = t < ngrid ? x.gslot[t] : -1;
        const int pos = s_nb + block_scan(sl >= 0);
        if (sl >= 0) x.active[pos] = sl;
        __syncthreads();
        if (tid == 0) s_nb += s_chunk;
        __syncthreads();
    }
    const int nact = s_nb;
    if (tid == 0) *x.nactive = nact;
    if (x.world > 1) {  // this rank's launch list, coordinate order
        __syncthreads();
        if (tid == 0) s_nb = 0;
        __syncthreads();
        for (int base = 0; base < ngrid; base += NT) {
            const int t = base + tid;
            const int sl = t < ngrid ? x.gslot[t] : -1;
            const bool mine = sl >= 0 && x.owner[sl] % x.world == x.rank;
            const int pos = s_nb + block_scan(mine);
            if (mine) x.lactive[pos] = sl;
            __syncthreads();
            if (tid == 0) s_nb += s_chunk;
            __syncthreads();
        }
        if (tid == 0) *x.nlactive = s_nb;
    }
    // routes (engine.cu compute_routes: faces, then edges hopping along the
    // higher axis first; an absent hop gives the ambient slot), trigger masks
    for (int k = tid; k < nact; k += NT) {
        const int s = x.active[k];
        const int* c = &x.coords[3 * s];
        int* out = x.route_psi + size_t(s) * 18;
        uint8_t bm = 0, om = 0;
        for (int f = 0; f < 6; ++f) {
            int q[3] = {c[0], c[1], c[2]};
            q[f >> 1] += (f & 1) ? 1 : -1;
            if (!wrap(q)) {
                out[f] = x.amb;
                om |= uint8_t(1u << f);
                continue;
            }
            const int ns = x.gslot[lin(q)];
            out[f] = ns >= 0 ? ns : x.amb;
            if (ns < 0) bm |= uint8_t(1u << f);
        }
        x.bmask[s] = bm;
        x.omask[s] = om;
        const int pairs[3][2] = {{0, 1}, {0, 2}, {1, 2}};
        for (int p = 0; p < 3; ++p)
            for (int da = -1; da <= 1; da += 2)
                for (int db = -1; db <= 1; db += 2) {
                    const int a = pairs[p][0], b = pairs[p][1];
                    int r = x.amb;
                    int q1[3] = {c[0], c[1], c[2]};
                    q1[b] += db;
                    if (wrap(q1) && x.gslot[lin(q1)] >= 0) {
                        int q2[3] = {q1[0], q1[1], q1[2]};
                        q2[a] += da;
                        if (wrap(q2) && x.gslot[lin(q2)] >= 0) r = x.gslot[lin(q2)];
                    }
                    out[edge_class(a, b, da, db)] = r;
                }
        // geometric neighbours of the new map (A-A store targets)
        int* ow = x.route_w + size_t(s) * 18;
        for (int f = 0; f < 6; ++f) ow[f] = out[f];
        for (int p = 0; p < 3; ++p)
            for (int da = -1; da <= 1; da += 2)
                for (int db = -1; db <= 1; db += 2) {
                    const int a = pairs[p][0], b = pairs[p][1];
                    int q[3] = {c[0], c[1], c[2]};
                    q[a] += da;
                    q[b] += db;
                    const int ns = wrap(q) ? x.gslot[lin(q)] : -1;
                    ow[edge_class(a, b, da, db)] = ns >= 0 ? ns : x.amb;
                }
    }
    // modeled step bytes (engine.cu recompute_step_bytes)
    unsigned long long sb[3] = {0, 0, 0};
    for (int k = tid; k < nact * 6; k += NT) {
        const int s = x.active[k / 6], f = k % 6;
        int q[3] = {x.coords[3 * s], x.coords[3 * s + 1], x.coords[3 * s + 2]};
        q[f >> 1] += (f & 1) ? 1 : -1;
        if (!wrap(q)) continue;
        const int ns = x.gslot[lin(q)];
        if (ns < 0) continue;
        const int a = x.owner[s], bo = x.owner[ns];
        const int cls = a == bo ? 0 : (x.p2p[a * x.devices + bo] ? 1 : 2);
        sb[cls] += 2ull * x.face_xfer;
    }
    for (int c = 0; c < 3; ++c) {
        unsigned long long v = sb[c];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        sb[c] = v;
    }
    __shared__ unsigned long long s_sb[3];
    if (tid < 3) s_sb[tid] = 0;
    __syncthreads();
    if ((tid & 31) == 0)
        for (int c = 0; c < 3; ++c) atomicAdd(&s_sb[c], sb[c]);
    __syncthreads();
    if (tid == 0)
        for (int c = 0; c < 3; ++c) x.acc[5 + c] = s_sb[c];
}

// Device-side barrier of the ranks of one run (one process per GPU, pools
// and sync blocks mapped over NVLink): every rank stores `epoch` into slot
// `rank` of every peer's flag words (system-scope release after the fence:
// the kernels queued before this one on the stream have completed, so their
// stores are ordered before the flag), then waits until every peer's epoch
// reached its own flag words.  Launched with identical epochs on every rank
// (the host counts barriers; every rank queues the same sequence).  A peer
// that never arrives (it died) turns into an error after `timeout_ns`
// instead of a hang.
struct PeerFlags {
    unsigned long long* p[8];
};
static __global__ void k_rank_barrier(unsigned long long* flags, PeerFlags peers, int world, int rank,
                               unsigned long long epoch, unsigned long long* err, long iter,
                               unsigned long long timeout_ns, const unsigned long long* cnt,
                               unsigned long long* snap) {
    const int t = threadIdx.x;
    // (the step's second barrier) this rank's diagnostic counters into the
    // step-parity slot peers sum after the barrier
    if (snap && t < CNT_N) snap[t] = cnt[t];
    __syncwarp();
    if (t < world && t != rank) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(peers.p[t] + rank), "l"(epoch) : "memory");
        const unsigned long long t0 = global_ns();
        unsigned long long v = 0;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(flags + t) : "memory");
            if (v >= epoch) break;
            if (global_ns() - t0 > timeout_ns) {
                atomicMin(err, ((unsigned long long)iter << 37) | ERR_PEER_TIMEOUT);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
}

// After each step's main kernel: the modes of the tiles born at the end of
// the previous step go back to PULL, and the pull routes catch up with the
// psi routes (engine.cu step_main's memset / copy, here device-driven).
static __global__ void k_post_main(uint8_t* mode, int* route_pull, const int* route_psi, int nslot,
                            int* post_flags, const int* halt) {
    if (*(volatile const int*)halt != 0) return;
    const int f = *(volatile int*)post_flags;
    if (!f) return;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nslot * 18; k += gridDim.x * blockDim.x) {
        if (k < nslot && (f & 1)) mode[k] = MODE_PULL;
        if (f & 2) route_pull[k] = route_psi[k];
    }
}

// Solid slicing of the initial tiles (create_tile, tilemap.cpp:94-127: the
// tile's (E+2)^3 box incl. the ghost ring from the domain geometry, periodic
// wrap, ambient fluid outside a non-periodic domain) on the device: one CTA
// per tile, the mask built in shared memory, fluid count and has_solid out.
template <int E>
__global__ void __launch_bounds__(256) k_slice(const int* __restrict__ slots, const int* __restrict__ coords,
                                               int n, const uint8_t* __restrict__ geom, int dx, int dy,
                                               int dz, int px, int py, int pz, uint32_t* solid,
                                               int solid_words, uint8_t* has_solid, int* fluid_out) {
    constexpr int G = E + 2;
    constexpr int W = (G * G * G + 31) / 32;
    __shared__ uint32_t bits[W];
    __shared__ int s_fluid, s_any;
    const int k = blockIdx.x;
    if (k >= n) return;
    const int slot = slots[k];
    const int t[3] = {coords[3 * k], coords[3 * k + 1], coords[3 * k + 2]};
    const int dom[3] = {dx, dy, dz}, per[3] = {px, py, pz};
    for (int w = threadIdx.x; w < W; w += blockDim.x) bits[w] = 0u;
    if (threadIdx.x == 0) s_fluid = s_any = 0;
    __syncthreads();
    int fluid = 0, any = 0;
    for (int c = threadIdx.x; c < G * G * G; c += blockDim.x) {
        const int l[3] = {c % G - 1, (c / G) % G - 1, c / (G * G) - 1};
        int g[3];
        bool outside = false;
        for (int a = 0; a < 3; ++a) {
            g[a] = t[a] * E + l[a];
            if (g[a] < 0 || g[a] >= dom[a]) {
                if (per[a]) g[a] = (g[a] + dom[a]) % dom[a];
                else outside = true;
            }
        }
        const bool sol = !outside && geom[size_t(g[0]) + size_t(dom[0]) * (size_t(g[1]) + size_t(dom[1]) * g[2])];
        if (sol) {
            atomicOr(&bits[c >> 5], 1u << (c & 31));
            any = 1;
        } else if (l[0] >= 0 && l[0] < E && l[1] >= 0 && l[1] < E && l[2] >= 0 && l[2] < E) {
            ++fluid;
        }
    }
    fluid = __reduce_add_sync(0xffffffffu, fluid);
    any = __any_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_fluid, fluid);
        if (any) s_any = 1;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < solid_words; w += blockDim.x) solid[size_t(slot) * solid_words + w] = bits[w];
    if (threadIdx.x == 0) {
        has_solid[k] = uint8_t(s_any);
        fluid_out[k] = s_fluid;
    }
}

}  // namespace plbm
