"""Scenario description shared by every engine behind the step-loop boundary.

Python mirror of ``include/plbm_scenario.h`` (ctypes structs) plus the
builders for the benchmark configurations of BASELINE.json / SURVEY §8(d).
Field names and defaults follow the reference's ``ScenarioConfig`` and
``ComponentParams`` (proj/include/plbm/scenario.hpp:32-59,
proj/include/plbm/physics.hpp:14-30).
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

Q = 19
MAX_COMP = 4
MAX_SEEDS = 64

MODE_STATIC, MODE_PROGRESSIVE = 0, 1
POLICY_SIMPLE, POLICY_OPTIMIZED = 0, 1
SEED_BOX, SEED_SPHERE = 0, 1

FIELD_F, FIELD_RHO, FIELD_UX, FIELD_UY, FIELD_UZ = 0, 1, 2, 3, 4
FIELD_PUX, FIELD_PUY, FIELD_PUZ, FIELD_PSI = 5, 6, 7, 8
FACE_NAMES = ("-x", "+x", "-y", "+y", "-z", "+z")

CS2 = 1.0 / 3.0  # proj/include/plbm/stencil.hpp:20


class ComponentDesc(C.Structure):
    _fields_ = [("tau", C.c_double), ("rho_ambient", C.c_double),
                ("g_self", C.c_double), ("beta", C.c_double),
                ("gravity", C.c_double * 3),
                ("a", C.c_double), ("b", C.c_double), ("R", C.c_double),
                ("T", C.c_double), ("Tc", C.c_double), ("omega", C.c_double)]


class SeedDesc(C.Structure):
    _fields_ = [("shape", C.c_int32), ("component", C.c_int32),
                ("box_min", C.c_double * 3), ("box_max", C.c_double * 3),
                ("center", C.c_double * 3), ("radius", C.c_double),
                ("rho", C.c_double), ("velocity", C.c_double * 3)]


class ScenarioDesc(C.Structure):
    _fields_ = [("domain", C.c_int32 * 3), ("tile_extent", C.c_int32),
                ("mode", C.c_int32), ("threshold", C.c_double),
                ("devices", C.c_int32), ("policy", C.c_int32),
                ("weight_p2p", C.c_double), ("weight_staged", C.c_double),
                ("p2p", C.POINTER(C.c_uint8)),
                ("periodic", C.c_int32 * 3),
                ("n_components", C.c_int32),
                ("components", C.POINTER(ComponentDesc)),
                ("coupling", C.POINTER(C.c_double)),
                ("n_seeds", C.c_int32),
                ("seeds", C.POINTER(SeedDesc)),
                ("geometry", C.POINTER(C.c_uint8))]


class CreationEvent(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("coords", C.c_int32 * 3),
                ("trigger", C.c_int32), ("owner", C.c_int32), ("pad", C.c_int32)]


class Counters(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("cell_updates", C.c_uint64),
                ("negative_populations", C.c_uint64), ("psi_clamps", C.c_uint64),
                ("zero_rho_forcings", C.c_uint64),
                ("suppressed_expansions", C.c_uint64),
                ("bytes", C.c_uint64 * 3), ("tiles", C.c_uint64),
                ("active_cells", C.c_uint64), ("bytes_resident", C.c_uint64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "bytes"}
        d["bytes"] = tuple(self.bytes)
        return d


class Error(C.Structure):
    _fields_ = [("code", C.c_int32), ("tile", C.c_int32 * 3),
                ("iteration", C.c_int64), ("phase", C.c_char * 8),
                ("message", C.c_char * 240)]


class EngineError(RuntimeError):
    """Mirror of plbm::engine::EngineError (proj/include/plbm/engine.hpp:64-74)."""

    def __init__(self, err: Error):
        self.code = err.code
        self.iteration = err.iteration
        self.tile = tuple(err.tile)
        self.phase = err.phase.decode()
        super().__init__(err.message.decode())


@dataclass
class Component:
    """proj/include/plbm/physics.hpp:14-30 (defaults included)."""
    tau: float = 1.0
    rho_ambient: float = 1.0
    g_self: float = -1.0
    beta: float = 1.16
    gravity: Sequence[float] = (0.0, 0.0, 0.0)
    a: float = 0.0
    b: float = 0.0
    R: float = 1.0
    T: float = CS2
    Tc: float = 0.0
    omega: float = 0.0


@dataclass
class Seed:
    """proj/include/plbm/scenario.hpp:18-30."""
    shape: int = SEED_BOX
    component: int = 0
    box_min: Sequence[float] = (0.0, 0.0, 0.0)
    box_max: Sequence[float] = (0.0, 0.0, 0.0)
    center: Sequence[float] = (0.0, 0.0, 0.0)
    radius: float = 0.0
    rho: float = 1.0
    velocity: Sequence[float] = (0.0, 0.0, 0.0)


@dataclass
class Scenario:
    domain: Sequence[int] = (64, 64, 64)
    tile_extent: int = 16
    mode: int = MODE_PROGRESSIVE
    threshold: float = 0.0
    devices: int = 1
    policy: int = POLICY_OPTIMIZED
    weight_p2p: float = 0.5
    weight_staged: float = 1.0
    p2p: Optional[np.ndarray] = None
    periodic: Sequence[int] = (0, 0, 0)
    components: List[Component] = field(default_factory=lambda: [Component()])
    coupling: Optional[np.ndarray] = None
    seeds: List[Seed] = field(default_factory=list)
    geometry: Optional[np.ndarray] = None  # uint8 [nz, ny, nx] (x-fastest)
    name: str = "scenario"

    @property
    def n_components(self) -> int:
        return len(self.components)

    @property
    def tile_grid(self):
        return tuple(d // self.tile_extent for d in self.domain)

    def to_c(self) -> "CScenario":
        return CScenario(self)

    def to_toml(self, path: str, iterations: int = 10, report_interval: int = 10,
                snapshot_interval: int = 0, snapshot_fields=("rho",), snapshot_pgm: bool = False,
                output: str = "out", workers: int = 0) -> None:
        """The reference's scenario file (proj/src/scenario.cpp:185-290, read by
        iobench::load_config); a geometry is written next to it as LBMGEO v1."""
        def num(v):
            return repr(float(v))

        def arr(vs, f=num):
            return "[" + ", ".join(f(v) for v in vs) + "]"
        lines = [f'name = "{self.name}"', 'stencil = "D3Q19"',
                 f"domain = {arr(self.domain, str)}", f"tile_extent = {self.tile_extent}",
                 f'mode = "{"static" if self.mode == MODE_STATIC else "progressive"}"',
                 f"iterations = {iterations}", f"report_interval = {report_interval}",
                 f"snapshot_interval = {snapshot_interval}", f"threshold = {num(self.threshold)}",
                 f"devices = {self.devices}",
                 f'policy = "{"simple" if self.policy == POLICY_SIMPLE else "optimized"}"',
                 f"weight_p2p = {num(self.weight_p2p)}", f"weight_staged = {num(self.weight_staged)}",
                 f'output = "{output}"',
                 "snapshot_fields = [" + ", ".join(f'"{f}"' for f in snapshot_fields) + "]",
                 f"snapshot_pgm = {'true' if snapshot_pgm else 'false'}", f"workers = {workers}",
                 "boundary = [" + ", ".join('"periodic"' if p else '"ambient"' for p in self.periodic) + "]"]
        if self.p2p is not None:
            raise ValueError("to_toml: a custom P2P topology is not written")
        if self.geometry is not None:
            geo = os.path.splitext(path)[0] + ".lbmgeo"
            save_lbmgeo(self.geometry, geo)
            lines.append(f'geometry = "{os.path.basename(geo)}"')
        for c in self.components:
            lines += ["", "[[component]]", f"tau = {num(c.tau)}", f"rho_ambient = {num(c.rho_ambient)}",
                      f"g_self = {num(c.g_self)}", f"beta = {num(c.beta)}", f"gravity = {arr(c.gravity)}",
                      f"a = {num(c.a)}", f"b = {num(c.b)}", f"R = {num(c.R)}", f"T = {num(c.T)}",
                      f"Tc = {num(c.Tc)}", f"omega = {num(c.omega)}"]
        n = len(self.components)
        if self.coupling is not None:
            g = np.asarray(self.coupling, float)
            for a in range(n):
                for b in range(a + 1, n):
                    if g[a, b] != 0.0:
                        lines += ["", "[[coupling]]", f"pair = [{a}, {b}]", f"g = {num(g[a, b])}"]
        for sd in self.seeds:
            lines += ["", "[[seed]]"]
            if sd.shape == SEED_SPHERE:
                lines += ['shape = "sphere"', f"center = {arr(sd.center)}", f"radius = {num(sd.radius)}"]
            else:
                lines += ['shape = "box"', f"min = {arr(sd.box_min)}", f"max = {arr(sd.box_max)}"]
            lines += [f"component = {sd.component}", f"rho = {num(sd.rho)}", f"velocity = {arr(sd.velocity)}"]
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")


class CScenario:
    """Owns the ctypes buffers behind one ScenarioDesc."""

    def __init__(self, sc: Scenario):
        n = sc.n_components
        if not (1 <= n <= MAX_COMP):
            raise ValueError("1..4 components supported")
        self._comps = (ComponentDesc * n)()
        for k, c in enumerate(sc.components):
            d = self._comps[k]
            d.tau, d.rho_ambient, d.g_self, d.beta = c.tau, c.rho_ambient, c.g_self, c.beta
            for a in range(3):
                d.gravity[a] = c.gravity[a]
            d.a, d.b, d.R, d.T, d.Tc, d.omega = c.a, c.b, c.R, c.T, c.Tc, c.omega
        ns = len(sc.seeds)
        self._seeds = (SeedDesc * max(ns, 1))()
        for k, s in enumerate(sc.seeds):
            d = self._seeds[k]
            d.shape, d.component = s.shape, s.component
            for a in range(3):
                d.box_min[a], d.box_max[a] = s.box_min[a], s.box_max[a]
                d.center[a], d.velocity[a] = s.center[a], s.velocity[a]
            d.radius, d.rho = s.radius, s.rho
        cp = np.zeros((n, n)) if sc.coupling is None else np.asarray(sc.coupling, np.float64)
        self._coupling = np.ascontiguousarray(cp, dtype=np.float64)
        self._geom = None
        if sc.geometry is not None:
            g = np.ascontiguousarray(sc.geometry, dtype=np.uint8)
            if g.shape != (sc.domain[2], sc.domain[1], sc.domain[0]):
                raise ValueError("geometry must be [nz, ny, nx]")
            self._geom = g
        self._p2p = None
        if sc.p2p is not None:
            self._p2p = np.ascontiguousarray(sc.p2p, dtype=np.uint8)
        d = ScenarioDesc()
        for a in range(3):
            d.domain[a] = sc.domain[a]
            d.periodic[a] = int(sc.periodic[a])
        d.tile_extent, d.mode, d.threshold = sc.tile_extent, sc.mode, sc.threshold
        d.devices, d.policy = sc.devices, sc.policy
        d.weight_p2p, d.weight_staged = sc.weight_p2p, sc.weight_staged
        d.p2p = (self._p2p.ctypes.data_as(C.POINTER(C.c_uint8))
                 if self._p2p is not None else None)
        d.n_components = n
        d.components = C.cast(self._comps, C.POINTER(ComponentDesc))
        d.coupling = self._coupling.ctypes.data_as(C.POINTER(C.c_double))
        d.n_seeds = ns
        d.seeds = C.cast(self._seeds, C.POINTER(SeedDesc))
        d.geometry = (self._geom.ctypes.data_as(C.POINTER(C.c_uint8))
                      if self._geom is not None else None)
        self.desc = d

    def ptr(self):
        return C.byref(self.desc)


# ---------------------------------------------------------------------------
# Component presets (parameters from proj/tests/acceptance.cpp:623-660).

def ideal_gas(tau: float = 1.0, rho_ambient: float = 1.0) -> Component:
    """Single-component ideal gas: R T = cs2 makes psi = 0 (physics.hpp:19)."""
    return Component(tau=tau, rho_ambient=rho_ambient)


def pr_heavy() -> Component:
    """Peng-Robinson liquid/vapour component (acceptance.cpp:625-634)."""
    Tc = 0.072922004074134239
    return Component(tau=1.0, a=2.0 / 49.0, b=2.0 / 21.0, R=1.0, Tc=Tc,
                     T=0.85 * Tc, omega=0.344, g_self=-1.0,
                     rho_ambient=0.34130948026364294)


def ideal_light() -> Component:
    """Ideal-like light component, psi = sqrt(2 rho) (acceptance.cpp:636-640)."""
    return Component(tau=1.0, T=2.0 / 3.0, g_self=1.0, rho_ambient=0.4)


def _ramp01(frac: float) -> float:
    return 0.5 * (1.0 - math.cos(frac * 3.14159265358979323846))


def ramped_sphere_seeds(center, r_core: float, rho_l: float, rho_v: float,
                        ramp: int = 6, component: int = 0) -> List[Seed]:
    """Concentric spheres: outermost first so inner shells overwrite (seeds are
    applied in list order, proj/src/engine.cpp:43-76) -- a cosine ramp from
    rho_v to rho_l over `ramp` cells, then the liquid core."""
    seeds = []
    for i in range(ramp):  # shell i covers r <= r_core + ramp - i
        s = _ramp01((i + 0.5) / ramp)
        seeds.append(Seed(shape=SEED_SPHERE, component=component, center=tuple(center),
                          radius=r_core + ramp - i, rho=rho_v + (rho_l - rho_v) * s))
    seeds.append(Seed(shape=SEED_SPHERE, component=component, center=tuple(center),
                      radius=r_core, rho=rho_l))
    return seeds


def config1(threshold: float = 0.0, mode: int = MODE_PROGRESSIVE, n: int = 64,
            extent: int = 16) -> Scenario:
    """C1: D3Q19 single component, inflow emulated by a moving seeded box into an
    empty 64^3 domain, 16^3 subdomains."""
    q = n // 4
    return Scenario(domain=(n, n, n), tile_extent=extent, mode=mode, threshold=threshold,
                    components=[ideal_gas(tau=0.8)],
                    seeds=[Seed(box_min=(0, q, q), box_max=(q, 3 * q, 3 * q), rho=1.1,
                                velocity=(0.05, 0.0, 0.0))],
                    name="c1")


def mpmc_release(n: int = 256, extent: int = 32, mode: int = MODE_PROGRESSIVE,
                 threshold: float = 1e-9, r_core: Optional[float] = None,
                 devices: int = 1, n_components: int = 2,
                 domain: Optional[Sequence[int]] = None) -> Scenario:
    """C2/C3/C5: two-component MPMC (Peng-Robinson liquid/vapour + ideal-like
    light gas) released from a ramped liquid sphere at the domain centre
    (SURVEY §8(d) C2).  n_components=3 adds a second ideal-like component
    coupled to both (C5)."""
    dom = tuple(domain) if domain is not None else (n, n, n)
    comps = [pr_heavy(), ideal_light()]
    if n_components == 1:  # single-component multiphase (PR liquid/vapour only)
        comps = [pr_heavy()]
    if n_components == 3:
        comps.append(Component(tau=1.0, T=2.0 / 3.0, g_self=1.0, rho_ambient=0.3))
    nc = len(comps)
    g = np.full((nc, nc), 0.08)
    np.fill_diagonal(g, 0.0)
    if r_core is None:
        r_core = min(dom) / 8.0
    center = tuple(d / 2.0 for d in dom)
    heavy = comps[0]
    seeds = ramped_sphere_seeds(center, r_core, 6.5, heavy.rho_ambient, 6, 0)
    return Scenario(domain=dom, tile_extent=extent, mode=mode, threshold=threshold,
                    devices=devices, components=comps, coupling=g, seeds=seeds,
                    name="mpmc_release")


BENCH_DEVICES = 16  # simulated devices of the bench workload (placement only)


def bench_c2(mode: int = MODE_PROGRESSIVE) -> Scenario:
    """The benchmark workload (BASELINE.json configs[1]):
    256^3, 32^3 subdomains, two-component MPMC sphere release, S = 1e-9.
    Owners are placed over BENCH_DEVICES simulated devices so the reference
    CPU engine can spread the tiles over that many worker threads
    (engine.cpp:214-218: tile owner % W); on the GPU the owner is placement
    metadata only (byte classes, creation log)."""
    return mpmc_release(n=256, extent=32, mode=mode, threshold=1e-9, devices=BENCH_DEVICES)


def mpmc_release_weak(n_blocks: int, n: int = 256, extent: int = 32, threshold: float = 1e-9) -> Scenario:
    """Weak-scaling form of C2 for N GPUs: N 256^3 blocks side by side along x,
    each with its own ramped liquid sphere (the single-GPU case is exactly
    mpmc_release(256)); owners = GPUs (devices = N)."""
    sc = mpmc_release(n=n, extent=extent, threshold=threshold, devices=n_blocks,
                      domain=(n * n_blocks, n, n))
    heavy = sc.components[0]
    seeds = []
    for b in range(n_blocks):
        seeds += ramped_sphere_seeds((n * b + n / 2.0, n / 2.0, n / 2.0), n / 8.0, 6.5,
                                     heavy.rho_ambient, 6, 0)
    sc.seeds = seeds
    sc.name = f"mpmc_release_weak_x{n_blocks}"
    return sc


# ---- 3-D channel network --------------------------
def channel_network(nx: int = 1024, ny: int = 512, nz: int = 512, seed: int = 1510,
                    radius: Optional[float] = None) -> np.ndarray:
    """Deterministic 3-D channel network in solid rock, uint8 [nz, ny, nx]
    (x fastest, 1 = solid), the geometry of BASELINE config 4.

    An inlet channel runs along +x from x = 0 on the domain axis; at a quarter
    of the length it splits into four branches that wander (seeded random
    turns) towards the far end, each splitting once more.  Channels are
    capsules (cylinders with round ends) of radius r (r/2 for the last
    level).  Every dimension scales with the domain, so a 64 x 32 x 32 copy
    is the parity-test version of the same network (three branching levels,
    radius r, 0.8 r, 0.65 r, 0.5 r; r = ny / 14 by default)."""
    rng = np.random.default_rng(seed)
    r0 = radius if radius is not None else max(2.0, ny / 14.0)
    g = np.ones((nz, ny, nx), np.uint8)
    zz, yy, xx = (np.arange(n, dtype=np.float64) + 0.5 for n in (nz, ny, nx))

    def capsule(p, q, r):
        p, q = np.asarray(p, float), np.asarray(q, float)
        lo = np.maximum(np.floor(np.minimum(p, q) - r - 1).astype(int), 0)
        hi = np.minimum(np.ceil(np.maximum(p, q) + r + 1).astype(int), (nx, ny, nz))
        if np.any(hi <= lo):
            return
        X = xx[lo[0]:hi[0]][None, None, :]
        Y = yy[lo[1]:hi[1]][None, :, None]
        Z = zz[lo[2]:hi[2]][:, None, None]
        d = q - p
        L2 = float(d @ d) or 1.0
        t = np.clip(((X - p[0]) * d[0] + (Y - p[1]) * d[1] + (Z - p[2]) * d[2]) / L2, 0.0, 1.0)
        dist2 = (X - p[0] - t * d[0]) ** 2 + (Y - p[1] - t * d[1]) ** 2 + (Z - p[2] - t * d[2]) ** 2
        sub = g[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        sub[dist2 <= r * r] = 0

    def wander(p, direction, length, r, steps):
        pts = [np.asarray(p, float)]
        d = np.asarray(direction, float)
        d /= np.linalg.norm(d)
        for _ in range(steps):
            turn = rng.normal(0.0, 0.35, 3)
            turn[0] = abs(turn[0]) * 0.2  # keep heading downstream
            d = d + turn
            d[0] = max(d[0], 0.35)
            d /= np.linalg.norm(d)
            q = pts[-1] + d * (length / steps)
            q = np.clip(q, [0, r + 1, r + 1], [nx - 1, ny - r - 1, nz - r - 1])
            capsule(pts[-1], q, r)
            pts.append(q)
        return pts[-1], d

    inlet = np.array([0.0, ny / 2.0, nz / 2.0])
    junction = np.array([nx / 4.0, ny / 2.0, nz / 2.0])
    capsule(inlet, junction, r0)
    for dy, dz in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
        end, d = wander(junction, (1.0, 0.6 * dy, 0.6 * dz), nx * 0.3, r0 * 0.8, 6)
        for s in (1, -1):
            end2, d2 = wander(end, (1.0, d[1] + 0.5 * s, d[2] - 0.5 * s), nx * 0.25, r0 * 0.65, 5)
            for t in (1, -1):
                wander(end2, (1.0, d2[1] - 0.5 * t, d2[2] + 0.5 * t), nx * 0.25, r0 * 0.5, 5)
    return g


def mpmc_channel(nx: int = 1024, ny: int = 512, nz: int = 512, extent: int = 32,
                 threshold: float = 1e-9, mode: int = MODE_PROGRESSIVE, devices: int = 1,
                 seed: int = 1510) -> Scenario:
    """C4: C2's two-component MPMC with the ramped liquid sphere wholly inside
    the inlet channel of the 3-D channel network."""
    geo = channel_network(nx, ny, nz, seed)
    comps = [pr_heavy(), ideal_light()]
    g = np.full((2, 2), 0.08)
    np.fill_diagonal(g, 0.0)
    r0 = max(2.0, ny / 14.0)
    core = r0 * 0.5
    center = (nx / 8.0, ny / 2.0, nz / 2.0)
    seeds = ramped_sphere_seeds(center, core, 6.5, comps[0].rho_ambient, max(1, int(r0 * 0.4)), 0)
    return Scenario(domain=(nx, ny, nz), tile_extent=extent, mode=mode, threshold=threshold,
                    devices=devices, components=comps, coupling=g, seeds=seeds, geometry=geo,
                    name="mpmc_channel")


def save_lbmgeo(mask: np.ndarray, path: str) -> None:
    """LBMGEO v1 (proj/src/geometry.cpp:64-75): 'LBMGEO v1 nx ny nz\\n' + bytes."""
    nz, ny, nx = mask.shape
    with open(path, "wb") as fh:
        fh.write(f"LBMGEO v1 {nx} {ny} {nz}\n".encode())
        fh.write(np.ascontiguousarray(mask, np.uint8).tobytes())
