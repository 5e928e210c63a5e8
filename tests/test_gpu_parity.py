"""GPU parity: the B200 engine (through the C-ABI) against the oracle
restatement, bit for bit in FP64 — every field of every tile, the creation
log (activation set + order + trigger + owner), the diagnostics counters and
the modeled byte classes."""
import pytest

from paper_1510_03560_b200 import capi
from tests import scenarios
from tests.compare import assert_same_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [0, 20, 26, 27, 1, 21, 22, 100, 200], ids=["default", "percomp_wholetile", "percomp_halftile", "percomp_quartertile", "plain", "percomp_late_head", "percomp_lag2", "percomp_fused_face", "percomp_strided_xfaces"])
@pytest.mark.parametrize("name", sorted(scenarios.ALL))
def test_gpu_matches_oracle(built, name, variant):
    make, steps = scenarios.ALL[name]
    sc = make()
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    gpu.set_kernel_variant(variant)
    assert_same_state(orc, gpu, label=f"{name}@0")
    orc.step(1)
    gpu.step(1)
    assert_same_state(orc, gpu, label=f"{name}@1")
    orc.step(steps - 1)
    gpu.step(steps - 1)
    assert_same_state(orc, gpu, label=f"{name}@{steps}")


@pytest.mark.parametrize("name", sorted(__import__("tests.golden_check", fromlist=["x"]).load_golden()))
def test_gpu_reproduces_reference_golden_states(built, name):
    """Against the state the reference itself produced (tests/golden/)."""
    from tests.golden_check import assert_matches_golden
    make, steps = scenarios.ALL[name]
    gpu = capi.gpu_engine(make(), capture=True)
    gpu.step(steps)
    assert_matches_golden(gpu, name)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32", "c1_static"])
def test_poked_nan_matches_reference(built, name, variant):
    """proj/tests/test_engine.cpp:284-310: a NaN written into one f_read
    population between steps -> the same EngineError (iteration, tile, phase)
    as the reference, and no advance of iteration / cell_updates.  (A finite
    poke is not comparable: the reference's collision then mixes the poked
    f_read with the u of the previous P5, which this engine recomputes.)"""
    value = float("nan")
    from tests.conftest import have_ref
    from paper_1510_03560_b200.scenario import EngineError
    if not have_ref():
        pytest.skip("reference shim not built")
    make, _ = scenarios.ALL[name]
    sc = make()
    ref = capi.ref_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    gpu.set_kernel_variant(variant)
    ref.step(3)
    gpu.step(3)
    coords = ref.tiles()[0][0]
    E = sc.tile_extent
    local = (E // 2, E // 2 - 1, E // 2 + 1)
    ref.poke_f(coords, 0, 7, local, value)
    gpu.poke_f(coords, 0, 7, local, value)
    errs = []
    for eng in (ref, gpu):
        try:
            eng.step(3)
            errs.append(None)
        except EngineError as e:
            errs.append((e.iteration, tuple(e.tile), e.phase))
    assert errs[0] == errs[1], errs
    assert errs[0] is not None
    for k in ("iteration", "cell_updates"):
        assert ref.counters()[k] == gpu.counters()[k]


@pytest.mark.parametrize("mode", ["device", "host_overflow", "host"])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "c1_progressive_S0", "mpmc_channel_e16", "mpmc_e32", "mpmc_e64"])
def test_expansion_paths_match_oracle(built, name, mode, monkeypatch):
    """The device-side expansion (k_check_expand), its overflow to the host
    (births beyond the launched grid, headroom 0) and the host-only path give
    the reference's creation log, owners, counters and fields."""
    if mode == "host":
        monkeypatch.setenv("PLBM_DEVICE_EXPAND", "0")
    if mode == "host_overflow":
        monkeypatch.setenv("PLBM_EXPAND_HEADROOM", "0")
    make, steps = scenarios.ALL[name]
    sc = make()
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    for chunk in (1, steps - 1):
        orc.step(chunk)
        gpu.step(chunk)
        assert_same_state(orc, gpu, label=f"{name}/{mode}")


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32", "mpmc_s0_3dev", "mpmc3_e32"])
def test_interior_blowup_reports_p5_like_reference(built, name, variant):
    """An interior blow-up created by the collision itself must be reported
    the way the reference reports it: EngineError(k, tile, "P5") from the
    post-stream moments scan of EVERY fluid cell (proj/src/engine.cpp:
    500-512), not one step later as a P1 density NaN.

    Drive: a huge rest population (f_0 = 1e308, e_0 = 0) is written into an
    interior cell of the ideal-like component that is exactly at rest (u == 0,
    so both engines collide it with u = 0: the reference with its stored P5
    u, this engine with u recomputed from the poked populations).  P1 passes
    (rho finite, no pole for a = b = 0), psi overflows to +inf, the cell's
    Shan-Chen force is inf * 0 = NaN and its post-collision populations are
    NaN, which the P5 scan of the same step finds inside the tile.  Counters
    after the abort: iteration / cell_updates not advanced, the failing step's
    exchange bytes counted (P2 and P4 ran), diagnostics of the whole step."""
    import numpy as np
    from tests.conftest import have_ref
    from paper_1510_03560_b200.scenario import EngineError, FIELD_UX, FIELD_UY, FIELD_UZ
    if not have_ref():
        pytest.skip("reference shim not built")
    make, _ = scenarios.ALL[name]
    sc = make()
    ref = capi.ref_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    assert gpu.set_kernel_variant(variant) in (None, 0)
    ref.step(3)
    gpu.step(3)
    E = sc.tile_extent
    comp = 1
    coords = None
    for tc, _, _ in ref.tiles():
        u = [ref.read_tile(tc, comp, f) for f in (FIELD_UX, FIELD_UY, FIELD_UZ)]
        rest = (u[0] == 0) & (u[1] == 0) & (u[2] == 0)
        inner = np.zeros_like(rest)
        inner[3:E - 3, 3:E - 3, 3:E - 3] = True
        zz, yy, xx = np.nonzero(rest & inner)
        if len(xx):
            coords, local = tc, (int(xx[0]), int(yy[0]), int(zz[0]))
            break
    assert coords is not None, "no interior cell at rest"
    ref.poke_f(coords, comp, 0, local, 1e308)
    gpu.poke_f(coords, comp, 0, local, 1e308)
    errs = []
    for eng in (ref, gpu):
        try:
            eng.step(3)
            errs.append(None)
        except EngineError as e:
            errs.append((e.iteration, tuple(e.tile), e.phase))
    assert errs[0] == errs[1], errs
    assert errs[0] == (4, tuple(coords), "P5"), errs
    rc, gc = ref.counters(), gpu.counters()
    for k in ("iteration", "cell_updates", "bytes", "negative_populations", "psi_clamps",
              "zero_rho_forcings", "tiles", "suppressed_expansions"):
        assert rc[k] == gc[k], (k, rc[k], gc[k])


@pytest.mark.parametrize("name", ["c1_static", "mpmc_progressive_e16"])
def test_p5_screen_has_no_false_alarm(built, name):
    """Huge but finite populations (outside the screen's range, so the tile is
    checked exactly every step) must not raise anything the reference does not
    raise: a psi-free single component with f_0 = 1e300 stays finite."""
    from tests.conftest import have_ref
    from paper_1510_03560_b200.scenario import EngineError
    if not have_ref():
        pytest.skip("reference shim not built")
    make, steps = scenarios.ALL[name]
    sc = make()
    ref = capi.ref_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    ref.step(2)
    gpu.step(2)
    coords = ref.tiles()[0][0]
    E = sc.tile_extent
    comp = sc.n_components - 1
    local = (E // 2, E // 2, E // 2)
    ref.poke_f(coords, comp, 0, local, 1e300 if sc.n_components == 1 else 1e-320)
    gpu.poke_f(coords, comp, 0, local, 1e300 if sc.n_components == 1 else 1e-320)
    errs = []
    for eng in (ref, gpu):
        try:
            eng.step(3)
            errs.append(None)
        except EngineError as e:
            errs.append((e.iteration, tuple(e.tile), e.phase))
    assert errs[0] == errs[1], errs
    for k in ("iteration", "cell_updates"):
        assert ref.counters()[k] == gpu.counters()[k]


def _aa_scenarios():
    # A-A runs on the fused cluster kernels (whole or split tiles) or on one
    # CTA per tile (E <= 32): every parity scenario
    return sorted(scenarios.ALL)


@pytest.mark.parametrize("variant", [20, 26, 27], ids=["wholetile", "halftile", "quartertile"])
@pytest.mark.parametrize("name", _aa_scenarios())
def test_aa_storage_matches_oracle(built, name, variant):
    """A-A in-place streaming (one population buffer): the
    same bit-exact state as the oracle after the first step (an AA_LOCAL
    step), after the second (AA_NEIGH) and at the end — the read-back itself
    goes through the A-A addressing of the next step's kind."""
    make, steps = scenarios.ALL[name]
    sc = make()
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True, storage="aa")
    if variant == 20 and sc.tile_extent == 64 and sc.n_components == 3:
        with pytest.raises(ValueError):  # no whole-tile cluster (24 CTAs) at this shape
            gpu.set_kernel_variant(variant)
        return
    gpu.set_kernel_variant(variant)
    for k in (1, 1, steps - 2):
        orc.step(k)
        gpu.step(k)
        assert_same_state(orc, gpu, label=f"{name}/aa@{orc.counters()['iteration']}")


@pytest.mark.parametrize("mode", ["device", "host"])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "c1_progressive_S0", "mpmc_channel_e16", "mpmc_e32"])
def test_aa_expansion_paths_match_oracle(built, name, mode, monkeypatch):
    """A-A with births: stores into newborn tiles follow ROUTE_W, whether the
    device (k_check_expand) or the host mirror grows the map."""
    if mode == "host":
        monkeypatch.setenv("PLBM_DEVICE_EXPAND", "0")
    make, steps = scenarios.ALL[name]
    sc = make()
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True, storage="aa")
    for chunk in (1, 2, steps - 3):
        orc.step(chunk)
        gpu.step(chunk)
        assert_same_state(orc, gpu, label=f"{name}/aa/{mode}")


def test_aa_halves_population_memory(built, monkeypatch):
    """The A-A engine allocates one population buffer: the device memory an
    engine takes drops by about the size of one buffer (pools allocated up
    front, PLBM_LAZY_POOL=0, so the whole pool is counted)."""
    import torch
    monkeypatch.setenv("PLBM_LAZY_POOL", "0")
    sc = scenarios.ALL["mpmc_e32"][0]()
    free0 = torch.cuda.mem_get_info()[0]
    ab = capi.gpu_engine(sc)
    free_ab = torch.cuda.mem_get_info()[0]
    ab.close()
    free1 = torch.cuda.mem_get_info()[0]
    aa = capi.gpu_engine(sc, storage="aa")
    free_aa = torch.cuda.mem_get_info()[0]
    aa.close()
    used_ab, used_aa = free0 - free_ab, free1 - free_aa
    n = 1
    for d in sc.domain:
        n *= d
    one_buffer = n * sc.n_components * 19 * 8
    assert used_ab - used_aa >= 0.9 * one_buffer, (used_ab, used_aa, one_buffer)


def test_e64_three_components_run_on_split_clusters(built):
    """E = 64 with three components: a whole-tile cluster would need 24 CTAs,
    so k_main_pc runs with 2 or 4 clusters per tile (12 / 6 CTAs) — A-B and
    A-A, bit-exact against the oracle — and the whole-tile variant falls back
    to the plain kernel (A-B) or is refused (A-A)."""
    make, steps = scenarios.ALL["mpmc3_e64_solid"]
    for storage in ("ab", "aa"):
        for v in (26, 27):
            sc = make()
            orc = capi.oracle_engine(sc)
            gpu = capi.gpu_engine(sc, capture=True, storage=storage)
            gpu.set_kernel_variant(v)
            orc.step(steps)
            gpu.step(steps)
            assert_same_state(orc, gpu, label=f"e64c3/{storage}/{v}")


@pytest.mark.parametrize("storage", ["ab", "aa"])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32"])
def test_eos_pole_matches_reference(built, name, storage):
    """proj/src/physics.cpp:12-27: pr_pressure throws when b * rho >= 1.  A
    rest population of 20 poked into a Peng-Robinson cell (b = 2/21, so rho
    > 1/b) must give the reference's EngineError (iteration, tile, "P1") and
    leave iteration / cell_updates where the reference leaves them."""
    from tests.conftest import have_ref
    from paper_1510_03560_b200.scenario import EngineError
    if not have_ref():
        pytest.skip("reference shim not built")
    make, _ = scenarios.ALL[name]
    sc = make()
    ref = capi.ref_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True, storage=storage)
    ref.step(3)
    gpu.step(3)
    tiles = [t[0] for t in ref.tiles()]
    coords = tiles[len(tiles) // 2]
    E = sc.tile_extent
    local = (E // 2 + 1, E // 2, E // 2 - 1)
    ref.poke_f(coords, 0, 0, local, 20.0)
    gpu.poke_f(coords, 0, 0, local, 20.0)
    errs = []
    for eng in (ref, gpu):
        try:
            eng.step(2)
            errs.append(None)
        except EngineError as e:
            errs.append((e.iteration, tuple(e.tile), e.phase, "pole" in str(e).lower()))
    assert errs[0] is not None and errs[0] == errs[1], errs
    for k in ("iteration", "cell_updates"):
        assert ref.counters()[k] == gpu.counters()[k], k


@pytest.mark.parametrize("storage", ["ab", "aa"])
def test_lazy_pool_follows_active_tiles(built, storage):
    """One-rank pools are a reserved address range backed only for the tiles
    the launches can reach (plus the mapper thread's look-ahead): a
    progressive run starts with a fraction of the pool mapped, maps more as
    the mesh grows, and stays bit-exact."""
    from paper_1510_03560_b200 import scenario as S
    steps = 12
    sc = S.mpmc_channel(nx=256, ny=128, nz=128, extent=16, threshold=1e-10)  # 1024-tile capacity
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True, storage=storage)
    m0 = gpu.memory()
    assert 0 < m0["pool_mapped_bytes"] < m0["pool_reserved_bytes"], m0
    orc.step(steps)
    gpu.step(steps)
    assert_same_state(orc, gpu, label=f"lazy/{storage}")
    m1 = gpu.memory()
    assert m1["pool_reserved_bytes"] == m0["pool_reserved_bytes"]
    assert m1["pool_mapped_bytes"] >= m0["pool_mapped_bytes"]
    # backed: the tiles (+ headroom and the ambient slot) rounded up to
    # granules per buffer, never the whole capacity of a sparse mesh
    nb = 1 if storage == "aa" else 2
    tiles = len(gpu.tiles())
    slot = m1["pool_reserved_bytes"] / nb / (sc.domain[0] * sc.domain[1] * sc.domain[2] // sc.tile_extent ** 3 + 1)
    launch = tiles + max(64, tiles // 4)                               # launch_tiles_
    ahead = launch + max(launch // 4, int(m1["granule_bytes"] // slot))  # the mapper's target
    bound = nb * ((ahead + 1) * slot + 2 * m1["granule_bytes"])
    assert m1["pool_mapped_bytes"] <= bound, (m1, tiles, slot)


def test_eager_pool_matches_oracle(built, monkeypatch):
    """PLBM_LAZY_POOL=0 (whole pool allocated up front) is the same engine."""
    monkeypatch.setenv("PLBM_LAZY_POOL", "0")
    make, steps = scenarios.ALL["mpmc_channel_e16"]
    sc = make()
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    m = gpu.memory()
    assert m["pool_mapped_bytes"] == m["pool_reserved_bytes"]
    orc.step(steps)
    gpu.step(steps)
    assert_same_state(orc, gpu, label="eager")
