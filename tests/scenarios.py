"""Small parity scenarios (sizes the CPU oracle finishes in seconds).

Each covers a different part of the path: ghost routing, progressive
activation at S = 0 (rounding-noise driven) and S > 0, periodic
self-neighbours, solids (bounce-back + solid ghost psi), gravity, placement
on several simulated devices, two and three MPMC components.
"""
import numpy as np

from paper_1510_03560_b200 import scenario as S


def c1_progressive(extent=8, n=32, threshold=1e-12):
    return S.config1(threshold=threshold, n=n, extent=extent)


def c1_static(extent=8, n=32):
    return S.config1(n=n, extent=extent, mode=S.MODE_STATIC)


def mpmc_progressive(extent=16, n=32, threshold=1e-9, devices=1):
    return S.mpmc_release(n=n, extent=extent, threshold=threshold, r_core=5, devices=devices)


def mpmc_s0(extent=8, n=32):
    return S.mpmc_release(n=n, extent=extent, threshold=0.0, r_core=5, devices=3)


def periodic_solid_gravity(extent=8, n=32):
    sc = S.config1(threshold=1e-12, n=n, extent=extent)
    sc.periodic = (1, 0, 1)
    sc.devices = 4
    sc.policy = S.POLICY_SIMPLE
    g = np.zeros((n, n, n), np.uint8)
    g[:, :, 20:22] = 1
    g[5:9, 3:30, 3:18] = 1
    sc.geometry = g
    sc.components[0].gravity = (1e-5, 0.0, -2e-5)
    return sc


def closed_box(n=32, extent=16):
    """Acceptance criterion 2 shape (proj/tests/acceptance.cpp:206-237)."""
    sc = S.Scenario(domain=(n, n, n), tile_extent=extent, mode=S.MODE_STATIC,
                    components=[S.Component(tau=0.9)],
                    seeds=[S.Seed(box_min=(8, 8, 8), box_max=(24, 24, 24), rho=1.2,
                                  velocity=(0.04, 0.02, 0.01))])
    g = np.zeros((n, n, n), np.uint8)
    g[0, :, :] = g[-1, :, :] = g[:, 0, :] = g[:, -1, :] = g[:, :, 0] = g[:, :, -1] = 1
    sc.geometry = g
    return sc


def mpmc3_static(extent=8, n=16):
    return S.mpmc_release(n=n, extent=extent, mode=S.MODE_STATIC, r_core=3, n_components=3)


def mpmc_periodic_solid(extent=8, n=32):
    sc = S.mpmc_release(n=n, extent=extent, threshold=1e-10, r_core=5, devices=2)
    sc.periodic = (0, 1, 0)
    g = np.zeros((n, n, n), np.uint8)
    g[:, 2:5, 24:28] = 1
    sc.geometry = g
    sc.components[1].gravity = (0.0, 0.0, -1e-6)
    return sc


ALL = {
    "c1_progressive": (c1_progressive, 20),
    "c1_static": (c1_static, 10),
    "c1_progressive_S0": (lambda: c1_progressive(threshold=0.0), 12),
    "mpmc_progressive_e16": (mpmc_progressive, 15),
    "mpmc_s0_3dev": (mpmc_s0, 12),
    "periodic_solid_gravity": (periodic_solid_gravity, 25),
    "closed_box": (closed_box, 20),
    "mpmc3_static": (mpmc3_static, 10),
    "mpmc_periodic_solid": (mpmc_periodic_solid, 20),
}


def mpmc_e32(n=64, threshold=1e-9):
    """C2 physics at E = 32 (the benchmark tile size; 4-CTA cluster kernel)."""
    return S.mpmc_release(n=n, extent=32, threshold=threshold, r_core=8)


def mpmc_e32_solid_periodic(n=64):
    sc = S.mpmc_release(n=n, extent=32, mode=S.MODE_STATIC, r_core=8, devices=2)
    sc.domain = (64, 32, 64)
    sc.seeds = S.ramped_sphere_seeds((32.0, 16.0, 32.0), 8, 6.5, sc.components[0].rho_ambient, 6)
    sc.periodic = (1, 1, 0)
    g = np.zeros((64, 32, 64), np.uint8)
    g[40:44, :, 10:20] = 1
    g[:, 5:7, 50:60] = 1
    sc.geometry = g
    sc.components[0].gravity = (0.0, 1e-6, 0.0)
    return sc


def mpmc3_e32(n=32):
    return S.mpmc_release(n=n, extent=32, mode=S.MODE_STATIC, r_core=6, n_components=3)


def mpmc_e16_solid(n=32):
    sc = S.mpmc_release(n=n, extent=16, threshold=0.0, r_core=5, devices=4)
    g = np.zeros((n, n, n), np.uint8)
    g[20:23, 3:29, 10:14] = 1
    sc.geometry = g
    sc.periodic = (0, 0, 1)
    return sc


def mpmc_channel_e16():
    """C4 geometry at test scale: the 3-D channel network, liquid sphere in the
    inlet channel, progressive."""
    return S.mpmc_channel(nx=128, ny=64, nz=64, extent=16, threshold=1e-10)


ALL.update({
    "mpmc_channel_e16": (mpmc_channel_e16, 16),
    "mpmc_e32": (mpmc_e32, 8),
    "mpmc_e32_solid_periodic": (mpmc_e32_solid_periodic, 6),
    "mpmc3_e32": (mpmc3_e32, 6),
    "mpmc_e16_solid_S0": (mpmc_e16_solid, 10),
})


def mpmc_e64():
    """C5's largest tile size (E = 64, plain kernel with 16-row y-chunks):
    progressive at S = 0, liquid sphere next to the tile boundary."""
    sc = S.mpmc_release(extent=64, threshold=0.0, r_core=3, devices=2, domain=(128, 64, 64))
    sc.seeds = S.ramped_sphere_seeds((54.0, 32.0, 32.0), 3, 6.5, sc.components[0].rho_ambient, 6)
    return sc


def mpmc3_e64_solid():
    sc = S.mpmc_release(extent=64, mode=S.MODE_STATIC, r_core=6, n_components=3, domain=(64, 64, 128))
    sc.seeds = S.ramped_sphere_seeds((32.0, 32.0, 60.0), 6, 6.5, sc.components[0].rho_ambient, 6)
    sc.periodic = (0, 1, 0)
    g = np.zeros((128, 64, 64), np.uint8)  # [z, y, x]
    g[60:70, 10:50, 20:24] = 1
    sc.geometry = g
    return sc


def mp1_e64():
    """single-component PR multiphase at E = 64 (smallest psi ring)."""
    sc = S.mpmc_release(extent=64, mode=S.MODE_STATIC, r_core=6, n_components=1, domain=(64, 128, 64))
    sc.seeds = S.ramped_sphere_seeds((32.0, 60.0, 32.0), 6, 6.5, sc.components[0].rho_ambient, 6)
    return sc


ALL.update({
    "mp1_e64": (mp1_e64, 4),
    "mpmc_e64": (mpmc_e64, 8),
    "mpmc3_e64_solid": (mpmc3_e64_solid, 4),
})


def mpmc_islands():
    """Optimized placement on a non-uniform topology: 4 devices in two NVLink
    islands (p2p inside, staged across), S = 0 growth from an off-centre
    sphere — exercises classify / gamma_cost with all three link classes."""
    sc = S.mpmc_release(n=64, extent=16, threshold=0.0, r_core=4, devices=4)
    sc.seeds = S.ramped_sphere_seeds((20.0, 30.0, 34.0), 4, 6.5, sc.components[0].rho_ambient, 4)
    sc.p2p = np.array([[1, 1, 0, 0], [1, 1, 0, 0], [0, 0, 1, 1], [0, 0, 1, 1]], np.uint8)
    sc.weight_p2p, sc.weight_staged = 0.4, 1.3
    return sc


ALL.update({
    "mpmc_islands": (mpmc_islands, 12),
})


def mp1_e16():
    """single-component PR liquid/vapour at E = 16 (k_main_pc<16, 1>),
    progressive S = 1e-9, gravity."""
    sc = S.mpmc_release(n=64, extent=16, threshold=1e-9, r_core=5, n_components=1, devices=2)
    sc.components[0].gravity = (0.0, -1e-6, 0.0)
    return sc


def mp1_e32_solid():
    """single-component PR at E = 32 (k_main_pc<32, 1>), static, periodic in
    x, a solid slab through the sphere's edge."""
    sc = S.mpmc_release(extent=32, mode=S.MODE_STATIC, r_core=7, n_components=1, domain=(64, 32, 64))
    sc.seeds = S.ramped_sphere_seeds((32.0, 16.0, 32.0), 7, 6.5, sc.components[0].rho_ambient, 6)
    sc.periodic = (1, 0, 0)
    g = np.zeros((64, 32, 64), np.uint8)  # [z, y, x]
    g[20:26, 4:28, 36:40] = 1
    sc.geometry = g
    return sc


def mpmc3_e16():
    """three components at E = 16 (k_main_pc<16, 3>: 6-CTA clusters),
    progressive at S = 0 on 3 simulated devices."""
    return S.mpmc_release(n=64, extent=16, threshold=0.0, r_core=5, n_components=3, devices=3)


ALL.update({
    "mp1_e16": (mp1_e16, 14),
    "mp1_e32_solid": (mp1_e32_solid, 6),
    "mpmc3_e16": (mpmc3_e16, 10),
})
