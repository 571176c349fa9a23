"""fp32 throughput mode (BASELINE.json north_star: forces, torques and tangential histories within
1e-5 relative in fp32 mode). The fp64 parity path is the reference here (it is
itself bitwise with the CPU oracle, tests/test_gpu_parity.py). Relative means relative to the
particle's sum of contact-force magnitudes (net forces in dense packs nearly cancel).
"""
import numpy as np
import pytest

import paper_1503_03553_b200 as dem

pytestmark = pytest.mark.gpu

TOL = 1e-5


def contact_scale(ps, o, p, d):
    """Per particle, the sum over its contacts of the magnitudes of the force terms
    (contact_mechanics.cpp:28-33, 48-55): Hertz k_n dn^1.5, tangential spring k_t |delta_t| and
    damping eta (|v_rel| + spin), default material. Walls use r_eff = r, m_eff = m."""
    m = dem.MaterialParams()
    young_sum = 2.0 * (2.0 - m.poisson_ratio ** 2) / m.youngs_modulus
    shear_sum = 2.0 * (2.0 - m.poisson_ratio) / m.shear_modulus
    le = np.log(m.restitution)
    alpha = -2.0 * le / np.sqrt(np.pi ** 2 + le ** 2)
    pp = p >= 0
    i, j = o[pp], p[pp]
    x, v, w, r, ms = ps.positions, ps.velocities, ps.angular_velocities, ps.radii, ps.masses
    dist = np.linalg.norm(x[j] - x[i], axis=1)
    dn = np.maximum(r[i] + r[j] - dist, 0.0)
    r_eff = r[i] * r[j] / (r[i] + r[j])
    m_eff = ms[i] * ms[j] / (ms[i] + ms[j])
    kn = (4.0 / 3.0) * np.sqrt(r_eff) / young_sum
    kt = 8.0 * np.sqrt(r_eff * dn) / shear_sum
    eta = alpha * np.sqrt(m_eff * kn * np.sqrt(dn))
    vmag = (np.linalg.norm(v[i] - v[j], axis=1) + np.linalg.norm(w[i], axis=1) * r[i]
            + np.linalg.norm(w[j], axis=1) * r[j])
    term = kn * dn * np.sqrt(dn) + kt * np.linalg.norm(d[pp], axis=1) + eta * vmag
    s = np.zeros(len(ps.ids))
    np.add.at(s, i, term)
    return s


def history_map(sim):
    ps = sim.particles()
    o, p, d = sim.contacts()
    return {(int(ps.ids[a]), int(ps.ids[b]) if b >= 0 else int(b)): dt for a, b, dt in zip(o, p, d)}


def make(n, poly, seed, precision):
    ps, dmax = dem.gen_packing(n, s=1.4 if poly else 1.8, jit=0.2, poly=poly, seed=seed,
                               omega_half=50.0 if poly else 0.5)
    cfg = dem.packing_config(dmax, poly=poly)
    cfg.precision = precision
    return dem.Simulation(ps, cfg)


@pytest.mark.parametrize("n,poly,seed", [(32768, False, 41), (32768, True, 42)])
def test_fp32_forces_within_1e5_of_fp64(cuda, n, poly, seed):
    a, b = make(n, poly, seed, 0), make(n, poly, seed, 1)
    for k in range(4):  # the priming pass (no history) and 3 steps with history
        if k:
            ma, mb = a.step(), b.step()
            assert ma.contacts == mb.contacts and ma.pp_contact_events == mb.pp_contact_events
        pa, pb = a.particles(), b.particles()
        assert np.array_equal(pa.ids, pb.ids)
        o, p, d = a.contacts()
        scale = contact_scale(pa, o, p, d)
        has = scale > 0
        fa, fb = a.forces(), b.forces()
        ef = np.linalg.norm(fa.force - fb.force, axis=1)
        et = np.linalg.norm(fa.torque - fb.torque, axis=1)
        assert (ef[has] <= TOL * scale[has]).all(), (k, (ef[has] / scale[has]).max())
        assert (et[has] <= TOL * scale[has] * pa.radii[has]).all(), (k, (et[has] / (scale[has] * pa.radii[has])).max())
        # history: relative to |delta_t| plus one step's increment scale |v_rel| dt (the fp32
        # tangential projection of v_rel cancels when v_rel is nearly normal)
        ha, hb = history_map(a), history_map(b)
        assert ha.keys() == hb.keys()
        o, p, d = a.contacts()
        pp = p >= 0
        v, w, r = pa.velocities, pa.angular_velocities, pa.radii
        inc = np.linalg.norm(v[o], axis=1) + np.linalg.norm(w[o], axis=1) * r[o]
        inc[pp] = (np.linalg.norm(v[o[pp]] - v[p[pp]], axis=1) + np.linalg.norm(w[o[pp]], axis=1) * r[o[pp]]
                   + np.linalg.norm(w[p[pp]], axis=1) * r[p[pp]])
        dt = 1e-5
        keys = [(int(pa.ids[x]), int(pa.ids[y]) if y >= 0 else int(y)) for x, y in zip(o, p)]
        db = np.array([hb[k_] for k_ in keys]).reshape(-1, 3)
        ref = np.linalg.norm(d, axis=1) + inc * dt
        assert (np.linalg.norm(d - db, axis=1) <= TOL * ref).all(), (k, (np.linalg.norm(d - db, axis=1) / ref).max())


def test_fp32_statistics_track_fp64(cuda):
    """Trajectories are chaotic, so multi-step runs are compared by kinetic energy and
    coordination number (north_star): 200 steps of the dense packing."""
    a, b = make(8000, False, 43, 0), make(8000, False, 43, 1)
    for k in range(200):
        ma, mb = a.step(), b.step()
        if k % 20 == 19:
            ka = dem.total_kinetic_energy(a.particles())
            kb = dem.total_kinetic_energy(b.particles())
            assert abs(ka - kb) <= 1e-5 * ka, (k, ka, kb)
            assert abs(ma.contacts - mb.contacts) <= 1e-3 * ma.contacts


def test_fp32_rejects_single_loop(cuda):
    ps, dmax = dem.gen_packing(512, seed=1)
    cfg = dem.packing_config(dmax)
    cfg.precision = 1
    cfg.collide_variant = dem.BASELINE
    with pytest.raises(dem.ConfigError):
        dem.Simulation(ps, cfg)
