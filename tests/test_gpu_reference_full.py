"""GPU parity against the LIVE reference at BASELINE.json's full sizes (oracle/_ref, the reference
core compiled from its own sources; prebuilt, it travels to the GPU box).

* configs[1] (262,144 dense monodisperse) and configs[2] (1,048,576 polydisperse 1:2 with the
  friction cap engaged, K = 32): the constructor's priming pass and two steps on the B200 and on
  the reference Simulation from identical inputs. After each, per stable id:
  - the contact-pair sets (owner id, partner id) are identical, bit-exact;
  - forces and torques agree within 1e-9 relative to the particle's sum of contribution
    magnitudes, sum_k |F_k| (+ |m g|) and sum_k |T_k| (SURVEY §8a notes: not |net F|, which nearly
    cancels in dense packs; the sums come from the CPU restatement on the same inputs);
  - tangential displacements agree within 1e-9 relative to |delta_t| (+ 1e-300).
  The two differ only in the in-cell order (canonical stable-id order here, the bitonic network's
  tie order there), so the sums are accumulated in different orders and agree to ulps, not bits.
* configs[0] (4,096 settling spheres in the walled box, built by the reference's own
  parse_config + build_initial_state): 1,000 steps on the B200 and on the reference; the
  kinetic-energy series agrees within 1e-9 relative at every step and the coordination series
  (pp contacts per particle) exactly — the tolerance DESIGN.md §1 states for multi-step runs
  (observed on the CPU restatement, which is bitwise the B200 path: KE within 2e-15, coordination
  identical; the chaotic divergence has not grown past round-off in 1,000 steps of settling).
"""
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ref_mod = pytest.importorskip("oracle.oracle")


@pytest.fixture(scope="module")
def ref():
    if not ref_mod.have_ref():
        pytest.skip("oracle/_ref/libdemforge_ref.so not built")
    r = ref_mod.RefLib()
    r.set_threads(os.cpu_count() or 1)
    return r


def _pairs(owner, partner, ids):
    """(owner id, partner id) for particle partners; walls as (owner id, -(w+1) as int)."""
    o = ids[owner.astype(np.int64)].astype(np.int64)
    p = partner.astype(np.int64)
    pid = np.where(p >= 0, ids[np.clip(p, 0, None)].astype(np.int64), p)
    return o, pid


def _check_step(sim, rsim, osim, label):
    import paper_1503_03553_b200 as dem  # noqa: F401
    a, r = sim.particles(), rsim.state()
    o = osim.state()
    fa, ta = sim.forces().force, sim.forces().torque
    fr, tr = rsim.forces()
    fs, ts = osim.force_scale()
    ia, ir, io = np.argsort(a.ids), np.argsort(r.ids), np.argsort(o.ids)
    assert np.array_equal(a.ids[ia], r.ids[ir]) and np.array_equal(a.ids[ia], o.ids[io])
    sf, st = fs[io][:, None], ts[io][:, None]
    df = np.abs(fa[ia] - fr[ir])
    dt_ = np.abs(ta[ia] - tr[ir])
    assert np.all(df <= 1e-9 * sf), f"{label}: force rel {np.max(df / np.maximum(sf, 1e-300)):.3e}"
    assert np.all(dt_ <= 1e-9 * np.maximum(st, 1e-300)), f"{label}: torque rel {np.max(dt_ / np.maximum(st, 1e-300)):.3e}"
    # contact pairs and tangential histories, keyed by stable ids
    co, cp, cd = sim.contacts()
    ro, rp, rt, rd = rsim.table()
    keep = rt  # touched entries: this phase's contacts (contact_table.cpp:15-35)
    ko, kp = _pairs(co, cp, a.ids)
    ro2, rp2 = _pairs(ro[keep], rp[keep], r.ids)
    kb = np.stack([ko, kp], 1)
    kr = np.stack([ro2, rp2], 1)
    ob, orr = np.lexsort((kb[:, 1], kb[:, 0])), np.lexsort((kr[:, 1], kr[:, 0]))
    assert len(kb) == len(kr) and np.array_equal(kb[ob], kr[orr]), f"{label}: contact sets differ"
    db, dr = cd[ob], rd[keep][orr]
    scale = np.linalg.norm(dr, axis=1)[:, None]
    assert np.all(np.abs(db - dr) <= 1e-9 * scale + 1e-300), f"{label}: delta_t differs"
    return len(kb)


@pytest.mark.parametrize("case", ["configs1_262144", "configs2_1M_poly_friction"])
def test_full_size_one_step_vs_reference(cuda, ref, case):
    dem = cuda
    from oracle.oracle import Oracle, OracleSim, RefSim
    if case == "configs1_262144":
        ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, poly=False, seed=1)
        cfg = dem.packing_config(dmax)
    else:
        ps, dmax = dem.gen_packing(1 << 20, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
        cfg = dem.packing_config(dmax, poly=True)
    sim = dem.Simulation(ps, cfg)
    rsim = RefSim(ref, ps, cfg)
    osim = OracleSim(Oracle(), ps, cfg)
    contacts = _check_step(sim, rsim, osim, "priming pass")
    capped = 0
    for k in range(2):
        m = sim.step()
        rsim.step()
        osim.step()
        capped += m.capped_contacts
        contacts = _check_step(sim, rsim, osim, f"step {k + 1}")
    assert contacts > 0
    if case != "configs1_262144":
        assert capped > 0  # the friction cap is engaged (divergence stress case)


def test_config0_1000_steps_statistics_vs_reference(cuda, ref):
    """configs[0]: 4,096 settling spheres, 5 walls, 1,000 steps."""
    dem = cuda
    from oracle.oracle import RefSim
    text = open(os.path.join(ROOT, "configs", "settle4096.cfg")).read()
    cfg_c, mats, rects, lines, st, nsteps = ref.parse_and_build(text)
    assert nsteps == 1000 and len(st.ids) == 4096
    cfg = dem.SimConfig()
    cfg.dt = cfg_c.dt
    cfg.gravity = tuple(cfg_c.gravity)
    cfg.domain_min = tuple(cfg_c.domain_min)
    cfg.domain_max = tuple(cfg_c.domain_max)
    for k, m in enumerate(mats):
        cfg.materials.add(f"m{k}", dem.MaterialParams(m.poisson_ratio, m.shear_modulus, m.youngs_modulus,
                                                      m.restitution, m.sliding_friction))
    cfg.rect_walls = [dem.RectWall(tuple(w.corner), tuple(w.edge_u), tuple(w.edge_v), w.material_id) for w in rects]
    cfg.line_walls = [dem.LineWall(tuple(w.a), tuple(w.b), w.material_id) for w in lines]
    cfg.contact_capacity = cfg_c.contact_capacity
    ps = dem.ParticleSet(len(st.ids))
    ps.ids[:], ps.positions[:], ps.velocities[:] = st.ids, st.positions, st.velocities
    ps.angular_velocities[:], ps.radii[:], ps.masses[:], ps.material_ids[:] = (
        st.angular_velocities, st.radii, st.masses, st.material_ids)
    sim = dem.Simulation(ps, cfg)
    rsim = RefSim(ref, ps, cfg)

    def ke(s):  # particle_set.cpp:71-79
        return float((0.5 * s.masses * (s.velocities ** 2).sum(1)).sum()
                     + (0.5 * (0.4 * s.masses * s.radii * s.radii) * (s.angular_velocities ** 2).sum(1)).sum())

    kb, kr, cb, cr = [], [], [], []
    for _ in range(nsteps):
        mb = sim.step()
        mr = rsim.step()
        kb.append(ke(sim.particles()))
        kr.append(ke(rsim.state()))
        cb.append(mb.pp_contact_events)
        cr.append(mr.pp_contact_events)
    kb, kr = np.array(kb), np.array(kr)
    rel = np.abs(kb - kr) / np.abs(kr)
    print(f"KE end {kb[-1]:.6e} (reference {kr[-1]:.6e}); max rel {rel.max():.2e}; "
          f"mean coordination {np.mean(cb) / 4096:.4f} (reference {np.mean(cr) / 4096:.4f})")
    assert np.all(rel <= 1e-9)
    assert cb == cr
    assert abs(kr[-1] - 0.17712) < 5e-5  # KE_end printed 1.7712e-01 J


@pytest.mark.parametrize("case", ["configs1_262144", "configs2_1M_poly_friction"])
def test_fp32_mode_priming_pass_vs_reference(cuda, ref, case):
    """north_star's fp32 bar against the LIVE reference (not only against the GPU's own fp64 path):
    the fp32 throughput mode's priming pass on identical inputs at BASELINE.json's full sizes.
    * Contact-pair sets are identical (detection stays the exact fp64 classification).
    * Forces within 1e-5 and torques within 1e-5 r of the particle's sum of contact-term
      magnitudes (Hertz k_n dn^1.5 + spring k_t |delta_t| + damping eta |v_rel|, the scale of
      tests/test_fp32_mode.py): an fp32 evaluation is accurate relative to the terms it sums, and
      in the configs[2] stress case (spins up to 50 rad/s) a separating contact's elastic and
      damping terms cancel to 1/400 of their size, so 1e-5 of the net |F| would ask fp32 for
      ~4e-8 relative accuracy per term. The error relative to sum |F_k| is printed alongside.
    * New tangential displacements (delta_t = v_t dt in the priming pass) within 1e-5 relative to
      |delta_t| + |v_rel| dt, |v_rel| <= |v_i - v_j| + |w_i| r_i + |w_j| r_j."""
    dem = cuda
    from oracle.oracle import Oracle, OracleSim, RefSim
    from test_fp32_mode import contact_scale
    if case == "configs1_262144":
        ps, dmax = dem.gen_packing(262144, s=1.8, jit=0.2, poly=False, seed=1)
        cfg = dem.packing_config(dmax)
    else:
        ps, dmax = dem.gen_packing(1 << 20, s=1.4, jit=0.2, poly=True, seed=3, omega_half=50.0)
        cfg = dem.packing_config(dmax, poly=True)
    rsim = RefSim(ref, ps, cfg)
    osim = OracleSim(Oracle(), ps, cfg)
    cfg.precision = 1
    sim = dem.Simulation(ps, cfg)
    a, r, o = sim.particles(), rsim.state(), osim.state()
    ia, ir, io = np.argsort(a.ids), np.argsort(r.ids), np.argsort(o.ids)
    assert np.array_equal(a.ids[ia], r.ids[ir]) and np.array_equal(a.ids[ia], o.ids[io])
    fa, ta = sim.forces().force[ia], sim.forces().torque[ia]
    fr, tr = (x[ir] for x in rsim.forces())
    co, cp, cd = sim.contacts()
    scale = contact_scale(a, co, cp, cd)[ia]
    has = scale > 0
    ef = np.linalg.norm(fa - fr, axis=1)
    et = np.linalg.norm(ta - tr, axis=1)
    rad = a.radii[ia]
    fs = np.maximum(osim.force_scale()[0][io], 1e-300)
    print(f"{case}: fp32 vs reference: force {np.max(ef[has] / scale[has]):.2e}, torque "
          f"{np.max(et[has] / (scale[has] * rad[has])):.2e} of the contact-term sums; force "
          f"{np.max(np.abs(fa - fr).max(1) / fs):.2e} of sum |F_k|")
    assert np.all(ef[~has] == 0.0) and np.all(et[~has] == 0.0)
    assert np.all(ef[has] <= 1e-5 * scale[has]) and np.all(et[has] <= 1e-5 * scale[has] * rad[has])
    ro, rp, rt, rd = rsim.table()
    ko, kp = _pairs(co, cp, a.ids)
    ro2, rp2 = _pairs(ro[rt], rp[rt], r.ids)
    kb, kr = np.stack([ko, kp], 1), np.stack([ro2, rp2], 1)
    ob, orr = np.lexsort((kb[:, 1], kb[:, 0])), np.lexsort((kr[:, 1], kr[:, 0]))
    assert len(kb) == len(kr) and np.array_equal(kb[ob], kr[orr]), "contact sets differ"
    # |v_rel| bound per contact, from the reference state by stable id (walls: partner terms 0)
    pos_of = np.empty(int(r.ids.max()) + 1, dtype=np.int64)
    pos_of[r.ids] = np.arange(len(r.ids))
    oi = pos_of[kb[ob][:, 0]]
    pj = kb[ob][:, 1]
    wall = pj < 0
    ji = pos_of[np.where(wall, r.ids[0], pj)]
    v, w, rr = r.velocities, r.angular_velocities, r.radii
    vrel = (np.linalg.norm(v[oi] - np.where(wall[:, None], 0.0, v[ji]), axis=1)
            + np.linalg.norm(w[oi], axis=1) * rr[oi]
            + np.where(wall, 0.0, np.linalg.norm(w[ji], axis=1) * rr[ji]))
    db, dr = cd[ob], rd[rt][orr]
    sd = np.linalg.norm(dr, axis=1) + vrel * cfg.dt
    ed = np.max(np.linalg.norm(db - dr, axis=1) / np.maximum(sd, 1e-300))
    print(f"{case}: fp32 vs reference: delta_t {ed:.2e}")
    assert ed <= 1e-5
