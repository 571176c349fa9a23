"""GPU parity at BASELINE.json's large sizes through size-independent properties (the CPU oracle
and the reference cannot step 8M-33M particles in a test; configs[1] and configs[2] are compared
with the live reference in test_gpu_reference_full.py).

Every operation of a pair evaluation is round-to-nearest symmetric (x - y = -(y - x), products and
sums of negated operands negate exactly, sums commute), and the classification depends on d^2 and
r_i + r_j only, so in a box without shear:
* the contact-pair set is symmetric: (i, j) is a contact of i exactly when (j, i) is one of j;
* the tangential displacements of the two sides are exact negatives, bit for bit (both start at 0
  when the contact forms and are updated, and capped, by negated operations);
* with no walls and no gravity the per-particle forces sum to zero up to the rounding of the
  per-particle sums (|sum F| <= 1e-12 sum |F|; a dropped or doubled contact gives ~1e-2).
configs[4]'s north-star pack (33,554,432 dense frictional spheres) and an 8M dense pack are
checked after the priming pass and two steps, in fp64 and in the fp32 mode; configs[3]'s 8M
Lees-Edwards box for the symmetric contact-pair set."""
import numpy as np
import pytest

from helpers import bits

import paper_1503_03553_b200 as dem

pytestmark = pytest.mark.gpu


def _symmetric_pairs(sim, histories=True):
    ps = sim.particles()
    o, p, d = sim.contacts()
    pp = p >= 0
    a = ps.ids[o[pp]].astype(np.uint64)
    b = ps.ids[p[pp].astype(np.int64)].astype(np.uint64)
    dt = d[pp]
    fwd = (a << np.uint64(32)) | b
    rev = (b << np.uint64(32)) | a
    of, orv = np.argsort(fwd, kind="stable"), np.argsort(rev, kind="stable")
    assert np.array_equal(fwd[of], rev[orv]), "contact-pair set not symmetric"
    if histories:
        assert np.array_equal(bits(dt[of]), bits(-dt[orv])), "tangential displacements not antisymmetric"
    return len(fwd)


def _momentum(sim):
    f = sim.forces().force
    return float(np.max(np.abs(f.sum(axis=0))) / np.abs(f).sum())


@pytest.mark.parametrize("precision", [0, 1])
def test_8m_dense_pair_symmetry_and_momentum(cuda, precision):
    ps, dmax = dem.gen_packing(1 << 23, s=1.8, jit=0.2, seed=4)
    cfg = dem.packing_config(dmax)
    cfg.precision = precision
    sim = dem.Simulation(ps, cfg)
    del ps
    for k in range(3):  # the priming pass, then two steps (histories carried, friction cap engaged)
        if k:
            m = sim.step()
            assert m.capped_contacts > 0
        assert _symmetric_pairs(sim) > 0
        assert _momentum(sim) <= 1e-12


def test_32m_north_star_momentum_and_counts(cuda):
    """configs[4] at s = 1.8 (north_star: 32M dense frictional): momentum balance after two steps,
    and the contact count is even (each pair appears once per side)."""
    ps, dmax = dem.gen_packing(1 << 25, s=1.8, jit=0.2, seed=5)
    sim = dem.Simulation(ps, dem.packing_config(dmax))
    del ps
    for _ in range(2):
        m = sim.step()
    assert m.contacts > 0 and m.contacts % 2 == 0 and m.contacts == m.pp_contact_events
    assert _momentum(sim) <= 1e-12


def test_8m_periodic_lees_edwards_pair_symmetry(cuda):
    """configs[3] (8,388,608 spheres, periodic box, Lees-Edwards shear) after two steps: the
    minimum image of (j, i) is the negated one of (i, j) bit for bit (the shear offset enters as
    -(d - delta) = -d + delta), so the contact-pair set is symmetric. (The two sides' tangential
    histories are not exact negatives here: the partner image's velocity offset is added on each
    side's own velocity.)"""
    ps, L = dem.gen_periodic_packing(1 << 23, s=1.8, jit=0.2, seed=4)
    sim = dem.Simulation(ps, dem.periodic_config(L, shear_rate=1.0))
    del ps
    sim.steps(2)
    assert _symmetric_pairs(sim, histories=False) > 0
