"""Traversal traces and the warp model: Simulation::traces()
(pipeline.hpp:97, recorded in kernel_collide, pipeline.cpp:191-231) downloaded from the device
(dem_get_traces), against the reference's own traces on the same input, and the reference's warp
model (warp_model.cpp) evaluated over both."""
import numpy as np
import pytest

from helpers import basic_config, box_for, random_dense_state, settling_state, walled_config

pytestmark = pytest.mark.gpu


def canon(off, cand, hit, ids, keys):
    """{owner id: sorted [(candidate cell key, candidate id, contact)]}; also checks that each
    lane visits cells in nondecreasing key order (z, y, x outer-to-inner, grid.cpp:60-82)."""
    out = {}
    for i in range(len(off) - 1):
        a, b = int(off[i]), int(off[i + 1])
        c = cand[a:b]
        k = keys[c]
        assert np.all(np.diff(k.astype(np.int64)) >= 0), i
        assert np.all(c != i)
        out[int(ids[i])] = sorted(zip(k.tolist(), ids[c].tolist(), hit[a:b].tolist()))
    return out


def ref_traces_after_step(ref, st, cfg):
    from oracle.oracle import RefSim
    rs = RefSim(ref, st, cfg)
    ref.L.ref_sim_set_record_traces(rs.h, 1)
    rs.step()
    return rs


@pytest.mark.parametrize("n,seed", [(1000, 3), (1331, 5)])
def test_traces_match_reference(cuda, ref, n, seed):
    dem = cuda
    cfg = basic_config(box_for(n))
    st = random_dense_state(n, seed)
    sim = dem.Simulation(st, cfg)
    m = sim.step()
    rs = ref_traces_after_step(ref, st, cfg)
    off, cand, hit = sim.traces()
    ps = sim.particles()
    keys, _ = sim.order()
    got = canon(off, cand, hit, ps.ids, keys)
    roff, rcand, rhit = rs.traces()
    rps = rs.state()
    g = sim.grid()  # same config -> same grid
    # reference keys from its own positions through calc_hash semantics (same grid)
    rel = (rps.positions - np.array(g.origin)) * (1.0 / g.cell_size)
    c = np.floor(rel).astype(np.int64)
    c = np.clip(c, 0, np.array([g.nx - 1, g.ny - 1, g.nz - 1]))
    rkeys = (c[:, 0] + g.nx * (c[:, 1] + g.ny * c[:, 2])).astype(np.uint32)
    want = canon(roff, rcand, rhit, rps.ids, rkeys)
    assert got == want
    assert hit.sum() == m.pp_contact_events > 0
    # the reference warp model over both trace sets: identical warp count, close values (lanes
    # move between warps when the in-cell order differs)
    a = ref.model_report(off, hit)
    b = ref.model_report(roff, rhit)
    assert a["warp_count"] == b["warp_count"]
    for k in ("cycles_baseline", "cycles_two_phase", "utilization_baseline", "utilization_two_phase"):
        assert abs(a[k] - b[k]) <= 0.05 * abs(b[k]), (k, a[k], b[k])
    assert a["utilization_baseline"] < a["utilization_two_phase"]


def test_traces_contact_events_are_the_pair_set(cuda, orc):
    """Contact events of the traces == brute-force pairs (the verify completeness check,
    runner.cpp:298-311), including the first step of a walled settling run."""
    dem = cuda
    cfg = walled_config(8)
    sim = dem.Simulation(settling_state(512, 4), cfg)
    for _ in range(3):
        sim.step()
    off, cand, hit = sim.traces()
    ps = sim.particles()
    pairs = set()
    for i in range(len(off) - 1):
        for j, h in zip(cand[off[i]:off[i + 1]], hit[off[i]:off[i + 1]]):
            if h:
                pairs.add((min(i, int(j)), max(i, int(j))))
    ii, jj = orc.contact_pairs(ps.positions, ps.radii, binned=False)
    assert pairs == set(zip(ii.tolist(), jj.tolist()))


def test_traces_identical_for_both_variants_and_invalidated_by_set_particles(cuda):
    dem = cuda
    cfg = basic_config(box_for(1000))
    a = dem.Simulation(random_dense_state(1000, 9), cfg)
    b = a.clone()
    b.set_collide_variant(dem.BASELINE)
    a.step()
    b.step()
    ta, tb = a.traces(), b.traces()
    for x, y in zip(ta, tb):
        assert np.array_equal(x, y)
    # a clone carries the binning: its traces are the source's
    c = a.clone()
    for x, y in zip(c.traces(), ta):
        assert np.array_equal(x, y)
    a.set_particles(a.particles())
    with pytest.raises(Exception):
        a.traces()
    a.step()
    assert a.traces()[0][-1] > 0  # valid again after a force phase
