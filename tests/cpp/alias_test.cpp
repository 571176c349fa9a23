// alias_test.cpp — the drop-in switch itself: a program written against the reference API
// (demforge::Simulation and its value types, /root/reference/proj/core/include/demforge/
// pipeline.hpp:50-136) compiled with `namespace demforge = demb200;` instead of the reference
// headers. Every public member and free function of pipeline.hpp:50-107 is called, so a missing
// or differently-typed entry point is a compile error; the run checks the results are coherent.
// Built by tests/cpp/Makefile (needs only this repo's headers); run on the GPU box by
// tests/test_cpp_drop_in.py.
#include <cmath>
#include <cstdio>
#include <string>
#include <type_traits>

#include "demb200/simulation.hpp"

namespace demforge = demb200;

static int failures = 0;
#define EXPECT(c)                                                                               \
    do {                                                                                        \
        if (!(c)) { std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); ++failures; }     \
    } while (0)

static demforge::SimConfig make_config(double box) {
    demforge::SimConfig cfg;
    cfg.dt = 1e-5;
    cfg.gravity = {0.0, 0.0, -9.81};
    cfg.domain_min = {0.0, 0.0, 0.0};
    cfg.domain_max = {box, box, box};
    demforge::MaterialParams m;
    m.shear_modulus = 3.85e5;
    cfg.materials.add("bead", m);
    cfg.contact_capacity = 16;
    return cfg;
}

int main() {
    const double r0 = 0.005, sp = 1.8 * r0;
    const int side = 8;
    demforge::ParticleSet ps;
    for (int i = 0; i < side * side * side; ++i) {
        const double x = 2 * r0 + (i % side) * sp, y = 2 * r0 + (i / side % side) * sp, z = 2 * r0 + (i / side / side) * sp;
        ps.push_back(static_cast<std::uint32_t>(1000 + i), {x, y, z}, {0.1 * std::sin(i), 0.1 * std::cos(i), 0.0},
                     {0.0, 0.0, 1.0}, r0, 1e-3, 0);
    }
    const demforge::SimConfig cfg = make_config(4 * r0 + side * sp);
    demforge::Simulation sim(ps, cfg);

    // accessors with the reference's exact return types (pipeline.hpp:88-107)
    static_assert(std::is_same_v<decltype(sim.grid()), const demforge::UniformGrid&>);
    static_assert(std::is_same_v<decltype(std::as_const(sim).particles()), const demforge::ParticleSet&>);
    static_assert(std::is_same_v<decltype(sim.particles()), demforge::ParticleSet&>);
    static_assert(std::is_same_v<decltype(std::as_const(sim).forces()), const demforge::ForceAccumulator&>);
    static_assert(std::is_same_v<decltype(sim.contact_table()), demforge::ContactTable&>);
    static_assert(std::is_same_v<decltype(sim.order()), const demforge::SortedOrder&>);
    static_assert(std::is_same_v<decltype(sim.config()), const demforge::SimConfig&>);
    static_assert(std::is_same_v<decltype(sim.step()), demforge::StepMetrics>);
    static_assert(std::is_same_v<decltype(sim.neighborhood_sufficient()), bool>);

    const demforge::UniformGrid& g = sim.grid();
    EXPECT(g.cell_size >= 2 * r0 && g.nx >= side);
    EXPECT(sim.neighborhood_sufficient());
    EXPECT(sim.step_index() == 0);

    sim.set_record_traces(true);
    sim.set_collide_variant(demforge::CollideVariant::two_phase);
    const demforge::StepMetrics m = sim.step();
    EXPECT(m.step == 1 && sim.step_index() == 1);
    EXPECT(m.contacts > 0 && m.pp_contact_events == m.contacts);
    EXPECT(sim.traces().size() == ps.size());
    EXPECT(sim.last_clamp_count() == 0);
    EXPECT(std::abs(sim.mean_coordination() - double(m.pp_contact_events) / double(ps.size())) == 0.0);
    EXPECT(sim.order().sorted_keys.size() == ps.size());
    EXPECT(sim.contact_table().particle_count() == ps.size() && sim.contact_table().max_live_count() > 0);

    // the per-kernel methods compose one step (pipeline.hpp:77-86), like Simulation::step()
    demforge::Simulation a(sim), b(sim);
    a.step();
    b.kernel_integrate();
    b.kernel_calc_hash();
    b.kernel_bitonic_sort();
    b.kernel_find_cell_bounds_and_reorder();
    b.zero_forces();
    b.kernel_force_gravity();
    b.kernel_initialize_contact_ids();
    b.kernel_collide(demforge::CollideVariant::two_phase, false);
    b.kernel_collide_rectangle();
    b.kernel_collide_line();
    EXPECT(a.particles() == b.particles());
    EXPECT(a.forces() == b.forces());

    // the free functions (pipeline.hpp:50-56) on the host copies: integrating the device state
    // with the device forces is what the next step's Integrate does
    demforge::ParticleSet host = sim.particles();
    demforge::ForceAccumulator f = sim.forces();
    demforge::integrate(host, f, cfg.dt);
    demforge::Simulation c(sim);
    c.kernel_integrate();
    c.kernel_find_cell_bounds_and_reorder();
    {
        // c's state after Integrate + reorder is `host` permuted into c's slot order
        const auto& cs = c.particles();
        std::size_t matched = 0;
        for (std::size_t i = 0; i < cs.size(); ++i)
            for (std::size_t j = 0; j < host.size(); ++j)
                if (host.ids[j] == cs.ids[i]) { matched += host.positions[j] == cs.positions[i] && host.velocities[j] == cs.velocities[i]; break; }
        EXPECT(matched == host.size());
    }
    demforge::ForceAccumulator zero;
    zero.force.assign(host.size(), demforge::Vec3{});
    zero.torque.assign(host.size(), demforge::Vec3{});
    demforge::force_gravity(host, zero, cfg.gravity);
    EXPECT(zero.force[0].z == -9.81 * host.masses[0] && zero.torque[0].z == 0.0);

    // error types (error.hpp:10-49): a non-finite force is the reference's KernelError("Integrate")
    zero.force[3].x = NAN;
    bool threw = false;
    try { demforge::integrate(host, zero, cfg.dt); } catch (const demforge::KernelError& e) { threw = e.kernel() == "Integrate"; }
    EXPECT(threw);
    threw = false;
    try {
        demforge::SimConfig bad = cfg;
        bad.dt = -1.0;
        demforge::Simulation s2(ps, bad);
    } catch (const demforge::ConfigError&) { threw = true; }
    EXPECT(threw);

    std::printf("%s\n", failures ? "FAILED" : "PASSED");
    return failures ? 1 : 0;
}
