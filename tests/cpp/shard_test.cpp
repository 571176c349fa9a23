// shard_test.cpp — the C++ multi-GPU entry point with no Python in the loop: demb200::
// ShardedSimulation (include/demb200/sharded.hpp over dem_create_sharded / dem_shard_*) for 1-4
// ranks of one process on one device, stepped with launch/wait, against demb200::Simulation:
// positions, velocities, forces and torques of every particle by stable id, bitwise. Walled box
// with plane crossings, and a periodic Lees-Edwards ring. Built by tests/cpp/Makefile; run by
// tests/test_cpp_drop_in.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "demb200/host.hpp"
#include "demb200/sharded.hpp"

namespace b2 = demb200;

static int failures = 0;
#define EXPECT(c)                                                                              \
    do {                                                                                       \
        if (!(c)) { std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); ++failures; }    \
    } while (0)

static bool same(const b2::Vec3& a, const b2::Vec3& b) { return std::memcmp(&a, &b, sizeof a) == 0; }

static b2::ParticleSet lattice(int side, double s, std::uint64_t seed, double kick, double* box) {
    b2::ParticleSet ps;
    b2::XorShift64Star rng(seed);
    const double r0 = 0.005;
    for (int i = 0; i < side * side * side; ++i) {
        const double x = 2 * r0 + (i % side) * s * r0 + rng.next_in(-0.2 * r0, 0.2 * r0);
        const double y = 2 * r0 + (i / side % side) * s * r0 + rng.next_in(-0.2 * r0, 0.2 * r0);
        const double z = 2 * r0 + (i / side / side) * s * r0 + rng.next_in(-0.2 * r0, 0.2 * r0);
        const double vz = rng.next_in(-0.5, 0.5) + (i % 2 ? kick : -kick);
        ps.push_back(static_cast<std::uint32_t>(i), {x, y, z}, {rng.next_in(-0.5, 0.5), rng.next_in(-0.5, 0.5), vz},
                     {rng.next_in(-0.5, 0.5), rng.next_in(-0.5, 0.5), rng.next_in(-0.5, 0.5)}, r0, 1e-3, 0);
    }
    *box = side * s * r0 + 4 * r0;
    return ps;
}

static void run_case(bool periodic, int nranks, int steps) {
    double box = 0.0;
    const b2::ParticleSet ps = lattice(24, 1.8, 7 + nranks, 30.0, &box);
    b2::SimConfig cfg;
    cfg.dt = 1e-5;
    cfg.gravity = {0.0, 0.0, 0.0};
    cfg.domain_min = {0.0, 0.0, 0.0};
    cfg.domain_max = {box, box, box};
    cfg.materials.add("bead", b2::MaterialParams{});
    if (periodic) {
        cfg.periodic = 7;
        cfg.shear_rate = 30.0;
    }
    b2::Simulation one(ps, cfg);
    for (int k = 0; k < steps; ++k) one.step();
    std::vector<std::unique_ptr<b2::ShardedSimulation>> shards;
    for (int r = 0; r < nranks; ++r) shards.push_back(std::make_unique<b2::ShardedSimulation>(ps, cfg, 0, r, nranks));
    for (int r = 0; r < nranks; ++r) {
        b2::ShardedSimulation* lo = (periodic || r > 0) ? shards[(r - 1 + nranks) % nranks].get() : nullptr;
        b2::ShardedSimulation* hi = (periodic || r < nranks - 1) ? shards[(r + 1) % nranks].get() : nullptr;
        shards[r]->connect_local(lo, hi);
    }
    std::printf("  created %d ranks\n", nranks);
    for (auto& sh : shards) sh->launch(steps);
    std::printf("  launched\n");
    std::int64_t contacts = 0;
    for (auto& sh : shards) contacts += sh->wait().contacts;
    std::map<std::uint32_t, std::size_t> at;
    const b2::ParticleSet& s1 = one.particles();
    const b2::ForceAccumulator& f1 = one.forces();
    for (std::size_t i = 0; i < s1.size(); ++i) at[s1.ids[i]] = i;
    std::size_t seen = 0, equal = 0;
    for (auto& sh : shards) {
        const b2::ParticleSet p = sh->owned_particles();
        const b2::ForceAccumulator f = sh->owned_forces();
        for (std::size_t k = 0; k < p.size(); ++k) {
            const std::size_t i = at.at(p.ids[k]);
            ++seen;
            equal += same(p.positions[k], s1.positions[i]) && same(p.velocities[k], s1.velocities[i]) &&
                     same(f.force[k], f1.force[i]) && same(f.torque[k], f1.torque[i]);
        }
    }
    std::printf("  %s, %d ranks, %d steps: %zu particles, %zu bitwise equal, %lld contacts\n",
                periodic ? "periodic Lees-Edwards" : "walled", nranks, steps, seen, equal, static_cast<long long>(contacts));
    EXPECT(seen == ps.size() && equal == seen && contacts > 0);
}

int main() {
    try {
        for (int r : {1, 2, 3, 4}) run_case(false, r, 12);
        for (int r : {1, 2, 3}) run_case(true, r, 12);
    } catch (const std::exception& e) {
        std::printf("FAIL: exception %s\n", e.what());
        ++failures;
    }
    std::printf("%s\n", failures ? "FAILED" : "PASSED");
    return failures ? 1 : 0;
}
