// sharded.hpp — the multi-GPU counterpart of demb200::Simulation (simulation.hpp): one rank of
// the host-free z-slab decomposition over the C ABI's dem_create_sharded / dem_shard_* entry
// points (dem_b200.h; SURVEY §8b "dem_create_sharded", §8e). A C++ caller gets multi-GPU stepping
// with no Python and no host round trip inside a step.
//
//   // one process (or host thread) per GPU; every rank passes the same global initial set
//   demb200::ShardedSimulation sim(all, cfg, device, rank, nranks,
//       [&](const void* mine, void* all, std::size_t bytes) {   // any all-gather:
//           ncclAllGather(d_mine, d_all, bytes, ncclUint8, comm, stream); ... // or MPI_Allgather
//       });
//   for (...) sim.step();
//   const demb200::ParticleSet& mine = sim.owned_particles();   // this slab's particles
//
// Ranks of ONE process are wired with ShardedSimulation::connect_local and stepped with
// launch() on every rank, then wait() on every rank (step() would block on its neighbours).
#pragma once

#include <functional>

#include "simulation.hpp"

namespace demb200 {

class ShardedSimulation {
  public:
    using AllGather = std::function<void(const void* mine, void* all, std::size_t bytes_per_rank)>;

    /// dem_create_sharded + dem_shard_handle + allgather + dem_shard_connect.
    ShardedSimulation(const ParticleSet& all, SimConfig config, int device, int rank, int nranks,
                      const AllGather& allgather)
        : ShardedSimulation(all, std::move(config), device, rank, nranks) {
        unsigned char mine[64];
        check(dem_shard_handle(ctx_.get(), mine));
        std::vector<unsigned char> handles(64 * static_cast<std::size_t>(nranks));
        allgather(mine, handles.data(), 64);
        check(dem_shard_connect(ctx_.get(), handles.data()));
    }

    /// Unconnected rank (connect_local wires ranks of one process).
    ShardedSimulation(const ParticleSet& all, SimConfig config, int device, int rank, int nranks) : cfg_(std::move(config)) {
        build_config();
        dem_particles p = view(all);
        dem_ctx* c = nullptr;
        const int rc = dem_create_sharded(&cc_.c, &p, device, rank, nranks, &c);
        if (rc != DEM_OK) rethrow(nullptr, rc);
        ctx_.reset(c);
    }

    ShardedSimulation(const ShardedSimulation&) = delete;
    ShardedSimulation& operator=(const ShardedSimulation&) = delete;
    ShardedSimulation(ShardedSimulation&&) = default;

    /// dem_shard_connect_local: lo / hi are the z-neighbours (nullptr at a non-periodic edge).
    void connect_local(ShardedSimulation* lo, ShardedSimulation* hi) {
        check(dem_shard_connect_local(ctx_.get(), lo ? lo->ctx_.get() : nullptr, hi ? hi->ctx_.get() : nullptr));
    }

    /// pipeline.hpp:68 for this rank (every rank steps together; the first call primes, :83).
    StepMetrics step(int n = 1) {
        dem_step_metrics m{};
        check(dem_step(ctx_.get(), n, &m));
        return convert(m);
    }
    void launch(int n = 1) { check(dem_shard_launch(ctx_.get(), n)); }
    StepMetrics wait() {
        dem_step_metrics m{};
        check(dem_shard_wait(ctx_.get(), &m));
        return convert(m);
    }

    int z_lo() const { return info().z_lo; }
    int z_hi() const { return info().z_hi; }
    std::uint64_t owned_count() const { return info().owned; }

    /// This slab's owned particles (halo copies dropped), in the slab's canonical slot order, and
    /// their forces.
    ParticleSet owned_particles() const {
        ParticleSet all;
        ForceAccumulator f;
        fetch(all, f);
        return select(all, f).first;
    }
    ForceAccumulator owned_forces() const {
        ParticleSet all;
        ForceAccumulator f;
        fetch(all, f);
        return select(all, f).second;
    }
    const SimConfig& config() const { return cfg_; }

  private:
    struct CtxDeleter { void operator()(dem_ctx* c) const { dem_destroy(c); } };
    struct Info { int z_lo, z_hi; std::uint64_t owned; };
    SimConfig cfg_;
    detail::CConfig cc_;
    std::unique_ptr<dem_ctx, CtxDeleter> ctx_;

    Info info() const {
        std::int32_t lo = 0, hi = 0;
        std::uint64_t n = 0;
        check(dem_shard_info(ctx_.get(), &lo, &hi, &n));
        return Info{lo, hi, n};
    }
    void check(int rc) const { if (rc != DEM_OK) rethrow(ctx_.get(), rc); }
    [[noreturn]] static void rethrow(const dem_ctx* c, int rc) { detail::rethrow(c, rc); }
    static StepMetrics convert(const dem_step_metrics& m) {
        StepMetrics r;
        r.step = m.step;
        r.contacts = m.contacts;
        r.pp_contact_events = m.pp_contact_events;
        r.max_contacts_per_particle = m.max_contacts_per_particle;
        r.clamps = m.clamps;
        r.friction_max_ratio = m.friction_max_ratio;
        r.capped_contacts = m.capped_contacts;
        return r;
    }
    static dem_particles view(const ParticleSet& s) { return detail::view(const_cast<ParticleSet&>(s)); }
    void build_config() { cc_.build(cfg_); }
    void fetch(ParticleSet& all, ForceAccumulator& f) const {
        const std::size_t n = dem_size(ctx_.get());
        all.ids.resize(n); all.positions.resize(n); all.velocities.resize(n); all.angular_velocities.resize(n);
        all.radii.resize(n); all.masses.resize(n); all.material_ids.resize(n);
        f.force.resize(n);
        f.torque.resize(n);
        if (!n) return;
        dem_particles p = view(all);
        check(dem_get_particles(ctx_.get(), &p));
        check(dem_get_forces(ctx_.get(), &f.force.data()->x, &f.torque.data()->x));
    }
    static std::pair<ParticleSet, ForceAccumulator> select(const ParticleSet& all, const ForceAccumulator& f) {
        ParticleSet o;
        ForceAccumulator of;
        for (std::size_t i = 0; i < all.size(); ++i) {
            if (all.material_ids[i] & 0x80000000u) continue;  // halo copy of a neighbour's particle
            o.push_back(all.ids[i], all.positions[i], all.velocities[i], all.angular_velocities[i], all.radii[i],
                        all.masses[i], all.material_ids[i]);
            of.force.push_back(f.force[i]);
            of.torque.push_back(f.torque[i]);
        }
        return {std::move(o), std::move(of)};
    }
};

}  // namespace demb200
