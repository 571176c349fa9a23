// host_test.cpp — CPU check of the host side against the reference
// itself: config parsing (config_io.cpp), initial states (lattice.cpp), snapshot formatting
// (snapshot_io.cpp). Runs without a GPU. Built by tests/cpp/Makefile.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <random>
#include <sstream>

#include "demb200/host.hpp"
#include "demb200/simulation.hpp"
#include "demforge/config_io.hpp"
#include "demforge/pipeline.hpp"
#include "demforge/error.hpp"
#include "demforge/lattice.hpp"
#include "demforge/snapshot_io.hpp"
#include "demforge/warp_model.hpp"

static int failures = 0;
#define EXPECT(c) do { if (!(c)) { std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); ++failures; } } while (0)

static std::string slurp(const std::string& p) {
    std::ifstream f(p, std::ios::binary);
    std::stringstream s;
    s << f.rdbuf();
    return s.str();
}

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }
template <class A, class B> static bool same3(const A& a, const B& b) { return same(a.x, b.x) && same(a.y, b.y) && same(a.z, b.z); }

static void compare_config(const std::string& text, const char* label) {
    const auto r = demforge::parse_config_text(text, "cfg");
    const auto b = demb200::parse_config_text(text, "cfg");
    EXPECT(same(r.dt, b.dt) && same3(r.gravity, b.gravity) && same3(r.domain_min, b.domain_min) && same3(r.domain_max, b.domain_max));
    EXPECT(r.materials.size() == b.materials.size());
    for (std::uint32_t k = 0; k < r.materials.size(); ++k) {
        const auto& x = r.materials.params(k);
        const auto& y = b.materials.params(k);
        EXPECT(same(x.poisson_ratio, y.poisson_ratio) && same(x.shear_modulus, y.shear_modulus) &&
               same(x.youngs_modulus, y.youngs_modulus) && same(x.restitution, y.restitution) &&
               same(x.sliding_friction, y.sliding_friction));
        for (std::uint32_t j = 0; j < r.materials.size(); ++j) EXPECT(same(r.materials.pair_restitution(k, j), b.materials.pair_restitution(k, j)));
    }
    EXPECT(r.rect_walls.size() == b.rect_walls.size() && r.line_walls.size() == b.line_walls.size());
    for (std::size_t k = 0; k < r.rect_walls.size(); ++k)
        EXPECT(same3(r.rect_walls[k].corner, b.rect_walls[k].corner) && same3(r.rect_walls[k].edge_u, b.rect_walls[k].edge_u) &&
               same3(r.rect_walls[k].edge_v, b.rect_walls[k].edge_v) && r.rect_walls[k].material_id == b.rect_walls[k].material_id);
    EXPECT(r.contact_capacity == b.contact_capacity && r.seed == b.seed && same(r.grid_cell_size, b.grid_cell_size));
    EXPECT(r.run.steps == b.run.steps && r.run.warmup_steps == b.run.warmup_steps && r.run.snapshot_every == b.run.snapshot_every);
    EXPECT((r.run.collide_variant == demforge::CollideVariant::baseline) == (b.run.collide_variant == demb200::CollideVariant::baseline));
    const auto rs = demforge::build_initial_state(r);
    const auto bs = demb200::build_initial_state(b);
    EXPECT(rs.size() == bs.size());
    bool ok = rs.size() == bs.size();
    for (std::size_t i = 0; ok && i < rs.size(); ++i)
        ok = rs.ids[i] == bs.ids[i] && same3(rs.positions[i], bs.positions[i]) && same3(rs.velocities[i], bs.velocities[i]) &&
             same(rs.radii[i], bs.radii[i]) && same(rs.masses[i], bs.masses[i]) && rs.material_ids[i] == bs.material_ids[i];
    EXPECT(ok);
    // snapshot bytes
    const auto dir = std::filesystem::temp_directory_path() / "dem_b200_host_test";
    std::filesystem::create_directories(dir);
    demforge::write_snapshot(dir / "r.csv", rs);
    demb200::write_snapshot(dir / "b.csv", bs);
    EXPECT(slurp((dir / "r.csv").string()) == slurp((dir / "b.csv").string()));
    std::printf("  %s: %zu particles, %zu walls, identical\n", label, bs.size(), b.rect_walls.size() + b.line_walls.size());
}

static void expect_same_error(const std::string& text) {
    std::string rm, bm;
    try { demforge::parse_config_text(text, "cfg"); } catch (const demforge::ConfigError& e) { rm = e.what(); }
    try { demb200::parse_config_text(text, "cfg"); } catch (const demb200::ConfigError& e) { bm = e.what(); }
    if (rm != bm) std::printf("  error mismatch:\n    ref:  %s\n    b200: %s\n", rm.c_str(), bm.c_str());
    EXPECT(!rm.empty() && rm == bm);
}

int main(int argc, char** argv) {
    const std::string root = argc > 1 ? argv[1] : ".";
    for (const char* c : {"configs/headon.cfg", "configs/settle512.cfg", "configs/settle4096.cfg"})
        compare_config(slurp(root + "/" + c), c);
    const std::string head = slurp(root + "/configs/headon.cfg");
    expect_same_error(head + "\nbogus.key = 1\n");
    expect_same_error(head + "\ndt = 2e-5\n");
    expect_same_error(head + "\nwall.rect.1.corner = 0 0 0\n");
    expect_same_error(head + "\nwall.box.0.corner = 0 0 0\n");
    expect_same_error(head + "\nrestitution_pair.bead.nope = 0.5\n");
    expect_same_error(head + "\nrun.collide_variant2 = x\n");
    expect_same_error("dt = 1e-5\n");
    expect_same_error(head + "\nparticles.jitter = abc\n");
    expect_same_error("dt 1e-5\n");
    // the format_double shortest round trip on random doubles
    std::mt19937_64 rng(3);
    std::uniform_real_distribution<double> u(-1e3, 1e3);
    bool fd = true;
    for (int k = 0; k < 100000; ++k) {
        const double v = u(rng) * std::pow(10.0, static_cast<int>(rng() % 40) - 20);
        fd = fd && demforge::format_double(v) == demb200::format_double(v);
    }
    EXPECT(fd);
    // the warp model (warp_model.cpp) on random traces: every field bitwise, several warp sizes
    // and non-integer costs (so the summation order matters)
    for (int trial = 0; trial < 40; ++trial) {
        const std::size_t lanes = 1 + rng() % 300;
        std::vector<demforge::LaneTrace> rt(lanes);
        std::vector<demb200::LaneTrace> bt(lanes);
        const double dens = 0.02 + 0.5 * (rng() % 1000) / 1000.0;
        for (std::size_t i = 0; i < lanes; ++i) {
            const int len = static_cast<int>(rng() % 90);
            for (int k = 0; k < len; ++k) {
                const bool hit = (rng() % 1000) < dens * 1000;
                rt[i].push_back({k, hit});
                bt[i].push_back({k, hit});
            }
        }
        demforge::WarpCostParams rp;
        demb200::WarpCostParams bp;
        const int ws[] = {32, 7, 1, 64};
        rp.warp_size = bp.warp_size = ws[trial % 4];
        if (trial % 2) {
            rp.c_check = bp.c_check = 0.37; rp.c_force = bp.c_force = 19.3;
            rp.c_store = bp.c_store = 1.1; rp.c_load = bp.c_load = 0.7;
        }
        const auto r = demforge::model_report(rt, rp);
        const auto b = demb200::model_report(bt, bp);
        EXPECT(same(r.cycles_baseline, b.cycles_baseline) && same(r.cycles_two_phase, b.cycles_two_phase));
        EXPECT(same(r.utilization_baseline, b.utilization_baseline) && same(r.utilization_two_phase, b.utilization_two_phase));
        EXPECT(same(r.useful_baseline, b.useful_baseline) && same(r.occupied_two_phase, b.occupied_two_phase));
        EXPECT(r.warp_count == b.warp_count && same(r.speedup(), b.speedup()));
        const auto rw = demforge::group_warps(rt, rp.warp_size);
        const auto bw = demb200::group_warps(bt, bp.warp_size);
        EXPECT(rw.size() == bw.size());
        for (std::size_t w = 0; w < rw.size() && w < bw.size(); ++w)
            for (auto [rv, bv] : {std::pair{demforge::CollideVariant::baseline, demb200::CollideVariant::baseline},
                                  std::pair{demforge::CollideVariant::two_phase, demb200::CollideVariant::two_phase}})
                EXPECT(same(demforge::utilization(rw[w], rp, rv), demb200::utilization(bw[w], bp, bv)));
        // merge of per-step reports (runner.cpp:128-129)
        auto rm = r; rm.merge(r);
        auto bm = b; bm.merge(b);
        EXPECT(same(rm.utilization_two_phase, bm.utilization_two_phase) && same(rm.cycles_baseline, bm.cycles_baseline));
        // metrics rows carrying the model columns (snapshot_io.cpp:70-94)
        demforge::StepMetrics rsm;
        demb200::StepMetrics bsm;
        rsm.step = bsm.step = trial + 1;
        rsm.model_cycles_baseline = bsm.model_cycles_baseline = r.cycles_baseline;
        rsm.model_cycles_two_phase = bsm.model_cycles_two_phase = r.cycles_two_phase;
        rsm.utilization_baseline = bsm.utilization_baseline = r.utilization_baseline;
        rsm.utilization_two_phase = bsm.utilization_two_phase = r.utilization_two_phase;
        rsm.contacts = bsm.contacts = 17 * trial;
        rsm.max_contacts_per_particle = bsm.max_contacts_per_particle = trial % 7;
        rsm.clamps = bsm.clamps = trial % 3;
        std::string ro, bo;
        demforge::append_metrics_rows(ro, rsm, true);
        demb200::append_metrics_rows(bo, bsm.step, bsm, nullptr, true);
        EXPECT(ro == bo);
    }
    {
        demb200::WarpCostParams bad;
        bad.c_force = 0.5;
        bool threw = false;
        try { bad.validate(); } catch (const demb200::ConfigError& e) { threw = std::string(e.what()) == "simt.c_force must exceed simt.c_check"; }
        EXPECT(threw);
    }
    {
        // the free functions of pipeline.hpp:50-56 (host utilities in both): bitwise equal, and the
        // same KernelError on a non-finite force
        std::mt19937_64 rng(11);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        demforge::ParticleSet rs;
        demb200::ParticleSet bs;
        demforge::ForceAccumulator rf;
        demb200::ForceAccumulator bf;
        for (std::uint32_t i = 0; i < 257; ++i) {
            const double p[3] = {u(rng), u(rng), u(rng)}, v[3] = {u(rng), u(rng), u(rng)}, w[3] = {u(rng), u(rng), u(rng)};
            const double r = 0.004 + 0.001 * std::abs(u(rng)), m = 1e-3 * (1.5 + u(rng));
            rs.push_back(i, {p[0], p[1], p[2]}, {v[0], v[1], v[2]}, {w[0], w[1], w[2]}, r, m, 0);
            bs.push_back(i, {p[0], p[1], p[2]}, {v[0], v[1], v[2]}, {w[0], w[1], w[2]}, r, m, 0);
            const double f[3] = {u(rng), u(rng), u(rng)}, t[3] = {1e-3 * u(rng), 1e-3 * u(rng), 1e-3 * u(rng)};
            rf.force.push_back({f[0], f[1], f[2]}); rf.torque.push_back({t[0], t[1], t[2]});
            bf.force.push_back({f[0], f[1], f[2]}); bf.torque.push_back({t[0], t[1], t[2]});
        }
        demforge::force_gravity(rs, rf, {0.1, -0.2, -9.81});
        demb200::force_gravity(bs, bf, {0.1, -0.2, -9.81});
        for (int k = 0; k < 3; ++k) {
            demforge::integrate(rs, rf, 1e-4);
            demb200::integrate(bs, bf, 1e-4);
        }
        bool eq = true;
        for (std::size_t i = 0; i < rs.size(); ++i)
            eq = eq && same3(rf.force[i], bf.force[i]) && same3(rs.positions[i], bs.positions[i]) &&
                 same3(rs.velocities[i], bs.velocities[i]) && same3(rs.angular_velocities[i], bs.angular_velocities[i]);
        EXPECT(eq);
        rf.torque[9].y = NAN;
        bf.torque[9].y = NAN;
        std::string rw, bw;
        try { demforge::integrate(rs, rf, 1e-4); } catch (const demforge::KernelError& e) { rw = std::string(e.kernel()) + ":" + e.what(); }
        try { demb200::integrate(bs, bf, 1e-4); } catch (const demb200::KernelError& e) { bw = e.kernel() + ":" + e.what(); }
        if (rw != bw) std::printf("reference: %s\nb200:      %s\n", rw.c_str(), bw.c_str());
        EXPECT(!rw.empty() && rw == bw);
    }
    std::printf("%s\n", failures ? "FAILED" : "PASSED");
    return failures ? 1 : 0;
}
