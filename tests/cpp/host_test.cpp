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
#include "demforge/config_io.hpp"
#include "demforge/error.hpp"
#include "demforge/lattice.hpp"
#include "demforge/snapshot_io.hpp"

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
    std::printf("%s\n", failures ? "FAILED" : "PASSED");
    return failures ? 1 : 0;
}
