// runner.cpp — the run / bench / verify drivers (reference core/src/runner.cpp:35-417) over the
// B200 Simulation. run writes byte-deterministic snapshot and metrics CSVs; bench times both
// Collide variants on identical states on the device and aborts if they ever differ bitwise;
// verify checks contact completeness against a host brute-force pair scan, variant equivalence,
// the friction bound, momentum conservation and energy dissipation.
#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <set>
#include <sstream>

#include "../../include/demb200/host.hpp"

namespace demb200 {

namespace {

std::filesystem::path snapshot_path(const std::filesystem::path& dir, std::int64_t step) {
    char name[40];
    std::snprintf(name, sizeof(name), "snapshot_%06" PRId64 ".csv", step);
    return dir / name;
}

KernelError at_step(const KernelError& e, std::int64_t step) {  // runner.cpp:29-31
    return KernelError(e.kernel(), "aborted at step " + std::to_string(step) + ": " + e.what());
}

bool same_bits(const std::vector<Vec3>& a, const std::vector<Vec3>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(Vec3)) == 0;
}

bool same_tables(const ContactTable& a, const ContactTable& b) {
    if (a.particle_count() != b.particle_count() || a.capacity() != b.capacity()) return false;
    for (std::uint32_t p = 0; p < a.particle_count(); ++p)
        for (int s = 0; s < a.capacity(); ++s) {
            const ContactSlot &x = a.row(p)[s], &y = b.row(p)[s];
            if (x.partner != y.partner || std::memcmp(&x.delta_t, &y.delta_t, sizeof(Vec3)) != 0) return false;
        }
    return true;
}

Vec3 momentum(const ParticleSet& s) {  // particle_set.cpp:65-69
    Vec3 p;
    for (std::size_t i = 0; i < s.size(); ++i) {
        p.x += s.velocities[i].x * s.masses[i];
        p.y += s.velocities[i].y * s.masses[i];
        p.z += s.velocities[i].z * s.masses[i];
    }
    return p;
}

double kinetic_energy(const ParticleSet& s) {  // particle_set.cpp:71-79
    double e = 0.0;
    for (std::size_t i = 0; i < s.size(); ++i) {
        const double inertia = 0.4 * s.masses[i] * s.radii[i] * s.radii[i];
        const Vec3& v = s.velocities[i];
        const Vec3& w = s.angular_velocities[i];
        e += 0.5 * s.masses[i] * (v.x * v.x + v.y * v.y + v.z * v.z) + 0.5 * inertia * (w.x * w.x + w.y * w.y + w.z * w.z);
    }
    return e;
}

double vnorm(const Vec3& a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

// Host brute-force contact pairs (i < j, slot indices): every pair, the plain distance test of
// oracle.cpp:11-24. The completeness reference for the 27-cell neighbourhood search.
std::vector<std::pair<std::uint32_t, std::uint32_t>> brute_pairs(const ParticleSet& s) {
    std::vector<std::pair<std::uint32_t, std::uint32_t>> out;
    for (std::uint32_t i = 0; i < s.size(); ++i)
        for (std::uint32_t j = i + 1; j < s.size(); ++j) {
            const Vec3 d{s.positions[j].x - s.positions[i].x, s.positions[j].y - s.positions[i].y,
                         s.positions[j].z - s.positions[i].z};
            if (vnorm(d) < s.radii[i] + s.radii[j]) out.emplace_back(i, j);
        }
    return out;
}

// Contact pairs (i < j) seen by the traversal: the contact events of the traces (runner.cpp:245-256).
std::vector<std::pair<std::uint32_t, std::uint32_t>> trace_pairs(const std::vector<LaneTrace>& traces) {
    std::set<std::pair<std::uint32_t, std::uint32_t>> out;
    for (std::uint32_t i = 0; i < traces.size(); ++i)
        for (const TraceEvent& e : traces[i]) {
            if (!e.contact) continue;
            const auto j = static_cast<std::uint32_t>(e.candidate);
            out.emplace(std::min(i, j), std::max(i, j));
        }
    return {out.begin(), out.end()};
}

ParticleSet seeded_state(const SimConfig& cfg) {  // runner.cpp:233-243
    ParticleSet s = build_initial_state(cfg);
    XorShift64Star rng(cfg.seed ^ 0x7E57AB1E5EEDULL);
    for (std::size_t i = 0; i < s.size(); ++i) {
        s.velocities[i] = Vec3{0.1 + rng.next_in(-0.5, 0.5), rng.next_in(-0.5, 0.5), rng.next_in(-0.5, 0.5)};
        s.angular_velocities[i] = Vec3{rng.next_in(-10.0, 10.0), rng.next_in(-10.0, 10.0), rng.next_in(-10.0, 10.0)};
    }
    return s;
}

}  // namespace

RunSummary run_simulation(const SimConfig& cfg, const std::filesystem::path& out_dir, int device) {
    std::filesystem::create_directories(out_dir);
    Simulation sim(build_initial_state(cfg), cfg, device);
    RunSummary summary;
    write_snapshot(snapshot_path(out_dir, 0), sim.particles());
    ++summary.snapshots_written;
    sim.set_record_traces(false);
    for (std::int64_t s = 1; s <= cfg.run.warmup_steps; ++s) {
        try {
            sim.step();
        } catch (const KernelError& e) {
            throw at_step(e, -s);  // negative marks a warm-up step
        }
    }
    summary.metrics_path = out_dir / "metrics.csv";
    std::string text = std::string(kMetricsHeader) + "\n";
    sim.set_record_traces(true);  // model columns of the metrics rows (runner.cpp:57)
    for (std::int64_t s = 1; s <= cfg.run.steps; ++s) {
        StepMetrics m;
        try {
            m = sim.step();
        } catch (const KernelError& e) {
            throw at_step(e, s);
        }
        append_metrics_rows(text, s, m, nullptr, /*zero_wall_time=*/true);
        const bool cadence = cfg.run.snapshot_every > 0 && s % cfg.run.snapshot_every == 0;
        if (cadence || s == cfg.run.steps) {
            write_snapshot(snapshot_path(out_dir, s), sim.particles());
            ++summary.snapshots_written;
        }
        ++summary.steps_run;
    }
    std::ofstream f(summary.metrics_path, std::ios::binary);
    if (!f) throw ConfigError("cannot open " + summary.metrics_path.string());
    f << text;
    return summary;
}

namespace {

// Each measured step: fork the simulation, advance the fork with the single-loop Collide and the
// original with two-phase, on the device with per-kernel events; both must agree bitwise.
BenchPhase measure(Simulation& sim, std::int64_t steps, const std::string& label) {
    BenchPhase ph;
    ph.label = label;
    ph.steps = steps;
    double coord = 0.0;
    for (std::int64_t s = 0; s < steps; ++s) {
        Simulation fork = sim;
        fork.set_record_traces(false);
        fork.set_collide_variant(CollideVariant::baseline);
        double kb[DEM_DEVICE_KERNEL_COUNT], kt[DEM_DEVICE_KERNEL_COUNT];
        fork.profile_step(kb);
        sim.set_collide_variant(CollideVariant::two_phase);
        const StepMetrics m = sim.profile_step(kt);
        if (!same_bits(fork.particles().positions, sim.particles().positions) ||
            !same_bits(fork.forces().force, sim.forces().force) || !same_bits(fork.forces().torque, sim.forces().torque) ||
            !same_tables(fork.contact_table(), sim.contact_table()))
            throw KernelError("Collide", "bench: variant outputs differ bitwise");
        ph.collide_us_baseline += 1e3 * kb[DEM_DK_DETECT];
        ph.collide_us_two_phase += 1e3 * (kt[DEM_DK_DETECT] + kt[DEM_DK_FORCE_REDUCE]);
        for (int k = 0; k < DEM_DEVICE_KERNEL_COUNT; ++k) ph.kernel_us[k] += 1e3 * kt[k];
        coord += sim.mean_coordination();
        ph.model.merge(model_report(sim.traces(), sim.config().warp));
        (void)m;
    }
    const double inv = 1.0 / static_cast<double>(std::max<std::int64_t>(1, steps));
    ph.collide_us_baseline *= inv;
    ph.collide_us_two_phase *= inv;
    for (double& v : ph.kernel_us) v *= inv;
    ph.mean_coordination = coord * inv;
    return ph;
}

void format_phase(std::ostringstream& os, const BenchPhase& ph) {
    static const char* names[DEM_DEVICE_KERNEL_COUNT] = {"k_phase_begin", "k_integrate_hash", "k_scan_cells",
                                                         "k_scatter", "k_reorder", "k_detect", "k_force_reduce"};
    os << "[" << ph.label << "] measured steps: " << ph.steps << ", mean coordination: " << ph.mean_coordination << "\n";
    os << "  device time per step (us, two-phase step):\n";
    for (int k = 0; k < DEM_DEVICE_KERNEL_COUNT; ++k) os << "    " << names[k] << ": " << ph.kernel_us[k] << "\n";
    os << "  Collide single loop (Alg. 1):           " << ph.collide_us_baseline << " us\n";
    os << "  Collide two-phase (detect + force):     " << ph.collide_us_two_phase << " us\n";
    os << "  Collide ratio single-loop / two-phase:  " << ph.ratio() << "\n";
    os << "  modeled warp cycles baseline:          " << ph.model.cycles_baseline << "\n";
    os << "  modeled warp cycles two_phase:         " << ph.model.cycles_two_phase << "\n";
    os << "  modeled ratio baseline/two_phase:      " << ph.model.speedup() << "\n";
    os << "  modeled utilization baseline:          " << ph.model.utilization_baseline << "\n";
    os << "  modeled utilization two_phase:         " << ph.model.utilization_two_phase << "\n";
}

}  // namespace

std::string BenchReport::format() const {
    std::ostringstream os;
    format_phase(os, sparse);
    os << "\n";
    format_phase(os, dense);
    return os.str();
}

BenchReport bench(const SimConfig& cfg, int device) {  // runner.cpp:193-214
    Simulation sim(build_initial_state(cfg), cfg, device);
    sim.set_record_traces(false);  // the model is taken once per measured step, in measure()
    BenchReport r;
    const std::int64_t measured = std::max<std::int64_t>(1, cfg.run.steps);
    r.sparse = measure(sim, std::min<std::int64_t>(5, measured), "sparse (pre-warm-up)");
    for (std::int64_t s = 0; s < cfg.run.warmup_steps; ++s) {
        try {
            sim.step();
        } catch (const KernelError& e) {
            throw at_step(e, s + 1);
        }
    }
    r.dense = measure(sim, measured, "dense (warm-started)");
    return r;
}

bool VerifyReport::all_pass() const {
    return std::all_of(properties.begin(), properties.end(), [](const PropertyResult& p) { return p.pass; });
}

std::string VerifyReport::format() const {
    std::ostringstream os;
    for (const auto& p : properties) os << (p.pass ? "PASS" : "FAIL") << "  " << p.name << ": " << p.detail << "\n";
    return os.str();
}

VerifyReport verify(const SimConfig& cfg, int device) {  // runner.cpp:274-417
    VerifyReport rep;
    {
        Simulation sim(seeded_state(cfg), cfg, device);
        sim.set_record_traces(false);
        bool complete = true, variants = true;
        std::int64_t pairs = 0, missing = 0, events = 0;
        double friction = 0.0;
        int checkpoints = 0;
        for (std::int64_t s = 0; s <= 500; ++s) {
            if (s % 100 == 0) {
                ++checkpoints;
                Simulation a = sim, b = sim;  // fork at the pre-collide point (runner.cpp:261-270)
                a.set_collide_variant(CollideVariant::two_phase);
                b.set_collide_variant(CollideVariant::baseline);
                a.advance_and_collide();
                b.advance_and_collide();
                const auto found = trace_pairs(b.traces());
                const auto expect = brute_pairs(b.particles());
                pairs += static_cast<std::int64_t>(expect.size());
                if (found != expect) {
                    complete = false;
                    for (const auto& p : expect)
                        if (!std::binary_search(found.begin(), found.end(), p)) ++missing;
                }
                if (!same_bits(a.forces().force, b.forces().force) || !same_bits(a.forces().torque, b.forces().torque) ||
                    !same_tables(a.contact_table(), b.contact_table()))
                    variants = false;
            }
            if (s < 500) {
                StepMetrics m;
                try {
                    m = sim.step();
                } catch (const KernelError& e) {
                    throw at_step(e, s + 1);
                }
                friction = std::max(friction, m.friction_max_ratio);
                events += m.contacts;
            }
        }
        rep.properties.push_back({"contact-completeness", complete,
                                  complete ? "27-neighborhood found all " + std::to_string(pairs) + " brute-force pairs over " +
                                                 std::to_string(checkpoints) + " checkpoints"
                                           : std::to_string(missing) + " contacting pairs missed"});
        rep.properties.push_back({"collide-variant-equivalence", variants,
                                  variants ? "single-loop and two-phase Collide bitwise identical at " + std::to_string(checkpoints) +
                                                 " checkpoints"
                                           : "single-loop and two-phase Collide differ"});
        rep.properties.push_back({"friction-bound", friction <= 1.0 + 1e-9,
                                  "max |F_t| / (mu |F_n|) = " + format_double(friction) + " over " + std::to_string(events) +
                                      " contact events"});
    }
    {
        SimConfig free_cfg = cfg;
        free_cfg.gravity = Vec3{};
        free_cfg.rect_walls.clear();
        free_cfg.line_walls.clear();
        Simulation sim(seeded_state(free_cfg), free_cfg, device);
        sim.set_record_traces(false);
        const Vec3 p0 = momentum(sim.particles());
        const double p0n = vnorm(p0);
        double ke_last = kinetic_energy(sim.particles()), worst = 0.0;
        bool free_last = true;
        std::int64_t seen = 0;
        for (std::int64_t s = 1; s <= 1000; ++s) {
            StepMetrics m;
            try {
                m = sim.step();
            } catch (const KernelError& e) {
                throw at_step(e, s);
            }
            seen += m.contacts;
            if (s % 10 == 0) {
                const bool contact_free = m.contacts == 0;
                if (contact_free) {
                    const double ke = kinetic_energy(sim.particles());
                    if (free_last) worst = std::max(worst, ke / ke_last);
                    ke_last = ke;
                }
                free_last = contact_free;
            }
        }
        const Vec3 p1 = momentum(sim.particles());
        const double drift = vnorm(Vec3{p1.x - p0.x, p1.y - p0.y, p1.z - p0.z});
        const double rel = p0n > 0.0 ? drift / p0n : drift;
        rep.properties.push_back({"momentum-conservation", rel <= 1e-9,
                                  "relative drift " + format_double(rel) + " over 1000 steps (g = 0, no walls)"});
        rep.properties.push_back({"energy-dissipation", worst <= 1.0 + 1e-9,
                                  "worst contact-free kinetic energy ratio " + (worst > 0.0 ? format_double(worst) : std::string("n/a")) +
                                      ", " + std::to_string(seen) + " contact events seen"});
    }
    return rep;
}

}  // namespace demb200
