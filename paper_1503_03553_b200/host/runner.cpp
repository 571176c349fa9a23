// runner.cpp — the run / bench / verify drivers (reference core/src/runner.cpp:35-417) over the
// B200 Simulation. run writes byte-deterministic snapshot and metrics CSVs; bench times both
// Collide variants on identical states on the device and aborts if they ever differ bitwise;
// verify checks the reference's five properties: contact completeness against a host brute-force
// pair scan, force-oracle equivalence of both Collide variants against an independent O(N^2) host
// oracle, the friction bound, momentum conservation and energy dissipation.
#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <unordered_map>

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

// ---- the O(N^2) force oracle of verify (reference oracle.cpp:47-105) ---------------------------
// An independent host restatement of Collide: every other particle in the 27 surrounding cells is
// a candidate, ordered by (neighbour-visit index, slot) — the Collide traversal order — then the
// reference's contact_geometry (geometry.cpp:24-58), contact_coefficients (contact_mechanics.cpp:
// 14-41), lookup_or_insert (contact_table.cpp:15-35), update_tangential_displacement (:43-46) and
// contact_force (:48-85), evaluated in the reference's association order (this file is compiled
// with -ffp-contract=off). It shares no code with the device path, so a force-kernel regression
// that hits both Collide variants alike still fails `force-oracle-equivalence`.
namespace oracle {

Vec3 add(Vec3 a, Vec3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
Vec3 sub(Vec3 a, Vec3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
Vec3 mul(Vec3 a, double k) { return {a.x * k, a.y * k, a.z * k}; }
Vec3 divv(Vec3 a, double k) { return {a.x / k, a.y / k, a.z / k}; }
double dot(Vec3 a, Vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
Vec3 cross(Vec3 a, Vec3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double norm(Vec3 a) { return std::sqrt(dot(a, a)); }

struct Slot {
    std::int32_t partner = INT32_MIN;
    bool touched = false;
    Vec3 delta_t{};
};

struct Result {
    std::vector<Vec3> force, torque;
    std::vector<std::vector<Slot>> rows;  // the table after the collide (live + touched flags)
    bool capacity_error = false;
};

double restitution_alpha(double e) {  // contact_mechanics.cpp:7-12
    if (e >= 1.0) return 0.0;
    const double ln_eps = std::log(e);
    constexpr double pi = 3.14159265358979323846;
    return -2.0 * ln_eps / std::sqrt(pi * pi + ln_eps * ln_eps);
}

// `rows`: the table at the pre-collide point (after the sweep), indexed by the state's slots
Result collide(const ParticleSet& st, const SimConfig& cfg, const UniformGrid& g, std::vector<std::vector<Slot>> rows) {
    const std::size_t n = st.size();
    Result out;
    out.force.assign(n, Vec3{});
    out.torque.assign(n, Vec3{});
    const double inv_h = 1.0 / g.cell_size;
    auto axis = [&](double v, double o, int dim) {
        const int c = static_cast<int>(std::floor((v - o) * inv_h));
        return std::clamp(c, 0, dim - 1);
    };
    std::vector<std::array<int, 3>> cell(n);
    for (std::size_t i = 0; i < n; ++i)
        cell[i] = {axis(st.positions[i].x, g.origin.x, g.nx), axis(st.positions[i].y, g.origin.y, g.ny),
                   axis(st.positions[i].z, g.origin.z, g.nz)};
    std::vector<std::pair<int, std::uint32_t>> cand;
    for (std::size_t i = 0; i < n; ++i) {
        cand.clear();
        for (std::size_t j = 0; j < n; ++j) {
            if (j == i) continue;
            const int dx = cell[j][0] - cell[i][0], dy = cell[j][1] - cell[i][1], dz = cell[j][2] - cell[i][2];
            if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) continue;
            cand.emplace_back(((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1), static_cast<std::uint32_t>(j));
        }
        std::sort(cand.begin(), cand.end());
        const Vec3 p1 = st.positions[i], v1 = st.velocities[i], w1 = st.angular_velocities[i];
        const double r1 = st.radii[i], m1 = st.masses[i];
        for (const auto& [visit, j] : cand) {
            (void)visit;
            // contact_geometry (geometry.cpp:24-49)
            const Vec3 diff = sub(st.positions[j], p1);
            const double dist = norm(diff);
            const double r2 = st.radii[j], reach = r1 + r2;
            if (dist >= reach) continue;
            if (dist < 1e-12) throw DegenerateContactError("Collide", "Collide: coincident centers: contact normal undefined");
            const Vec3 nrm = divv(diff, dist);
            const double overlap = reach - dist;
            const Vec3 rv = sub(v1, st.velocities[j]);
            const Vec3 spin = add(mul(w1, r1), mul(st.angular_velocities[j], r2));
            const Vec3 vt = add(sub(rv, mul(nrm, dot(rv, nrm))), cross(spin, nrm));
            // contact_coefficients (contact_mechanics.cpp:14-41)
            const MaterialParams& ma = cfg.materials.params(st.material_ids[i]);
            const MaterialParams& mb = cfg.materials.params(st.material_ids[j]);
            const double m2 = st.masses[j];
            const double r_eff = r1 * r2 / (r1 + r2), m_eff = m1 * m2 / (m1 + m2);
            const double shear_sum = (2.0 - ma.poisson_ratio) / ma.shear_modulus + (2.0 - mb.poisson_ratio) / mb.shear_modulus;
            const double young_sum = (2.0 - ma.poisson_ratio * ma.poisson_ratio) / ma.youngs_modulus +
                                     (2.0 - mb.poisson_ratio * mb.poisson_ratio) / mb.youngs_modulus;
            const double k_t = 8.0 * std::sqrt(r_eff * overlap) / shear_sum;
            const double k_n = (4.0 / 3.0) * std::sqrt(r_eff) / young_sum;
            const double alpha = restitution_alpha(cfg.materials.pair_restitution(st.material_ids[i], st.material_ids[j]));
            const double eta = alpha * std::sqrt(m_eff * k_n * std::sqrt(overlap));
            // lookup_or_insert (contact_table.cpp:15-35)
            auto& row = rows[i];
            Slot* slot = nullptr;
            for (auto& sl : row)
                if (sl.partner == static_cast<std::int32_t>(j)) { slot = &sl; break; }
            if (!slot) {
                for (auto& sl : row)
                    if (sl.partner == INT32_MIN) { slot = &sl; sl = Slot{static_cast<std::int32_t>(j), false, Vec3{}}; break; }
                if (!slot) { out.capacity_error = true; return out; }
            }
            slot->touched = true;
            // update_tangential_displacement + contact_force (contact_mechanics.cpp:43-85)
            const Vec3 d = add(sub(slot->delta_t, mul(nrm, dot(slot->delta_t, nrm))), mul(vt, cfg.dt));
            const Vec3 v_n = mul(nrm, dot(rv, nrm));
            const Vec3 force = sub(sub(sub(mul(d, -k_t), mul(vt, eta)), mul(nrm, k_n * overlap * std::sqrt(overlap))), mul(v_n, eta));
            const Vec3 f_normal = mul(nrm, dot(force, nrm));
            Vec3 f_tan = sub(force, f_normal);
            Vec3 d_new = d;
            const double ft = norm(f_tan);
            const double mu = std::sqrt(ma.sliding_friction * mb.sliding_friction);
            const double limit = mu * norm(f_normal);
            if (ft > limit) {
                if (ft < 1e-15) {
                    f_tan = Vec3{};
                    d_new = Vec3{};
                } else {
                    f_tan = mul(f_tan, limit / ft);
                    d_new = mul(f_tan, -1.0 / k_t);
                }
            }
            slot->delta_t = d_new;
            const Vec3 fo = add(f_normal, f_tan);
            out.force[i] = add(out.force[i], fo);
            out.torque[i] = add(out.torque[i], mul(cross(nrm, fo), r1));
        }
    }
    out.rows = std::move(rows);
    return out;
}

}  // namespace oracle

// The table of `sim` at its pre-collide point, re-indexed into the slot order `after` (the next
// phase's order): rows by stable id, particle partners mapped slot -> id -> slot, walls kept.
std::vector<std::vector<oracle::Slot>> table_before(const ContactTable& t, const ParticleSet& before, const ParticleSet& after) {
    std::unordered_map<std::uint32_t, std::uint32_t> slot_of;
    for (std::uint32_t k = 0; k < after.size(); ++k) slot_of[after.ids[k]] = k;
    std::vector<std::vector<oracle::Slot>> rows(after.size(), std::vector<oracle::Slot>(t.capacity()));
    for (std::uint32_t p = 0; p < t.particle_count(); ++p) {
        auto& row = rows[slot_of.at(before.ids[p])];
        for (int s = 0; s < t.capacity(); ++s) {
            const ContactSlot& c = t.row(p)[s];
            if (c.empty()) continue;
            const std::int32_t partner = c.partner < 0 ? c.partner : static_cast<std::int32_t>(slot_of.at(before.ids[c.partner]));
            row[s] = oracle::Slot{partner, false, c.delta_t};
        }
    }
    return rows;
}

// Forces bitwise, and per owner the touched oracle slots equal the device's contacts (same
// partners, bitwise delta_t; the device lists them in traversal order, the oracle keeps the
// reference's row positions, so they are compared as maps).
bool matches_oracle(const Simulation& sim, const oracle::Result& o) {
    if (o.capacity_error) return false;
    if (!same_bits(sim.forces().force, o.force) || !same_bits(sim.forces().torque, o.torque)) return false;
    const ContactTable& t = sim.contact_table();
    for (std::uint32_t p = 0; p < t.particle_count(); ++p) {
        std::map<std::int32_t, Vec3> a, b;
        for (int s = 0; s < t.capacity(); ++s)
            if (!t.row(p)[s].empty() && t.row(p)[s].partner >= 0) a[t.row(p)[s].partner] = t.row(p)[s].delta_t;
        for (const auto& sl : o.rows[p])
            if (sl.touched) b[sl.partner] = sl.delta_t;
        if (a.size() != b.size()) return false;
        for (const auto& [k, v] : a) {
            const auto it = b.find(k);
            if (it == b.end() || std::memcmp(&v, &it->second, sizeof(Vec3)) != 0) return false;
        }
    }
    return true;
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
        bool complete = true, oracle_ok = true;
        std::int64_t pairs = 0, missing = 0, events = 0;
        double friction = 0.0;
        int checkpoints = 0;
        for (std::int64_t s = 0; s <= 500; ++s) {
            if (s % 100 == 0) {
                ++checkpoints;
                // the table at the pre-collide point: the last phase's contacts (the sweep keeps
                // exactly those, contact_table.cpp:37-46) — read before the forks advance
                const ParticleSet before = sim.particles();
                const ContactTable tb = sim.contact_table();
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
                // force-oracle-equivalence (runner.cpp:313-318): both Collide variants against
                // the independent O(N^2) host oracle, bitwise
                const oracle::Result o = oracle::collide(b.particles(), cfg, b.grid(), table_before(tb, before, b.particles()));
                if (!matches_oracle(a, o) || !matches_oracle(b, o) || !(a.particles() == b.particles())) oracle_ok = false;
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
        rep.properties.push_back({"force-oracle-equivalence", oracle_ok,
                                  oracle_ok ? "Collide forces and delta_t table bitwise-match the O(N^2) oracle at " +
                                                  std::to_string(checkpoints) + " checkpoints"
                                            : "mismatch against the O(N^2) oracle"});
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
