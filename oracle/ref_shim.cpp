// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference core (demforge, compiled from
// its own sources under /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libdemforge_ref.so). It lets the Python tests and bench.py's
// reference arm drive demforge::Simulation, oracle_collide and the L2 physics
// functions on identical inputs. Nothing here re-implements reference logic:
// every entry point converts plain arrays to the reference's own types and
// calls its public API (pipeline.hpp:62-136, oracle.hpp:24-33, ...).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "demforge/compare.hpp"
#include "demforge/config_io.hpp"
#include "demforge/contact_mechanics.hpp"
#include "demforge/error.hpp"
#include "demforge/geometry.hpp"
#include "demforge/grid.hpp"
#include "demforge/lattice.hpp"
#include "demforge/oracle.hpp"
#include "demforge/parallel.hpp"
#include "demforge/pipeline.hpp"

#include "dem_oracle.h"  // plain-data structs shared with the C restatement

using namespace demforge;

namespace {

thread_local std::string g_last_error;

int classify(const std::exception& e) {
    if (dynamic_cast<const CapacityError*>(&e)) return ORC_ERR_CAPACITY;
    if (dynamic_cast<const DegenerateContactError*>(&e)) return ORC_ERR_DEGENERATE;
    if (dynamic_cast<const KernelError*>(&e)) return ORC_ERR_KERNEL;
    if (dynamic_cast<const ConfigError*>(&e)) return ORC_ERR_CONFIG;
    return 99;
}

Vec3 v(const double* p) { return Vec3{p[0], p[1], p[2]}; }

MaterialParams mat_of(const orc_material& m) {
    MaterialParams p;
    p.poisson_ratio = m.poisson_ratio;
    p.shear_modulus = m.shear_modulus;
    p.youngs_modulus = m.youngs_modulus;
    p.restitution = m.restitution;
    p.sliding_friction = m.sliding_friction;
    return p;
}

SimConfig config_of(const orc_config* c, std::size_t n, double r0, double m0) {
    SimConfig cfg;
    cfg.dt = c->dt;
    cfg.gravity = v(c->gravity);
    cfg.domain_min = v(c->domain_min);
    cfg.domain_max = v(c->domain_max);
    for (std::uint32_t k = 0; k < c->material_count; ++k) {
        cfg.materials.add("m" + std::to_string(k), mat_of(c->materials[k]));
    }
    if (c->pair_restitution) {
        for (std::uint32_t a = 0; a < c->material_count; ++a)
            for (std::uint32_t b = a; b < c->material_count; ++b)
                cfg.materials.set_pair_restitution(a, b, c->pair_restitution[a * c->material_count + b]);
    }
    for (std::uint32_t k = 0; k < c->rect_count; ++k) {
        const orc_rect& w = c->rects[k];
        cfg.rect_walls.push_back({v(w.corner), v(w.edge_u), v(w.edge_v), w.material_id});
    }
    for (std::uint32_t k = 0; k < c->line_count; ++k) {
        const orc_line& w = c->lines[k];
        cfg.line_walls.push_back({v(w.a), v(w.b), w.material_id});
    }
    cfg.grid_cell_size = c->grid_cell_size;
    cfg.contact_capacity = c->contact_capacity;
    cfg.run.collide_variant = CollideVariant::two_phase;
    cfg.particles.count = static_cast<std::uint32_t>(n);
    cfg.particles.radius = r0;
    cfg.particles.mass = m0;
    cfg.particles.material = "m0";
    return cfg;
}

ParticleSet state_of(std::size_t n, const std::uint32_t* ids, const double* pos, const double* vel,
                     const double* omg, const double* rad, const double* mass,
                     const std::uint32_t* mat) {
    ParticleSet s;
    for (std::size_t i = 0; i < n; ++i) {
        s.push_back(ids[i], v(pos + 3 * i), v(vel + 3 * i), v(omg + 3 * i), rad[i], mass[i], mat[i]);
    }
    return s;
}

void put(double* p, const Vec3& a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }
void ref_set_threads(int n) { set_thread_count(n); }
int ref_thread_count() { return thread_count(); }

void* ref_sim_create(const orc_config* c, std::size_t n, const std::uint32_t* ids, const double* pos,
                     const double* vel, const double* omg, const double* rad, const double* mass,
                     const std::uint32_t* mat, int* code) {
    try {
        *code = 0;
        return new Simulation(state_of(n, ids, pos, vel, omg, rad, mass, mat),
                              config_of(c, n, n ? rad[0] : 1.0, n ? mass[0] : 1.0));
    } catch (const std::exception& e) {
        g_last_error = e.what();
        *code = classify(e);
        return nullptr;
    }
}

void* ref_sim_clone(void* h) { return new Simulation(*static_cast<Simulation*>(h)); }
void ref_sim_destroy(void* h) { delete static_cast<Simulation*>(h); }
void ref_sim_set_record_traces(void* h, int on) { static_cast<Simulation*>(h)->set_record_traces(on != 0); }

int ref_sim_step(void* h, int nsteps, orc_metrics* m) {
    auto* sim = static_cast<Simulation*>(h);
    try {
        for (int k = 0; k < nsteps; ++k) {
            const StepMetrics sm = sim->step();
            if (m) {
                m->step = sm.step;
                m->contacts = sm.contacts;
                m->pp_contact_events = sm.pp_contact_events;
                m->max_contacts_per_particle = sm.max_contacts_per_particle;
                m->clamps = sm.clamps;
                m->friction_max_ratio = sm.friction_max_ratio;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return classify(e);
    }
}

// Individual kernels in Simulation order (pipeline.hpp:77-86).
int ref_sim_run_kernel(void* h, int which, int variant) {
    auto* sim = static_cast<Simulation*>(h);
    try {
        switch (which) {
            case 0: sim->kernel_integrate(); break;
            case 1: sim->kernel_calc_hash(); break;
            case 2: sim->kernel_bitonic_sort(); break;
            case 3: sim->kernel_find_cell_bounds_and_reorder(); break;
            case 4: sim->zero_forces(); break;
            case 5: sim->kernel_force_gravity(); break;
            case 6: sim->kernel_initialize_contact_ids(); break;
            case 7: sim->kernel_collide(variant & 1 ? CollideVariant::two_phase : CollideVariant::baseline, (variant & 2) != 0); break;
            case 8: sim->kernel_collide_rectangle(); break;
            case 9: sim->kernel_collide_line(); break;
            default: return -1;
        }
        return 0;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return classify(e);
    }
}

std::size_t ref_sim_size(void* h) { return static_cast<Simulation*>(h)->particles().size(); }

void ref_sim_get_state(void* h, std::uint32_t* ids, double* pos, double* vel, double* omg,
                       double* rad, double* mass, std::uint32_t* mat) {
    const ParticleSet& s = static_cast<Simulation*>(h)->particles();
    for (std::size_t i = 0; i < s.size(); ++i) {
        if (ids) ids[i] = s.ids[i];
        if (pos) put(pos + 3 * i, s.positions[i]);
        if (vel) put(vel + 3 * i, s.velocities[i]);
        if (omg) put(omg + 3 * i, s.angular_velocities[i]);
        if (rad) rad[i] = s.radii[i];
        if (mass) mass[i] = s.masses[i];
        if (mat) mat[i] = s.material_ids[i];
    }
}

void ref_sim_get_forces(void* h, double* f, double* t) {
    const ForceAccumulator& a = static_cast<Simulation*>(h)->forces();
    for (std::size_t i = 0; i < a.force.size(); ++i) {
        if (f) put(f + 3 * i, a.force[i]);
        if (t) put(t + 3 * i, a.torque[i]);
    }
}

void ref_sim_get_grid(void* h, orc_grid* g) {
    const UniformGrid& u = static_cast<Simulation*>(h)->grid();
    g->origin[0] = u.origin.x; g->origin[1] = u.origin.y; g->origin[2] = u.origin.z;
    g->cell_size = u.cell_size; g->nx = u.nx; g->ny = u.ny; g->nz = u.nz;
}

double ref_sim_mean_coordination(void* h) { return static_cast<Simulation*>(h)->mean_coordination(); }

// Traversal traces of the last kernel_collide with record_traces (pipeline.hpp:97), flattened:
// offsets[n+1], then candidate slot / contact flag per event. Returns the event count.
std::int64_t ref_sim_traces(void* h, std::uint64_t* offsets, std::int32_t* cand, std::uint8_t* contact,
                            std::int64_t cap) {
    const auto& tr = static_cast<Simulation*>(h)->traces();
    std::int64_t k = 0;
    for (std::size_t i = 0; i < tr.size(); ++i) {
        if (offsets) offsets[i] = static_cast<std::uint64_t>(k);
        for (const TraceEvent& e : tr[i]) {
            if (k < cap) { cand[k] = e.candidate; contact[k] = e.contact ? 1 : 0; }
            ++k;
        }
    }
    if (offsets) offsets[tr.size()] = static_cast<std::uint64_t>(k);
    return k;
}

// The reference warp model (warp_model.cpp:118-136) over flattened traces.
// out: cycles_baseline, cycles_two_phase, utilization_baseline, utilization_two_phase, warp_count.
void ref_model_report(std::size_t n, const std::uint64_t* offsets, const std::uint8_t* contact,
                      int warp_size, double c_check, double c_force, double c_store, double c_load,
                      double out[5]) {
    std::vector<LaneTrace> tr(n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::uint64_t k = offsets[i]; k < offsets[i + 1]; ++k)
            tr[i].push_back({static_cast<std::int32_t>(k - offsets[i]), contact[k] != 0});
    WarpCostParams p;
    p.warp_size = warp_size; p.c_check = c_check; p.c_force = c_force; p.c_store = c_store; p.c_load = c_load;
    const WarpReport r = model_report(tr, p);
    out[0] = r.cycles_baseline; out[1] = r.cycles_two_phase;
    out[2] = r.utilization_baseline; out[3] = r.utilization_two_phase;
    out[4] = static_cast<double>(r.warp_count);
}

// Live contact-table slots as (owner slot, partner, touched, delta_t), row order.
std::int64_t ref_sim_table(void* h, std::uint32_t* owner, std::int32_t* partner, std::uint8_t* touched,
                           double* dt, std::int64_t cap) {
    const ContactTable& t = static_cast<Simulation*>(h)->contact_table();
    std::int64_t k = 0;
    for (std::uint32_t p = 0; p < t.particle_count(); ++p) {
        const ContactSlot* row = t.row(p);
        for (int s = 0; s < t.capacity(); ++s) {
            if (row[s].empty()) continue;
            if (k < cap) {
                owner[k] = p; partner[k] = row[s].partner; touched[k] = row[s].touched ? 1 : 0;
                put(dt + 3 * k, row[s].delta_t);
            }
            ++k;
        }
    }
    return k;
}

// oracle_collide (oracle.cpp:47-105) on a state in the caller's slot order. table_in holds the
// live entries after the sweep, as (owner slot, partner slot or wall id, delta_t).
std::int64_t ref_oracle_collide(const orc_config* c, std::size_t n, const std::uint32_t* ids,
                                const double* pos, const double* vel, const double* omg,
                                const double* rad, const double* mass, const std::uint32_t* mat,
                                const orc_grid* g, std::int64_t nin, const std::uint32_t* in_owner,
                                const std::int32_t* in_partner, const double* in_dt, double* forces,
                                double* torques, std::uint32_t* out_owner, std::int32_t* out_partner,
                                double* out_dt, std::uint32_t* ev_owner, std::uint32_t* ev_partner,
                                std::int64_t cap, std::int64_t* n_events) {
    try {
        const SimConfig cfg = config_of(c, n, n ? rad[0] : 1.0, n ? mass[0] : 1.0);
        const ParticleSet state = state_of(n, ids, pos, vel, omg, rad, mass, mat);
        UniformGrid grid;
        grid.origin = v(g->origin);
        grid.cell_size = g->cell_size;
        grid.nx = g->nx; grid.ny = g->ny; grid.nz = g->nz;
        ContactTable table(static_cast<std::uint32_t>(n), c->contact_capacity);
        for (std::int64_t k = 0; k < nin; ++k) {
            table.lookup_or_insert(in_owner[k], in_partner[k], "Oracle").delta_t = v(in_dt + 3 * k);
        }
        table.initialize_contact_ids();  // entries alive, touched flags cleared (post-sweep)
        const OracleResult r = oracle_collide(state, cfg.materials, grid, c->dt, table);
        for (std::size_t i = 0; i < n; ++i) {
            put(forces + 3 * i, r.forces.force[i]);
            put(torques + 3 * i, r.forces.torque[i]);
        }
        std::int64_t k = 0;
        for (std::uint32_t p = 0; p < r.table.particle_count(); ++p) {
            const ContactSlot* row = r.table.row(p);
            for (int s = 0; s < r.table.capacity(); ++s) {
                if (row[s].empty() || !row[s].touched) continue;
                if (k < cap) { out_owner[k] = p; out_partner[k] = row[s].partner; put(out_dt + 3 * k, row[s].delta_t); }
                ++k;
            }
        }
        std::int64_t e = 0;
        for (const auto& ev : r.contact_events) {
            if (e < cap) { ev_owner[e] = ev.first; ev_partner[e] = ev.second; }
            ++e;
        }
        *n_events = e;
        return k;
    } catch (const std::exception& ex) {
        g_last_error = ex.what();
        return -classify(ex);
    }
}

std::int64_t ref_brute_force_pairs(std::size_t n, const double* pos, const double* rad,
                                   std::uint32_t* out_i, std::uint32_t* out_j, std::int64_t cap) {
    ParticleSet s;
    for (std::size_t i = 0; i < n; ++i) s.push_back(static_cast<std::uint32_t>(i), v(pos + 3 * i), {}, {}, rad[i], 1.0, 0);
    const auto pairs = brute_force_contact_pairs(s);
    std::int64_t k = 0;
    for (const auto& p : pairs) {
        if (k < cap) { out_i[k] = p.first; out_j[k] = p.second; }
        ++k;
    }
    return k;
}

// ---- L2 functions, for golden-vector pinning of the C restatement ----
double ref_restitution_alpha(double e) { return restitution_alpha(e); }

void ref_contact_coefficients(double dn, const orc_material* a, const orc_material* b, double r1,
                              double r2, double m1, double m2, double alpha, int wall, double out[4]) {
    const ContactCoefficients c =
        contact_coefficients_with_alpha(dn, mat_of(*a), mat_of(*b), r1, r2, m1, m2, alpha, wall != 0);
    out[0] = c.k_t; out[1] = c.k_n; out[2] = c.eta_n; out[3] = c.eta_t;
}

int ref_contact_geometry(const double p1[3], double r1, const double v1[3], const double w1[3],
                         const double pp[3], int wall, double r2, const double v2[3],
                         const double w2[3], double out[10]) {
    try {
        std::optional<ContactGeometry> g;
        if (wall) {
            g = contact_geometry(v(p1), r1, v(v1), v(w1), v(pp),
                                 ContactPartner::make_wall(PartnerKind::rectangle_wall, 0));
        } else {
            g = contact_geometry(v(p1), r1, v(pp), r2, v(v1), v(v2), v(w1), v(w2));
        }
        if (!g) return 0;
        put(out, g->normal); out[3] = g->overlap; put(out + 4, g->relative_velocity);
        put(out + 7, g->tangential_velocity);
        return 1;
    } catch (const DegenerateContactError&) {
        return -1;
    }
}

void ref_contact_force(const double g[10], const double c[4], const double dlt[3], double mu,
                       double r1, double out[12]) {
    ContactGeometry geom;
    geom.normal = v(g); geom.overlap = g[3]; geom.relative_velocity = v(g + 4);
    geom.tangential_velocity = v(g + 7);
    ContactCoefficients co; co.k_t = c[0]; co.k_n = c[1]; co.eta_n = c[2]; co.eta_t = c[3];
    const ContactForce f = contact_force(geom, co, v(dlt), mu, r1);
    put(out, f.force); put(out + 3, f.torque); put(out + 6, f.new_tangential_displacement);
    out[9] = f.normal_magnitude; out[10] = f.tangential_magnitude; out[11] = f.capped ? 1.0 : 0.0;
}

void ref_update_tangential(const double o[3], const double n[3], const double vt[3], double dt,
                           double out[3]) {
    put(out, update_tangential_displacement(v(o), v(n), v(vt), dt));
}

int ref_make_grid(const double bmin[3], const double bmax[3], double r_max, double h, orc_grid* g) {
    try {
        const UniformGrid u = make_grid(v(bmin), v(bmax), r_max, h);
        g->origin[0] = u.origin.x; g->origin[1] = u.origin.y; g->origin[2] = u.origin.z;
        g->cell_size = u.cell_size; g->nx = u.nx; g->ny = u.ny; g->nz = u.nz;
        return 0;
    } catch (const std::exception&) {
        return ORC_ERR_CONFIG;
    }
}

std::uint32_t ref_calc_hash(const double p[3], const orc_grid* g, int* clamped) {
    UniformGrid u; u.origin = v(g->origin); u.cell_size = g->cell_size; u.nx = g->nx; u.ny = g->ny; u.nz = g->nz;
    bool c = false;
    const std::uint32_t k = calc_hash(v(p), u, &c);
    if (clamped) *clamped = c ? 1 : 0;
    return k;
}

int ref_neighbor_cells(std::uint32_t cell, const orc_grid* g, std::uint32_t out[27]) {
    UniformGrid u; u.origin = v(g->origin); u.cell_size = g->cell_size; u.nx = g->nx; u.ny = g->ny; u.nz = g->nz;
    std::array<std::uint32_t, 27> a{};
    const int n = neighbor_cells(cell, u, a);
    for (int k = 0; k < n; ++k) out[k] = a[k];
    return n;
}

void ref_closest_point_rect(const double p[3], const orc_rect* w, double out[4]) {
    const ClosestPoint cp = closest_point_rectangle(v(p), RectWall{v(w->corner), v(w->edge_u), v(w->edge_v), w->material_id});
    put(out, cp.point); out[3] = cp.distance;
}

void ref_closest_point_line(const double p[3], const orc_line* w, double out[4]) {
    const ClosestPoint cp = closest_point_line(v(p), LineWall{v(w->a), v(w->b), w->material_id});
    put(out, cp.point); out[3] = cp.distance;
}

// ---- config-file path (config_io.cpp + lattice.cpp): builds config-1 inputs ----
// Returns particle count; fills arrays when non-null (call twice). Materials/walls are written
// into caller buffers sized by the first call's *n_mat/*n_rect/*n_line.
std::int64_t ref_parse_and_build(const char* text, orc_config* out_cfg, orc_material* mats,
                                 orc_rect* rects, orc_line* lines, std::uint32_t* ids, double* pos,
                                 double* vel, double* omg, double* rad, double* mass,
                                 std::uint32_t* mat, std::int64_t* steps) {
    try {
        const SimConfig cfg = parse_config_text(std::string(text), "<text>");
        const ParticleSet s = build_initial_state(cfg);
        out_cfg->dt = cfg.dt;
        put(out_cfg->gravity, cfg.gravity);
        put(out_cfg->domain_min, cfg.domain_min);
        put(out_cfg->domain_max, cfg.domain_max);
        out_cfg->material_count = static_cast<std::uint32_t>(cfg.materials.size());
        out_cfg->rect_count = static_cast<std::uint32_t>(cfg.rect_walls.size());
        out_cfg->line_count = static_cast<std::uint32_t>(cfg.line_walls.size());
        out_cfg->grid_cell_size = cfg.grid_cell_size;
        out_cfg->contact_capacity = cfg.contact_capacity;
        if (steps) *steps = cfg.run.steps;
        if (mats) {
            for (std::uint32_t k = 0; k < cfg.materials.size(); ++k) {
                const MaterialParams& p = cfg.materials.params(k);
                mats[k] = {p.poisson_ratio, p.shear_modulus, p.youngs_modulus, p.restitution, p.sliding_friction};
            }
        }
        if (rects) {
            for (std::size_t k = 0; k < cfg.rect_walls.size(); ++k) {
                const RectWall& w = cfg.rect_walls[k];
                put(rects[k].corner, w.corner); put(rects[k].edge_u, w.edge_u); put(rects[k].edge_v, w.edge_v);
                rects[k].material_id = w.material_id;
            }
        }
        if (lines) {
            for (std::size_t k = 0; k < cfg.line_walls.size(); ++k) {
                const LineWall& w = cfg.line_walls[k];
                put(lines[k].a, w.a); put(lines[k].b, w.b); lines[k].material_id = w.material_id;
            }
        }
        if (ids) {
            for (std::size_t i = 0; i < s.size(); ++i) {
                ids[i] = s.ids[i]; put(pos + 3 * i, s.positions[i]); put(vel + 3 * i, s.velocities[i]);
                put(omg + 3 * i, s.angular_velocities[i]); rad[i] = s.radii[i]; mass[i] = s.masses[i];
                mat[i] = s.material_ids[i];
            }
        }
        return static_cast<std::int64_t>(s.size());
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -classify(e);
    }
}

}  // extern "C"

// run_simulation (runner.cpp:35-82) on a config text: writes the reference's snapshot and
// metrics CSVs into out_dir. Returns the steps run or a negative error code.
#include "demforge/runner.hpp"
extern "C" std::int64_t ref_run_simulation(const char* text, const char* out_dir) {
    try {
        const demforge::SimConfig cfg = demforge::parse_config_text(std::string(text), "<text>");
        return demforge::run_simulation(cfg, out_dir).steps_run;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -classify(e);
    }
}
