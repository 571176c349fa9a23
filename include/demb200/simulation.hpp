// demb200/simulation.hpp — header-only C++ drop-in for the reference demforge::Simulation API
// (/root/reference/proj/core/include/demforge/pipeline.hpp:62-136 and its value types), built on
// the C ABI in dem_b200.h. Types live in namespace demb200 so a program can link this and the
// reference (demforge::) side by side; `namespace demforge = demb200;` makes it a drop-in.
//
// Semantics kept from the reference:
//  * the constructor validates, uploads and runs the priming force pass (pipeline.cpp:52-84);
//  * step() runs Integrate then the force phase and returns StepMetrics (pipeline.cpp:366-378);
//  * particles()/forces()/contact_table() return references into host mirrors that are synced
//    lazily from the device; the non-const overloads mark the mirror dirty and the next kernel
//    call uploads it (the reference lets callers mutate state between kernels, runner.cpp:131);
//  * errors are rethrown as ConfigError / KernelError / CapacityError / DegenerateContactError
//    with the reference kernel names (error.hpp:10-49, pipeline.cpp:16-29);
//  * the class is copyable (a device-side clone, runner.cpp:261-270).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../dem_b200.h"

namespace demb200 {

// ---- vec3.hpp ----------------------------------------------------------------------------------
struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
    constexpr Vec3() = default;
    constexpr Vec3(double x_, double y_, double z_) : x(x_), y(y_), z(z_) {}
    bool operator==(const Vec3&) const = default;
};

// ---- error.hpp ---------------------------------------------------------------------------------
class ConfigError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
class KernelError : public std::runtime_error {
  public:
    KernelError(std::string kernel, const std::string& what)
        : std::runtime_error(what), kernel_(std::move(kernel)) {}
    const std::string& kernel() const { return kernel_; }

  private:
    std::string kernel_;
};
class CapacityError : public KernelError {
  public:
    CapacityError(std::string kernel, const std::string& what, std::uint32_t particle)
        : KernelError(std::move(kernel), what), particle_(particle) {}
    std::uint32_t particle() const { return particle_; }

  private:
    std::uint32_t particle_;
};
class DegenerateContactError : public KernelError {
  public:
    using KernelError::KernelError;
};
class DeviceError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

// ---- materials.hpp / geometry.hpp / sim_config.hpp --------------------------------------------
struct MaterialParams {
    double poisson_ratio = 0.3, shear_modulus = 4e5, youngs_modulus = 1e6, restitution = 0.9,
           sliding_friction = 0.3;
};

class MaterialTable {
  public:
    std::uint32_t add(std::string name, const MaterialParams& p) {
        for (const auto& n : names_)
            if (n == name) throw ConfigError("material '" + name + "' defined twice");
        names_.push_back(std::move(name));
        mats_.push_back(p);
        return static_cast<std::uint32_t>(mats_.size() - 1);
    }
    std::uint32_t index_of(const std::string& name) const {
        for (std::size_t i = 0; i < names_.size(); ++i)
            if (names_[i] == name) return static_cast<std::uint32_t>(i);
        throw ConfigError("unknown material '" + name + "'");
    }
    const MaterialParams& params(std::uint32_t i) const { return mats_[i]; }
    std::size_t size() const { return mats_.size(); }
    void set_pair_restitution(std::uint32_t a, std::uint32_t b, double eps) {
        if (a > b) std::swap(a, b);
        for (auto& o : over_)
            if (o.a == a && o.b == b) { o.eps = eps; return; }
        over_.push_back({a, b, eps});
    }
    double pair_restitution(std::uint32_t a, std::uint32_t b) const {  // materials.cpp:58-64
        if (a > b) std::swap(a, b);
        for (const auto& o : over_)
            if (o.a == a && o.b == b) return o.eps;
        return std::sqrt(mats_[a].restitution * mats_[b].restitution);
    }
    bool contains(const std::string& name) const {
        for (const auto& n : names_)
            if (n == name) return true;
        return false;
    }
    const std::string& name(std::uint32_t i) const { return names_[i]; }

  private:
    struct Override { std::uint32_t a, b; double eps; };
    std::vector<std::string> names_;
    std::vector<MaterialParams> mats_;
    std::vector<Override> over_;
};

struct RectWall { Vec3 corner, edge_u, edge_v; std::uint32_t material_id = 0; };
struct LineWall { Vec3 a, b; std::uint32_t material_id = 0; };
enum class CollideVariant { baseline, two_phase };

// sim_config.hpp:15-37: how `run` builds the initial state, and the run control block.
enum class InitMode { lattice, headon };
struct ParticleInitConfig {
    InitMode mode = InitMode::lattice;
    std::uint32_t count = 0;
    double radius = 0.0, mass = 0.0;
    std::string material;
    double jitter = -1.0;          // < 0: 0.1 * (spacing - 2 r)
    double lattice_spacing = 0.0;  // 0: fit to the domain
    double headon_gap = -1.0;      // < 0: 0.1 r
    double headon_speed = 1.0;
};
struct RunControlConfig {
    std::int64_t steps = 0, warmup_steps = 0, snapshot_every = 0;
    CollideVariant collide_variant = CollideVariant::two_phase;
};
// ---- warp_model.hpp ----------------------------------------------------------------------------
// The paper's lockstep SIMT cost model (warp_model.hpp:9-88), evaluated on the host over the
// traversal traces the device records (dem_get_traces). It is a model of a hypothetical warp, kept
// for the reference's metrics columns and bench report; the B200 kernels' real divergence is
// measured with ncu (profiles/). Sums run in the reference's order (warp by warp, lane by lane),
// so a report over the same traces is bitwise the reference's.
struct WarpCostParams {
    int warp_size = 32;
    double c_check = 1.0, c_force = 20.0, c_store = 1.0, c_load = 1.0;
    void validate() const {  // warp_model.cpp:9-18
        if (warp_size < 1) throw ConfigError("simt.warp_size must be >= 1");
        if (c_check < 0.0 || c_force < 0.0 || c_store < 0.0 || c_load < 0.0)
            throw ConfigError("simt cost parameters must be >= 0");
        if (!(c_force > c_check)) throw ConfigError("simt.c_force must exceed simt.c_check");
    }
};

struct TraceEvent {
    std::int32_t candidate = 0;  // slot index of the inspected partner
    bool contact = false;        // check_pair succeeded
    bool operator==(const TraceEvent&) const = default;
};
using LaneTrace = std::vector<TraceEvent>;

inline std::size_t contact_count(const LaneTrace& t) {
    std::size_t k = 0;
    for (const auto& e : t) k += e.contact ? 1 : 0;
    return k;
}

/// Lanes [w*warp_size, (w+1)*warp_size) form warp w; the last may be partial.
inline std::vector<std::span<const LaneTrace>> group_warps(std::span<const LaneTrace> lanes, int warp_size) {
    std::vector<std::span<const LaneTrace>> out;
    const std::size_t w = static_cast<std::size_t>(warp_size);
    for (std::size_t b = 0; b < lanes.size(); b += w) out.push_back(lanes.subspan(b, std::min(w, lanes.size() - b)));
    return out;
}

namespace detail {
// Lockstep shape of one warp: per iteration j (up to the longest trace) whether some lane hits,
// and the largest per-lane contact count.
struct WarpShape {
    std::vector<char> any_hit;
    std::size_t max_contacts = 0;
};
inline WarpShape warp_shape(std::span<const LaneTrace> warp) {
    WarpShape s;
    std::size_t len = 0;
    for (const auto& lane : warp) {
        len = std::max(len, lane.size());
        s.max_contacts = std::max(s.max_contacts, contact_count(lane));
    }
    s.any_hit.assign(len, 0);
    for (const auto& lane : warp)
        for (std::size_t j = 0; j < lane.size(); ++j) s.any_hit[j] |= lane[j].contact ? 1 : 0;
    return s;
}
}  // namespace detail

/// Single loop: each iteration costs a check, plus a force when any lane hits (warp_model.hpp:45-48).
inline double warp_cycles_baseline(std::span<const LaneTrace> warp, const WarpCostParams& c) {
    double cycles = 0.0;
    for (char hit : detail::warp_shape(warp).any_hit) {
        cycles += c.c_check;
        if (hit) cycles += c.c_force;
    }
    return cycles;
}

/// Two loops: check (+ store when any lane hits), then max-contacts force iterations (:50-52).
inline double warp_cycles_two_phase(std::span<const LaneTrace> warp, const WarpCostParams& c) {
    const auto s = detail::warp_shape(warp);
    double loop1 = 0.0;
    for (char hit : s.any_hit) {
        loop1 += c.c_check;
        if (hit) loop1 += c.c_store;
    }
    return loop1 + static_cast<double>(s.max_contacts) * (c.c_load + c.c_force);
}

inline double warp_useful_cycles(std::span<const LaneTrace> warp, const WarpCostParams& c, CollideVariant v) {
    double useful = 0.0;
    for (const auto& lane : warp) {
        const double hits = static_cast<double>(contact_count(lane));
        useful += static_cast<double>(lane.size()) * c.c_check + hits * c.c_force;
        if (v == CollideVariant::two_phase) useful += hits * (c.c_store + c.c_load);
    }
    return useful;
}

inline double utilization(std::span<const LaneTrace> warp, const WarpCostParams& c, CollideVariant v) {
    const double cycles = v == CollideVariant::baseline ? warp_cycles_baseline(warp, c) : warp_cycles_two_phase(warp, c);
    if (cycles == 0.0) return 1.0;
    return warp_useful_cycles(warp, c, v) / (static_cast<double>(warp.size()) * cycles);
}

struct WarpReport {
    double cycles_baseline = 0.0, cycles_two_phase = 0.0;
    double utilization_baseline = 1.0, utilization_two_phase = 1.0;
    std::size_t warp_count = 0;
    double useful_baseline = 0.0, useful_two_phase = 0.0;
    double occupied_baseline = 0.0, occupied_two_phase = 0.0;
    double speedup() const { return cycles_two_phase == 0.0 ? 1.0 : cycles_baseline / cycles_two_phase; }
    void refresh() {
        if (occupied_baseline > 0.0) utilization_baseline = useful_baseline / occupied_baseline;
        if (occupied_two_phase > 0.0) utilization_two_phase = useful_two_phase / occupied_two_phase;
    }
    void merge(const WarpReport& o) {
        cycles_baseline += o.cycles_baseline;
        cycles_two_phase += o.cycles_two_phase;
        warp_count += o.warp_count;
        useful_baseline += o.useful_baseline;
        useful_two_phase += o.useful_two_phase;
        occupied_baseline += o.occupied_baseline;
        occupied_two_phase += o.occupied_two_phase;
        refresh();
    }
};

inline WarpReport model_report(std::span<const LaneTrace> traces, const WarpCostParams& c) {
    WarpReport r;
    for (const auto warp : group_warps(traces, c.warp_size)) {
        const double lanes = static_cast<double>(warp.size());
        const double base = warp_cycles_baseline(warp, c), two = warp_cycles_two_phase(warp, c);
        ++r.warp_count;
        r.cycles_baseline += base;
        r.cycles_two_phase += two;
        r.useful_baseline += warp_useful_cycles(warp, c, CollideVariant::baseline);
        r.useful_two_phase += warp_useful_cycles(warp, c, CollideVariant::two_phase);
        r.occupied_baseline += lanes * base;
        r.occupied_two_phase += lanes * two;
    }
    r.refresh();
    return r;
}

struct SimConfig {
    double dt = 0.0;
    Vec3 gravity{0.0, 0.0, -9.81};
    Vec3 domain_min, domain_max;
    MaterialTable materials;
    std::vector<RectWall> rect_walls;
    std::vector<LineWall> line_walls;
    double grid_cell_size = 0.0;
    int contact_capacity = 16;
    WarpCostParams warp;
    RunControlConfig run;
    ParticleInitConfig particles;
    std::uint64_t seed = 1;
    // beyond the reference (dem_b200.h): periodic axes (bit 0 x, 1 y, 2 z) and a
    // Lees-Edwards shear rate; 0 / 0.0 is the reference's walled box
    std::uint32_t periodic = 0;
    double shear_rate = 0.0;
    int precision = 0;  // 0 fp64 parity, 1 fp32 throughput
};

// ---- particle_set.hpp --------------------------------------------------------------------------
struct ParticleSet {
    std::vector<std::uint32_t> ids;
    std::vector<Vec3> positions, velocities, angular_velocities;
    std::vector<double> radii, masses;
    std::vector<std::uint32_t> material_ids;
    std::size_t size() const { return positions.size(); }
    void push_back(std::uint32_t id, const Vec3& p, const Vec3& v, const Vec3& w, double r, double m,
                   std::uint32_t mat) {
        ids.push_back(id); positions.push_back(p); velocities.push_back(v);
        angular_velocities.push_back(w); radii.push_back(r); masses.push_back(m); material_ids.push_back(mat);
    }
    bool operator==(const ParticleSet&) const = default;
};

struct ForceAccumulator {
    std::vector<Vec3> force, torque;
    bool operator==(const ForceAccumulator&) const = default;
};

// ---- contact_table.hpp (read API) ----------------------------------------------------------------
struct ContactSlot {
    std::int32_t partner = INT32_MIN;
    bool touched = false;
    Vec3 delta_t{};
    bool empty() const { return partner == INT32_MIN; }
};

class ContactTable {
  public:
    ContactTable() = default;
    ContactTable(std::uint32_t n, int capacity) : n_(n), cap_(capacity), slots_(std::size_t(n) * capacity) {}
    static std::int32_t wall_id(int w) { return -(w + 1); }
    static bool is_wall(std::int32_t p) { return p < 0; }
    std::uint32_t particle_count() const { return n_; }
    int capacity() const { return cap_; }
    const ContactSlot* row(std::uint32_t p) const { return slots_.data() + std::size_t(p) * cap_; }
    ContactSlot* row(std::uint32_t p) { return slots_.data() + std::size_t(p) * cap_; }
    int live_count(std::uint32_t p) const {
        int k = 0;
        for (int s = 0; s < cap_; ++s) k += row(p)[s].empty() ? 0 : 1;
        return k;
    }
    int max_live_count() const {
        int m = 0;
        for (std::uint32_t p = 0; p < n_; ++p) m = std::max(m, live_count(p));
        return m;
    }
    std::int64_t total_live() const {
        std::int64_t k = 0;
        for (const auto& s : slots_) k += s.empty() ? 0 : 1;
        return k;
    }
    bool operator==(const ContactTable&) const = default;
    const ContactSlot* find(std::uint32_t p, std::int32_t partner) const {
        for (int s = 0; s < cap_; ++s)
            if (!row(p)[s].empty() && row(p)[s].partner == partner) return &row(p)[s];
        return nullptr;
    }

  private:
    std::uint32_t n_ = 0;
    int cap_ = 0;
    std::vector<ContactSlot> slots_;
};

// sorted_order.hpp:13-19 (no BitonicStats: the B200 sort is a one-digit counting sort)
struct SortedOrder {
    std::vector<std::uint32_t> sorted_keys;  // nondecreasing cell keys per slot
    std::vector<std::uint32_t> permutation;  // new slot -> previous slot
    std::vector<std::uint32_t> cell_start, cell_end;  // untouched cells: start == end == 0
};

struct UniformGrid {
    Vec3 origin;
    double cell_size = 0.0;
    int nx = 1, ny = 1, nz = 1;
    std::int64_t cell_count() const { return std::int64_t(nx) * ny * nz; }
};

// ---- pipeline.hpp ------------------------------------------------------------------------------
inline constexpr int kKernelCount = DEM_KERNEL_COUNT;  // pipeline.hpp:19-31
struct StepMetrics {  // pipeline.hpp:35-48
    std::int64_t step = 0;
    // The reference's host wall time per reference kernel; the B200 step is one CUDA graph, so
    // these stay 0 (per-device-kernel times: Simulation::profile_step).
    std::array<std::int64_t, kKernelCount> kernel_wall_ns{};
    double model_cycles_baseline = 0.0, model_cycles_two_phase = 0.0;  // with record_traces
    double utilization_baseline = 1.0, utilization_two_phase = 1.0;
    std::int64_t contacts = 0, pp_contact_events = 0;
    int max_contacts_per_particle = 0;
    std::int64_t clamps = 0;
    double friction_max_ratio = 0.0;
    std::int64_t capped_contacts = 0;  // new counter: contacts whose friction cap engaged
};

/// pipeline.hpp:50-53 (pipeline.cpp:31-44): semi-implicit update of a host particle set from
/// host forces — v += F (dt / m), x += v dt (new v), w += T (dt / I), I = ((0.4 m) r) r; throws
/// KernelError("Integrate") on a non-finite force or torque, naming the particle. A host utility
/// like the reference's (the device step integrates inside its own graph); compiled under the
/// reference's -ffp-contract=off it is bitwise the reference's.
inline void integrate(ParticleSet& state, const ForceAccumulator& forces, double dt) {
    const auto finite = [](const Vec3& v) { return std::isfinite(v.x) && std::isfinite(v.y) && std::isfinite(v.z); };
    for (std::size_t i = 0; i < state.size(); ++i) {
        const Vec3& f = forces.force[i];
        const Vec3& t = forces.torque[i];
        if (!finite(f) || !finite(t))
            throw KernelError("Integrate", "Integrate: non-finite force on particle " + std::to_string(state.ids[i]));
        const double s = dt / state.masses[i];
        Vec3& v = state.velocities[i];
        v = Vec3{v.x + f.x * s, v.y + f.y * s, v.z + f.z * s};
        Vec3& x = state.positions[i];
        x = Vec3{x.x + v.x * dt, x.y + v.y * dt, x.z + v.z * dt};
        const double inertia = 0.4 * state.masses[i] * state.radii[i] * state.radii[i];
        const double s2 = dt / inertia;
        Vec3& w = state.angular_velocities[i];
        w = Vec3{w.x + t.x * s2, w.y + t.y * s2, w.z + t.z * s2};
    }
}

/// pipeline.hpp:55-56 (pipeline.cpp:46-50): F += g m per particle; torques untouched.
inline void force_gravity(const ParticleSet& state, ForceAccumulator& forces, const Vec3& gravity) {
    for (std::size_t i = 0; i < state.size(); ++i) {
        const double m = state.masses[i];
        Vec3& f = forces.force[i];
        f = Vec3{f.x + gravity.x * m, f.y + gravity.y * m, f.z + gravity.z * m};
    }
}

namespace detail {

// SimConfig -> dem_config (the arrays it points into live here)
struct CConfig {
    dem_config c{};
    std::vector<dem_material> mats;
    std::vector<double> pair;
    std::vector<dem_rect_wall> rects;
    std::vector<dem_line_wall> lines;

    void build(const SimConfig& cfg) {
        const auto m = cfg.materials.size();
        mats.resize(m);
        pair.resize(m * m);
        for (std::size_t k = 0; k < m; ++k) {
            const auto& q = cfg.materials.params(std::uint32_t(k));
            mats[k] = dem_material{q.poisson_ratio, q.shear_modulus, q.youngs_modulus, q.restitution, q.sliding_friction};
        }
        for (std::size_t a = 0; a < m; ++a)
            for (std::size_t b = 0; b < m; ++b) pair[a * m + b] = cfg.materials.pair_restitution(std::uint32_t(a), std::uint32_t(b));
        rects.clear();
        for (const auto& w : cfg.rect_walls)
            rects.push_back(dem_rect_wall{{w.corner.x, w.corner.y, w.corner.z}, {w.edge_u.x, w.edge_u.y, w.edge_u.z},
                                          {w.edge_v.x, w.edge_v.y, w.edge_v.z}, w.material_id});
        lines.clear();
        for (const auto& w : cfg.line_walls)
            lines.push_back(dem_line_wall{{w.a.x, w.a.y, w.a.z}, {w.b.x, w.b.y, w.b.z}, w.material_id});
        c = dem_config{};
        c.dt = cfg.dt;
        c.gravity[0] = cfg.gravity.x; c.gravity[1] = cfg.gravity.y; c.gravity[2] = cfg.gravity.z;
        c.domain_min[0] = cfg.domain_min.x; c.domain_min[1] = cfg.domain_min.y; c.domain_min[2] = cfg.domain_min.z;
        c.domain_max[0] = cfg.domain_max.x; c.domain_max[1] = cfg.domain_max.y; c.domain_max[2] = cfg.domain_max.z;
        c.material_count = std::uint32_t(m);
        c.materials = mats.data();
        c.pair_restitution = pair.data();
        c.rect_wall_count = std::uint32_t(rects.size());
        c.rect_walls = rects.data();
        c.line_wall_count = std::uint32_t(lines.size());
        c.line_walls = lines.data();
        c.grid_cell_size = cfg.grid_cell_size;
        c.contact_capacity = cfg.contact_capacity;
        c.collide_variant = cfg.run.collide_variant == CollideVariant::two_phase ? 1 : 0;
        c.periodic = cfg.periodic;
        c.shear_rate = cfg.shear_rate;
        c.precision = cfg.precision;
    }
};

// a ParticleSet's arrays as dem_particles (data(): valid for empty sets too)
inline dem_particles view(ParticleSet& s) {
    dem_particles p{};
    p.count = s.size();
    p.ids = s.ids.data();
    p.positions = &s.positions.data()->x;
    p.velocities = &s.velocities.data()->x;
    p.angular_velocities = &s.angular_velocities.data()->x;
    p.radii = s.radii.data();
    p.masses = s.masses.data();
    p.material_ids = s.material_ids.data();
    return p;
}

// a dem_status as the reference's exception (error.hpp:10-49) with the reference kernel name
[[noreturn]] inline void rethrow(const dem_ctx* c, int rc) {
    dem_error e{};
    dem_last_error(c, &e);
    static const char* names[] = {"Integrate", "CalcHash", "BitonicSort", "FindCellBoundsAndReorder",
                                  "ForceGravity", "InitializeContactIDs", "Collide", "CollideRectangle",
                                  "CollideLine"};
    const std::string kernel = (e.kernel >= 0 && e.kernel < DEM_KERNEL_COUNT) ? names[e.kernel] : "?";
    switch (rc) {
        case DEM_ERR_CONFIG: throw ConfigError(e.message);
        case DEM_ERR_CAPACITY: throw CapacityError(kernel, e.message, e.particle_slot);
        case DEM_ERR_DEGENERATE: throw DegenerateContactError("Collide", e.message);
        case DEM_ERR_KERNEL: throw KernelError(kernel, e.message);
        case DEM_ERR_ARGUMENT: throw std::invalid_argument(e.message[0] ? e.message : "dem_b200: invalid argument at the C ABI");
        default: throw DeviceError(e.message);
    }
}

}  // namespace detail

class Simulation {
  public:
    Simulation(ParticleSet initial, SimConfig config, int device = 0) : cfg_(std::move(config)) {
        build_c_config();
        dem_particles p = view(initial);
        dem_ctx* c = nullptr;
        const int rc = dem_create(&ccfg_, &p, device, &c);
        if (rc != DEM_OK) rethrow(nullptr, rc);
        ctx_.reset(c);
        double r_max = 0.0;
        for (double r : initial.radii) r_max = std::max(r_max, r);
        load_grid(r_max);
        state_ = std::move(initial);
        state_fresh_ = false;
    }

    Simulation(const Simulation& o) : cfg_(o.cfg_) {
        grid_ = o.grid_;
        neighborhood_sufficient_ = o.neighborhood_sufficient_;
        o.run_pending();
        o.flush();
        build_c_config();
        dem_ctx* c = nullptr;
        const int rc = dem_clone(o.ctx_.get(), &c);
        if (rc != DEM_OK) rethrow(o.ctx_.get(), rc);
        ctx_.reset(c);
    }
    Simulation& operator=(const Simulation& o) {
        if (this != &o) { Simulation t(o); *this = std::move(t); }
        return *this;
    }
    Simulation(Simulation&&) = default;
    Simulation& operator=(Simulation&&) = default;

    StepMetrics step() { return run([&](dem_step_metrics* m) { return dem_step(ctx_.get(), 1, m); }, true); }
    /// Whether step() records traversal traces and runs the warp model (pipeline.hpp:70-71;
    /// on by default like the reference). Costs a trace download per step.
    void set_record_traces(bool on) { record_traces_ = on; }
    /// Per-slot traversal traces of the last force phase (pipeline.hpp:97), fetched on demand.
    const std::vector<LaneTrace>& traces() const { sync_traces(); return traces_; }
    void set_collide_variant(CollideVariant v) {
        cfg_.run.collide_variant = v;
        check(dem_set_collide_variant(ctx_.get(), v == CollideVariant::two_phase ? 1 : 0));
    }
    /// The reference's per-kernel methods (pipeline.hpp:77-86). The B200 step fuses kernels, so
    /// calls compose into one force phase in pipeline order (Integrate, CalcHash, BitonicSort,
    /// FindCellBoundsAndReorder, ZeroForces, ForceGravity, InitializeContactIDs, Collide,
    /// CollideRectangle, CollideLine) that runs when a result is observed (particles(), forces(),
    /// contact_table(), order(), traces(), step(), ...) or when a kernel earlier in that order is
    /// called again. Every composed phase bins and starts from zeroed accumulators, as every
    /// reference caller does (tests/test_pipeline.cpp:69-76, runner.cpp:261-270); errors surface
    /// when the phase runs.
    void kernel_integrate() { compose(0, DEM_PHASE_INTEGRATE); }
    void kernel_calc_hash() { compose(1, 0); }
    void kernel_bitonic_sort() { compose(2, 0); }
    void kernel_find_cell_bounds_and_reorder() { compose(3, 0); }
    void zero_forces() { compose(4, 0); }
    void kernel_force_gravity() { compose(5, DEM_PHASE_GRAVITY); }
    void kernel_initialize_contact_ids() { compose(6, 0); }
    void kernel_collide(CollideVariant variant, bool /*record_traces: traces are produced on demand*/) {
        compose(7, DEM_PHASE_PP);
        pending_variant_ = variant == CollideVariant::two_phase ? 1 : 0;
    }
    void kernel_collide_rectangle() { compose(8, DEM_PHASE_RECT); }
    void kernel_collide_line() { compose(9, DEM_PHASE_LINE); }

    /// advance_to_collide + kernel_collide (tests/test_pipeline.cpp:69-76): pp only, no gravity.
    StepMetrics advance_and_collide() {
        return run([&](dem_step_metrics* m) { return dem_force_phase(ctx_.get(), DEM_PHASE_INTEGRATE | DEM_PHASE_PP, m); }, false);
    }
    StepMetrics force_phase(std::uint32_t flags) {
        return run([&](dem_step_metrics* m) { return dem_force_phase(ctx_.get(), flags, m); }, false);
    }
    /// One step() without graphs; per-B200-kernel device ms (dem_device_kernel order) in `ms`.
    StepMetrics profile_step(double ms[DEM_DEVICE_KERNEL_COUNT], std::size_t flush_bytes = 0) {
        dem_step_metrics raw{};
        StepMetrics r = run([&](dem_step_metrics* m) {
            const int rc = dem_profile_step(ctx_.get(), flush_bytes, m);
            raw = *m;
            return rc;
        }, true);
        for (int k = 0; k < DEM_DEVICE_KERNEL_COUNT; ++k) ms[k] = raw.device_kernel_ms[k];
        return r;
    }

    const SimConfig& config() const { return cfg_; }
    const UniformGrid& grid() const { return grid_; }  // fixed at construction (make_grid, grid.cpp:10-28)
    /// pipeline.hpp:101-103: the cell size admits the 27-cell neighbourhood guarantee, h >= 2 r_max
    /// of the initial set (pipeline.cpp:60).
    bool neighborhood_sufficient() const { return neighborhood_sufficient_; }
    const ParticleSet& particles() const { sync_state(); return state_; }
    ParticleSet& particles() { sync_state(); state_dirty_ = true; return state_; }
    const ForceAccumulator& forces() const { sync_forces(); return forces_; }
    ForceAccumulator& forces() { sync_forces(); forces_dirty_ = true; return forces_; }
    const ContactTable& contact_table() const { sync_table(); return table_; }
    /// Mutable, as the reference's bench uses it to restore a saved table (runner.cpp:131-132):
    /// touched, non-empty slots are uploaded before the next kernel (dem_set_contacts); the
    /// phase's sweep would delete the untouched ones (contact_table.cpp:37-46).
    ContactTable& contact_table() { sync_table(); table_dirty_ = true; return table_; }
    const SortedOrder& order() const { sync_order(); return order_; }
    std::int64_t step_index() const { return dem_step_index(ctx_.get()); }
    std::int64_t last_clamp_count() const { run_pending(); return last_.clamps; }
    double mean_coordination() const {
        run_pending();
        const auto n = dem_size(ctx_.get());
        return n ? double(last_.pp_contact_events) / double(n) : 0.0;
    }

  private:
    UniformGrid grid_;
    bool neighborhood_sufficient_ = true;
    void load_grid(double r_max) {
        dem_grid g{};
        check(dem_get_grid(ctx_.get(), &g));
        grid_ = UniformGrid{Vec3{g.origin[0], g.origin[1], g.origin[2]}, g.cell_size, g.nx, g.ny, g.nz};
        neighborhood_sufficient_ = grid_.cell_size >= 2.0 * r_max;
    }
    struct CtxDeleter { void operator()(dem_ctx* c) const { dem_destroy(c); } };
    std::uint32_t pending_ = 0;    // composed per-kernel calls (kernel_integrate ...)
    int pending_last_ = -1;
    int pending_variant_ = -1;

    template <typename F>
    StepMetrics run(F&& fn, bool record) {
        if (pending_last_ >= 0) run_pending();
        flush();
        dem_step_metrics m{};
        const int rc = fn(&m);
        state_fresh_ = forces_fresh_ = table_fresh_ = false;
        if (rc != DEM_OK) rethrow(ctx_.get(), rc);
        traces_fresh_ = order_fresh_ = false;
        last_ = StepMetrics{};
        last_.step = m.step;
        last_.contacts = m.contacts;
        last_.pp_contact_events = m.pp_contact_events;
        last_.max_contacts_per_particle = m.max_contacts_per_particle;
        last_.clamps = m.clamps;
        last_.friction_max_ratio = m.friction_max_ratio;
        last_.capped_contacts = m.capped_contacts;
        if (record && record_traces_ && !cfg_.periodic) {  // pipeline.cpp:356-362 (no traces in periodic boxes)
            const WarpReport r = model_report(traces(), cfg_.warp);
            last_.model_cycles_baseline = r.cycles_baseline;
            last_.model_cycles_two_phase = r.cycles_two_phase;
            last_.utilization_baseline = r.utilization_baseline;
            last_.utilization_two_phase = r.utilization_two_phase;
        }
        return last_;
    }

    void compose(int k, std::uint32_t flag) {
        if (k <= pending_last_) run_pending();
        pending_ |= flag;
        pending_last_ = k;
    }
    // runs the composed force phase (see kernel_integrate); a no-op without pending kernels
    void run_pending() const {
        auto* self = const_cast<Simulation*>(this);
        if (pending_last_ < 0) return;
        const std::uint32_t flags = pending_;
        const int variant = pending_variant_;
        self->pending_ = 0;
        self->pending_last_ = -1;
        self->pending_variant_ = -1;
        const int current = cfg_.run.collide_variant == CollideVariant::two_phase ? 1 : 0;
        if (variant >= 0 && variant != current) self->check(dem_set_collide_variant(ctx_.get(), variant));
        self->run([&](dem_step_metrics* m) { return dem_force_phase(ctx_.get(), flags, m); }, false);
        if (variant >= 0 && variant != current) self->check(dem_set_collide_variant(ctx_.get(), current));
    }

    void flush() const {
        auto* self = const_cast<Simulation*>(this);
        if (state_dirty_) {
            dem_particles p = view(self->state_);
            self->check(dem_set_particles(ctx_.get(), &p));
            self->state_dirty_ = false;
        }
        if (forces_dirty_) {
            self->check(dem_set_forces(ctx_.get(), &self->forces_.force[0].x, &self->forces_.torque[0].x));
            self->forces_dirty_ = false;
        }
        if (table_dirty_) {
            std::vector<std::uint32_t> o;
            std::vector<std::int32_t> pr;
            std::vector<double> d;
            for (std::uint32_t i = 0; i < table_.particle_count(); ++i)
                for (int k = 0; k < table_.capacity(); ++k) {
                    const ContactSlot& c = table_.row(i)[k];
                    if (c.empty() || !c.touched) continue;
                    o.push_back(i);
                    pr.push_back(c.partner);
                    d.insert(d.end(), {c.delta_t.x, c.delta_t.y, c.delta_t.z});
                }
            self->check(dem_set_contacts(ctx_.get(), o.data(), pr.data(), d.data(), static_cast<std::int64_t>(o.size())));
            self->table_dirty_ = false;
        }
    }

    void sync_state() const {
        run_pending();
        if (state_fresh_ || state_dirty_) return;
        auto* self = const_cast<Simulation*>(this);
        const auto n = dem_size(ctx_.get());
        ParticleSet& s = self->state_;
        s.ids.resize(n); s.positions.resize(n); s.velocities.resize(n); s.angular_velocities.resize(n);
        s.radii.resize(n); s.masses.resize(n); s.material_ids.resize(n);
        dem_particles p = view(s);
        self->check(dem_get_particles(ctx_.get(), &p));
        self->state_fresh_ = true;
    }
    void sync_forces() const {
        run_pending();
        if (forces_fresh_ || forces_dirty_) return;
        auto* self = const_cast<Simulation*>(this);
        const auto n = dem_size(ctx_.get());
        self->forces_.force.resize(n);
        self->forces_.torque.resize(n);
        if (n)
            self->check(dem_get_forces(ctx_.get(), &self->forces_.force.data()->x, &self->forces_.torque.data()->x));
        self->forces_fresh_ = true;
    }
    void sync_table() const {
        run_pending();
        if (table_fresh_) return;
        auto* self = const_cast<Simulation*>(this);
        const auto n = static_cast<std::uint32_t>(dem_size(ctx_.get()));
        const std::int64_t c = dem_get_contacts(ctx_.get(), nullptr, nullptr, nullptr, 0);
        if (c < 0) self->check(static_cast<int>(c));  // an error code, not a count
        std::vector<std::uint32_t> o(c);
        std::vector<std::int32_t> p(c);
        std::vector<double> d(3 * c);
        const std::int64_t c2 = dem_get_contacts(ctx_.get(), o.data(), p.data(), d.data(), c);
        if (c2 < 0) self->check(static_cast<int>(c2));
        self->table_ = ContactTable(n, cfg_.contact_capacity);
        std::vector<int> fill(n, 0);
        for (std::int64_t k = 0; k < c; ++k) {
            ContactSlot& s = self->table_.row(o[k])[fill[o[k]]++];
            s.partner = p[k];
            s.touched = true;
            s.delta_t = Vec3{d[3 * k], d[3 * k + 1], d[3 * k + 2]};
        }
        self->table_fresh_ = true;
    }

    void sync_order() const {
        run_pending();
        if (order_fresh_) return;
        auto* self = const_cast<Simulation*>(this);
        const auto n = dem_size(ctx_.get());
        SortedOrder& o = self->order_;
        o.sorted_keys.assign(n, 0);
        o.permutation.assign(n, 0);
        check(dem_get_order(ctx_.get(), o.sorted_keys.data(), o.permutation.data()));
        const auto m = static_cast<std::size_t>(grid().cell_count());
        o.cell_start.assign(m, 0);
        o.cell_end.assign(m, 0);
        for (std::size_t i = 0; i < n; ++i) {  // sorted_order.cpp:17-29
            const std::uint32_t k = o.sorted_keys[i];
            if (i == 0 || o.sorted_keys[i - 1] != k) o.cell_start[k] = static_cast<std::uint32_t>(i);
            o.cell_end[k] = static_cast<std::uint32_t>(i + 1);
        }
        self->order_fresh_ = true;
    }

    void sync_traces() const {
        run_pending();
        if (traces_fresh_) return;
        auto* self = const_cast<Simulation*>(this);
        const auto n = dem_size(ctx_.get());
        std::vector<std::uint64_t> off(n + 1);
        const std::int64_t total = dem_get_traces(ctx_.get(), off.data(), nullptr, 0);
        if (total < 0) rethrow(ctx_.get(), static_cast<int>(-total));
        std::vector<dem_trace_event> ev(static_cast<std::size_t>(total));
        if (total > 0 && dem_get_traces(ctx_.get(), nullptr, ev.data(), total) != total) rethrow(ctx_.get(), DEM_ERR_CUDA);
        self->traces_.assign(n, LaneTrace{});
        for (std::size_t i = 0; i < n; ++i) {
            LaneTrace& t = self->traces_[i];
            t.reserve(off[i + 1] - off[i]);
            for (std::uint64_t k = off[i]; k < off[i + 1]; ++k) t.push_back(TraceEvent{ev[k].candidate, ev[k].contact != 0});
        }
        self->traces_fresh_ = true;
    }

    static dem_particles view(ParticleSet& s) { return detail::view(s); }

    void build_c_config() {
        cc_.build(cfg_);
        ccfg_ = cc_.c;
    }

    void check(int rc) const { if (rc != DEM_OK) rethrow(ctx_.get(), rc); }

    [[noreturn]] static void rethrow(const dem_ctx* c, int rc) { detail::rethrow(c, rc); }

    SimConfig cfg_;
    detail::CConfig cc_;
    dem_config ccfg_{};
    std::unique_ptr<dem_ctx, CtxDeleter> ctx_;
    mutable ParticleSet state_;
    mutable ForceAccumulator forces_;
    mutable ContactTable table_;
    mutable std::vector<LaneTrace> traces_;
    mutable SortedOrder order_;
    mutable bool state_fresh_ = false, forces_fresh_ = false, table_fresh_ = false, traces_fresh_ = false,
                 order_fresh_ = false;
    mutable bool state_dirty_ = false, forces_dirty_ = false, table_dirty_ = false;
    StepMetrics last_;
    bool record_traces_ = true;
};

}  // namespace demb200
