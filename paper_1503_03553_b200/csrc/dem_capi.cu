// dem_capi.cu — the C ABI (include/dem_b200.h): context lifetime, validation, host<->device
// layout conversion, CUDA-graph step execution and error mapping.
//
// Host arithmetic that feeds the kernels (grid, per-material-pair tables) is compiled with
// -ffp-contract=off so it rounds exactly as the reference does (core/CMakeLists.txt:32-37).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dem_b200.h"
#include "dem_internal.h"

using namespace demb200;

namespace {

const char* kKernelNames[DEM_KERNEL_COUNT] = {
    "Integrate", "CalcHash", "BitonicSort", "FindCellBoundsAndReorder", "ForceGravity",
    "InitializeContactIDs", "Collide", "CollideRectangle", "CollideLine"};  // pipeline.cpp:16-29
const char* kDeviceKernelNames[DEM_DEVICE_KERNEL_COUNT] = {
    "k_phase_begin", "k_integrate_hash", "k_scan_cells", "k_scatter",
    "k_reorder",     "k_detect",         "k_force_reduce"};

}  // namespace

struct dem_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;

    // configuration
    double dt = 0.0, gravity[3] = {0, 0, 0};
    double domain_min[3] = {0, 0, 0}, domain_max[3] = {0, 0, 0};
    std::vector<dem_material> materials;
    std::vector<double> pair_rest;
    std::vector<dem_rect_wall> rects;
    std::vector<dem_line_wall> lines;
    double grid_cell_size = 0.0;
    int K = 16;
    int collide_variant = 1;
    dem_grid grid{};
    uint32_t periodic = 0;
    int precision = 0;               // 0 fp64 parity, 1 fp32 throughput
    double shear_rate = 0.0;
    double cell_extent[3] = {0, 0, 0};
    uint64_t n = 0;
    uint32_t M = 0;
    size_t cap = 0;

    // device memory
    StateBuf state[2]{};
    StateBuf pre{};  // single context: the force kernel's pre-integrated state (DevCtl::preint_phase)
    HistBuf hist[2]{};
    double* ft = nullptr;
    uint32_t *key = nullptr, *skey = nullptr, *loc = nullptr, *cnt = nullptr, *cstart = nullptr;
    uint32_t *tmp_src = nullptr, *tmp_id = nullptr, *prev_slot = nullptr;
    uint2* prev_row = nullptr;
    uint32_t *pair_i = nullptr, *pair_j = nullptr;
    unsigned long long *status_scan = nullptr, *status_det = nullptr;
    uint32_t n_tiles_scan = 0, n_tiles_det = 0;
    DevCtl* ctl = nullptr;
    MatPairH* d_pairs = nullptr;
    RectW* d_rects = nullptr;
    LineW* d_lines = nullptr;
    std::vector<void*> allocations;
    uint64_t device_bytes = 0;

    // execution state
    uint64_t phase_count = 0;  // force phases executed (parity selects buffers)
    uint64_t replaced_at = ~0ull;  // phase_count when dem_set_particles last replaced the state
    bool state_invalid = false;     // the last upload was rejected (REQUIRE_STATE)
    uint32_t* idmap = nullptr;      // duplicate-id screen of uploads (upload_state), idmask + 1 bits
    uint32_t idmask = 0;
    int64_t step_index = 0;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    cudaGraphExec_t graph_async[2] = {nullptr, nullptr};  // + the state-ready event node (dem_step_async)
    void* flush_buf = nullptr;
    size_t flush_bytes = 0;
    DevCtl* h_ctl = nullptr;  // pinned readback
    dem_error last_error{};

    // slab decomposition (dem_create_slab). Single-GPU contexts: kz0 = 0, nz_loc = nz.
    bool slab = false;
    int kz0 = 0, nz_loc = 0;
    int z_lo = 0, z_hi = 0;
    uint64_t n_cap = 0;           // slot capacity (owned + ghosts)
    uint64_t n_own = 0;           // owned slots assembled into Y
    uint64_t n_asm = 0;           // assembled slots (owned + ghosts)
    int sstate = 0, shist = 0;    // X = state[sstate], history = hist[shist]
    bool integrated = false;      // the pending assembly came from an integrating migrate
    uint32_t* hrm_pos = nullptr;
    uint32_t* hrm_cnt = nullptr;
    uint32_t* counters = nullptr;
    uint32_t* h_counters = nullptr;
    size_t tile_pairs = 0, imp_cap = 0, imp_used = 0;
    uint32_t rec_bytes = 0, rec_dt_off = 0, ghost_bytes = 0;

    // host-free sharded stepping (dem_create_sharded): device-resident counts, the
    // inbox block the neighbours store into, their inboxes, one graph per history parity
    bool shard = false;
    int rank = 0, nranks = 1;
    uint32_t* dn = nullptr;              // [0] phase slots (owned + ghosts), [1] owned slots
    uint8_t* inbox = nullptr;
    size_t inbox_bytes = 0;
    uint64_t cap_rec = 0;                // records per inbox region
    uint8_t* peer[2] = {nullptr, nullptr};  // lower / upper neighbour's inbox (nullptr: none)
    bool peer_ipc[2] = {false, false};   // opened with cudaIpcOpenMemHandle (closed at destroy)
    bool connected = false, primed = false, launched = false;
    bool stream_wait = true;             // flag waits as stream memory operations (else k_shard_wait)
    cudaGraphExec_t shard_graph[2] = {nullptr, nullptr};
    uint64_t launch_pb = 0;
    int64_t launch_sb = 0;

    // asynchronous stepping (dem_step_async): steps launched but not yet collected, and the
    // readback stream that overlaps dem_get_particles with the tail of the last step
    bool inflight = false;
    uint64_t inflight_pb = 0;
    int64_t inflight_sb = 0;
    dem_step_metrics async_last{};
    cudaStream_t side = nullptr;
    cudaEvent_t ev_state[2] = {nullptr, nullptr};  // recorded by step graph [parity] after k_reorder

    // device staging in the host layout for get/set (allocated on first use)
    double* raw_d = nullptr;
    uint32_t* raw_u = nullptr;
    uint64_t raw_n = 0;
};

namespace {

int state_cur(const dem_ctx* c) { return c->slab ? c->sstate : static_cast<int>(c->phase_count & 1); }
int hist_cur(const dem_ctx* c) { return c->slab ? c->shist : static_cast<int>(c->phase_count & 1); }
uint64_t ft_stride(const dem_ctx* c) { return c->slab ? c->n_cap : c->n; }

int set_error(dem_ctx* c, int code, int kernel, uint32_t slot, uint32_t id, int64_t step, const std::string& msg) {
    if (c) {
        c->last_error.code = code;
        c->last_error.kernel = kernel;
        c->last_error.particle_slot = slot;
        c->last_error.particle_id = id;
        c->last_error.step = step;
        std::snprintf(c->last_error.message, sizeof(c->last_error.message), "%s", msg.c_str());
    }
    return code;
}

thread_local dem_error g_create_error{};

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            return set_error(ctx, DEM_ERR_CUDA, -1, 0, 0, ctx ? ctx->step_index : 0,     \
                             std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #expr); \
        }                                                                                \
    } while (0)

template <typename T>
cudaError_t dalloc(dem_ctx* c, T** p, size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    if (e == cudaSuccess) {
        c->allocations.push_back(*p);
        c->device_bytes += bytes;
        e = cudaMemsetAsync(*p, 0, bytes, c->stream);
    }
    return e;
}

bool finite3(const double* p) { return std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2]); }

// SimConfig::validate (sim_config.cpp:10-60) for the fields the step consumes, and
// ParticleSet::validate (particle_set.cpp:40-58).
int validate(const dem_config* cfg, const dem_particles* p, std::string* why) {
    auto fail = [&](const std::string& s) { *why = s; return DEM_ERR_CONFIG; };
    if (!(cfg->dt > 0.0)) return fail("dt: must be > 0");
    if (!finite3(cfg->gravity)) return fail("gravity: must be finite");
    for (int a = 0; a < 3; ++a)
        if (!(cfg->domain_max[a] - cfg->domain_min[a] > 0.0))
            return fail("domain: min must be strictly below max on every axis");
    if (cfg->material_count == 0 || !cfg->materials) return fail("no materials defined");
    if (cfg->material_count > static_cast<uint32_t>(kMaxMaterials)) return fail("too many materials for the B200 tables (max 16)");
    for (uint32_t k = 0; k < cfg->material_count; ++k) {
        const dem_material& m = cfg->materials[k];
        const std::string w = "material." + std::to_string(k) + ".";
        if (!(m.poisson_ratio >= 0.0 && m.poisson_ratio < 0.5)) return fail(w + "poisson: must satisfy 0 <= sigma < 0.5");
        if (!(m.shear_modulus > 0.0)) return fail(w + "shear_modulus: must be > 0");
        if (!(m.youngs_modulus > 0.0)) return fail(w + "youngs_modulus: must be > 0");
        if (!(m.restitution > 0.0 && m.restitution <= 1.0)) return fail(w + "restitution: must satisfy 0 < eps <= 1");
        if (!(m.sliding_friction >= 0.0)) return fail(w + "mu_d: must be >= 0");
    }
    if (cfg->grid_cell_size < 0.0) return fail("grid.cell_size: must be > 0");
    if (cfg->periodic & ~7u) return fail("periodic: bits 0-2 (x, y, z) only");
    if (!std::isfinite(cfg->shear_rate)) return fail("shear_rate: must be finite");
    if (cfg->shear_rate != 0.0 && (cfg->periodic & 3u) != 3u)
        return fail("shear_rate: Lees-Edwards shear needs periodic x and y");
    if (cfg->periodic && cfg->collide_variant == 0)
        return fail("periodic boxes run the two_phase collide variant");
    if (cfg->precision != 0 && cfg->precision != 1) return fail("precision: 0 (fp64) or 1 (fp32)");
    if (cfg->precision == 1 && cfg->collide_variant == 0)
        return fail("the fp32 throughput mode runs the two_phase collide variant");
    if (cfg->contact_capacity < 1) return fail("contacts.capacity: must be >= 1");
    // k_detect stages 2K + 1 partner words + up to 38 row bounds per thread (256 threads) in its
    // 200 KB of shared memory: K <= 80 holds in periodic and walled boxes
    if (cfg->contact_capacity > kMaxContactCapacity)
        return fail("contacts.capacity: the B200 build supports at most " + std::to_string(kMaxContactCapacity));
    if (cfg->rect_wall_count + cfg->line_wall_count > static_cast<uint32_t>(kMaxWalls)) return fail("too many walls (max 64)");
    for (uint32_t k = 0; k < cfg->rect_wall_count; ++k) {
        const dem_rect_wall& w = cfg->rect_walls[k];
        const std::string where = "wall.rect." + std::to_string(k);
        const double lu = std::sqrt(w.edge_u[0] * w.edge_u[0] + w.edge_u[1] * w.edge_u[1] + w.edge_u[2] * w.edge_u[2]);
        const double lv = std::sqrt(w.edge_v[0] * w.edge_v[0] + w.edge_v[1] * w.edge_v[1] + w.edge_v[2] * w.edge_v[2]);
        if (!(lu > 0.0) || !(lv > 0.0)) return fail(where + ": degenerate rectangle (zero-length edge)");
        const double d = w.edge_u[0] * w.edge_v[0] + w.edge_u[1] * w.edge_v[1] + w.edge_u[2] * w.edge_v[2];
        if (std::abs(d) > 1e-9 * lu * lv) return fail(where + ": edge_u and edge_v must be orthogonal");
        if (w.material_id >= cfg->material_count) return fail(where + ": bad material");
    }
    for (uint32_t k = 0; k < cfg->line_wall_count; ++k) {
        const dem_line_wall& w = cfg->line_walls[k];
        const std::string where = "wall.line." + std::to_string(k);
        const double dx = w.b[0] - w.a[0], dy = w.b[1] - w.a[1], dz = w.b[2] - w.a[2];
        if (!(std::sqrt(dx * dx + dy * dy + dz * dz) > 0.0)) return fail(where + ": zero-length segment");
        if (w.material_id >= cfg->material_count) return fail(where + ": bad material");
    }
    if (p->count >= (1ull << 31)) return fail("particle count must be < 2^31");
    for (uint64_t i = 0; i < p->count; ++i) {
        if (!(p->radii[i] > 0.0)) return fail("particle " + std::to_string(p->ids[i]) + ": radius must be > 0");
        if (!(p->masses[i] > 0.0)) return fail("particle " + std::to_string(p->ids[i]) + ": mass must be > 0");
        if (!finite3(p->positions + 3 * i) || !finite3(p->velocities + 3 * i) || !finite3(p->angular_velocities + 3 * i))
            return fail("particle " + std::to_string(p->ids[i]) + ": non-finite state");
        if (p->material_ids[i] >= cfg->material_count) return fail("particle " + std::to_string(p->ids[i]) + ": bad material");
    }
    return DEM_OK;
}

// make_grid, grid.cpp:10-28
int make_grid(const dem_config* cfg, double r_max, dem_grid* g, std::string* why) {
    const double ex = cfg->domain_max[0] - cfg->domain_min[0];
    const double ey = cfg->domain_max[1] - cfg->domain_min[1];
    const double ez = cfg->domain_max[2] - cfg->domain_min[2];
    if (!(ex > 0.0 && ey > 0.0 && ez > 0.0)) { *why = "domain box is degenerate (min must be strictly below max)"; return DEM_ERR_CONFIG; }
    double h = cfg->grid_cell_size;
    if (h <= 0.0) h = 2.0 * r_max * (1.0 + 1e-6);
    if (!(h > 0.0)) { *why = "grid.cell_size must be positive"; return DEM_ERR_CONFIG; }
    for (int a = 0; a < 3; ++a) g->origin[a] = cfg->domain_min[a];
    g->cell_size = h;
    g->nx = std::max(1, static_cast<int>(std::ceil(ex / h)));
    g->ny = std::max(1, static_cast<int>(std::ceil(ey / h)));
    g->nz = std::max(1, static_cast<int>(std::ceil(ez / h)));
    // periodic axes: n = floor(L / h) cells of extent L / n >= h
    const double ext[3] = {ex, ey, ez};
    int32_t* dims[3] = {&g->nx, &g->ny, &g->nz};
    for (int a = 0; a < 3; ++a) {
        if (!(cfg->periodic & (1u << a))) continue;
        const int na = static_cast<int>(std::floor(ext[a] / h));
        if (na < 3) { *why = "periodic axis needs at least 3 cells (domain length >= 3 h)"; return DEM_ERR_CONFIG; }
        if (a == 0 && cfg->shear_rate != 0.0 && na < 4) { *why = "sheared box needs at least 4 cells along x"; return DEM_ERR_CONFIG; }
        *dims[a] = na;
    }
    const int64_t cells = static_cast<int64_t>(g->nx) * g->ny * g->nz;
    if (cells > (int64_t{1} << 31)) { *why = "grid has more than 2^31 cells; increase grid.cell_size"; return DEM_ERR_CONFIG; }
    if (cells >= (int64_t{1} << 31) - 1) { *why = "grid too large for 32-bit cell keys"; return DEM_ERR_CONFIG; }
    return DEM_OK;
}

double restitution_alpha(double restitution) {  // contact_mechanics.cpp:7-12
    if (restitution >= 1.0) return 0.0;
    const double ln_eps = std::log(restitution);
    constexpr double pi = 3.14159265358979323846;
    return -2.0 * ln_eps / std::sqrt(pi * pi + ln_eps * ln_eps);
}

// periodic box fields of a context: cell extent L / n on periodic axes
void set_periodic(dem_ctx* c, const dem_config* cfg) {
    c->periodic = cfg->periodic & 7u;
    c->shear_rate = c->periodic ? cfg->shear_rate : 0.0;
    const int n[3] = {c->grid.nx, c->grid.ny, c->grid.nz};
    for (int a = 0; a < 3; ++a) {
        const double L = cfg->domain_max[a] - cfg->domain_min[a];
        c->cell_extent[a] = (c->periodic & (1u << a)) ? L / static_cast<double>(n[a]) : c->grid.cell_size;
    }
}

StepParams make_params(const dem_ctx* c, uint32_t flags) {
    StepParams p{};
    p.ox = c->grid.origin[0]; p.oy = c->grid.origin[1]; p.oz = c->grid.origin[2];
    p.h = c->grid.cell_size;
    p.inv_h = 1.0 / c->grid.cell_size;  // grid.cpp:32
    p.nx = c->grid.nx; p.ny = c->grid.ny; p.nz = c->grid.nz;
    p.kz0 = c->kz0;
    p.nz_loc = c->nz_loc;
    p.M = c->M;
    p.dt = c->dt;
    p.gx = c->gravity[0]; p.gy = c->gravity[1]; p.gz = c->gravity[2];
    p.n = static_cast<uint32_t>(c->slab ? c->n_asm : c->n);
    p.K = c->K;
    p.nmat = static_cast<int>(c->materials.size());
    p.nrect = static_cast<int>(c->rects.size());
    p.nline = static_cast<int>(c->lines.size());
    p.flags = flags;
    p.det_lo = 1.0 - 0x1p-40;  // see k_detect
    p.det_hi = 1.0 + 0x1p-40;
    p.det_tiny = 4e-24;
    p.periodic = c->periodic;
    const double inv[3] = {1.0 / c->cell_extent[0], 1.0 / c->cell_extent[1], 1.0 / c->cell_extent[2]};
    p.inv_x = (c->periodic & 1u) ? inv[0] : p.inv_h;
    p.inv_y = (c->periodic & 2u) ? inv[1] : p.inv_h;
    p.inv_z = (c->periodic & 4u) ? inv[2] : p.inv_h;
    p.Lx = c->domain_max[0] - c->domain_min[0];
    p.Ly = c->domain_max[1] - c->domain_min[1];
    p.Lz = c->domain_max[2] - c->domain_min[2];
    p.half_x = 0.5 * p.Lx; p.half_y = 0.5 * p.Ly; p.half_z = 0.5 * p.Lz;
    p.shear_rate = c->shear_rate;
    p.shear_u = c->shear_rate * p.Ly;
    if (c->precision == 1) p.flags |= kPhaseFp32;
    if (!c->slab) p.flags |= kPhasePreint;
    if (c->periodic && (!(c->periodic & 1u) || c->grid.nx >= 5) && (!(c->periodic & 2u) || c->grid.ny >= 5) &&
        (!(c->periodic & 4u) || c->grid.nz >= 5))
        p.flags |= kPhaseInterior;
    p.pairs = c->d_pairs;
    p.rects = c->d_rects;
    p.lines = c->d_lines;
    return p;
}

// Buffers of force phase number `phase` (1-based): state (phase-1)%2 -> phase%2.
PhaseBufs make_bufs(const dem_ctx* c, uint64_t phase) {
    PhaseBufs b{};
    const int cur = static_cast<int>(phase & 1), prev = cur ^ 1;
    b.src = c->state[prev];
    b.dst = c->state[cur];
    b.old_h = c->hist[prev];
    b.cur_h = c->hist[cur];
    b.ft = c->ft;
    b.pre = c->pre;
    b.key = c->key; b.skey = c->skey; b.loc = c->loc; b.cnt = c->cnt; b.cstart = c->cstart;
    b.tmp_src = c->tmp_src; b.tmp_id = c->tmp_id; b.prev_slot = c->prev_slot; b.prev_row = c->prev_row;
    b.pair_i = c->pair_i; b.pair_j = c->pair_j;
    b.status_scan = c->status_scan; b.status_det = c->status_det;
    b.n_tiles_scan = c->n_tiles_scan; b.n_tiles_det = c->n_tiles_det;
    b.cap = c->cap;
    b.ft_stride = static_cast<uint32_t>(c->slab ? c->n_cap : c->n);
    b.ctl = c->ctl;
    if (c->slab) {
        // slab phase: bin the assembly Y into X; previous history rows reached through the
        // remapped / imported index (hrm_*), new history into the other history buffer
        b.src = c->state[c->sstate ^ 1];
        b.dst = c->state[c->sstate];
        b.old_h = c->hist[c->shist];
        b.old_h.pos = c->hrm_pos;
        b.old_h.cnt = c->hrm_cnt;
        b.cur_h = c->hist[c->shist ^ 1];
        b.n_tiles_det = detect_tiles(static_cast<uint32_t>(c->n_asm));
    }
    return b;
}

// Enqueue one force phase; with `ev` (9 events) records an event after each kernel.
// state_ready (graphs only): an external event node after k_reorder — the phase's particle state
// is final there (detection and forces only read it), so a readback can overlap them.
void enqueue_phase(const dem_ctx* c, uint32_t flags, uint64_t phase, cudaEvent_t* ev,
                   cudaEvent_t state_ready = nullptr) {
    const StepParams p = make_params(c, flags);
    const PhaseBufs b = make_bufs(c, phase);
    cudaStream_t s = c->stream;
    if (ev) cudaEventRecord(ev[0], s);
    launch_phase_begin(p, b, s);
    if (ev) cudaEventRecord(ev[1], s);
    launch_integrate_hash(p, b, (flags & DEM_PHASE_INTEGRATE) != 0, s);
    if (ev) cudaEventRecord(ev[2], s);
    launch_scan_cells(p, b, s);
    if (ev) cudaEventRecord(ev[3], s);
    launch_scatter(p, b, s);
    if (ev) cudaEventRecord(ev[4], s);
    launch_reorder(p, b, s);
    if (ev) cudaEventRecord(ev[5], s);
    if (state_ready) cudaEventRecordWithFlags(state_ready, s, cudaEventRecordExternal);
    if (c->collide_variant == 0) {
        // Alg. 1, single loop (pipeline.cpp:209-217): detection and forces in one divergent loop
        launch_collide_single_loop(p, b, s);
        if (ev) cudaEventRecord(ev[6], s);
        if (ev) cudaEventRecord(ev[7], s);
    } else {
        launch_detect(p, b, s);
        if (ev) cudaEventRecord(ev[6], s);
        launch_force_reduce(p, b, s);
        if (ev) cudaEventRecord(ev[7], s);
    }
}

// Step graphs per phase parity; the asynchronous ones also record ev_state after k_reorder (an
// event node between kernels costs ~1 us of launch latency, so dem_step runs without it).
int build_graphs(dem_ctx* ctx) {
    for (int par = 0; par < 2; ++par) {
        if (!ctx->ev_state[par]) CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_state[par], cudaEventDisableTiming));
        for (int async = 0; async < 2; ++async) {
            cudaGraphExec_t& ge = async ? ctx->graph_async[par] : ctx->graph[par];
            if (ge) { cudaGraphExecDestroy(ge); ge = nullptr; }
            cudaGraph_t g;
            CUDA_TRY(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            enqueue_phase(ctx, DEM_PHASE_STEP, static_cast<uint64_t>(par), nullptr, async ? ctx->ev_state[par] : nullptr);
            CUDA_TRY(cudaStreamEndCapture(ctx->stream, &g));
            CUDA_TRY(cudaGraphInstantiate(&ge, g, 0));
            cudaGraphDestroy(g);
        }
    }
    return DEM_OK;
}

// Reads the control block after a sync; maps a device error to last_error.
int collect(dem_ctx* ctx, dem_step_metrics* m, uint64_t phase_before, int64_t step_before, bool is_step,
            bool fetched = false) {
    if (!fetched) {
        CUDA_TRY(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        CUDA_TRY(cudaGetLastError());
    }
    const DevCtl& d = *ctx->h_ctl;
    if (d.err_key != kNoError) {
        const uint64_t fail_phase = d.err_phase;
        ctx->phase_count = d.phase;  // phases after the failing one were halted
        const int64_t done = static_cast<int64_t>(fail_phase - phase_before);
        const int64_t fail_step = is_step ? step_before + done : ctx->step_index;
        ctx->step_index = is_step ? fail_step : ctx->step_index;
        const int kernel = static_cast<int>(d.err_key >> 56);
        const uint32_t slot = static_cast<uint32_t>((d.err_key >> 8) & 0xffffffffull);
        const int code = static_cast<int>(d.err_key & 0xff);
        const uint32_t id = static_cast<uint32_t>(d.err_sid[kernel] & 0xffffffffull);
        std::string what;
        const char* kname = kKernelNames[kernel];
        if (code == DEM_ERR_KERNEL) {
            what = std::string(kname) + ": non-finite force on particle " + std::to_string(id);  // pipeline.cpp:35-38
        } else if (code == DEM_ERR_CAPACITY) {
            what = std::string(kname) + ": contact capacity exceeded for particle " + std::to_string(slot) +
                   " (capacity " + std::to_string(ctx->K) + ")";  // error.hpp:30-42
        } else {
            kname = "Collide";  // geometry.cpp:32 tags every degenerate contact "Collide"
            what = std::string(kname) + ": coincident centers: contact normal undefined";
        }
        set_error(ctx, code, kernel, slot, id, fail_step, what);
        // reset the device error word so the context can be inspected / reused
        DevCtl clean = d;
        clean.err_key = kNoError;
        for (auto& s : clean.err_sid) s = kNoError;
        clean.halted = 0;
        clean.preint_phase = ~0ull;  // the failed phase's state is what the caller inspects
        clean.deferred[0] = clean.deferred[1] = ~0ull;
        CUDA_TRY(cudaMemcpyAsync(ctx->ctl, &clean, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return code;
    }
    if (m) {
        m->step = ctx->step_index;
        m->contacts = static_cast<int64_t>(d.contacts);
        m->pp_contact_events = static_cast<int64_t>(d.pp_events);
        m->max_contacts_per_particle = static_cast<int32_t>(d.max_per);
        m->clamps = static_cast<int64_t>(d.clamps);
        double fm;
        std::memcpy(&fm, &d.fric_bits, sizeof(double));
        m->friction_max_ratio = fm;
        m->capped_contacts = static_cast<int64_t>(d.capped);
        m->cells = ctx->M;
    }
    return DEM_OK;
}

// Collects steps launched by dem_step_async (sync, error mapping, metrics of the last one). Every
// entry point that reads or replaces device state settles first, so an asynchronous step's error
// surfaces at the next such call, attributed to the step that failed.
int settle(dem_ctx* ctx) {
    if (!ctx->inflight) return DEM_OK;
    ctx->inflight = false;
    std::memset(&ctx->async_last, 0, sizeof(ctx->async_last));
    return collect(ctx, &ctx->async_last, ctx->inflight_pb, ctx->inflight_sb, true);
}
#define SETTLE(ctx)                                  \
    do {                                             \
        const int settle_rc_ = settle(ctx);          \
        if (settle_rc_ != DEM_OK) return settle_rc_; \
    } while (0)
// entry points that run phases on the state: refused after a rejected dem_set_particles
#define REQUIRE_STATE(ctx)                                                                          \
    do {                                                                                            \
        if ((ctx)->state_invalid)                                                                   \
            return set_error(ctx, DEM_ERR_CONFIG, -1, 0, 0, (ctx)->step_index,                      \
                             "particle state was rejected by dem_set_particles; upload a valid one"); \
    } while (0)

void free_ctx(dem_ctx* c) {
    if (!c) return;
    if (c->device >= 0) cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);
    for (auto& g : c->graph) if (g) cudaGraphExecDestroy(g);
    for (auto& g : c->shard_graph) if (g) cudaGraphExecDestroy(g);
    for (int k = 0; k < 2; ++k)
        if (c->peer_ipc[k] && c->peer[k] && !(k == 1 && c->peer_ipc[0] && c->peer[0] == c->peer[1]))
            cudaIpcCloseMemHandle(c->peer[k]);
    for (auto& g : c->graph_async) if (g) cudaGraphExecDestroy(g);
    for (auto& e : c->ev_state) if (e) cudaEventDestroy(e);
    if (c->side) cudaStreamDestroy(c->side);
    for (void* p : c->allocations) cudaFree(p);
    if (c->flush_buf) cudaFree(c->flush_buf);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    if (c->h_counters) cudaFreeHost(c->h_counters);
    if (c->raw_d) cudaFree(c->raw_d);
    if (c->raw_u) cudaFree(c->raw_u);
    if (c->idmap) cudaFree(c->idmap);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int allocate(dem_ctx* ctx) {
    const uint64_t n = ctx->slab ? ctx->n_cap : ctx->n;  // slot capacity
    ctx->n_tiles_scan = scan_tiles(ctx->M);
    ctx->n_tiles_det = detect_tiles(static_cast<uint32_t>(n));
    ctx->tile_pairs = static_cast<size_t>(ctx->n_tiles_det) * 32u * static_cast<size_t>(ctx->K);  // tile regions
    ctx->cap = ctx->tile_pairs + ctx->imp_cap * static_cast<size_t>(ctx->K);  // + history import region
    if (ctx->slab) {
        CUDA_TRY(dalloc(ctx, &ctx->hrm_pos, n));
        CUDA_TRY(dalloc(ctx, &ctx->hrm_cnt, n));
        CUDA_TRY(dalloc(ctx, &ctx->counters, 8));
        CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_counters), 8 * sizeof(uint32_t)));
    }
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(dalloc(ctx, &ctx->state[b].pos_r, n));
        CUDA_TRY(dalloc(ctx, &ctx->state[b].vel_m, n));
        CUDA_TRY(dalloc(ctx, &ctx->state[b].omg, n));
        CUDA_TRY(dalloc(ctx, &ctx->state[b].idm, n));
        CUDA_TRY(dalloc(ctx, &ctx->state[b].pos_f, n));
        CUDA_TRY(dalloc(ctx, &ctx->hist[b].pos, n));
        CUDA_TRY(dalloc(ctx, &ctx->hist[b].cnt, n));
        CUDA_TRY(dalloc(ctx, &ctx->hist[b].key, ctx->cap));
        CUDA_TRY(dalloc(ctx, &ctx->hist[b].dt, 3 * ctx->cap));
    }
    if (!ctx->slab) {
        CUDA_TRY(dalloc(ctx, &ctx->pre.pos_r, n));
        CUDA_TRY(dalloc(ctx, &ctx->pre.vel_m, n));
        CUDA_TRY(dalloc(ctx, &ctx->pre.omg, n));
    }
    CUDA_TRY(dalloc(ctx, &ctx->ft, 6 * n));
    CUDA_TRY(dalloc(ctx, &ctx->key, n));
    CUDA_TRY(dalloc(ctx, &ctx->skey, n));
    CUDA_TRY(dalloc(ctx, &ctx->loc, n));
    CUDA_TRY(dalloc(ctx, &ctx->cnt, static_cast<size_t>(ctx->M) + 4));
    CUDA_TRY(dalloc(ctx, &ctx->cstart, static_cast<size_t>(ctx->M) + 4));
    CUDA_TRY(dalloc(ctx, &ctx->tmp_src, n));
    CUDA_TRY(dalloc(ctx, &ctx->tmp_id, n));
    CUDA_TRY(dalloc(ctx, &ctx->prev_slot, n));
    CUDA_TRY(dalloc(ctx, &ctx->prev_row, n));
    CUDA_TRY(dalloc(ctx, &ctx->pair_i, ctx->cap));
    CUDA_TRY(dalloc(ctx, &ctx->pair_j, ctx->cap));
    CUDA_TRY(dalloc(ctx, &ctx->status_scan, ctx->n_tiles_scan + 1));
    CUDA_TRY(dalloc(ctx, &ctx->status_det, ctx->n_tiles_det + 1));
    CUDA_TRY(dalloc(ctx, &ctx->ctl, 1));
    CUDA_TRY(dalloc(ctx, &ctx->d_pairs, kMaxMaterials * kMaxMaterials));
    CUDA_TRY(dalloc(ctx, &ctx->d_rects, kMaxWalls));
    CUDA_TRY(dalloc(ctx, &ctx->d_lines, kMaxWalls));
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_ctl), sizeof(DevCtl)));
    return DEM_OK;
}

int upload_tables(dem_ctx* ctx) {
    const size_t m = ctx->materials.size();
    std::vector<MatPairH> tab(m * m);
    for (size_t a = 0; a < m; ++a)
        for (size_t b = 0; b < m; ++b) {
            const dem_material& ma = ctx->materials[a];
            const dem_material& mb = ctx->materials[b];
            MatPairH& t = tab[a * m + b];
            t.shear_sum = (2.0 - ma.poisson_ratio) / ma.shear_modulus + (2.0 - mb.poisson_ratio) / mb.shear_modulus;
            t.young_sum = (2.0 - ma.poisson_ratio * ma.poisson_ratio) / ma.youngs_modulus +
                          (2.0 - mb.poisson_ratio * mb.poisson_ratio) / mb.youngs_modulus;
            double eps;
            if (!ctx->pair_rest.empty()) {
                eps = ctx->pair_rest[a * m + b];
            } else {
                const size_t lo = std::min(a, b), hi = std::max(a, b);  // materials.cpp:58-64
                eps = std::sqrt(ctx->materials[lo].restitution * ctx->materials[hi].restitution);
            }
            t.alpha = restitution_alpha(eps);
            t.mu = std::sqrt(ma.sliding_friction * mb.sliding_friction);  // materials.cpp:66-68
        }
    std::vector<RectW> rw(ctx->rects.size());
    for (size_t k = 0; k < rw.size(); ++k) {
        for (int a = 0; a < 3; ++a) {
            rw[k].c[a] = ctx->rects[k].corner[a];
            rw[k].u[a] = ctx->rects[k].edge_u[a];
            rw[k].v[a] = ctx->rects[k].edge_v[a];
        }
        rw[k].mat = ctx->rects[k].material_id;
    }
    std::vector<LineW> lw(ctx->lines.size());
    for (size_t k = 0; k < lw.size(); ++k) {
        for (int a = 0; a < 3; ++a) { lw[k].a[a] = ctx->lines[k].a[a]; lw[k].b[a] = ctx->lines[k].b[a]; }
        lw[k].mat = ctx->lines[k].material_id;
    }
    if (!tab.empty()) CUDA_TRY(cudaMemcpyAsync(ctx->d_pairs, tab.data(), tab.size() * sizeof(MatPairH), cudaMemcpyHostToDevice, ctx->stream));
    if (!rw.empty()) CUDA_TRY(cudaMemcpyAsync(ctx->d_rects, rw.data(), rw.size() * sizeof(RectW), cudaMemcpyHostToDevice, ctx->stream));
    if (!lw.empty()) CUDA_TRY(cudaMemcpyAsync(ctx->d_lines, lw.data(), lw.size() * sizeof(LineW), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DEM_OK;
}

// Staging buffers in the caller's layout (11 doubles + 2 u32 per particle).
int ensure_raw(dem_ctx* ctx, uint64_t n) {
    if (ctx->raw_n >= n && ctx->raw_d) return DEM_OK;
    if (ctx->raw_d) { cudaFree(ctx->raw_d); cudaFree(ctx->raw_u); ctx->raw_d = nullptr; ctx->raw_u = nullptr; }
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&ctx->raw_d), std::max<uint64_t>(n, 1) * 11 * sizeof(double)));
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&ctx->raw_u), std::max<uint64_t>(n, 1) * 2 * sizeof(uint32_t)));
    uint64_t bits = 1024;
    while (bits < 4 * n && bits < (1ull << 32)) bits <<= 1;
    if (ctx->idmap) cudaFree(ctx->idmap);
    ctx->idmap = nullptr;
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&ctx->idmap), bits / 8));
    ctx->idmask = static_cast<uint32_t>(bits - 1);
    ctx->raw_n = n;
    return DEM_OK;
}

RawState raw_view(const dem_ctx* ctx, uint64_t n) {
    RawState r{};
    r.pos = ctx->raw_d;
    r.vel = ctx->raw_d + 3 * n;
    r.omg = ctx->raw_d + 6 * n;
    r.rad = ctx->raw_d + 9 * n;
    r.mass = ctx->raw_d + 10 * n;
    r.ids = ctx->raw_u;
    r.mat = ctx->raw_u + n;
    return r;
}

// ParticleSet ids must be unique for the B200 path: its contact history is keyed by the partner's
// stable id (the reference keys it by slot, contact_table.hpp:16-24). Exact, O(n log n) on a copy:
// at creation, and after an upload whose device screen saw a possible duplicate (upload_state).
int check_unique_ids(const uint32_t* ids, uint64_t n, std::string* why) {
    if (!ids) return DEM_OK;
    std::vector<uint32_t> v(ids, ids + n);
    std::sort(v.begin(), v.end());
    const auto d = std::adjacent_find(v.begin(), v.end());
    if (d != v.end()) {
        *why = "particle " + std::to_string(*d) + ": duplicate stable id (the B200 contact history is keyed by id)";
        return DEM_ERR_CONFIG;
    }
    if (n && v.back() > 0xFFFFFFBFu) {
        *why = "particle " + std::to_string(v.back()) + ": stable id in the reserved wall-key range (>= 0xFFFFFFC0)";
        return DEM_ERR_CONFIG;
    }
    return DEM_OK;
}

// Host arrays -> device staging (plain copies; pinned callers get full PCIe bandwidth) -> SoA.
// (Zero-copy packing straight from page-locked arrays was measured: no faster on the way in,
// slower on the way out.)
int upload_state(dem_ctx* ctx, const dem_particles* p, int buf) {
    const uint64_t n = ctx->n;
    if (!n) return DEM_OK;
    cudaStream_t s = ctx->stream;
    int rc = ensure_raw(ctx, n);
    if (rc != DEM_OK) return rc;
    RawState r = raw_view(ctx, n);
    // ids, radii, masses, material ids may be NULL (dem_set_particles): the slots keep theirs
    if (!p->radii) r.rad = nullptr;
    if (!p->masses) r.mass = nullptr;
    if (!p->ids) r.ids = nullptr;
    if (!p->material_ids) r.mat = nullptr;
    CUDA_TRY(cudaMemcpyAsync(r.pos, p->positions, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(r.vel, p->velocities, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(r.omg, p->angular_velocities, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
    if (r.rad) CUDA_TRY(cudaMemcpyAsync(r.rad, p->radii, n * sizeof(double), cudaMemcpyHostToDevice, s));
    if (r.mass) CUDA_TRY(cudaMemcpyAsync(r.mass, p->masses, n * sizeof(double), cudaMemcpyHostToDevice, s));
    if (r.ids) CUDA_TRY(cudaMemcpyAsync(r.ids, p->ids, n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    if (r.mat) CUDA_TRY(cudaMemcpyAsync(r.mat, p->material_ids, n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    // + r_ref, m_ref = particle 0's radius and mass: the monodisperse detection shortcut compares
    // every radius with r_ref (k_integrate_hash); k_force_reduce memoises r_eff, m_eff, k_n for
    // contacts of two particles equal to them (kept when radii / masses are kept)
    // every packed particle is validated on the device as it is packed (ParticleSet::validate,
    // particle_set.cpp:40-58; material ids < count, since they index the force kernel's shared
    // material table; stable ids below the wall keys): free for the host-coupled stepping loop
    // Duplicate ids are screened on the device too: the ids hash into a bitmap of >= 4n bits
    // (id mod 2^k: a permutation of 0..n-1, the usual ids, never collides); only a collision
    // sends the ids through the exact host check.
    CUDA_TRY(cudaMemsetAsync(&ctx->ctl->bad_upload, 0xff, sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(&ctx->ctl->maybe_dup, 0, sizeof(unsigned int), s));
    CUDA_TRY(cudaMemsetAsync(&ctx->ctl->preint_phase, 0xff, sizeof(unsigned long long), s));  // new state
    if (r.ids) CUDA_TRY(cudaMemsetAsync(ctx->idmap, 0, (static_cast<size_t>(ctx->idmask) + 1) / 8, s));
    const PackCheck chk{ctx->ctl, static_cast<uint32_t>(ctx->materials.size()), r.ids ? ctx->idmap : nullptr, ctx->idmask};
    launch_pack_state(ctx->state[buf], r, static_cast<uint32_t>(n), true, s, &chk,
                      r.rad && r.mass ? &ctx->ctl->r_ref : nullptr);
    struct { unsigned long long bad; unsigned int dup; } flags{~0ull, 0u};
    CUDA_TRY(cudaMemcpyAsync(&flags.bad, &ctx->ctl->bad_upload, sizeof(flags.bad), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&flags.dup, &ctx->ctl->maybe_dup, sizeof(flags.dup), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    const unsigned long long bad = flags.bad;
    if (bad == ~0ull && flags.dup) {
        std::string why;
        if (check_unique_ids(p->ids, n, &why) != DEM_OK) {
            ctx->state_invalid = true;
            return set_error(ctx, DEM_ERR_CONFIG, -1, 0, 0, ctx->step_index, why);
        }
    }
    if (bad != ~0ull) {
        // the buffer now holds the rejected particles: no phase may run on it until a valid upload
        ctx->state_invalid = true;
        const uint64_t slot = bad >> 8;
        static const char* const why[] = {"?", "radius must be > 0", "mass must be > 0", "non-finite state",
                                          "bad material", "stable id in the reserved wall-key range (>= 0xFFFFFFC0)"};
        const uint32_t code = static_cast<uint32_t>(bad & 0xff);
        const uint32_t id = p->ids ? p->ids[slot] : 0u;
        char raw[64];
        std::snprintf(raw, sizeof(raw), " (slot %llu, check word 0x%llx)", static_cast<unsigned long long>(slot), bad);
        return set_error(ctx, DEM_ERR_CONFIG, -1, static_cast<uint32_t>(slot), id, ctx->step_index,
                         "particle " + std::to_string(id) + ": " + why[code < 6 ? code : 0] + (code < 6 && code ? "" : raw));
    }
    ctx->state_invalid = false;
    return DEM_OK;
}


int run_phase(dem_ctx* ctx, uint32_t flags, dem_step_metrics* m, bool is_step) {
    if (ctx->n == 0) {
        if (is_step) ++ctx->step_index;
        if (m) { std::memset(m, 0, sizeof(*m)); m->step = ctx->step_index; }
        return DEM_OK;
    }
    const uint64_t pb = ctx->phase_count;
    const int64_t sb = ctx->step_index;
    ++ctx->phase_count;
    if (is_step) ++ctx->step_index;
    if (flags == DEM_PHASE_STEP && ctx->graph[ctx->phase_count & 1]) {
        CUDA_TRY(cudaGraphLaunch(ctx->graph[ctx->phase_count & 1], ctx->stream));
    } else {
        enqueue_phase(ctx, flags, ctx->phase_count, nullptr);
    }
    return collect(ctx, m, pb, sb, is_step);
}

}  // namespace

extern "C" {

int dem_abi_version(void) { return DEM_B200_ABI_VERSION; }

const char* dem_device_kernel_name(int k) {
    return (k >= 0 && k < DEM_DEVICE_KERNEL_COUNT) ? kDeviceKernelNames[k] : "?";
}

int dem_create(const dem_config* cfg, const dem_particles* particles, int device, dem_ctx** out) {
    dem_ctx* ctx = nullptr;
    if (!cfg || !particles || !out) return DEM_ERR_ARGUMENT;
    *out = nullptr;
    std::string why;
    int rc = validate(cfg, particles, &why);
    if (rc == DEM_OK) rc = check_unique_ids(particles->ids, particles->count, &why);
    if (rc != DEM_OK) {
        std::snprintf(g_create_error.message, sizeof(g_create_error.message), "%s", why.c_str());
        g_create_error.code = rc;
        return rc;
    }
    double r_max = 0.0;
    for (uint64_t i = 0; i < particles->count; ++i) r_max = std::max(r_max, particles->radii[i]);
    dem_grid grid{};
    rc = make_grid(cfg, r_max, &grid, &why);
    if (rc != DEM_OK) {
        std::snprintf(g_create_error.message, sizeof(g_create_error.message), "%s", why.c_str());
        g_create_error.code = rc;
        return rc;
    }
    ctx = new (std::nothrow) dem_ctx();
    if (!ctx) return DEM_ERR_ARGUMENT;
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
        std::snprintf(g_create_error.message, sizeof(g_create_error.message), "CUDA device %d unavailable", device);
        g_create_error.code = DEM_ERR_CUDA;
        free_ctx(ctx);
        return DEM_ERR_CUDA;
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    init_device_attributes();
    ctx->dt = cfg->dt;
    for (int a = 0; a < 3; ++a) {
        ctx->gravity[a] = cfg->gravity[a];
        ctx->domain_min[a] = cfg->domain_min[a];
        ctx->domain_max[a] = cfg->domain_max[a];
    }
    ctx->materials.assign(cfg->materials, cfg->materials + cfg->material_count);
    if (cfg->pair_restitution)
        ctx->pair_rest.assign(cfg->pair_restitution, cfg->pair_restitution + cfg->material_count * cfg->material_count);
    if (cfg->rect_wall_count) ctx->rects.assign(cfg->rect_walls, cfg->rect_walls + cfg->rect_wall_count);
    if (cfg->line_wall_count) ctx->lines.assign(cfg->line_walls, cfg->line_walls + cfg->line_wall_count);
    ctx->grid_cell_size = cfg->grid_cell_size;
    ctx->K = cfg->contact_capacity;
    ctx->collide_variant = cfg->collide_variant;
    ctx->grid = grid;
    set_periodic(ctx, cfg);
    ctx->precision = cfg->precision;
    ctx->n = particles->count;
    ctx->kz0 = 0;
    ctx->nz_loc = grid.nz;
    ctx->M = static_cast<uint32_t>(static_cast<int64_t>(grid.nx) * grid.ny * grid.nz);
    rc = allocate(ctx);
    if (rc == DEM_OK) rc = upload_tables(ctx);
    if (rc == DEM_OK) {
        DevCtl init{};
        init.err_key = kNoError;
        for (auto& s : init.err_sid) s = kNoError;
        init.preint_phase = ~0ull;
        init.deferred[0] = init.deferred[1] = ~0ull;
        // on the context's stream: a legacy cudaMemcpy from pageable memory may complete its DMA after
        // later work on this non-blocking stream (upload_state's check-word reset)
        if (cudaMemcpyAsync(ctx->ctl, &init, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = DEM_ERR_CUDA;
    }
    if (rc == DEM_OK) rc = upload_state(ctx, particles, 0);
    if (rc == DEM_OK) rc = build_graphs(ctx);
    // priming force pass, pipeline.cpp:83
    if (rc == DEM_OK) rc = run_phase(ctx, DEM_PHASE_GRAVITY | DEM_PHASE_PP | DEM_PHASE_RECT | DEM_PHASE_LINE, nullptr, false);
    if (rc != DEM_OK) {
        g_create_error = ctx->last_error;
        g_create_error.code = rc;
        free_ctx(ctx);
        return rc;
    }
    *out = ctx;
    return DEM_OK;
}

int dem_clone(const dem_ctx* src, dem_ctx** out) {
    if (!src || !out || src->slab) return DEM_ERR_ARGUMENT;
    cudaSetDevice(src->device);
    SETTLE(const_cast<dem_ctx*>(src));
    dem_ctx* ctx = new (std::nothrow) dem_ctx();
    if (!ctx) return DEM_ERR_ARGUMENT;
    ctx->device = src->device;
    cudaSetDevice(ctx->device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) { free_ctx(ctx); return DEM_ERR_CUDA; }
    ctx->num_sms = src->num_sms;
    init_device_attributes();
    ctx->dt = src->dt;
    std::memcpy(ctx->gravity, src->gravity, sizeof(ctx->gravity));
    std::memcpy(ctx->domain_min, src->domain_min, sizeof(ctx->domain_min));
    std::memcpy(ctx->domain_max, src->domain_max, sizeof(ctx->domain_max));
    ctx->materials = src->materials; ctx->pair_rest = src->pair_rest;
    ctx->rects = src->rects; ctx->lines = src->lines;
    ctx->grid_cell_size = src->grid_cell_size; ctx->K = src->K; ctx->collide_variant = src->collide_variant;
    ctx->grid = src->grid; ctx->n = src->n; ctx->M = src->M;
    ctx->periodic = src->periodic; ctx->shear_rate = src->shear_rate; ctx->precision = src->precision;
    std::memcpy(ctx->cell_extent, src->cell_extent, sizeof(ctx->cell_extent));
    ctx->kz0 = src->kz0; ctx->nz_loc = src->nz_loc;
    int rc = allocate(ctx);
    if (rc == DEM_OK) {
        // allocations were made in the same order with the same sizes: copy pairwise
        size_t k = 0;
        auto copy = [&](void* dst, const void* s, size_t bytes) {
            if (rc == DEM_OK && cudaMemcpyAsync(dst, s, bytes, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess) rc = DEM_ERR_CUDA;
        };
        const uint64_t n = src->n;
        for (int b = 0; b < 2; ++b) {
            copy(ctx->state[b].pos_r, src->state[b].pos_r, n * sizeof(double4));
            copy(ctx->state[b].vel_m, src->state[b].vel_m, n * sizeof(double4));
            copy(ctx->state[b].omg, src->state[b].omg, n * sizeof(double4));
            copy(ctx->state[b].idm, src->state[b].idm, n * sizeof(uint2));
            copy(ctx->hist[b].pos, src->hist[b].pos, n * sizeof(uint32_t));
            copy(ctx->hist[b].cnt, src->hist[b].cnt, n * sizeof(uint32_t));
            copy(ctx->hist[b].key, src->hist[b].key, src->cap * sizeof(uint32_t));
            copy(ctx->hist[b].dt, src->hist[b].dt, 3 * src->cap * sizeof(double));
        }
        copy(ctx->ft, src->ft, 6 * n * sizeof(double));
        copy(ctx->skey, src->skey, n * sizeof(uint32_t));
        copy(ctx->cstart, src->cstart, (static_cast<size_t>(src->M) + 1) * sizeof(uint32_t));
        copy(ctx->prev_slot, src->prev_slot, n * sizeof(uint32_t));
        copy(ctx->prev_row, src->prev_row, n * sizeof(uint2));
        copy(ctx->pair_i, src->pair_i, src->cap * sizeof(uint32_t));
        copy(ctx->pair_j, src->pair_j, src->cap * sizeof(uint32_t));
        copy(ctx->ctl, src->ctl, sizeof(DevCtl));
        if (rc == DEM_OK && cudaMemsetAsync(&ctx->ctl->preint_phase, 0xff, sizeof(unsigned long long), ctx->stream) != cudaSuccess)
            rc = DEM_ERR_CUDA;  // the pre-integrated state is not copied: the clone integrates from its state
        copy(ctx->d_pairs, src->d_pairs, kMaxMaterials * kMaxMaterials * sizeof(MatPairH));
        copy(ctx->d_rects, src->d_rects, kMaxWalls * sizeof(RectW));
        copy(ctx->d_lines, src->d_lines, kMaxWalls * sizeof(LineW));
        (void)k;
        if (rc == DEM_OK && cudaStreamSynchronize(ctx->stream) != cudaSuccess) rc = DEM_ERR_CUDA;
    }
    ctx->phase_count = src->phase_count;
    ctx->replaced_at = src->replaced_at;
    ctx->state_invalid = src->state_invalid;
    ctx->step_index = src->step_index;
    ctx->last_error = src->last_error;
    if (rc == DEM_OK) rc = build_graphs(ctx);
    if (rc != DEM_OK) { free_ctx(ctx); return rc; }
    *out = ctx;
    return DEM_OK;
}

void dem_destroy(dem_ctx* ctx) { free_ctx(ctx); }

int dem_step(dem_ctx* ctx, int nsteps, dem_step_metrics* last) {
    if (!ctx || nsteps < 0) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    REQUIRE_STATE(ctx);
    if (ctx->shard) {  // host-free sharded steps: every rank's process (or thread) calls this
        const int rc = dem_shard_launch(ctx, nsteps);
        return rc != DEM_OK ? rc : dem_shard_wait(ctx, last);
    }
    if (ctx->n == 0) {
        ctx->step_index += nsteps;
        if (last) { std::memset(last, 0, sizeof(*last)); last->step = ctx->step_index; }
        return DEM_OK;
    }
    const uint64_t pb = ctx->phase_count;
    const int64_t sb = ctx->step_index;
    for (int k = 0; k < nsteps; ++k) {
        ++ctx->phase_count;
        ++ctx->step_index;
        CUDA_TRY(cudaGraphLaunch(ctx->graph[ctx->phase_count & 1], ctx->stream));
    }
    return collect(ctx, last, pb, sb, true);
}

int dem_step_async(dem_ctx* ctx, int nsteps) {
    if (!ctx || nsteps < 0 || ctx->slab) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    REQUIRE_STATE(ctx);
    if (ctx->n == 0) {
        ctx->step_index += nsteps;
        return DEM_OK;
    }
    if (!ctx->inflight) {
        ctx->inflight = true;
        ctx->inflight_pb = ctx->phase_count;
        ctx->inflight_sb = ctx->step_index;
    }
    for (int k = 0; k < nsteps; ++k) {
        ++ctx->phase_count;
        ++ctx->step_index;
        CUDA_TRY(cudaGraphLaunch(ctx->graph_async[ctx->phase_count & 1], ctx->stream));
    }
    return DEM_OK;
}

int dem_sync(dem_ctx* ctx, dem_step_metrics* last) {
    if (!ctx) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    const int rc = settle(ctx);
    if (last) *last = ctx->async_last;
    return rc;
}

int dem_force_phase(dem_ctx* ctx, uint32_t flags, dem_step_metrics* m) {
    if (!ctx || (flags & ~static_cast<uint32_t>(DEM_PHASE_STEP))) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    REQUIRE_STATE(ctx);
    return run_phase(ctx, flags, m, flags == DEM_PHASE_STEP);
}

int dem_set_collide_variant(dem_ctx* ctx, int variant) {
    if (!ctx || (variant != 0 && variant != 1)) return DEM_ERR_ARGUMENT;
    if ((ctx->periodic || ctx->precision) && variant == 0)
        return set_error(ctx, DEM_ERR_CONFIG, -1, 0, 0, ctx->step_index, "periodic boxes and the fp32 mode run the two_phase collide variant");
    if (ctx->collide_variant == variant) return DEM_OK;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    ctx->collide_variant = variant;
    cudaSetDevice(ctx->device);
    return ctx->slab ? DEM_OK : build_graphs(ctx);  // step graphs embed the Collide kernels
}

uint64_t dem_size(const dem_ctx* ctx) { return ctx ? ctx->n : 0; }
int64_t dem_step_index(const dem_ctx* ctx) { return ctx ? ctx->step_index : 0; }
uint64_t dem_device_bytes(const dem_ctx* ctx) { return ctx ? ctx->device_bytes : 0; }
int dem_kernels_per_step(const dem_ctx*) { return DEM_DEVICE_KERNEL_COUNT; }

int dem_get_particles(dem_ctx* ctx, dem_particles* out) {
    if (!ctx || !out || out->count != ctx->n) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    const uint64_t n = ctx->n;
    if (!n) return settle(ctx);
    int rc = ensure_raw(ctx, n);
    if (rc != DEM_OK) return rc;
    const RawState r = raw_view(ctx, n);
    cudaStream_t s = ctx->stream;
    // After dem_step_async the last step's state is final once its k_reorder has run: the
    // readback goes on the side stream from there and overlaps the step's detection and forces.
    const bool overlap = ctx->inflight && !ctx->slab;
    if (overlap) {
        if (!ctx->side) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        s = ctx->side;
        CUDA_TRY(cudaStreamWaitEvent(s, ctx->ev_state[ctx->phase_count & 1], 0));
    } else {
        SETTLE(ctx);
    }
    launch_pack_state(ctx->state[state_cur(ctx)], r, static_cast<uint32_t>(n), false, s);
    if (out->positions) CUDA_TRY(cudaMemcpyAsync(out->positions, r.pos, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out->velocities) CUDA_TRY(cudaMemcpyAsync(out->velocities, r.vel, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out->angular_velocities) CUDA_TRY(cudaMemcpyAsync(out->angular_velocities, r.omg, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out->radii) CUDA_TRY(cudaMemcpyAsync(out->radii, r.rad, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out->masses) CUDA_TRY(cudaMemcpyAsync(out->masses, r.mass, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out->ids) CUDA_TRY(cudaMemcpyAsync(out->ids, r.ids, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    if (out->material_ids) CUDA_TRY(cudaMemcpyAsync(out->material_ids, r.mat, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    rc = overlap ? settle(ctx) : DEM_OK;  // the step's own completion and error check
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    return rc;
}

int dem_set_particles(dem_ctx* ctx, const dem_particles* in) {
    if (!ctx || !in || in->count != ctx->n) return DEM_ERR_ARGUMENT;
    if (!in->positions || !in->velocities || !in->angular_velocities) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    ctx->replaced_at = ctx->phase_count;  // the binning no longer matches the state (traces)
    return upload_state(ctx, in, state_cur(ctx));
}

int dem_get_forces(dem_ctx* ctx, double* force, double* torque) {
    if (!ctx) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    const uint64_t n = ctx->n, fs = ft_stride(ctx);
    if (!n) return DEM_OK;
    int rc = ensure_raw(ctx, n);
    if (rc != DEM_OK) return rc;
    double* f = ctx->raw_d;           // 6n doubles of staging: F[3n] | T[3n]
    double* t = ctx->raw_d + 3 * n;
    launch_ft_layout(ctx->ft, static_cast<uint32_t>(fs), f, t, static_cast<uint32_t>(n), true, ctx->stream);
    if (force) CUDA_TRY(cudaMemcpyAsync(force, f, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (torque) CUDA_TRY(cudaMemcpyAsync(torque, t, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaGetLastError());
    return DEM_OK;
}

int dem_set_forces(dem_ctx* ctx, const double* force, const double* torque) {
    if (!ctx || !force || !torque) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    const uint64_t n = ctx->n, fs = ft_stride(ctx);
    if (!n) return DEM_OK;
    int rc = ensure_raw(ctx, n);
    if (rc != DEM_OK) return rc;
    double* f = ctx->raw_d;
    double* t = ctx->raw_d + 3 * n;
    CUDA_TRY(cudaMemcpyAsync(f, force, 3 * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(t, torque, 3 * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    launch_ft_layout(ctx->ft, static_cast<uint32_t>(fs), f, t, static_cast<uint32_t>(n), false, ctx->stream);
    CUDA_TRY(cudaMemsetAsync(&ctx->ctl->preint_phase, 0xff, sizeof(unsigned long long), ctx->stream));  // new forces
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaGetLastError());
    return DEM_OK;
}

int dem_get_grid(const dem_ctx* ctx, dem_grid* out) {
    if (!ctx || !out) return DEM_ERR_ARGUMENT;
    *out = ctx->grid;
    return DEM_OK;
}

int dem_get_periodic_box(dem_ctx* ctx, double cell_extent[3], double* shear_offset) {
    if (!ctx) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    if (cell_extent) for (int a = 0; a < 3; ++a) cell_extent[a] = ctx->cell_extent[a];
    if (shear_offset) {
        cudaSetDevice(ctx->device);
        CUDA_TRY(cudaMemcpy(shear_offset, &ctx->ctl->le_delta, sizeof(double), cudaMemcpyDeviceToHost));
    }
    return DEM_OK;
}

int dem_get_order(dem_ctx* ctx, uint32_t* sorted_keys, uint32_t* permutation) {
    if (!ctx) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    const uint64_t n = ctx->n;
    if (n && sorted_keys) CUDA_TRY(cudaMemcpyAsync(sorted_keys, ctx->skey, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    if (n && permutation) CUDA_TRY(cudaMemcpyAsync(permutation, ctx->prev_slot, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DEM_OK;
}

int dem_set_contacts(dem_ctx* ctx, const uint32_t* owner_slot, const int32_t* partner, const double* delta_t,
                     int64_t count) {
    if (!ctx || ctx->slab || count < 0 || (count && (!owner_slot || !partner || !delta_t))) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    const uint64_t n = ctx->n;
    if (n == 0) return count ? DEM_ERR_ARGUMENT : DEM_OK;
    const uint32_t K = static_cast<uint32_t>(ctx->K);
    // stable ids of the current slots: the history keys partners by id (walls by their code)
    std::vector<uint2> idm(n);
    CUDA_TRY(cudaMemcpy(idm.data(), ctx->state[state_cur(ctx)].idm, n * sizeof(uint2), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> cnt(n, 0), pos(n, 0);
    for (int64_t k = 0; k < count; ++k) {
        if (owner_slot[k] >= n) return DEM_ERR_ARGUMENT;
        if (partner[k] >= 0 && static_cast<uint64_t>(partner[k]) >= n) return DEM_ERR_ARGUMENT;
        if (++cnt[owner_slot[k]] > K) return DEM_ERR_ARGUMENT;
    }
    // tile-compacted layout: owner i's row inside tile i/32's region, slot order
    for (uint64_t t0 = 0; t0 < n; t0 += 32) {
        uint32_t q = static_cast<uint32_t>(t0 * K);
        for (uint64_t i = t0; i < std::min<uint64_t>(n, t0 + 32); ++i) { pos[i] = q; q += cnt[i]; }
    }
    const size_t cap = ctx->cap;
    std::vector<uint32_t> key(cap, 0), pj(cap, 0), fill(n, 0);
    std::vector<double> dt(3 * cap, 0.0);
    for (int64_t k = 0; k < count; ++k) {
        const uint32_t i = owner_slot[k];
        const uint32_t q = pos[i] + fill[i]++;
        const uint32_t kk = partner[k] >= 0 ? idm[partner[k]].x : static_cast<uint32_t>(partner[k]);
        for (uint32_t r = pos[i]; r < q; ++r)
            if (key[r] == kk) return DEM_ERR_ARGUMENT;  // one entry per partner (contact_table.cpp:15-35)
        key[q] = kk;
        pj[q] = static_cast<uint32_t>(partner[k]);
        for (int a = 0; a < 3; ++a) dt[a * cap + q] = delta_t[3 * k + a];
    }
    const HistBuf& h = ctx->hist[hist_cur(ctx)];
    // on the context's (non-blocking) stream, so the next phase is ordered after the DMA
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaMemcpyAsync(h.pos, pos.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(h.cnt, cnt.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(h.key, key.data(), cap * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(h.dt, dt.data(), 3 * cap * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->pair_j, pj.data(), cap * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return DEM_OK;
}

int64_t dem_get_contacts(dem_ctx* ctx, uint32_t* owner_slot, int32_t* partner, double* delta_t, int64_t cap) {
    if (!ctx) return -DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    if (const int rc_ = settle(ctx)) return -rc_;
    const uint64_t n = ctx->n;
    if (n == 0) return 0;
    const HistBuf& h = ctx->hist[hist_cur(ctx)];
    std::vector<uint32_t> pos(n), cnt(n);
    if (cudaMemcpy(pos.data(), h.pos, n * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) return -DEM_ERR_CUDA;
    if (cudaMemcpy(cnt.data(), h.cnt, n * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) return -DEM_ERR_CUDA;
    int64_t C = 0;
    for (uint64_t i = 0; i < n; ++i) C += cnt[i];
    if (cap <= 0 || !owner_slot || !partner || !delta_t) return C;
    // tile regions -> dense list in slot order (per-owner accumulation order)
    std::vector<uint32_t> pj(ctx->cap);
    std::vector<double> dt(3 * ctx->cap);
    if (cudaMemcpy(pj.data(), ctx->pair_j, ctx->cap * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) return -DEM_ERR_CUDA;
    if (cudaMemcpy(dt.data(), h.dt, 3 * ctx->cap * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) return -DEM_ERR_CUDA;
    int64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t q = pos[i]; q < pos[i] + cnt[i] && k < cap; ++q, ++k) {
            owner_slot[k] = static_cast<uint32_t>(i);
            partner[k] = static_cast<int32_t>(pj[q]);  // wall codes ~w == -(w+1) (contact_table.hpp:35)
            for (int a = 0; a < 3; ++a) delta_t[3 * k + a] = dt[a * ctx->cap + q];
        }
    return C;
}

int64_t dem_get_traces(dem_ctx* ctx, uint64_t* offsets, dem_trace_event* events, int64_t capacity) {
    if (!ctx || ctx->slab || ctx->periodic || ctx->phase_count == 0 || ctx->replaced_at == ctx->phase_count) return -DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    if (const int rc_ = settle(ctx)) return -rc_;
    const uint64_t n = ctx->n;
    if (n == 0) {
        if (offsets) offsets[0] = 0;
        return 0;
    }
    const StepParams p = make_params(ctx, DEM_PHASE_PP);
    const PhaseBufs b = make_bufs(ctx, ctx->phase_count);
    cudaStream_t s = ctx->stream;
    uint32_t* d_count = nullptr;
    unsigned long long* d_off = nullptr;
    int2* d_ev = nullptr;
    int64_t result = -DEM_ERR_CUDA;
    std::vector<uint32_t> cnt(n);
    std::vector<unsigned long long> off(n + 1);
    do {
        if (cudaMalloc(&d_count, n * sizeof(uint32_t)) != cudaSuccess) break;
        launch_trace(p, b, nullptr, nullptr, d_count, s);
        if (cudaMemcpyAsync(cnt.data(), d_count, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s) != cudaSuccess) break;
        if (cudaStreamSynchronize(s) != cudaSuccess) break;
        off[0] = 0;
        for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + cnt[i];
        const uint64_t total = off[n];
        if (offsets) std::memcpy(offsets, off.data(), (n + 1) * sizeof(uint64_t));
        result = static_cast<int64_t>(total);
        if (!events || capacity < static_cast<int64_t>(total) || total == 0) break;
        result = -DEM_ERR_CUDA;
        if (cudaMalloc(&d_off, (n + 1) * sizeof(unsigned long long)) != cudaSuccess) break;
        if (cudaMalloc(&d_ev, total * sizeof(int2)) != cudaSuccess) break;
        if (cudaMemcpyAsync(d_off, off.data(), (n + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice, s) != cudaSuccess) break;
        launch_trace(p, b, d_off, d_ev, nullptr, s);
        static_assert(sizeof(dem_trace_event) == sizeof(int2), "event layout");
        if (cudaMemcpyAsync(events, d_ev, total * sizeof(int2), cudaMemcpyDeviceToHost, s) != cudaSuccess) break;
        if (cudaStreamSynchronize(s) != cudaSuccess) break;
        result = static_cast<int64_t>(total);
    } while (false);
    cudaFree(d_count);
    cudaFree(d_off);
    cudaFree(d_ev);
    if (cudaGetLastError() != cudaSuccess) result = -DEM_ERR_CUDA;
    if (result == -DEM_ERR_CUDA) set_error(ctx, DEM_ERR_CUDA, -1, 0, 0, ctx->step_index, "CUDA failure in dem_get_traces");
    return result;
}

int dem_last_error(const dem_ctx* ctx, dem_error* out) {
    if (!out) return DEM_ERR_ARGUMENT;
    *out = ctx ? ctx->last_error : g_create_error;
    return DEM_OK;
}

namespace {
int shard_collect(dem_ctx* c, dem_step_metrics* m);  // host-free sharded stepping, below
}  // namespace

int dem_time_steps(dem_ctx* ctx, int nsteps, size_t flush_bytes, float* step_ms, dem_step_metrics* last) {
    if (!ctx || nsteps < 0 || (nsteps && !step_ms)) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    REQUIRE_STATE(ctx);
    if (flush_bytes && flush_bytes != ctx->flush_bytes) {
        if (ctx->flush_buf) cudaFree(ctx->flush_buf);
        ctx->flush_buf = nullptr;
        CUDA_TRY(cudaMalloc(&ctx->flush_buf, flush_bytes));
        ctx->flush_bytes = flush_bytes;
    }
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(nsteps));
    for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
    const uint64_t pb = ctx->phase_count;
    const int64_t sb = ctx->step_index;
    if (ctx->shard && (!ctx->primed || ctx->launched)) return DEM_ERR_ARGUMENT;  // dem_step first
    if (ctx->shard) { ctx->launch_pb = pb; ctx->launch_sb = sb; ctx->launched = true; }
    for (int k = 0; k < nsteps; ++k) {
        if (flush_bytes) launch_flush(ctx->flush_buf, flush_bytes, ctx->stream);
        CUDA_TRY(cudaEventRecord(ev[2 * k], ctx->stream));
        if (ctx->shard) {
            // a sharded step includes the waits for the neighbours' records
            CUDA_TRY(cudaGraphLaunch(ctx->shard_graph[ctx->shist], ctx->stream));
            ctx->shist ^= 1;
        } else {
            CUDA_TRY(cudaGraphLaunch(ctx->graph[(ctx->phase_count + 1) & 1], ctx->stream));
        }
        ++ctx->phase_count;
        ++ctx->step_index;
        CUDA_TRY(cudaEventRecord(ev[2 * k + 1], ctx->stream));
    }
    int rc = ctx->shard ? shard_collect(ctx, last) : collect(ctx, last, pb, sb, true);
    for (int k = 0; k < nsteps; ++k) cudaEventElapsedTime(&step_ms[k], ev[2 * k], ev[2 * k + 1]);
    for (auto& e : ev) cudaEventDestroy(e);
    return rc;
}

int dem_profile_step(dem_ctx* ctx, size_t flush_bytes, dem_step_metrics* m) {
    if (!ctx || !m) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    SETTLE(ctx);
    REQUIRE_STATE(ctx);
    if (flush_bytes && flush_bytes != ctx->flush_bytes) {
        if (ctx->flush_buf) cudaFree(ctx->flush_buf);
        ctx->flush_buf = nullptr;
        CUDA_TRY(cudaMalloc(&ctx->flush_buf, flush_bytes));
        ctx->flush_bytes = flush_bytes;
    }
    cudaEvent_t ev[DEM_DEVICE_KERNEL_COUNT + 1];
    for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
    if (flush_bytes) launch_flush(ctx->flush_buf, flush_bytes, ctx->stream);
    const uint64_t pb = ctx->phase_count;
    const int64_t sb = ctx->step_index;
    ++ctx->phase_count;
    ++ctx->step_index;
    enqueue_phase(ctx, DEM_PHASE_STEP, ctx->phase_count, ev);
    int rc = collect(ctx, m, pb, sb, true);
    for (int k = 0; k < DEM_DEVICE_KERNEL_COUNT; ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
        m->device_kernel_ms[k] = ms;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return rc;
}

// ---------------------------------------------------------------------------------------------
// Slab decomposition. The host moves records between neighbours
// (NCCL over NVLink in production, gloo / loopback in tests); these calls only touch device
// memory they are given.

namespace {

SlabBufs make_slab(const dem_ctx* c, void* send_lo, void* send_hi, uint64_t cap_records) {
    SlabBufs s{};
    s.X = c->state[c->sstate];
    s.Y = c->state[c->sstate ^ 1];
    s.ft = c->ft;
    s.ft_stride = static_cast<uint32_t>(c->n_cap);
    s.H_old = c->hist[c->shist];
    s.hrm_pos = c->hrm_pos;
    s.hrm_cnt = c->hrm_cnt;
    s.n_x = static_cast<uint32_t>(c->n);
    s.counters = c->counters;
    s.send_lo = static_cast<uint8_t*>(send_lo);
    s.send_hi = static_cast<uint8_t*>(send_hi);
    s.cap_send = static_cast<uint32_t>(std::min<uint64_t>(cap_records, 0xffffffffull));
    s.rec_bytes = c->rec_bytes;
    s.rec_dt_off = c->rec_dt_off;
    s.ghost_bytes = c->ghost_bytes;
    s.z_lo = c->z_lo;
    s.z_hi = c->z_hi;
    s.imp_base = c->tile_pairs;
    s.hcap = c->cap;
    s.K = static_cast<uint32_t>(c->K);
    s.ctl = c->ctl;
    return s;
}

int read_counters(dem_ctx* ctx) {
    CUDA_TRY(cudaMemcpyAsync(ctx->h_counters, ctx->counters, 8 * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaGetLastError());
    return DEM_OK;
}

}  // namespace

int dem_create_slab(const dem_config* cfg, const dem_particles* owned, int device, int32_t z_lo, int32_t z_hi,
                    uint64_t capacity, dem_ctx** out) {
    if (!cfg || !owned || !out) return DEM_ERR_ARGUMENT;
    *out = nullptr;
    std::string why;
    int rc = validate(cfg, owned, &why);
    if (rc == DEM_OK && !(cfg->grid_cell_size > 0.0)) {
        why = "grid.cell_size: a slab context needs the global cell size (2 r_max (1 + 1e-6) of all ranks)";
        rc = DEM_ERR_CONFIG;
    }
    dem_grid grid{};
    if (rc == DEM_OK) rc = make_grid(cfg, 0.0, &grid, &why);
    if (rc == DEM_OK && !(z_lo >= 0 && z_lo < z_hi && z_hi <= grid.nz)) {
        why = "slab planes must satisfy 0 <= z_lo < z_hi <= nz";
        rc = DEM_ERR_CONFIG;
    }
    if (rc != DEM_OK) {
        std::snprintf(g_create_error.message, sizeof(g_create_error.message), "%s", why.c_str());
        g_create_error.code = rc;
        return rc;
    }
    dem_ctx* ctx = new (std::nothrow) dem_ctx();
    if (!ctx) return DEM_ERR_ARGUMENT;
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
        free_ctx(ctx);
        return DEM_ERR_CUDA;
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    init_device_attributes();
    ctx->dt = cfg->dt;
    for (int a = 0; a < 3; ++a) {
        ctx->gravity[a] = cfg->gravity[a];
        ctx->domain_min[a] = cfg->domain_min[a];
        ctx->domain_max[a] = cfg->domain_max[a];
    }
    ctx->materials.assign(cfg->materials, cfg->materials + cfg->material_count);
    if (cfg->pair_restitution)
        ctx->pair_rest.assign(cfg->pair_restitution, cfg->pair_restitution + cfg->material_count * cfg->material_count);
    if (cfg->rect_wall_count) ctx->rects.assign(cfg->rect_walls, cfg->rect_walls + cfg->rect_wall_count);
    if (cfg->line_wall_count) ctx->lines.assign(cfg->line_walls, cfg->line_walls + cfg->line_wall_count);
    ctx->grid_cell_size = cfg->grid_cell_size;
    ctx->K = cfg->contact_capacity;
    ctx->collide_variant = cfg->collide_variant;
    ctx->grid = grid;
    set_periodic(ctx, cfg);
    ctx->precision = cfg->precision;
    ctx->slab = true;
    ctx->z_lo = z_lo;
    ctx->z_hi = z_hi;
    // keyed planes: the slab plus one ghost plane each side (beyond the grid only if z is periodic,
    // where the neighbours form a ring)
    const bool zring = (cfg->periodic & 4u) != 0;
    ctx->kz0 = zring ? z_lo - 1 : std::max(z_lo - 1, 0);
    ctx->nz_loc = (zring ? z_hi + 1 : std::min(z_hi + 1, grid.nz)) - ctx->kz0;
    ctx->M = static_cast<uint32_t>(static_cast<int64_t>(grid.nx) * grid.ny * ctx->nz_loc);
    ctx->n = owned->count;
    ctx->n_cap = std::max<uint64_t>(capacity, owned->count) + 32;
    ctx->imp_cap = ctx->n_cap / 4 + 1024;
    const uint32_t keys_bytes = ((4u * ctx->K) + 7u) & ~7u;
    ctx->rec_dt_off = 112u + keys_bytes;
    ctx->rec_bytes = (ctx->rec_dt_off + 24u * ctx->K + 31u) & ~31u;
    ctx->ghost_bytes = 128u;
    ctx->sstate = 0;
    ctx->shist = 0;
    rc = allocate(ctx);
    if (rc == DEM_OK) rc = upload_tables(ctx);
    if (rc == DEM_OK) {
        DevCtl init{};
        init.err_key = kNoError;
        for (auto& s : init.err_sid) s = kNoError;
        init.preint_phase = ~0ull;
        init.deferred[0] = init.deferred[1] = ~0ull;
        // on the context's stream: a legacy cudaMemcpy from pageable memory may complete its DMA after
        // later work on this non-blocking stream (upload_state's check-word reset)
        if (cudaMemcpyAsync(ctx->ctl, &init, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = DEM_ERR_CUDA;
    }
    if (rc == DEM_OK) rc = upload_state(ctx, owned, 0);
    if (rc != DEM_OK) {
        g_create_error = ctx->last_error;
        g_create_error.code = rc;
        free_ctx(ctx);
        return rc;
    }
    *out = ctx;
    return DEM_OK;
}

int dem_slab_record_bytes(const dem_ctx* ctx, uint64_t* migrant_bytes, uint64_t* ghost_bytes) {
    if (!ctx || !ctx->slab) return DEM_ERR_ARGUMENT;
    if (migrant_bytes) *migrant_bytes = ctx->rec_bytes;
    if (ghost_bytes) *ghost_bytes = ctx->ghost_bytes;
    return DEM_OK;
}

uint64_t dem_slab_owned(const dem_ctx* ctx) { return ctx && ctx->slab ? ctx->n_own : 0; }

int dem_slab_migrate(dem_ctx* ctx, int integrate, void* send_lo, void* send_hi, uint64_t cap_records,
                     uint64_t* n_lo, uint64_t* n_hi) {
    if (!ctx || !ctx->slab || ctx->shard || !n_lo || !n_hi) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    CUDA_TRY(cudaMemsetAsync(ctx->counters, 0, 8 * sizeof(uint32_t), ctx->stream));
    const StepParams p = make_params(ctx, 0);
    launch_slab_migrate(p, make_slab(ctx, send_lo, send_hi, cap_records), integrate != 0, ctx->stream);
    // one synchronisation for the record counts and the error word
    CUDA_TRY(cudaMemcpyAsync(ctx->h_counters, ctx->counters, 8 * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(cudaGetLastError());
    const int rc = collect(ctx, nullptr, ctx->phase_count, ctx->step_index, false, true);
    if (rc != DEM_OK) return rc;
    if (ctx->h_counters[4]) return set_error(ctx, DEM_ERR_CAPACITY, -1, 0, 0, ctx->step_index, "slab: migrant send buffer too small");
    ctx->n_own = ctx->h_counters[0];
    ctx->n_asm = ctx->n_own;
    ctx->imp_used = 0;
    ctx->integrated = integrate != 0;
    *n_lo = ctx->h_counters[1];
    *n_hi = ctx->h_counters[2];
    return DEM_OK;
}

int dem_slab_import(dem_ctx* ctx, const void* recs_lo, uint64_t n_lo, const void* recs_hi, uint64_t n_hi) {
    if (!ctx || !ctx->slab || ctx->shard) return DEM_ERR_ARGUMENT;
    if (ctx->n_own + n_lo + n_hi > ctx->n_cap || (ctx->imp_used / ctx->K) + n_lo + n_hi > ctx->imp_cap)
        return set_error(ctx, DEM_ERR_CAPACITY, -1, 0, 0, ctx->step_index, "slab: context capacity exceeded by imports");
    cudaSetDevice(ctx->device);
    const SlabBufs s = make_slab(ctx, nullptr, nullptr, 0);
    launch_slab_import(s, recs_lo, static_cast<uint32_t>(n_lo), static_cast<uint32_t>(ctx->n_own), ctx->imp_used, ctx->stream);
    ctx->n_own += n_lo;
    ctx->imp_used += n_lo * ctx->K;
    launch_slab_import(s, recs_hi, static_cast<uint32_t>(n_hi), static_cast<uint32_t>(ctx->n_own), ctx->imp_used, ctx->stream);
    ctx->n_own += n_hi;
    ctx->imp_used += n_hi * ctx->K;
    ctx->n_asm = ctx->n_own;
    CUDA_TRY(cudaGetLastError());  // stream-ordered: dem_slab_halo follows on the same stream
    return DEM_OK;
}

int dem_slab_halo(dem_ctx* ctx, void* send_lo, void* send_hi, uint64_t cap_records, uint64_t* n_lo, uint64_t* n_hi) {
    if (!ctx || !ctx->slab || ctx->shard || !n_lo || !n_hi) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    CUDA_TRY(cudaMemsetAsync(ctx->counters, 0, 8 * sizeof(uint32_t), ctx->stream));
    const StepParams p = make_params(ctx, 0);
    launch_slab_halo(p, make_slab(ctx, send_lo, send_hi, cap_records), static_cast<uint32_t>(ctx->n_own), ctx->stream);
    int rc = read_counters(ctx);
    if (rc != DEM_OK) return rc;
    if (ctx->h_counters[4]) return set_error(ctx, DEM_ERR_CAPACITY, -1, 0, 0, ctx->step_index, "slab: halo send buffer too small");
    *n_lo = ctx->h_counters[5];
    *n_hi = ctx->h_counters[6];
    return DEM_OK;
}

int dem_slab_ghosts(dem_ctx* ctx, const void* recs_lo, uint64_t n_lo, const void* recs_hi, uint64_t n_hi) {
    if (!ctx || !ctx->slab || ctx->shard) return DEM_ERR_ARGUMENT;
    if (ctx->n_own + n_lo + n_hi > ctx->n_cap)
        return set_error(ctx, DEM_ERR_CAPACITY, -1, 0, 0, ctx->step_index, "slab: context capacity exceeded by ghosts");
    cudaSetDevice(ctx->device);
    const SlabBufs s = make_slab(ctx, nullptr, nullptr, 0);
    launch_slab_ghosts(s, recs_lo, static_cast<uint32_t>(n_lo), static_cast<uint32_t>(ctx->n_own), false, ctx->stream);
    launch_slab_ghosts(s, recs_hi, static_cast<uint32_t>(n_hi), static_cast<uint32_t>(ctx->n_own + n_lo), true, ctx->stream);
    ctx->n_asm = ctx->n_own + n_lo + n_hi;
    CUDA_TRY(cudaGetLastError());  // stream-ordered: dem_slab_force follows on the same stream
    return DEM_OK;
}

int dem_slab_force(dem_ctx* ctx, uint32_t flags, dem_step_metrics* m) {
    if (!ctx || !ctx->slab || ctx->shard) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    flags = (flags & ~static_cast<uint32_t>(DEM_PHASE_INTEGRATE)) | kPhaseSlab;
    const uint64_t pb = ctx->phase_count;
    const int64_t sb = ctx->step_index;
    ++ctx->phase_count;
    if (ctx->integrated) ++ctx->step_index;
    enqueue_phase(ctx, flags, ctx->phase_count, nullptr);
    const int rc = collect(ctx, m, pb, sb, ctx->integrated);
    ctx->integrated = false;
    if (rc != DEM_OK) return rc;
    ctx->n = ctx->n_asm;
    ctx->shist ^= 1;
    return DEM_OK;
}

int dem_ipc_alloc(int device, uint64_t bytes, void** ptr) {
    if (!ptr) return DEM_ERR_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(ptr, bytes ? bytes : 16) != cudaSuccess) return DEM_ERR_CUDA;
    return DEM_OK;
}
int dem_ipc_free(int device, void* ptr) {
    if (cudaSetDevice(device) != cudaSuccess) return DEM_ERR_CUDA;
    return cudaFree(ptr) == cudaSuccess ? DEM_OK : DEM_ERR_CUDA;
}
int dem_ipc_handle(int device, void* ptr, void* handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
    if (!ptr || !handle64) return DEM_ERR_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return DEM_ERR_CUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return DEM_ERR_CUDA;
    std::memcpy(handle64, &h, sizeof(h));
    return DEM_OK;
}
int dem_ipc_open(int device, const void* handle64, void** ptr) {
    if (!handle64 || !ptr) return DEM_ERR_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return DEM_ERR_CUDA;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? DEM_OK : DEM_ERR_CUDA;
}
int dem_ipc_close(int device, void* ptr) {
    if (cudaSetDevice(device) != cudaSuccess) return DEM_ERR_CUDA;
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? DEM_OK : DEM_ERR_CUDA;
}

// ---- host-free sharded stepping --------------------------------------
// dem_create_sharded builds rank `rank` of a z-slab decomposition from the GLOBAL initial set (the
// same partition on every rank); the caller all-gathers the 64-byte inbox handles
// (dem_shard_handle) with whatever it has (NCCL, MPI, torch.distributed) and connects
// (dem_shard_connect), or wires contexts of one process directly (dem_shard_connect_local). Steps
// then run without the host: record counts stay on the device, neighbours store into each other's
// inbox blocks and signal with release flags, and each step is one CUDA graph.
namespace {

using CuWaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
CuWaitFn g_cu_wait = nullptr;
bool g_cu_wait_probed = false;

CuWaitFn cu_stream_wait() {
    if (!g_cu_wait_probed) {
        g_cu_wait_probed = true;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_cu_wait = reinterpret_cast<CuWaitFn>(fn);
    }
    return g_cu_wait;
}

SlabBufs make_shard(const dem_ctx* c, int hpar) {
    SlabBufs s = make_slab(c, nullptr, nullptr, c->cap_rec);
    s.H_old = c->hist[hpar];
    s.dn = c->dn;
    s.inbox = c->inbox;
    s.peer_lo = c->peer[0];
    s.peer_hi = c->peer[1];
    s.n_cap = static_cast<uint32_t>(c->n_cap);
    s.imp_cap = static_cast<uint32_t>(c->imp_cap);
    return s;
}

int shard_wait(dem_ctx* c, const SlabBufs& s, uint32_t kind) {
    if (c->stream_wait) {
        CuWaitFn w = cu_stream_wait();
        for (uint32_t side = 0; side < 2; ++side) {
            if (!c->peer[side]) continue;
            const CUdeviceptr f = reinterpret_cast<CUdeviceptr>(c->inbox + 4 * (2 * kind + side));
            if (!w || w(reinterpret_cast<CUstream>(c->stream), f, 1u, CU_STREAM_WAIT_VALUE_EQ) != CUDA_SUCCESS)
                return DEM_ERR_CUDA;
        }
        return DEM_OK;
    }
    launch_shard_wait(s, kind, c->stream);
    return DEM_OK;
}

// One force phase of the sharded step, history parity hpar (hist[hpar] -> hist[hpar ^ 1]):
// migrate -> post -> wait -> import -> halo -> post -> wait -> ghosts -> the 7 force-phase kernels
// over the device-resident slot count.
int enqueue_shard_phase(dem_ctx* c, bool integrate, uint32_t flags, int hpar) {
    dem_ctx* const ctx = c;  // CUDA_TRY reports into ctx
    const SlabBufs s = make_shard(c, hpar);
    StepParams p = make_params(c, 0);
    cudaStream_t st = c->stream;
    CUDA_TRY(cudaMemsetAsync(c->counters, 0, 8 * sizeof(uint32_t), st));
    launch_shard_migrate(p, s, integrate, st);
    launch_shard_post(s, 0, st);
    int rc = shard_wait(c, s, 0);
    if (rc != DEM_OK) return rc;
    launch_shard_import(s, st);
    launch_shard_halo(p, s, st);
    launch_shard_post(s, 1, st);
    rc = shard_wait(c, s, 1);
    if (rc != DEM_OK) return rc;
    launch_shard_ghosts(s, st);
    // the force phase: bins Y into X, detects and forces for owned slots; n from dn[0]
    p = make_params(c, (flags & ~static_cast<uint32_t>(DEM_PHASE_INTEGRATE)) | kPhaseSlab);
    p.n = static_cast<uint32_t>(c->n_cap);
    PhaseBufs b = make_bufs(c, 0);
    b.old_h = c->hist[hpar];
    b.old_h.pos = c->hrm_pos;
    b.old_h.cnt = c->hrm_cnt;
    b.cur_h = c->hist[hpar ^ 1];
    b.n_tiles_det = detect_tiles(static_cast<uint32_t>(c->n_cap));
    b.dn = c->dn;
    launch_phase_begin(p, b, st);
    launch_integrate_hash(p, b, false, st);
    launch_scan_cells(p, b, st);
    launch_scatter(p, b, st);
    launch_reorder(p, b, st);
    launch_detect(p, b, st);
    launch_force_reduce(p, b, st);
    CUDA_TRY(cudaGetLastError());
    return DEM_OK;
}

int build_shard_graphs(dem_ctx* c) {
    dem_ctx* const ctx = c;  // CUDA_TRY reports into ctx
    for (int par = 0; par < 2; ++par) {
        cudaGraphExec_t& ge = c->shard_graph[par];
        if (ge) { cudaGraphExecDestroy(ge); ge = nullptr; }
        cudaGraph_t g;
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue_shard_phase(c, true, DEM_PHASE_STEP, par);
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (rc != DEM_OK || e != cudaSuccess) {
            cudaGetLastError();
            if (e == cudaSuccess) cudaGraphDestroy(g);
            return DEM_ERR_CUDA;
        }
        const cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) { cudaGetLastError(); return DEM_ERR_CUDA; }
    }
    return DEM_OK;
}

// rank r's slab of the global set: whole cell planes along z, balanced by particle count
// (slab.py's global_grid / cell_planes / slab_bounds, the same arithmetic)
int shard_partition(const dem_config* cfg, const dem_particles* all, int rank, int nranks, double* h_out,
                    int32_t* z_lo, int32_t* z_hi, std::vector<uint64_t>* owned, uint64_t* ghosts, uint64_t* cap_rec,
                    std::string* why) {
    double r_max = 0.0;
    for (uint64_t i = 0; i < all->count; ++i) r_max = std::max(r_max, all->radii[i]);
    dem_grid g{};
    int rc = make_grid(cfg, r_max, &g, why);
    if (rc != DEM_OK) return rc;
    const double ez = cfg->domain_max[2] - cfg->domain_min[2];
    const double inv_z = (cfg->periodic & 4u) ? 1.0 / (ez / g.nz) : 1.0 / g.cell_size;
    if (nranks > g.nz) { *why = std::to_string(nranks) + " slabs need at least as many cell planes (grid has " + std::to_string(g.nz) + ")"; return DEM_ERR_CONFIG; }
    std::vector<int> plane(all->count);
    std::vector<double> hist(g.nz, 0.0);
    for (uint64_t i = 0; i < all->count; ++i) {
        double f = std::floor((all->positions[3 * i + 2] - cfg->domain_min[2]) * inv_z);
        if (!std::isfinite(f)) f = -1.0;
        const int z = static_cast<int>(std::min<double>(std::max<double>(f, 0.0), g.nz - 1));
        plane[i] = z;
        hist[z] += 1.0;
    }
    std::vector<double> cum(g.nz);
    double acc = 0.0;
    for (int z = 0; z < g.nz; ++z) cum[z] = (acc += hist[z]);
    const double total = g.nz ? cum[g.nz - 1] : 0.0;
    std::vector<int> cuts{0};
    for (int k = 1; k < nranks; ++k) {
        const double target = total * k / nranks;
        int z = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin()) + 1;
        z = std::max(z, cuts.back() + 1);
        z = std::min(z, g.nz - (nranks - k));
        cuts.push_back(z);
    }
    cuts.push_back(g.nz);
    // records per inbox region: the same on every rank (the neighbours compute the inbox layout
    // from their own value): two of the fullest cell planes, at least N / (4 nranks) and 4096
    double max_plane = 0.0;
    for (int z = 0; z < g.nz; ++z) max_plane = std::max(max_plane, hist[z]);
    *cap_rec = std::max<uint64_t>({4096, static_cast<uint64_t>(2.0 * max_plane) + 1024, all->count / (4 * nranks)});
    *z_lo = cuts[rank];
    *z_hi = cuts[rank + 1];
    *h_out = g.cell_size;
    owned->clear();
    *ghosts = 0;
    const bool ring = (cfg->periodic & 4u) != 0;
    const int below = ring ? (*z_lo - 1 + g.nz) % g.nz : *z_lo - 1, above = ring ? *z_hi % g.nz : *z_hi;
    for (uint64_t i = 0; i < all->count; ++i) {
        if (plane[i] >= *z_lo && plane[i] < *z_hi) owned->push_back(i);
        else if (plane[i] == below || plane[i] == above) ++*ghosts;
    }
    return DEM_OK;
}

int shard_collect(dem_ctx* c, dem_step_metrics* m) {
    dem_ctx* const ctx = c;  // CUDA_TRY reports into ctx
    uint32_t dn[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(dn, c->dn, sizeof(dn), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaGetLastError());
    c->launched = false;
    const int rc = collect(c, m, c->launch_pb, c->launch_sb, true, true);
    c->n = c->n_asm = dn[0];
    c->n_own = dn[1];
    return rc;
}

}  // namespace

int dem_create_sharded(const dem_config* cfg, const dem_particles* all, int device, int rank, int nranks,
                       dem_ctx** out) {
    if (!cfg || !all || !out || nranks < 1 || rank < 0 || rank >= nranks) return DEM_ERR_ARGUMENT;
    *out = nullptr;
    std::string why;
    int rc = validate(cfg, all, &why);
    if (rc == DEM_OK) rc = check_unique_ids(all->ids, all->count, &why);
    if (rc == DEM_OK && cfg->collide_variant == 0) { why = "sharded contexts run the two_phase collide variant"; rc = DEM_ERR_CONFIG; }
    double h = 0.0;
    int32_t z_lo = 0, z_hi = 0;
    std::vector<uint64_t> idx;
    uint64_t ghosts = 0, cap_rec = 0;
    if (rc == DEM_OK) rc = shard_partition(cfg, all, rank, nranks, &h, &z_lo, &z_hi, &idx, &ghosts, &cap_rec, &why);
    if (rc != DEM_OK) {
        std::snprintf(g_create_error.message, sizeof(g_create_error.message), "%s", why.c_str());
        g_create_error.code = rc;
        return rc;
    }
    // the owned subset, then a slab context with the global cell size
    const uint64_t n = idx.size();
    std::vector<uint32_t> ids(n), mat(n);
    std::vector<double> pos(3 * n), vel(3 * n), omg(3 * n), rad(n), mass(n);
    for (uint64_t k = 0; k < n; ++k) {
        const uint64_t i = idx[k];
        ids[k] = all->ids[i];
        mat[k] = all->material_ids[i];
        rad[k] = all->radii[i];
        mass[k] = all->masses[i];
        for (int a = 0; a < 3; ++a) {
            pos[3 * k + a] = all->positions[3 * i + a];
            vel[3 * k + a] = all->velocities[3 * i + a];
            omg[3 * k + a] = all->angular_velocities[3 * i + a];
        }
    }
    dem_particles owned{n, ids.data(), pos.data(), vel.data(), omg.data(), rad.data(), mass.data(), mat.data()};
    dem_config scfg = *cfg;
    scfg.grid_cell_size = h;
    const uint64_t capacity = 1024 + (3 * (n + ghosts)) / 2;
    dem_ctx* ctx = nullptr;
    rc = dem_create_slab(&scfg, &owned, device, z_lo, z_hi, capacity, &ctx);
    if (rc != DEM_OK) return rc;
    ctx->shard = true;
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->cap_rec = cap_rec;
    ctx->inbox_bytes = inbox_region(1, 1, ctx->cap_rec, ctx->rec_bytes, ctx->ghost_bytes) + ctx->cap_rec * ctx->ghost_bytes;
    uint8_t* box = nullptr;
    cudaError_t e = dalloc(ctx, &box, ctx->inbox_bytes);
    if (e == cudaSuccess) e = dalloc(ctx, &ctx->dn, 2);
    if (e == cudaSuccess) {
        ctx->inbox = box;
        const uint32_t dn0[2] = {static_cast<uint32_t>(n), static_cast<uint32_t>(n)};
        e = cudaMemcpyAsync(ctx->dn, dn0, sizeof(dn0), cudaMemcpyHostToDevice, ctx->stream);  // X holds the owned set
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    }
    if (e != cudaSuccess) {
        free_ctx(ctx);
        std::snprintf(g_create_error.message, sizeof(g_create_error.message), "CUDA allocation of the shard inbox failed");
        g_create_error.code = DEM_ERR_CUDA;
        return DEM_ERR_CUDA;
    }
    *out = ctx;
    return DEM_OK;
}

int dem_shard_info(const dem_ctx* ctx, int32_t* z_lo, int32_t* z_hi, uint64_t* owned) {
    if (!ctx || !ctx->shard) return DEM_ERR_ARGUMENT;
    if (z_lo) *z_lo = ctx->z_lo;
    if (z_hi) *z_hi = ctx->z_hi;
    if (owned) *owned = ctx->n_own ? ctx->n_own : ctx->n;
    return DEM_OK;
}

int dem_shard_handle(const dem_ctx* ctx, void* handle64) {
    if (!ctx || !ctx->shard || !handle64) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, ctx->inbox) != cudaSuccess) return DEM_ERR_CUDA;
    std::memcpy(handle64, &h, sizeof(h));
    return DEM_OK;
}

namespace {
int shard_finish_connect(dem_ctx* ctx) {
    ctx->connected = true;
    ctx->stream_wait = cu_stream_wait() != nullptr;
    if (build_shard_graphs(ctx) != DEM_OK) {  // no stream memory operations in graphs: spin waits
        ctx->stream_wait = false;
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        if (build_shard_graphs(ctx) != DEM_OK) return set_error(ctx, DEM_ERR_CUDA, -1, 0, 0, ctx->step_index, "shard graph capture failed");
    }
    return DEM_OK;
}
}  // namespace

int dem_shard_connect(dem_ctx* ctx, const void* handles) {
    if (!ctx || !ctx->shard || !handles || ctx->connected) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    const bool ring = (ctx->periodic & 4u) != 0;
    const int R = ctx->nranks, r = ctx->rank;
    const int nb[2] = {ring || r > 0 ? (r - 1 + R) % R : -1, ring || r < R - 1 ? (r + 1) % R : -1};
    for (int side = 0; side < 2; ++side) {
        if (nb[side] < 0) continue;
        if (nb[side] == r) { ctx->peer[side] = ctx->inbox; continue; }
        if (side == 1 && nb[1] == nb[0] && ctx->peer_ipc[0]) { ctx->peer[1] = ctx->peer[0]; ctx->peer_ipc[1] = true; continue; }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + 64 * nb[side], sizeof(h));
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            return set_error(ctx, DEM_ERR_CUDA, -1, 0, 0, ctx->step_index,
                             "shard: cannot open the inbox of rank " + std::to_string(nb[side]) + " (no peer access?)");
        ctx->peer[side] = static_cast<uint8_t*>(ptr);
        ctx->peer_ipc[side] = true;
    }
    return shard_finish_connect(ctx);
}

int dem_shard_connect_local(dem_ctx* ctx, dem_ctx* lo, dem_ctx* hi) {
    if (!ctx || !ctx->shard || ctx->connected) return DEM_ERR_ARGUMENT;
    if ((lo && !lo->shard) || (hi && !hi->shard)) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    for (dem_ctx* o : {lo, hi})
        if (o && o->device != ctx->device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return DEM_ERR_CUDA;
            cudaGetLastError();
        }
    ctx->peer[0] = lo ? lo->inbox : nullptr;
    ctx->peer[1] = hi ? hi->inbox : nullptr;
    return shard_finish_connect(ctx);
}

int dem_shard_launch(dem_ctx* ctx, int nsteps) {
    if (!ctx || !ctx->shard || !ctx->connected || nsteps < 0 || ctx->launched) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    ctx->launch_pb = ctx->phase_count;
    ctx->launch_sb = ctx->step_index;
    if (!ctx->primed) {  // the constructor's force-only pass (pipeline.cpp:83), collectively
        const int rc = enqueue_shard_phase(ctx, false, DEM_PHASE_GRAVITY | DEM_PHASE_PP | DEM_PHASE_RECT | DEM_PHASE_LINE,
                                           ctx->shist);
        if (rc != DEM_OK) return rc;
        ctx->shist ^= 1;
        ++ctx->phase_count;
        ctx->primed = true;
        ctx->launch_pb = ctx->phase_count;
    }
    for (int k = 0; k < nsteps; ++k) {
        CUDA_TRY(cudaGraphLaunch(ctx->shard_graph[ctx->shist], ctx->stream));
        ctx->shist ^= 1;
        ++ctx->phase_count;
        ++ctx->step_index;
    }
    ctx->launched = true;
    return DEM_OK;
}

int dem_shard_wait(dem_ctx* ctx, dem_step_metrics* last) {
    if (!ctx || !ctx->shard) return DEM_ERR_ARGUMENT;
    cudaSetDevice(ctx->device);
    if (!ctx->launched) {
        if (last) { std::memset(last, 0, sizeof(*last)); last->step = ctx->step_index; }
        return DEM_OK;
    }
    return shard_collect(ctx, last);
}

int dem_selftest_division(int device, uint64_t n, uint64_t seed, uint64_t* mismatches) {
    if (!mismatches) return DEM_ERR_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return DEM_ERR_CUDA;
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return DEM_ERR_CUDA;
    unsigned long long h = 0;
    cudaError_t e = cudaMemset(d, 0, sizeof(*d));
    if (e == cudaSuccess) {
        launch_selftest_division(n, seed, d, 0);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    *mismatches = h;
    return e == cudaSuccess ? DEM_OK : DEM_ERR_CUDA;
}

}  // extern "C"
