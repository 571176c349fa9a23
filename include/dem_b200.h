/*
 * dem_b200.h — C ABI of the B200-native DEM step (drop-in for the reference
 * demforge::Simulation path, arxiv/paper_1503_03553).
 *
 * The reference exposes the hot path as the C++ class demforge::Simulation
 * (/root/reference/proj/core/include/demforge/pipeline.hpp:62-136) plus its
 * value types. There is no FFI in the reference; this header is what a
 * reference-side binding (C++ wrapper, ctypes, cgo, ...) binds instead. Each
 * entry point cites the reference member it replaces. Plain pointers and sizes
 * only; no CUDA or torch types cross the boundary.
 *
 * Ownership: a dem_ctx owns all device memory (one device, one stream); host
 * buffers passed in/out are caller-owned. A context is single-owner and not
 * thread-safe (same contract as demforge::Simulation, pipeline.hpp:58-61).
 * Errors: functions return a dem_status; details (kernel name, particle) are
 * available from dem_last_error(), mirroring the exception taxonomy of
 * core/include/demforge/error.hpp:10-49.
 */
#ifndef DEM_B200_H
#define DEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DEM_B200_ABI_VERSION 2

/* Status codes <-> reference exception types (error.hpp). */
typedef enum {
    DEM_OK = 0,
    DEM_ERR_CONFIG = 1,     /* ConfigError            error.hpp:10-13 (CLI exit 2) */
    DEM_ERR_KERNEL = 2,     /* KernelError            error.hpp:17-26 (CLI exit 3) */
    DEM_ERR_CAPACITY = 3,   /* CapacityError          error.hpp:30-42              */
    DEM_ERR_DEGENERATE = 4, /* DegenerateContactError error.hpp:46-49              */
    DEM_ERR_ARGUMENT = 5,   /* bad pointer / size at the ABI boundary              */
    DEM_ERR_CUDA = 6        /* device / driver failure                             */
} dem_status;

/* Kernel identifiers, in step order (pipeline.hpp:21-31). */
typedef enum {
    DEM_KERNEL_INTEGRATE = 0,
    DEM_KERNEL_CALC_HASH = 1,
    DEM_KERNEL_SORT = 2, /* reference: BitonicSort; here a one-digit (radix = cell count) counting sort */
    DEM_KERNEL_FIND_CELL_BOUNDS_AND_REORDER = 3,
    DEM_KERNEL_FORCE_GRAVITY = 4,
    DEM_KERNEL_INITIALIZE_CONTACT_IDS = 5,
    DEM_KERNEL_COLLIDE = 6,
    DEM_KERNEL_COLLIDE_RECTANGLE = 7,
    DEM_KERNEL_COLLIDE_LINE = 8,
    DEM_KERNEL_COUNT = 9
} dem_kernel;

/* The B200 kernels one step() launches, in order. */
typedef enum {
    DEM_DK_PHASE_BEGIN = 0,   /* control-block reset                                  */
    DEM_DK_INTEGRATE_HASH,    /* Integrate + CalcHash + cell histogram                */
    DEM_DK_SCAN_CELLS,        /* cell_start scan (FindCellBounds)                     */
    DEM_DK_SCATTER,           /* counting-sort scatter (BitonicSort replacement)      */
    DEM_DK_REORDER,           /* canonical in-cell order + SoA gather (Reorder)       */
    DEM_DK_DETECT,            /* 27-cell detection -> compacted pair list (loop 1)    */
    DEM_DK_FORCE_REDUCE,      /* Hertz-Mindlin per contact + history merge (loop 2)   */
                              /* + per-particle deterministic sum, gravity, capacity  */
    DEM_DEVICE_KERNEL_COUNT
} dem_device_kernel;

/* MaterialParams, materials.hpp:10-21 */
typedef struct {
    double poisson_ratio;
    double shear_modulus;
    double youngs_modulus;
    double restitution;
    double sliding_friction;
} dem_material;

/* RectWall, geometry.hpp:55-61 */
typedef struct {
    double corner[3];
    double edge_u[3];
    double edge_v[3];
    uint32_t material_id;
} dem_rect_wall;

/* LineWall, geometry.hpp:63-67 */
typedef struct {
    double a[3];
    double b[3];
    uint32_t material_id;
} dem_line_wall;

/* SimConfig, sim_config.hpp:42-63 (the fields the step reads). */
typedef struct {
    double dt;
    double gravity[3];
    double domain_min[3];
    double domain_max[3];
    uint32_t material_count;
    const dem_material* materials;
    /* material_count^2 row-major pair restitution after overrides
     * (MaterialTable::pair_restitution, materials.cpp:58-64); NULL = sqrt(eps_a eps_b). */
    const double* pair_restitution;
    uint32_t rect_wall_count;
    const dem_rect_wall* rect_walls;
    uint32_t line_wall_count;
    const dem_line_wall* line_walls;
    double grid_cell_size;   /* 0 => 2 r_max (1 + 1e-6), grid.cpp:15 */
    int32_t contact_capacity; /* K, contact_table.hpp:30-74 */
    int32_t collide_variant;  /* 0 baseline (Alg. 1), 1 two_phase (warp_model.hpp:9) */
    /* Beyond the reference; zero = the reference's box.
     * periodic: bit 0 x, bit 1 y, bit 2 z. A periodic axis of length L gets n = floor(L / h)
     * cells of extent L / n (n >= 3). shear_rate: Lees-Edwards shear (flow x, gradient y; needs
     * x and y periodic, n_x >= 4). Periodic boxes run the two-phase variant on one GPU. */
    uint32_t periodic;
    double shear_rate;
    /* 0: fp64 parity mode (the reference's arithmetic, bit for bit). 1: fp32 throughput mode —
     * the force kernel evaluates each contact in fp32 around an fp64 geometry core (displacement,
     * distance, overlap) and sums in fp64; north_star tolerance 1e-5 relative. */
    int32_t precision;
} dem_config;

/* ParticleSet, particle_set.hpp:13-37, flattened (Vec3 = 3 doubles). */
typedef struct {
    uint64_t count;
    uint32_t* ids;
    double* positions;          /* 3*count */
    double* velocities;         /* 3*count */
    double* angular_velocities; /* 3*count */
    double* radii;
    double* masses;
    uint32_t* material_ids;
} dem_particles;

/* StepMetrics, pipeline.hpp:35-48 (+ device times per kernel when profiled). */
typedef struct {
    int64_t step;
    int64_t contacts;
    int64_t pp_contact_events;
    int32_t max_contacts_per_particle;
    int32_t reserved0;
    int64_t clamps;
    double friction_max_ratio;
    int64_t capped_contacts;          /* new counter: contacts where the friction cap engaged */
    int64_t cells;                    /* grid cells M (for byte accounting) */
    /* filled by dem_profile_step only: device ms per B200 kernel, index = dem_device_kernel */
    double device_kernel_ms[DEM_DEVICE_KERNEL_COUNT];
} dem_step_metrics;

/* UniformGrid, grid.hpp:14-31 */
typedef struct {
    double origin[3];
    double cell_size;
    int32_t nx, ny, nz;
} dem_grid;

typedef struct {
    int32_t code;            /* dem_status */
    int32_t kernel;          /* dem_kernel, or -1 */
    uint32_t particle_slot;  /* sorted slot at the failing step */
    uint32_t particle_id;    /* stable id */
    int64_t step;            /* step index (0 = constructor priming pass) */
    char message[256];       /* same text shape as the reference exception what() */
} dem_error;

/* Force-phase composition flags (Simulation::run_force_phase, pipeline.cpp:317-364, and the
 * advance_to_collide / fork_at_collide compositions used by tests and verify,
 * tests/test_pipeline.cpp:69-76, runner.cpp:261-270). */
typedef enum {
    DEM_PHASE_INTEGRATE = 1,
    DEM_PHASE_GRAVITY = 2,
    DEM_PHASE_PP = 4,
    DEM_PHASE_RECT = 8,
    DEM_PHASE_LINE = 16,
    DEM_PHASE_STEP = 31
} dem_phase_flags;

typedef struct dem_ctx dem_ctx;

int dem_abi_version(void);

/* Simulation(ParticleSet, SimConfig) — pipeline.hpp:64, pipeline.cpp:52-84. Validates
 * (sim_config.cpp:10-60, particle_set.cpp:40-58), uploads, runs the priming force pass. */
int dem_create(const dem_config* config, const dem_particles* particles, int device, dem_ctx** out);

/* Copy constructor — the reference class is copyable and forked by verify (runner.cpp:261-270). */
int dem_clone(const dem_ctx* ctx, dem_ctx** out);

void dem_destroy(dem_ctx* ctx);

/* Simulation::step() x nsteps — pipeline.hpp:68, pipeline.cpp:366-378. `last` (nullable)
 * receives the last step's metrics. Stops at the first failing step. */
int dem_step(dem_ctx* ctx, int nsteps, dem_step_metrics* last);

/* Asynchronous stepping for host-coupled callers (B200 addition): enqueue nsteps and return at
 * once. The next call that reads or replaces the state collects them — an error of an
 * asynchronous step is reported there, attributed to the failing step — and dem_sync collects
 * explicitly, returning the last step's metrics. dem_get_particles right after dem_step_async
 * reads the state back while the last step's detection and forces still run (its state is final
 * after the reorder), then waits for the step. Not for slab contexts. */
int dem_step_async(dem_ctx* ctx, int nsteps);
int dem_sync(dem_ctx* ctx, dem_step_metrics* last);

/* A composed force phase (flags, see dem_phase_flags). DEM_PHASE_STEP == step(). */
int dem_force_phase(dem_ctx* ctx, uint32_t flags, dem_step_metrics* metrics);

/* set_collide_variant, pipeline.hpp:74 */
int dem_set_collide_variant(dem_ctx* ctx, int variant);

/* Accessors — particles()/forces()/contact_table()/order()/grid()/step_index(),
 * pipeline.hpp:88-99. Arrays are in the current sorted slot order. */
uint64_t dem_size(const dem_ctx* ctx);
int64_t dem_step_index(const dem_ctx* ctx);
int dem_get_particles(dem_ctx* ctx, dem_particles* out);
/* positions, velocities, angular_velocities are required; ids, radii, masses, material_ids may be
 * NULL, in which case every slot keeps its current value (the given arrays are then in the current
 * slot order, as dem_get_particles returns it) — a host-coupled caller that changes only the
 * motion moves 72 of the 96 bytes per particle. In dem_get_particles any array may be NULL. */
int dem_set_particles(dem_ctx* ctx, const dem_particles* in);
int dem_get_forces(dem_ctx* ctx, double* force, double* torque);
int dem_set_forces(dem_ctx* ctx, const double* force, const double* torque);
int dem_get_grid(const dem_ctx* ctx, dem_grid* out);
/* Periodic box: cell extent per axis (the grid's cell_size on non-periodic axes)
 * and the current Lees-Edwards image offset of the upper box along x. */
int dem_get_periodic_box(dem_ctx* ctx, double cell_extent[3], double* shear_offset);
/* sorted cell keys (SortedOrder::sorted_keys) and, per new slot, the previous slot
 * (SortedOrder::permutation, sorted_order.hpp:13-19) */
int dem_get_order(dem_ctx* ctx, uint32_t* sorted_keys, uint32_t* permutation);

/* Live contact history after the last force phase (ContactTable touched slots,
 * contact_table.hpp:53-66): owner slot, partner (slot >= 0, or wall id -(w+1)),
 * delta_t (3 per entry), in per-owner accumulation order. Returns the count; fills up to cap. */
/* Replace the live contact history (the mutable ContactTable the reference's bench restores,
 * runner.cpp:131-132): `count` entries (owner slot, partner slot >= 0 or wall id -(w+1), delta_t),
 * in the current slot order; each owner's entries keep their given order. The next force phase
 * merges tangential history from it exactly as from a history the step produced. Owners with more
 * than contact_capacity entries, repeated (owner, partner) pairs or out-of-range slots are
 * DEM_ERR_ARGUMENT. Single-GPU contexts. */
int dem_set_contacts(dem_ctx* ctx, const uint32_t* owner_slot, const int32_t* partner, const double* delta_t,
                     int64_t count);
int64_t dem_get_contacts(dem_ctx* ctx, uint32_t* owner_slot, int32_t* partner, double* delta_t,
                         int64_t cap);

/* Traversal traces of the last force phase — Simulation::traces() (pipeline.hpp:97), recorded by
 * kernel_collide (pipeline.cpp:191-231): per owner slot i, in the traversal order (27 cells z, y,
 * x outer-to-inner, ascending slot, j != i), one event per candidate slot j with the check_pair
 * outcome. Identical for both Collide variants. offsets (nullable, n+1 entries) receives the
 * per-slot event ranges; events (nullable) is filled when capacity >= the total. Returns the total
 * event count, or a negative dem_status. Available after a force phase with DEM_PHASE_PP until
 * the state is replaced (dem_set_particles); single-GPU contexts only. */
typedef struct dem_trace_event {
    int32_t candidate; /* TraceEvent::candidate, warp_model.hpp:28-33 (a slot index) */
    int32_t contact;   /* TraceEvent::contact (0/1) */
} dem_trace_event;
int64_t dem_get_traces(dem_ctx* ctx, uint64_t* offsets, dem_trace_event* events, int64_t capacity);

/* Last error (what(), kernel, particle). */
int dem_last_error(const dem_ctx* ctx, dem_error* out);

/* ---- measurement helpers (used by bench.py; kernels run on the context's stream) ---- */
/* Runs nsteps step()s as CUDA-graph launches. Before each step, when flush_bytes > 0, a
 * buffer of that size is overwritten to evict L2; each step is timed with CUDA events on
 * the launching stream and written to step_ms[k]. */
int dem_time_steps(dem_ctx* ctx, int nsteps, size_t flush_bytes, float* step_ms,
                   dem_step_metrics* last);
/* One step() without graphs with events between kernels; per-kernel device ms in
 * metrics->kernel_ms (index = dem_kernel). */
int dem_profile_step(dem_ctx* ctx, size_t flush_bytes, dem_step_metrics* metrics);
/* Number of kernel launches one step() issues, and their names. */
int dem_kernels_per_step(const dem_ctx* ctx);
const char* dem_device_kernel_name(int k);
/* Bytes of device memory the context holds. */
uint64_t dem_device_bytes(const dem_ctx* ctx);

/* ---- slab domain decomposition (multi-GPU; no reference counterpart:
 * the reference is single-process) ----
 * A slab context owns the particles whose global cell plane z is in [z_lo, z_hi). Each step the
 * host runs, per rank:
 *   dem_slab_migrate(integrate=1) -> exchange migrant records with the z-neighbours ->
 *   dem_slab_import -> dem_slab_halo -> exchange ghost records -> dem_slab_ghosts ->
 *   dem_slab_force(DEM_PHASE_STEP)
 * (the constructor-equivalent priming pass is the same with integrate=0 and flags
 * GRAVITY|PP|RECT|LINE). Record buffers are DEVICE pointers owned by the caller (e.g. torch
 * tensors exchanged with NCCL); record sizes come from dem_slab_record_bytes. Results are
 * bitwise identical to a single-GPU context because the in-cell order is canonical.
 * config->grid_cell_size must be the global cell size (2 r_max (1 + 1e-6) over all ranks). */
int dem_create_slab(const dem_config* config, const dem_particles* owned, int device, int32_t z_lo,
                    int32_t z_hi, uint64_t capacity, dem_ctx** out);
int dem_slab_record_bytes(const dem_ctx* ctx, uint64_t* migrant_bytes, uint64_t* ghost_bytes);
uint64_t dem_slab_owned(const dem_ctx* ctx);
int dem_slab_migrate(dem_ctx* ctx, int integrate, void* send_lo, void* send_hi, uint64_t cap_records,
                     uint64_t* n_lo, uint64_t* n_hi);
int dem_slab_import(dem_ctx* ctx, const void* recs_lo, uint64_t n_lo, const void* recs_hi, uint64_t n_hi);
int dem_slab_halo(dem_ctx* ctx, void* send_lo, void* send_hi, uint64_t cap_records, uint64_t* n_lo,
                  uint64_t* n_hi);
int dem_slab_ghosts(dem_ctx* ctx, const void* recs_lo, uint64_t n_lo, const void* recs_hi, uint64_t n_hi);
int dem_slab_force(dem_ctx* ctx, uint32_t flags, dem_step_metrics* metrics);

/* Peer-memory record exchange (one process per GPU, NVLink P2P): a rank allocates its receive
 * buffers here, shares them with its z-neighbours as CUDA IPC handles (64 bytes each), and passes
 * the neighbours' opened buffers as dem_slab_migrate / dem_slab_halo send buffers — the pack
 * kernels then store the records straight into the neighbour's memory over NVLink, and only the
 * record counts travel through the host. */
int dem_ipc_alloc(int device, uint64_t bytes, void** ptr);
int dem_ipc_free(int device, void* ptr);
int dem_ipc_handle(int device, void* ptr, void* handle64);
int dem_ipc_open(int device, const void* handle64, void** ptr);
int dem_ipc_close(int device, void* ptr);

/* ---- host-free sharded stepping: the multi-GPU Simulation (SURVEY §8b "dem_create_sharded";
 * §8e). Replaces, for N GPUs, the reference's single-process Simulation(ParticleSet, SimConfig)
 * (pipeline.hpp:64) + step() (:68); no reference counterpart for the decomposition itself
 * (SPEC.md:382-383 lists multi-node as a non-goal).
 *
 *   dem_create_sharded(cfg, ALL particles, device, rank, nranks, &ctx)   every rank, same inputs:
 *       rank `rank` keeps the z-slab of whole cell planes the deterministic, count-balanced
 *       partition assigns it (plus a one-plane halo each step)
 *   dem_shard_handle(ctx, handle64)        64 bytes: this rank's inbox (a CUDA IPC handle)
 *   -- the caller all-gathers the nranks handles (ncclAllGather, MPI_Allgather, torch) --
 *   dem_shard_connect(ctx, handles)        nranks * 64 bytes, rank order; opens the neighbours'
 *                                          inboxes (one process per GPU, NVLink peer memory)
 *   dem_shard_connect_local(ctx, lo, hi)   instead: contexts of ONE process (lo / hi = the
 *                                          z-neighbours' contexts, NULL at a non-periodic edge)
 *   dem_step(ctx, n, &m)                   n steps (the first call also runs the priming pass)
 *
 * A step is one CUDA graph with no host round trip: record counts stay on the device, the
 * migrate / halo pack kernels store records and counts straight into the neighbours' inboxes and
 * raise a flag (release store, system scope), and the stream waits for the neighbours' flags
 * (stream memory operation; a spin kernel where unavailable). Every rank must step the same number
 * of times: dem_step on ranks of one process would wait for each other, so there call
 * dem_shard_launch on every rank, then dem_shard_wait on every rank. Results are bitwise identical
 * to one context (canonical in-cell order). dem_get_particles / dem_get_forces / dem_get_contacts
 * return the slab's slots, owned and halo: halo copies have material_ids bit 31 set.
 * dem_time_steps times graph-launched steps (after a first dem_step). Tear-down: destroy every
 * rank only after all ranks have finished stepping (their stores target each other's memory). */
int dem_create_sharded(const dem_config* config, const dem_particles* all_particles, int device, int rank,
                       int nranks, dem_ctx** out);
int dem_shard_info(const dem_ctx* ctx, int32_t* z_lo, int32_t* z_hi, uint64_t* owned);
int dem_shard_handle(const dem_ctx* ctx, void* handle64);
int dem_shard_connect(dem_ctx* ctx, const void* handles);
int dem_shard_connect_local(dem_ctx* ctx, dem_ctx* lo, dem_ctx* hi);
int dem_shard_launch(dem_ctx* ctx, int nsteps);
int dem_shard_wait(dem_ctx* ctx, dem_step_metrics* last);

/* Diagnostics: the force kernel's shared-reciprocal division against the plain IEEE '/' on n
 * seeded random operand pairs (random bit patterns, exponents around the
 * fast-path bounds, contact-like magnitudes). *mismatches = results that differ in any bit. */
int dem_selftest_division(int device, uint64_t n, uint64_t seed, uint64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif /* DEM_B200_H */
