/*
 * dem_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A single-threaded plain-C restatement of the reference DEM step
 * (arxiv/paper_1503_03553, "demforge", /root/reference/proj/core). It is the
 * parity checker for the B200 path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product
 * path (paper_1503_03553_b200) never links or calls it.
 *
 * Parity pinning: every function below is checked against the reference
 * itself compiled from its own sources (oracle/_ref, see oracle/Makefile) and
 * against the known-answer values of the reference tests
 * (proj/tests/test_physics.cpp, test_grid.cpp, test_pipeline.cpp).
 *
 * Arithmetic contract (reference core/CMakeLists.txt:32-37): fp64, every
 * + - * / individually rounded (compiled with -ffp-contract=off), IEEE sqrt,
 * strict left-to-right evaluation exactly as the reference writes it.
 */
#ifndef DEM_ORACLE_H
#define DEM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (mirror include/dem_b200.h). */
enum {
    ORC_OK = 0,
    ORC_ERR_CONFIG = 1,      /* ConfigError            (error.hpp:10-13)  */
    ORC_ERR_KERNEL = 2,      /* KernelError            (error.hpp:17-26)  */
    ORC_ERR_CAPACITY = 3,    /* CapacityError          (error.hpp:30-42)  */
    ORC_ERR_DEGENERATE = 4,  /* DegenerateContactError (error.hpp:46-49)  */
    ORC_ERR_BUFFER = 5       /* caller buffer too small                   */
};

/* Kernel names for error reporting (pipeline.cpp:16-29). */
enum {
    ORC_K_INTEGRATE = 0, ORC_K_CALC_HASH, ORC_K_SORT, ORC_K_REORDER, ORC_K_GRAVITY,
    ORC_K_SWEEP, ORC_K_COLLIDE, ORC_K_COLLIDE_RECT, ORC_K_COLLIDE_LINE
};

typedef struct {
    double poisson_ratio, shear_modulus, youngs_modulus, restitution, sliding_friction;
} orc_material;

typedef struct { double corner[3], edge_u[3], edge_v[3]; uint32_t material_id; } orc_rect;
typedef struct { double a[3], b[3]; uint32_t material_id; } orc_line;

typedef struct {
    double dt;
    double gravity[3];
    double domain_min[3], domain_max[3];
    uint32_t material_count;
    const orc_material* materials;
    const double* pair_restitution; /* material_count^2, row-major; NULL = sqrt(ea*eb) */
    uint32_t rect_count;
    const orc_rect* rects;
    uint32_t line_count;
    const orc_line* lines;
    double grid_cell_size;          /* 0 = 2 r_max (1+1e-6) */
    int32_t contact_capacity;
    /* Beyond the reference: periodic axes (bit 0 x, 1 y,
     * 2 z) and a Lees-Edwards shear rate (flow x, gradient y; needs x and y periodic). 0, 0 is
     * the reference's walled box, bit for bit. */
    uint32_t periodic;
    double shear_rate;
} orc_config;

typedef struct {
    double origin[3];
    double cell_size;
    int32_t nx, ny, nz;
} orc_grid;

/* ---- L2 pure functions (golden-vector tests) ---- */
double orc_restitution_alpha(double eps);                               /* contact_mechanics.cpp:7-12 */
void orc_contact_coefficients(double delta_n, const orc_material* m1, const orc_material* m2,
                              double r1, double r2, double m1_, double m2_, double alpha,
                              int partner_is_wall, double out[4]);      /* :14-33 -> k_t,k_n,eta_n,eta_t */
/* geometry: returns 1 contact, 0 none, -1 degenerate. out: normal[3], overlap, rel_vel[3], vt[3] */
int orc_contact_geometry(const double p1[3], double r1, const double v1[3], const double w1[3],
                         const double partner_point[3], int partner_is_wall, double r2,
                         const double v2[3], const double w2[3], double out[10]); /* geometry.cpp:24-51 */
/* force: in geom[10] as above; out: F[3], T[3], dt_new[3], fn, ft, capped */
void orc_contact_force(const double geom[10], const double coeffs[4], const double delta_t[3],
                       double mu, double r1, double out[12]);           /* contact_mechanics.cpp:48-85 */
void orc_update_tangential(const double old[3], const double n[3], const double vt[3], double dt,
                           double out[3]);                              /* :43-46 */
int orc_make_grid(const double bmin[3], const double bmax[3], double r_max, double h,
                  orc_grid* out);                                       /* grid.cpp:10-28 */
uint32_t orc_calc_hash(const double p[3], const orc_grid* g, int* clamped); /* grid.cpp:30-58 */
int orc_neighbor_cells(uint32_t cell, const orc_grid* g, uint32_t out[27]); /* grid.cpp:60-82 */
void orc_closest_point_rect(const double p[3], const orc_rect* w, double out[4]); /* geometry.cpp:60-68 */
void orc_closest_point_line(const double p[3], const orc_line* w, double out[4]); /* geometry.cpp:70-75 */

/* ---- Oracles ---- */
/* All unordered contacting pairs (i<j, slot indices), oracle.cpp:11-24. O(N^2) when
 * binned==0; binned==1 uses an equivalent independent grid (exact same test). Pairs are
 * returned sorted by (i, j). Returns count, or -1 if cap too small (count in *needed). */
int64_t orc_contact_pairs(size_t n, const double* pos, const double* rad, int binned,
                          uint32_t* out_i, uint32_t* out_j, int64_t cap);

/* History entry keyed by stable ids: partner key = partner stable id, or the reference wall
 * id -(w+1) reinterpreted as uint32 (contact_table.hpp:35). */
typedef struct {
    uint32_t owner_id;
    uint32_t partner_key;
    double delta_t[3];
} orc_hist;

/* Permutation-agnostic pp collide replay (oracle.cpp:47-105): candidates of slot i are
 * visited by (neighbour visit index, slot); pp only, no gravity, no walls. Forces/torques are
 * written per slot (3n each, zero-initialised then accumulated). hist_in: previous live
 * entries (any order). hist_out: entries touched here, in event order (<= cap).
 * events: (owner slot, partner slot) pairs in accumulation order.
 * Returns the number of events or a negative error code. */
int64_t orc_collide(size_t n, const uint32_t* ids, const double* pos, const double* vel,
                    const double* omg, const double* rad, const double* mass,
                    const uint32_t* mat, const orc_config* cfg, const orc_grid* grid,
                    const orc_hist* hist_in, int64_t hist_in_count, double* forces,
                    double* torques, orc_hist* hist_out, uint32_t* ev_owner,
                    uint32_t* ev_partner, int64_t cap);

/* ---- Full step restatement (pipeline.cpp:31-378) with canonical (cell, stable id) order ---- */
typedef struct orc_sim orc_sim;

typedef struct {
    int64_t step;
    int64_t contacts;           /* incl. walls */
    int64_t pp_contact_events;
    int32_t max_contacts_per_particle;
    int64_t clamps;
    double friction_max_ratio;
} orc_metrics;

typedef struct {
    int32_t code;
    int32_t kernel;
    uint32_t particle_slot;
    uint32_t particle_id;
    int64_t step;
} orc_error;

/* flags for orc_sim_force_phase */
enum { ORC_PH_INTEGRATE = 1, ORC_PH_GRAVITY = 2, ORC_PH_PP = 4, ORC_PH_RECT = 8, ORC_PH_LINE = 16,
       ORC_PH_ALL = 31 };

orc_sim* orc_sim_create(const orc_config* cfg, size_t n, const uint32_t* ids, const double* pos,
                        const double* vel, const double* omg, const double* rad,
                        const double* mass, const uint32_t* mat, orc_error* err);
void orc_sim_destroy(orc_sim* s);
int orc_sim_step(orc_sim* s, int nsteps, orc_metrics* m, orc_error* err);
int orc_sim_force_phase(orc_sim* s, int flags, orc_metrics* m, orc_error* err);
size_t orc_sim_size(const orc_sim* s);
void orc_sim_get_state(const orc_sim* s, uint32_t* ids, double* pos, double* vel, double* omg,
                       double* rad, double* mass, uint32_t* mat);
void orc_sim_get_forces(const orc_sim* s, double* forces, double* torques);
void orc_sim_get_keys(const orc_sim* s, uint32_t* sorted_keys);
/* per slot, the last phase's sum of |F| and |T| contributions (gravity, contacts, walls): the scale
 * of the 1e-9 relative parity criterion (SURVEY §8a notes) */
void orc_sim_get_force_scale(const orc_sim* s, double* f_abs, double* t_abs);
int64_t orc_sim_history_count(const orc_sim* s);
void orc_sim_get_history(const orc_sim* s, orc_hist* out);
void orc_sim_get_grid(const orc_sim* s, orc_grid* g);
/* periodic box of a simulation: cell extents per axis and the current Lees-Edwards offset */
void orc_sim_get_pbox(const orc_sim* s, double cell_extent[3], double* shear_offset, int64_t* shear_steps);

/* bench input generator G(N, s, jit, poly, seed) of SURVEY.md §8d (bench_support.hpp:10-44, rng.hpp) */
int orc_gen_packing(uint64_t n, double s, double jit, int poly, uint64_t seed, double omega_half,
                    uint32_t* ids, double* pos, double* vel, double* omg, double* rad, double* mass,
                    uint32_t* mat, double domain_max[3]);

#ifdef __cplusplus
}
#endif
#endif
