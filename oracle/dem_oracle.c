/*
 * dem_oracle.c — TEST INFRASTRUCTURE ONLY (see dem_oracle.h).
 *
 * Plain-C restatement of the reference DEM step. Compile with
 * -ffp-contract=off (oracle/Makefile) so every operation rounds exactly as the
 * reference core does (core/CMakeLists.txt:32-37). Each function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/core/.
 */
#include "dem_oracle.h"

#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y, z; } v3;

static inline v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 ld3(const double* p) { return mk(p[0], p[1], p[2]); }
static inline void st3(double* p, v3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
/* vec3.hpp:38-53 */
static inline v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 muls(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static inline v3 divs(v3 a, double s) { return mk(a.x / s, a.y / s, a.z / s); }
static inline double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 cross(v3 a, v3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double norm(v3 a) { return sqrt(dot(a, a)); }
static inline int finite3(v3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }
/* std::clamp(v, lo, hi) */
static inline double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

static const double kDegenerateDistance = 1e-12; /* geometry.cpp:11 */

/* contact_mechanics.cpp:7-12 */
double orc_restitution_alpha(double e) {
    if (e >= 1.0) return 0.0;
    const double ln_eps = log(e);
    const double pi = 3.14159265358979323846;
    return -2.0 * ln_eps / sqrt(pi * pi + ln_eps * ln_eps);
}

static inline double shear_sum(const orc_material* a, const orc_material* b) {
    return (2.0 - a->poisson_ratio) / a->shear_modulus + (2.0 - b->poisson_ratio) / b->shear_modulus;
}
static inline double young_sum(const orc_material* a, const orc_material* b) {
    return (2.0 - a->poisson_ratio * a->poisson_ratio) / a->youngs_modulus +
           (2.0 - b->poisson_ratio * b->poisson_ratio) / b->youngs_modulus;
}

/* contact_mechanics.cpp:14-33 */
void orc_contact_coefficients(double delta_n, const orc_material* m1, const orc_material* m2,
                              double r1, double r2, double ma, double mb, double alpha,
                              int wall, double out[4]) {
    const double r_eff = wall ? r1 : r1 * r2 / (r1 + r2);
    const double m_eff = wall ? ma : ma * mb / (ma + mb);
    const double ss = shear_sum(m1, m2);
    const double ys = young_sum(m1, m2);
    const double k_t = 8.0 * sqrt(r_eff * delta_n) / ss;
    const double k_n = (4.0 / 3.0) * sqrt(r_eff) / ys;
    const double eta = alpha * sqrt(m_eff * k_n * sqrt(delta_n));
    out[0] = k_t; out[1] = k_n; out[2] = eta; out[3] = eta;
}

/* geometry.cpp:24-51 (contact_point is not needed by the force path) */
int orc_contact_geometry(const double p1[3], double r1, const double v1_[3], const double w1_[3],
                         const double pp[3], int wall, double r2, const double v2_[3],
                         const double w2_[3], double out[10]) {
    const v3 diff = sub(ld3(pp), ld3(p1));
    const double dist = norm(diff);
    const double reach = wall ? r1 : r1 + r2;
    if (dist >= reach) return 0;
    if (dist < kDegenerateDistance) return -1;
    const v3 n = divs(diff, dist);
    const double overlap = reach - dist;
    const v3 v1 = ld3(v1_), w1 = ld3(w1_);
    const v3 v2 = wall ? mk(0.0, 0.0, 0.0) : ld3(v2_);
    const v3 rv = sub(v1, v2);
    const v3 spin = wall ? muls(w1, r1) : add(muls(w1, r1), muls(ld3(w2_), r2));
    const v3 vt = add(sub(rv, muls(n, dot(rv, n))), cross(spin, n));
    st3(out, n); out[3] = overlap; st3(out + 4, rv); st3(out + 7, vt);
    return 1;
}

/* contact_mechanics.cpp:43-46 */
void orc_update_tangential(const double o[3], const double n_[3], const double vt[3], double dt,
                           double out[3]) {
    const v3 old = ld3(o), n = ld3(n_);
    st3(out, add(sub(old, muls(n, dot(old, n))), muls(ld3(vt), dt)));
}

/* contact_mechanics.cpp:48-85. out: F[3], T[3], delta_new[3], |F_n|, |F_t| (after cap), capped */
void orc_contact_force(const double g[10], const double c[4], const double dlt[3], double mu,
                       double r1, double out[12]) {
    const v3 n = ld3(g), rv = ld3(g + 4), vt = ld3(g + 7);
    const double overlap = g[3];
    const double k_t = c[0], k_n = c[1], eta_n = c[2], eta_t = c[3];
    const v3 d = ld3(dlt);
    const v3 v_n = muls(n, dot(rv, n));
    const v3 force = sub(sub(sub(muls(d, -k_t), muls(vt, eta_t)),
                             muls(n, k_n * overlap * sqrt(overlap))),
                         muls(v_n, eta_n));
    const v3 f_normal = muls(n, dot(force, n));
    v3 f_tangent = sub(force, f_normal);
    v3 dnew = d;
    const double fn = norm(f_normal);
    const double ft = norm(f_tangent);
    const double limit = mu * fn;
    double tmag;
    int capped = 0;
    if (ft > limit) {
        capped = 1;
        if (ft < 1e-15) {
            f_tangent = mk(0.0, 0.0, 0.0);
            dnew = mk(0.0, 0.0, 0.0);
            tmag = 0.0;
        } else {
            f_tangent = muls(f_tangent, limit / ft);
            dnew = muls(f_tangent, -1.0 / k_t);
            tmag = norm(f_tangent);
        }
    } else {
        tmag = ft;
    }
    const v3 fo = add(f_normal, f_tangent);
    const v3 to = muls(cross(n, fo), r1);
    st3(out, fo); st3(out + 3, to); st3(out + 6, dnew);
    out[9] = fn; out[10] = tmag; out[11] = capped;
}

/* grid.cpp:10-28 */
int orc_make_grid(const double bmin[3], const double bmax[3], double r_max, double h, orc_grid* g) {
    const v3 ext = sub(ld3(bmax), ld3(bmin));
    if (!(ext.x > 0.0 && ext.y > 0.0 && ext.z > 0.0)) return ORC_ERR_CONFIG;
    if (h <= 0.0) h = 2.0 * r_max * (1.0 + 1e-6);
    if (!(h > 0.0)) return ORC_ERR_CONFIG;
    g->origin[0] = bmin[0]; g->origin[1] = bmin[1]; g->origin[2] = bmin[2];
    g->cell_size = h;
    int nx = (int)ceil(ext.x / h), ny = (int)ceil(ext.y / h), nz = (int)ceil(ext.z / h);
    g->nx = nx < 1 ? 1 : nx; g->ny = ny < 1 ? 1 : ny; g->nz = nz < 1 ? 1 : nz;
    if ((int64_t)g->nx * g->ny * g->nz > ((int64_t)1 << 31)) return ORC_ERR_CONFIG;
    return ORC_OK;
}

/* static_cast<int>(double) as x86-64 cvttsd2si executes it: out-of-range and NaN give INT_MIN. */
static inline int to_int_x86(double f) {
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return INT_MIN;
    return (int)f;
}

static inline int clamp_axis(int c, int dim, int* clamped) {
    if (c < 0) { *clamped = 1; return 0; }
    if (c >= dim) { *clamped = 1; return dim - 1; }
    return c;
}

static inline uint32_t linear_index(const orc_grid* g, int cx, int cy, int cz) { /* grid.hpp:23-25 */
    return (uint32_t)(cx + g->nx * (cy + (int64_t)g->ny * cz));
}

/* grid.cpp:30-58 */
uint32_t orc_calc_hash(const double p[3], const orc_grid* g, int* clamped) {
    const v3 rel = sub(ld3(p), ld3(g->origin));
    const double inv_h = 1.0 / g->cell_size;
    int cl = 0;
    int cx = to_int_x86(floor(rel.x * inv_h));
    int cy = to_int_x86(floor(rel.y * inv_h));
    int cz = to_int_x86(floor(rel.z * inv_h));
    cx = clamp_axis(cx, g->nx, &cl);
    cy = clamp_axis(cy, g->ny, &cl);
    cz = clamp_axis(cz, g->nz, &cl);
    if (clamped) *clamped = cl;
    return linear_index(g, cx, cy, cz);
}

/* grid.cpp:60-82 */
int orc_neighbor_cells(uint32_t cell, const orc_grid* g, uint32_t out[27]) {
    const int cx = (int)(cell % (uint32_t)g->nx);
    const int rest = (int)(cell / (uint32_t)g->nx);
    const int cy = rest % g->ny;
    const int cz = rest / g->ny;
    int count = 0;
    for (int dz = -1; dz <= 1; ++dz) {
        const int z = cz + dz;
        if (z < 0 || z >= g->nz) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            const int y = cy + dy;
            if (y < 0 || y >= g->ny) continue;
            for (int dx = -1; dx <= 1; ++dx) {
                const int x = cx + dx;
                if (x < 0 || x >= g->nx) continue;
                out[count++] = linear_index(g, x, y, z);
            }
        }
    }
    return count;
}

/* geometry.cpp:60-68; out = point[3], distance */
void orc_closest_point_rect(const double p_[3], const orc_rect* w, double out[4]) {
    const v3 p = ld3(p_), c = ld3(w->corner), u = ld3(w->edge_u), v = ld3(w->edge_v);
    const v3 rel = sub(p, c);
    const double uu = dot(u, u);
    const double vv = dot(v, v);
    const double s = clampd(dot(rel, u) / uu, 0.0, 1.0);
    const double t = clampd(dot(rel, v) / vv, 0.0, 1.0);
    const v3 point = add(add(c, muls(u, s)), muls(v, t));
    st3(out, point); out[3] = norm(sub(p, point));
}

/* geometry.cpp:70-75 */
void orc_closest_point_line(const double p_[3], const orc_line* w, double out[4]) {
    const v3 p = ld3(p_), a = ld3(w->a), b = ld3(w->b);
    const v3 dir = sub(b, a);
    const double t = clampd(dot(sub(p, a), dir) / dot(dir, dir), 0.0, 1.0);
    const v3 point = add(a, muls(dir, t));
    st3(out, point); out[3] = norm(sub(p, point));
}

/* ------------------------------------------------------------------------ */
/* Contact pair oracle, oracle.cpp:11-24                                     */

typedef struct { uint64_t key; uint32_t idx; } keyidx;
static int cmp_keyidx(const void* a, const void* b) {
    const keyidx* x = (const keyidx*)a; const keyidx* y = (const keyidx*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
typedef struct { uint32_t i, j; } pairu;
static int cmp_pair(const void* a, const void* b) {
    const pairu* x = (const pairu*)a; const pairu* y = (const pairu*)b;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j);
}

int64_t orc_contact_pairs(size_t n, const double* pos, const double* rad, int binned,
                          uint32_t* out_i, uint32_t* out_j, int64_t cap) {
    int64_t count = 0;
#define EMIT(I, J) do { if (count < cap) { out_i[count] = (uint32_t)(I); out_j[count] = (uint32_t)(J); } ++count; } while (0)
    if (!binned) {
        for (size_t i = 0; i < n; ++i)
            for (size_t j = i + 1; j < n; ++j) {
                const double dist = norm(sub(ld3(pos + 3 * j), ld3(pos + 3 * i)));
                if (dist < rad[i] + rad[j]) EMIT(i, j);
            }
        return count <= cap ? count : -count;
    }
    /* Independent grid (cell >= max reach): any pair with dist < r_i + r_j <= 2 r_max lies in
     * adjacent cells, so this enumerates exactly the same set with the same test. */
    double rmax = 0.0, lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (size_t i = 0; i < n; ++i) {
        if (rad[i] > rmax) rmax = rad[i];
        for (int a = 0; a < 3; ++a) {
            if (pos[3 * i + a] < lo[a]) lo[a] = pos[3 * i + a];
            if (pos[3 * i + a] > hi[a]) hi[a] = pos[3 * i + a];
        }
    }
    if (n == 0) return 0;
    const double h = 2.0 * rmax * 1.01 + 1e-300;
    int64_t dim[3];
    for (int a = 0; a < 3; ++a) dim[a] = (int64_t)floor((hi[a] - lo[a]) / h) + 1;
    keyidx* ki = (keyidx*)malloc(n * sizeof(keyidx));
    int64_t* cc = (int64_t*)malloc(n * 3 * sizeof(int64_t));
    for (size_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            int64_t c = (int64_t)floor((pos[3 * i + a] - lo[a]) / h);
            if (c < 0) c = 0;
            if (c >= dim[a]) c = dim[a] - 1;
            cc[3 * i + a] = c;
        }
        ki[i].key = (uint64_t)(cc[3 * i] + dim[0] * (cc[3 * i + 1] + dim[1] * cc[3 * i + 2]));
        ki[i].idx = (uint32_t)i;
    }
    qsort(ki, n, sizeof(keyidx), cmp_keyidx);
    pairu* pr = NULL; int64_t pcap = 0;
    for (size_t i = 0; i < n; ++i) {
        for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
            const int64_t x = cc[3 * i] + dx, y = cc[3 * i + 1] + dy, z = cc[3 * i + 2] + dz;
            if (x < 0 || y < 0 || z < 0 || x >= dim[0] || y >= dim[1] || z >= dim[2]) continue;
            const uint64_t key = (uint64_t)(x + dim[0] * (y + dim[1] * z));
            /* lower bound */
            size_t a = 0, b = n;
            while (a < b) { size_t m = (a + b) / 2; if (ki[m].key < key) a = m + 1; else b = m; }
            for (size_t q = a; q < n && ki[q].key == key; ++q) {
                const size_t j = ki[q].idx;
                if (j <= i) continue;
                const double dist = norm(sub(ld3(pos + 3 * j), ld3(pos + 3 * i)));
                if (dist < rad[i] + rad[j]) {
                    if (count >= pcap) { pcap = pcap ? 2 * pcap : 1024; pr = (pairu*)realloc(pr, pcap * sizeof(pairu)); }
                    pr[count].i = (uint32_t)i; pr[count].j = (uint32_t)j; ++count;
                }
            }
        }
    }
    qsort(pr, count, sizeof(pairu), cmp_pair);
    for (int64_t k = 0; k < count && k < cap; ++k) { out_i[k] = pr[k].i; out_j[k] = pr[k].j; }
    free(pr); free(ki); free(cc);
#undef EMIT
    return count <= cap ? count : -count;
}

/* ------------------------------------------------------------------------ */
/* History keyed by stable ids (replaces ContactTable rows, contact_table.cpp:15-63) */

static int cmp_hist(const void* a, const void* b) {
    const orc_hist* x = (const orc_hist*)a; const orc_hist* y = (const orc_hist*)b;
    if (x->owner_id != y->owner_id) return x->owner_id < y->owner_id ? -1 : 1;
    return x->partner_key < y->partner_key ? -1 : (x->partner_key > y->partner_key);
}

/* [lo, hi) range of owner in a (owner, partner)-sorted history */
static void hist_owner_range(const orc_hist* h, int64_t n, uint32_t owner, int64_t* lo, int64_t* hi) {
    int64_t a = 0, b = n;
    while (a < b) { int64_t m = (a + b) / 2; if (h[m].owner_id < owner) a = m + 1; else b = m; }
    *lo = a;
    b = n;
    while (a < b) { int64_t m = (a + b) / 2; if (h[m].owner_id <= owner) a = m + 1; else b = m; }
    *hi = a;
}

static const orc_hist* hist_find(const orc_hist* h, int64_t lo, int64_t hi, uint32_t key) {
    for (int64_t k = lo; k < hi; ++k) if (h[k].partner_key == key) return &h[k];
    return NULL;
}

static inline uint32_t wall_key(int w) { return (uint32_t)(int32_t)(-(w + 1)); } /* contact_table.hpp:35 */

/* Per-material-pair tables, pipeline.cpp:70-78 + materials.cpp:58-68 */
typedef struct {
    uint32_t m;
    orc_material* mats;
    double* alpha;  /* m*m */
    double* mu;     /* m*m */
    double* rest;   /* m*m */
} mat_tables;

static void build_tables(const orc_config* cfg, mat_tables* t) {
    const uint32_t m = cfg->material_count;
    t->m = m;
    t->mats = (orc_material*)malloc(m * sizeof(orc_material));
    memcpy(t->mats, cfg->materials, m * sizeof(orc_material));
    t->alpha = (double*)malloc(m * m * sizeof(double));
    t->mu = (double*)malloc(m * m * sizeof(double));
    t->rest = (double*)malloc(m * m * sizeof(double));
    for (uint32_t a = 0; a < m; ++a)
        for (uint32_t b = 0; b < m; ++b) {
            const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
            const double e = cfg->pair_restitution ? cfg->pair_restitution[a * m + b]
                                                   : sqrt(t->mats[lo].restitution * t->mats[hi].restitution);
            t->rest[a * m + b] = e;
            t->alpha[a * m + b] = orc_restitution_alpha(e);
            t->mu[a * m + b] = sqrt(t->mats[a].sliding_friction * t->mats[b].sliding_friction);
        }
}
static void free_tables(mat_tables* t) { free(t->mats); free(t->alpha); free(t->mu); free(t->rest); }

/* ------------------------------------------------------------------------ */
/* oracle_collide, oracle.cpp:47-105                                         */

typedef struct { int visit; uint32_t j; } cand;

int64_t orc_collide(size_t n, const uint32_t* ids, const double* pos, const double* vel,
                    const double* omg, const double* rad, const double* mass,
                    const uint32_t* mat, const orc_config* cfg, const orc_grid* grid,
                    const orc_hist* hist_in, int64_t hist_in_count, double* forces,
                    double* torques, orc_hist* hist_out, uint32_t* ev_owner,
                    uint32_t* ev_partner, int64_t cap) {
    mat_tables T;
    build_tables(cfg, &T);
    const int K = cfg->contact_capacity;
    orc_hist* old = (orc_hist*)malloc((hist_in_count + 1) * sizeof(orc_hist));
    if (hist_in_count) memcpy(old, hist_in, hist_in_count * sizeof(orc_hist));
    qsort(old, hist_in_count, sizeof(orc_hist), cmp_hist);

    /* oracle.cpp:35-43: per-particle cells by the documented rule */
    int* cell = (int*)malloc(n * 3 * sizeof(int));
    const double inv_h = 1.0 / grid->cell_size;
    const int dims[3] = {grid->nx, grid->ny, grid->nz};
    for (size_t i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            int c = to_int_x86(floor((pos[3 * i + a] - grid->origin[a]) * inv_h));
            int dummy = 0;
            cell[3 * i + a] = clamp_axis(c, dims[a], &dummy);
        }
    /* Bin by cell (equivalent to the O(N^2) scan: candidates sorted by (visit, slot)). */
    keyidx* ki = (keyidx*)malloc((n + 1) * sizeof(keyidx));
    for (size_t i = 0; i < n; ++i) {
        ki[i].key = (uint64_t)linear_index(grid, cell[3 * i], cell[3 * i + 1], cell[3 * i + 2]);
        ki[i].idx = (uint32_t)i;
    }
    qsort(ki, n, sizeof(keyidx), cmp_keyidx);

    memset(forces, 0, 3 * n * sizeof(double));
    memset(torques, 0, 3 * n * sizeof(double));
    int64_t events = 0, touched = 0;
    int64_t rc = 0;
    cand* cands = (cand*)malloc(4096 * sizeof(cand));
    size_t ccap = 4096;
    for (size_t i = 0; i < n && rc == 0; ++i) {
        size_t nc = 0;
        for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
            const int x = cell[3 * i] + dx, y = cell[3 * i + 1] + dy, z = cell[3 * i + 2] + dz;
            if (x < 0 || y < 0 || z < 0 || x >= dims[0] || y >= dims[1] || z >= dims[2]) continue;
            const uint64_t key = linear_index(grid, x, y, z);
            size_t a = 0, b = n;
            while (a < b) { size_t m = (a + b) / 2; if (ki[m].key < key) a = m + 1; else b = m; }
            const int visit = ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1);
            for (size_t q = a; q < n && ki[q].key == key; ++q) {
                if (ki[q].idx == i) continue;
                if (nc == ccap) { ccap *= 2; cands = (cand*)realloc(cands, ccap * sizeof(cand)); }
                cands[nc].visit = visit; cands[nc].j = ki[q].idx; ++nc;
            }
        }
        /* already in (visit, slot) order: visits ascend with the loop, slots ascend per cell */
        int64_t olo, ohi;
        hist_owner_range(old, hist_in_count, ids[i], &olo, &ohi);
        int row_live = (int)(ohi - olo);
        for (size_t c = 0; c < nc; ++c) {
            const uint32_t j = cands[c].j;
            double g[10];
            const int hit = orc_contact_geometry(pos + 3 * i, rad[i], vel + 3 * i, omg + 3 * i,
                                                 pos + 3 * j, 0, rad[j], vel + 3 * j, omg + 3 * j, g);
            if (hit < 0) { rc = -ORC_ERR_DEGENERATE; break; }
            if (!hit) continue;
            const uint32_t mi = mat[i], mj = mat[j];
            double co[4];
            orc_contact_coefficients(g[3], &T.mats[mi], &T.mats[mj], rad[i], rad[j], mass[i], mass[j],
                                     orc_restitution_alpha(T.rest[mi * T.m + mj]), 0, co);
            const orc_hist* h = hist_find(old, olo, ohi, ids[j]);
            double d0[3] = {0.0, 0.0, 0.0};
            if (h) { d0[0] = h->delta_t[0]; d0[1] = h->delta_t[1]; d0[2] = h->delta_t[2]; }
            else if (++row_live > K) { rc = -ORC_ERR_CAPACITY; break; }
            double dt_[3];
            orc_update_tangential(d0, g, g + 7, cfg->dt, dt_);
            double f[12];
            orc_contact_force(g, co, dt_, T.mu[mi * T.m + mj], rad[i], f);
            st3(forces + 3 * i, add(ld3(forces + 3 * i), ld3(f)));
            st3(torques + 3 * i, add(ld3(torques + 3 * i), ld3(f + 3)));
            if (events < cap) {
                ev_owner[events] = (uint32_t)i; ev_partner[events] = j;
                hist_out[touched].owner_id = ids[i]; hist_out[touched].partner_key = ids[j];
                hist_out[touched].delta_t[0] = f[6]; hist_out[touched].delta_t[1] = f[7];
                hist_out[touched].delta_t[2] = f[8];
            }
            ++events; ++touched;
        }
    }
    free(cands); free(ki); free(cell); free(old); free_tables(&T);
    if (rc) return rc;
    return events <= cap ? events : -ORC_ERR_BUFFER;
}

/* ------------------------------------------------------------------------ */
/* Periodic boundaries and Lees-Edwards shear. The reference has neither (grid.cpp:60-82
 * clips at the box); this is the repo's own specification, restated here
 * independently of the GPU code. With no periodic axis every function below is bypassed, so
 * the step is the reference's bit for bit. */
typedef struct {
    uint32_t mask;                 /* bit k: axis k periodic */
    double lo[3], L[3], half[3];   /* box origin, length, L/2 */
    double inv[3];                 /* 1 / cell extent per axis */
    int n[3];
    double rate, U;                /* shear rate, image velocity rate * L_y */
    int64_t le_steps;              /* integrates so far */
    double delta;                  /* image offset of the upper box along x */
} pbox;

static void pb_update_delta(pbox* b, double dt) {
    const double t = (double)b->le_steps * dt;
    const double d = b->U * t;
    b->delta = d - b->L[0] * floor(d / b->L[0]);
}

/* wrap a position (and the LE velocity jump) back into the box after integration */
static void pb_wrap(const pbox* b, double* p, double* v) {
    if (b->mask & 2u) {
        const double ky = floor((p[1] - b->lo[1]) / b->L[1]);
        if (ky != 0.0) {
            p[1] = p[1] - b->L[1] * ky;
            if (b->rate != 0.0) { p[0] = p[0] - b->delta * ky; v[0] = v[0] - b->U * ky; }
        }
    }
    if (b->mask & 1u) {
        const double kx = floor((p[0] - b->lo[0]) / b->L[0]);
        if (kx != 0.0) p[0] = p[0] - b->L[0] * kx;
    }
    if (b->mask & 4u) {
        const double kz = floor((p[2] - b->lo[2]) / b->L[2]);
        if (kz != 0.0) p[2] = p[2] - b->L[2] * kz;
    }
}

/* cell key with per-axis extents; periodic axes clamp silently (rounding at the upper face) */
static uint32_t pb_hash(const pbox* b, const orc_grid* g, const double p[3], int* clamped) {
    int c[3];
    const int dims[3] = {g->nx, g->ny, g->nz};
    int cl = 0;
    for (int k = 0; k < 3; ++k) {
        const double rel = p[k] - g->origin[k];
        int ck = to_int_x86(floor(rel * b->inv[k]));
        if (b->mask & (1u << k)) ck = ck < 0 ? 0 : (ck >= dims[k] ? dims[k] - 1 : ck);
        else ck = clamp_axis(ck, dims[k], &cl);
        c[k] = ck;
    }
    if (clamped) *clamped = cl;
    return linear_index(g, c[0], c[1], c[2]);
}

/* minimum-image displacement partner - owner, plus the x velocity of the partner's image */
static v3 pb_min_image(const pbox* b, v3 d, double* dvx) {
    *dvx = 0.0;
    if (b->mask & 2u) {
        if (d.y > b->half[1]) {
            d.y = d.y - b->L[1];
            if (b->rate != 0.0) { d.x = d.x - b->delta; *dvx = -b->U; }
        } else if (d.y < -b->half[1]) {
            d.y = d.y + b->L[1];
            if (b->rate != 0.0) { d.x = d.x + b->delta; *dvx = b->U; }
        }
    }
    if ((b->mask & 1u) && fabs(d.x) > b->half[0]) d.x = d.x - b->L[0] * rint(d.x / b->L[0]);
    if ((b->mask & 4u) && fabs(d.z) > b->half[2]) d.z = d.z - b->L[2] * rint(d.z / b->L[2]);
    return d;
}

/* Candidate cells of an owner cell as x-ranges [xa, xb] of rows (y, z), in visit order: z, y
 * outer to inner (dz, dy = -1, 0, 1, wrapped on periodic axes, clipped otherwise), then x
 * ascending from the row's first cell: cx-1 .. cx+1, or, on a row seen through the sheared
 * y-boundary, the 4 cells lo .. lo+3 with lo = floor((cx-1) - s/e_x), s = -+delta the image
 * offset. Wrapped x splits a row into two ranges. Returns the number of ranges (<= 18). */
static int pb_ranges(const pbox* b, const orc_grid* g, uint32_t cell, int out[18][4]) {
    const int nx = g->nx, ny = g->ny, nz = g->nz;
    const int cx = (int)(cell % (uint32_t)nx);
    const int rest = (int)(cell / (uint32_t)nx);
    const int cy = rest % ny, cz = rest / ny;
    int cnt = 0;
    for (int dz = -1; dz <= 1; ++dz) {
        int z = cz + dz;
        if (z < 0 || z >= nz) {
            if (!(b->mask & 4u)) continue;
            z = (z + nz) % nz;
        }
        for (int dy = -1; dy <= 1; ++dy) {
            int y = cy + dy, ysh = 0;
            if (y < 0 || y >= ny) {
                if (!(b->mask & 2u)) continue;
                ysh = y < 0 ? -1 : 1;
                y = (y + ny) % ny;
            }
            int xa, xb;
            if (ysh != 0 && b->rate != 0.0) {
                const double sx = ysh < 0 ? -b->delta : b->delta;
                xa = (int)floor((double)(cx - 1) - sx * b->inv[0]);
                xb = xa + 3;
            } else {
                xa = cx - 1; xb = cx + 1;
                if (!(b->mask & 1u)) { if (xa < 0) xa = 0; if (xb >= nx) xb = nx - 1; }
            }
            if (!(b->mask & 1u)) {
                out[cnt][0] = xa; out[cnt][1] = xb; out[cnt][2] = y; out[cnt][3] = z; ++cnt;
                continue;
            }
            const int wa = ((xa % nx) + nx) % nx;
            const int wb = wa + (xb - xa);
            if (wb < nx) {
                out[cnt][0] = wa; out[cnt][1] = wb; out[cnt][2] = y; out[cnt][3] = z; ++cnt;
            } else {
                out[cnt][0] = wa; out[cnt][1] = nx - 1; out[cnt][2] = y; out[cnt][3] = z; ++cnt;
                out[cnt][0] = 0; out[cnt][1] = wb - nx; out[cnt][2] = y; out[cnt][3] = z; ++cnt;
            }
        }
    }
    return cnt;
}

/* ------------------------------------------------------------------------ */
/* Full step, pipeline.cpp:31-378, with canonical in-cell order by stable id */

struct orc_sim {
    double dt, g[3];
    orc_config cfg;
    mat_tables T;
    orc_rect* rects; uint32_t nrect;
    orc_line* lines; uint32_t nline;
    int K;
    orc_grid grid;
    size_t n;
    uint32_t *ids, *mat, *keys;
    double *pos, *vel, *omg, *rad, *mass, *F, *Tq;
    double *Fabs, *Tabs; /* per particle: sum of |contribution| (the 1e-9 parity scale) */
    orc_hist* hist; int64_t nhist, hcap;
    int64_t step_index, clamps;
    /* per-particle counters for metrics */
    uint32_t *pp_count, *wall_count;
    double* fric;
    /* scratch */
    uint32_t *cstart, *cend;
    pbox pb;
};

size_t orc_sim_size(const orc_sim* s) { return s->n; }

static void set_err(orc_error* e, int code, int kernel, uint32_t slot, uint32_t id, int64_t step) {
    if (!e) return;
    e->code = code; e->kernel = kernel; e->particle_slot = slot; e->particle_id = id; e->step = step;
}

static int g_sort_n;
static const uint32_t* g_sort_keys;
static const uint32_t* g_sort_ids;
static int cmp_canonical(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    if (g_sort_keys[x] != g_sort_keys[y]) return g_sort_keys[x] < g_sort_keys[y] ? -1 : 1;
    return g_sort_ids[x] < g_sort_ids[y] ? -1 : (g_sort_ids[x] > g_sort_ids[y]);
}

#define PERMUTE(arr, type, width)                                                  \
    do {                                                                           \
        type* tmp = (type*)malloc(s->n * (width) * sizeof(type));                  \
        for (size_t q = 0; q < s->n; ++q)                                          \
            for (int w = 0; w < (width); ++w) tmp[q * (width) + w] = s->arr[perm[q] * (width) + w]; \
        free(s->arr); s->arr = tmp;                                                \
    } while (0)

typedef struct { int64_t contacts, pp; int32_t maxc; double fric; } phase_acc;

/* apply_pair_contact / apply_wall_contact, pipeline.cpp:155-180, 244-270 */
static int apply_contact(orc_sim* s, size_t i, const double g[10], uint32_t mi, uint32_t mj,
                         double rj, double mj_mass, int wall, uint32_t pkey, const orc_hist* old,
                         int64_t olo, int64_t ohi, int* row_live, orc_hist* out, int64_t* nout) {
    const double* co_alpha = &s->T.alpha[mi * s->T.m + mj];
    double co[4];
    orc_contact_coefficients(g[3], &s->T.mats[mi], &s->T.mats[mj], s->rad[i], rj, s->mass[i], mj_mass,
                             *co_alpha, wall, co);
    const orc_hist* h = hist_find(old, olo, ohi, pkey);
    double d0[3] = {0.0, 0.0, 0.0};
    if (h) { d0[0] = h->delta_t[0]; d0[1] = h->delta_t[1]; d0[2] = h->delta_t[2]; }
    else if (++*row_live > s->K) return ORC_ERR_CAPACITY;
    double dt_[3];
    orc_update_tangential(d0, g, g + 7, s->dt, dt_);
    const double mu = s->T.mu[mi * s->T.m + mj];
    double f[12];
    orc_contact_force(g, co, dt_, mu, s->rad[i], f);
    st3(s->F + 3 * i, add(ld3(s->F + 3 * i), ld3(f)));
    st3(s->Tq + 3 * i, add(ld3(s->Tq + 3 * i), ld3(f + 3)));
    s->Fabs[i] += norm(ld3(f));
    s->Tabs[i] += norm(ld3(f + 3));
    if (wall) ++s->wall_count[i]; else ++s->pp_count[i];
    const double limit = mu * f[9];
    if (limit > 0.0) {
        const double r = f[10] / limit;
        if (r > s->fric[i]) s->fric[i] = r;   /* std::max(fric, r) */
    }
    out[*nout].owner_id = s->ids[i]; out[*nout].partner_key = pkey;
    out[*nout].delta_t[0] = f[6]; out[*nout].delta_t[1] = f[7]; out[*nout].delta_t[2] = f[8];
    ++*nout;
    return ORC_OK;
}

int orc_sim_force_phase(orc_sim* s, int flags, orc_metrics* m, orc_error* err) {
    const size_t n = s->n;
    const int64_t step = s->step_index;
    /* Integrate, pipeline.cpp:31-44 */
    if (flags & ORC_PH_INTEGRATE) ++s->pb.le_steps;
    if (s->pb.mask) pb_update_delta(&s->pb, s->dt);
    if (flags & ORC_PH_INTEGRATE) {
        for (size_t i = 0; i < n; ++i) {
            const v3 f = ld3(s->F + 3 * i), t = ld3(s->Tq + 3 * i);
            if (!finite3(f) || !finite3(t)) {
                set_err(err, ORC_ERR_KERNEL, ORC_K_INTEGRATE, (uint32_t)i, s->ids[i], step);
                return ORC_ERR_KERNEL;
            }
            const double m_ = s->mass[i];
            v3 v = add(ld3(s->vel + 3 * i), muls(f, s->dt / m_));
            st3(s->vel + 3 * i, v);
            st3(s->pos + 3 * i, add(ld3(s->pos + 3 * i), muls(v, s->dt)));
            const double inertia = 0.4 * m_ * s->rad[i] * s->rad[i];
            st3(s->omg + 3 * i, add(ld3(s->omg + 3 * i), muls(t, s->dt / inertia)));
            if (s->pb.mask) pb_wrap(&s->pb, s->pos + 3 * i, s->vel + 3 * i);
        }
    }
    /* CalcHash, pipeline.cpp:107-121 */
    int64_t clamps = 0;
    for (size_t i = 0; i < n; ++i) {
        int cl = 0;
        s->keys[i] = s->pb.mask ? pb_hash(&s->pb, &s->grid, s->pos + 3 * i, &cl)
                                : orc_calc_hash(s->pos + 3 * i, &s->grid, &cl);
        clamps += cl;
    }
    s->clamps = clamps;
    /* Sort: canonical (cell key, stable id) order — replaces the bitonic network whose tie
     * order is network-defined (bitonic_sort.cpp:16-63). */
    uint32_t* perm = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    g_sort_keys = s->keys; g_sort_ids = s->ids; g_sort_n = (int)n;
    qsort(perm, n, sizeof(uint32_t), cmp_canonical);
    /* FindCellBoundsAndReorder, sorted_order.cpp:17-29 + particle_set.cpp:30-38 */
    PERMUTE(ids, uint32_t, 1); PERMUTE(mat, uint32_t, 1); PERMUTE(keys, uint32_t, 1);
    PERMUTE(pos, double, 3); PERMUTE(vel, double, 3); PERMUTE(omg, double, 3);
    PERMUTE(rad, double, 1); PERMUTE(mass, double, 1);
    free(perm);
    const int64_t M = (int64_t)s->grid.nx * s->grid.ny * s->grid.nz;
    memset(s->cstart, 0, M * sizeof(uint32_t));
    memset(s->cend, 0, M * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) {
        const uint32_t c = s->keys[i];
        if (i == 0 || s->keys[i - 1] != c) s->cstart[c] = (uint32_t)i;
        if (i + 1 == n || s->keys[i + 1] != c) s->cend[c] = (uint32_t)(i + 1);
    }
    /* zero_forces + ForceGravity, pipeline.cpp:137-139, 46-50 */
    memset(s->F, 0, 3 * n * sizeof(double));
    memset(s->Tq, 0, 3 * n * sizeof(double));
    memset(s->Fabs, 0, n * sizeof(double));
    memset(s->Tabs, 0, n * sizeof(double));
    if (flags & ORC_PH_GRAVITY) {
        const v3 g = ld3(s->g);
        for (size_t i = 0; i < n; ++i) {
            st3(s->F + 3 * i, add(ld3(s->F + 3 * i), muls(g, s->mass[i])));
            s->Fabs[i] = norm(muls(g, s->mass[i]));
        }
    }
    /* InitializeContactIDs (sweep): the live entries are exactly the previous phase's touched
     * ones, which is what s->hist holds (contact_table.cpp:37-46). */
    orc_hist* old = s->hist;
    const int64_t nold = s->nhist;
    orc_hist* out = (orc_hist*)malloc((size_t)(n * (size_t)s->K + 1) * sizeof(orc_hist));
    int64_t nout = 0;
    memset(s->pp_count, 0, n * sizeof(uint32_t));
    memset(s->wall_count, 0, n * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) s->fric[i] = 0.0;
    int* row_live = (int*)malloc((n + 1) * sizeof(int));
    int64_t* olo = (int64_t*)malloc((n + 1) * sizeof(int64_t));
    int64_t* ohi = (int64_t*)malloc((n + 1) * sizeof(int64_t));
    for (size_t i = 0; i < n; ++i) {
        hist_owner_range(old, nold, s->ids[i], &olo[i], &ohi[i]);
        row_live[i] = (int)(ohi[i] - olo[i]);
    }
    int rc = ORC_OK;
    /* Collide (two-phase), pipeline.cpp:182-242 */
    if (flags & ORC_PH_PP) {
        uint32_t* local = (uint32_t*)malloc(((size_t)s->K + 1) * sizeof(uint32_t));
        for (size_t i = 0; i < n && rc == ORC_OK && s->pb.mask; ++i) {
            int rg[18][4];
            const int nrg = pb_ranges(&s->pb, &s->grid, s->keys[i], rg);
            int cnt = 0;
            const v3 pi = ld3(s->pos + 3 * i);
            const double zero3[3] = {0.0, 0.0, 0.0};
            for (int c = 0; c < nrg && rc == ORC_OK; ++c) {
                const uint32_t ka = linear_index(&s->grid, rg[c][0], rg[c][2], rg[c][3]);
                const uint32_t kb = linear_index(&s->grid, rg[c][1], rg[c][2], rg[c][3]);
                for (uint32_t cc = ka; cc <= kb && rc == ORC_OK; ++cc)
                for (uint32_t j = s->cstart[cc]; j < s->cend[cc]; ++j) {
                    if (j == i) continue;
                    double dvx;
                    const v3 diff = pb_min_image(&s->pb, sub(ld3(s->pos + 3 * j), pi), &dvx);
                    const double reach = s->rad[i] + s->rad[j];
                    const double reach2 = reach * reach;
                    if (dot(diff, diff) >= reach2 + reach2 * 1e-9) continue;
                    double dd[3], vj[3], g[10];
                    st3(dd, diff);
                    st3(vj, ld3(s->vel + 3 * j));
                    if (dvx != 0.0) vj[0] = vj[0] + dvx;
                    const int hit = orc_contact_geometry(zero3, s->rad[i], s->vel + 3 * i, s->omg + 3 * i, dd, 0,
                                                         s->rad[j], vj, s->omg + 3 * j, g);
                    if (hit < 0) {
                        set_err(err, ORC_ERR_DEGENERATE, ORC_K_COLLIDE, (uint32_t)i, s->ids[i], step);
                        rc = ORC_ERR_DEGENERATE; break;
                    }
                    if (!hit) continue;
                    if (cnt >= s->K) {
                        set_err(err, ORC_ERR_CAPACITY, ORC_K_COLLIDE, (uint32_t)i, s->ids[i], step);
                        rc = ORC_ERR_CAPACITY; break;
                    }
                    local[cnt++] = j;
                }
            }
            for (int c = 0; c < cnt && rc == ORC_OK; ++c) {
                const uint32_t j = local[c];
                double dvx, dd[3], vj[3], g[10];
                st3(dd, pb_min_image(&s->pb, sub(ld3(s->pos + 3 * j), pi), &dvx));
                st3(vj, ld3(s->vel + 3 * j));
                if (dvx != 0.0) vj[0] = vj[0] + dvx;
                orc_contact_geometry(zero3, s->rad[i], s->vel + 3 * i, s->omg + 3 * i, dd, 0, s->rad[j], vj,
                                     s->omg + 3 * j, g);
                if (apply_contact(s, i, g, s->mat[i], s->mat[j], s->rad[j], s->mass[j], 0, s->ids[j],
                                  old, olo[i], ohi[i], &row_live[i], out, &nout) != ORC_OK) {
                    set_err(err, ORC_ERR_CAPACITY, ORC_K_COLLIDE, (uint32_t)i, s->ids[i], step);
                    rc = ORC_ERR_CAPACITY;
                }
            }
        }
        for (size_t i = 0; i < n && rc == ORC_OK && !s->pb.mask; ++i) {
            uint32_t cells[27];
            const int nc = orc_neighbor_cells(s->keys[i], &s->grid, cells);
            int cnt = 0;
            const v3 pi = ld3(s->pos + 3 * i);
            for (int c = 0; c < nc && rc == ORC_OK; ++c) {
                for (uint32_t j = s->cstart[cells[c]]; j < s->cend[cells[c]]; ++j) {
                    if (j == i) continue;
                    /* check_pair, pipeline.cpp:143-153 */
                    const v3 diff = sub(ld3(s->pos + 3 * j), pi);
                    const double reach = s->rad[i] + s->rad[j];
                    const double reach2 = reach * reach;
                    if (dot(diff, diff) >= reach2 + reach2 * 1e-9) continue;
                    double g[10];
                    const int hit = orc_contact_geometry(s->pos + 3 * i, s->rad[i], s->vel + 3 * i,
                                                         s->omg + 3 * i, s->pos + 3 * j, 0, s->rad[j],
                                                         s->vel + 3 * j, s->omg + 3 * j, g);
                    if (hit < 0) {
                        set_err(err, ORC_ERR_DEGENERATE, ORC_K_COLLIDE, (uint32_t)i, s->ids[i], step);
                        rc = ORC_ERR_DEGENERATE; break;
                    }
                    if (!hit) continue;
                    if (cnt >= s->K) {
                        set_err(err, ORC_ERR_CAPACITY, ORC_K_COLLIDE, (uint32_t)i, s->ids[i], step);
                        rc = ORC_ERR_CAPACITY; break;
                    }
                    local[cnt++] = j;
                }
            }
            for (int c = 0; c < cnt && rc == ORC_OK; ++c) {
                const uint32_t j = local[c];
                double g[10];
                orc_contact_geometry(s->pos + 3 * i, s->rad[i], s->vel + 3 * i, s->omg + 3 * i,
                                     s->pos + 3 * j, 0, s->rad[j], s->vel + 3 * j, s->omg + 3 * j, g);
                if (apply_contact(s, i, g, s->mat[i], s->mat[j], s->rad[j], s->mass[j], 0, s->ids[j],
                                  old, olo[i], ohi[i], &row_live[i], out, &nout) != ORC_OK) {
                    set_err(err, ORC_ERR_CAPACITY, ORC_K_COLLIDE, (uint32_t)i, s->ids[i], step);
                    rc = ORC_ERR_CAPACITY;
                }
            }
        }
        free(local);
    }
    /* CollideRectangle, pipeline.cpp:272-289 */
    if (rc == ORC_OK && (flags & ORC_PH_RECT)) {
        for (size_t i = 0; i < n && rc == ORC_OK; ++i)
            for (uint32_t w = 0; w < s->nrect; ++w) {
                double cp[4];
                orc_closest_point_rect(s->pos + 3 * i, &s->rects[w], cp);
                if (cp[3] >= s->rad[i]) continue;
                double g[10];
                const int hit = orc_contact_geometry(s->pos + 3 * i, s->rad[i], s->vel + 3 * i,
                                                     s->omg + 3 * i, cp, 1, 0.0, NULL, NULL, g);
                if (hit < 0) { set_err(err, ORC_ERR_DEGENERATE, ORC_K_COLLIDE_RECT, (uint32_t)i, s->ids[i], step); rc = ORC_ERR_DEGENERATE; break; }
                if (!hit) continue;
                if (apply_contact(s, i, g, s->mat[i], s->rects[w].material_id, 0.0, 0.0, 1, wall_key((int)w),
                                  old, olo[i], ohi[i], &row_live[i], out, &nout) != ORC_OK) {
                    set_err(err, ORC_ERR_CAPACITY, ORC_K_COLLIDE_RECT, (uint32_t)i, s->ids[i], step);
                    rc = ORC_ERR_CAPACITY; break;
                }
            }
    }
    /* CollideLine, pipeline.cpp:291-308 */
    if (rc == ORC_OK && (flags & ORC_PH_LINE)) {
        for (size_t i = 0; i < n && rc == ORC_OK; ++i)
            for (uint32_t w = 0; w < s->nline; ++w) {
                double cp[4];
                orc_closest_point_line(s->pos + 3 * i, &s->lines[w], cp);
                if (cp[3] >= s->rad[i]) continue;
                double g[10];
                const int hit = orc_contact_geometry(s->pos + 3 * i, s->rad[i], s->vel + 3 * i,
                                                     s->omg + 3 * i, cp, 1, 0.0, NULL, NULL, g);
                if (hit < 0) { set_err(err, ORC_ERR_DEGENERATE, ORC_K_COLLIDE_LINE, (uint32_t)i, s->ids[i], step); rc = ORC_ERR_DEGENERATE; break; }
                if (!hit) continue;
                if (apply_contact(s, i, g, s->mat[i], s->lines[w].material_id, 0.0, 0.0, 1,
                                  wall_key((int)(s->nrect + w)), old, olo[i], ohi[i], &row_live[i], out,
                                  &nout) != ORC_OK) {
                    set_err(err, ORC_ERR_CAPACITY, ORC_K_COLLIDE_LINE, (uint32_t)i, s->ids[i], step);
                    rc = ORC_ERR_CAPACITY; break;
                }
            }
    }
    free(row_live); free(olo); free(ohi);
    qsort(out, nout, sizeof(orc_hist), cmp_hist);
    free(s->hist);
    s->hist = out; s->nhist = nout;
    if (rc != ORC_OK) return rc;
    if (m) { /* pipeline.cpp:338-363 */
        m->step = step;
        m->clamps = s->clamps;
        int64_t contacts = 0, pp = 0; int32_t mx = 0; double fm = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const int per = (int)(s->pp_count[i] + s->wall_count[i]);
            contacts += per; pp += s->pp_count[i];
            if (per > mx) mx = per;
            if (s->fric[i] > fm) fm = s->fric[i];
        }
        m->contacts = contacts; m->pp_contact_events = pp; m->max_contacts_per_particle = mx;
        m->friction_max_ratio = fm;
    }
    return ORC_OK;
}

orc_sim* orc_sim_create(const orc_config* cfg, size_t n, const uint32_t* ids, const double* pos,
                        const double* vel, const double* omg, const double* rad,
                        const double* mass, const uint32_t* mat, orc_error* err) {
    orc_sim* s = (orc_sim*)calloc(1, sizeof(orc_sim));
    s->cfg = *cfg;
    s->dt = cfg->dt;
    s->g[0] = cfg->gravity[0]; s->g[1] = cfg->gravity[1]; s->g[2] = cfg->gravity[2];
    build_tables(cfg, &s->T);
    s->nrect = cfg->rect_count; s->nline = cfg->line_count;
    s->rects = (orc_rect*)malloc((s->nrect + 1) * sizeof(orc_rect));
    s->lines = (orc_line*)malloc((s->nline + 1) * sizeof(orc_line));
    if (s->nrect) memcpy(s->rects, cfg->rects, s->nrect * sizeof(orc_rect));
    if (s->nline) memcpy(s->lines, cfg->lines, s->nline * sizeof(orc_line));
    s->cfg.materials = s->T.mats; s->cfg.rects = s->rects; s->cfg.lines = s->lines;
    s->cfg.pair_restitution = NULL;
    s->K = cfg->contact_capacity;
    s->n = n;
#define ALLOC_COPY(dst, src, type, width) do { s->dst = (type*)malloc((n * (width) + 1) * sizeof(type)); memcpy(s->dst, src, n * (width) * sizeof(type)); } while (0)
    ALLOC_COPY(ids, ids, uint32_t, 1); ALLOC_COPY(mat, mat, uint32_t, 1);
    ALLOC_COPY(pos, pos, double, 3); ALLOC_COPY(vel, vel, double, 3); ALLOC_COPY(omg, omg, double, 3);
    ALLOC_COPY(rad, rad, double, 1); ALLOC_COPY(mass, mass, double, 1);
#undef ALLOC_COPY
    s->keys = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    s->F = (double*)calloc(3 * n + 1, sizeof(double));
    s->Tq = (double*)calloc(3 * n + 1, sizeof(double));
    s->Fabs = (double*)calloc(n + 1, sizeof(double));
    s->Tabs = (double*)calloc(n + 1, sizeof(double));
    s->pp_count = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    s->wall_count = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    s->fric = (double*)calloc(n + 1, sizeof(double));
    s->hist = (orc_hist*)malloc(sizeof(orc_hist)); s->nhist = 0; s->hcap = 1;
    double rmax = 0.0;
    for (size_t i = 0; i < n; ++i) if (rad[i] > rmax) rmax = rad[i];
    if (orc_make_grid(cfg->domain_min, cfg->domain_max, rmax, cfg->grid_cell_size, &s->grid) != ORC_OK) {
        set_err(err, ORC_ERR_CONFIG, -1, 0, 0, 0);
        orc_sim_destroy(s);
        return NULL;
    }
    /* periodic axes: n = floor(L / h) cells of extent L / n (>= h); n >= 3 (x: >= 4 with shear) */
    s->pb.mask = cfg->periodic & 7u;
    s->pb.rate = s->pb.mask ? cfg->shear_rate : 0.0;
    {
        int* dims[3] = {&s->grid.nx, &s->grid.ny, &s->grid.nz};
        int bad = (s->pb.rate != 0.0) && ((s->pb.mask & 3u) != 3u);
        for (int k = 0; k < 3; ++k) {
            s->pb.lo[k] = cfg->domain_min[k];
            s->pb.L[k] = cfg->domain_max[k] - cfg->domain_min[k];
            s->pb.half[k] = 0.5 * s->pb.L[k];
            s->pb.inv[k] = 1.0 / s->grid.cell_size;
            if (s->pb.mask & (1u << k)) {
                const int nk = (int)floor(s->pb.L[k] / s->grid.cell_size);
                if (nk < 3 || (k == 0 && s->pb.rate != 0.0 && nk < 4)) bad = 1;
                *dims[k] = nk < 1 ? 1 : nk;
                s->pb.inv[k] = 1.0 / (s->pb.L[k] / (double)nk);
            }
            s->pb.n[k] = *dims[k];
        }
        s->pb.U = s->pb.rate * s->pb.L[1];
        if (bad) {
            set_err(err, ORC_ERR_CONFIG, -1, 0, 0, 0);
            orc_sim_destroy(s);
            return NULL;
        }
    }
    const int64_t M = (int64_t)s->grid.nx * s->grid.ny * s->grid.nz;
    s->cstart = (uint32_t*)calloc(M + 1, sizeof(uint32_t));
    s->cend = (uint32_t*)calloc(M + 1, sizeof(uint32_t));
    /* priming force pass, pipeline.cpp:83 */
    if (orc_sim_force_phase(s, ORC_PH_GRAVITY | ORC_PH_PP | ORC_PH_RECT | ORC_PH_LINE, NULL, err) != ORC_OK) {
        orc_sim_destroy(s);
        return NULL;
    }
    return s;
}

void orc_sim_destroy(orc_sim* s) {
    if (!s) return;
    free_tables(&s->T); free(s->rects); free(s->lines);
    free(s->ids); free(s->mat); free(s->keys); free(s->pos); free(s->vel); free(s->omg);
    free(s->rad); free(s->mass); free(s->F); free(s->Tq); free(s->Fabs); free(s->Tabs); free(s->hist);
    free(s->pp_count); free(s->wall_count); free(s->fric); free(s->cstart); free(s->cend);
    free(s);
}

/* Simulation::step, pipeline.cpp:366-378 */
int orc_sim_step(orc_sim* s, int nsteps, orc_metrics* m, orc_error* err) {
    for (int k = 0; k < nsteps; ++k) {
        ++s->step_index;
        const int rc = orc_sim_force_phase(s, ORC_PH_ALL, m, err);
        if (rc != ORC_OK) return rc;
    }
    return ORC_OK;
}

void orc_sim_get_state(const orc_sim* s, uint32_t* ids, double* pos, double* vel, double* omg,
                       double* rad, double* mass, uint32_t* mat) {
    const size_t n = s->n;
    if (ids) memcpy(ids, s->ids, n * sizeof(uint32_t));
    if (pos) memcpy(pos, s->pos, 3 * n * sizeof(double));
    if (vel) memcpy(vel, s->vel, 3 * n * sizeof(double));
    if (omg) memcpy(omg, s->omg, 3 * n * sizeof(double));
    if (rad) memcpy(rad, s->rad, n * sizeof(double));
    if (mass) memcpy(mass, s->mass, n * sizeof(double));
    if (mat) memcpy(mat, s->mat, n * sizeof(uint32_t));
}
void orc_sim_get_forces(const orc_sim* s, double* f, double* t) {
    if (f) memcpy(f, s->F, 3 * s->n * sizeof(double));
    if (t) memcpy(t, s->Tq, 3 * s->n * sizeof(double));
}
void orc_sim_get_force_scale(const orc_sim* s, double* fabs_, double* tabs_) {
    memcpy(fabs_, s->Fabs, s->n * sizeof(double));
    memcpy(tabs_, s->Tabs, s->n * sizeof(double));
}
void orc_sim_get_keys(const orc_sim* s, uint32_t* k) { memcpy(k, s->keys, s->n * sizeof(uint32_t)); }
int64_t orc_sim_history_count(const orc_sim* s) { return s->nhist; }
void orc_sim_get_history(const orc_sim* s, orc_hist* out) { memcpy(out, s->hist, s->nhist * sizeof(orc_hist)); }
void orc_sim_get_grid(const orc_sim* s, orc_grid* g) { *g = s->grid; }
void orc_sim_get_pbox(const orc_sim* s, double ext[3], double* off, int64_t* steps) {
    for (int k = 0; k < 3; ++k) ext[k] = 1.0 / s->pb.inv[k];
    if (off) *off = s->pb.delta;
    if (steps) *steps = s->pb.le_steps;
}

/* ---- bench input generator (TEST INFRASTRUCTURE: the reference arm builds its inputs here so it
 * never loads the product library) ---------------------------------------------------------------
 * SURVEY.md §8d's G(N, s, jit, poly, seed): the reference benchmark packing shape
 * (benchmarks/bench_support.hpp:10-44) drawn with the reference's xorshift64* (rng.hpp:11-33).
 * Draw order per particle: jx, jy, jz, [r], vx, vy, vz, wx, wy, wz. Bitwise the same arrays as the
 * product's dem_gen_packing (tests/test_oracle_golden.py checks it). */
static uint64_t orc_xs_next(uint64_t* st) {                              /* rng.hpp:19-26 */
    uint64_t x = *st;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    *st = x;
    return x * 0x2545F4914F6CDD1DULL;
}
static double orc_xs_in(uint64_t* st, double lo, double hi) {            /* rng.hpp:28-33 */
    const double u = (double)(orc_xs_next(st) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

int orc_gen_packing(uint64_t n, double s, double jit, int poly, uint64_t seed, double omega_half,
                    uint32_t* ids, double* pos, double* vel, double* omg, double* rad, double* mass,
                    uint32_t* mat, double domain_max[3]) {
    const double r0 = 0.005, m0 = 1e-3, r_max = r0;
    const uint64_t side = (uint64_t)ceil(cbrt((double)n));
    const double spacing = s * r0;
    uint64_t st = seed != 0 ? seed : 0x9E3779B97F4A7C15ULL;              /* rng.hpp:13-15 */
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t ix = i % side, iy = (i / side) % side, iz = i / (side * side);
        const double jx = orc_xs_in(&st, -jit * r0, jit * r0);
        const double jy = orc_xs_in(&st, -jit * r0, jit * r0);
        const double jz = orc_xs_in(&st, -jit * r0, jit * r0);
        double r = r0, m = m0;
        if (poly) {
            r = r0 * orc_xs_in(&st, 0.5, 1.0);
            const double q = r / r0;
            m = m0 * q * q * q;
        }
        ids[i] = (uint32_t)i;
        pos[3 * i + 0] = 2.0 * r_max + (double)ix * spacing + jx;
        pos[3 * i + 1] = 2.0 * r_max + (double)iy * spacing + jy;
        pos[3 * i + 2] = 2.0 * r_max + (double)iz * spacing + jz;
        for (int a = 0; a < 3; ++a) vel[3 * i + a] = orc_xs_in(&st, -0.5, 0.5);
        for (int a = 0; a < 3; ++a) omg[3 * i + a] = orc_xs_in(&st, -omega_half, omega_half);
        rad[i] = r;
        mass[i] = m;
        mat[i] = 0;
    }
    domain_max[0] = domain_max[1] = domain_max[2] = (double)side * spacing + 4.0 * r_max;
    return 0;
}
