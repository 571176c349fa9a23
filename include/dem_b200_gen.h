/*
 * dem_b200_gen.h — synthetic input generator for the benchmark and parity configs
 * (SURVEY.md §8d generator G; template: reference benchmarks/bench_support.hpp:10-44,
 * RNG: core/include/demforge/rng.hpp:11-33). Not part of the drop-in boundary.
 */
#ifndef DEM_B200_GEN_H
#define DEM_B200_GEN_H

#include "dem_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* G(n, s, jit, poly, seed): lattice spacing s*r0 (r0 = 0.005 m, m0 = 1e-3 kg), jitter
 * U(-jit r0, jit r0) per axis, radius r0 or r0*U(0.5, 1) (poly, mass m0 (r/r0)^3),
 * v ~ U(-0.5, 0.5)^3, omega ~ U(-omega_half, omega_half)^3. Draw order per particle:
 * jx, jy, jz, [r], vx, vy, vz, wx, wy, wz. out->count must equal n and all arrays be sized.
 * domain_max receives the cube extent side*s*r0 + 4 r_max (domain_min = 0). */
int dem_gen_packing(uint64_t n, double s, double jit, int poly, uint64_t seed, double omega_half,
                    dem_particles* out, double domain_max[3]);

#ifdef __cplusplus
}
#endif
#endif
