// dem_gen.cpp — synthetic packing generator G(N, s, jit, poly, seed) of SURVEY.md §8d.
//
// Same shape as the reference benchmark packing (benchmarks/bench_support.hpp:10-44), drawn
// with the reference's portable xorshift64* (core/include/demforge/rng.hpp:11-33) so that a
// seed names one packing on every host. Input generation only: it feeds identical arrays to the
// B200 path and to the reference CPU path; nothing here is on the timed path.
#include <cmath>
#include <cstdint>

#include "../../include/dem_b200_gen.h"

namespace {

struct XorShift64Star {  // rng.hpp:11-33
    uint64_t state;
    explicit XorShift64Star(uint64_t seed) : state(seed != 0 ? seed : 0x9E3779B97F4A7C15ULL) {}
    uint64_t next_u64() {
        uint64_t x = state;
        x ^= x >> 12;
        x ^= x << 25;
        x ^= x >> 27;
        state = x;
        return x * 0x2545F4914F6CDD1DULL;
    }
    double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_in(double lo, double hi) { return lo + (hi - lo) * next_unit(); }
};

}  // namespace

extern "C" int dem_gen_packing(uint64_t n, double s, double jit, int poly, uint64_t seed,
                               double omega_half, dem_particles* out, double domain_max[3]) {
    if (!out || out->count != n || !domain_max) return DEM_ERR_ARGUMENT;
    const double r0 = 0.005, m0 = 1e-3;
    const double r_max = r0;
    const int side = static_cast<int>(std::ceil(std::cbrt(static_cast<double>(n))));
    const double spacing = s * r0;
    XorShift64Star rng(seed);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t ix = i % side, iy = (i / side) % side, iz = i / (static_cast<uint64_t>(side) * side);
        const double jx = rng.next_in(-jit * r0, jit * r0);
        const double jy = rng.next_in(-jit * r0, jit * r0);
        const double jz = rng.next_in(-jit * r0, jit * r0);
        double r = r0, m = m0;
        if (poly) {
            r = r0 * rng.next_in(0.5, 1.0);
            const double q = r / r0;
            m = m0 * q * q * q;
        }
        out->ids[i] = static_cast<uint32_t>(i);
        out->positions[3 * i + 0] = 2.0 * r_max + static_cast<double>(ix) * spacing + jx;
        out->positions[3 * i + 1] = 2.0 * r_max + static_cast<double>(iy) * spacing + jy;
        out->positions[3 * i + 2] = 2.0 * r_max + static_cast<double>(iz) * spacing + jz;
        for (int a = 0; a < 3; ++a) out->velocities[3 * i + a] = rng.next_in(-0.5, 0.5);
        for (int a = 0; a < 3; ++a) out->angular_velocities[3 * i + a] = rng.next_in(-omega_half, omega_half);
        out->radii[i] = r;
        out->masses[i] = m;
        out->material_ids[i] = 0;
    }
    const double extent = side * spacing + 4.0 * r_max;
    domain_max[0] = domain_max[1] = domain_max[2] = extent;
    return DEM_OK;
}
