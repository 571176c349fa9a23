// dem_periodic.cuh — periodic boxes and Lees-Edwards shear, device side, shared
// by the step kernels (dem_kernels.cu) and the slab kernels (dem_slab.cu).
#pragma once

#include "dem_internal.h"
#include "dem_math.cuh"

namespace demb200 {

// Periodic boundaries and Lees-Edwards shear (flow x, gradient y). The reference has neither
// (grid.cpp:60-82 clips at the box); the specification is DESIGN.md §6 and the CPU
// restatement the parity tests use is oracle/dem_oracle.c (pb_*). With p.periodic == 0 none of
// this runs and the step is the reference's.

// Wrap an integrated position back into the box; crossing the y faces of a sheared box moves
// the particle by the image offset and its x velocity by the image velocity.
__device__ __forceinline__ void wrap_periodic(const StepParams& p, double delta, double4& pr, double4& vm) {
    if (p.periodic & 2u) {
        const double ky = floor((pr.y - p.oy) / p.Ly);
        if (ky != 0.0) {
            pr.y = pr.y - p.Ly * ky;
            if (p.shear_rate != 0.0) { pr.x = pr.x - delta * ky; vm.x = vm.x - p.shear_u * ky; }
        }
    }
    if (p.periodic & 1u) {
        const double kx = floor((pr.x - p.ox) / p.Lx);
        if (kx != 0.0) pr.x = pr.x - p.Lx * kx;
    }
    if (p.periodic & 4u) {
        const double kz = floor((pr.z - p.oz) / p.Lz);
        if (kz != 0.0) pr.z = pr.z - p.Lz * kz;
    }
}

// Minimum-image displacement partner - owner (d = Pj - Pi as the reference computes it, then
// corrected on periodic axes); *dvx receives the x velocity of the partner's image.
__device__ __forceinline__ V3 min_image(const StepParams& p, V3 d, double delta, double* dvx) {
    *dvx = 0.0;
    if (p.periodic & 2u) {
        if (d.y > p.half_y) {
            d.y = d.y - p.Ly;
            if (p.shear_rate != 0.0) { d.x = d.x - delta; *dvx = -p.shear_u; }
        } else if (d.y < -p.half_y) {
            d.y = d.y + p.Ly;
            if (p.shear_rate != 0.0) { d.x = d.x + delta; *dvx = p.shear_u; }
        }
    }
    if ((p.periodic & 1u) && fabs(d.x) > p.half_x) d.x = d.x - p.Lx * rint(d.x / p.Lx);
    if ((p.periodic & 4u) && fabs(d.z) > p.half_z) d.z = d.z - p.Lz * rint(d.z / p.Lz);
    return d;
}

// Lees-Edwards clock: `advance` counts one more integrate; the image offset of the upper box is
// Delta = U t - L_x floor(U t / L_x), U = rate L_y, t = le_steps dt (oracle pb_update_delta).
__device__ __forceinline__ void le_clock(const StepParams& p, DevCtl* ctl, bool advance) {
    if (advance) ctl->le_steps += 1;
    if (p.periodic) {
        const double t = static_cast<double>(ctl->le_steps) * p.dt;
        const double d = p.shear_u * t;
        ctl->le_delta = d - p.Lx * floor(d / p.Lx);
    }
}

}  // namespace demb200
