// dem_slab.cu — slab domain decomposition kernels.
//
// A slab context owns the particles whose GLOBAL cell z lies in [z_lo, z_hi) and holds, for
// each step, a one-plane halo of neighbour particles (ghosts) below and above. Per step:
//   k_slab_migrate  integrate the owned particles (pipeline.cpp:31-44), classify them by their
//                   new cell plane, compact the stayers into the assembly buffer Y (carrying the
//                   index of their previous history row) and write leavers, with their history
//                   rows keyed by stable id, as migrant records for the neighbour;
//   k_slab_import   append received migrants to Y and their history rows to the import region;
//   k_slab_halo     write boundary-plane owned particles as ghost records for the neighbours;
//   k_slab_ghosts   append received ghosts to Y, flagged (idm.y bit 31).
// The force phase then bins Y (owned + ghosts) into X and detects / computes forces for owned
// slots only. Because the in-cell order is canonical (cell, stable id), every owned particle
// sees exactly the candidate sequence of a single-GPU run: results are bitwise identical to
// one GPU. The order in which records are written here (atomics) does not matter for that.
#include <cuda_runtime.h>

#include "dem_internal.h"
#include "dem_math.cuh"
#include "dem_periodic.cuh"

namespace demb200 {

namespace {

constexpr uint32_t kGhost = 0x80000000u;
constexpr uint32_t kGhostHi = 0x40000000u;  // the halo copy came from the z_hi side

__device__ __forceinline__ void raise_err(DevCtl* ctl, int kernel, uint32_t slot, uint32_t id, int code) {
    const unsigned long long key = (static_cast<unsigned long long>(kernel) << 56) |
                                   (static_cast<unsigned long long>(slot) << 8) | static_cast<unsigned long long>(code);
    atomicMin(&ctl->err_key, key);
    atomicMin(&ctl->err_sid[kernel], (static_cast<unsigned long long>(slot) << 32) | id);
    ctl->err_phase = ctl->phase;
}

// global cell plane of a position: the z part of calc_hash (grid.cpp:30-52)
__device__ __forceinline__ int cell_z(const StepParams& p, double z) {
    int cz = to_int_x86(floor((z - p.oz) * p.inv_z));
    return cz < 0 ? 0 : (cz >= p.nz ? p.nz - 1 : cz);
}

// warp-aggregated counter increment among lanes with the same `cls`
__device__ __forceinline__ uint32_t agg_add(uint32_t* ctr, int cls) {
    const unsigned active = __activemask();
    const unsigned peers = __match_any_sync(active, cls);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(ctr, static_cast<uint32_t>(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    return base + __popc(peers & ((1u << lane) - 1u));
}

__device__ __forceinline__ void put_state(StateBuf& y, uint32_t s, double4 pr, double4 vm, double4 om, uint2 idm) {
    st4(&y.pos_r[s], pr);
    st4(&y.vel_m[s], vm);
    st4(&y.omg[s], om);
    y.idm[s] = idm;
}

__device__ __forceinline__ void put_record(uint8_t* rec, double4 pr, double4 vm, double4 om, uint2 idm) {
    double4* d = reinterpret_cast<double4*>(rec);
    st4(&d[0], pr);
    st4(&d[1], vm);
    st4(&d[2], om);
    *reinterpret_cast<uint2*>(rec + 96) = idm;
}

template <bool INTEGRATE>
__global__ void __launch_bounds__(256) k_slab_migrate(StepParams p, SlabBufs s) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.n_x) return;
    const uint2 idm = s.X.idm[i];
    if (idm.y & kGhost) return;  // last step's halo copies are dropped
    double4 pr = ld4(&s.X.pos_r[i]);
    double4 vm = ld4(&s.X.vel_m[i]);
    double4 om = ld4(&s.X.omg[i]);
    if (INTEGRATE) {  // pipeline.cpp:31-44, same arithmetic as k_integrate_hash
        const uint32_t n = s.ft_stride;
        const V3 f = v3(s.ft[i], s.ft[n + i], s.ft[2 * n + i]);
        const V3 t = v3(s.ft[3 * n + i], s.ft[4 * n + i], s.ft[5 * n + i]);
        if (!finite3(f) || !finite3(t)) {
            raise_err(s.ctl, 0, i, idm.x, 2 /*DEM_ERR_KERNEL*/);
        } else {
            const double m = vm.w, r = pr.w;
            const double sc = p.dt / m;
            vm.x = vm.x + f.x * sc; vm.y = vm.y + f.y * sc; vm.z = vm.z + f.z * sc;
            pr.x = pr.x + vm.x * p.dt; pr.y = pr.y + vm.y * p.dt; pr.z = pr.z + vm.z * p.dt;
            const double inertia = 0.4 * m * r * r;
            const double s2 = p.dt / inertia;
            om.x = om.x + t.x * s2; om.y = om.y + t.y * s2; om.z = om.z + t.z * s2;
        }
    }
    int cls;
    if (p.periodic) {
        // periodic z: the direction comes from the unwrapped plane (a particle leaving the top of
        // the last slab goes up the ring, to slab 0), then the position is wrapped
        int cz = cell_z(p, pr.z);
        if (p.periodic & 4u) cz = to_int_x86(floor((pr.z - p.oz) * p.inv_z));
        if (INTEGRATE) wrap_periodic(p, s.ctl->le_delta, pr, vm);
        cls = cz < s.z_lo ? 1 : (cz >= s.z_hi ? 2 : 0);
    } else {
        const int cz = cell_z(p, pr.z);
        cls = cz < s.z_lo ? 1 : (cz >= s.z_hi ? 2 : 0);
    }
    const uint32_t slot = agg_add(&s.counters[cls], cls);
    const uint32_t hpos = s.H_old.pos[i], hcnt = s.H_old.cnt[i];
    if (cls == 0) {
        put_state(s.Y, slot, pr, vm, om, idm);
        s.hrm_pos[slot] = hpos;
        s.hrm_cnt[slot] = hcnt;
        return;
    }
    if (slot >= s.cap_send) { atomicMax(&s.counters[4], 1u); return; }
    uint8_t* rec = (cls == 1 ? s.send_lo : s.send_hi) + static_cast<size_t>(slot) * s.rec_bytes;
    put_record(rec, pr, vm, om, idm);
    uint32_t* hdr = reinterpret_cast<uint32_t*>(rec + 104);
    hdr[0] = hcnt;
    uint32_t* keys = reinterpret_cast<uint32_t*>(rec + 112);
    double* dts = reinterpret_cast<double*>(rec + s.rec_dt_off);
    for (uint32_t k = 0; k < hcnt; ++k) {
        keys[k] = s.H_old.key[hpos + k];
        dts[3 * k + 0] = s.H_old.dt[hpos + k];
        dts[3 * k + 1] = s.H_old.dt[s.hcap + hpos + k];
        dts[3 * k + 2] = s.H_old.dt[2 * s.hcap + hpos + k];
    }
}

__global__ void __launch_bounds__(256) k_slab_import(SlabBufs s, const uint8_t* recs, uint32_t n, uint32_t base,
                                                      size_t imp_off) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint8_t* rec = recs + static_cast<size_t>(t) * s.rec_bytes;
    const double4* d = reinterpret_cast<const double4*>(rec);
    const uint2 idm = *reinterpret_cast<const uint2*>(rec + 96);
    put_state(s.Y, base + t, ld4(&d[0]), ld4(&d[1]), ld4(&d[2]), idm);
    const uint32_t hcnt = reinterpret_cast<const uint32_t*>(rec + 104)[0];
    const uint32_t* keys = reinterpret_cast<const uint32_t*>(rec + 112);
    const double* dts = reinterpret_cast<const double*>(rec + s.rec_dt_off);
    const size_t hpos = s.imp_base + imp_off + static_cast<size_t>(t) * s.K;
    for (uint32_t k = 0; k < hcnt; ++k) {
        s.H_old.key[hpos + k] = keys[k];
        s.H_old.dt[hpos + k] = dts[3 * k];
        s.H_old.dt[s.hcap + hpos + k] = dts[3 * k + 1];
        s.H_old.dt[2 * s.hcap + hpos + k] = dts[3 * k + 2];
    }
    s.hrm_pos[base + t] = static_cast<uint32_t>(hpos);
    s.hrm_cnt[base + t] = hcnt;
}

// the Lees-Edwards clock advances with the integrating migrate (the slab force phase does not
// integrate)
__global__ void k_le_advance(StepParams p, DevCtl* ctl) {
    if (threadIdx.x == 0 && ctl->err_key == kNoError) le_clock(p, ctl, true);
}

// owned particles of Y[0, n_own) on the boundary planes become ghost records for the neighbours
__global__ void __launch_bounds__(256) k_slab_halo(StepParams p, SlabBufs s, uint32_t n_own) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_own) return;
    const double4 pr = ld4(&s.Y.pos_r[i]);
    const int cz = cell_z(p, pr.z);
    const bool lo = cz == s.z_lo, hi = cz == s.z_hi - 1;
    if (!lo && !hi) return;
    const double4 vm = ld4(&s.Y.vel_m[i]), om = ld4(&s.Y.omg[i]);
    const uint2 idm = s.Y.idm[i];
    if (lo) {
        const uint32_t slot = atomicAdd(&s.counters[5], 1u);
        if (slot < s.cap_send) put_record(s.send_lo + static_cast<size_t>(slot) * s.ghost_bytes, pr, vm, om, idm);
        else atomicMax(&s.counters[4], 1u);
    }
    if (hi) {
        const uint32_t slot = atomicAdd(&s.counters[6], 1u);
        if (slot < s.cap_send) put_record(s.send_hi + static_cast<size_t>(slot) * s.ghost_bytes, pr, vm, om, idm);
        else atomicMax(&s.counters[4], 1u);
    }
}

__global__ void __launch_bounds__(256) k_slab_ghosts(SlabBufs s, const uint8_t* recs, uint32_t n, uint32_t base,
                                                      bool from_hi) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint8_t* rec = recs + static_cast<size_t>(t) * s.ghost_bytes;
    const double4* d = reinterpret_cast<const double4*>(rec);
    uint2 idm = *reinterpret_cast<const uint2*>(rec + 96);
    idm.y |= kGhost | (from_hi ? kGhostHi : 0u);
    put_state(s.Y, base + t, ld4(&d[0]), ld4(&d[1]), ld4(&d[2]), idm);
    s.hrm_pos[base + t] = 0;
    s.hrm_cnt[base + t] = 0;
}

// ---------------------------------------------------------------------------------------------
// Host-free sharded stepping. The same per-step protocol as above, but every size
// is device-resident: the kernels are launched for the capacity and read the counts (s.dn, the
// counters, the inbox header); the migrant / ghost records are stored straight into the
// neighbours' inbox blocks (peer memory: CUDA IPC across processes, direct peer pointers in one
// process; over NVLink on an HGX box), the counts follow, then a flag is raised with a release
// store at system scope. The receiver's stream waits for the flag (a stream memory-operation wait,
// or k_shard_wait), consumes the records and clears the flag. No count crosses the host, so the
// whole step is one CUDA graph per history parity.
//
// Reuse of an inbox is ordered by the protocol itself: a neighbour writes my migrant inbox again
// only after it has seen my ghost flag of the current step, raised after I consumed my migrants
// (and symmetrically for ghosts), so one buffer per (kind, side) suffices.

__device__ __forceinline__ uint32_t* inbox_flags(uint8_t* box) { return reinterpret_cast<uint32_t*>(box); }
__device__ __forceinline__ uint32_t* inbox_counts(uint8_t* box) { return reinterpret_cast<uint32_t*>(box) + 4; }
__device__ __forceinline__ uint8_t* inbox_records(const SlabBufs& s, uint8_t* box, uint32_t kind, uint32_t side) {
    return box + inbox_region(kind, side, s.cap_send, s.rec_bytes, s.ghost_bytes);
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// k_slab_migrate over X[0, dn[0]) with the leavers stored into the neighbours' migrant inboxes
// (my "down" records arrive in the lower neighbour's from-above region, and vice versa).
template <bool INTEGRATE>
__global__ void __launch_bounds__(256) k_shard_migrate(StepParams p, SlabBufs s) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.dn[0] || s.ctl->err_key != kNoError) return;
    const uint2 idm = s.X.idm[i];
    if (idm.y & kGhost) return;
    double4 pr = ld4(&s.X.pos_r[i]);
    double4 vm = ld4(&s.X.vel_m[i]);
    double4 om = ld4(&s.X.omg[i]);
    if (INTEGRATE) {  // pipeline.cpp:31-44, as k_slab_migrate
        const uint32_t n = s.ft_stride;
        const V3 f = v3(s.ft[i], s.ft[n + i], s.ft[2 * n + i]);
        const V3 t = v3(s.ft[3 * n + i], s.ft[4 * n + i], s.ft[5 * n + i]);
        if (!finite3(f) || !finite3(t)) {
            raise_err(s.ctl, 0, i, idm.x, 2 /*DEM_ERR_KERNEL*/);
        } else {
            const double m = vm.w, r = pr.w;
            const double sc = p.dt / m;
            vm.x = vm.x + f.x * sc; vm.y = vm.y + f.y * sc; vm.z = vm.z + f.z * sc;
            pr.x = pr.x + vm.x * p.dt; pr.y = pr.y + vm.y * p.dt; pr.z = pr.z + vm.z * p.dt;
            const double inertia = 0.4 * m * r * r;
            const double s2 = p.dt / inertia;
            om.x = om.x + t.x * s2; om.y = om.y + t.y * s2; om.z = om.z + t.z * s2;
        }
    }
    int cz = cell_z(p, pr.z);
    if (p.periodic) {
        if (p.periodic & 4u) cz = to_int_x86(floor((pr.z - p.oz) * p.inv_z));
        if (INTEGRATE) wrap_periodic(p, s.ctl->le_delta, pr, vm);
    }
    int cls = cz < s.z_lo ? 1 : (cz >= s.z_hi ? 2 : 0);
    uint8_t* peer = cls == 1 ? s.peer_lo : (cls == 2 ? s.peer_hi : nullptr);
    if (cls != 0 && !peer) {  // no neighbour that side: cannot happen with clamped planes
        raise_err(s.ctl, 0, i, idm.x, 2);
        return;
    }
    const uint32_t slot = agg_add(&s.counters[cls], cls);
    const uint32_t hpos = s.H_old.pos[i], hcnt = s.H_old.cnt[i];
    if (cls == 0) {
        if (slot >= s.n_cap) { atomicMax(&s.counters[4], 1u); return; }
        put_state(s.Y, slot, pr, vm, om, idm);
        s.hrm_pos[slot] = hpos;
        s.hrm_cnt[slot] = hcnt;
        return;
    }
    if (slot >= s.cap_send) { atomicMax(&s.counters[4], 1u); return; }
    uint8_t* rec = inbox_records(s, peer, 0, cls == 1 ? 1u : 0u) + static_cast<size_t>(slot) * s.rec_bytes;
    put_record(rec, pr, vm, om, idm);
    reinterpret_cast<uint32_t*>(rec + 104)[0] = hcnt;
    uint32_t* keys = reinterpret_cast<uint32_t*>(rec + 112);
    double* dts = reinterpret_cast<double*>(rec + s.rec_dt_off);
    for (uint32_t k = 0; k < hcnt; ++k) {
        keys[k] = s.H_old.key[hpos + k];
        dts[3 * k + 0] = s.H_old.dt[hpos + k];
        dts[3 * k + 1] = s.H_old.dt[s.hcap + hpos + k];
        dts[3 * k + 2] = s.H_old.dt[2 * s.hcap + hpos + k];
    }
}

// after a pack: counts into the neighbours' inbox headers, then their flags (release, system
// scope). kind 0 also publishes the stayer count as this rank's owned-slot base.
__global__ void k_shard_post(SlabBufs s, uint32_t kind) {
    if (threadIdx.x != 0) return;
    uint32_t n_lo = s.counters[kind == 0 ? 1 : 5], n_hi = s.counters[kind == 0 ? 2 : 6];
    if (s.counters[4]) {  // a send buffer (or the assembly) overflowed: stop this rank's step
        raise_err(s.ctl, 6, 0, 0, 3 /*DEM_ERR_CAPACITY*/);
        n_lo = min(n_lo, s.cap_send);
        n_hi = min(n_hi, s.cap_send);
    }
    if (kind == 0) s.dn[1] = min(s.counters[0], s.n_cap);
    if (s.peer_lo) inbox_counts(s.peer_lo)[2 * kind + 1] = n_lo;
    if (s.peer_hi) inbox_counts(s.peer_hi)[2 * kind + 0] = n_hi;
    __threadfence_system();
    if (s.peer_lo) st_release_sys(&inbox_flags(s.peer_lo)[2 * kind + 1], 1u);
    if (s.peer_hi) st_release_sys(&inbox_flags(s.peer_hi)[2 * kind + 0], 1u);
}

// the spin fallback of the stream wait: both expected flags of `kind` raised
__global__ void k_shard_wait(SlabBufs s, uint32_t kind) {
    if (threadIdx.x != 0) return;
    uint32_t* f = inbox_flags(s.inbox);
    if (s.peer_lo) while (ld_acquire_sys(&f[2 * kind + 0]) == 0u) __nanosleep(200);
    if (s.peer_hi) while (ld_acquire_sys(&f[2 * kind + 1]) == 0u) __nanosleep(200);
}

// received migrants appended after the stayers, with their history rows in the import region
__global__ void __launch_bounds__(256) k_shard_import(SlabBufs s) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t* cnt = inbox_counts(s.inbox);
    const uint32_t n_lo = s.peer_lo ? cnt[0] : 0u, n_hi = s.peer_hi ? cnt[1] : 0u;
    const uint32_t base = min(s.counters[0], s.n_cap);  // the stayers (dn[1] is rewritten below)
    const bool fits = base + n_lo + n_hi <= s.n_cap && n_lo + n_hi <= s.imp_cap;
    if (t == 0) {
        uint32_t* f = inbox_flags(s.inbox);
        f[0] = 0u;
        f[1] = 0u;
        if (!fits) raise_err(s.ctl, 6, 0, 0, 3 /*DEM_ERR_CAPACITY*/);
    }
    if (t >= n_lo + n_hi || !fits) return;
    if (t == 0) s.dn[1] = base + n_lo + n_hi;
    const uint32_t side = t < n_lo ? 0u : 1u;
    const uint32_t r = side ? t - n_lo : t;
    const uint8_t* rec = inbox_records(s, s.inbox, 0, side) + static_cast<size_t>(r) * s.rec_bytes;
    const double4* d = reinterpret_cast<const double4*>(rec);
    const uint2 idm = *reinterpret_cast<const uint2*>(rec + 96);
    put_state(s.Y, base + t, ld4(&d[0]), ld4(&d[1]), ld4(&d[2]), idm);
    const uint32_t hcnt = reinterpret_cast<const uint32_t*>(rec + 104)[0];
    const uint32_t* keys = reinterpret_cast<const uint32_t*>(rec + 112);
    const double* dts = reinterpret_cast<const double*>(rec + s.rec_dt_off);
    const size_t hpos = s.imp_base + static_cast<size_t>(t) * s.K;
    for (uint32_t k = 0; k < hcnt; ++k) {
        s.H_old.key[hpos + k] = keys[k];
        s.H_old.dt[hpos + k] = dts[3 * k];
        s.H_old.dt[s.hcap + hpos + k] = dts[3 * k + 1];
        s.H_old.dt[2 * s.hcap + hpos + k] = dts[3 * k + 2];
    }
    s.hrm_pos[base + t] = static_cast<uint32_t>(hpos);
    s.hrm_cnt[base + t] = hcnt;
}

// boundary-plane owned particles of Y[0, dn[1]) as ghost records into the neighbours' inboxes
__global__ void __launch_bounds__(256) k_shard_halo(StepParams p, SlabBufs s) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.dn[1] || s.ctl->err_key != kNoError) return;
    const double4 pr = ld4(&s.Y.pos_r[i]);
    const int cz = cell_z(p, pr.z);
    const bool lo = cz == s.z_lo && s.peer_lo, hi = cz == s.z_hi - 1 && s.peer_hi;
    if (!lo && !hi) return;
    const double4 vm = ld4(&s.Y.vel_m[i]), om = ld4(&s.Y.omg[i]);
    const uint2 idm = s.Y.idm[i];
    if (lo) {
        const uint32_t slot = atomicAdd(&s.counters[5], 1u);
        if (slot < s.cap_send)
            put_record(inbox_records(s, s.peer_lo, 1, 1) + static_cast<size_t>(slot) * s.ghost_bytes, pr, vm, om, idm);
        else atomicMax(&s.counters[4], 1u);
    }
    if (hi) {
        const uint32_t slot = atomicAdd(&s.counters[6], 1u);
        if (slot < s.cap_send)
            put_record(inbox_records(s, s.peer_hi, 1, 0) + static_cast<size_t>(slot) * s.ghost_bytes, pr, vm, om, idm);
        else atomicMax(&s.counters[4], 1u);
    }
}

// received ghosts appended after the owned slots; dn[0] = the force phase's slot count
__global__ void __launch_bounds__(256) k_shard_ghosts(SlabBufs s) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t* cnt = inbox_counts(s.inbox);
    const uint32_t g_lo = s.peer_lo ? cnt[2] : 0u, g_hi = s.peer_hi ? cnt[3] : 0u;
    const uint32_t base = s.dn[1];
    const bool fits = base + g_lo + g_hi <= s.n_cap;
    if (t == 0) {
        uint32_t* f = inbox_flags(s.inbox);
        f[2] = 0u;
        f[3] = 0u;
        s.dn[0] = fits ? base + g_lo + g_hi : base;
        if (!fits) raise_err(s.ctl, 6, 0, 0, 3 /*DEM_ERR_CAPACITY*/);
    }
    if (t >= g_lo + g_hi || !fits) return;
    const bool from_hi = t >= g_lo;
    const uint32_t r = from_hi ? t - g_lo : t;
    const uint8_t* rec = inbox_records(s, s.inbox, 1, from_hi ? 1u : 0u) + static_cast<size_t>(r) * s.ghost_bytes;
    const double4* d = reinterpret_cast<const double4*>(rec);
    uint2 idm = *reinterpret_cast<const uint2*>(rec + 96);
    idm.y |= kGhost | (from_hi ? kGhostHi : 0u);
    put_state(s.Y, base + t, ld4(&d[0]), ld4(&d[1]), ld4(&d[2]), idm);
    s.hrm_pos[base + t] = 0;
    s.hrm_cnt[base + t] = 0;
}

inline unsigned blocks(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

void launch_shard_migrate(const StepParams& p, const SlabBufs& s, bool integrate, cudaStream_t st) {
    if (integrate && p.periodic) k_le_advance<<<1, 32, 0, st>>>(p, s.ctl);
    if (integrate) k_shard_migrate<true><<<blocks(s.n_cap), 256, 0, st>>>(p, s);
    else k_shard_migrate<false><<<blocks(s.n_cap), 256, 0, st>>>(p, s);
}
void launch_shard_post(const SlabBufs& s, uint32_t kind, cudaStream_t st) { k_shard_post<<<1, 32, 0, st>>>(s, kind); }
void launch_shard_wait(const SlabBufs& s, uint32_t kind, cudaStream_t st) { k_shard_wait<<<1, 32, 0, st>>>(s, kind); }
void launch_shard_import(const SlabBufs& s, cudaStream_t st) {
    k_shard_import<<<blocks(2 * static_cast<size_t>(s.cap_send)), 256, 0, st>>>(s);
}
void launch_shard_halo(const StepParams& p, const SlabBufs& s, cudaStream_t st) {
    k_shard_halo<<<blocks(s.n_cap), 256, 0, st>>>(p, s);
}
void launch_shard_ghosts(const SlabBufs& s, cudaStream_t st) {
    k_shard_ghosts<<<blocks(2 * static_cast<size_t>(s.cap_send)), 256, 0, st>>>(s);
}

void launch_slab_migrate(const StepParams& p, const SlabBufs& s, bool integrate, cudaStream_t st) {
    if (integrate && p.periodic) k_le_advance<<<1, 32, 0, st>>>(p, s.ctl);
    if (!s.n_x) return;
    if (integrate) k_slab_migrate<true><<<blocks(s.n_x), 256, 0, st>>>(p, s);
    else k_slab_migrate<false><<<blocks(s.n_x), 256, 0, st>>>(p, s);
}
void launch_slab_import(const SlabBufs& s, const void* recs, uint32_t n, uint32_t base, size_t imp_off, cudaStream_t st) {
    if (n) k_slab_import<<<blocks(n), 256, 0, st>>>(s, static_cast<const uint8_t*>(recs), n, base, imp_off);
}
void launch_slab_halo(const StepParams& p, const SlabBufs& s, uint32_t n_own, cudaStream_t st) {
    if (n_own) k_slab_halo<<<blocks(n_own), 256, 0, st>>>(p, s, n_own);
}
void launch_slab_ghosts(const SlabBufs& s, const void* recs, uint32_t n, uint32_t base, bool from_hi, cudaStream_t st) {
    if (n) k_slab_ghosts<<<blocks(n), 256, 0, st>>>(s, static_cast<const uint8_t*>(recs), n, base, from_hi);
}

}  // namespace demb200
