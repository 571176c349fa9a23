// dem_internal.h — device data layout and kernel launchers shared by dem_kernels.cu
// (the sm_100a kernels) and dem_capi.cu (the C ABI / context / CUDA graphs).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace demb200 {

constexpr int kMaxMaterials = 16;
constexpr int kMaxWalls = 64;
constexpr int kMaxContactCapacity = 80;  // k_detect's shared-memory rows (dem_kernels.cu launch_detect)
constexpr uint32_t kWallBit = 0x80000000u;  // partner codes >= this are walls: ~code = wall index
constexpr unsigned long long kNoError = ~0ull;
constexpr uint32_t kPhaseSlab = 64u;  // internal phase flag: slab context (ghost-aware kernels)
constexpr uint32_t kPhaseInterior = 128u;  // internal: every periodic axis has >= 5 cells (k_detect)
constexpr uint32_t kPhaseFp32 = 256u;      // internal: fp32 throughput mode (k_force_reduce)
constexpr uint32_t kPhasePreint = 512u;    // internal: single context; k_force_reduce pre-integrates (PhaseBufs::pre)

struct MatPairH {  // host mirror of MatPair (dem_math.cuh)
    double shear_sum, young_sum, alpha, mu;
};
struct RectW {
    double c[3], u[3], v[3];
    uint32_t mat, pad;
};
struct LineW {
    double a[3], b[3];
    uint32_t mat, pad;
};

// Uniform per-phase parameters, passed by value.
struct StepParams {
    double ox, oy, oz;   // grid origin
    double h, inv_h;     // cell size, 1.0 / h (grid.cpp:32)
    int nx, ny, nz;      // GLOBAL grid (grid.cpp:10-28)
    int kz0, nz_loc;     // keyed z-planes [kz0, kz0+nz_loc) (slab context; else 0, nz)
    uint32_t M;          // keyed cells nx*ny*nz_loc
    double dt;
    double gx, gy, gz;
    uint32_t n;          // particles
    int K;               // contact capacity
    int nmat;
    int nrect, nline;
    uint32_t flags;      // dem_phase_flags
    double det_lo, det_hi, det_tiny;  // k_detect classification constants (kept in the param bank)
    // periodic box (beyond the reference). periodic == 0: the reference's box.
    uint32_t periodic;   // bit k: axis k periodic
    double inv_x, inv_y, inv_z;  // 1 / cell extent per axis (all inv_h when nothing is periodic)
    double Lx, Ly, Lz;           // box lengths
    double half_x, half_y, half_z;
    double shear_rate, shear_u;  // Lees-Edwards rate and image velocity rate * Ly
    const MatPairH* pairs;  // nmat*nmat, [owner][partner]
    const RectW* rects;
    const LineW* lines;
};

// Control block (device memory): error word, phase counter, per-phase metrics, tile counters.
struct DevCtl {
    unsigned long long err_key;                 // (kernel<<56)|(slot<<8)|code, atomicMin
    unsigned long long err_sid[9];              // per kernel: (slot<<32)|stable id, atomicMin
    unsigned long long err_phase;               // phase of the error
    unsigned long long phase;                   // phases begun
    unsigned int halted;                        // set by a phase begun after an error
    unsigned int tile_ctr_scan;
    unsigned int tile_ctr_detect;
    unsigned int max_per;
    unsigned long long clamps;
    unsigned long long pp_events;
    unsigned long long capped;
    unsigned long long fric_bits;               // max of non-negative doubles as bits
    unsigned long long contacts;
    unsigned int odd_radius;                    // a radius outside [1e-100, 1e100] (or NaN) was binned
    unsigned int poly;                          // a radius != r_ref was binned this phase
    double r_ref;                               // particle 0's radius (set on upload; k_pack_state)
    double m_ref;                               // its mass (force memo); must follow r_ref
    long long le_steps;                         // integrating phases so far (Lees-Edwards clock)
    double le_delta;                            // Lees-Edwards image offset of the upper box
    unsigned long long bad_upload;              // (slot<<8)|reason of the first invalid uploaded particle, atomicMin
    unsigned int maybe_dup;                     // an uploaded id hashed onto an occupied idmap bit
    // Pre-integration (single context): the force kernel of phase `preint_phase` wrote the next
    // Integrate's result (its state advanced with the forces it just computed) into PhaseBufs::pre;
    // the next phase uses it when it integrates and preint_phase == phase - 1 (~0: invalid; every
    // host-side change of state or forces invalidates it). A non-finite force seen there is the next
    // Integrate's KernelError, deferred to that phase: deferred[q & 1] = min (slot<<32)|id of phase q.
    unsigned long long preint_phase;
    unsigned long long deferred[2];
};

// Structure-of-arrays particle state for one buffer (sorted slot order).
struct StateBuf {
    double4* pos_r;   // x, y, z, radius
    double4* vel_m;   // vx, vy, vz, mass
    double4* omg;     // wx, wy, wz, 0
    uint2* idm;       // stable id, material id
    float4* pos_f;    // x, y, z, radius rounded to fp32 (k_reorder; k_detect's conservative prefilter)
};

// Contacts of one force phase, tile-compacted: warp tile t (slots 32t..32t+31) owns the pair
// slots [32 K t, 32 K (t+1)); inside it the contacts of its particles are dense, in slot order,
// each particle's in accumulation order.
struct HistBuf {
    uint32_t* pos;    // n: first pair slot of particle i
    uint32_t* cnt;    // n: number of contacts of particle i
    uint32_t* key;    // cap: partner stable id, or wall code
    double* dt;       // 3 * cap (SoA: x | y | z): tangential displacement after this phase
};

struct PhaseBufs {
    StateBuf src, dst;       // reorder gathers src -> dst
    StateBuf pre;            // single context: pos_r / vel_m / omg pre-integrated by k_force_reduce (src slot order)
    HistBuf old_h, cur_h;    // history of previous phase / written this phase
    double* ft;              // 6 * n (fx|fy|fz|tx|ty|tz), per slot
    uint32_t* key;           // n: cell key per (pre-sort) slot, later sorted keys
    uint32_t* skey;          // n: sorted keys (new slot order)
    uint32_t* loc;           // n: arrival rank in cell
    uint32_t* cnt;           // M: cell counts (kept zero between phases)
    uint32_t* cstart;        // M+1
    uint32_t* tmp_src;       // n
    uint32_t* tmp_id;        // n
    uint32_t* prev_slot;     // n
    uint2* prev_row;         // n: {pos, cnt} of the slot's previous history row (written by k_reorder)
    uint32_t* pair_i;        // cap
    uint32_t* pair_j;        // cap
    unsigned long long* status_scan;
    unsigned long long* status_det;
    uint32_t n_tiles_scan, n_tiles_det;
    size_t cap;              // pair slots in key/dt (SoA stride of dt)
    uint32_t ft_stride;      // SoA stride of ft (n, or the slab context's slot capacity)
    DevCtl* ctl;
    // host-free (sharded) phases: the slot count lives in device memory (written by the slab
    // exchange kernels) and the grids are sized for the capacity; nullptr: StepParams::n
    const uint32_t* dn;
};

// Slab decomposition buffers (dem_slab.cu). X: state after the previous force phase (owned and
// ghosts); Y: the assembly buffer the next force phase bins from.
struct SlabBufs {
    StateBuf X, Y;
    const double* ft;
    uint32_t ft_stride;
    HistBuf H_old;           // previous phase's history (pos/cnt per X slot), + import region
    uint32_t* hrm_pos;       // per Y slot: previous history row (remapped / imported)
    uint32_t* hrm_cnt;
    uint32_t n_x;
    uint32_t* counters;      // [0] stayers [1] to lo [2] to hi [4] overflow [5] halo lo [6] halo hi
    uint8_t* send_lo;
    uint8_t* send_hi;
    uint32_t cap_send;       // records per send buffer
    uint32_t rec_bytes, rec_dt_off, ghost_bytes;
    int z_lo, z_hi;          // owned global planes
    size_t imp_base;         // first pair slot of the history import region
    size_t hcap;             // pair slots in key/dt (SoA stride)
    uint32_t K;
    DevCtl* ctl;
    // host-free (sharded) stepping: device-resident counts and the inboxes
    uint32_t* dn;            // [0] slots of the force phase (owned + ghosts) [1] owned slots
    uint8_t* inbox;          // this rank's inbox block (kInboxHeader + 4 record regions)
    uint8_t* peer_lo;        // the z-neighbours' inbox blocks (nullptr: no neighbour that side)
    uint8_t* peer_hi;
    uint32_t n_cap, imp_cap; // slot capacity, history-import capacity (records)
};

// Inbox block of a sharded rank: a header (flags[4], counts[4]; index 2 kind + side, kind 0
// migrants / 1 ghosts, side 0 = from the lower neighbour / 1 = from the upper) and four record
// regions in that order, cap_send records each. Neighbours store records and counts into it and
// raise the flag; the owner waits for the flag, consumes, and clears it.
constexpr size_t kInboxHeader = 256;
__host__ __device__ inline size_t inbox_region(uint32_t kind, uint32_t side, size_t cap, size_t rec_bytes, size_t ghost_bytes) {
    const size_t mig = cap * rec_bytes, gh = cap * ghost_bytes;
    return kInboxHeader + (kind == 0 ? side * mig : 2 * mig + side * gh);
}

void launch_shard_migrate(const StepParams& p, const SlabBufs& s, bool integrate, cudaStream_t st);
void launch_shard_post(const SlabBufs& s, uint32_t kind, cudaStream_t st);
void launch_shard_wait(const SlabBufs& s, uint32_t kind, cudaStream_t st);  // spin fallback of the stream wait
void launch_shard_import(const SlabBufs& s, cudaStream_t st);
void launch_shard_halo(const StepParams& p, const SlabBufs& s, cudaStream_t st);
void launch_shard_ghosts(const SlabBufs& s, cudaStream_t st);

void launch_slab_migrate(const StepParams& p, const SlabBufs& s, bool integrate, cudaStream_t st);
void launch_slab_import(const SlabBufs& s, const void* recs, uint32_t n, uint32_t base, size_t imp_off, cudaStream_t st);
void launch_slab_halo(const StepParams& p, const SlabBufs& s, uint32_t n_own, cudaStream_t st);
void launch_slab_ghosts(const SlabBufs& s, const void* recs, uint32_t n, uint32_t base, bool from_hi, cudaStream_t st);

constexpr int kScanThreads = 256;
#ifndef DEM_SCAN_ITEMS
#define DEM_SCAN_ITEMS 16
#endif
constexpr int kScanItems = DEM_SCAN_ITEMS;  // cells per thread of k_scan_cells (tile = 256 x this)
#ifndef DEM_DET_THREADS
#define DEM_DET_THREADS 128
#endif
// 4 warps per block (8: polydisperse detection 37 us slower at configs[2] — a block's slots free
// only when its slowest tile is done); a detection tile is one warp (32 slots)
constexpr int kDetectThreads = DEM_DET_THREADS;

inline uint32_t scan_tiles(uint32_t M) { return (M + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems); }
// warp tiles launched (a multiple of the warps per block)
// k_detect's per-thread shared-memory list: the fp32 prefilter's kept candidates (up to
// detect_pass_cap; more sends the lane to the one-stage walk), then its contacts compacted in
// place (<= K + 1), plus one scratch entry; odd stride, so the lanes' appends are conflict-free.
// The prefilter keeps the contacts and the pairs within ~2^-18 relative of touching, so K
// entries hold every list short of a CapacityError (a lane with more survivors takes the exact
// one-stage walk, which also counts an overflow exactly); the smaller rows let more detection
// blocks share an SM and leave more L1 (profiles/r02_force_variants.md: configs[2] detection
// -17 %, configs[1] -4 %; DEM_PF_CAP_EXTRA < 0: 2K, the earlier sizing).
#ifndef DEM_PF_CAP_EXTRA
#define DEM_PF_CAP_EXTRA 0
#endif
__host__ __device__ inline uint32_t detect_pass_cap(uint32_t K) {
    return DEM_PF_CAP_EXTRA < 0 ? 2u * K : K + static_cast<uint32_t>(DEM_PF_CAP_EXTRA);
}
__host__ __device__ inline uint32_t detect_row_stride(uint32_t K) { return (detect_pass_cap(K) + 1u) | 1u; }
inline uint32_t detect_tiles(uint32_t n) { return ((n + kDetectThreads - 1) / kDetectThreads) * (kDetectThreads / 32); }

// Launchers (dem_kernels.cu). Each enqueues exactly one kernel on `s`.
void launch_phase_begin(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_integrate_hash(const StepParams& p, const PhaseBufs& b, bool integrate, cudaStream_t s);
void launch_scan_cells(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_scatter(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_reorder(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_detect(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_force_reduce(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_collide_single_loop(const StepParams& p, const PhaseBufs& b, cudaStream_t s);
void launch_flush(void* buf, size_t bytes, cudaStream_t s);
// traversal traces of the phase whose buffers `b` names (ev == nullptr: per-slot counts)
void launch_selftest_division(uint64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t s);
void launch_trace(const StepParams& p, const PhaseBufs& b, const unsigned long long* off, int2* ev,
                  uint32_t* count, cudaStream_t s);

// Device staging in the caller's (host) layout: positions[3n], ..., ids[n], material_ids[n].
struct RawState {
    double *pos, *vel, *omg, *rad, *mass;
    uint32_t *ids, *mat;
};
// Upload validation done by the pack kernel (ParticleSet::validate, particle_set.cpp:40-58, plus
// the B200 id rules): the first invalid slot lands in ctl->bad_upload; uploaded ids are hashed into
// idmap (a bitmap of idmask + 1 bits, zeroed by the caller) and a set bit already present raises
// ctl->maybe_dup (a duplicate id, or a hash collision the host then resolves exactly).
struct PackCheck {
    DevCtl* ctl;
    uint32_t nmat;
    uint32_t* idmap;   // nullptr: ids not uploaded (kept), no duplicate screen
    uint32_t idmask;
};
// pack: host layout -> SoA, and (ref non-null) ref[0], ref[1] = particle 0's radius and mass
void launch_pack_state(const StateBuf& s, const RawState& r, uint32_t n, bool pack, cudaStream_t st,
                       const PackCheck* check = nullptr, double* ref = nullptr);
void launch_ft_layout(double* ft, uint32_t stride, double* f, double* t, uint32_t n, bool to_interleaved, cudaStream_t st);
cudaError_t init_device_attributes();

}  // namespace demb200
