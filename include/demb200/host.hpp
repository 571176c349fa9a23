// demb200/host.hpp — the host side around the B200 Simulation: config files, initial states,
// on-disk formats and the run / bench / verify drivers (reference
// core/include/demforge/{config_io,lattice,snapshot_io,runner}.hpp). Compiled into
// libdem_b200.so from paper_1503_03553_b200/host/*.cpp; the `dem_b200` CLI
// (paper_1503_03553_b200/host/cli.cpp) mirrors tools/demforge.cpp.
#pragma once

#include <cstdint>
#include <filesystem>
#include <string>
#include <vector>

#include "simulation.hpp"

namespace demb200 {

// ---- config_io.hpp: flat `key = value` files --------------------------------------------------
SimConfig parse_config(const std::filesystem::path& path);
SimConfig parse_config_text(const std::string& text, const std::string& origin = "config");
/// Cross-field validation (sim_config.cpp:10-60); throws ConfigError naming the key.
void validate_config(const SimConfig& cfg);
std::uint32_t particle_material_id(const SimConfig& cfg);

// ---- lattice.hpp: initial states --------------------------------------------------------------
/// xorshift64* (rng.hpp:11-33)
class XorShift64Star {
  public:
    explicit XorShift64Star(std::uint64_t seed) : state_(seed != 0 ? seed : 0x9E3779B97F4A7C15ULL) {}
    std::uint64_t next_u64() {
        std::uint64_t x = state_;
        x ^= x >> 12;
        x ^= x << 25;
        x ^= x >> 27;
        state_ = x;
        return x * 0x2545F4914F6CDD1DULL;
    }
    double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_in(double lo, double hi) { return lo + (hi - lo) * next_unit(); }

  private:
    std::uint64_t state_;
};
double resolve_lattice_spacing(const SimConfig& cfg);
ParticleSet build_initial_state(const SimConfig& cfg);

// ---- snapshot_io.hpp ----------------------------------------------------------------------------
std::string format_double(double value);  // shortest round-trip decimal
void write_snapshot(const std::filesystem::path& path, const ParticleSet& state);
inline constexpr const char* kMetricsHeader =
    "step,kernel,wall_ns,model_cycles_baseline,model_cycles_two_phase,"
    "utilization_baseline,utilization_two_phase,contacts,max_contacts_per_particle,clamps";
/// Nine kernel rows per step (snapshot_io.cpp:70-94). The Collide row carries the warp model of the
/// step's traversal traces (StepMetrics::model_*, filled when traces are recorded); wall_ns is the
/// device time of the B200 kernels mapped onto the reference kernel rows, or 0 when
/// `zero_wall_time`.
void append_metrics_rows(std::string& out, std::int64_t step, const StepMetrics& m,
                         const double* kernel_ms /* nullable, dem_device_kernel order */,
                         bool zero_wall_time);

// ---- runner.hpp ---------------------------------------------------------------------------------
struct RunSummary {
    std::int64_t steps_run = 0;
    int snapshots_written = 0;
    std::filesystem::path metrics_path;
};
RunSummary run_simulation(const SimConfig& cfg, const std::filesystem::path& out_dir, int device = 0);

struct BenchPhase {
    std::string label;
    std::int64_t steps = 0;
    double collide_us_baseline = 0.0, collide_us_two_phase = 0.0;
    double kernel_us[DEM_DEVICE_KERNEL_COUNT] = {};
    double mean_coordination = 0.0;
    WarpReport model;  // the warp model over the measured steps' traces (runner.cpp:126-129)
    double ratio() const { return collide_us_two_phase > 0 ? collide_us_baseline / collide_us_two_phase : 1.0; }
};
struct BenchReport {
    BenchPhase sparse, dense;
    std::string format() const;
};
BenchReport bench(const SimConfig& cfg, int device = 0);

struct PropertyResult {
    std::string name;
    bool pass = false;
    std::string detail;
};
struct VerifyReport {
    std::vector<PropertyResult> properties;
    bool all_pass() const;
    std::string format() const;
};
VerifyReport verify(const SimConfig& cfg, int device = 0);

}  // namespace demb200
