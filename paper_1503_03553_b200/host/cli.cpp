// cli.cpp — `dem_b200 run|bench|verify <config>`: the reference CLI (tools/demforge.cpp:16-103)
// over the B200 path. Same subcommands, options (--out-dir --steps --variant --seed) and exit
// codes (0 ok, 2 config error, 3 runtime error, 4 verify failed); plus --device.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>

#include "../../include/demb200/host.hpp"

namespace {

constexpr int kOk = 0, kConfig = 2, kRuntime = 3, kVerifyFailed = 4;

int usage() {
    std::cerr << "usage: dem_b200 {run|bench|verify} <config> [--out-dir DIR] [--steps N] "
                 "[--variant baseline|two_phase] [--seed S] [--device D]\n";
    return kConfig;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) return usage();
    const std::string cmd = argv[1];
    if (cmd != "run" && cmd != "bench" && cmd != "verify") return usage();
    std::string config = argv[2], out_dir = "out", variant;
    long long steps = -1, seed = -1;
    int device = 0;
    for (int k = 3; k < argc; ++k) {
        const std::string a = argv[k];
        auto next = [&]() -> std::string {
            if (k + 1 >= argc) { usage(); std::exit(kConfig); }
            return argv[++k];
        };
        if (a == "--out-dir") out_dir = next();
        else if (a == "--steps") steps = std::atoll(next().c_str());
        else if (a == "--variant") {
            variant = next();
            if (variant != "baseline" && variant != "two_phase") return usage();
        } else if (a == "--seed") seed = std::atoll(next().c_str());
        else if (a == "--device") device = std::atoi(next().c_str());
        else return usage();
    }
    try {
        demb200::SimConfig cfg = demb200::parse_config(config);
        if (steps >= 0) cfg.run.steps = steps;
        if (!variant.empty())
            cfg.run.collide_variant = variant == "baseline" ? demb200::CollideVariant::baseline : demb200::CollideVariant::two_phase;
        if (seed >= 0) cfg.seed = static_cast<std::uint64_t>(seed);
        if (cmd == "run") {
            const auto s = demb200::run_simulation(cfg, out_dir, device);
            std::cout << "ran " << s.steps_run << " steps, wrote " << s.snapshots_written << " snapshots and "
                      << s.metrics_path.string() << "\n";
            return kOk;
        }
        if (cmd == "bench") {
            const std::string text = demb200::bench(cfg, device).format();
            std::cout << text;
            if (!out_dir.empty()) {
                std::filesystem::create_directories(out_dir);
                std::ofstream(std::filesystem::path(out_dir) / "bench_report.txt") << text;
            }
            return kOk;
        }
        const auto rep = demb200::verify(cfg, device);
        std::cout << rep.format();
        return rep.all_pass() ? kOk : kVerifyFailed;
    } catch (const demb200::ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return kConfig;
    } catch (const demb200::KernelError& e) {
        std::cerr << "runtime error: " << e.what() << "\n";
        return kRuntime;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kRuntime;
    }
}
