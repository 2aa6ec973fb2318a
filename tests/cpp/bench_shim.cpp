// bench_shim.cpp -- config 1 end to end through the C++ drop-in shim
// (include/ccwsim_gpu.hpp): the reference's own types in and out
// (CategoricalGrid of std::vector<int>, simulate_ensemble returning
// std::vector<SimResult>), i.e. what a reference user's code pays.
//   bench_shim <ti.bin (500*500 codes)> <steps> <warmup>
// prints one JSON object: ms per step and cells/s.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <vector>

#include "ccwsim_gpu.hpp"

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    std::ifstream f(argv[1], std::ios::binary);
    std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (bytes.size() != 500u * 500u) return 3;
    ccwsim::CategoricalGrid ti(500, 500, 3, std::vector<int>(bytes.begin(), bytes.end()));
    ccwsim::SimConfig cfg;
    cfg.sg_height = cfg.sg_width = 1000;
    cfg.template_size = 64;
    cfg.overlap = 16;
    cfg.dwt_level = 2;
    cfg.candidates = 5;
    cfg.n_realizations = 100;
    cfg.master_seed = 20240441;
    const int steps = std::atoi(argv[2]), warmup = std::atoi(argv[3]);
    long long checksum = 0;
    for (int i = 0; i < warmup; ++i) checksum += ccwsim::simulate_ensemble(ti, cfg, 8).size();
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) {
        const auto res = ccwsim::simulate_ensemble(ti, cfg, 8);
        checksum += res.back().realization.at(999, 999);
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"ms_per_step\": %.4f, \"cells_per_s\": %.6e, \"steps\": %d, \"checksum\": %lld}\n",
                1e3 * s / steps, 100.0 * 1e6 * steps / s, steps, checksum);
    return 0;
}
