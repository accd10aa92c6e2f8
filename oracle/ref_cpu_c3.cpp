// The reference's CPU path for the C3 scenario, timed on this host.
// TEST / BASELINE INFRASTRUCTURE ONLY (bench.py --impl reference, cpu_baseline).
//
// The reference itself is an analytic model (proj/src/sim.cpp:121-215): its own
// CPU path "executes" a C3 scenario by predicting it. This driver reports both:
//   * the executed CPU C3 of BASELINE.json configs[0]: fp32 GEMM MxNxK on all
//     host threads concurrently with the all-gather the REFERENCE planner emits
//     (plan_all_gather, proj/src/conccl.cpp:24-53) replayed by memcpy on one
//     extra thread (oracle/c3oracle.c c3o_cpu_c3), 6 warm-up + 9 measured
//     (PAPER.md:158), medians;
//   * the reference simulate() prediction for the same scenario on the
//     machine file given (speedup/ideal/fraction for c3_base and conccl).
//
// usage: c3sim_ref_cpu_c3 M N K n_ranks payload_bytes threads warmup iters machine.json [kind]
// kind: all-gather (default; plan_all_gather), all-to-all or reduce-scatter
// (plan_all_to_all, conccl.cpp:55-84 -- the reduce-scatter copy phase -- then a
// local fp32 reduce).
// prints one JSON object.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "c3oracle.h"
#include "c3sim/conccl.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/sim.hpp"
#include "c3sim/taxonomy.hpp"

using namespace c3sim;

int main(int argc, char** argv) {
    if (argc < 10) {
        std::fprintf(stderr, "usage: M N K n_ranks payload threads warmup iters machine.json\n");
        return 2;
    }
    const long long M = std::stoll(argv[1]), N = std::stoll(argv[2]), K = std::stoll(argv[3]);
    const int n = std::stoi(argv[4]);
    const long long payload = std::stoll(argv[5]);
    int threads = std::stoi(argv[6]);
    const int warmup = std::stoi(argv[7]), iters = std::stoi(argv[8]);
    if (threads <= 0) threads = std::max(1u, std::thread::hardware_concurrency());
    try {
        const MachineDescriptor md = load_machine_file(argv[9]);
        const std::string kind = argc > 10 ? argv[10] : "all-gather";
        const int k = kind == "all-gather" ? 0 : kind == "all-to-all" ? 1 : kind == "reduce-scatter" ? 2 : -1;
        if (k < 0) throw std::runtime_error("unknown collective kind " + kind);
        const TransferPlan plan =
            k == 0 ? plan_all_gather(n, payload / n, md) : plan_all_to_all(n, payload / n, md);
        std::vector<c3o_transfer> ts;
        for (const auto& t : plan.transfers)
            ts.push_back({t.src_gpu, t.dst_gpu, t.src_offset, t.dst_offset, t.length, t.engine_id,
                          t.seq});
        double out[3] = {0, 0, 0};
        if (c3o_cpu_c3_kind(M, N, K, threads, ts.data(), (int)ts.size(), n, plan.buffers.src_bytes,
                            plan.buffers.dst_bytes, k, warmup, iters, out) != 0)
            return 4;
        const double serial = out[0] + out[1];
        const double speedup = serial / out[2];
        const double ideal = ideal_speedup(out[0], out[1]);
        const double frac = ideal > 1 ? fraction_of_ideal(speedup, ideal) : 0.0;
        std::printf(
            "{\"t_gemm_s\": %.9g, \"t_comm_s\": %.9g, \"t_concurrent_s\": %.9g, "
            "\"speedup\": %.9g, \"ideal\": %.9g, \"fraction_of_ideal\": %.9g, "
            "\"threads\": %d, \"transfers\": %zu, \"kind\": \"%s\", \"warmup\": %d, \"iters\": %d}\n",
            out[0], out[1], out[2], speedup, ideal, frac, threads, ts.size(), kind.c_str(), warmup, iters);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_cpu_c3: %s\n", e.what());
        return 4;
    }
    return 0;
}
