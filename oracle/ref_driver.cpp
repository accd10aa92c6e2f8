// Driver over the UNMODIFIED reference c3sim_core (oracle/_ref/libc3sim_ref.a).
// TEST INFRASTRUCTURE: generates golden fixtures (tests/golden/) and answers
// point queries for the parity tests. Written here; links the reference lib.
//
//   c3sim_ref_driver sweep <machine.json> <dataset.json> <tables.csv> <params.json> [zero]
//       -> reference sweep_to_csv over all strategies (proj/src/sim.cpp:256-334)
//   c3sim_ref_driver plan <all-gather|all-to-all> <n> <chunk> <machine.json>
//       -> reference to_json(plan) (proj/src/conccl.cpp:24-84,231-249)
//   c3sim_ref_driver cost <all-gather|all-to-all> <n> <chunk> <machine.json> <params.json>
//       -> plan_cost total/wire (proj/src/conccl.cpp:200-229)
#include <cstdio>
#include <iostream>
#include <string>
#include <vector>

#include "c3sim/conccl.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/params_io.hpp"
#include "c3sim/sim.hpp"

using namespace c3sim;

int main(int argc, char** argv) {
    try {
        if (argc < 2) return 2;
        const std::string cmd = argv[1];
        if (cmd == "sweep" && argc >= 6) {
            MachineDescriptor md = load_machine_file(argv[2]);
            const auto scenarios = load_dataset(argv[3]);
            SlowdownTableSet tables = load_slowdown_tables(argv[4], md.min_cu_grain);
            RunParams p = load_params_file(argv[5]);
            if (argc >= 7 && std::string(argv[6]) == "zero")
                apply_zero_interference(tables, p.penalties, p.eff, md);
            SimOptions opt;
            opt.freeze_phase2_allocation = p.freeze_phase2_allocation;
            const std::vector<Strategy> all(std::begin(kAllStrategies), std::end(kAllStrategies));
            std::cout << sweep_to_csv(sweep(scenarios, all, md, tables, p.penalties, p.eff, opt));
            return 0;
        }
        if ((cmd == "plan" || cmd == "cost") && argc >= 6) {
            const CollectiveKind kind = collective_kind_from_string(argv[2]);
            const int n = std::stoi(argv[3]);
            const long long chunk = std::stoll(argv[4]);
            const MachineDescriptor md = load_machine_file(argv[5]);
            const TransferPlan plan = kind == CollectiveKind::AllGather
                                          ? plan_all_gather(n, chunk, md)
                                          : plan_all_to_all(n, chunk, md);
            if (cmd == "plan") {
                std::cout << to_json(plan);
            } else {
                RunParams p = argc >= 7 ? load_params_file(argv[6]) : RunParams{};
                const PlanCost c = plan_cost(plan, md, p.eff);
                std::printf("%.17g %.17g\n", c.total, c.wire);
            }
            return 0;
        }
    } catch (const std::exception& e) {
        std::cerr << "ref_driver: " << e.what() << "\n";
        return 4;
    }
    std::cerr << "usage: see header\n";
    return 2;
}
