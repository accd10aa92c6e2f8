// c3-b200 extension: co-residency in the interference model
// (include/c3sim/coresident.hpp). Same two-phase fluid form as simulate()
// (reference proj/src/sim.cpp:121-215), with the GEMM on every CU and the
// collective beside it instead of a CU partition.
#include "c3sim/coresident.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>

#include "c3sim/errors.hpp"
#include "c3sim/taxonomy.hpp"
#include "json.hpp"

namespace c3sim {

using nlohmann::json;

void validate(const CommCurve& c) {
    if (c.ctas.size() != c.seconds.size()) throw ValidationError("comm curve: ctas/seconds size mismatch");
    for (std::size_t i = 0; i < c.ctas.size(); ++i) {
        if (c.ctas[i] < 1) throw ValidationError("comm curve: ctas must be >= 1");
        if (!(c.seconds[i] > 0) || !std::isfinite(c.seconds[i]))
            throw ValidationError("comm curve: times must be positive and finite");
        if (i && c.ctas[i] <= c.ctas[i - 1]) throw ValidationError("comm curve: ctas must be strictly increasing");
    }
}

double CommCurve::time_at(int cus) const {
    if (ctas.empty()) throw ValidationError("comm curve: empty");
    if (cus <= ctas.front()) return seconds.front() * ctas.front() / std::max(cus, 1);
    if (cus >= ctas.back()) return seconds.back();
    const auto hi = std::upper_bound(ctas.begin(), ctas.end(), cus) - ctas.begin();
    const auto lo = hi - 1;
    const double f = static_cast<double>(cus - ctas[lo]) / (ctas[hi] - ctas[lo]);
    return seconds[lo] + f * (seconds[hi] - seconds[lo]);
}

SlowdownTable CommCurve::as_table(KernelClass cls, const MachineDescriptor& md) const {
    validate(*this);
    SlowdownTable t{cls, {}};
    const int grain = std::max(md.min_cu_grain, 1);
    const double full = time_at(md.cus_per_gpu);
    for (int c = grain; c < md.cus_per_gpu; c += grain)
        t.points.push_back({c, std::max(1.0, time_at(c) / full)});
    t.points.push_back({md.cus_per_gpu, 1.0});
    return t;
}

void validate(const CoResidentParams& p) {
    for (double v : {p.gemm_compute_bound, p.gemm_memory_bound, p.comm})
        if (!(v >= 1.0) || !std::isfinite(v)) throw ValidationError("co-resident penalties must be finite and >= 1");
    if (!(p.comm_all_to_all == 0.0 || (p.comm_all_to_all >= 1.0 && std::isfinite(p.comm_all_to_all))))
        throw ValidationError("co-resident all-to-all cost factor must be 0 (= comm) or >= 1");
    if (!(p.comm_memory_bound == 0.0 || (p.comm_memory_bound >= 1.0 && std::isfinite(p.comm_memory_bound))))
        throw ValidationError("co-resident memory-bound cost factor must be 0 (= class factor) or >= 1");
    if (!(p.rate_exponent > 0) || !std::isfinite(p.rate_exponent))
        throw ValidationError("co-resident rate exponent must be finite and > 0");
    if (!(p.comm_reduce_scatter == 0.0 || (p.comm_reduce_scatter >= 1.0 && std::isfinite(p.comm_reduce_scatter))))
        throw ValidationError("co-resident reduce-scatter cost factor must be 0 (= all-to-all class) or >= 1");
    if (!(p.comm_all_gather_two_ranks == 0.0 ||
          (p.comm_all_gather_two_ranks >= 1.0 && std::isfinite(p.comm_all_gather_two_ranks))))
        throw ValidationError("co-resident two-rank all-gather cost factor must be 0 (= all-to-all class) or >= 1");
    if (!(p.cta_cost >= 0.0) || !std::isfinite(p.cta_cost))
        throw ValidationError("co-resident CTA cost must be finite and >= 0");
}

CoResidentParams load_coresident_params(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open file: " + path.string());
    std::ostringstream os;
    os << f.rdbuf();
    json j;
    try {
        j = json::parse(os.str());
    } catch (const json::exception& e) {
        throw IoError("co-resident params: " + std::string(e.what()));
    }
    CoResidentParams p;
    try {
        p.gemm_compute_bound = j.at("gemm-compute-bound").get<double>();
        p.gemm_memory_bound = j.at("gemm-memory-bound").get<double>();
        p.comm = j.value("comm", 1.0);
        p.rate_exponent = j.value("rate-exponent", 1.0);
        p.comm_all_to_all = j.value("comm-all-to-all", 0.0);
        p.all_gather_by_ranks = j.value("all-gather-by-ranks", false);
        p.comm_memory_bound = j.value("comm-memory-bound", 0.0);
        p.cta_cost = j.value("cta-cost", 0.0);
        p.comm_reduce_scatter = j.value("comm-reduce-scatter", 0.0);
        p.comm_all_gather_two_ranks = j.value("comm-all-gather-2", 0.0);
    } catch (const json::exception& e) {
        throw ValidationError("co-resident params: " + std::string(e.what()));
    }
    validate(p);
    return p;
}

std::string save_coresident_params(const CoResidentParams& p) {
    json j = {{"gemm-compute-bound", p.gemm_compute_bound},
              {"gemm-memory-bound", p.gemm_memory_bound},
              {"comm", p.comm},
              {"comm-all-to-all", p.comm_all_to_all},
              {"rate-exponent", p.rate_exponent}};
    if (p.all_gather_by_ranks) j["all-gather-by-ranks"] = true;
    if (p.comm_memory_bound > 0.0) j["comm-memory-bound"] = p.comm_memory_bound;
    if (p.cta_cost > 0.0) j["cta-cost"] = p.cta_cost;
    if (p.comm_reduce_scatter > 0.0) j["comm-reduce-scatter"] = p.comm_reduce_scatter;
    if (p.comm_all_gather_two_ranks > 0.0) j["comm-all-gather-2"] = p.comm_all_gather_two_ranks;
    return j.dump(2) + "\n";
}

int coresident_comm_ctas(int cus_comm, const CoResidentParams& p, KernelClass comm_class, int n_ranks,
                         KernelClass gemm_class) {
    validate(p);
    return std::max(1, static_cast<int>(std::lround(cus_comm / p.comm_factor(comm_class, n_ranks, gemm_class))));
}

SimTimeline simulate_coresident(double t_gemm, double t_comm_at_ctas, double t_comm_full, int cus,
                                int cus_comm, KernelClass gemm_class, const CoResidentParams& p,
                                double rate_ratio, double t_comm_alone_at_ctas) {
    if (!(t_comm_alone_at_ctas > 0)) t_comm_alone_at_ctas = t_comm_at_ctas;
    validate(p);
    if (!(t_gemm > 0) || !(t_comm_at_ctas > 0) || !(t_comm_full > 0))
        throw ValidationError("simulate_coresident: isolated times must be positive");
    if (!(rate_ratio > 0) || rate_ratio > 1.0 + 1e-12)
        throw ValidationError("simulate_coresident: rate_ratio must be in (0, 1]");
    SimTimeline tl;
    tl.serial_time = t_gemm + t_comm_full;
    tl.ideal = ideal_speedup(t_gemm, t_comm_full);
    tl.work_gemm = t_gemm;
    tl.work_comm = t_comm_full;
    // phase 1: both resident; rates in units of each kernel's isolated work
    const double rg = 1.0 / (1.0 + (p.gemm(gemm_class) - 1.0) * std::pow(rate_ratio, p.rate_exponent) +
                             p.cta_cost * static_cast<double>(cus_comm) / static_cast<double>(cus));
    const double rc = t_comm_full / t_comm_at_ctas;
    const double end_g = t_gemm / rg, end_c = t_comm_full / rc;
    const double t1 = std::min(end_g, end_c);
    tl.phases.push_back({0.0, t1, rg, rc, cus, cus_comm});
    if (end_c < end_g) {  // GEMM finishes alone at its isolated rate
        tl.makespan = t1 + (t_gemm - t1 * rg);
        tl.phases.push_back({t1, tl.makespan, 1.0, 0.0, cus, 0});
    } else if (end_g < end_c) {  // the collective finishes alone on its CTAs
        // its CTAs alone on their SMs now: the curve's time, no co-residency factor
        tl.makespan = t1 + (t_comm_full - t1 * rc) * (t_comm_alone_at_ctas / t_comm_full);
        tl.phases.push_back({t1, tl.makespan, 0.0, t_comm_full / t_comm_alone_at_ctas, 0, cus_comm});
    } else {
        tl.makespan = t1;
    }
    tl.speedup = tl.serial_time / tl.makespan;
    tl.fraction_of_ideal = fraction_of_ideal(tl.speedup, tl.ideal);
    return tl;
}

double fit_coresident_gemm_penalty(double t_gemm, double t_comm_at_ctas, double makespan) {
    // makespan = T1 + t_gemm - T1 / p_g with T1 = t_comm_at_ctas (p_c = 1)
    const double T1 = t_comm_at_ctas;
    if (!(t_gemm > 0 && T1 > 0 && makespan > 0) || T1 >= makespan) return 1.0;
    const double done = t_gemm + T1 - makespan;  // GEMM work done during phase 1
    if (done <= 0) return 100.0;
    return std::clamp(T1 / done, 1.0, 100.0);
}

}  // namespace c3sim
