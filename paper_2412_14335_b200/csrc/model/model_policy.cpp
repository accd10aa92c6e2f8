// C3 runtime policy and predictor: CU/SM-loss tables, co-run penalties, the
// paper's strategies (allocation + launch order), the RP partition heuristic,
// the ConCCL_rp rule and the two-phase fluid simulator used as the runtime
// heuristic's predictor.
//
// Reference semantics (/root/reference/proj):
//   SlowdownTable validate / slowdown_at        src/interference.cpp:14-48
//   comm_saturation_cus / default_comm_table    src/interference.cpp:50-68
//   shared_memory_factor                        src/interference.cpp:70-77
//   CoRunPenalty defaults / ones / validate     src/interference.cpp:170-208
//   schedule_priority_order                     src/strategy.cpp:23-33
//   candidate_cu_allocations / partition_heuristic  src/strategy.cpp:35-94
//   conccl_rp_plan                              src/strategy.cpp:96-113
//   Strategy names, allocate_cus                src/sim.cpp:13-100
//   dma_comm_work, simulate                     src/sim.cpp:104-215
//   work_conservation_check                     src/sim.cpp:217-237
//   sweep, sweep_to_csv                         src/sim.cpp:241-334
//   apply_zero_interference                     src/sim.cpp:336-347
// Extension: reduce-scatter maps to the all-to-all kernel class; its DMA work is
// the transpose plan's cost plus the local n-slot reduce at HBM speed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <map>
#include <numeric>
#include <sstream>

#include "c3sim/errors.hpp"
#include "c3sim/sim.hpp"

namespace c3sim {

// ------------------------------------------------------------ interference --

void validate(const SlowdownTable& t, int min_cu_grain) {
    const std::string who = "slowdown table " + to_string(t.kernel_class) + ": ";
    if (t.points.empty()) throw ValidationError(who + "empty");
    int prev = 0;
    for (std::size_t i = 0; i < t.points.size(); ++i) {
        const SlowdownPoint& pt = t.points[i];
        if (!(pt.slowdown > 0))
            throw ValidationError(who + "slowdown must be > 0 at cus=" + std::to_string(pt.cus));
        if (pt.cus < 1) throw ValidationError(who + "cus must be >= 1");
        if (min_cu_grain > 1 && pt.cus % min_cu_grain)
            throw ValidationError(who + "cus=" + std::to_string(pt.cus) +
                                  " is not a multiple of the CU grain");
        if (i > 0 && prev >= pt.cus)
            throw ValidationError(who + "cus values must be strictly increasing");
        prev = pt.cus;
    }
    if (t.points.back().slowdown != 1.0)
        throw ValidationError(who + "slowdown at max CUs must be 1.0");
}

double slowdown_at(const SlowdownTable& t, int cus) {
    const auto& pts = t.points;
    if (pts.empty()) throw ValidationError("slowdown_at: empty table");
    if (cus <= pts.front().cus) return pts.front().slowdown;
    if (cus >= pts.back().cus) return pts.back().slowdown;
    // first knot at or above `cus`; cus is strictly inside the covered range
    const auto hi = std::lower_bound(pts.begin(), pts.end(), cus,
                                     [](const SlowdownPoint& p, int c) { return p.cus < c; });
    const auto lo = hi - 1;
    const double f = static_cast<double>(cus - lo->cus) / static_cast<double>(hi->cus - lo->cus);
    return lo->slowdown + f * (hi->slowdown - lo->slowdown);
}

int comm_saturation_cus(CollectiveKind kind) {
    return kind == CollectiveKind::AllGather ? 32 : 64;
}

SlowdownTable default_comm_table(CollectiveKind kind, const MachineDescriptor& md) {
    const int grain = md.min_cu_grain > 1 ? md.min_cu_grain : 1;
    int sat = std::min(comm_saturation_cus(kind), md.cus_per_gpu);
    sat = std::max(sat - sat % grain, grain);
    SlowdownTable t{comm_kernel_class(kind), {}};
    for (int c = grain; c < sat; c += grain) t.points.push_back({c, static_cast<double>(sat) / c});
    t.points.push_back({sat, 1.0});
    if (md.cus_per_gpu > sat) t.points.push_back({md.cus_per_gpu, 1.0});
    validate(t, md.min_cu_grain);
    return t;
}

std::vector<double> shared_memory_factor(const std::vector<double>& demands,
                                         double effective_peak) {
    if (!(effective_peak > 0))
        throw ValidationError("shared_memory_factor: effective_peak must be > 0");
    const double sum = std::accumulate(demands.begin(), demands.end(), 0.0);
    return std::vector<double>(demands.size(), sum <= effective_peak ? 1.0 : sum / effective_peak);
}

const SlowdownTable& SlowdownTableSet::at(KernelClass c) const {
    return tables[static_cast<std::size_t>(c)];
}
SlowdownTable& SlowdownTableSet::at(KernelClass c) { return tables[static_cast<std::size_t>(c)]; }

double CoRunPenalty::get(KernelClass c, CommBackend b) const {
    return factor[static_cast<std::size_t>(c)][static_cast<std::size_t>(b)];
}
void CoRunPenalty::set(KernelClass c, CommBackend b, double v) {
    factor[static_cast<std::size_t>(c)][static_cast<std::size_t>(b)] = v;
}

CoRunPenalty CoRunPenalty::defaults() {
    // {CU, DMA} per class: the reference's calibration on its bundled sweep.
    CoRunPenalty p;
    p.factor = {{{1.02, 1.02}, {1.08, 1.05}, {1.40, 1.35}, {3.50, 1.80}}};
    return p;
}

CoRunPenalty CoRunPenalty::ones() {
    CoRunPenalty p;
    for (auto& row : p.factor) row.fill(1.0);
    return p;
}

void validate(const CoRunPenalty& p) {
    for (int c = 0; c < kNumKernelClasses; ++c) {
        const auto cls = static_cast<KernelClass>(c);
        const double cu = p.get(cls, CommBackend::CU), dma = p.get(cls, CommBackend::DMA);
        if (!(cu >= 1.0) || !(dma >= 1.0))
            throw ValidationError("co-run penalty " + to_string(cls) + ": factors must be >= 1");
        if (dma > cu)
            throw ValidationError("co-run penalty " + to_string(cls) +
                                  ": DMA factor must not exceed CU factor");
    }
}

KernelClass comm_kernel_class(CollectiveKind kind) {
    return kind == CollectiveKind::AllGather ? KernelClass::AllGather : KernelClass::AllToAll;
}

KernelClass gemm_kernel_class(const GemmKernel& g, double machine_ratio) {
    return classify_gemm_boundedness(g, machine_ratio) == Boundedness::MemoryBound
               ? KernelClass::GemmMemoryBound
               : KernelClass::GemmComputeBound;
}

std::string to_string(KernelClass c) {
    switch (c) {
        case KernelClass::GemmComputeBound: return "gemm-compute-bound";
        case KernelClass::GemmMemoryBound: return "gemm-memory-bound";
        case KernelClass::AllGather: return "all-gather";
        case KernelClass::AllToAll: return "all-to-all";
    }
    return "?";
}

KernelClass kernel_class_from_string(const std::string& s) {
    for (int c = 0; c < kNumKernelClasses; ++c)
        if (to_string(static_cast<KernelClass>(c)) == s) return static_cast<KernelClass>(c);
    throw ValidationError("unknown kernel class '" + s + "'");
}

// ---------------------------------------------------------------- strategy --

void validate(const PartitionPlan& p, const MachineDescriptor& md) {
    const int g = md.min_cu_grain;
    if (p.cus_comm + p.cus_gemm + p.cus_idle != md.cus_per_gpu)
        throw ValidationError("partition plan: CU counts must sum to cus_per_gpu");
    if (p.cus_comm % g || p.cus_gemm % g || p.cus_idle % g)
        throw ValidationError("partition plan: CU counts must be grain multiples");
    if (p.comm_backend == CommBackend::CU && p.cus_comm < g)
        throw ValidationError("partition plan: CU backend needs at least one grain for comm");
    if (p.cus_comm < 0 || p.cus_gemm < 0 || p.cus_idle < 0)
        throw ValidationError("partition plan: CU counts must be non-negative");
}

std::vector<KernelDemand> schedule_priority_order(std::vector<KernelDemand> kernels) {
    if (std::any_of(kernels.begin(), kernels.end(),
                    [](const KernelDemand& k) { return k.workgroups < 1; }))
        throw ValidationError("schedule_priority_order: workgroups must be >= 1");
    std::stable_sort(kernels.begin(), kernels.end(), [](const KernelDemand& a, const KernelDemand& b) {
        return a.workgroups != b.workgroups ? a.workgroups < b.workgroups : (a.is_comm && !b.is_comm);
    });
    return kernels;
}

std::vector<int> candidate_cu_allocations(const MachineDescriptor& md) {
    std::vector<int> out;
    for (int c = 8; c <= 256; c *= 2)
        if (c < md.cus_per_gpu && c % md.min_cu_grain == 0 && md.cus_per_gpu - c >= md.min_cu_grain)
            out.push_back(c);
    if (out.empty())
        throw ValidationError("partition heuristic: no feasible CU candidate on this machine");
    return out;
}

namespace {
std::string gemm_name(const C3Scenario& s) { return s.gemm.tag.empty() ? "gemm" : s.gemm.tag; }
}  // namespace

PartitionSweep partition_heuristic(const C3Scenario& scenario, const MachineDescriptor& md,
                                   const SlowdownTableSet& tables,
                                   const EfficiencyParams& params) {
    const double ratio = machine_op_to_byte(md);
    const SlowdownTable& gt = tables.at(gemm_kernel_class(scenario.gemm, ratio));
    const SlowdownTable& ct = tables.at(comm_kernel_class(scenario.collective.kind));
    const double tg = roofline_gemm_time(scenario.gemm, md, params);
    const double tc = roofline_collective_time(scenario.collective, md, params, true);

    PartitionSweep out;
    double best = std::numeric_limits<double>::infinity();
    int best_c = -1;
    for (int c : candidate_cu_allocations(md)) {
        CandidateEval e{c, tg * slowdown_at(gt, md.cus_per_gpu - c), tc * slowdown_at(ct, c), 0.0};
        e.predicted = std::max(e.gemm_term, e.comm_term);
        if (e.predicted < best) {  // strict: ties keep the earlier (smaller) c
            best = e.predicted;
            best_c = c;
        }
        out.candidates.push_back(e);
    }
    PartitionPlan& plan = out.plan;
    plan.comm_backend = CommBackend::CU;
    plan.cus_comm = best_c;
    plan.cus_gemm = md.cus_per_gpu - best_c;
    plan.cus_idle = 0;
    plan.predicted_makespan = best;
    const auto order = schedule_priority_order(
        {{gemm_name(scenario), false, estimate_workgroups(scenario.gemm)},
         {to_string(scenario.collective.kind), true, estimate_workgroups(scenario.collective)}});
    for (const KernelDemand& k : order) plan.schedule_order.push_back(k.name);
    validate(plan, md);
    return out;
}

PartitionPlan conccl_rp_plan(const C3Scenario& scenario, const MachineDescriptor& md,
                             const SlowdownTableSet& /*tables: the rule needs only boundedness*/) {
    const bool mb = classify_gemm_boundedness(scenario.gemm, machine_op_to_byte(md)) ==
                    Boundedness::MemoryBound;
    PartitionPlan plan;
    plan.comm_backend = CommBackend::DMA;
    plan.cus_comm = 0;
    plan.cus_idle = mb ? md.min_cu_grain : 0;
    plan.cus_gemm = md.cus_per_gpu - plan.cus_idle;
    plan.schedule_order = {to_string(scenario.collective.kind), gemm_name(scenario)};
    validate(plan, md);
    return plan;
}

// ------------------------------------------------------------------- sim ---

std::string to_string(Strategy s) {
    static const char* const names[] = {"serial", "c3_base", "c3_sp",    "c3_rp",
                                        "c3_sp_rp", "conccl", "conccl_rp"};
    const int i = static_cast<int>(s);
    return i >= 0 && i < 7 ? names[i] : "?";
}

Strategy strategy_from_string(const std::string& s) {
    for (Strategy st : kAllStrategies)
        if (to_string(st) == s) return st;
    throw UnknownEntityError("unknown strategy '" + s + "'");
}

Allocation allocate_cus(const C3Scenario& scenario, Strategy strategy,
                        const MachineDescriptor& md, const SlowdownTableSet& tables,
                        const EfficiencyParams& params) {
    const int C = md.cus_per_gpu, grain = md.min_cu_grain;
    const auto to_grain = [grain](int v) { return (v + grain - 1) / grain * grain; };
    Allocation a;
    switch (strategy) {
        case Strategy::Serial:  // each kernel alone on the whole GPU
            a.cus_gemm = C;
            a.cus_comm = C;
            break;
        case Strategy::C3Base: {
            // The GEMM, launched first, takes one CU per pending workgroup; the
            // late collective gets what is left but never less than a grain.
            const int gemm_wants = std::min(to_grain(estimate_workgroups(scenario.gemm)), C);
            a.cus_comm = std::max(C - gemm_wants, grain);
            a.cus_gemm = C - a.cus_comm;
            break;
        }
        case Strategy::C3Sp:  // collective first with its saturation CUs
            a.cus_comm = std::clamp(to_grain(comm_saturation_cus(scenario.collective.kind)), grain,
                                    C - grain);
            a.cus_gemm = C - a.cus_comm;
            a.comm_first = true;
            break;
        case Strategy::C3Rp:
        case Strategy::C3SpRp: {
            const PartitionSweep ps = partition_heuristic(scenario, md, tables, params);
            a.cus_comm = ps.plan.cus_comm;
            a.cus_gemm = ps.plan.cus_gemm;
            a.comm_first = true;
            break;
        }
        case Strategy::Conccl:
            a.cus_gemm = C;
            a.comm_backend = CommBackend::DMA;
            a.comm_first = true;
            break;
        case Strategy::ConcclRp: {
            const PartitionPlan p = conccl_rp_plan(scenario, md, tables);
            a.cus_gemm = p.cus_gemm;
            a.cus_comm = p.cus_comm;
            a.cus_idle = p.cus_idle;
            a.comm_backend = CommBackend::DMA;
            a.comm_first = true;
            break;
        }
    }
    return a;
}

namespace {

// Seconds the DMA backend spends on the collective: the ConCCL plan's event
// cost (plus, for reduce-scatter, the local reduce of n staged slots).
double dma_work(const C3Scenario& s, const MachineDescriptor& md, const EfficiencyParams& p) {
    const CollectiveOp& c = s.collective;
    const std::int64_t chunk = c.n_ranks > 0 ? c.payload_bytes / c.n_ranks : 0;
    const std::int64_t plan_chunk = std::max<std::int64_t>(chunk, 1);
    TransferPlan plan;
    switch (c.kind) {
        case CollectiveKind::AllGather: plan = plan_all_gather(c.n_ranks, plan_chunk, md); break;
        case CollectiveKind::AllToAll: plan = plan_all_to_all(c.n_ranks, plan_chunk, md); break;
        case CollectiveKind::ReduceScatter:
            plan = plan_reduce_scatter(c.n_ranks, plan_chunk, md);
            break;
    }
    if (chunk == 0 && c.n_ranks > 1)  // nothing to move: overheads only
        return static_cast<double>(plan.transfers.size() - 1) * md.cpu_launch_overhead +
               md.dma_sync_overhead;
    double t = plan_cost(plan, md, p).total;
    if (c.kind == CollectiveKind::ReduceScatter)
        t += static_cast<double>(c.payload_bytes + chunk) / (p.efficiency * md.hbm_bandwidth);
    return t;
}

}  // namespace

SimTimeline simulate(const C3Scenario& scenario, Strategy strategy,
                     const MachineDescriptor& md, const SlowdownTableSet& tables,
                     const CoRunPenalty& penalties, const EfficiencyParams& params,
                     const SimOptions& options) {
    validate(params);
    validate(penalties);
    validate(scenario.gemm);
    validate(scenario.collective);

    const KernelClass gcls = gemm_kernel_class(scenario.gemm, machine_op_to_byte(md));
    const KernelClass ccls = comm_kernel_class(scenario.collective.kind);
    const double tg = roofline_gemm_time(scenario.gemm, md, params);
    const double tc = roofline_collective_time(scenario.collective, md, params, true);
    if (!(tg > 0) || !(tc > 0)) throw ValidationError("simulate: isolated times must be positive");

    SimTimeline tl;
    tl.serial_time = tg + tc;
    tl.ideal = ideal_speedup(tg, tc);
    tl.work_gemm = tg;

    if (strategy == Strategy::Serial) {
        tl.work_comm = tc;
        tl.phases = {{0.0, tg, 1.0, 0.0, md.cus_per_gpu, 0},
                     {tg, tg + tc, 0.0, 1.0, 0, md.cus_per_gpu}};
        tl.makespan = tg + tc;
        tl.speedup = tl.serial_time / tl.makespan;
        tl.fraction_of_ideal = fraction_of_ideal(tl.speedup, tl.ideal);
        return tl;
    }

    Allocation a = allocate_cus(scenario, strategy, md, tables, params);
    if (options.force_cus_comm && (strategy == Strategy::C3Rp || strategy == Strategy::C3SpRp)) {
        a.cus_comm = *options.force_cus_comm;
        a.cus_gemm = md.cus_per_gpu - a.cus_comm;
        a.cus_idle = 0;
    }
    const bool dma = a.comm_backend == CommBackend::DMA;
    const double wc = dma ? dma_work(scenario, md, params) : tc;
    tl.work_comm = wc;

    // Phase 1: both kernels resident.
    const double sg = slowdown_at(tables.at(gcls), a.cus_gemm);
    const double sc = dma ? 1.0 : slowdown_at(tables.at(ccls), a.cus_comm);
    const double mem = shared_memory_factor({gemm_bandwidth_demand(scenario.gemm, md, params),
                                             collective_bandwidth_demand(scenario.collective, md, params)},
                                            params.efficiency * md.hbm_bandwidth)[0];
    const double rg = 1.0 / (sg * mem * penalties.get(gcls, a.comm_backend));
    const double rc = 1.0 / (sc * mem * penalties.get(ccls, a.comm_backend));
    if (!(rg > 0) || !(rc > 0)) throw ValidationError("simulate: non-positive phase rate");
    const double end_g = tg / rg, end_c = wc / rc;
    const double t1 = std::min(end_g, end_c);
    tl.phases.push_back({0.0, t1, rg, rc, a.cus_gemm, a.cus_comm});

    // Phase 2: the survivor runs alone (isolated rate unless frozen).
    const bool freeze = options.freeze_phase2_allocation;
    if (end_g == end_c) {
        tl.makespan = t1;
    } else if (end_g < end_c) {
        const double left = std::max(0.0, wc - t1 * rc);
        const double r2 = freeze && !dma ? 1.0 / sc : 1.0;
        const int cus2 = freeze ? a.cus_comm : (dma ? 0 : md.cus_per_gpu);
        tl.makespan = t1 + left / r2;
        tl.phases.push_back({t1, tl.makespan, 0.0, r2, 0, cus2});
    } else {
        const double left = std::max(0.0, tg - t1 * rg);
        const double r2 = freeze ? 1.0 / sg : 1.0;
        const int cus2 = freeze ? a.cus_gemm : md.cus_per_gpu;
        tl.makespan = t1 + left / r2;
        tl.phases.push_back({t1, tl.makespan, r2, 0.0, cus2, 0});
    }
    tl.speedup = tl.serial_time / tl.makespan;
    tl.fraction_of_ideal = fraction_of_ideal(tl.speedup, tl.ideal);
    return tl;
}

void work_conservation_check(const SimTimeline& tl) {
    double g = 0.0, c = 0.0, cursor = 0.0;
    const double tol = 1e-9 * std::max(1.0, tl.makespan);
    for (const PhaseRecord& ph : tl.phases) {
        if (std::abs(ph.start - cursor) > tol)
            throw ValidationError("work conservation: phases are not contiguous");
        const double d = ph.end - ph.start;
        if (d < 0) throw ValidationError("work conservation: negative phase duration");
        g += d * ph.rate_gemm;
        c += d * ph.rate_comm;
        cursor = ph.end;
    }
    const auto check = [](double done, double work, const char* what) {
        const double rel = std::abs(done - work) / std::max(work, 1e-300);
        if (rel > 1e-9)
            throw ValidationError(std::string("work conservation: ") + what +
                                  " progress off by relative " + std::to_string(rel));
    };
    check(g, tl.work_gemm, "gemm");
    check(c, tl.work_comm, "comm");
}

SweepResult sweep(const std::vector<C3Scenario>& scenarios,
                  const std::vector<Strategy>& strategies, const MachineDescriptor& md,
                  const SlowdownTableSet& tables, const CoRunPenalty& penalties,
                  const EfficiencyParams& params, const SimOptions& options) {
    SweepResult res;
    for (const C3Scenario& s : scenarios) {
        TaxonomyClass tax;
        if (s.expected_taxonomy) {
            tax = *s.expected_taxonomy;
        } else {
            tax = classify_c3(roofline_gemm_time(s.gemm, md, params),
                              roofline_collective_time(s.collective, md, params, true))
                      .value;
        }
        for (Strategy st : strategies) {
            const SimTimeline tl = simulate(s, st, md, tables, penalties, params, options);
            work_conservation_check(tl);
            res.rows.push_back({s.id, s.collective.kind, tax, st, tl.makespan, tl.speedup, tl.ideal,
                                tl.fraction_of_ideal});
        }
    }
    std::stable_sort(res.rows.begin(), res.rows.end(), [](const SweepRow& a, const SweepRow& b) {
        if (a.scenario_id != b.scenario_id) return a.scenario_id < b.scenario_id;
        if (a.collective != b.collective) return static_cast<int>(a.collective) < static_cast<int>(b.collective);
        return static_cast<int>(a.strategy) < static_cast<int>(b.strategy);
    });

    struct Sum {
        int n = 0;
        double speedup = 0.0, ideal = 0.0, frac = 0.0;
        void add(const SweepRow& r) {
            ++n;
            speedup += r.speedup;
            ideal += r.ideal;
            frac += r.fraction_of_ideal;
        }
    };
    for (Strategy st : strategies) {
        std::map<std::pair<int, int>, Sum> by_group;  // (collective, taxonomy), ordered
        Sum all;
        for (const SweepRow& r : res.rows) {
            if (r.strategy != st) continue;
            by_group[{static_cast<int>(r.collective), static_cast<int>(r.taxonomy)}].add(r);
            all.add(r);
        }
        for (const auto& [key, s] : by_group)
            res.aggregates.push_back({static_cast<CollectiveKind>(key.first),
                                      static_cast<TaxonomyClass>(key.second), st, s.n,
                                      s.speedup / s.n, s.ideal / s.n, s.frac / s.n});
        if (all.n > 0)
            res.aggregates.push_back({std::nullopt, std::nullopt, st, all.n, all.speedup / all.n,
                                      all.ideal / all.n, all.frac / all.n});
    }
    return res;
}

namespace {
std::string g12(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.12g", v);
    return buf;
}
}  // namespace

std::string sweep_to_csv(const SweepResult& result) {
    std::ostringstream os;
    os << "scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal\n";
    for (const SweepRow& r : result.rows)
        os << r.scenario_id << ',' << to_string(r.collective) << ',' << to_string(r.taxonomy) << ','
           << to_string(r.strategy) << ',' << g12(r.makespan) << ',' << g12(r.speedup) << ','
           << g12(r.ideal) << ',' << g12(r.fraction_of_ideal) << '\n';
    for (const AggregateRow& a : result.aggregates)
        os << "mean," << (a.collective ? to_string(*a.collective) : std::string("all")) << ','
           << (a.taxonomy ? to_string(*a.taxonomy) : std::string("all")) << ','
           << to_string(a.strategy) << ",," << g12(a.mean_speedup) << ',' << g12(a.mean_ideal)
           << ',' << g12(a.mean_fraction_of_ideal) << '\n';
    return os.str();
}

void apply_zero_interference(SlowdownTableSet& tables, CoRunPenalty& penalties,
                             EfficiencyParams& params, MachineDescriptor& md) {
    for (int i = 0; i < kNumKernelClasses; ++i)
        tables.tables[static_cast<std::size_t>(i)] = {static_cast<KernelClass>(i), {{md.cus_per_gpu, 1.0}}};
    penalties = CoRunPenalty::ones();
    params.comm_launch_overhead_cu = 0.0;
    md.cpu_launch_overhead = 0.0;
    md.dma_sync_overhead = 0.0;
}

}  // namespace c3sim
