// c3-b200 extension (no counterpart in the reference): co-residency in the
// interference model.
//
// The reference partitions CUs: a kernel pair shares the GPU as
// cus_gemm + cus_comm <= C (sim.cpp:40-100), and the SM strategies pay the
// GEMM's CU-loss slowdown. On B200 a P2P collective's CTA (512 threads, no
// shared memory) fits on the same SM as the persistent GEMM's CTA, so the
// GEMM keeps all C SMs and the collective runs on `cus_comm` CTAs beside it
// (DESIGN.md §5.4). This header models that execution mode with the same
// two-phase fluid form as simulate() (sim.cpp:121-215):
//   phase 1: GEMM rate 1/p_g, collective rate 1/(t_c(c)/t_c * p_c)
//   phase 2: the survivor alone at rate 1.
// t_c(c) comes from a measured CommCurve (collective time vs CTA count under
// the world's link conditions), p_g / p_c are co-residency penalties fitted
// on measured co-resident runs (tools/calibrate_coresident.py).
#pragma once

#include <filesystem>
#include <string>
#include <vector>

#include "c3sim/interference.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/sim.hpp"

namespace c3sim {

/// Measured isolated collective time (seconds) vs CTA count, under the world's
/// real (or emulated) link rate. Points sorted by ctas, times > 0.
struct CommCurve {
    std::vector<int> ctas;
    std::vector<double> seconds;

    bool empty() const { return ctas.empty(); }
    /// Linear between points; below the first point time scales as 1/ctas
    /// (bandwidth per CTA), above the last it stays flat.
    double time_at(int cus) const;
    /// Slowdown table over grain multiples up to C: t(c) / t(C), last point 1.0.
    SlowdownTable as_table(KernelClass cls, const MachineDescriptor& md) const;
};

void validate(const CommCurve& c);

/// Co-residency penalties (1.0 = no interference): the GEMM's residual
/// slowdown while a collective runs beside it, and the collective CTA's cost
/// factor: a CTA sharing its SM with the GEMM moves data like 1/comm isolated
/// CTAs, so the collective on c co-resident CTAs takes t_comm(c / comm)
/// (coresident_comm_ctas).
struct CoResidentParams {
    double gemm_compute_bound = 1.0;
    double gemm_memory_bound = 1.0;
    double comm = 1.0;
    /// The cost factor of the all-to-all class (all-to-all and reduce-scatter
    /// kernels: one store per load, or n loads per store); 0 = `comm`.
    double comm_all_to_all = 0.0;
    /// Comm pacing: the GEMM penalty's excess scales with the collective's
    /// rate as (rate / link rate)^rate_exponent; 1 = linear (pacing neutral),
    /// > 1 = spreading the collective over the GEMM pays.
    double rate_exponent = 1.0;
    /// The all-gather kernel stores each loaded vector n-1 times, so with few
    /// ranks it behaves like the all-to-all class: with this set, beside a
    /// compute-bound GEMM its factor is comm + (comm_all_to_all - comm) / (n-1)^2
    /// (measured: n = 2 / 4 / 8 fit 1.8 / 1.1 / 1.0, profiles/r01_size_sweep.csv).
    /// Beside a memory-bound GEMM (single-CTA tiles, light issue load) it stays `comm`.
    bool all_gather_by_ranks = false;
    /// The collective CTA's factor beside a memory-bound GEMM (single-CTA
    /// tiles: light issue and register pressure), any collective class;
    /// 0 = the class factor. Measured ~1.0 (RMS 30% -> 12% over 228 rows).
    double comm_memory_bound = 0.0;
    /// The GEMM's extra slowdown per resident collective CTA unit, whatever
    /// the collective's rate: excess += cta_cost * cus_comm / cus. Resident
    /// collective warps take issue slots, registers and L1 from the GEMM's
    /// CTAs even while they sleep (paced) or stall; measured: 64 all-to-all
    /// units beside the cfg4 GEMM 10% slower than 16, both collectives done
    /// well before the GEMM (profiles/r02_c3_sweep_link770.csv). 0 = off.
    double cta_cost = 0.0;
    /// The reduce-scatter pull's CTA factor (n loads and an fp32 sum per
    /// store: heavier beside the GEMM than the all-to-all push of its kernel
    /// class); 0 = the all-to-all class factor. Applied by for_kind().
    double comm_reduce_scatter = 0.0;
    /// With all_gather_by_ranks: the all-gather factor at n = 2, the limit the
    /// rank-dependent factor tends to (its one peer means one store per load,
    /// but the all-gather kernel's 32-byte vectors and 4 in flight per thread
    /// lose more beside the GEMM than the all-to-all push); 0 = comm_all_to_all.
    /// Fitted on the world-2 / 4 size sweep (profiles/r02_size_sweep_final.csv:
    /// 4.0 against the all-to-all's 2.4, pick regret at world 2 9.3% -> ~1%).
    double comm_all_gather_two_ranks = 0.0;

    /// These parameters as seen by a collective of `kind`: a reduce-scatter
    /// uses comm_reduce_scatter as its all-to-all class factor when set.
    CoResidentParams for_kind(CollectiveKind kind) const {
        CoResidentParams q = *this;
        if (kind == CollectiveKind::ReduceScatter && comm_reduce_scatter > 0.0)
            q.comm_all_to_all = comm_reduce_scatter;
        return q;
    }

    double gemm(KernelClass gemm_class) const {
        return gemm_class == KernelClass::GemmMemoryBound ? gemm_memory_bound : gemm_compute_bound;
    }
    double comm_factor(KernelClass comm_class) const {
        return comm_class == KernelClass::AllToAll && comm_all_to_all > 0.0 ? comm_all_to_all : comm;
    }
    /// n_ranks <= 1: no rank dependence (the class factor above).
    double comm_factor(KernelClass comm_class, int n_ranks, KernelClass gemm_class) const {
        if (gemm_class == KernelClass::GemmMemoryBound && comm_memory_bound > 0.0) return comm_memory_bound;
        if (comm_class != KernelClass::AllGather || !all_gather_by_ranks || n_ranks <= 1 ||
            gemm_class == KernelClass::GemmMemoryBound)
            return comm_factor(comm_class);
        const double two = comm_all_gather_two_ranks > 0.0 ? comm_all_gather_two_ranks
                           : comm_all_to_all > 0.0         ? comm_all_to_all
                                                           : comm;
        const double s = n_ranks - 1;
        return comm + (two - comm) / (s * s);
    }
};

void validate(const CoResidentParams& p);

/// JSON: {"gemm-compute-bound": pg, "gemm-memory-bound": pg, "comm": pc,
///        "comm-all-to-all": pc (optional), "rate-exponent": g (optional, default 1),
///        "all-gather-by-ranks": bool (optional, default false),
///        "comm-memory-bound": pc (optional, 0 = the class factor),
///        "cta-cost": c (optional, default 0),
///        "comm-reduce-scatter": pc (optional, 0 = the all-to-all class factor),
///        "comm-all-gather-2": pc (optional, 0 = the all-to-all class factor)}.
CoResidentParams load_coresident_params(const std::filesystem::path& path);
std::string save_coresident_params(const CoResidentParams& p);

/// Isolated-equivalent CTA count of `cus_comm` co-resident collective CTAs
/// of the given collective kernel class (n_ranks > 1 and the GEMM's class:
/// the rank-dependent all-gather factor, CoResidentParams::all_gather_by_ranks).
int coresident_comm_ctas(int cus_comm, const CoResidentParams& p,
                         KernelClass comm_class = KernelClass::AllGather, int n_ranks = 0,
                         KernelClass gemm_class = KernelClass::GemmComputeBound);

/// Two-phase fluid prediction of a co-resident run: GEMM on all CUs
/// (t_gemm seconds alone), collective on cus_comm CTAs (t_comm_at_ctas =
/// the isolated collective's time on coresident_comm_ctas(cus_comm) CTAs).
/// serial_time / ideal use t_comm_full, the collective's isolated time on the
/// whole GPU (the paper's t_comm).
/// rate_ratio (<= 1): the collective's actual rate beside the GEMM over its
/// unpaced full-GPU rate (t_comm_full / t_comm_at_ctas: pacing or few CTAs);
/// the GEMM penalty's excess scales by rate_ratio^rate_exponent.
/// A paced collective's t_comm_at_ctas is the longer of the curve time and
/// bytes / paced rate (the caller's).
/// t_comm_alone_at_ctas (> 0): the collective's time on its cus_comm CTAs once
/// the GEMM is gone (phase 2: no co-residency cost factor); 0 = t_comm_at_ctas.
SimTimeline simulate_coresident(double t_gemm, double t_comm_at_ctas, double t_comm_full, int cus,
                                int cus_comm, KernelClass gemm_class, const CoResidentParams& p,
                                double rate_ratio = 1.0, double t_comm_alone_at_ctas = 0.0);

/// Penalty p_g that makes simulate_coresident reproduce a measured makespan
/// (collective finishing first, p_c = 1); clamped to [1, 100]. Returns 1.0
/// when the GEMM finished first or the inputs leave no overlap to explain.
double fit_coresident_gemm_penalty(double t_gemm, double t_comm_at_ctas, double makespan);

}  // namespace c3sim
