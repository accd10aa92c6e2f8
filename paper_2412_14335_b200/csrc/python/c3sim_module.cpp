// _c3sim — Python extension over the PRODUCT model layer (libc3sim) and the B200
// execution API (include/c3sim/exec.hpp -> libc3cuda). Module name, class,
// enum, function and keyword names follow the reference's Python surface
// (/root/reference/proj/python/bindings.cpp:16-290, consumed through
// proj/python/c3sim/__init__.py), so the reference's own `c3sim` package and
// its tests/python/test_smoke.py run unchanged on top of this .so
// (tests/test_pymodule.py).
//
// Extensions: CollectiveKind.REDUCE_SCATTER, plan_reduce_scatter, DeviceError,
// and the execution layer: World, ExecResult, execute(), measure_isolated().
#include <pybind11/functional.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>
#include <pybind11/stl/filesystem.h>

#include <cstring>
#include <optional>

#include "c3sim/calibrate.hpp"
#include "c3sim/conccl.hpp"
#include "c3sim/coresident.hpp"
#include "c3sim/errors.hpp"
#include "c3sim/exec.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/params_io.hpp"
#include "c3sim/sim.hpp"
#include "c3sim/strategy.hpp"

namespace py = pybind11;
namespace cs = c3sim;

// Field-binding shorthands: RW = read/write attribute, RO = read-only.
#define RW(T, f) def_readwrite(#f, &T::f)
#define RO(T, f) def_readonly(#f, &T::f)

namespace {

void add_errors(py::module_& m) {
    py::register_exception<cs::IoError>(m, "IoError");
    py::register_exception<cs::UnknownEntityError>(m, "UnknownEntityError");
    auto validation = py::register_exception<cs::ValidationError>(m, "ValidationError");
    py::register_exception<cs::FitError>(m, "FitError");
    py::register_exception<cs::DeviceError>(m, "DeviceError");
    py::register_exception<cs::UnsupportedError>(m, "UnsupportedError", validation.ptr());
}

void add_enums(py::module_& m) {
    py::enum_<cs::Topology>(m, "Topology").value("FULLY_CONNECTED", cs::Topology::FullyConnected);
    py::enum_<cs::CollectiveKind>(m, "CollectiveKind")
        .value("ALL_GATHER", cs::CollectiveKind::AllGather)
        .value("ALL_TO_ALL", cs::CollectiveKind::AllToAll)
        .value("REDUCE_SCATTER", cs::CollectiveKind::ReduceScatter);
    py::enum_<cs::Boundedness>(m, "Boundedness")
        .value("COMPUTE_BOUND", cs::Boundedness::ComputeBound)
        .value("MEMORY_BOUND", cs::Boundedness::MemoryBound);
    py::enum_<cs::CommBoundedness>(m, "CommBoundedness")
        .value("LATENCY_BOUND", cs::CommBoundedness::LatencyBound)
        .value("BANDWIDTH_BOUND", cs::CommBoundedness::BandwidthBound);
    py::enum_<cs::TaxonomyClass>(m, "TaxonomyClass")
        .value("G_LONG", cs::TaxonomyClass::GLong)
        .value("C_LONG", cs::TaxonomyClass::CLong)
        .value("GC_EQUAL", cs::TaxonomyClass::GCEqual);
    py::enum_<cs::KernelClass>(m, "KernelClass")
        .value("GEMM_COMPUTE_BOUND", cs::KernelClass::GemmComputeBound)
        .value("GEMM_MEMORY_BOUND", cs::KernelClass::GemmMemoryBound)
        .value("ALL_GATHER", cs::KernelClass::AllGather)
        .value("ALL_TO_ALL", cs::KernelClass::AllToAll);
    py::enum_<cs::CommBackend>(m, "CommBackend")
        .value("CU", cs::CommBackend::CU)
        .value("DMA", cs::CommBackend::DMA);
    py::enum_<cs::Strategy> st(m, "Strategy");
    const char* names[] = {"SERIAL", "C3_BASE", "C3_SP", "C3_RP", "C3_SP_RP", "CONCCL", "CONCCL_RP"};
    for (cs::Strategy s : cs::kAllStrategies) st.value(names[static_cast<int>(s)], s);
}

void add_machine(py::module_& m) {
    using M = cs::MachineDescriptor;
    py::class_<M>(m, "MachineDescriptor")
        .def(py::init<>())
        .RW(M, gpus_per_node).RW(M, cus_per_gpu).RW(M, xcds_per_gpu).RW(M, cus_per_xcd)
        .RW(M, min_cu_grain).RW(M, dma_engines_per_gpu).RW(M, peak_compute_flops)
        .RW(M, hbm_bandwidth).RW(M, llc_capacity).RW(M, link_bandwidth_unidir)
        .RW(M, links_per_gpu).RW(M, topology).RW(M, cpu_launch_overhead).RW(M, dma_sync_overhead);
    m.def("load_machine", &cs::load_machine, py::arg("config_text"));
    m.def("load_machine_file", &cs::load_machine_file, py::arg("path"));
    m.def("save_machine", &cs::save_machine, py::arg("machine"));
    m.def("machine_op_to_byte", &cs::machine_op_to_byte, py::arg("machine"));
}

void add_workload(py::module_& m) {
    using G = cs::GemmKernel;
    using C = cs::CollectiveOp;
    using S = cs::C3Scenario;
    using E = cs::EfficiencyParams;
    py::class_<G>(m, "GemmKernel")
        .def(py::init<>())
        .RW(G, tag).RW(G, m).RW(G, n).RW(G, k).RW(G, dtype_bytes)
        .RW(G, measured_op_to_byte).RW(G, measured_time).RW(G, boundedness_override);
    py::class_<C>(m, "CollectiveOp")
        .def(py::init<>())
        .RW(C, kind).RW(C, payload_bytes).RW(C, n_ranks).RW(C, measured_time);
    py::class_<S>(m, "C3Scenario")
        .def(py::init<>())
        .RW(S, id).RW(S, gemm).RW(S, collective).RW(S, source).RW(S, expected_taxonomy);
    py::class_<E>(m, "EfficiencyParams")
        .def(py::init<>())
        .RW(E, efficiency).RW(E, comm_launch_overhead_cu);

    m.def("gemm_flops", &cs::gemm_flops);
    m.def("gemm_min_bytes", &cs::gemm_min_bytes);
    m.def("classify_gemm_boundedness", &cs::classify_gemm_boundedness);
    m.def("classify_collective_boundedness", &cs::classify_collective_boundedness);
    m.def("roofline_gemm_time", &cs::roofline_gemm_time);
    m.def("roofline_collective_time", &cs::roofline_collective_time, py::arg("collective"),
          py::arg("machine"), py::arg("params"), py::arg("include_overhead"));
    m.def("estimate_gemm_workgroups",
          [](const G& g, int tile) { return cs::estimate_workgroups(g, tile); }, py::arg("gemm"),
          py::arg("tile") = 128);
    m.def("estimate_collective_workgroups", [](const C& c) { return cs::estimate_workgroups(c); });
    m.def("gemm_bandwidth_demand", &cs::gemm_bandwidth_demand);
    m.def("collective_bandwidth_demand", &cs::collective_bandwidth_demand);
    m.def("load_dataset", &cs::load_dataset, py::arg("path"));
    m.def("parse_dataset", &cs::parse_dataset);

    using MC = cs::ModelConfig;
    using MW = cs::ModelWorkload;
    py::class_<MC>(m, "ModelConfig")
        .def(py::init<>())
        .RW(MC, hidden).RW(MC, ffn).RW(MC, tokens).RW(MC, dtype_bytes).RW(MC, shards);
    py::class_<MW>(m, "ModelWorkload").RO(MW, gemms).RO(MW, all_gathers);
    m.def("ingest_model", &cs::ingest_model);
}

void add_taxonomy(py::module_& m) {
    using L = cs::TaxonomyLabel;
    py::class_<L>(m, "TaxonomyLabel").RO(L, value).RO(L, threshold);
    m.def("classify_c3", &cs::classify_c3, py::arg("t_gemm"), py::arg("t_comm"),
          py::arg("threshold") = 1.15);
    m.def("ideal_speedup", &cs::ideal_speedup);
    m.def("fraction_of_ideal", &cs::fraction_of_ideal);
}

void add_interference(py::module_& m) {
    using P = cs::SlowdownPoint;
    using T = cs::SlowdownTable;
    using R = cs::CoRunPenalty;
    py::class_<P>(m, "SlowdownPoint").RW(P, cus).RW(P, slowdown);
    py::class_<T>(m, "SlowdownTable").RW(T, kernel_class).RW(T, points);
    py::class_<cs::SlowdownTableSet>(m, "SlowdownTableSet")
        .def("at", [](const cs::SlowdownTableSet& s, cs::KernelClass c) -> const T& { return s.at(c); },
             py::return_value_policy::reference_internal)
        .def("set", [](cs::SlowdownTableSet& s, cs::KernelClass c, const T& t) { s.at(c) = t; });
    m.def("slowdown_at", &cs::slowdown_at);
    m.def("comm_saturation_cus", &cs::comm_saturation_cus);
    m.def("default_comm_table", &cs::default_comm_table);
    m.def("shared_memory_factor", &cs::shared_memory_factor);
    m.def("load_slowdown_tables", &cs::load_slowdown_tables, py::arg("path"), py::arg("min_cu_grain") = 1);
    m.def("save_slowdown_tables", &cs::save_slowdown_tables);
    py::class_<R>(m, "CoRunPenalty")
        .def(py::init([] { return R::defaults(); }))
        .def_static("defaults", &R::defaults)
        .def_static("ones", &R::ones)
        .def("get", &R::get)
        .def("set", &R::set);

    using RP = cs::RunParams;
    py::class_<RP>(m, "RunParams")
        .def(py::init<>())
        .RW(RP, eff).RW(RP, penalties).RW(RP, freeze_phase2_allocation);
    m.def("load_params_file", &cs::load_params_file, py::arg("path"));
    m.def("save_params", &cs::save_params);
}

void add_strategy(py::module_& m) {
    using PP = cs::PartitionPlan;
    using CE = cs::CandidateEval;
    using PS = cs::PartitionSweep;
    py::class_<PP>(m, "PartitionPlan")
        .RO(PP, comm_backend).RO(PP, cus_comm).RO(PP, cus_gemm).RO(PP, cus_idle)
        .RO(PP, schedule_order).RO(PP, predicted_makespan);
    py::class_<CE>(m, "CandidateEval").RO(CE, cus_comm).RO(CE, gemm_term).RO(CE, comm_term).RO(CE, predicted);
    py::class_<PS>(m, "PartitionSweep").RO(PS, plan).RO(PS, candidates);
    m.def("partition_heuristic", &cs::partition_heuristic);
    m.def("conccl_rp_plan", &cs::conccl_rp_plan);
}

void add_conccl(py::module_& m) {
    using X = cs::Transfer;
    using TP = cs::TransferPlan;
    py::class_<X>(m, "Transfer")
        .RO(X, src_gpu).RO(X, dst_gpu).RO(X, src_offset).RO(X, dst_offset).RO(X, length)
        .RO(X, engine_id).RO(X, seq);
    py::class_<TP>(m, "TransferPlan").RO(TP, kind).RO(TP, n_ranks).RO(TP, chunk_bytes).RO(TP, transfers);
    py::class_<cs::PlanCheck>(m, "PlanCheck").RO(cs::PlanCheck, ok).RO(cs::PlanCheck, error);
    py::class_<cs::PlanCost>(m, "PlanCost")
        .RO(cs::PlanCost, total).RO(cs::PlanCost, per_engine).RO(cs::PlanCost, wire);
    m.def("plan_all_gather", &cs::plan_all_gather);
    m.def("plan_all_to_all", &cs::plan_all_to_all);
    m.def("plan_reduce_scatter", &cs::plan_reduce_scatter);
    m.def("validate_plan", &cs::validate_plan);
    m.def("plan_cost", &cs::plan_cost);
    m.def("plan_to_json", [](const TP& p) { return cs::to_json(p); });
}

void add_sim(py::module_& m) {
    using PR = cs::PhaseRecord;
    using TL = cs::SimTimeline;
    using SO = cs::SimOptions;
    using A = cs::Allocation;
    py::class_<PR>(m, "PhaseRecord")
        .RO(PR, start).RO(PR, end).RO(PR, rate_gemm).RO(PR, rate_comm).RO(PR, cus_gemm).RO(PR, cus_comm);
    py::class_<TL>(m, "SimTimeline")
        .RO(TL, phases).RO(TL, makespan).RO(TL, serial_time).RO(TL, speedup).RO(TL, ideal)
        .RO(TL, fraction_of_ideal).RO(TL, work_gemm).RO(TL, work_comm);
    py::class_<SO>(m, "SimOptions").def(py::init<>()).RW(SO, freeze_phase2_allocation).RW(SO, force_cus_comm);
    py::class_<A>(m, "Allocation")
        .RO(A, cus_gemm).RO(A, cus_comm).RO(A, cus_idle).RO(A, comm_backend).RO(A, comm_first);
    m.def("allocate_cus", &cs::allocate_cus);
    m.def("simulate", &cs::simulate, py::arg("scenario"), py::arg("strategy"), py::arg("machine"),
          py::arg("tables"), py::arg("penalties"), py::arg("params"), py::arg("options") = SO{});
    m.def("work_conservation_check", &cs::work_conservation_check);

    // B200 extension: co-residency in the model (c3sim/coresident.hpp)
    using CC = cs::CommCurve;
    py::class_<CC>(m, "CommCurve")
        .def(py::init<>())
        .def(py::init([](std::vector<int> c, std::vector<double> t) { return CC{std::move(c), std::move(t)}; }),
             py::arg("ctas"), py::arg("seconds"))
        .RW(CC, ctas).RW(CC, seconds)
        .def("time_at", &CC::time_at)
        .def("as_table", &CC::as_table);
    using CRP = cs::CoResidentParams;
    py::class_<CRP>(m, "CoResidentParams")
        .def(py::init<>())
        .RW(CRP, gemm_compute_bound).RW(CRP, gemm_memory_bound).RW(CRP, comm).RW(CRP, comm_all_to_all)
        .RW(CRP, rate_exponent).RW(CRP, all_gather_by_ranks).RW(CRP, comm_memory_bound).RW(CRP, cta_cost)
        .RW(CRP, comm_reduce_scatter).RW(CRP, comm_all_gather_two_ranks).def("for_kind", &CRP::for_kind);
    m.def("load_coresident_params", &cs::load_coresident_params);
    m.def("save_coresident_params", &cs::save_coresident_params);
    m.def("simulate_coresident", &cs::simulate_coresident, py::arg("t_gemm"), py::arg("t_comm_at_ctas"),
          py::arg("t_comm_full"), py::arg("cus"), py::arg("cus_comm"), py::arg("gemm_class"), py::arg("params"),
          py::arg("rate_ratio") = 1.0, py::arg("t_comm_alone_at_ctas") = 0.0);
    m.def("fit_coresident_gemm_penalty", &cs::fit_coresident_gemm_penalty);
    m.def("coresident_comm_ctas", &cs::coresident_comm_ctas, py::arg("cus_comm"), py::arg("params"),
          py::arg("comm_class") = cs::KernelClass::AllGather, py::arg("n_ranks") = 0,
          py::arg("gemm_class") = cs::KernelClass::GemmComputeBound);

    using SR = cs::SweepRow;
    using AR = cs::AggregateRow;
    py::class_<SR>(m, "SweepRow")
        .RO(SR, scenario_id).RO(SR, collective).RO(SR, taxonomy).RO(SR, strategy).RO(SR, makespan)
        .RO(SR, speedup).RO(SR, ideal).RO(SR, fraction_of_ideal);
    py::class_<AR>(m, "AggregateRow")
        .RO(AR, collective).RO(AR, taxonomy).RO(AR, strategy).RO(AR, count).RO(AR, mean_speedup)
        .RO(AR, mean_ideal).RO(AR, mean_fraction_of_ideal);
    py::class_<cs::SweepResult>(m, "SweepResult").RO(cs::SweepResult, rows).RO(cs::SweepResult, aggregates);
    m.def("sweep", &cs::sweep, py::arg("scenarios"), py::arg("strategies"), py::arg("machine"),
          py::arg("tables"), py::arg("penalties"), py::arg("params"), py::arg("options") = SO{});
    m.def("sweep_to_csv", &cs::sweep_to_csv);
}

void add_calibrate(py::module_& m) {
    using MS = cs::MeasuredSample;
    using FR = cs::FitResult;
    py::class_<MS>(m, "MeasuredSample")
        .def(py::init<>())
        .RW(MS, scenario_id).RW(MS, collective).RW(MS, strategy).RW(MS, measured_speedup);
    py::class_<FR>(m, "FitResult").RO(FR, penalties).RO(FR, rms_residual).RO(FR, iterations);
    m.def("load_measured_csv", &cs::load_measured_csv, py::arg("path"));
    m.def("fit_penalties", &cs::fit_penalties);
    m.def("strategy_name", [](cs::Strategy s) { return cs::to_string(s); });
    m.def("taxonomy_name", [](cs::TaxonomyClass t) { return cs::to_string(t); });
    m.def("collective_name", [](cs::CollectiveKind k) { return cs::to_string(k); });
}

// ---- execution (no reference counterpart: the reference only models) ----

cs::ExecMode mode_of(const py::object& s) {
    if (py::isinstance<cs::Strategy>(s)) return cs::to_mode(s.cast<cs::Strategy>());
    return cs::exec_mode_from_string(s.cast<std::string>());
}

// Python transport: allgather(bytes) -> bytes (rank-ordered concatenation), barrier().
std::unique_ptr<cs::HostTransport> transport_of(const py::object& allgather, const py::object& barrier) {
    if (allgather.is_none()) return nullptr;
    auto t = std::make_unique<cs::HostTransport>();
    t->allgather = [allgather](const void* mine, void* all, std::size_t bytes) {
        py::bytes out = allgather(py::bytes(static_cast<const char*>(mine), bytes));
        const std::string s = out;
        if (s.size() % bytes) throw cs::ValidationError("allgather returned a ragged buffer");
        std::memcpy(all, s.data(), s.size());
    };
    if (!barrier.is_none()) t->barrier = [barrier] { barrier(); };
    return t;
}

void add_exec(py::module_& m) {
    py::class_<cs::World>(m, "World")
        .def(py::init<int, int, int, bool>(), py::arg("rank"), py::arg("n_ranks"), py::arg("device") = 0,
             py::arg("loopback") = false)
        .def_property_readonly("sm_count", [](const cs::World& w) { return w.info().sm_count; })
        .def_property_readonly("rank", [](const cs::World& w) { return w.info().rank; })
        .def_property_readonly("n_ranks", [](const cs::World& w) { return w.info().n_ranks; })
        .def_property_readonly("loopback", [](const cs::World& w) { return w.info().loopback != 0; });
    using R = cs::ExecResult;
    py::class_<R>(m, "ExecResult")
        .RO(R, scenario_id).RO(R, t_gemm).RO(R, t_comm).RO(R, t_comm_dma).RO(R, makespan)
        .RO(R, serial_time).RO(R, speedup).RO(R, ideal).RO(R, fraction_of_ideal).RO(R, taxonomy)
        .RO(R, gemm_ctas).RO(R, comm_ctas).RO(R, partition).RO(R, launches).RO(R, steps)
        .def_property_readonly("strategy", [](const R& r) { return cs::to_string(r.mode); });
    m.def(
        "execute",
        [](const cs::C3Scenario& sc, const py::object& strategy, cs::World& w, int warmup, int reps,
           std::uint64_t seed, const py::object& allgather, const py::object& barrier, double link_gbps,
           std::optional<int> cus_gemm, std::optional<int> cus_comm, std::optional<double> comm_pace_gbps) {
            cs::ExecOptions o;
            o.warmup = warmup;
            o.reps = reps;
            o.seed = seed;
            o.link_gbps = link_gbps;
            auto t = transport_of(allgather, barrier);
            cs::Session s(w, sc, t.get());
            const cs::ExecMode mode = mode_of(strategy);
            if (cus_gemm || cus_comm || comm_pace_gbps) {
                o.use_alloc = true;
                o.alloc = s.default_alloc(mode);
                if (cus_gemm) o.alloc.cus_gemm = *cus_gemm;
                if (cus_comm) o.alloc.cus_comm = *cus_comm;
                if (comm_pace_gbps) o.alloc.comm_pace_gbps = static_cast<float>(*comm_pace_gbps);
            }
            return cs::execute(s, sc, mode, o);
        },
        py::arg("scenario"), py::arg("strategy"), py::arg("world"), py::arg("warmup") = 6,
        py::arg("reps") = 9, py::arg("seed") = 20241217ull, py::arg("allgather") = py::none(),
        py::arg("barrier") = py::none(), py::arg("link_gbps") = 0.0, py::arg("cus_gemm") = py::none(),
        py::arg("cus_comm") = py::none(), py::arg("comm_pace_gbps") = py::none(),
        "Run the scenario on this GPU under a strategy (Strategy or name, incl. 'c3_fused'); "
        "measured seconds and the reference's speedup arithmetic. B200 options: link_gbps "
        "(NVLink-rate emulation of a loopback world), an explicit allocation (cus_gemm, cus_comm: "
        "all SMs + c units = co-resident) and comm_pace_gbps (comm pacing).");
    m.def(
        "measure_isolated",
        [](cs::C3Scenario sc, cs::World& w, int warmup, int reps, const py::object& allgather,
           const py::object& barrier) {
            cs::ExecOptions o;
            o.warmup = warmup;
            o.reps = reps;
            auto t = transport_of(allgather, barrier);
            cs::Session s(w, sc, t.get());
            s.fill(o.seed);
            cs::measure_isolated(s, sc, o);
            return sc;
        },
        py::arg("scenario"), py::arg("world"), py::arg("warmup") = 6, py::arg("reps") = 9,
        py::arg("allgather") = py::none(), py::arg("barrier") = py::none(),
        "Copy of the scenario with gemm.measured_time / collective.measured_time set from B200 runs.");
}

}  // namespace

PYBIND11_MODULE(_c3sim, m) {
    m.doc() = "c3-b200: C3 performance model (drop-in for the reference c3sim) and B200 execution";
    add_errors(m);
    add_enums(m);
    add_machine(m);
    add_workload(m);
    add_taxonomy(m);
    add_interference(m);
    add_strategy(m);
    add_conccl(m);
    add_sim(m);
    add_calibrate(m);
    add_exec(m);
}
