// c3-b200 — C++ execution API: runs a c3sim::C3Scenario on B200 under a
// c3sim::Strategy and returns MEASURED times in the units and with the metric
// arithmetic of the reference model (seconds; speedup / ideal /
// fraction_of_ideal from taxonomy.hpp, /root/reference/proj/src/taxonomy.cpp:9-33).
//
// The reference only predicts (simulate, sim.hpp:70-73); this header is the
// execution counterpart SURVEY §8(b)(2) names:
//     ExecResult execute(const C3Scenario&, Strategy, World&, const ExecOptions&)
// Its isolated times are exactly what GemmKernel::measured_time /
// CollectiveOp::measured_time (workload.hpp:22-23,34) take, so
// `measure_isolated` + simulate() is the B200 calibration loop.
//
// Header-only, over the thin C ABI (include/c3cuda.h, libc3cuda.so): link
// with -lc3cuda -lc3sim. C-ABI status codes are rethrown as the reference's
// error types (errors.hpp: 2 IoError, 3 UnknownEntityError, 4
// ValidationError, 5 FitError); C3_ERR_UNSUPPORTED as UnsupportedError (a
// ValidationError); CUDA / driver failures (100, 101) as DeviceError. No CPU
// fallback: without a B200, World's constructor throws.
//
// Process model: one World per GPU-owning process. A multi-process world needs
// a HostTransport (MPI, torch.distributed, a file ...) to exchange the
// session's IPC handles and to act as the copy-engine strategies' completion
// barrier; a loopback world (n virtual ranks on one GPU) needs none.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "c3cuda.h"
#include "c3sim/errors.hpp"
#include "c3sim/sim.hpp"
#include "c3sim/taxonomy.hpp"
#include "c3sim/workload.hpp"

namespace c3sim {

/// CUDA runtime / driver failure or a non-B200 device (C-ABI status >= 100).
struct DeviceError : Error {
    int status;
    DeviceError(int st, const std::string& what) : Error(what), status(st) {}
};

/// The scenario cannot run in the requested mode on this device (C-ABI status
/// C3_ERR_UNSUPPORTED, e.g. c3_fused on a GEMM too small for the CTA-pair
/// kernel, or a non-B200 device). A ValidationError, so sweeps can skip it.
struct UnsupportedError : ValidationError {
    using ValidationError::ValidationError;
};

/// Execution-only modes next to the seven reference strategies (c3cuda.h).
enum class ExecMode : int {
    Serial = C3_SERIAL, C3Base = C3_C3_BASE, C3Sp = C3_C3_SP, C3Rp = C3_C3_RP,
    C3SpRp = C3_C3_SP_RP, Conccl = C3_CONCCL, ConcclRp = C3_CONCCL_RP,
    Fused = C3_FUSED,  // collective inside the CTA-pair GEMM (B200 extension)
    GemmOnly = C3_GEMM_ONLY, CommOnlyCu = C3_COMM_ONLY_CU, CommOnlyDma = C3_COMM_ONLY_DMA,
};

inline ExecMode to_mode(Strategy s) { return static_cast<ExecMode>(static_cast<int>(s)); }

inline std::string to_string(ExecMode m) {
    if (static_cast<int>(m) <= C3_CONCCL_RP) return to_string(static_cast<Strategy>(static_cast<int>(m)));
    switch (m) {
        case ExecMode::Fused: return "c3_fused";
        case ExecMode::GemmOnly: return "gemm_only";
        case ExecMode::CommOnlyCu: return "comm_only_cu";
        case ExecMode::CommOnlyDma: return "comm_only_dma";
        default: return "mode_" + std::to_string(static_cast<int>(m));
    }
}

inline ExecMode exec_mode_from_string(const std::string& s) {
    if (s == "c3_fused") return ExecMode::Fused;
    if (s == "gemm_only") return ExecMode::GemmOnly;
    if (s == "comm_only_cu") return ExecMode::CommOnlyCu;
    if (s == "comm_only_dma") return ExecMode::CommOnlyDma;
    return to_mode(strategy_from_string(s));  // throws UnknownEntityError
}

/// Throw the reference error type matching a C-ABI status.
inline void check_status(int rc, const char* what) {
    if (rc == C3_OK) return;
    const char* detail = c3_last_error();
    const std::string msg = std::string(what) + ": " + (detail ? detail : "");
    switch (rc) {
        case C3_ERR_IO: throw IoError(msg);
        case C3_ERR_UNKNOWN: throw UnknownEntityError(msg);
        case C3_ERR_VALIDATION: throw ValidationError(msg);
        case C3_ERR_FIT: throw FitError(msg);
        case C3_ERR_UNSUPPORTED: throw UnsupportedError(msg);
        default: throw DeviceError(rc, msg);
    }
}

/// Host-side exchange between the ranks of a multi-process world.
struct HostTransport {
    /// all[r*bytes .. (r+1)*bytes) <- rank r's `mine`, for every rank r.
    std::function<void(const void* mine, void* all, std::size_t bytes)> allgather;
    /// Cross-rank barrier (completion of the copy-engine collectives).
    std::function<void()> barrier;
};

/// One rank's view of the node: device, streams, green contexts, peer access.
class World {
public:
    World(int rank, int n_ranks, int device, bool loopback) {
        check_status(c3_world_create(rank, n_ranks, device, loopback ? 1 : 0, &w_), "c3_world_create");
    }
    World(const World&) = delete;
    World& operator=(const World&) = delete;
    World(World&& o) noexcept : w_(std::exchange(o.w_, nullptr)) {}
    ~World() {
        if (w_) c3_world_destroy(w_);
    }
    c3_world* get() const { return w_; }
    c3_world_info info() const {
        c3_world_info i{};
        check_status(c3_world_get_info(w_, &i), "c3_world_get_info");
        return i;
    }

private:
    c3_world* w_ = nullptr;
};

/// One scenario's operands on this rank, peer-mapped, ready to run.
class Session {
public:
    Session(World& w, const C3Scenario& sc, const HostTransport* transport = nullptr) {
        if (sc.gemm.dtype_bytes != 2 && sc.gemm.dtype_bytes != 4)
            throw ValidationError("execute: the B200 GEMM is bf16 (dtype_bytes 2) or fp32 on the TF32 tensor "
                                  "cores (4), scenario '" + sc.id + "' has dtype_bytes " +
                                  std::to_string(sc.gemm.dtype_bytes));
        const c3_world_info wi = w.info();
        if (sc.collective.n_ranks != wi.n_ranks)
            throw ValidationError("execute: scenario '" + sc.id + "' has n_ranks " +
                                  std::to_string(sc.collective.n_ranks) + ", the world " +
                                  std::to_string(wi.n_ranks));
        if (!wi.loopback && wi.n_ranks > 1 && (!transport || !transport->allgather))
            throw ValidationError("execute: a multi-process world needs a HostTransport");
        const c3_scenario_desc d{sc.gemm.m, sc.gemm.n, sc.gemm.k,
                                 static_cast<int32_t>(sc.collective.kind), sc.collective.n_ranks,
                                 sc.collective.payload_bytes, static_cast<int32_t>(sc.gemm.dtype_bytes)};
        check_status(c3_session_create(w.get(), &d, &s_), "c3_session_create");
        n_ranks_ = wi.n_ranks;
        if (!wi.loopback && wi.n_ranks > 1) {
            transport_ = std::make_unique<HostTransport>(*transport);
            std::vector<unsigned char> mine(C3_SESSION_HANDLE_BYTES),
                all(static_cast<std::size_t>(C3_SESSION_HANDLE_BYTES) * wi.n_ranks);
            check_status(c3_session_export(s_, mine.data()), "c3_session_export");
            transport_->allgather(mine.data(), all.data(), mine.size());
            check_status(c3_session_import(s_, all.data()), "c3_session_import");
            if (transport_->barrier)
                check_status(c3_session_set_barrier(s_, &Session::barrier_tramp, transport_.get()),
                             "c3_session_set_barrier");
        }
    }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    ~Session() {
        if (s_) c3_session_destroy(s_);
    }

    c3_session* get() const { return s_; }
    const HostTransport* transport() const { return transport_.get(); }
    int n_ranks() const { return n_ranks_; }

    void fill(std::uint64_t seed) { check_status(c3_session_fill(s_, seed), "c3_session_fill"); }

    c3_alloc default_alloc(ExecMode m) const {
        c3_alloc a{};
        check_status(c3_session_default_alloc(s_, static_cast<int>(m), &a), "c3_session_default_alloc");
        return a;
    }

    /// One device-timed step (this rank's share of the collective).
    c3_timing run(ExecMode m, const c3_alloc* alloc = nullptr) {
        c3_timing t{};
        check_status(c3_session_run(s_, static_cast<int>(m), alloc, &t), "c3_session_run");
        return t;
    }

    /// One step on host buffers (c3_session_run_host): A and this rank's
    /// collective input copied in, the first out_bytes of C copied back.
    c3_timing run_host(ExecMode m, const c3_alloc* alloc, const void* host_a, const void* host_send,
                       void* host_out, std::int64_t out_bytes) {
        c3_timing t{};
        check_status(c3_session_run_host(s_, static_cast<int>(m), alloc, host_a, host_send, host_out,
                                         out_bytes, &t),
                     "c3_session_run_host");
        return t;
    }

    /// Link-rate emulation for loopback worlds (c3_session_set_link_rate); 0 = off.
    void set_link_rate(double gbps) {
        check_status(c3_session_set_link_rate(s_, gbps), "c3_session_set_link_rate");
    }

    /// The runtime heuristic's inputs: measured interference tables, co-run
    /// penalties (optional) and the B200 co-residency parameters (optional).
    void load_model(const std::string& tables_csv, const std::string& params_json = {},
                    const std::string& coresident_json = {}) {
        check_status(c3_session_load_tables(s_, tables_csv.c_str()), "c3_session_load_tables");
        if (!params_json.empty())
            check_status(c3_session_load_params(s_, params_json.c_str()), "c3_session_load_params");
        if (!coresident_json.empty())
            check_status(c3_session_load_coresident(s_, coresident_json.c_str()), "c3_session_load_coresident");
    }

    /// The collective's measured time (seconds) vs CTA units (co-residency model).
    void set_comm_curve(const std::vector<std::pair<int, double>>& pts) {
        std::vector<int> c;
        std::vector<double> ms;
        for (const auto& [ctas, sec] : pts) {
            c.push_back(ctas);
            ms.push_back(sec * 1e3);
        }
        check_status(c3_session_set_comm_curve(s_, c.data(), ms.data(), static_cast<int>(c.size())),
                     "c3_session_set_comm_curve");
    }

    /// c3_session_choose on measured isolated times (seconds): the mode and
    /// allocation the runtime heuristic picks, and its predicted makespan.
    std::pair<ExecMode, c3_alloc> choose(double t_gemm, double t_comm, double t_comm_dma, bool allow_dma,
                                         double* predicted = nullptr) {
        int st = 0;
        c3_alloc a{};
        double pred_ms = 0;
        check_status(c3_session_choose(s_, t_gemm * 1e3, t_comm * 1e3, t_comm_dma * 1e3, allow_dma ? 1 : 0,
                                       &st, &a, &pred_ms),
                     "c3_session_choose");
        if (predicted) *predicted = pred_ms * 1e-3;
        return {static_cast<ExecMode>(st), a};
    }

private:
    static int barrier_tramp(void* ctx) {
        try {
            static_cast<HostTransport*>(ctx)->barrier();
            return 0;
        } catch (...) {
            return 1;
        }
    }
    c3_session* s_ = nullptr;
    int n_ranks_ = 1;
    std::unique_ptr<HostTransport> transport_;
};

struct ExecOptions {
    int warmup = 6;   // the paper's protocol: 6 warm-up + 9 measured, median
    int reps = 9;
    std::uint64_t seed = 20241217;
    bool fill = true;
    /// Override the strategy's own allocation (allocate_cus semantics).
    bool use_alloc = false;
    c3_alloc alloc{};
    /// Link-rate emulation of the (loopback) collective, GB/s per direction; 0 = off.
    double link_gbps = 0.0;
};

struct ExecResult {
    std::string scenario_id;
    ExecMode mode = ExecMode::Serial;
    c3_alloc alloc{};
    double t_gemm = 0;     // isolated GEMM, whole GPU, median seconds
    double t_comm = 0;     // isolated SM collective, whole GPU, median seconds
    double t_comm_dma = 0; // isolated copy-engine collective (DMA modes only)
    double makespan = 0;   // the strategy's step, median seconds
    double serial_time = 0, speedup = 0, ideal = 0, fraction_of_ideal = 0;
    TaxonomyClass taxonomy = TaxonomyClass::GCEqual;
    int gemm_ctas = 0, comm_ctas = 0, partition = 0, launches = 0;
    std::vector<double> steps;  // per-rep makespans (max over ranks), seconds
};

namespace detail {

inline double median(std::vector<double> v) {
    if (v.empty()) return 0;
    std::sort(v.begin(), v.end());
    const std::size_t h = v.size() / 2;
    return v.size() % 2 ? v[h] : 0.5 * (v[h - 1] + v[h]);
}

/// Elementwise max over ranks (identity without a transport).
inline std::vector<double> max_over_ranks(const Session& s, std::vector<double> v) {
    const HostTransport* t = s.transport();
    if (!t || s.n_ranks() <= 1 || v.empty()) return v;
    std::vector<double> all(v.size() * static_cast<std::size_t>(s.n_ranks()));
    t->allgather(v.data(), all.data(), v.size() * sizeof(double));
    for (int r = 0; r < s.n_ranks(); ++r)
        for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::max(v[i], all[r * v.size() + i]);
    return v;
}

}  // namespace detail

/// Isolated GEMM / SM collective / copy-engine collective times (seconds,
/// median over `reps` after `warmup`, max over ranks), interleaved so the
/// three see the same thermal and power state. Writes them into the
/// scenario's measured_time fields — the reference model then predicts with
/// B200 numbers (roofline_gemm_time honours measured_time, workload.cpp:74).
inline void measure_isolated(Session& s, C3Scenario& sc, const ExecOptions& o = {},
                             double* t_comm_dma = nullptr) {
    const int C = s.default_alloc(ExecMode::GemmOnly).cus_gemm;
    c3_alloc comm = s.default_alloc(ExecMode::CommOnlyCu);
    comm.cus_comm = C;
    std::vector<double> g, c, d;
    for (int r = 0; r < o.warmup + o.reps; ++r) {
        const c3_timing tg = s.run(ExecMode::GemmOnly);
        const c3_timing tc = s.run(ExecMode::CommOnlyCu, &comm);
        c3_timing td{};
        if (t_comm_dma) td = s.run(ExecMode::CommOnlyDma);
        if (r < o.warmup) continue;
        g.push_back((tg.gemm_end_ms - tg.gemm_start_ms) * 1e-3);
        c.push_back((tc.comm_end_ms - tc.comm_start_ms) * 1e-3);
        if (t_comm_dma) d.push_back((td.comm_end_ms - td.comm_start_ms) * 1e-3);
    }
    sc.gemm.measured_time = detail::median(detail::max_over_ranks(s, g));
    sc.collective.measured_time = detail::median(detail::max_over_ranks(s, c));
    if (t_comm_dma) *t_comm_dma = detail::median(detail::max_over_ranks(s, d));
}

/// Execute one scenario under one mode on an existing session: isolated
/// kernels and the concurrent step in rotating round-robin order, medians, the
/// reference's metric arithmetic (serial = t_gemm + t_comm on the CU backend,
/// sim.cpp:143; ideal and fraction from taxonomy.hpp).
inline ExecResult execute(Session& s, const C3Scenario& sc, ExecMode mode, const ExecOptions& o = {}) {
    if (o.reps < 1 || o.warmup < 0) throw ValidationError("execute: reps >= 1 and warmup >= 0 required");
    if (o.fill) s.fill(o.seed);
    s.set_link_rate(o.link_gbps);
    ExecResult res;
    res.scenario_id = sc.id;
    res.mode = mode;
    res.alloc = o.use_alloc ? o.alloc : s.default_alloc(mode);
    const bool dma = mode == ExecMode::Conccl || mode == ExecMode::ConcclRp;
    const int C = s.default_alloc(ExecMode::GemmOnly).cus_gemm;
    c3_alloc comm = s.default_alloc(ExecMode::CommOnlyCu);
    comm.cus_comm = C;

    // jobs: 0 GEMM alone, 1 SM collective alone, 2 copy-engine collective alone, 3 the step
    std::vector<int> jobs = {0, 1, 3};
    if (dma) jobs.insert(jobs.begin() + 2, 2);
    std::vector<double> g, c, d, m;
    c3_timing last{};
    for (int r = 0; r < o.warmup + o.reps; ++r) {
        const std::size_t rot = static_cast<std::size_t>(r) % jobs.size();
        for (std::size_t j = 0; j < jobs.size(); ++j) {
            const int job = jobs[(j + rot) % jobs.size()];
            c3_timing t{};
            if (job == 0) t = s.run(ExecMode::GemmOnly);
            if (job == 1) t = s.run(ExecMode::CommOnlyCu, &comm);
            if (job == 2) t = s.run(ExecMode::CommOnlyDma);
            if (job == 3) t = last = s.run(mode, &res.alloc);
            if (r < o.warmup) continue;
            if (job == 0) g.push_back((t.gemm_end_ms - t.gemm_start_ms) * 1e-3);
            if (job == 1) c.push_back((t.comm_end_ms - t.comm_start_ms) * 1e-3);
            if (job == 2) d.push_back((t.comm_end_ms - t.comm_start_ms) * 1e-3);
            if (job == 3) m.push_back(t.total_ms * 1e-3);
        }
    }
    res.t_gemm = detail::median(detail::max_over_ranks(s, g));
    res.t_comm = detail::median(detail::max_over_ranks(s, c));
    if (dma) res.t_comm_dma = detail::median(detail::max_over_ranks(s, d));
    res.steps = detail::max_over_ranks(s, m);
    res.makespan = detail::median(res.steps);
    res.serial_time = res.t_gemm + res.t_comm;
    res.speedup = res.serial_time / res.makespan;
    res.ideal = ideal_speedup(res.t_gemm, res.t_comm);
    res.fraction_of_ideal = fraction_of_ideal(res.speedup, res.ideal);
    res.taxonomy = classify_c3(res.t_gemm, res.t_comm).value;
    res.gemm_ctas = last.gemm_ctas;
    res.comm_ctas = last.comm_ctas;
    res.partition = last.partition;
    res.launches = last.launches;
    return res;
}

/// The SURVEY §8(b) form: one scenario, one reference strategy, a fresh session.
inline ExecResult execute(const C3Scenario& sc, Strategy strategy, World& w, const ExecOptions& o = {},
                          const HostTransport* transport = nullptr) {
    Session s(w, sc, transport);
    return execute(s, sc, to_mode(strategy), o);
}

}  // namespace c3sim
