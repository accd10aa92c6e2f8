// c3sim — product CLI over libc3sim (the model layer). Same subcommands, flags,
// report formats and exit codes as the reference front-end
// (/root/reference/proj/tools/c3sim_main.cpp:28-417): classify, plan,
// conccl-plan, sweep, calibrate; exit 0 ok, 2 I/O, 3 unknown entity,
// 4 validation, 5 fit. Argument parsing is self-contained (no CLI11).
// Reports are written atomically (temp file + rename).
//
// New subcommand `run` EXECUTES scenarios on the local B200 through the C++
// execution API (include/c3sim/exec.hpp -> libc3cuda.so): measured isolated
// times, the strategy's measured makespan, speedup / ideal / fraction of
// ideal, and — given --machine and --tables — the model's prediction from the
// same measured isolated times next to it. Single process, so the n ranks of
// the scenario run as a loopback world on one GPU. Exit 6 = device error
// (CUDA / driver / no B200).
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "c3sim/calibrate.hpp"
#include "c3sim/conccl.hpp"
#include "c3sim/errors.hpp"
#include "c3sim/exec.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/params_io.hpp"
#include "c3sim/sim.hpp"
#include "c3sim/strategy.hpp"
#include "json.hpp"

using namespace c3sim;
using nlohmann::json;

namespace {

std::string g12(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.12g", v);
    return b;
}

void write_report(const std::optional<std::string>& path, const std::string& text) {
    if (!path) {
        std::cout << text;
        return;
    }
    const std::string tmp = *path + ".tmp";
    {
        std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
        if (!f) throw IoError("cannot write file: " + *path);
        f << text;
        if (!f.good()) throw IoError("write failed: " + *path);
    }
    std::filesystem::rename(tmp, *path);
}

struct Args {
    std::string cmd;
    std::map<std::string, std::string> opt;  // --name -> value
    bool zero = false;

    bool has(const std::string& k) const { return opt.count(k) > 0; }
    std::string get(const std::string& k, const std::string& dflt = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? dflt : it->second;
    }
    std::string need(const std::string& k) const {
        if (!has(k)) throw std::invalid_argument("missing required option --" + k);
        return opt.at(k);
    }
    std::optional<std::string> out() const {
        return has("out") ? std::optional<std::string>(opt.at("out")) : std::nullopt;
    }
};

struct Inputs {
    MachineDescriptor md;
    std::vector<C3Scenario> scenarios;
    SlowdownTableSet tables;
    RunParams params;
};

Inputs load_inputs(const Args& a, bool dataset, bool tables) {
    Inputs in;
    in.md = load_machine_file(a.need("machine"));
    if (dataset) in.scenarios = load_dataset(a.need("dataset"));
    if (a.has("params")) in.params = load_params_file(a.get("params"));
    if (tables) {
        if (!a.has("tables")) throw IoError("--tables is required");
        in.tables = load_slowdown_tables(a.get("tables"), in.md.min_cu_grain);
    } else {
        for (int i = 0; i < kNumKernelClasses; ++i)
            in.tables.tables[static_cast<std::size_t>(i)] = {static_cast<KernelClass>(i), {{in.md.cus_per_gpu, 1.0}}};
    }
    if (a.zero) apply_zero_interference(in.tables, in.params.penalties, in.params.eff, in.md);
    return in;
}

TaxonomyClass label_of(const C3Scenario& s, const Inputs& in) {
    if (s.expected_taxonomy) return *s.expected_taxonomy;
    return classify_c3(roofline_gemm_time(s.gemm, in.md, in.params.eff),
                       roofline_collective_time(s.collective, in.md, in.params.eff, true))
        .value;
}

std::vector<C3Scenario> filtered(const Args& a, const Inputs& in) {
    std::optional<CollectiveKind> kind;
    std::optional<TaxonomyClass> tax;
    if (!a.get("filter-collective").empty()) kind = collective_kind_from_string(a.get("filter-collective"));
    if (!a.get("filter-taxonomy").empty()) tax = taxonomy_from_string(a.get("filter-taxonomy"));
    std::vector<C3Scenario> out;
    for (const auto& s : in.scenarios)
        if ((!kind || s.collective.kind == *kind) && (!tax || label_of(s, in) == *tax)) out.push_back(s);
    return out;
}

void check_format(const std::string& f) {
    if (f != "csv" && f != "structured-text")
        throw ValidationError("--format must be csv or structured-text, got '" + f + "'");
}

int classify_cmd(const Args& a) {
    const std::string format = a.get("format", "csv");
    check_format(format);
    const Inputs in = load_inputs(a, true, false);
    const double ratio = machine_op_to_byte(in.md);
    std::ostringstream csv;
    csv << "scenario_id,collective,gemm_tag,gemm_boundedness,collective_boundedness,"
           "t_gemm_s,t_comm_s,taxonomy,ideal_speedup,expected_taxonomy,match\n";
    json rows = json::array();
    int bad = 0;
    const auto list = filtered(a, in);
    for (const auto& s : list) {
        const double tg = roofline_gemm_time(s.gemm, in.md, in.params.eff);
        const double tc = roofline_collective_time(s.collective, in.md, in.params.eff, true);
        const auto lab = classify_c3(tg, tc).value;
        const auto gb = classify_gemm_boundedness(s.gemm, ratio);
        const auto cb = classify_collective_boundedness(s.collective, in.md, in.params.eff);
        const double ideal = ideal_speedup(tg, tc);
        const std::string exp = s.expected_taxonomy ? to_string(*s.expected_taxonomy) : "";
        const bool match = !s.expected_taxonomy || *s.expected_taxonomy == lab;
        bad += !match;
        csv << s.id << ',' << to_string(s.collective.kind) << ',' << s.gemm.tag << ','
            << to_string(gb) << ',' << to_string(cb) << ',' << g12(tg) << ',' << g12(tc) << ','
            << to_string(lab) << ',' << g12(ideal) << ',' << exp << ',' << (match ? "yes" : "NO") << '\n';
        rows.push_back({{"scenario_id", s.id}, {"collective", to_string(s.collective.kind)},
                        {"gemm_tag", s.gemm.tag}, {"gemm_boundedness", to_string(gb)},
                        {"collective_boundedness", to_string(cb)}, {"t_gemm_s", tg},
                        {"t_comm_s", tc}, {"taxonomy", to_string(lab)}, {"ideal_speedup", ideal},
                        {"expected_taxonomy", exp}, {"match", match}});
    }
    write_report(a.out(), format == "csv" ? csv.str() : rows.dump(2) + "\n");
    std::cerr << list.size() << " scenarios classified, " << bad << " taxonomy mismatches\n";
    return 0;
}

TransferPlan plan_for(CollectiveKind kind, int n, std::int64_t chunk, const MachineDescriptor& md) {
    switch (kind) {
        case CollectiveKind::AllGather: return plan_all_gather(n, chunk, md);
        case CollectiveKind::AllToAll: return plan_all_to_all(n, chunk, md);
        case CollectiveKind::ReduceScatter: return plan_reduce_scatter(n, chunk, md);
    }
    throw ValidationError("unknown collective kind");
}

int plan_cmd(const Args& a) {
    const Inputs in = load_inputs(a, true, true);
    const Strategy st = strategy_from_string(a.need("strategy"));
    const std::string id = a.need("scenario");
    std::optional<CollectiveKind> kind;
    if (!a.get("filter-collective").empty()) kind = collective_kind_from_string(a.get("filter-collective"));
    const C3Scenario* s = nullptr;  // prefer the all-gather instance of the id
    for (const auto& x : in.scenarios)
        if (x.id == id && (!kind || x.collective.kind == *kind) &&
            (!s || x.collective.kind == CollectiveKind::AllGather))
            s = &x;
    if (!s) throw UnknownEntityError("unknown scenario id '" + id + "'");

    PartitionPlan plan;
    std::ostringstream audit;
    if (st == Strategy::Conccl || st == Strategy::ConcclRp) {
        plan = conccl_rp_plan(*s, in.md, in.tables);
        if (st == Strategy::Conccl) {
            plan.cus_gemm = in.md.cus_per_gpu;
            plan.cus_idle = 0;
        }
        const auto& c = s->collective;
        const TransferPlan xfer =
            plan_for(c.kind, c.n_ranks, std::max<std::int64_t>(c.payload_bytes / c.n_ranks, 1), in.md);
        const auto& gt = in.tables.at(gemm_kernel_class(s->gemm, machine_op_to_byte(in.md)));
        plan.predicted_makespan =
            std::max(roofline_gemm_time(s->gemm, in.md, in.params.eff) * slowdown_at(gt, plan.cus_gemm),
                     plan_cost(xfer, in.md, in.params.eff).total);
    } else if (st == Strategy::C3Rp || st == Strategy::C3SpRp) {
        const PartitionSweep ps = partition_heuristic(*s, in.md, in.tables, in.params.eff);
        plan = ps.plan;
        audit << "cus_comm,gemm_term_s,comm_term_s,predicted_s\n";
        for (const auto& c : ps.candidates)
            audit << c.cus_comm << ',' << g12(c.gemm_term) << ',' << g12(c.comm_term) << ','
                  << g12(c.predicted) << '\n';
    } else {
        throw UnknownEntityError("cmd plan supports c3_rp, c3_sp_rp, conccl and conccl_rp");
    }
    std::cout << "scenario " << s->id << " (" << to_string(s->collective.kind) << "), strategy "
              << to_string(st) << "\n"
              << to_json(plan);
    if (audit.tellp() > 0) std::cout << "candidate sweep:\n" << audit.str();
    if (a.out()) write_report(a.out(), to_json(plan));
    return 0;
}

int conccl_plan_cmd(const Args& a) {
    const Inputs in = load_inputs(a, false, false);
    const CollectiveKind kind = collective_kind_from_string(a.need("kind"));
    const int n = std::stoi(a.need("ranks"));
    const std::int64_t payload = std::stoll(a.need("payload-bytes"));
    if (n < 1) throw ValidationError("--ranks must be >= 1");
    if (payload < 0) throw ValidationError("--payload-bytes must be >= 0");
    if (n > 1 && payload % n) throw ValidationError("--payload-bytes must be divisible by --ranks");
    std::int64_t chunk = payload / n;
    if (n == 1 && chunk == 0) chunk = 1;
    const TransferPlan plan = plan_for(kind, n, chunk, in.md);
    const PlanCheck ok = validate_plan(plan, in.md);
    if (a.out()) write_report(a.out(), to_json(plan));
    const PlanCost cost = plan_cost(plan, in.md, in.params.eff);
    std::cout << to_string(kind) << " plan: " << plan.transfers.size() << " transfers, " << n
              << " ranks, chunk " << plan.chunk_bytes << " B\n"
              << "cost: total " << g12(cost.total) << " s, wire " << g12(cost.wire) << " s (launch "
              << g12(in.md.cpu_launch_overhead) << " s/transfer, sync "
              << g12(in.md.dma_sync_overhead) << " s)\n"
              << "validation: " << (ok.ok ? "ok" : "FAILED: " + ok.error) << "\n";
    return ok.ok ? 0 : 4;
}

int sweep_cmd(const Args& a) {
    const std::string format = a.get("format", "csv");
    check_format(format);
    const Inputs in = load_inputs(a, true, true);
    const auto list = filtered(a, in);
    std::vector<Strategy> sts;
    const std::string name = a.get("strategy", "all");
    if (name.empty() || name == "all")
        sts.assign(std::begin(kAllStrategies), std::end(kAllStrategies));
    else
        sts.push_back(strategy_from_string(name));
    SimOptions opt;
    opt.freeze_phase2_allocation = in.params.freeze_phase2_allocation;
    const SweepResult r = sweep(list, sts, in.md, in.tables, in.params.penalties, in.params.eff, opt);
    if (format == "csv") {
        write_report(a.out(), sweep_to_csv(r));
        return 0;
    }
    json rows = json::array(), aggs = json::array();
    for (const auto& x : r.rows)
        rows.push_back({{"scenario_id", x.scenario_id}, {"collective", to_string(x.collective)},
                        {"taxonomy", to_string(x.taxonomy)}, {"strategy", to_string(x.strategy)},
                        {"makespan_s", x.makespan}, {"speedup", x.speedup}, {"ideal", x.ideal},
                        {"fraction_of_ideal", x.fraction_of_ideal}});
    for (const auto& g : r.aggregates)
        aggs.push_back({{"collective", g.collective ? to_string(*g.collective) : "all"},
                        {"taxonomy", g.taxonomy ? to_string(*g.taxonomy) : "all"},
                        {"strategy", to_string(g.strategy)}, {"count", g.count},
                        {"mean_speedup", g.mean_speedup}, {"mean_ideal", g.mean_ideal},
                        {"mean_fraction_of_ideal", g.mean_fraction_of_ideal}});
    write_report(a.out(), json({{"rows", rows}, {"aggregates", aggs}}).dump(2) + "\n");
    return 0;
}

int calibrate_cmd(const Args& a) {
    const Inputs in = load_inputs(a, true, true);
    const auto samples = load_measured_csv(a.need("measured"));
    const FitResult fit = fit_penalties(in.scenarios, samples, in.md, in.tables, in.params.eff,
                                        in.params.penalties);
    RunParams out = in.params;
    out.penalties = fit.penalties;
    const std::string text = save_params(out);
    if (a.out()) write_report(a.out(), text);
    std::cout << text;
    std::cerr << "fit: rms residual " << g12(fit.rms_residual) << " over " << samples.size()
              << " samples, " << fit.iterations << " iterations\n";
    return 0;
}

C3Scenario run_scenario(const Args& a) {
    if (a.has("scenario")) {
        const auto all = load_dataset(a.need("dataset"));
        std::optional<CollectiveKind> kind;
        if (!a.get("filter-collective").empty()) kind = collective_kind_from_string(a.get("filter-collective"));
        for (const auto& x : all)
            if (x.id == a.get("scenario") && (!kind || x.collective.kind == *kind)) return x;
        throw UnknownEntityError("unknown scenario id '" + a.get("scenario") + "'");
    }
    C3Scenario sc;
    sc.id = a.get("id", "custom");
    sc.gemm.tag = "gemm";
    sc.gemm.m = std::stoll(a.need("m"));
    sc.gemm.n = std::stoll(a.need("n"));
    sc.gemm.k = std::stoll(a.need("k"));
    sc.collective.kind = collective_kind_from_string(a.get("kind", "all-gather"));
    sc.collective.n_ranks = std::stoi(a.need("ranks"));
    sc.collective.payload_bytes = std::stoll(a.need("payload-bytes"));
    validate(sc.gemm);
    validate(sc.collective);
    return sc;
}

int run_cmd(const Args& a) {
    const std::string format = a.get("format", "csv");
    check_format(format);
    C3Scenario sc = run_scenario(a);
    std::vector<ExecMode> modes;
    const std::string name = a.get("strategy", "all");
    const bool autopick = name == "auto";
    if (name == "all") {
        for (Strategy s : kAllStrategies) modes.push_back(to_mode(s));
        modes.push_back(ExecMode::Fused);
    } else if (!autopick) {
        modes.push_back(exec_mode_from_string(name));
    }
    ExecOptions o;
    o.warmup = std::stoi(a.get("warmup", "6"));
    o.reps = std::stoi(a.get("reps", "9"));
    o.seed = std::stoull(a.get("seed", "20241217"));
    o.link_gbps = std::stod(a.get("link-gbps", "0"));
    // explicit allocation (B200: --cus-gemm all SMs + --cus-comm c = co-resident)
    const bool explicit_alloc = a.has("cus-gemm") || a.has("cus-comm") || a.has("comm-pace-gbps");

    // optional model side: predict every strategy from the measured isolated times
    std::optional<Inputs> model;
    if (a.has("machine") && a.has("tables")) model = load_inputs(a, false, true);

    World world(0, sc.collective.n_ranks, std::stoi(a.get("device", "0")), /*loopback=*/true);
    Session session(world, sc);
    std::optional<c3_alloc> picked;
    if (autopick) {
        // the runtime heuristic: measured isolated times and comm curve ->
        // c3_session_choose (reference model + B200 co-residency) -> execute
        if (!a.has("tables")) throw ValidationError("run --strategy auto needs --tables");
        session.load_model(a.get("tables"), a.get("params", ""), a.get("coresident", ""));
        session.fill(o.seed);
        session.set_link_rate(o.link_gbps);
        C3Scenario msc = sc;
        ExecOptions mo = o;
        measure_isolated(session, msc, mo);
        std::vector<std::pair<int, double>> curve;
        for (int c : {8, 16, 24, 32, 48, 64}) {
            c3_alloc ca = session.default_alloc(ExecMode::CommOnlyCu);
            ca.cus_comm = c;
            std::vector<double> ts;
            for (int r = 0; r < 3 + o.warmup; ++r) {
                const c3_timing t = session.run(ExecMode::CommOnlyCu, &ca);
                if (r >= o.warmup) ts.push_back((t.comm_end_ms - t.comm_start_ms) * 1e-3);
            }
            curve.emplace_back(c, detail::median(ts));
        }
        const int C = session.default_alloc(ExecMode::GemmOnly).cus_gemm;
        const double tg = msc.gemm.measured_time.value(), tc = msc.collective.measured_time.value();
        curve.emplace_back(C, std::min(tc, curve.back().second));
        session.set_comm_curve(curve);
        const auto [mode, alloc] = session.choose(tg, tc, 0.0, /*allow_dma=*/false);
        std::cerr << "auto: picked " << to_string(mode) << " cus_gemm " << alloc.cus_gemm << " cus_comm "
                  << alloc.cus_comm << " pace " << alloc.comm_pace_gbps << " GB/s\n";
        modes.push_back(mode);
        picked = alloc;
        o.fill = false;
    }
    std::ostringstream csv;
    csv << "scenario_id,collective,strategy,cus_gemm,cus_comm,backend,t_gemm_s,t_comm_s,t_comm_dma_s,"
           "makespan_s,speedup,ideal,fraction_of_ideal,taxonomy,predicted_makespan_s,predicted_speedup,"
           "comm_pace_gbps\n";
    json rows = json::array();
    for (ExecMode m : modes) {
        ExecResult r;
        try {
            if (picked) {
                o.use_alloc = true;
                o.alloc = *picked;
            } else if (explicit_alloc) {
                o.use_alloc = true;
                o.alloc = session.default_alloc(m);
                if (a.has("cus-gemm")) o.alloc.cus_gemm = std::stoi(a.get("cus-gemm"));
                if (a.has("cus-comm")) o.alloc.cus_comm = std::stoi(a.get("cus-comm"));
                if (a.has("comm-pace-gbps")) o.alloc.comm_pace_gbps = std::stof(a.get("comm-pace-gbps"));
            }
            r = execute(session, sc, m, o);
            o.fill = false;  // operands stay resident across strategies
        } catch (const ValidationError& e) {  // e.g. c3_fused on a shape without the pair GEMM
            std::cerr << "skip " << to_string(m) << ": " << e.what() << "\n";
            continue;
        }
        std::string pred_ms, pred_sp;
        double pm = 0;
        if (model && static_cast<int>(m) <= C3_CONCCL_RP) {
            C3Scenario msc = sc;
            msc.gemm.measured_time = r.t_gemm;
            msc.collective.measured_time = r.t_comm;
            SimOptions so;
            so.freeze_phase2_allocation = model->params.freeze_phase2_allocation;
            const SimTimeline tl = simulate(msc, static_cast<Strategy>(static_cast<int>(m)), model->md,
                                            model->tables, model->params.penalties, model->params.eff, so);
            pm = tl.makespan;
            pred_ms = g12(tl.makespan);
            pred_sp = g12(tl.speedup);
        }
        const char* backend = r.alloc.backend == C3_BACKEND_DMA ? "dma"
                              : r.alloc.backend == C3_BACKEND_TMA ? "tma" : "cu";
        csv << sc.id << ',' << to_string(sc.collective.kind) << ',' << to_string(m) << ','
            << r.gemm_ctas << ',' << r.comm_ctas << ',' << backend << ',' << g12(r.t_gemm) << ','
            << g12(r.t_comm) << ',' << g12(r.t_comm_dma) << ',' << g12(r.makespan) << ','
            << g12(r.speedup) << ',' << g12(r.ideal) << ',' << g12(r.fraction_of_ideal) << ','
            << to_string(r.taxonomy) << ',' << pred_ms << ',' << pred_sp << ',' << g12(r.alloc.comm_pace_gbps)
            << '\n';
        json row = {{"scenario_id", sc.id}, {"collective", to_string(sc.collective.kind)},
                    {"strategy", to_string(m)}, {"cus_gemm", r.gemm_ctas}, {"cus_comm", r.comm_ctas},
                    {"backend", backend}, {"t_gemm_s", r.t_gemm}, {"t_comm_s", r.t_comm},
                    {"t_comm_dma_s", r.t_comm_dma}, {"makespan_s", r.makespan}, {"speedup", r.speedup},
                    {"ideal", r.ideal}, {"fraction_of_ideal", r.fraction_of_ideal},
                    {"taxonomy", to_string(r.taxonomy)}, {"steps_s", r.steps},
                    {"comm_pace_gbps", r.alloc.comm_pace_gbps}};
        if (!pred_ms.empty()) row["predicted_makespan_s"] = pm;
        rows.push_back(row);
    }
    if (rows.empty()) throw ValidationError("run: no strategy could execute this scenario");
    write_report(a.out(), format == "csv" ? csv.str() : rows.dump(2) + "\n");
    return 0;
}

void usage() {
    std::cerr << "usage: c3sim {classify|plan|conccl-plan|sweep|calibrate} --machine FILE "
                 "[--dataset FILE] [--tables FILE] [--params FILE] [--out FILE] "
                 "[--zero-interference] [subcommand options]\n"
                 "       c3sim run {--dataset FILE --scenario ID | --m M --n N --k K --ranks R "
                 "--payload-bytes P [--kind all-gather|all-to-all|reduce-scatter]} "
                 "[--strategy NAME|all|auto] [--cus-gemm N] [--cus-comm N] [--comm-pace-gbps X] "
                 "[--link-gbps X] [--coresident FILE] [--warmup W] [--reps K] [--device D] "
                 "[--machine FILE --tables FILE [--params FILE]] [--format csv|structured-text] "
                 "[--out FILE]\n";
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    if (argc < 2) {
        usage();
        return 2;
    }
    a.cmd = argv[1];
    try {
        for (int i = 2; i < argc; ++i) {
            std::string k = argv[i];
            if (k.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument '" + k + "'");
            k = k.substr(2);
            if (k == "zero-interference") {
                a.zero = true;
                continue;
            }
            const auto eq = k.find('=');
            if (eq != std::string::npos) {
                a.opt[k.substr(0, eq)] = k.substr(eq + 1);
            } else {
                if (i + 1 >= argc) throw std::invalid_argument("option --" + k + " needs a value");
                a.opt[k] = argv[++i];
            }
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        usage();
        return 2;
    }
    try {
        if (a.cmd == "classify") return classify_cmd(a);
        if (a.cmd == "plan") return plan_cmd(a);
        if (a.cmd == "conccl-plan") return conccl_plan_cmd(a);
        if (a.cmd == "sweep") return sweep_cmd(a);
        if (a.cmd == "calibrate") return calibrate_cmd(a);
        if (a.cmd == "run") return run_cmd(a);
        usage();
        return 2;
    } catch (const DeviceError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 6;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const UnknownEntityError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const FitError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 5;
    } catch (const Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 4;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
