// File formats of the model layer: machine / dataset / params JSON, slowdown
// CSV, transfer-plan and partition-plan JSON. Strict parsing: unknown fields
// are rejected, missing required fields are ValidationErrors, unreadable files
// are IoErrors — the same contracts as the reference loaders
// (/root/reference/proj: src/machine.cpp:52-119, src/workload.cpp:134-215,
// src/params_io.cpp:14-70, src/interference.cpp:106-168,
// src/conccl.cpp:231-280, src/strategy.cpp:115-124).
// JSON is nlohmann/json 3.11.3 (third-party header, found at build time).
#include <cstdio>
#include <fstream>
#include <set>
#include <sstream>

#include "c3sim/conccl.hpp"
#include "c3sim/errors.hpp"
#include "c3sim/interference.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/params_io.hpp"
#include "c3sim/strategy.hpp"
#include "c3sim/workload.hpp"
#include "json.hpp"

namespace c3sim {

using nlohmann::json;

namespace {

std::string slurp(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open file: " + path.string());
    std::ostringstream os;
    os << f.rdbuf();
    return os.str();
}

json parse_or_throw(const std::string& text, const char* what) {
    try {
        return json::parse(text);
    } catch (const json::exception& e) {
        throw ValidationError(std::string(what) + ": parse failure: " + e.what());
    }
}

void reject_unknown(const json& j, const std::set<std::string>& known, const std::string& what) {
    for (const auto& item : j.items())
        if (!known.count(item.key())) throw ValidationError(what + " '" + item.key() + "'");
}

const std::set<std::string> kMachineFields = {
    "gpus_per_node",         "cus_per_gpu",   "xcds_per_gpu", "cus_per_xcd",
    "min_cu_grain",          "dma_engines_per_gpu", "peak_compute_flops", "hbm_bandwidth",
    "llc_capacity",          "link_bandwidth_unidir", "links_per_gpu", "topology",
    "cpu_launch_overhead",   "dma_sync_overhead"};

}  // namespace

// ---------------------------------------------------------------- machine ---

MachineDescriptor load_machine(const std::string& text) {
    const json j = parse_or_throw(text, "machine");
    if (!j.is_object()) throw ValidationError("machine: top-level value must be an object");
    reject_unknown(j, kMachineFields, "machine: unknown field");
    for (const auto& k : kMachineFields)
        if (!j.contains(k)) throw ValidationError("machine: missing field '" + k + "'");
    MachineDescriptor md;
    try {
        j.at("gpus_per_node").get_to(md.gpus_per_node);
        j.at("cus_per_gpu").get_to(md.cus_per_gpu);
        j.at("xcds_per_gpu").get_to(md.xcds_per_gpu);
        j.at("cus_per_xcd").get_to(md.cus_per_xcd);
        j.at("min_cu_grain").get_to(md.min_cu_grain);
        j.at("dma_engines_per_gpu").get_to(md.dma_engines_per_gpu);
        j.at("peak_compute_flops").get_to(md.peak_compute_flops);
        j.at("hbm_bandwidth").get_to(md.hbm_bandwidth);
        j.at("llc_capacity").get_to(md.llc_capacity);
        j.at("link_bandwidth_unidir").get_to(md.link_bandwidth_unidir);
        j.at("links_per_gpu").get_to(md.links_per_gpu);
        j.at("cpu_launch_overhead").get_to(md.cpu_launch_overhead);
        j.at("dma_sync_overhead").get_to(md.dma_sync_overhead);
        const std::string topo = j.at("topology").get<std::string>();
        if (topo != "fully-connected")
            throw ValidationError("machine: unsupported topology '" + topo + "'");
        md.topology = Topology::FullyConnected;
    } catch (const json::exception& e) {
        throw ValidationError(std::string("machine: bad field type: ") + e.what());
    }
    validate(md);
    return md;
}

MachineDescriptor load_machine_file(const std::filesystem::path& path) {
    return load_machine(slurp(path));
}

std::string save_machine(const MachineDescriptor& md) {
    json j = {{"gpus_per_node", md.gpus_per_node},
              {"cus_per_gpu", md.cus_per_gpu},
              {"xcds_per_gpu", md.xcds_per_gpu},
              {"cus_per_xcd", md.cus_per_xcd},
              {"min_cu_grain", md.min_cu_grain},
              {"dma_engines_per_gpu", md.dma_engines_per_gpu},
              {"peak_compute_flops", md.peak_compute_flops},
              {"hbm_bandwidth", md.hbm_bandwidth},
              {"llc_capacity", md.llc_capacity},
              {"link_bandwidth_unidir", md.link_bandwidth_unidir},
              {"links_per_gpu", md.links_per_gpu},
              {"topology", "fully-connected"},
              {"cpu_launch_overhead", md.cpu_launch_overhead},
              {"dma_sync_overhead", md.dma_sync_overhead}};
    return j.dump(2) + "\n";
}

// ---------------------------------------------------------------- dataset ---

namespace {

GemmKernel gemm_of(const json& j) {
    reject_unknown(j, {"tag", "m", "n", "k", "dtype_bytes", "measured_op_to_byte", "measured_time",
                       "boundedness_override"},
                   "dataset: unknown gemm field");
    GemmKernel g;
    g.tag = j.at("tag").get<std::string>();
    g.m = j.at("m").get<std::int64_t>();
    g.n = j.at("n").get<std::int64_t>();
    g.k = j.at("k").get<std::int64_t>();
    g.dtype_bytes = j.at("dtype_bytes").get<int>();
    if (j.contains("measured_op_to_byte")) g.measured_op_to_byte = j.at("measured_op_to_byte").get<double>();
    if (j.contains("measured_time")) g.measured_time = j.at("measured_time").get<double>();
    if (j.contains("boundedness_override")) {
        const std::string b = j.at("boundedness_override").get<std::string>();
        if (b == "compute-bound")
            g.boundedness_override = Boundedness::ComputeBound;
        else if (b == "memory-bound")
            g.boundedness_override = Boundedness::MemoryBound;
        else
            throw ValidationError("dataset: bad boundedness_override '" + b + "'");
    }
    validate(g);
    return g;
}

CollectiveOp collective_of(const json& j) {
    reject_unknown(j, {"kind", "payload_bytes", "n_ranks", "measured_time"},
                   "dataset: unknown collective field");
    CollectiveOp c;
    c.kind = collective_kind_from_string(j.at("kind").get<std::string>());
    c.payload_bytes = j.at("payload_bytes").get<std::int64_t>();
    c.n_ranks = j.at("n_ranks").get<int>();
    if (j.contains("measured_time")) c.measured_time = j.at("measured_time").get<double>();
    validate(c);
    return c;
}

}  // namespace

std::vector<C3Scenario> parse_dataset(const std::string& text) {
    const json j = parse_or_throw(text, "dataset");
    if (!j.is_array()) throw ValidationError("dataset: top-level value must be an array");
    std::vector<C3Scenario> out;
    std::set<std::pair<std::string, std::string>> ids;
    for (const json& item : j) {
        reject_unknown(item, {"id", "source", "expected_taxonomy", "gemm", "collective"},
                       "dataset: unknown scenario field");
        C3Scenario s;
        s.id = item.at("id").get<std::string>();
        s.source = item.value("source", std::string("synthetic"));
        s.gemm = gemm_of(item.at("gemm"));
        s.collective = collective_of(item.at("collective"));
        if (item.contains("expected_taxonomy"))
            s.expected_taxonomy = taxonomy_from_string(item.at("expected_taxonomy").get<std::string>());
        if (!ids.emplace(s.id, to_string(s.collective.kind)).second)
            throw ValidationError("dataset: duplicate scenario '" + s.id + "' for " +
                                  to_string(s.collective.kind));
        out.push_back(std::move(s));
    }
    return out;
}

std::vector<C3Scenario> load_dataset(const std::filesystem::path& path) {
    return parse_dataset(slurp(path));
}

// ----------------------------------------------------------------- params ---

RunParams load_params(const std::string& text) {
    const json j = parse_or_throw(text, "params");
    reject_unknown(j, {"efficiency", "comm_launch_overhead_cu", "co_run_penalty", "freeze_phase2_allocation"},
                   "params: unknown field");
    RunParams p;
    try {
        p.eff.efficiency = j.at("efficiency").get<double>();
        p.eff.comm_launch_overhead_cu = j.at("comm_launch_overhead_cu").get<double>();
        if (j.contains("freeze_phase2_allocation"))
            p.freeze_phase2_allocation = j.at("freeze_phase2_allocation").get<bool>();
        if (j.contains("co_run_penalty"))
            for (const auto& item : j.at("co_run_penalty").items()) {
                const KernelClass cls = kernel_class_from_string(item.key());
                p.penalties.set(cls, CommBackend::CU, item.value().at("cu").get<double>());
                p.penalties.set(cls, CommBackend::DMA, item.value().at("dma").get<double>());
            }
    } catch (const json::exception& e) {
        throw ValidationError(std::string("params: bad field: ") + e.what());
    }
    validate(p.eff);
    validate(p.penalties);
    return p;
}

RunParams load_params_file(const std::filesystem::path& path) { return load_params(slurp(path)); }

std::string save_params(const RunParams& p) {
    json pen = json::object();
    for (int c = 0; c < kNumKernelClasses; ++c) {
        const auto cls = static_cast<KernelClass>(c);
        pen[to_string(cls)] = {{"cu", p.penalties.get(cls, CommBackend::CU)},
                               {"dma", p.penalties.get(cls, CommBackend::DMA)}};
    }
    json j = {{"efficiency", p.eff.efficiency},
              {"comm_launch_overhead_cu", p.eff.comm_launch_overhead_cu},
              {"co_run_penalty", pen},
              {"freeze_phase2_allocation", p.freeze_phase2_allocation}};
    return j.dump(2) + "\n";
}

// ------------------------------------------------------- slowdown tables ---

namespace {
std::string strip(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return {};
    return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}
}  // namespace

SlowdownTableSet parse_slowdown_tables(const std::string& text, int min_cu_grain) {
    std::istringstream in(text);
    std::string line;
    if (!std::getline(in, line) || strip(line) != "kernel_class,cus,slowdown")
        throw ValidationError("slowdown tables: expected header kernel_class,cus,slowdown");
    SlowdownTableSet set;
    bool seen[kNumKernelClasses] = {};
    for (int i = 0; i < kNumKernelClasses; ++i) set.tables[static_cast<std::size_t>(i)].kernel_class = static_cast<KernelClass>(i);
    for (int lineno = 2; std::getline(in, line); ++lineno) {
        const std::string row = strip(line);
        if (row.empty()) continue;
        std::vector<std::string> cells;
        std::istringstream cs(row);
        for (std::string cell; std::getline(cs, cell, ',');) cells.push_back(cell);
        if (cells.size() < 3)
            throw ValidationError("slowdown tables: malformed row at line " + std::to_string(lineno));
        if (cells.size() > 3)
            throw ValidationError("slowdown tables: too many cells at line " + std::to_string(lineno));
        const KernelClass cls = kernel_class_from_string(strip(cells[0]));
        SlowdownPoint pt{};
        try {
            pt.cus = std::stoi(strip(cells[1]));
            pt.slowdown = std::stod(strip(cells[2]));
        } catch (const std::exception&) {
            throw ValidationError("slowdown tables: bad number at line " + std::to_string(lineno));
        }
        set.at(cls).points.push_back(pt);
        seen[static_cast<int>(cls)] = true;
    }
    for (int i = 0; i < kNumKernelClasses; ++i) {
        if (!seen[i])
            throw ValidationError("slowdown tables: missing class " + to_string(static_cast<KernelClass>(i)));
        validate(set.tables[static_cast<std::size_t>(i)], min_cu_grain);
    }
    return set;
}

SlowdownTableSet load_slowdown_tables(const std::filesystem::path& path, int min_cu_grain) {
    return parse_slowdown_tables(slurp(path), min_cu_grain);
}

std::string save_slowdown_tables(const SlowdownTableSet& set) {
    std::ostringstream os;
    os << "kernel_class,cus,slowdown\n";
    for (const SlowdownTable& t : set.tables)
        for (const SlowdownPoint& p : t.points) {
            char num[64];
            std::snprintf(num, sizeof num, "%.17g", p.slowdown);
            os << to_string(t.kernel_class) << ',' << p.cus << ',' << num << '\n';
        }
    return os.str();
}

// ------------------------------------------------------------ plans JSON ---

std::string to_json(const TransferPlan& plan) {
    json ts = json::array();
    for (const Transfer& t : plan.transfers)
        ts.push_back({{"src", t.src_gpu}, {"dst", t.dst_gpu}, {"src_off", t.src_offset},
                      {"dst_off", t.dst_offset}, {"len", t.length}, {"engine", t.engine_id},
                      {"seq", t.seq}});
    json j = {{"kind", to_string(plan.kind)},
              {"n_ranks", plan.n_ranks},
              {"chunk_bytes", plan.chunk_bytes},
              {"src_buffer_bytes", plan.buffers.src_bytes},
              {"dst_buffer_bytes", plan.buffers.dst_bytes},
              {"transfers", ts}};
    return j.dump(2) + "\n";
}

TransferPlan plan_from_json(const std::string& text) {
    const json j = parse_or_throw(text, "transfer plan");
    TransferPlan plan;
    try {
        plan.kind = collective_kind_from_string(j.at("kind").get<std::string>());
        plan.n_ranks = j.at("n_ranks").get<int>();
        plan.chunk_bytes = j.at("chunk_bytes").get<std::int64_t>();
        plan.buffers.src_bytes = j.at("src_buffer_bytes").get<std::int64_t>();
        plan.buffers.dst_bytes = j.at("dst_buffer_bytes").get<std::int64_t>();
        for (const json& t : j.at("transfers"))
            plan.transfers.push_back({t.at("src").get<int>(), t.at("dst").get<int>(),
                                      t.at("src_off").get<std::int64_t>(),
                                      t.at("dst_off").get<std::int64_t>(),
                                      t.at("len").get<std::int64_t>(), t.at("engine").get<int>(),
                                      t.at("seq").get<int>()});
    } catch (const json::exception& e) {
        throw ValidationError(std::string("transfer plan: bad field: ") + e.what());
    }
    return plan;
}

std::string to_json(const PartitionPlan& p) {
    json j = {{"comm_backend", p.comm_backend == CommBackend::CU ? "CU" : "DMA"},
              {"cus_comm", p.cus_comm},
              {"cus_gemm", p.cus_gemm},
              {"cus_idle", p.cus_idle},
              {"schedule_order", p.schedule_order},
              {"predicted_makespan_s", p.predicted_makespan}};
    return j.dump(2) + "\n";
}

}  // namespace c3sim
