// Model primitives of the C3 hot path: machine invariants, the C3 taxonomy and
// metric, GEMM / collective rooflines and bandwidth demands.
//
// Semantics follow the reference model layer (paths under /root/reference/proj):
//   validate(MachineDescriptor)              src/machine.cpp:26-50
//   machine_op_to_byte                       src/machine.cpp:121-124
//   classify_c3 / ideal_speedup / fraction   src/taxonomy.cpp:9-33
//   validate(Gemm/Collective/Efficiency)     src/workload.cpp:16-41
//   gemm_flops / gemm_min_bytes              src/workload.cpp:43-53
//   boundedness classifiers                  src/workload.cpp:55-70
//   roofline_gemm_time / _collective_time    src/workload.cpp:72-91
//   estimate_workgroups                      src/workload.cpp:93-103
//   bandwidth demands                        src/workload.cpp:105-122
//   ingest_model                             src/workload.cpp:217-251
// Floating-point expressions keep the reference's operation order so results
// are bit-identical (tests/test_model.py compares the full sweep byte-for-byte).
#include <algorithm>
#include <string>

#include "c3sim/errors.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/taxonomy.hpp"
#include "c3sim/workload.hpp"

namespace c3sim {

// ---------------------------------------------------------------- machine ---

void validate(const MachineDescriptor& md) {
    const auto bad = [](const std::string& why) -> void { throw ValidationError("machine: " + why); };
    if (md.gpus_per_node < 1) bad("gpus_per_node must be >= 1");
    if (md.cus_per_gpu < 1) bad("cus_per_gpu must be >= 1");
    if (md.xcds_per_gpu < 1) bad("xcds_per_gpu must be >= 1");
    if (md.cus_per_xcd < 1) bad("cus_per_xcd must be >= 1");
    const int product = md.xcds_per_gpu * md.cus_per_xcd;
    if (md.cus_per_gpu != product)
        bad("cus_per_gpu (" + std::to_string(md.cus_per_gpu) + ") != xcds_per_gpu * cus_per_xcd (" +
            std::to_string(product) + ")");
    if (md.min_cu_grain < 1) bad("min_cu_grain must be >= 1");
    if (md.cus_per_gpu % md.min_cu_grain) bad("min_cu_grain must divide cus_per_gpu");
    if (md.dma_engines_per_gpu < 1) bad("dma_engines_per_gpu must be >= 1");
    if (!(md.peak_compute_flops > 0)) bad("peak_compute_flops must be > 0");
    if (!(md.hbm_bandwidth > 0)) bad("hbm_bandwidth must be > 0");
    if (md.llc_capacity <= 0) bad("llc_capacity must be > 0");
    if (!(md.link_bandwidth_unidir > 0)) bad("link_bandwidth_unidir must be > 0");
    if (md.links_per_gpu < 0) bad("links_per_gpu must be >= 0");
    if (md.topology == Topology::FullyConnected && md.links_per_gpu + 1 != md.gpus_per_node)
        bad("fully-connected topology requires links_per_gpu == gpus_per_node - 1");
    if (md.cpu_launch_overhead < 0) bad("cpu_launch_overhead must be >= 0");
    if (md.dma_sync_overhead < 0) bad("dma_sync_overhead must be >= 0");
}

double machine_op_to_byte(const MachineDescriptor& md) {
    if (!(md.hbm_bandwidth > 0)) throw ValidationError("machine: hbm_bandwidth must be > 0");
    return md.peak_compute_flops / md.hbm_bandwidth;
}

// --------------------------------------------------------------- taxonomy ---

TaxonomyLabel classify_c3(double t_gemm, double t_comm, double threshold) {
    if (!(t_gemm > 0 && t_comm > 0)) throw ValidationError("classify_c3: times must be positive");
    if (!(threshold > 1)) throw ValidationError("classify_c3: threshold must be > 1");
    TaxonomyLabel label{TaxonomyClass::GCEqual, threshold};
    if (t_gemm > threshold * t_comm)
        label.value = TaxonomyClass::GLong;
    else if (t_comm > threshold * t_gemm)
        label.value = TaxonomyClass::CLong;
    return label;
}

double ideal_speedup(double t_gemm, double t_comm) {
    if (!(t_gemm > 0 && t_comm > 0)) throw ValidationError("ideal_speedup: times must be positive");
    const double longest = t_gemm < t_comm ? t_comm : t_gemm;
    return (t_gemm + t_comm) / longest;
}

double fraction_of_ideal(double achieved_speedup, double ideal) {
    if (!(ideal > 1)) throw ValidationError("fraction_of_ideal: ideal must be > 1");
    return achieved_speedup < 1.0 ? 0.0 : (achieved_speedup - 1.0) / (ideal - 1.0);
}

std::string to_string(TaxonomyClass c) {
    if (c == TaxonomyClass::GLong) return "G-long";
    if (c == TaxonomyClass::CLong) return "C-long";
    if (c == TaxonomyClass::GCEqual) return "GC-equal";
    return "?";
}

TaxonomyClass taxonomy_from_string(const std::string& s) {
    for (TaxonomyClass c : {TaxonomyClass::GLong, TaxonomyClass::CLong, TaxonomyClass::GCEqual})
        if (to_string(c) == s) return c;
    throw ValidationError("unknown taxonomy label '" + s + "'");
}

// --------------------------------------------------------------- workload ---

void validate(const GemmKernel& g) {
    const std::string who = "gemm '" + g.tag + "': ";
    if (g.m < 1 || g.n < 1 || g.k < 1) throw ValidationError(who + "dimensions must be >= 1");
    switch (g.dtype_bytes) {
        case 1: case 2: case 4: case 8: break;
        default: throw ValidationError(who + "dtype_bytes must be 1, 2, 4 or 8");
    }
    if (g.measured_op_to_byte && !(*g.measured_op_to_byte > 0))
        throw ValidationError(who + "measured_op_to_byte must be > 0");
    if (g.measured_time && !(*g.measured_time > 0))
        throw ValidationError(who + "measured_time must be > 0");
}

void validate(const CollectiveOp& c) {
    if (c.payload_bytes < 0) throw ValidationError("collective: payload_bytes must be >= 0");
    if (c.n_ranks < 1) throw ValidationError("collective: n_ranks must be >= 1");
    if (c.payload_bytes % c.n_ranks)
        throw ValidationError("collective: payload_bytes must be divisible by n_ranks");
    if (c.measured_time && !(*c.measured_time > 0))
        throw ValidationError("collective: measured_time must be > 0");
}

void validate(const EfficiencyParams& p) {
    if (!(p.efficiency > 0 && p.efficiency <= 1))
        throw ValidationError("params: efficiency must be in (0, 1]");
    if (p.comm_launch_overhead_cu < 0)
        throw ValidationError("params: comm_launch_overhead_cu must be >= 0");
}

double gemm_flops(const GemmKernel& g) {
    double f = 2.0 * static_cast<double>(g.m);
    f *= static_cast<double>(g.n);
    return f * static_cast<double>(g.k);
}

double gemm_min_bytes(const GemmKernel& g) {
    const double m = static_cast<double>(g.m), n = static_cast<double>(g.n),
                 k = static_cast<double>(g.k);
    const double a = m * k, b = k * n, c = m * n;  // operand and result elements
    return static_cast<double>(g.dtype_bytes) * (a + b + c);
}

Boundedness classify_gemm_boundedness(const GemmKernel& g, double machine_ratio) {
    if (!(machine_ratio > 0))
        throw ValidationError("classify_gemm_boundedness: machine_ratio must be > 0");
    if (g.boundedness_override) return *g.boundedness_override;
    const double intensity = g.measured_op_to_byte.value_or(gemm_flops(g) / gemm_min_bytes(g));
    return intensity > machine_ratio ? Boundedness::ComputeBound : Boundedness::MemoryBound;
}

double roofline_gemm_time(const GemmKernel& g, const MachineDescriptor& md,
                          const EfficiencyParams& p) {
    if (g.measured_time) return *g.measured_time;
    const double t_flops = gemm_flops(g) / (p.efficiency * md.peak_compute_flops);
    const double t_bytes = gemm_min_bytes(g) / (p.efficiency * md.hbm_bandwidth);
    return t_flops < t_bytes ? t_bytes : t_flops;
}

double roofline_collective_time(const CollectiveOp& c, const MachineDescriptor& md,
                                const EfficiencyParams& p, bool include_overhead) {
    if (c.measured_time) return *c.measured_time;
    if (c.n_ranks > md.gpus_per_node)
        throw ValidationError("collective: n_ranks exceeds gpus_per_node");
    if (c.n_ranks == 1) return 0.0;
    const double per_peer = static_cast<double>(c.payload_bytes) / static_cast<double>(c.n_ranks);
    const double wire = per_peer / (p.efficiency * md.link_bandwidth_unidir);
    return include_overhead ? wire + p.comm_launch_overhead_cu : wire;
}

CommBoundedness classify_collective_boundedness(const CollectiveOp& c,
                                                const MachineDescriptor& md,
                                                const EfficiencyParams& p) {
    const double wire = roofline_collective_time(c, md, p, false);
    return p.comm_launch_overhead_cu >= wire ? CommBoundedness::LatencyBound
                                             : CommBoundedness::BandwidthBound;
}

int estimate_workgroups(const GemmKernel& g, int tile) {
    if (tile < 1) throw ValidationError("estimate_workgroups: tile must be >= 1");
    const std::int64_t tm = (g.m + tile - 1) / tile, tn = (g.n + tile - 1) / tile;
    return static_cast<int>(std::min<std::int64_t>(tm * tn, std::int64_t{1} << 30));
}

// Launch widths of the modeled CU collectives: all-gather 64 workgroups,
// all-to-all 56; a reduce-scatter runs the all-to-all exchange pattern.
int estimate_workgroups(const CollectiveOp& c) {
    return c.kind == CollectiveKind::AllGather ? 64 : 56;
}

double gemm_bandwidth_demand(const GemmKernel& g, const MachineDescriptor& md,
                             const EfficiencyParams& p) {
    const double t = roofline_gemm_time(g, md, p);
    if (!(t > 0)) throw ValidationError("gemm_bandwidth_demand: zero roofline time");
    return gemm_min_bytes(g) / t;
}

double collective_bandwidth_demand(const CollectiveOp& c, const MachineDescriptor& md,
                                   const EfficiencyParams& p) {
    if (c.n_ranks == 1 || c.payload_bytes == 0) return 0.0;
    const double wire = roofline_collective_time(c, md, p, false);
    if (!(wire > 0)) throw ValidationError("collective_bandwidth_demand: zero wire time");
    // HBM traffic per byte on the wire: an all-gather reads the own chunk and
    // writes the received ones (~14% below a full read+write); all-to-all and
    // the reduce-scatter exchange are a full read + write.
    const double factor = c.kind == CollectiveKind::AllGather ? 2.0 * 0.86 : 2.0;
    const double remote_share =
        static_cast<double>(c.n_ranks - 1) / static_cast<double>(c.n_ranks);
    return factor * remote_share * static_cast<double>(c.payload_bytes) / wire;
}

ModelWorkload ingest_model(const ModelConfig& cfg) {
    if (cfg.hidden < 1 || cfg.ffn < 1 || cfg.tokens < 1)
        throw ValidationError("ingest_model: dimensions must be >= 1");
    if (cfg.shards < 1) throw ValidationError("ingest_model: shards must be >= 1");
    struct Proj {
        const char* tag;
        std::int64_t n, k;
    };
    const Proj projections[] = {{"attn_qkv", 3 * cfg.hidden, cfg.hidden},
                                {"attn_out", cfg.hidden, cfg.hidden},
                                {"ffn_in", 2 * cfg.ffn, cfg.hidden},
                                {"ffn_out", cfg.hidden, cfg.ffn}};
    ModelWorkload w;
    for (const Proj& pr : projections) {
        GemmKernel g;
        g.tag = pr.tag;
        g.m = cfg.tokens;
        g.n = pr.n;
        g.k = pr.k;
        g.dtype_bytes = cfg.dtype_bytes;
        validate(g);
        w.gemms.push_back(g);
        if (cfg.shards == 1) continue;
        CollectiveOp ag;
        ag.kind = CollectiveKind::AllGather;
        ag.n_ranks = cfg.shards;
        ag.payload_bytes = pr.n * pr.k * cfg.dtype_bytes;  // whole weight after the gather
        const std::int64_t rem = ag.payload_bytes % ag.n_ranks;
        if (rem) ag.payload_bytes += ag.n_ranks - rem;      // pad to an even shard
        validate(ag);
        w.all_gathers.push_back(ag);
    }
    return w;
}

std::string to_string(CollectiveKind k) {
    switch (k) {
        case CollectiveKind::AllGather: return "all-gather";
        case CollectiveKind::AllToAll: return "all-to-all";
        case CollectiveKind::ReduceScatter: return "reduce-scatter";
    }
    return "?";
}

CollectiveKind collective_kind_from_string(const std::string& s) {
    for (CollectiveKind k :
         {CollectiveKind::AllGather, CollectiveKind::AllToAll, CollectiveKind::ReduceScatter})
        if (to_string(k) == s) return k;
    throw ValidationError("unknown collective kind '" + s + "'");
}

std::string to_string(Boundedness b) {
    return b == Boundedness::MemoryBound ? "memory-bound" : "compute-bound";
}

std::string to_string(CommBoundedness b) {
    return b == CommBoundedness::BandwidthBound ? "bandwidth-bound" : "latency-bound";
}

}  // namespace c3sim
