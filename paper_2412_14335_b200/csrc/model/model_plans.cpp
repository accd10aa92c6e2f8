// ConCCL collective decomposition: transfer plans, their exact validator and
// their event cost model. These plans are what the B200 copy-engine executor
// (csrc/cuda/runtime.cpp ce_run) runs: one batched submission per engine.
//
// Reference semantics (/root/reference/proj):
//   plan_all_gather   src/conccl.cpp:24-53   (peer-indexed engine, per-engine seq)
//   plan_all_to_all   src/conccl.cpp:55-84   (transpose)
//   validate_plan     src/conccl.cpp:102-198 (structure + byte-interval replay)
//   plan_cost         src/conccl.cpp:200-229 (serial CPU submitter, FIFO engines,
//                                             dedicated (src,dst) links, one sync)
// Extension: plan_reduce_scatter = the transpose into a staging buffer.
#include <algorithm>
#include <map>
#include <string>
#include <utility>

#include "c3sim/conccl.hpp"
#include "c3sim/errors.hpp"

namespace c3sim {

namespace {

void require_plan_args(int n_ranks, std::int64_t chunk, const MachineDescriptor& md) {
    if (n_ranks < 1) throw ValidationError("transfer plan: n_ranks must be >= 1");
    if (n_ranks > md.gpus_per_node)
        throw ValidationError("transfer plan: n_ranks exceeds gpus_per_node");
    if (n_ranks > 1 && chunk <= 0) throw ValidationError("transfer plan: chunk_bytes must be > 0");
}

// Shared builder: for each source rank g, one transfer to every other rank p.
// `src_slot(g, p)` / `dst_slot(g, p)` give the slot indices (times chunk).
template <class SrcSlot, class DstSlot>
TransferPlan direct_plan(CollectiveKind kind, int n, std::int64_t chunk, std::int64_t src_bytes,
                         const MachineDescriptor& md, SrcSlot src_slot, DstSlot dst_slot) {
    require_plan_args(n, chunk, md);
    TransferPlan plan;
    plan.kind = kind;
    plan.n_ranks = n;
    plan.chunk_bytes = chunk;
    plan.buffers.src_bytes = src_bytes;
    plan.buffers.dst_bytes = chunk * n;
    if (n == 1) return plan;
    const int engines = md.dma_engines_per_gpu;
    plan.transfers.reserve(static_cast<std::size_t>(n) * (n - 1));
    for (int g = 0; g < n; ++g) {
        std::vector<int> fifo_depth(static_cast<std::size_t>(engines), 0);
        int k = 0;  // index of p among g's peers
        for (int p = 0; p < n; ++p) {
            if (p == g) continue;
            Transfer t;
            t.src_gpu = g;
            t.dst_gpu = p;
            t.src_offset = static_cast<std::int64_t>(src_slot(g, p)) * chunk;
            t.dst_offset = static_cast<std::int64_t>(dst_slot(g, p)) * chunk;
            t.length = chunk;
            t.engine_id = k % engines;
            t.seq = fifo_depth[static_cast<std::size_t>(t.engine_id)]++;
            plan.transfers.push_back(t);
            ++k;
        }
    }
    return plan;
}

std::string where(int rank, std::int64_t offset, std::int64_t chunk) {
    return "(rank " + std::to_string(rank) + ", slot " + std::to_string(offset / chunk) + ")";
}

struct Written {  // one replayed write: [lo, hi) on the destination rank
    std::int64_t lo, hi;
    int src_rank;
    std::int64_t src_lo;
};

}  // namespace

TransferPlan plan_all_gather(int n_ranks, std::int64_t chunk_bytes, const MachineDescriptor& md) {
    return direct_plan(CollectiveKind::AllGather, n_ranks, chunk_bytes, chunk_bytes, md,
                       [](int, int) { return 0; }, [](int g, int) { return g; });
}

TransferPlan plan_all_to_all(int n_ranks, std::int64_t per_peer_bytes,
                             const MachineDescriptor& md) {
    return direct_plan(CollectiveKind::AllToAll, n_ranks, per_peer_bytes,
                       per_peer_bytes * n_ranks, md, [](int, int p) { return p; },
                       [](int g, int) { return g; });
}

TransferPlan plan_reduce_scatter(int n_ranks, std::int64_t per_peer_bytes,
                                 const MachineDescriptor& md) {
    TransferPlan plan = plan_all_to_all(n_ranks, per_peer_bytes, md);
    plan.kind = CollectiveKind::ReduceScatter;
    return plan;
}

PlanCheck validate_plan(const TransferPlan& plan, const MachineDescriptor& md) {
    const auto reject = [](std::string why) { return PlanCheck{false, std::move(why)}; };
    const int n = plan.n_ranks;
    if (n < 1) return reject("n_ranks must be >= 1");
    if (n > md.gpus_per_node) return reject("n_ranks exceeds gpus_per_node");
    const std::int64_t want_count = n >= 2 ? static_cast<std::int64_t>(n) * (n - 1) : 0;
    if (static_cast<std::int64_t>(plan.transfers.size()) != want_count)
        return reject("transfer count " + std::to_string(plan.transfers.size()) +
                      " != n*(n-1) = " + std::to_string(want_count));
    if (n == 1) return {};
    const std::int64_t chunk = plan.chunk_bytes;
    if (chunk <= 0) return reject("chunk_bytes must be > 0");
    const bool gather = plan.kind == CollectiveKind::AllGather;
    if (plan.buffers.src_bytes != (gather ? chunk : chunk * n) ||
        plan.buffers.dst_bytes != chunk * n)
        return reject("buffer extents do not match kind/chunk/n_ranks");

    std::map<std::pair<int, int>, std::vector<int>> fifo;  // (src rank, engine) -> seqs
    for (const Transfer& t : plan.transfers) {
        if (t.src_gpu == t.dst_gpu) return reject("self transfer on rank " + std::to_string(t.src_gpu));
        if (t.src_gpu < 0 || t.src_gpu >= n || t.dst_gpu < 0 || t.dst_gpu >= n)
            return reject("rank id out of range");
        if (t.length <= 0) return reject("non-positive transfer length");
        if (t.engine_id < 0 || t.engine_id >= md.dma_engines_per_gpu)
            return reject("engine_id out of range");
        if (t.src_offset < 0 || t.src_offset + t.length > plan.buffers.src_bytes)
            return reject("source range out of bounds on rank " + std::to_string(t.src_gpu));
        if (t.dst_offset < 0 || t.dst_offset + t.length > plan.buffers.dst_bytes)
            return reject("destination range out of bounds on rank " + std::to_string(t.dst_gpu));
        fifo[{t.src_gpu, t.engine_id}].push_back(t.seq);
    }
    for (auto& [key, seqs] : fifo) {
        std::sort(seqs.begin(), seqs.end());
        for (std::size_t i = 0; i < seqs.size(); ++i)
            if (seqs[i] != static_cast<int>(i))
                return reject("seq numbers not contiguous from 0 on gpu " + std::to_string(key.first) +
                              " engine " + std::to_string(key.second));
    }

    // Replay in plan order: any overlap with an earlier write is a double write.
    std::vector<std::vector<Written>> per_rank(static_cast<std::size_t>(n));
    for (const Transfer& t : plan.transfers) {
        auto& mine = per_rank[static_cast<std::size_t>(t.dst_gpu)];
        const Written w{t.dst_offset, t.dst_offset + t.length, t.src_gpu, t.src_offset};
        for (const Written& o : mine)
            if (w.lo < o.hi && o.lo < w.hi)
                return reject("overlapping writes at " + where(t.dst_gpu, w.lo, chunk));
        mine.push_back(w);
    }
    // The resident slot (own chunk / self slot) must stay untouched.
    for (int r = 0; r < n; ++r) {
        const std::int64_t lo = static_cast<std::int64_t>(r) * chunk, hi = lo + chunk;
        for (const Written& w : per_rank[static_cast<std::size_t>(r)])
            if (w.lo < hi && lo < w.hi) return reject("write into resident slot " + where(r, lo, chunk));
    }
    // Every other slot must be tiled exactly, from the right source bytes.
    for (int r = 0; r < n; ++r) {
        std::vector<Written> ws = per_rank[static_cast<std::size_t>(r)];
        std::sort(ws.begin(), ws.end(), [](const Written& a, const Written& b) { return a.lo < b.lo; });
        std::size_t next = 0;
        for (int slot = 0; slot < n; ++slot) {
            if (slot == r) continue;
            const std::int64_t base = static_cast<std::int64_t>(slot) * chunk, end = base + chunk;
            std::int64_t at = base;
            while (at < end) {
                if (next >= ws.size() || ws[next].lo != at)
                    return reject("incomplete coverage at " + where(r, at, chunk));
                const Written& w = ws[next];
                if (w.hi > end) return reject("write crosses slot boundary at " + where(r, at, chunk));
                // all-gather: slot s <- rank s's chunk; transpose kinds: slot s <-
                // rank s's source slot r.
                const std::int64_t want_src_lo =
                    gather ? at - base : static_cast<std::int64_t>(r) * chunk + (at - base);
                if (w.src_rank != slot || w.src_lo != want_src_lo)
                    return reject("wrong source data at " + where(r, at, chunk));
                at = w.hi;
                ++next;
            }
        }
        if (next != ws.size()) return reject("unexpected extra write on rank " + std::to_string(r));
    }
    return {};
}

PlanCost plan_cost(const TransferPlan& plan, const MachineDescriptor& md,
                   const EfficiencyParams& params) {
    PlanCost cost;
    cost.per_engine.assign(static_cast<std::size_t>(md.dma_engines_per_gpu), 0.0);
    if (plan.transfers.empty()) return cost;
    const double bw = params.efficiency * md.link_bandwidth_unidir;
    std::map<std::pair<int, int>, double> engine_busy_until, link_busy_until;
    double finish = 0.0, longest = 0.0;
    for (std::size_t i = 0; i < plan.transfers.size(); ++i) {
        const Transfer& t = plan.transfers[i];
        const double duration = static_cast<double>(t.length) / bw;
        longest = std::max(longest, duration);
        double& engine = engine_busy_until[{t.src_gpu, t.engine_id}];
        double& link = link_busy_until[{t.src_gpu, t.dst_gpu}];
        const double submitted = static_cast<double>(i) * md.cpu_launch_overhead;
        const double begin = std::max(std::max(submitted, engine), link);
        const double end = begin + duration;
        engine = end;
        link = end;
        double& pe = cost.per_engine[static_cast<std::size_t>(t.engine_id)];
        pe = std::max(pe, end);
        finish = std::max(finish, end);
    }
    cost.wire = longest;
    cost.total = finish + md.dma_sync_overhead;
    return cost;
}

}  // namespace c3sim
