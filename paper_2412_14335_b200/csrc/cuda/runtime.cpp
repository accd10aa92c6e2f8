// libc3cuda host runtime: error state, worlds (one device; real or loopback
// ranks), CUDA-IPC peer mapping, the copy-engine plan executor, and the C3
// session that executes one scenario under the paper's strategies.
//
// Strategy semantics are the reference's allocate_cus
// (/root/reference/proj/src/sim.cpp:40-100), turned into launch mechanics:
//   serial     GEMM then collective, back to back on one stream
//   c3_base    GEMM launched first (every SM), SM collective second with the
//              one grain the model leaves it, default priorities
//   c3_sp      SM collective launched first on the highest-priority stream
//              with its saturation CTAs; GEMM capped at cus_gemm CTAs
//   c3_rp      SM partition: green contexts (cuGreenCtx*) split the GPU into a
//              comm group of cus_comm SMs and a GEMM group (falls back to CTA
//              caps, reported in c3_timing.partition, if green contexts fail)
//   c3_sp_rp   c3_rp with the collective first on a high-priority stream
//   conccl     copy-engine collective (each TransferPlan transfer becomes a
//              cudaMemcpyAsync on the stream of its engine) + GEMM on all SMs
//   conccl_rp  copy-engine collective + GEMM capped at cus_gemm (one grain
//              idle for memory-bound GEMMs; conccl_rp_plan, strategy.cpp:96-113)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "c3cuda_internal.hpp"
#include "c3sim/conccl.hpp"
#include "c3sim/coresident.hpp"
#include "c3sim/errors.hpp"
#include "c3sim/machine.hpp"
#include "c3sim/params_io.hpp"
#include "c3sim/sim.hpp"

namespace c3k {

namespace {
thread_local std::string g_last_error;
}

const char* last_error_cstr() { return g_last_error.c_str(); }

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int set_cuda_error(cudaError_t e, const char* what) {
    return set_error(C3_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                      cudaGetErrorString(e) + ")");
}
int set_driver_error(CUresult r, const char* what) {
    const char* name = nullptr;
    if (drv().GetErrorName) drv().GetErrorName(r, &name);
    return set_error(C3_ERR_DRIVER,
                     std::string(what) + ": " + (name ? name : std::to_string(static_cast<int>(r))));
}

// Runs a model-layer call, mapping c3sim exceptions to status codes.
template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const c3sim::IoError& e) {
        return set_error(C3_ERR_IO, e.what());
    } catch (const c3sim::UnknownEntityError& e) {
        return set_error(C3_ERR_UNKNOWN, e.what());
    } catch (const c3sim::FitError& e) {
        return set_error(C3_ERR_FIT, e.what());
    } catch (const c3sim::Error& e) {
        return set_error(C3_ERR_VALIDATION, e.what());
    } catch (const std::exception& e) {
        return set_error(C3_ERR_VALIDATION, e.what());
    }
}

}  // namespace c3k

using namespace c3k;

// ------------------------------------------------------------------ world

struct GreenPartition {
    int comm_sms = 0, gemm_sms = 0;
    CUgreenCtx comm_ctx = nullptr, gemm_ctx = nullptr;
    CUstream comm_stream = nullptr, gemm_stream = nullptr;
};

struct c3_world {
    int rank = 0, n_ranks = 1, device = 0, loopback = 0;
    cudaDeviceProp prop{};
    int prio_lo = 0, prio_hi = 0;
    int green_ok = 0, green_grain = 0;
    CUdevice cu_dev = 0;
    std::vector<cudaStream_t> ce_streams;  // one per copy-engine index
    std::vector<cudaEvent_t> ce_events;
    cudaEvent_t fork_event = nullptr;
    std::map<int, GreenPartition> partitions;  // keyed by requested comm SMs
    int* gemm_counters = nullptr;              // pool for standalone c3_gemm_bf16 calls
    int gemm_counter_next = 0;
};
static constexpr int kGemmCounterSlots = 64;

namespace {

int probe_green(c3_world* w) {
    // The SM split granularity on sm_100 is not documented in the 12.9
    // headers: ask for a 1-SM group and read back what the driver grants.
    CUdevResource all{};
    const Driver& d = drv();
    if (!d.DeviceGetDevResource || !d.DevSmResourceSplitByCount || !d.GreenCtxCreate ||
        !d.GreenCtxStreamCreate || !d.DevResourceGenerateDesc)
        return 0;
    if (d.DeviceGetDevResource(w->cu_dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return 0;
    CUdevResource grp[1] = {};
    CUdevResource rest{};
    unsigned int nb = 1;
    if (d.DevSmResourceSplitByCount(grp, &nb, &all, &rest, 0, 1) != CUDA_SUCCESS || nb < 1) return 0;
    w->green_grain = static_cast<int>(grp[0].sm.smCount);
    return 1;
}

// Copy-engine stream of `engine` (mod the device's async engine count); with
// inbound = true the second bank of streams (the host-staged proxy's H2D
// half, so the two PCIe directions run side by side).
int ce_stream(c3_world* w, int engine, std::size_t* idx_out, bool inbound = false) {
    const int n_eng = std::max(1, w->prop.asyncEngineCount);
    const std::size_t idx = static_cast<std::size_t>(engine % n_eng + (inbound ? n_eng : 0));
    while (w->ce_streams.size() <= idx) {
        cudaStream_t s;
        cudaEvent_t e;
        C3_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, w->prio_hi));
        C3_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        w->ce_streams.push_back(s);
        w->ce_events.push_back(e);
    }
    *idx_out = idx;
    return C3_OK;
}

int green_partition(c3_world* w, int comm_sms, GreenPartition** out) {
    auto it = w->partitions.find(comm_sms);
    if (it != w->partitions.end()) {
        *out = &it->second;
        return C3_OK;
    }
    if (!w->green_ok) return set_error(C3_ERR_UNSUPPORTED, "green contexts unavailable on this device");
    CUdevResource all{};
    C3_CU(DeviceGetDevResource, w->cu_dev, &all, CU_DEV_RESOURCE_TYPE_SM);
    CUdevResource comm[1] = {};
    CUdevResource rest{};
    unsigned int nb = 1;
    C3_CU(DevSmResourceSplitByCount, comm, &nb, &all, &rest, 0, static_cast<unsigned>(comm_sms));
    if (nb < 1) return set_error(C3_ERR_UNSUPPORTED, "green context split produced no group");
    GreenPartition gp;
    gp.comm_sms = static_cast<int>(comm[0].sm.smCount);
    gp.gemm_sms = static_cast<int>(rest.sm.smCount);
    CUdevResourceDesc dc, dg;
    C3_CU(DevResourceGenerateDesc, &dc, comm, 1);
    C3_CU(DevResourceGenerateDesc, &dg, &rest, 1);
    C3_CU(GreenCtxCreate, &gp.comm_ctx, dc, w->cu_dev, CU_GREEN_CTX_DEFAULT_STREAM);
    C3_CU(GreenCtxCreate, &gp.gemm_ctx, dg, w->cu_dev, CU_GREEN_CTX_DEFAULT_STREAM);
    C3_CU(GreenCtxStreamCreate, &gp.comm_stream, gp.comm_ctx, CU_STREAM_NON_BLOCKING, w->prio_hi);
    C3_CU(GreenCtxStreamCreate, &gp.gemm_stream, gp.gemm_ctx, CU_STREAM_NON_BLOCKING, 0);
    *out = &w->partitions.emplace(comm_sms, gp).first->second;
    return C3_OK;
}

// Delivery flags of a multi-process copy-engine collective: after the copies
// on one engine stream, word [kSigCeDone + self] of every destination rank's
// signal array gets the step's epoch, so the receiver learns on the device
// that this rank's bytes have landed (no host barrier, nothing blocks the
// host before the GEMM is launched). A stream memop (cuStreamWriteValue32,
// which fences the stream's prior writes) when the driver has it, else a
// one-thread st.release.sys kernel.
struct CeDeliver {
    const Signals* sig = nullptr;  // peers' signal arrays, epoch, this rank
};

int ce_signal(const CeDeliver& dv, const std::vector<int>& dsts, cudaStream_t st) {
    const Signals& g = *dv.sig;
    uint32_t* words[C3_MAX_RANKS];
    int cnt = 0;
    for (int d : dsts)
        if (d != g.self) words[cnt++] = g.peers[d] + kSigCeDone + g.self;
    if (cnt == 0) return C3_OK;
    if (drv().StreamWriteValue32) {
        for (int i = 0; i < cnt; ++i)
            C3_CU(StreamWriteValue32, reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(words[i]),
                  g.epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
        return C3_OK;
    }
    return launch_flag_store(words, cnt, g.epoch, st);
}

// Copy-engine executor: fork from `parent`, one cudaMemcpyAsync per selected
// transfer on the stream of its engine_id, join back into `parent`.
// Measured on B200 (profiles/r01_ce_probe2.json): copies between two devices
// and host<->device copies run on copy engines; a copy whose source and
// destination are on the SAME device runs as a driver copy kernel on SMs
// (every runtime copy path). So the DMA backend is copy-engine only across
// devices; in a loopback world its "transfers" are SM copies.
// One submission per transfer: the reference's plan_cost charges
// cpu_launch_overhead per transfer (conccl.cpp:200-229), measured here at
// 1.5 us (data/b200-ce-overheads.json). (The batched submission API of CUDA
// 12.8+ is closed on this GPU pool after driver faults, so it is not used.)
// Transfers selected: src_gpu == src_filter, or (dst_filter >= 0) dst_gpu ==
// dst_filter; every transfer when both filters are < 0. Copies whose
// destination is dst_filter use the inbound stream bank.
int ce_run(c3_world* w, const c3_transfer* t, int nt, const void* const* src, void* const* dst,
           int src_filter, cudaStream_t parent, const CeDeliver* deliver = nullptr, int dst_filter = -1) {
    if (!w->fork_event) C3_CUDA(cudaEventCreateWithFlags(&w->fork_event, cudaEventDisableTiming));
    std::vector<char> used;
    std::vector<std::vector<int>> dst_ranks;  // destinations per engine stream (delivery flags)
    bool forked = false;
    for (int i = 0; i < nt; ++i) {
        const c3_transfer& x = t[i];
        const bool pick = (src_filter < 0 && dst_filter < 0) || x.src_gpu == src_filter || x.dst_gpu == dst_filter;
        if (!pick || x.length <= 0) continue;
        std::size_t idx = 0;
        C3_TRY(ce_stream(w, x.engine_id, &idx, dst_filter >= 0 && x.dst_gpu == dst_filter));
        if (!forked) {
            C3_CUDA(cudaEventRecord(w->fork_event, parent));
            forked = true;
        }
        if (used.size() <= idx) {
            used.resize(idx + 1, 0);
            dst_ranks.resize(idx + 1);
        }
        if (!used[idx]) {
            C3_CUDA(cudaStreamWaitEvent(w->ce_streams[idx], w->fork_event, 0));
            used[idx] = 1;
        }
        auto& dr = dst_ranks[idx];
        if (std::find(dr.begin(), dr.end(), x.dst_gpu) == dr.end()) dr.push_back(x.dst_gpu);
        void* d = static_cast<uint8_t*>(dst[x.dst_gpu]) + x.dst_offset;
        const void* sp = static_cast<const uint8_t*>(src[x.src_gpu]) + x.src_offset;
        C3_CUDA(cudaMemcpyAsync(d, sp, static_cast<size_t>(x.length), cudaMemcpyDefault, w->ce_streams[idx]));
    }
    for (std::size_t idx = 0; idx < used.size(); ++idx) {
        if (!used[idx]) continue;
        if (deliver) C3_TRY(ce_signal(*deliver, dst_ranks[idx], w->ce_streams[idx]));
        C3_CUDA(cudaEventRecord(w->ce_events[idx], w->ce_streams[idx]));
        C3_CUDA(cudaStreamWaitEvent(parent, w->ce_events[idx], 0));
    }
    return C3_OK;
}

// B200 machine descriptor for a world of `n` ranks, from the live device.
// Defaults = data/b200-node-n{n}.json (tools/make_machine.py): peaks from the
// driver-measured MEASURED_PEAKS.json of this pool, copy-engine overheads
// from data/b200-ce-overheads.json, the measured 770 GB/s peer copy shared by
// n-1 peers. c3_session_load_machine replaces it with a machine file.
c3sim::MachineDescriptor b200_machine(const c3_world* w, int n) {
    c3sim::MachineDescriptor md;
    md.gpus_per_node = n;
    md.cus_per_gpu = w->prop.multiProcessorCount;
    md.xcds_per_gpu = md.cus_per_gpu % 2 == 0 ? 2 : 1;
    md.cus_per_xcd = md.cus_per_gpu / md.xcds_per_gpu;
    md.min_cu_grain = md.cus_per_gpu % 4 == 0 ? 4 : (md.cus_per_gpu % 2 == 0 ? 2 : 1);
    md.dma_engines_per_gpu = std::max(1, w->prop.asyncEngineCount);
    md.peak_compute_flops = 1.6786e15;
    md.hbm_bandwidth = 6.5498e12;
    md.llc_capacity = w->prop.l2CacheSize;
    md.link_bandwidth_unidir = n > 1 ? 770e9 / (n - 1) : 770e9;
    md.links_per_gpu = n - 1;
    md.cpu_launch_overhead = 1.5e-6;
    md.dma_sync_overhead = 3.36e-5;
    c3sim::validate(md);
    return md;
}

// Placeholder interference tables until measured B200 tables are loaded:
// GEMMs scale with SMs (compute-bound: C/c; memory-bound saturating at C/2),
// collectives use the reference's bandwidth-proportional default.
c3sim::SlowdownTableSet default_tables(const c3sim::MachineDescriptor& md) {
    c3sim::SlowdownTableSet t;
    const int C = md.cus_per_gpu, g = md.min_cu_grain;
    auto& cb = t.at(c3sim::KernelClass::GemmComputeBound);
    auto& mb = t.at(c3sim::KernelClass::GemmMemoryBound);
    cb.kernel_class = c3sim::KernelClass::GemmComputeBound;
    mb.kernel_class = c3sim::KernelClass::GemmMemoryBound;
    for (int c = g; c < C; c += g) {
        cb.points.push_back({c, static_cast<double>(C) / c});
        mb.points.push_back({c, std::max(1.0, 0.5 * C / c)});
    }
    cb.points.push_back({C, 1.0});
    mb.points.push_back({C, 1.0});
    t.at(c3sim::KernelClass::AllGather) = c3sim::default_comm_table(c3sim::CollectiveKind::AllGather, md);
    t.at(c3sim::KernelClass::AllToAll) = c3sim::default_comm_table(c3sim::CollectiveKind::AllToAll, md);
    return t;
}

}  // namespace

// ---------------------------------------------------------------- session

namespace {
constexpr int kRunAllRanks = 1;
// Every step advances the session's epoch by this stride, whatever its
// collective launches: a pipelined host-input step runs up to kEpochStride
// pieces, piece k of P signalling epoch base + stride - (P - 1 - k), and a
// whole-slot collective signals the top epoch. A rank that runs one
// collective and a peer that runs P pieces therefore stay consistent: the top
// epoch is only reached once every piece is done (the epoch must
// not depend on per-call arguments).
constexpr uint32_t kEpochStride = 8;
}  // namespace

struct c3_session {
    c3_world* w = nullptr;
    c3_scenario_desc d{};
    int vr = 1;             // virtual ranks held by this process
    int n = 1;              // collective ranks
    int64_t chunk = 0;      // payload / n (bytes)
    int elem = 2;           // GEMM element bytes: 2 bf16, 4 fp32 (TF32 tensor cores)
    GemmPlan gemm;
    int* gemm_counters = nullptr;
    void *a = nullptr, *b = nullptr, *c = nullptr;
    void* gemm_ws = nullptr;  // the GEMM plan's workspace (gemm_workspace_bytes: fp32 split-K, bf16 stream-K)
    // per virtual rank: AG recv (payload, own chunk in place); RS in (payload),
    // out (chunk), staging (payload)
    std::vector<void*> recv, in, out, staging;
    // multi-process peer views, indexed by rank ([rank] = local)
    void* peer_coll[C3_MAX_RANKS] = {};     // AG recv / RS in
    void* peer_staging[C3_MAX_RANKS] = {};
    uint32_t* peer_sig[C3_MAX_RANKS] = {};
    std::vector<void*> imported;            // to close on destroy
    uint32_t* sig = nullptr;                // local signal array
    uint32_t* done = nullptr;               // [0] AG counter, [1] RS counter
    uint32_t epoch = 0;                     // top epoch of the current step (multiple of kEpochStride)
    int piece_k = 0, piece_n = 1;           // piece of the collective being enqueued (make_signals)
    uint64_t step_index = 0;                // steps run (copy-engine staging parity)
    uint32_t* err_host = nullptr;           // mapped pinned word: kWait* code of an expired device wait
    uint32_t* err_dev = nullptr;            // ... its device alias
    uint64_t wait_ns = kDefaultWaitNs;      // bound of every device-side cross-rank wait
    float fused_pace = 0.0f;                // C3_FUSED: copies finish by this share of the GEMM (0 = unpaced)
    int64_t fused_piece = 0;                // C3_FUSED: bytes per bulk copy; 0 = per collective (AG 8 KiB, A2A 16 KiB)
    int fused_mode = 0;                     // C3_FUSED: 0 TMA bulk copies, 1 LSU vectors
    double link_gbps = 0.0;                 // link emulation: peer-traffic budget per step (0 = off)
    double run_gbps = 0.0;                  // this run's pacing: link rate, or a concurrent run's comm pace
    bool solo_comm = false;                 // this run's collective has the GPU to itself (no GEMM beside it)
    c3_barrier_fn barrier = nullptr;        // host barrier across ranks (copy-engine path)
    void* barrier_ctx = nullptr;
    bool ready = false;                     // peers imported (or loopback)
    std::vector<c3_transfer> plan;          // validated ConCCL plan
    // host-staged copy-engine proxy (loopback, c3_session_set_ce_proxy): the
    // DMA backend's peers are pinned host buffers, one chunk each: the peer's
    // own data (source of its inbound copies) and what this rank sends it
    bool ce_proxy = false;
    void* proxy_send[C3_MAX_RANKS] = {};
    void* proxy_recv[C3_MAX_RANKS] = {};
    cudaStream_t main = nullptr, gemm_s = nullptr, comm_s = nullptr, comm_hi = nullptr;
    cudaEvent_t ev_start = nullptr, ev_gs = nullptr, ev_ge = nullptr, ev_cs = nullptr,
                ev_ce = nullptr, ev_end = nullptr, ev_h2d = nullptr;
    cudaStream_t h2d_s = nullptr;             // c3_session_run_host: the host-input copies
    cudaStream_t d2h_s = nullptr;             // ... the result read-back (C), beside the collective
    cudaEvent_t ev_d2h = nullptr;
    uint32_t* a_flags = nullptr;              // ... A row bands landed (RowGate)
    uint32_t a_epoch = 0;
    cudaEvent_t ev_piece[8] = {};             // ... one per landed piece of the collective's input
    c3sim::MachineDescriptor md;
    c3sim::SlowdownTableSet tables;
    c3sim::SlowdownTableSet tables_loaded;  // as loaded (tables' comm class may come from comm_curve)
    bool tables_from_file = false;
    c3sim::CoRunPenalty penalties = c3sim::CoRunPenalty::ones();  // c3_session_load_params
    bool freeze_phase2 = false;                                      // ... its freeze_phase2_allocation
    c3sim::C3Scenario scenario;
    c3sim::CommCurve comm_curve;            // c3_session_set_comm_curve (seconds)
    bool coresident = false;                // c3_session_load_coresident: model co-residency
    c3sim::CoResidentParams cores;
};

namespace {

bool multi_process(const c3_session* s) { return !s->w->loopback && s->n > 1; }
int staging_buffers(const c3_session* s) { return multi_process(s) ? 2 : 1; }

int session_alloc(c3_session* s) {
    const c3_scenario_desc& d = s->d;
    C3_CUDA(cudaMalloc(&s->a, static_cast<size_t>(d.m * d.k * s->elem)));
    C3_CUDA(cudaMalloc(&s->b, static_cast<size_t>(d.n * d.k * s->elem)));
    C3_CUDA(cudaMalloc(&s->c, static_cast<size_t>(d.m * d.n * s->elem)));
    C3_CUDA(cudaMalloc(&s->gemm_counters, 2 * sizeof(int)));
    C3_CUDA(cudaMemset(s->gemm_counters, 0, 2 * sizeof(int)));
    const size_t ws = static_cast<size_t>(gemm_workspace_bytes(d.m, d.n, d.k, s->elem, s->w->prop.multiProcessorCount));
    if (ws > 0) {
        C3_CUDA(cudaMalloc(&s->gemm_ws, ws));
        C3_CUDA(cudaMemset(s->gemm_ws, 0,
                           static_cast<size_t>(gemm_workspace_zero_bytes(d.m, d.n, d.k, s->elem,
                                                                         s->w->prop.multiProcessorCount))));
    }
    C3_TRY(gemm_plan_init(&s->gemm, s->a, s->b, s->c, d.m, d.n, d.k, s->gemm_counters,
                          s->w->prop.multiProcessorCount, s->elem, s->gemm_ws));
    const size_t payload = static_cast<size_t>(d.payload_bytes);
    for (int v = 0; v < s->vr; ++v) {
        void* p = nullptr;
        if (d.collective == C3_ALL_GATHER) {
            C3_CUDA(cudaMalloc(&p, std::max<size_t>(payload, 16)));
            s->recv.push_back(p);
        } else if (d.collective == C3_ALL_TO_ALL) {
            C3_CUDA(cudaMalloc(&p, std::max<size_t>(payload, 16)));
            s->in.push_back(p);
            C3_CUDA(cudaMalloc(&p, std::max<size_t>(payload, 16)));
            s->recv.push_back(p);
        } else {
            C3_CUDA(cudaMalloc(&p, std::max<size_t>(payload, 16)));
            s->in.push_back(p);
            C3_CUDA(cudaMalloc(&p, std::max<size_t>(static_cast<size_t>(s->chunk), 16)));
            s->out.push_back(p);
            // multi-process copy-engine reduce-scatter: two staging buffers,
            // used by step parity, so a peer one step ahead never writes into
            // the slots this rank's local reduce is still reading
            C3_CUDA(cudaMalloc(&p, std::max<size_t>(payload * static_cast<size_t>(staging_buffers(s)), 16)));
            s->staging.push_back(p);
        }
    }
    C3_CUDA(cudaMalloc(&s->sig, kSigWords * sizeof(uint32_t)));
    C3_CUDA(cudaMemset(s->sig, 0, kSigWords * sizeof(uint32_t)));
    C3_CUDA(cudaMalloc(&s->done, 4 * sizeof(uint32_t)));  // [0] AG/A2A [1] RS [2] fused
    C3_CUDA(cudaMemset(s->done, 0, 4 * sizeof(uint32_t)));
    C3_CUDA(cudaStreamCreateWithFlags(&s->main, cudaStreamNonBlocking));
    C3_CUDA(cudaStreamCreateWithPriority(&s->gemm_s, cudaStreamNonBlocking, s->w->prio_lo));
    C3_CUDA(cudaStreamCreateWithPriority(&s->comm_s, cudaStreamNonBlocking, s->w->prio_lo));
    C3_CUDA(cudaStreamCreateWithPriority(&s->comm_hi, cudaStreamNonBlocking, s->w->prio_hi));
    for (cudaEvent_t* e : {&s->ev_start, &s->ev_gs, &s->ev_ge, &s->ev_cs, &s->ev_ce, &s->ev_end})
        C3_CUDA(cudaEventCreate(e));
    C3_CUDA(cudaEventCreateWithFlags(&s->ev_h2d, cudaEventDisableTiming));
    for (cudaEvent_t& e : s->ev_piece) C3_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    C3_CUDA(cudaStreamCreateWithFlags(&s->h2d_s, cudaStreamNonBlocking));
    C3_CUDA(cudaStreamCreateWithFlags(&s->d2h_s, cudaStreamNonBlocking));
    C3_CUDA(cudaEventCreateWithFlags(&s->ev_d2h, cudaEventDisableTiming));
    C3_CUDA(cudaMalloc(&s->a_flags, 64 * sizeof(uint32_t)));
    C3_CUDA(cudaMemset(s->a_flags, 0, 64 * sizeof(uint32_t)));
    // error word of the device-side waits: mapped pinned host memory, so the
    // host reads it after the step's event without a copy
    C3_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->err_host), 64, cudaHostAllocMapped));
    *s->err_host = 0;
    C3_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->err_dev), s->err_host, 0));
    if (const char* e = std::getenv("C3_WAIT_TIMEOUT_MS")) {
        const double ms = std::atof(e);
        if (ms > 0) s->wait_ns = static_cast<uint64_t>(ms * 1e6);
    }
    return C3_OK;
}

// What a collective launch signals across processes (collectives.cu layout).
enum class SigUse {
    Push,    // AG / A2A push: entry (receivers free) + exit (stores landed)
    Rs,      // RS pull: entry (inputs ready) + exit (inputs read)
    Fused,   // fused C3: fixed slots inside the GEMM kernel
    CeEntry, // copy-engine AG / A2A: receivers free (post + wait), before the copies
    CeDone,  // copy-engine: wait for every peer's delivery flags (written by its CE streams)
};

// Epochs of a step (kEpochStride): the step's top epoch E = s->epoch and its
// base E - stride + 1. A collective split into P pieces (host-input steps)
// runs piece k with s->piece_k = k, s->piece_n = P; a whole-slot one with
// k = 0, P = 1. Entry of a push (receivers free) happens once per step, at the
// base epoch; entry of a pull (inputs up to piece k ready) at E - (P-1-k); the
// exit barrier only at the last piece, at E. Ranks that split the same step
// differently therefore neither deadlock nor pass early.
Signals make_signals(c3_session* s, SigUse use) {
    Signals g;
    if (s->w->loopback || s->n == 1) return g;
    g.enabled = true;
    g.mine = s->sig;
    for (int p = 0; p < s->n; ++p) g.peers[p] = s->peer_sig[p];
    const uint32_t top = s->epoch, base = s->epoch - kEpochStride + 1;
    const bool first = s->piece_k == 0, last = s->piece_k == s->piece_n - 1;
    g.epoch = top;
    g.entry_epoch = base;
    g.self = s->w->rank;
    g.err = s->err_dev;
    g.timeout_ns = s->wait_ns;
    switch (use) {
        case SigUse::Push:
            g.done = s->done + 0;
            g.entry_slot = first ? kSigPushEntry : -1;
            g.exit_slot = last ? kSigPushExit : -1;
            break;
        case SigUse::Rs:
            g.done = s->done + 1;
            g.entry_slot = kSigRsEntry;
            g.entry_epoch = top - static_cast<uint32_t>(s->piece_n - 1 - s->piece_k);
            g.exit_slot = last ? kSigRsExit : -1;
            break;
        case SigUse::Fused:
            g.done = s->done + 2;
            break;
        case SigUse::CeEntry:
            g.entry_slot = kSigPushEntry;
            break;
        case SigUse::CeDone:
            g.entry_slot = kSigCeDone;
            g.entry_post = false;
            g.entry_epoch = top;
            break;
    }
    return g;
}

// Enqueue this rank's share of the collective on `st`. Returns the number of
// kernels launched via *launches. Nothing here blocks the host: every
// cross-rank dependency is a device-side flag wait (bounded, see Signals).
// `off`/`len` (CU backend only): move bytes [off, off + len) of every slot,
// the piece of a pipelined host-input step (len < 0: the whole slot).
int enqueue_collective(c3_session* s, int backend, int n_ctas, int flags, cudaStream_t st,
                       int* launches, int64_t off = 0, int64_t len = -1) {
    c3_world* w = s->w;
    const int n = s->n;
    const int64_t chunk = s->chunk;
    const int64_t plen = len < 0 ? chunk : len;
    if (backend != C3_BACKEND_CU && (off != 0 || plen != chunk))
        return set_error(C3_ERR_VALIDATION, "slot ranges are for the SM collectives only");
    const bool loop = w->loopback != 0;
    const bool all = loop && (flags & kRunAllRanks);
    const int first = loop ? 0 : w->rank;
    const int last = loop ? (all ? n - 1 : 0) : w->rank;
    if (n == 1) return C3_OK;
    // copy-engine collectives across processes: delivery flags per engine
    // stream, and (AG / A2A, which write into the peers' result buffers) an
    // entry barrier before the copies
    const Signals ce_done = make_signals(s, SigUse::CeDone);
    CeDeliver dv;
    dv.sig = &ce_done;
    const CeDeliver* deliver = ce_done.enabled ? &dv : nullptr;
    const auto ce_entry = [&]() -> int {
        const Signals e = make_signals(s, SigUse::CeEntry);
        if (!e.enabled) return C3_OK;
        C3_TRY(launch_signal_wait(e, n, st));
        ++*launches;
        return C3_OK;
    };
    const auto ce_wait_delivered = [&]() -> int {
        if (!ce_done.enabled) return C3_OK;
        C3_TRY(launch_signal_wait(ce_done, n, st));
        ++*launches;
        return C3_OK;
    };
    // host-staged proxy (rank 0's share of a loopback world): rank 0's copies
    // to peer q land in q's pinned host buffer (D2H), q's copies to rank 0 come
    // from it (H2D), so every byte of this GPU's share crosses a copy engine
    const bool proxy = loop && s->ce_proxy && !all && backend == C3_BACKEND_DMA;
    const int dst_filter = proxy ? 0 : -1;
    if (s->d.collective == C3_ALL_GATHER) {
        MutPtrTable recv{};
        std::vector<const void*> src(static_cast<size_t>(n));
        std::vector<void*> dst(static_cast<size_t>(n));
        for (int p = 0; p < n; ++p) {
            void* base = loop ? s->recv[static_cast<size_t>(p)] : s->peer_coll[p];
            recv.p[p] = base;
            dst[static_cast<size_t>(p)] = base;
            src[static_cast<size_t>(p)] = static_cast<uint8_t*>(base) + chunk * p;
        }
        if (backend == C3_BACKEND_CU) {
            const Signals sig = make_signals(s, SigUse::Push);
            for (int v = first; v <= last; ++v) {
                // the kernel writes slot v at recv[q] + plen * v: shift the bases
                // so that lands on recv[q] + chunk * v + off
                MutPtrTable r = recv;
                for (int q = 0; q < n; ++q) r.p[q] = static_cast<uint8_t*>(recv.p[q]) + (chunk - plen) * v + off;
                C3_TRY(launch_allgather_push(v, n, static_cast<uint8_t*>(recv.p[v]) + chunk * v + off, r,
                                             plen, n_ctas, sig, st, s->run_gbps, s->solo_comm));
                ++*launches;
            }
        } else {
            // plan_all_gather (conccl.cpp:24-53) on the copy engines; the step
            // ends once every peer's chunk has landed here (delivery flags)
            if (proxy)
                for (int q = 1; q < n; ++q) {
                    src[static_cast<size_t>(q)] = s->proxy_send[q];  // plan src_offset = 0
                    dst[static_cast<size_t>(q)] = s->proxy_recv[q];  // rank 0's slot: dst_offset = 0
                }
            C3_TRY(ce_entry());
            C3_TRY(ce_run(w, s->plan.data(), static_cast<int>(s->plan.size()), src.data(), dst.data(),
                          all ? -1 : first, st, deliver, dst_filter));
            C3_TRY(ce_wait_delivered());
        }
        return C3_OK;
    }
    if (s->d.collective == C3_ALL_TO_ALL) {
        MutPtrTable recv{};
        std::vector<const void*> src(static_cast<size_t>(n));
        std::vector<void*> dst(static_cast<size_t>(n));
        for (int p = 0; p < n; ++p) {
            recv.p[p] = loop ? s->recv[static_cast<size_t>(p)] : s->peer_coll[p];
            dst[static_cast<size_t>(p)] = recv.p[p];
            src[static_cast<size_t>(p)] = loop ? s->in[static_cast<size_t>(p)] : s->in[0];
        }
        if (backend == C3_BACKEND_CU) {
            const Signals sig = make_signals(s, SigUse::Push);
            MutPtrTable r = recv;
            for (int q = 0; q < n; ++q) r.p[q] = static_cast<uint8_t*>(recv.p[q]) + off;
            for (int v = first; v <= last; ++v) {
                C3_TRY(launch_alltoall_push(v, n,
                                            static_cast<const uint8_t*>(loop ? s->in[static_cast<size_t>(v)] : s->in[0]) + off,
                                            r, plen, n_ctas, sig, st, s->run_gbps, chunk));
                ++*launches;
            }
        } else {
            // plan_all_to_all (conccl.cpp:55-84) on the copy engines; the self
            // slot is a local copy, not part of the plan
            if (proxy)
                for (int q = 1; q < n; ++q) {
                    src[static_cast<size_t>(q)] = s->proxy_send[q];  // q's send slot 0 (src_offset 0)
                    dst[static_cast<size_t>(q)] = s->proxy_recv[q];  // rank 0's slot (dst_offset 0)
                }
            C3_TRY(ce_entry());
            C3_TRY(ce_run(w, s->plan.data(), static_cast<int>(s->plan.size()), src.data(), dst.data(),
                          all ? -1 : first, st, deliver, dst_filter));
            for (int v = first; v <= last; ++v) {
                const size_t lv = loop ? static_cast<size_t>(v) : 0;
                C3_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(s->recv[lv]) + chunk * v,
                                        static_cast<const uint8_t*>(s->in[lv]) + chunk * v,
                                        static_cast<size_t>(chunk), cudaMemcpyDeviceToDevice, st));
            }
            C3_TRY(ce_wait_delivered());
        }
        return C3_OK;
    }
    // reduce-scatter
    const int64_t count = chunk / 2;
    if (backend == C3_BACKEND_CU) {
        PtrTable in{};
        for (int p = 0; p < n; ++p) in.p[p] = loop ? s->in[static_cast<size_t>(p)] : s->peer_coll[p];
        const Signals sig = make_signals(s, SigUse::Rs);
        for (int v = first; v <= last; ++v) {
            // the kernel reads in[g] + plen * v: shift to in[g] + chunk * v + off
            PtrTable r = in;
            for (int g = 0; g < n; ++g) r.p[g] = static_cast<const uint8_t*>(in.p[g]) + (chunk - plen) * v + off;
            void* out = static_cast<uint8_t*>(loop ? s->out[static_cast<size_t>(v)] : s->out[0]) + off;
            C3_TRY(launch_reduce_scatter_pull(v, n, r, out, plen / 2, n_ctas, sig, st, s->run_gbps));
            ++*launches;
        }
        return C3_OK;
    }
    // copy phase: rank g's slot p -> rank p's staging slot g (plan_reduce_scatter),
    // into the staging buffer of this step's parity (multi-process)
    const int64_t par = multi_process(s) ? static_cast<int64_t>(s->step_index % 2) * s->d.payload_bytes : 0;
    std::vector<const void*> src(static_cast<size_t>(n));
    std::vector<void*> dst(static_cast<size_t>(n));
    for (int p = 0; p < n; ++p) {
        src[static_cast<size_t>(p)] = loop ? s->in[static_cast<size_t>(p)] : s->peer_coll[p];
        dst[static_cast<size_t>(p)] =
            static_cast<uint8_t*>(loop ? s->staging[static_cast<size_t>(p)] : s->peer_staging[p]) + par;
    }
    if (!loop) src[static_cast<size_t>(w->rank)] = s->in[0];
    if (proxy)
        for (int q = 1; q < n; ++q) {
            src[static_cast<size_t>(q)] = s->proxy_send[q];  // q's input slot 0 (src_offset 0)
            dst[static_cast<size_t>(q)] = s->proxy_recv[q];  // rank 0's slot (dst_offset 0)
        }
    C3_TRY(ce_run(w, s->plan.data(), static_cast<int>(s->plan.size()), src.data(), dst.data(),
                  all ? -1 : first, st, deliver, dst_filter));
    // local reduce of the n slots (own slot straight from the input); across
    // processes its CTAs first wait for every peer's delivery flag
    for (int v = first; v <= last; ++v) {
        PtrTable slots{};
        const size_t lv = loop ? static_cast<size_t>(v) : 0;
        for (int g = 0; g < n; ++g)
            slots.p[g] = g == v ? static_cast<const uint8_t*>(s->in[lv]) + chunk * v
                                : static_cast<const uint8_t*>(s->staging[lv]) + par + chunk * g;
        C3_TRY(launch_reduce_scatter_pull(0, n, slots, s->out[lv], count, std::max(1, n_ctas), ce_done, st));
        ++*launches;
    }
    return C3_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

extern "C" {

const char* c3_last_error(void) { return last_error_cstr(); }
int c3_version(void) { return 1; }

int c3_world_create(int rank, int n_ranks, int device, int loopback, c3_world** out) {
    if (!out) return set_error(C3_ERR_VALIDATION, "c3_world_create: null out");
    if (n_ranks < 1 || n_ranks > C3_MAX_RANKS)
        return set_error(C3_ERR_VALIDATION, "c3_world_create: n_ranks must be in [1, 8]");
    if (rank < 0 || rank >= n_ranks) return set_error(C3_ERR_VALIDATION, "c3_world_create: bad rank");
    auto* w = new c3_world;
    w->rank = loopback ? 0 : rank;
    w->n_ranks = n_ranks;
    w->device = device;
    w->loopback = loopback ? 1 : 0;
    const auto fail = [&](int rc) {
        delete w;
        return rc;
    };
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(set_cuda_error(e, "cudaSetDevice"));
    e = cudaGetDeviceProperties(&w->prop, device);
    if (e != cudaSuccess) return fail(set_cuda_error(e, "cudaGetDeviceProperties"));
    if (w->prop.major != 10)
        return fail(set_error(C3_ERR_UNSUPPORTED, "libc3cuda is built for sm_100a (B200); device is sm_" +
                                                      std::to_string(w->prop.major * 10 + w->prop.minor)));
    cudaDeviceGetStreamPriorityRange(&w->prio_lo, &w->prio_hi);
    if (!drv().Init || !drv().DeviceGet || drv().Init(0) != CUDA_SUCCESS ||
        drv().DeviceGet(&w->cu_dev, device) != CUDA_SUCCESS)
        return fail(set_error(C3_ERR_DRIVER, "cuInit/cuDeviceGet failed"));
    w->green_ok = probe_green(w);
    e = cudaMalloc(&w->gemm_counters, 2 * kGemmCounterSlots * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(w->gemm_counters, 0, 2 * kGemmCounterSlots * sizeof(int));
    if (e != cudaSuccess) return fail(set_cuda_error(e, "cudaMalloc(gemm counters)"));
    *out = w;
    return C3_OK;
}

int c3_world_destroy(c3_world* w) {
    if (!w) return C3_OK;
    cudaSetDevice(w->device);
    for (auto& [k, gp] : w->partitions) {
        if (gp.comm_stream && drv().StreamDestroy) drv().StreamDestroy(gp.comm_stream);
        if (gp.gemm_stream && drv().StreamDestroy) drv().StreamDestroy(gp.gemm_stream);
        if (gp.comm_ctx && drv().GreenCtxDestroy) drv().GreenCtxDestroy(gp.comm_ctx);
        if (gp.gemm_ctx && drv().GreenCtxDestroy) drv().GreenCtxDestroy(gp.gemm_ctx);
    }
    for (auto s : w->ce_streams) cudaStreamDestroy(s);
    for (auto e : w->ce_events) cudaEventDestroy(e);
    if (w->fork_event) cudaEventDestroy(w->fork_event);
    if (w->gemm_counters) cudaFree(w->gemm_counters);
    delete w;
    return C3_OK;
}

int c3_world_get_info(const c3_world* w, c3_world_info* o) {
    if (!w || !o) return set_error(C3_ERR_VALIDATION, "c3_world_get_info: null argument");
    o->rank = w->rank;
    o->n_ranks = w->n_ranks;
    o->device = w->device;
    o->loopback = w->loopback;
    o->sm_count = w->prop.multiProcessorCount;
    o->async_engines = w->prop.asyncEngineCount;
    o->l2_bytes = w->prop.l2CacheSize;
    o->cc_major = w->prop.major;
    o->cc_minor = w->prop.minor;
    o->green_ctx = w->green_ok;
    o->sm_grain = w->green_grain;
    o->stream_prio_lo = w->prio_lo;
    o->stream_prio_hi = w->prio_hi;
    return C3_OK;
}

int c3_malloc(c3_world* w, int64_t bytes, void** ptr) {
    if (!w || !ptr || bytes < 0) return set_error(C3_ERR_VALIDATION, "c3_malloc: bad argument");
    C3_CUDA(cudaSetDevice(w->device));
    C3_CUDA(cudaMalloc(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 16))));
    return C3_OK;
}

int c3_free(c3_world* w, void* ptr) {
    if (!w) return set_error(C3_ERR_VALIDATION, "c3_free: null world");
    C3_CUDA(cudaFree(ptr));
    return C3_OK;
}

int c3_memcpy(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
    if (bytes <= 0) return C3_OK;
    C3_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), static_cast<cudaMemcpyKind>(kind),
                            static_cast<cudaStream_t>(stream)));
    return C3_OK;
}

int c3_stream_sync(void* stream) {
    C3_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return C3_OK;
}

int c3_device_sync(void) {
    C3_CUDA(cudaDeviceSynchronize());
    return C3_OK;
}

int c3_ipc_export(c3_world* w, void* ptr, void* handle_out) {
    if (!w || !ptr || !handle_out) return set_error(C3_ERR_VALIDATION, "c3_ipc_export: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == C3_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    C3_CUDA(cudaIpcGetMemHandle(&h, ptr));
    std::memcpy(handle_out, &h, sizeof h);
    return C3_OK;
}

int c3_ipc_import(c3_world* w, const void* handle, void** peer_ptr) {
    if (!w || !handle || !peer_ptr) return set_error(C3_ERR_VALIDATION, "c3_ipc_import: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    C3_CUDA(cudaSetDevice(w->device));
    C3_CUDA(cudaIpcOpenMemHandle(peer_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return C3_OK;
}

int c3_ipc_close(c3_world* w, void* peer_ptr) {
    if (!w) return set_error(C3_ERR_VALIDATION, "c3_ipc_close: null world");
    C3_CUDA(cudaIpcCloseMemHandle(peer_ptr));
    return C3_OK;
}

int c3_fill_bf16(void* dst, int64_t count, uint64_t seed, int rank, int tensor, void* stream) {
    return launch_fill_bf16(dst, count, seed, rank, tensor, static_cast<cudaStream_t>(stream));
}

int c3_fill_f32(void* dst, int64_t count, uint64_t seed, int rank, int tensor, void* stream) {
    return launch_fill_f32(dst, count, seed, rank, tensor, static_cast<cudaStream_t>(stream));
}

int c3_fill_labels(void* dst, int64_t bytes, uint64_t seed, int rank, int tensor, void* stream) {
    return launch_fill_labels(dst, bytes, seed, rank, tensor, static_cast<cudaStream_t>(stream));
}

static int world_gemm(c3_world* w, const void* A, const void* B, void* C, int64_t m, int64_t n, int64_t k,
                      int max_ctas, void* stream, int elem) {
    if (!w) return set_error(C3_ERR_VALIDATION, "gemm: null world");
    GemmPlan plan;
    // round-robin claim-counter pairs: up to kGemmCounterSlots GEMMs in flight
    int* ctr = w->gemm_counters + 2 * (w->gemm_counter_next++ % kGemmCounterSlots);
    C3_CUDA(cudaSetDevice(w->device));
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    void* ws = nullptr;  // stream-ordered workspace (fp32 split-K, bf16 stream-K), zeroed, freed behind the GEMM
    if (m < 1 || n < 1 || k < 1) return set_error(C3_ERR_VALIDATION, "gemm: dimensions must be >= 1");
    const size_t bytes = static_cast<size_t>(gemm_workspace_bytes(m, n, k, elem, w->prop.multiProcessorCount));
    if (bytes > 0) {
        C3_CUDA(cudaMallocAsync(&ws, bytes, st));
        C3_CUDA(cudaMemsetAsync(
            ws, 0, static_cast<size_t>(gemm_workspace_zero_bytes(m, n, k, elem, w->prop.multiProcessorCount)), st));
    }
    int rc = gemm_plan_init(&plan, A, B, C, m, n, k, ctr, w->prop.multiProcessorCount, elem, ws);
    if (rc == C3_OK) rc = gemm_plan_launch(&plan, max_ctas, w->prop.multiProcessorCount, st);
    if (ws) cudaFreeAsync(ws, st);
    return rc;
}

int c3_gemm_bf16(c3_world* w, const void* A, const void* B, void* C, int64_t m, int64_t n,
                 int64_t k, int max_ctas, void* stream) {
    return world_gemm(w, A, B, C, m, n, k, max_ctas, stream, 2);
}

int c3_gemm_f32(c3_world* w, const void* A, const void* B, void* C, int64_t m, int64_t n, int64_t k,
                int max_ctas, void* stream) {
    return world_gemm(w, A, B, C, m, n, k, max_ctas, stream, 4);
}

int c3_allgather_p2p(c3_world* w, int self, const void* send, void* const* recv,
                     int64_t chunk_bytes, int n_ctas, void* stream) {
    if (!w || !recv) return set_error(C3_ERR_VALIDATION, "c3_allgather_p2p: null argument");
    MutPtrTable t{};
    for (int p = 0; p < w->n_ranks; ++p) t.p[p] = recv[p];
    return launch_allgather_push(self, w->n_ranks, send, t, chunk_bytes, n_ctas, Signals{},
                                 static_cast<cudaStream_t>(stream));
}

int c3_alltoall_p2p(c3_world* w, int self, const void* send, void* const* recv,
                    int64_t per_peer_bytes, int n_ctas, void* stream) {
    if (!w || !recv) return set_error(C3_ERR_VALIDATION, "c3_alltoall_p2p: null argument");
    MutPtrTable t{};
    for (int p = 0; p < w->n_ranks; ++p) t.p[p] = recv[p];
    return launch_alltoall_push(self, w->n_ranks, send, t, per_peer_bytes, n_ctas, Signals{},
                                static_cast<cudaStream_t>(stream));
}

int c3_reduce_scatter_p2p(c3_world* w, int self, const void* const* in, void* out, int64_t count,
                          int n_ctas, void* stream) {
    if (!w || !in) return set_error(C3_ERR_VALIDATION, "c3_reduce_scatter_p2p: null argument");
    PtrTable t{};
    for (int p = 0; p < w->n_ranks; ++p) t.p[p] = in[p];
    return launch_reduce_scatter_pull(self, w->n_ranks, t, out, count, n_ctas, Signals{},
                                      static_cast<cudaStream_t>(stream));
}

int c3_reduce_local_bf16(const void* const* slots, int n_slots, void* out, int64_t count, int n_ctas,
                         void* stream) {
    if (!slots || n_slots < 1 || n_slots > C3_MAX_RANKS)
        return set_error(C3_ERR_VALIDATION, "c3_reduce_local_bf16: bad slots");
    PtrTable t{};
    for (int g = 0; g < n_slots; ++g) t.p[g] = slots[g];
    return launch_reduce_scatter_pull(0, n_slots, t, out, count, n_ctas, Signals{},
                                      static_cast<cudaStream_t>(stream));
}

int c3_ce_execute(c3_world* w, const c3_transfer* t, int n_transfers, const void* const* src,
                  void* const* dst, int src_filter, void* stream) {
    if (!w || (n_transfers > 0 && (!t || !src || !dst)))
        return set_error(C3_ERR_VALIDATION, "c3_ce_execute: null argument");
    for (int i = 0; i < n_transfers; ++i)
        if (t[i].src_gpu < 0 || t[i].src_gpu >= w->n_ranks || t[i].dst_gpu < 0 ||
            t[i].dst_gpu >= w->n_ranks || t[i].length < 0 || t[i].src_offset < 0 || t[i].dst_offset < 0)
            return set_error(C3_ERR_VALIDATION, "c3_ce_execute: transfer " + std::to_string(i) + " out of range");
    return ce_run(w, t, n_transfers, src, dst, src_filter, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------- sessions

int c3_plan_transfers(int kind, int n_ranks, int64_t chunk_bytes, int dma_engines, c3_transfer* out,
                      int capacity, int* count) {
    if (!count) return set_error(C3_ERR_VALIDATION, "c3_plan_transfers: null count");
    return guarded([&] {
        c3sim::MachineDescriptor md;
        md.gpus_per_node = std::max(1, n_ranks);
        md.dma_engines_per_gpu = dma_engines;
        c3sim::TransferPlan plan;
        switch (kind) {
            case C3_ALL_GATHER: plan = c3sim::plan_all_gather(n_ranks, chunk_bytes, md); break;
            case C3_ALL_TO_ALL: plan = c3sim::plan_all_to_all(n_ranks, chunk_bytes, md); break;
            case C3_REDUCE_SCATTER: plan = c3sim::plan_reduce_scatter(n_ranks, chunk_bytes, md); break;
            default: throw c3sim::UnknownEntityError("unknown collective kind " + std::to_string(kind));
        }
        if (dma_engines < 1) throw c3sim::ValidationError("dma_engines must be >= 1");
        const c3sim::PlanCheck chk = c3sim::validate_plan(plan, md);
        if (!chk.ok) throw c3sim::ValidationError("transfer plan invalid: " + chk.error);
        *count = static_cast<int>(plan.transfers.size());
        if (out) {
            if (capacity < *count) throw c3sim::ValidationError("c3_plan_transfers: capacity too small");
            for (int i = 0; i < *count; ++i) {
                const auto& t = plan.transfers[static_cast<std::size_t>(i)];
                out[i] = {t.src_gpu, t.dst_gpu, t.src_offset, t.dst_offset, t.length, t.engine_id, t.seq};
            }
        }
        return C3_OK;
    });
}

int c3_ingest_model(int64_t hidden, int64_t ffn, int64_t tokens, int dtype_bytes, int shards,
                    c3_scenario_desc* out, int capacity, int* count) {
    if (!count) return set_error(C3_ERR_VALIDATION, "c3_ingest_model: null count");
    return guarded([&] {
        c3sim::ModelConfig cfg;
        cfg.hidden = hidden;
        cfg.ffn = ffn;
        cfg.tokens = tokens;
        cfg.dtype_bytes = dtype_bytes;
        cfg.shards = shards;
        const c3sim::ModelWorkload w = c3sim::ingest_model(cfg);
        *count = static_cast<int>(w.gemms.size());
        if (out) {
            if (capacity < *count) throw c3sim::ValidationError("c3_ingest_model: capacity too small");
            for (int i = 0; i < *count; ++i) {
                const auto& g = w.gemms[static_cast<size_t>(i)];
                c3_scenario_desc d{};
                d.m = g.m;
                d.n = g.n;
                d.k = g.k;
                d.collective = C3_ALL_GATHER;
                d.n_ranks = shards;
                d.payload_bytes = w.all_gathers.empty() ? 0 : w.all_gathers[static_cast<size_t>(i)].payload_bytes;
                out[i] = d;
            }
        }
        return C3_OK;
    });
}

int c3_session_create(c3_world* w, const c3_scenario_desc* desc, c3_session** out) {
    if (!w || !desc || !out) return set_error(C3_ERR_VALIDATION, "c3_session_create: null argument");
    const c3_scenario_desc& d = *desc;
    if (d.n_ranks != w->n_ranks)
        return set_error(C3_ERR_VALIDATION, "c3_session_create: scenario n_ranks != world n_ranks");
    if (d.collective != C3_ALL_GATHER && d.collective != C3_REDUCE_SCATTER && d.collective != C3_ALL_TO_ALL)
        return set_error(C3_ERR_UNKNOWN, "c3_session_create: unknown collective kind");
    if (d.payload_bytes < 0 || d.payload_bytes % d.n_ranks)
        return set_error(C3_ERR_VALIDATION, "collective: payload_bytes must be divisible by n_ranks");
    if (d.collective == C3_REDUCE_SCATTER && (d.payload_bytes / d.n_ranks) % 2)
        return set_error(C3_ERR_VALIDATION, "reduce-scatter: per-rank slot must hold whole bf16 elements");
    if (d.dtype_bytes != 0 && d.dtype_bytes != 2 && d.dtype_bytes != 4)
        return set_error(C3_ERR_VALIDATION, "c3_session_create: dtype_bytes must be 2 (bf16) or 4 (fp32)");
    auto* s = new c3_session;
    s->elem = d.dtype_bytes == 4 ? 4 : 2;
    s->w = w;
    s->d = d;
    s->n = d.n_ranks;
    s->vr = w->loopback ? d.n_ranks : 1;
    s->chunk = d.payload_bytes / d.n_ranks;
    const auto fail = [&](int rc) {
        c3_session_destroy(s);
        return rc;
    };
    cudaSetDevice(w->device);
    int rc = session_alloc(s);
    if (rc != C3_OK) return fail(rc);
    rc = guarded([&] {
        s->md = b200_machine(w, s->n);
        s->tables = default_tables(s->md);
        c3sim::C3Scenario& sc = s->scenario;
        sc.id = "session";
        sc.gemm.tag = "gemm";
        sc.gemm.m = d.m;
        sc.gemm.n = d.n;
        sc.gemm.k = d.k;
        sc.gemm.dtype_bytes = s->elem;
        sc.collective.kind = d.collective == C3_ALL_GATHER   ? c3sim::CollectiveKind::AllGather
                             : d.collective == C3_ALL_TO_ALL ? c3sim::CollectiveKind::AllToAll
                                                             : c3sim::CollectiveKind::ReduceScatter;
        sc.collective.payload_bytes = d.payload_bytes;
        sc.collective.n_ranks = d.n_ranks;
        if (s->n > 1 && s->chunk > 0) {  // nothing to plan for an empty payload
            const c3sim::TransferPlan tp =
                d.collective == C3_ALL_GATHER   ? c3sim::plan_all_gather(s->n, s->chunk, s->md)
                : d.collective == C3_ALL_TO_ALL ? c3sim::plan_all_to_all(s->n, s->chunk, s->md)
                                                : c3sim::plan_reduce_scatter(s->n, s->chunk, s->md);
            const c3sim::PlanCheck chk = c3sim::validate_plan(tp, s->md);
            if (!chk.ok) throw c3sim::ValidationError("transfer plan invalid: " + chk.error);
            for (const auto& t : tp.transfers)
                s->plan.push_back({t.src_gpu, t.dst_gpu, t.src_offset, t.dst_offset, t.length,
                                   t.engine_id, t.seq});
        }
        return C3_OK;
    });
    if (rc != C3_OK) return fail(rc);
    if (w->loopback || s->n == 1) {
        s->ready = true;
        if (!w->loopback) {
            s->peer_coll[0] = d.collective == C3_REDUCE_SCATTER ? s->in[0] : s->recv[0];
            s->peer_sig[0] = s->sig;
        }
    }
    *out = s;
    return C3_OK;
}

int c3_session_destroy(c3_session* s) {
    if (!s) return C3_OK;
    cudaSetDevice(s->w->device);
    cudaDeviceSynchronize();
    for (void* p : s->imported) cudaIpcCloseMemHandle(p);
    for (auto* v : {&s->recv, &s->in, &s->out, &s->staging})
        for (void* p : *v) cudaFree(p);
    for (void* p : {s->a, s->b, s->c, s->gemm_ws, static_cast<void*>(s->sig),
                    static_cast<void*>(s->done), static_cast<void*>(s->gemm_counters)})
        if (p) cudaFree(p);
    for (cudaStream_t st : {s->main, s->gemm_s, s->comm_s, s->comm_hi})
        if (st) cudaStreamDestroy(st);
    for (cudaEvent_t e : s->ev_piece)
        if (e) cudaEventDestroy(e);
    if (s->h2d_s) cudaStreamDestroy(s->h2d_s);
    if (s->d2h_s) cudaStreamDestroy(s->d2h_s);
    if (s->ev_d2h) cudaEventDestroy(s->ev_d2h);
    if (s->a_flags) cudaFree(s->a_flags);
    if (s->err_host) cudaFreeHost(s->err_host);
    for (int q = 0; q < C3_MAX_RANKS; ++q) {
        if (s->proxy_send[q]) cudaFreeHost(s->proxy_send[q]);
        if (s->proxy_recv[q]) cudaFreeHost(s->proxy_recv[q]);
    }
    for (cudaEvent_t e : {s->ev_start, s->ev_gs, s->ev_ge, s->ev_cs, s->ev_ce, s->ev_end, s->ev_h2d})
        if (e) cudaEventDestroy(e);
    delete s;
    return C3_OK;
}

int c3_session_pointers(const c3_session* s, int v, c3_session_ptrs* o) {
    if (!s || !o) return set_error(C3_ERR_VALIDATION, "c3_session_pointers: null argument");
    if (v < 0 || v >= s->vr) return set_error(C3_ERR_VALIDATION, "c3_session_pointers: bad virtual rank");
    std::memset(o, 0, sizeof *o);
    const c3_scenario_desc& d = s->d;
    o->a = s->a;
    o->b = s->b;
    o->c = s->c;
    o->a_bytes = d.m * d.k * s->elem;
    o->b_bytes = d.n * d.k * s->elem;
    o->c_bytes = d.m * d.n * s->elem;
    const size_t sv = static_cast<size_t>(v);
    const int self = s->w->loopback ? v : s->w->rank;
    if (d.collective == C3_ALL_GATHER) {
        o->recv = s->recv[sv];
        o->recv_bytes = d.payload_bytes;
        o->send = static_cast<uint8_t*>(s->recv[sv]) + s->chunk * self;
        o->send_bytes = s->chunk;
    } else if (d.collective == C3_ALL_TO_ALL) {
        o->send = s->in[sv];
        o->send_bytes = d.payload_bytes;
        o->recv = s->recv[sv];
        o->recv_bytes = d.payload_bytes;
    } else {
        o->send = s->in[sv];
        o->send_bytes = d.payload_bytes;
        o->recv = s->out[sv];
        o->recv_bytes = s->chunk;
        o->staging = s->staging[sv];
        o->staging_bytes = d.payload_bytes;
    }
    o->virtual_ranks = s->vr;
    return C3_OK;
}

int c3_session_fill(c3_session* s, uint64_t seed) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_fill: null session");
    const c3_scenario_desc& d = s->d;
    cudaStream_t st = s->main;
    const int r0 = s->w->loopback ? 0 : s->w->rank;
    const auto fill = s->elem == 4 ? launch_fill_f32 : launch_fill_bf16;
    C3_TRY(fill(s->a, d.m * d.k, seed, r0, 0, st));
    C3_TRY(fill(s->b, d.n * d.k, seed, r0, 1, st));
    for (int v = 0; v < s->vr; ++v) {
        const int rank = s->w->loopback ? v : s->w->rank;
        const size_t sv = static_cast<size_t>(v);
        if (d.collective == C3_ALL_GATHER) {
            C3_CUDA(cudaMemsetAsync(s->recv[sv], 0, static_cast<size_t>(d.payload_bytes), st));
            C3_TRY(launch_fill_labels(static_cast<uint8_t*>(s->recv[sv]) + s->chunk * rank, s->chunk,
                                      seed, rank, 2, st));
        } else if (d.collective == C3_ALL_TO_ALL) {
            C3_CUDA(cudaMemsetAsync(s->recv[sv], 0, static_cast<size_t>(d.payload_bytes), st));
            C3_TRY(launch_fill_labels(s->in[sv], d.payload_bytes, seed, rank, 4, st));
        } else {
            C3_TRY(launch_fill_bf16(s->in[sv], d.payload_bytes / 2, seed, rank, 3, st));
        }
    }
    if (s->ce_proxy && s->chunk > 0) {
        // each proxy peer's own data (the oracle's labels / values of rank q):
        // generated on the device, staged into its pinned host buffer
        void* tmp = nullptr;
        C3_CUDA(cudaMalloc(&tmp, static_cast<size_t>(s->chunk)));
        for (int q = 1; q < s->n; ++q) {
            if (d.collective == C3_ALL_GATHER)
                C3_TRY(launch_fill_labels(tmp, s->chunk, seed, q, 2, st));
            else if (d.collective == C3_ALL_TO_ALL)
                C3_TRY(launch_fill_labels(tmp, s->chunk, seed, q, 4, st));  // q's send slot 0
            else
                C3_TRY(launch_fill_bf16(tmp, s->chunk / 2, seed, q, 3, st));  // q's input slot 0
            C3_CUDA(cudaMemcpyAsync(s->proxy_send[q], tmp, static_cast<size_t>(s->chunk), cudaMemcpyDefault, st));
            C3_CUDA(cudaStreamSynchronize(st));
            std::memset(s->proxy_recv[q], 0, static_cast<size_t>(s->chunk));
        }
        C3_CUDA(cudaFree(tmp));
    }
    C3_CUDA(cudaStreamSynchronize(st));
    return C3_OK;
}

int c3_sm_hog(c3_world* w, double ms, void* stream) {
    if (!w || !(ms > 0.0) || ms > 10000.0) return set_error(C3_ERR_VALIDATION, "c3_sm_hog: ms must be in (0, 10000]");
    C3_CUDA(cudaSetDevice(w->device));
    return launch_sm_hog(w->prop.multiProcessorCount, ms, static_cast<cudaStream_t>(stream));
}

int c3_session_set_ce_proxy(c3_session* s, int on) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_set_ce_proxy: null session");
    if (!on) {
        s->ce_proxy = false;
        return C3_OK;
    }
    if (!s->w->loopback || s->n < 2)
        return set_error(C3_ERR_VALIDATION, "c3_session_set_ce_proxy: needs a loopback world of >= 2 ranks");
    C3_CUDA(cudaSetDevice(s->w->device));
    const size_t bytes = static_cast<size_t>(std::max<int64_t>(s->chunk, 16));
    for (int q = 1; q < s->n; ++q) {
        if (!s->proxy_send[q]) C3_CUDA(cudaHostAlloc(&s->proxy_send[q], bytes, cudaHostAllocPortable));
        if (!s->proxy_recv[q]) C3_CUDA(cudaHostAlloc(&s->proxy_recv[q], bytes, cudaHostAllocPortable));
        std::memset(s->proxy_send[q], 0, bytes);  // c3_session_fill writes peer q's data
        std::memset(s->proxy_recv[q], 0, bytes);
    }
    s->ce_proxy = true;
    return C3_OK;
}

int c3_session_proxy_buffers(c3_session* s, int peer, void** host_send, void** host_recv) {
    if (!s || !host_send || !host_recv) return set_error(C3_ERR_VALIDATION, "c3_session_proxy_buffers: null argument");
    if (!s->ce_proxy || peer < 1 || peer >= s->n)
        return set_error(C3_ERR_VALIDATION, "c3_session_proxy_buffers: no proxy buffer for that peer");
    *host_send = s->proxy_send[peer];
    *host_recv = s->proxy_recv[peer];
    return C3_OK;
}

int c3_session_export(c3_session* s, void* blob) {
    if (!s || !blob) return set_error(C3_ERR_VALIDATION, "c3_session_export: null argument");
    if (s->w->loopback) return set_error(C3_ERR_VALIDATION, "c3_session_export: loopback session");
    std::memset(blob, 0, C3_SESSION_HANDLE_BYTES);
    uint8_t* b = static_cast<uint8_t*>(blob);
    void* coll = s->d.collective == C3_REDUCE_SCATTER ? s->in[0] : s->recv[0];
    C3_TRY(c3_ipc_export(s->w, coll, b));
    if (!s->staging.empty()) C3_TRY(c3_ipc_export(s->w, s->staging[0], b + C3_IPC_HANDLE_BYTES));
    C3_TRY(c3_ipc_export(s->w, s->sig, b + 2 * C3_IPC_HANDLE_BYTES));
    return C3_OK;
}

int c3_session_import(c3_session* s, const void* all) {
    if (!s || !all) return set_error(C3_ERR_VALIDATION, "c3_session_import: null argument");
    if (s->w->loopback) return set_error(C3_ERR_VALIDATION, "c3_session_import: loopback session");
    const uint8_t* b = static_cast<const uint8_t*>(all);
    for (int p = 0; p < s->n; ++p) {
        const uint8_t* blob = b + static_cast<size_t>(p) * C3_SESSION_HANDLE_BYTES;
        if (p == s->w->rank) {
            s->peer_coll[p] = s->d.collective == C3_REDUCE_SCATTER ? s->in[0] : s->recv[0];
            s->peer_staging[p] = s->staging.empty() ? nullptr : s->staging[0];
            s->peer_sig[p] = s->sig;
            continue;
        }
        void* ptr = nullptr;
        C3_TRY(c3_ipc_import(s->w, blob, &ptr));
        s->imported.push_back(ptr);
        s->peer_coll[p] = ptr;
        if (!s->staging.empty()) {
            C3_TRY(c3_ipc_import(s->w, blob + C3_IPC_HANDLE_BYTES, &ptr));
            s->imported.push_back(ptr);
            s->peer_staging[p] = ptr;
        }
        C3_TRY(c3_ipc_import(s->w, blob + 2 * C3_IPC_HANDLE_BYTES, &ptr));
        s->imported.push_back(ptr);
        s->peer_sig[p] = static_cast<uint32_t*>(ptr);
    }
    s->ready = true;
    return C3_OK;
}

int c3_session_load_tables(c3_session* s, const char* csv_path) {
    if (!s || !csv_path) return set_error(C3_ERR_VALIDATION, "c3_session_load_tables: null argument");
    return guarded([&] {
        s->tables = c3sim::load_slowdown_tables(csv_path, s->md.min_cu_grain);
        s->tables_loaded = s->tables;
        s->tables_from_file = true;
        if (!s->comm_curve.empty()) {
            const auto cls = c3sim::comm_kernel_class(s->scenario.collective.kind);
            s->tables.at(cls) = s->comm_curve.as_table(cls, s->md);
        }
        return C3_OK;
    });
}

namespace {

// Model-layer prediction of one strategy's makespan (seconds) from measured
// isolated times; see c3_session_choose.
double predict_makespan(c3_session* s, int st, double t_gemm_ms, double t_comm_cu_ms,
                        double t_comm_dma_ms) {
    c3sim::EfficiencyParams eff;
    eff.comm_launch_overhead_cu = 0.0;  // measured times include launch
    const c3sim::CoRunPenalty& pen = s->penalties;
    c3sim::C3Scenario x = s->scenario;
    x.gemm.measured_time = t_gemm_ms * 1e-3;
    x.gemm.boundedness_override =
        c3sim::classify_gemm_boundedness(s->scenario.gemm, c3sim::machine_op_to_byte(s->md));
    const bool dma = st == C3_CONCCL || st == C3_CONCCL_RP;
    x.collective.measured_time = (dma ? t_comm_dma_ms : t_comm_cu_ms) * 1e-3;
    if (st == C3_SERIAL) return (t_gemm_ms + t_comm_cu_ms) * 1e-3;
    c3sim::MachineDescriptor md = s->md;
    if (dma && s->chunk > 0) {
        // the link bandwidth at which the model's DMA work (plan_cost of the
        // ConCCL plan, conccl.cpp:200-229: per-engine FIFOs, so 7 transfers on
        // 4 engines take two transfer times; plus the reduce-scatter's local
        // reduce) reproduces the measured copy-engine time
        md.cpu_launch_overhead = 0.0;
        md.dma_sync_overhead = 0.0;
        md.link_bandwidth_unidir = 1.0;
        const c3sim::CollectiveKind kind = s->scenario.collective.kind;
        const c3sim::TransferPlan tp = kind == c3sim::CollectiveKind::AllGather
                                           ? c3sim::plan_all_gather(s->n, s->chunk, md)
                                       : kind == c3sim::CollectiveKind::AllToAll
                                           ? c3sim::plan_all_to_all(s->n, s->chunk, md)
                                           : c3sim::plan_reduce_scatter(s->n, s->chunk, md);
        const double at_unit = c3sim::plan_cost(tp, md, eff).total;  // seconds at 1 B/s
        const double fixed = kind == c3sim::CollectiveKind::ReduceScatter
                                 ? static_cast<double>(s->d.payload_bytes + s->chunk) /
                                       (eff.efficiency * md.hbm_bandwidth)
                                 : 0.0;
        const double t_dma = t_comm_dma_ms * 1e-3;
        md.link_bandwidth_unidir = at_unit / std::max(t_dma - fixed, 0.05 * t_dma);
    }
    c3sim::SimOptions opt;
    opt.freeze_phase2_allocation = s->freeze_phase2;
    return c3sim::simulate(x, static_cast<c3sim::Strategy>(st), md, s->tables, pen, eff, opt).makespan;
}

// Collective time (ms) on `ctas` CTAs given its measured full-GPU time: the
// measured comm curve's shape when set, else the loaded comm table.
double comm_ms_at(const c3_session* s, int ctas, double t_comm_cu_ms) {
    if (!s->comm_curve.empty())
        return t_comm_cu_ms * s->comm_curve.time_at(ctas) / s->comm_curve.time_at(s->md.cus_per_gpu);
    const auto cls = c3sim::comm_kernel_class(s->scenario.collective.kind);
    return t_comm_cu_ms * c3sim::slowdown_at(s->tables.at(cls), ctas);
}

// This rank's peer bytes per collective (AG / A2A pushed, RS pulled).
double peer_bytes(const c3_session* s) { return static_cast<double>(s->n - 1) * static_cast<double>(s->chunk); }

// The collective's unpaced rate in GB/s (= bytes/ns): the emulated link rate,
// else the measured full-GPU time's.
double link_rate_gbps(const c3_session* s, double t_comm_cu_ms) {
    return s->link_gbps > 0.0 ? s->link_gbps : peer_bytes(s) / (t_comm_cu_ms * 1e6);
}

// B200 co-resident prediction (include/c3sim/coresident.hpp): GEMM on all
// SMs, the SM collective on `ctas` CTAs beside it, paced to pace_gbps if > 0.
double predict_coresident(const c3_session* s, int ctas, double t_gemm_ms, double t_comm_cu_ms,
                          double pace_gbps = 0.0) {
    const auto gcls = c3sim::gemm_kernel_class(s->scenario.gemm, c3sim::machine_op_to_byte(s->md));
    const c3sim::CoResidentParams cores = s->cores.for_kind(s->scenario.collective.kind);
    const int eff = c3sim::coresident_comm_ctas(ctas, cores,
                                                c3sim::comm_kernel_class(s->scenario.collective.kind), s->n, gcls);
    double t_at = comm_ms_at(s, eff, t_comm_cu_ms);
    double t_alone = comm_ms_at(s, ctas, t_comm_cu_ms);  // after the GEMM: the same CTAs, alone
    const double link = link_rate_gbps(s, t_comm_cu_ms);
    if (pace_gbps > 0.0 && pace_gbps < link) {
        t_at = std::max(t_at, peer_bytes(s) / (pace_gbps * 1e6));
        t_alone = std::max(t_alone, peer_bytes(s) / (pace_gbps * 1e6));
    }
    // the collective's actual rate relative to its unpaced full-GPU rate: pacing
    // or too few co-resident CTAs both lower its intensity beside the GEMM
    const double ratio = std::min(1.0, t_comm_cu_ms / t_at);
    return c3sim::simulate_coresident(t_gemm_ms * 1e-3, t_at * 1e-3, t_comm_cu_ms * 1e-3, s->md.cus_per_gpu,
                                      ctas, gcls, cores, ratio, t_alone * 1e-3)
        .makespan;
}

bool is_coresident(const c3_session* s, int st, const c3_alloc* a) {
    return a && st >= C3_C3_BASE && st <= C3_C3_SP_RP && a->backend == C3_BACKEND_CU &&
           a->cus_gemm + a->cus_comm > s->md.cus_per_gpu;
}

}  // namespace

int c3_session_set_comm_curve(c3_session* s, const int* ctas, const double* ms, int n) {
    if (!s || n < 0 || (n > 0 && (!ctas || !ms)))
        return set_error(C3_ERR_VALIDATION, "c3_session_set_comm_curve: bad argument");
    return guarded([&] {
        const auto cls = c3sim::comm_kernel_class(s->scenario.collective.kind);
        if (n == 0) {
            s->comm_curve = {};
            s->tables.at(cls) = s->tables_loaded.at(cls);
            return C3_OK;
        }
        c3sim::CommCurve c;
        for (int i = 0; i < n; ++i) {
            c.ctas.push_back(ctas[i]);
            c.seconds.push_back(ms[i] * 1e-3);
        }
        c3sim::validate(c);
        s->tables.at(cls) = c.as_table(cls, s->md);
        s->comm_curve = std::move(c);
        return C3_OK;
    });
}

int c3_session_load_coresident(c3_session* s, const char* json_path) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_load_coresident: null session");
    if (!json_path) {
        s->coresident = false;
        return C3_OK;
    }
    return guarded([&] {
        s->cores = c3sim::load_coresident_params(json_path);
        s->coresident = true;
        return C3_OK;
    });
}

int c3_session_predict_alloc(c3_session* s, int strategy, const c3_alloc* alloc, double t_gemm_ms,
                             double t_comm_cu_ms, double t_comm_dma_ms, double* predicted_ms) {
    if (!s || !alloc || !predicted_ms) return set_error(C3_ERR_VALIDATION, "c3_session_predict_alloc: null argument");
    if (!is_coresident(s, strategy, alloc))
        return c3_session_predict(s, strategy, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms, predicted_ms);
    if (!(t_gemm_ms > 0 && t_comm_cu_ms > 0))
        return set_error(C3_ERR_VALIDATION, "c3_session_predict_alloc: isolated times must be positive");
    if (!s->coresident)
        return set_error(C3_ERR_VALIDATION, "c3_session_predict_alloc: co-resident allocation needs "
                                            "c3_session_load_coresident");
    return guarded([&] {
        *predicted_ms =
            predict_coresident(s, alloc->cus_comm, t_gemm_ms, t_comm_cu_ms, alloc->comm_pace_gbps) * 1e3;
        return C3_OK;
    });
}

int c3_session_load_machine(c3_session* s, const char* machine_json_path) {
    if (!s || !machine_json_path) return set_error(C3_ERR_VALIDATION, "c3_session_load_machine: null argument");
    return guarded([&] {
        const c3sim::MachineDescriptor md = c3sim::load_machine_file(machine_json_path);
        if (md.gpus_per_node != s->n)
            throw c3sim::ValidationError("machine: gpus_per_node " + std::to_string(md.gpus_per_node) +
                                         " != the session's " + std::to_string(s->n) + " ranks");
        if (md.cus_per_gpu != s->w->prop.multiProcessorCount)
            throw c3sim::ValidationError("machine: cus_per_gpu " + std::to_string(md.cus_per_gpu) +
                                         " != this device's " + std::to_string(s->w->prop.multiProcessorCount) +
                                         " SMs");
        s->md = md;
        if (!s->tables_from_file) s->tables = default_tables(s->md);
        return C3_OK;
    });
}

int c3_session_load_params(c3_session* s, const char* params_json_path) {
    if (!s || !params_json_path) return set_error(C3_ERR_VALIDATION, "c3_session_load_params: null argument");
    return guarded([&] {
        const c3sim::RunParams rp = c3sim::load_params_file(params_json_path);
        s->penalties = rp.penalties;
        // green-context partitions stay in place after the collective ends
        // (c3_rp / c3_sp_rp): the reference's freeze_phase2_allocation option
        s->freeze_phase2 = rp.freeze_phase2_allocation;
        return C3_OK;
    });
}

int c3_session_predict(c3_session* s, int strategy, double t_gemm_ms, double t_comm_cu_ms,
                       double t_comm_dma_ms, double* predicted_ms) {
    if (!s || !predicted_ms) return set_error(C3_ERR_VALIDATION, "c3_session_predict: null argument");
    if (strategy < C3_SERIAL || strategy > C3_CONCCL_RP)
        return set_error(C3_ERR_UNKNOWN, "unknown strategy " + std::to_string(strategy));
    const bool dma = strategy == C3_CONCCL || strategy == C3_CONCCL_RP;
    if (!(t_gemm_ms > 0 && t_comm_cu_ms > 0) || (dma && !(t_comm_dma_ms > 0)))
        return set_error(C3_ERR_VALIDATION, "c3_session_predict: isolated times must be positive");
    return guarded([&] {
        *predicted_ms = predict_makespan(s, strategy, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms) * 1e3;
        return C3_OK;
    });
}

// Runtime strategy heuristic: predict every strategy's makespan with the
// model layer's simulate() (sim.cpp:121-215) fed with this GPU's measured
// isolated times (GemmKernel/CollectiveOp::measured_time, workload.hpp:23,34)
// and the loaded (measured) interference tables; rp splits come from
// partition_heuristic (strategy.cpp:48-94). The DMA backend's link bandwidth
// is set so that plan_cost reproduces the measured copy-engine time. Serial
// wins when no concurrent strategy is predicted to beat it.
// a B200 co-resident pick must predict at least this much below serial
constexpr double kCoresidentMargin = 0.02;

int c3_session_choose(c3_session* s, double t_gemm_ms, double t_comm_cu_ms, double t_comm_dma_ms,
                      int allow_dma, int* strategy, c3_alloc* alloc, double* predicted_ms) {
    if (!s || !strategy || !alloc || !predicted_ms)
        return set_error(C3_ERR_VALIDATION, "c3_session_choose: null argument");
    if (!(t_gemm_ms > 0 && t_comm_cu_ms > 0))
        return set_error(C3_ERR_VALIDATION, "c3_session_choose: isolated times must be positive");
    return guarded([&] {
        const bool use_dma = allow_dma && t_comm_dma_ms > 0;
        double best = (t_gemm_ms + std::min(t_comm_cu_ms, use_dma ? t_comm_dma_ms : t_comm_cu_ms)) * 1e-3;
        const double serial = best;
        int best_st = C3_SERIAL;
        for (int st = C3_C3_BASE; st <= C3_CONCCL_RP; ++st) {
            const bool dma = st == C3_CONCCL || st == C3_CONCCL_RP;
            if (dma && !use_dma) continue;
            const double m = predict_makespan(s, st, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms);
            if (m < best) {
                best = m;
                best_st = st;
            }
        }
        // B200 co-resident candidates: GEMM on every SM, the collective on c
        // CTA units beside it, unpaced or paced to spread over 80% / 60% of
        // the GEMM (below its unpaced rate), every (c, pace) predicted jointly.
        // Among those within 1% of the best prediction the FEWEST CTAs win
        // (then the lowest prediction): extra resident CTAs cost the GEMM more
        // than the fluid model sees.
        int best_cores = 0;
        double best_pace = 0.0;
        if (s->coresident) {
            std::vector<int> cands = {8, 16, 24, 32, 48, 64};
            for (int c : s->comm_curve.ctas) cands.push_back(c);
            std::sort(cands.begin(), cands.end());
            cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
            const double link = link_rate_gbps(s, t_comm_cu_ms);
            struct Cand {
                int c;
                double pace, m;
            };
            std::vector<Cand> pred;
            double best_co = 1e300;
            // no counts below 16 unless the comm curve measured them: the curve's
            // time there is an extrapolation, and too few co-resident CTAs fall
            // behind even a paced collective's rate (size sweep, world 2)
            const int min_c = s->comm_curve.empty() ? 1 : std::min(16, s->comm_curve.ctas.front());
            for (int c : cands) {
                if (c < min_c || c >= s->md.cus_per_gpu) continue;
                pred.push_back({c, 0.0, predict_coresident(s, c, t_gemm_ms, t_comm_cu_ms)});
                for (double frac : {0.8, 0.6}) {
                    const double pace = peer_bytes(s) / (frac * t_gemm_ms * 1e6);
                    if (pace < link) pred.push_back({c, pace, predict_coresident(s, c, t_gemm_ms, t_comm_cu_ms, pace)});
                }
            }
            for (const Cand& x : pred) best_co = std::min(best_co, x.m);
            const Cand* pick = nullptr;
            for (const Cand& x : pred)  // ascending c
                if (x.m <= best_co * 1.01 && (!pick || (x.c == pick->c && x.m < pick->m))) {
                    if (pick && x.c != pick->c) break;
                    pick = &x;
                }
            // and it must beat serial by more than the co-residency model's error
            // (RMS ~4.7%): a collective that is a few % of the GEMM (full local
            // speed, small payloads) gains at most those few %, and a co-resident
            // or slow-paced collective there measured up to 6% SLOWER than serial
            // (profiles/r02p_layer_pipeline.csv, full-speed rows)
            if (pick && pick->m < best && pick->m < serial * (1.0 - kCoresidentMargin)) {
                best = pick->m;
                best_st = C3_C3_BASE;
                best_cores = pick->c;
                best_pace = pick->pace;
            }
        }
        *strategy = best_st;
        *predicted_ms = best * 1e3;
        if (best_cores) {
            alloc->cus_gemm = s->md.cus_per_gpu;
            alloc->cus_comm = best_cores;
            alloc->cus_idle = 0;
            alloc->backend = C3_BACKEND_CU;
            alloc->comm_first = 0;
            alloc->comm_pace_gbps = static_cast<float>(best_pace);
            return C3_OK;
        }
        c3sim::EfficiencyParams eff;
        eff.comm_launch_overhead_cu = 0.0;
        c3sim::C3Scenario x = s->scenario;
        x.gemm.measured_time = t_gemm_ms * 1e-3;
        x.collective.measured_time = t_comm_cu_ms * 1e-3;
        const c3sim::Allocation a =
            c3sim::allocate_cus(x, static_cast<c3sim::Strategy>(best_st), s->md, s->tables, eff);
        alloc->cus_gemm = a.cus_gemm;
        alloc->cus_comm = best_st == C3_SERIAL ? s->md.cus_per_gpu : a.cus_comm;
        alloc->cus_idle = a.cus_idle;
        alloc->backend = a.comm_backend == c3sim::CommBackend::DMA ? C3_BACKEND_DMA : C3_BACKEND_CU;
        alloc->comm_first = a.comm_first ? 1 : 0;
        alloc->comm_pace_gbps = 0.f;
        return C3_OK;
    });
}

int c3_session_autotune(c3_session* s, const int* strategies, const c3_alloc* allocs, int n,
                        int rounds, double* medians, int* best, double* best_ms) {
    if (!s || !strategies || !allocs || !medians || !best || !best_ms || n < 1 || rounds < 1)
        return set_error(C3_ERR_VALIDATION, "c3_session_autotune: bad argument");
    std::vector<std::vector<double>> t(static_cast<size_t>(n));
    // round-robin so clock drift hits all alike, starting one candidate later
    // each round: under the power cap a run's clocks depend on its predecessor
    for (int r = 0; r < rounds; ++r)
        for (int j = 0; j < n; ++j) {
            const int i = (j + r) % n;
            c3_timing tm;
            C3_TRY(c3_session_run(s, strategies[i], &allocs[i], &tm));
            t[static_cast<size_t>(i)].push_back(tm.total_ms);
        }
    *best = 0;
    *best_ms = 1e300;
    for (int i = 0; i < n; ++i) {
        auto v = t[static_cast<size_t>(i)];
        std::sort(v.begin(), v.end());
        const double med = v[v.size() / 2];
        medians[i] = med;
        if (med < *best_ms) {
            *best_ms = med;
            *best = i;
        }
    }
    return C3_OK;
}

int c3_session_set_fused_pace(c3_session* s, float pace, int piece_bytes) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_set_fused_pace: null session");
    if (piece_bytes == 0) {  // LSU mode: the copy warp's 32 lanes move 16-byte vectors
        s->fused_mode = 1;
        s->fused_pace = pace;
        return C3_OK;
    }
    s->fused_mode = 0;
    if (!(pace >= 0.f && pace <= 1.f)) return set_error(C3_ERR_VALIDATION, "pace must be in [0, 1]");
    if (piece_bytes < 16 || piece_bytes > 16384 || piece_bytes % 16)
        return set_error(C3_ERR_VALIDATION, "piece must be a multiple of 16 in [16, 16384]");
    s->fused_pace = pace;
    s->fused_piece = piece_bytes;
    return C3_OK;
}

int c3_session_set_link_rate(c3_session* s, double gbps) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_set_link_rate: null session");
    if (!(gbps >= 0.0)) return set_error(C3_ERR_VALIDATION, "link rate must be >= 0 GB/s");
    s->link_gbps = gbps;  // 1 GB/s = 1 byte/ns
    return C3_OK;
}

int c3_session_set_wait_timeout(c3_session* s, double ms) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_set_wait_timeout: null session");
    if (!(ms > 0.0)) return set_error(C3_ERR_VALIDATION, "wait timeout must be > 0 ms");
    s->wait_ns = static_cast<uint64_t>(ms * 1e6);
    return C3_OK;
}

int c3_session_set_barrier(c3_session* s, c3_barrier_fn fn, void* ctx) {
    if (!s) return set_error(C3_ERR_VALIDATION, "c3_session_set_barrier: null session");
    s->barrier = fn;
    s->barrier_ctx = ctx;
    return C3_OK;
}

int c3_session_default_alloc(c3_session* s, int strategy, c3_alloc* out) {
    if (!s || !out) return set_error(C3_ERR_VALIDATION, "c3_session_default_alloc: null argument");
    const int C = s->md.cus_per_gpu;
    if (strategy == C3_SERIAL_OVERLAP_IO) {
        *out = {C, C, 0, C3_BACKEND_CU, 0, 0.f};
        return C3_OK;
    }
    if (strategy >= C3_GEMM_ONLY) {
        *out = {C, strategy == C3_COMM_ONLY_CU ? 32 : 0, 0,
                strategy == C3_COMM_ONLY_DMA ? C3_BACKEND_DMA : C3_BACKEND_CU, 0, 0.f};
        return C3_OK;
    }
    if (strategy == C3_FUSED) {
        *out = {C, 0, 0, C3_BACKEND_TMA, 0, 0.f};
        return C3_OK;
    }
    if (strategy < C3_SERIAL || strategy > C3_CONCCL_RP)
        return set_error(C3_ERR_UNKNOWN, "unknown strategy " + std::to_string(strategy));
    return guarded([&] {
        const c3sim::Allocation a =
            c3sim::allocate_cus(s->scenario, static_cast<c3sim::Strategy>(strategy), s->md, s->tables,
                                c3sim::EfficiencyParams{});
        out->cus_gemm = a.cus_gemm;
        out->cus_comm = a.cus_comm;
        out->cus_idle = a.cus_idle;
        out->backend = a.comm_backend == c3sim::CommBackend::DMA ? C3_BACKEND_DMA : C3_BACKEND_CU;
        out->comm_first = a.comm_first ? 1 : 0;
        out->comm_pace_gbps = 0.f;
        if (strategy == C3_SERIAL) out->cus_comm = C;  // each kernel alone on the whole GPU
        return C3_OK;
    });
}

// Host buffers of c3_session_run_host: the step's inputs come from (pinned)
// host memory and its result goes back, all inside the step.
struct HostIO {
    const void* a = nullptr;     // A, M x K bf16
    const void* send = nullptr;  // this rank's collective input (c3_session_ptrs.send)
    void* out = nullptr;         // first out_bytes of C
    int64_t out_bytes = 0;
};

namespace {
// this rank's collective input in device memory (c3_session_pointers' send)
void* session_send(c3_session* s, int64_t* bytes) {
    const int self = s->w->loopback ? 0 : s->w->rank;
    if (s->d.collective == C3_ALL_GATHER) {
        *bytes = s->chunk;
        return static_cast<uint8_t*>(s->recv[0]) + s->chunk * self;
    }
    *bytes = s->d.payload_bytes;
    return s->in[0];
}

// Enqueue one H2D copy of the step's inputs on `st` (nothing if no buffer).
int h2d_a(c3_session* s, const HostIO* io, cudaStream_t st) {
    if (!io || !io->a) return C3_OK;
    C3_CUDA(cudaMemcpyAsync(s->a, io->a, static_cast<size_t>(s->d.m * s->d.k * s->elem), cudaMemcpyDefault, st));
    return C3_OK;
}
// Pieces of the collective's host input in a pipelined concurrent step: each
// piece's copy is followed by the collective on that piece while the next
// piece crosses PCIe (C3_H2D_PIECES, default 8: the last piece's collective is
// the exposed tail; 1 below 4 MiB slots). profiles/r01_e2e_pieces.txt
int h2d_pieces(const c3_session* s) {
    const char* e = std::getenv("C3_H2D_PIECES");
    const int env = e && std::atoi(e) > 0 ? std::min(std::atoi(e), static_cast<int>(kEpochStride)) : 8;
    // strided all-to-all slot ranges need 16-byte slots (launch_alltoall_push)
    if (s->d.collective == C3_ALL_TO_ALL && s->chunk % 16 != 0) return 1;
    return s->chunk >= (int64_t{4} << 20) ? env : 1;
}
void piece_range(const c3_session* s, int pieces, int k, int64_t* off, int64_t* len) {
    const int64_t pb = (s->chunk / pieces) & ~int64_t{4095};
    *off = pb * k;
    *len = k == pieces - 1 ? s->chunk - *off : pb;
}
// A in row bands (C3_H2D_A_PIECES, default 4; multiples of the pair tile's
// 256 rows): the CTA-pair GEMM starts on the first band while the rest cross
// PCIe (RowGate). 0 bands = A copied whole before the GEMM (other kernels).
int a_row_bands(const c3_session* s, int* rows_per_band) {
    // read per call (a test may change it between steps; getenv is cheap)
    const char* e = std::getenv("C3_H2D_A_PIECES");
    const int env = e && std::atoi(e) > 0 ? std::min(std::atoi(e), 32) : 4;
    const bool pair = s->gemm.kind == GemmPlan::kPair || s->gemm.kind == GemmPlan::kPair512;
    if (!pair || env < 2 || !drv().StreamWriteValue32) return 0;
    const int64_t rows = ((s->d.m + env - 1) / env + 255) / 256 * 256;
    *rows_per_band = static_cast<int>(rows);
    return static_cast<int>((s->d.m + rows - 1) / rows);
}

// bytes [off, off + len) of every slot of the collective's input
int h2d_send_piece(c3_session* s, const HostIO* io, int64_t off, int64_t len, cudaStream_t st) {
    int64_t bytes = 0;
    uint8_t* dst = static_cast<uint8_t*>(session_send(s, &bytes));
    const uint8_t* src = static_cast<const uint8_t*>(io->send);
    if (s->d.collective == C3_ALL_GATHER) {
        C3_CUDA(cudaMemcpyAsync(dst + off, src + off, static_cast<size_t>(len), cudaMemcpyDefault, st));
    } else {
        const size_t pitch = static_cast<size_t>(s->chunk);
        C3_CUDA(cudaMemcpy2DAsync(dst + off, pitch, src + off, pitch, static_cast<size_t>(len),
                                  static_cast<size_t>(s->n), cudaMemcpyDefault, st));
    }
    return C3_OK;
}

int h2d_send(c3_session* s, const HostIO* io, cudaStream_t st) {
    if (!io || !io->send) return C3_OK;
    int64_t bytes = 0;
    void* dst = session_send(s, &bytes);
    C3_CUDA(cudaMemcpyAsync(dst, io->send, static_cast<size_t>(bytes), cudaMemcpyDefault, st));
    return C3_OK;
}
int d2h_out(c3_session* s, const HostIO* io, cudaStream_t st) {
    if (!io || !io->out || io->out_bytes <= 0) return C3_OK;
    C3_CUDA(cudaMemcpyAsync(io->out, s->c, static_cast<size_t>(io->out_bytes), cudaMemcpyDefault, st));
    return C3_OK;
}
}  // namespace

namespace {
const char* wait_error_text(uint32_t code) {
    switch (code) {
        case kWaitEntry: return "a peer never reached the collective's entry barrier";
        case kWaitExit: return "a peer never finished the collective (exit barrier)";
        case kWaitCeDone: return "a peer's copy-engine deliveries never landed";
        case kWaitFusedExit: return "a peer never finished the fused collective";
        case kWaitFusedEntry: return "a peer never reached the fused collective";
        case kWaitRowGate: return "an A row band never landed (row gate)";
        default: return "a device-side wait expired";
    }
}
int check_wait_error(c3_session* s) {
    const uint32_t code = *static_cast<volatile uint32_t*>(s->err_host);
    if (code == 0) return C3_OK;
    *static_cast<volatile uint32_t*>(s->err_host) = 0;
    // drain the copies so nothing still reads the caller's host buffers
    cudaStreamSynchronize(s->h2d_s);
    for (cudaStream_t st : s->w->ce_streams) cudaStreamSynchronize(st);
    return set_error(C3_ERR_TIMEOUT, std::string("c3_session_run: ") + wait_error_text(code) + " (epoch " +
                                         std::to_string(s->epoch) + ", bound " + std::to_string(s->wait_ns / 1000000) +
                                         " ms)");
}
}  // namespace

static int session_run_impl(c3_session* s, int strategy, const c3_alloc* alloc_in, int flags,
                            c3_timing* t, const HostIO* io = nullptr) {
    if (!s->ready) return set_error(C3_ERR_VALIDATION, "c3_session_run: peers not imported");
    c3_alloc a;
    if (alloc_in)
        a = *alloc_in;
    else
        C3_TRY(c3_session_default_alloc(s, strategy, &a));
    c3_world* w = s->w;
    const int C = w->prop.multiProcessorCount;
    std::memset(t, 0, sizeof *t);
    s->epoch += kEpochStride;
    s->piece_k = 0;
    s->piece_n = 1;
    ++s->step_index;

    cudaStream_t gs = s->gemm_s, cs = s->comm_s;
    int gemm_ctas = std::max(1, std::min(a.cus_gemm > 0 ? a.cus_gemm : C, C));
    int comm_ctas = std::max(1, a.cus_comm > 0 ? a.cus_comm : 32);
    const bool sp = strategy == C3_C3_SP || strategy == C3_C3_SP_RP;
    const bool rp = strategy == C3_C3_RP || strategy == C3_C3_SP_RP;
    if (sp) cs = s->comm_hi;
    if (rp) {
        // the SM partition is the strategy (allocate_cus, sim.cpp:40-100): no
        // silent fallback to CTA caps, and no silent rounding of the split
        if (!w->green_ok)
            return set_error(C3_ERR_UNSUPPORTED, "c3_rp / c3_sp_rp need green contexts, unavailable on this device");
        if (w->green_grain > 0 && comm_ctas % w->green_grain != 0)
            return set_error(C3_ERR_VALIDATION, "c3_rp / c3_sp_rp: cus_comm " + std::to_string(comm_ctas) +
                                                    " is not a multiple of the green-context SM grain " +
                                                    std::to_string(w->green_grain));
        GreenPartition* gp = nullptr;
        C3_TRY(green_partition(w, comm_ctas, &gp));
        if (gp->comm_sms != comm_ctas)
            return set_error(C3_ERR_VALIDATION, "c3_rp: the driver granted " + std::to_string(gp->comm_sms) +
                                                    " SMs for a request of " + std::to_string(comm_ctas));
        gs = reinterpret_cast<cudaStream_t>(gp->gemm_stream);
        cs = reinterpret_cast<cudaStream_t>(gp->comm_stream);
        gemm_ctas = std::min(gemm_ctas, gp->gemm_sms);
        t->partition = 1;
    }
    t->gemm_ctas = gemm_ctas;
    t->comm_ctas = a.backend == C3_BACKEND_CU ? comm_ctas : 0;
    // pacing of this run's SM / fused collective: the emulated link rate, or
    // (concurrent runs) the allocation's comm pace when lower
    s->run_gbps = s->link_gbps;
    const bool serial_io = strategy == C3_SERIAL_OVERLAP_IO;
    const bool concurrent = strategy != C3_SERIAL && strategy != C3_GEMM_ONLY && !serial_io &&
                            strategy != C3_COMM_ONLY_CU && strategy != C3_COMM_ONLY_DMA;
    if (concurrent && a.comm_pace_gbps > 0.f &&
        (s->run_gbps <= 0.0 || static_cast<double>(a.comm_pace_gbps) < s->run_gbps))
        s->run_gbps = a.comm_pace_gbps;
    int launches = 0;

    if (strategy == C3_FUSED) {
        if (s->d.collective != C3_ALL_GATHER && s->d.collective != C3_ALL_TO_ALL)
            return set_error(C3_ERR_UNSUPPORTED, "fused C3 moves all-gather / all-to-all data only");
        FusedComm fc;
        fc.enabled = s->n > 1 ? 1 : 0;
        fc.kind = s->d.collective == C3_ALL_GATHER ? 0 : 1;
        fc.n = s->n;
        fc.chunk = s->chunk;
        fc.pace = s->fused_pace;
        // all-to-all moves one store per load: bigger pieces amortise the copy
        // warp's per-item cost (profiles/r01_fused_probe_ring64.txt)
        fc.piece = s->fused_piece > 0 ? s->fused_piece : (fc.kind == 0 ? 8192 : 16384);
        fc.mode = s->fused_mode;
        fc.link_bpns = s->run_gbps;
        const bool loop = w->loopback != 0;
        fc.self_begin = loop ? 0 : w->rank;
        fc.self_end = loop ? ((flags & kRunAllRanks) ? s->n : 1) : w->rank + 1;
        for (int q = 0; q < s->n; ++q) {
            const size_t lq = loop ? static_cast<size_t>(q) : 0;
            fc.dst[q] = static_cast<uint8_t*>(loop ? s->recv[lq] : s->peer_coll[q]);
            if (loop || q == w->rank) {
                fc.src[q] = fc.kind == 0 ? static_cast<const uint8_t*>(s->recv[lq]) + s->chunk * q
                                         : static_cast<const uint8_t*>(s->in[lq]);
            }
        }
        if (!loop && s->n > 1) {
            fc.sig = make_signals(s, SigUse::Fused);
        }
        t->gemm_ctas = gemm_ctas;
        C3_CUDA(cudaEventRecord(s->ev_start, s->main));
        C3_CUDA(cudaStreamWaitEvent(gs, s->ev_start, 0));
        C3_TRY(h2d_a(s, io, gs));  // the copy warp reads the send data from the first tile on
        C3_TRY(h2d_send(s, io, gs));
        C3_CUDA(cudaEventRecord(s->ev_gs, gs));
        C3_TRY(gemm_plan_launch(&s->gemm, gemm_ctas, C, gs, &fc));
        C3_CUDA(cudaEventRecord(s->ev_ge, gs));
        C3_CUDA(cudaStreamWaitEvent(s->main, s->ev_ge, 0));
        C3_TRY(d2h_out(s, io, s->main));
        C3_CUDA(cudaEventRecord(s->ev_end, s->main));
        C3_CUDA(cudaEventSynchronize(s->ev_end));
        C3_CUDA(cudaGetLastError());
        t->gemm_start_ms = t->comm_start_ms = elapsed(s->ev_start, s->ev_gs);
        t->gemm_end_ms = t->comm_end_ms = elapsed(s->ev_start, s->ev_ge);
        t->total_ms = elapsed(s->ev_start, s->ev_end);
        t->launches = 1;
        return check_wait_error(s);
    }

    C3_CUDA(cudaEventRecord(s->ev_start, s->main));
    const bool do_gemm = strategy != C3_COMM_ONLY_CU && strategy != C3_COMM_ONLY_DMA;
    const bool do_comm = strategy != C3_GEMM_ONLY;
    // loopback worlds only: over real NVLink the push is link-bound and the LSU
    // kernel is the one exercised across processes
    s->solo_comm = s->w->loopback && (strategy == C3_COMM_ONLY_CU || strategy == C3_SERIAL);
    const int backend = strategy == C3_COMM_ONLY_DMA ? C3_BACKEND_DMA
                        : strategy == C3_COMM_ONLY_CU || serial_io ? C3_BACKEND_CU
                                                                    : a.backend;
    if (serial_io) a.comm_first = 0;  // GEMM first, the collective after it
    bool gated = false;  // A arrives in row bands the GEMM waits on (RowGate)
    if (strategy == C3_SERIAL) {
        C3_CUDA(cudaStreamWaitEvent(gs, s->ev_start, 0));
        C3_TRY(h2d_a(s, io, gs));
        C3_TRY(h2d_send(s, io, gs));
        C3_CUDA(cudaEventRecord(s->ev_gs, gs));
        C3_TRY(gemm_plan_launch(&s->gemm, gemm_ctas, C, gs));
        launches += gemm_launches(s->gemm);
        C3_CUDA(cudaEventRecord(s->ev_ge, gs));
        C3_CUDA(cudaEventRecord(s->ev_cs, gs));
        C3_TRY(enqueue_collective(s, C3_BACKEND_CU, comm_ctas, flags, gs, &launches));
        C3_CUDA(cudaEventRecord(s->ev_ce, gs));
        C3_CUDA(cudaStreamWaitEvent(s->main, s->ev_ce, 0));
        C3_TRY(d2h_out(s, io, s->main));  // one stream: after everything
    } else {
        C3_CUDA(cudaStreamWaitEvent(gs, s->ev_start, 0));
        C3_CUDA(cudaStreamWaitEvent(cs, s->ev_start, 0));
        // Host inputs (c3_session_run_host) share one PCIe direction: they are
        // copied back to back on the copy stream, the first-launched kernel's
        // input first. The collective's input lands in pieces and the SM
        // collective runs per piece as it lands, so the copies overlap the GEMM
        // and the collective overlaps the remaining copies.
        const bool send_in = io && io->send && do_comm;
        const int pieces = send_in ? (backend == C3_BACKEND_CU && !serial_io ? h2d_pieces(s) : 1) : 0;
        // comm pacing spreads a device-resident collective over the GEMM; a
        // collective whose input arrives over PCIe in pieces is already spread,
        // and pacing each piece from its own start would only stretch the tail
        if (pieces > 1) s->run_gbps = s->link_gbps;
        RowGate gate;
        const int a_bands = io && io->a && do_gemm && !rp ? a_row_bands(s, &gate.rows_per_flag) : 0;
        if (a_bands > 0) {
            gate.flags = s->a_flags;
            gate.epoch = ++s->a_epoch;
            gate.timed_out = s->err_dev;
            gated = true;
        }
        if (io) {
            C3_CUDA(cudaStreamWaitEvent(s->h2d_s, s->ev_start, 0));
            const auto copy_a = [&]() -> int {
                if (!io->a) return C3_OK;
                if (a_bands > 0) {  // in row bands, each published by a flag the GEMM waits on
                    const size_t row_bytes = static_cast<size_t>(s->d.k * s->elem);
                    for (int b = 0; b < a_bands; ++b) {
                        const int64_t r0 = static_cast<int64_t>(b) * gate.rows_per_flag;
                        const int64_t nr = std::min<int64_t>(gate.rows_per_flag, s->d.m - r0);
                        C3_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(s->a) + r0 * row_bytes,
                                                static_cast<const uint8_t*>(io->a) + r0 * row_bytes,
                                                static_cast<size_t>(nr) * row_bytes, cudaMemcpyDefault, s->h2d_s));
                        C3_CU(StreamWriteValue32, reinterpret_cast<CUstream>(s->h2d_s),
                              reinterpret_cast<CUdeviceptr>(s->a_flags + b), gate.epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
                    }
                    return C3_OK;
                }
                C3_TRY(h2d_a(s, io, s->h2d_s));
                C3_CUDA(cudaEventRecord(s->ev_h2d, s->h2d_s));
                C3_CUDA(cudaStreamWaitEvent(gs, s->ev_h2d, 0));
                return C3_OK;
            };
            const auto copy_send = [&]() -> int {
                for (int k = 0; k < pieces; ++k) {
                    int64_t off = 0, len = 0;
                    piece_range(s, pieces, k, &off, &len);
                    C3_TRY(h2d_send_piece(s, io, off, len, s->h2d_s));
                    C3_CUDA(cudaEventRecord(s->ev_piece[k], s->h2d_s));
                }
                return C3_OK;
            };
            if (a.comm_first) {
                C3_TRY(copy_send());
                C3_TRY(copy_a());
            } else {
                C3_TRY(copy_a());
                C3_TRY(copy_send());
            }
        }
        const auto launch_gemm = [&]() -> int {
            C3_CUDA(cudaEventRecord(s->ev_gs, gs));
            if (do_gemm) {
                C3_TRY(gemm_plan_launch(&s->gemm, gemm_ctas, C, gs, nullptr, a_bands > 0 ? &gate : nullptr));
                launches += gemm_launches(s->gemm);
            }
            C3_CUDA(cudaEventRecord(s->ev_ge, gs));
            return C3_OK;
        };
        const auto launch_comm = [&]() -> int {
            if (pieces > 0) C3_CUDA(cudaStreamWaitEvent(cs, s->ev_piece[0], 0));
            if (serial_io) C3_CUDA(cudaStreamWaitEvent(cs, s->ev_ge, 0));  // kernels in sequence
            C3_CUDA(cudaEventRecord(s->ev_cs, cs));
            if (do_comm && pieces > 1) {
                for (int k = 0; k < pieces; ++k) {
                    int64_t off = 0, len = 0;
                    piece_range(s, pieces, k, &off, &len);
                    if (k > 0) C3_CUDA(cudaStreamWaitEvent(cs, s->ev_piece[k], 0));
                    // every piece is one collective across the ranks (epochs: make_signals)
                    s->piece_k = k;
                    s->piece_n = pieces;
                    C3_TRY(enqueue_collective(s, backend, comm_ctas, flags, cs, &launches, off, len));
                }
            } else if (do_comm) {
                C3_TRY(enqueue_collective(s, backend, comm_ctas, flags, cs, &launches));
            }
            C3_CUDA(cudaEventRecord(s->ev_ce, cs));
            return C3_OK;
        };
        if (a.comm_first) {
            C3_TRY(launch_comm());
            C3_TRY(launch_gemm());
        } else {
            C3_TRY(launch_gemm());
            C3_TRY(launch_comm());
        }
        C3_CUDA(cudaStreamWaitEvent(s->main, s->ev_ge, 0));
        C3_CUDA(cudaStreamWaitEvent(s->main, s->ev_ce, 0));
        if (io && io->out && io->out_bytes > 0) {
            // C goes back as soon as the GEMM is done, beside the collective
            C3_CUDA(cudaStreamWaitEvent(s->d2h_s, s->ev_ge, 0));
            C3_TRY(d2h_out(s, io, s->d2h_s));
            C3_CUDA(cudaEventRecord(s->ev_d2h, s->d2h_s));
            C3_CUDA(cudaStreamWaitEvent(s->main, s->ev_d2h, 0));
        }
    }
    C3_CUDA(cudaEventRecord(s->ev_end, s->main));
    C3_CUDA(cudaEventSynchronize(s->ev_end));
    C3_CUDA(cudaGetLastError());
    // a bounded device-side wait expired: a peer is dead or ran a mismatched
    // step, or (row gate) a band of A never landed
    C3_TRY(check_wait_error(s));
    (void)gated;
    t->gemm_start_ms = elapsed(s->ev_start, s->ev_gs);
    t->gemm_end_ms = elapsed(s->ev_start, s->ev_ge);
    t->comm_start_ms = elapsed(s->ev_start, s->ev_cs);
    t->comm_end_ms = elapsed(s->ev_start, s->ev_ce);
    t->total_ms = elapsed(s->ev_start, s->ev_end);
    t->launches = launches;
    return C3_OK;
}

int c3_session_run(c3_session* s, int strategy, const c3_alloc* alloc, c3_timing* out) {
    if (!s || !out) return set_error(C3_ERR_VALIDATION, "c3_session_run: null argument");
    C3_CUDA(cudaSetDevice(s->w->device));
    return session_run_impl(s, strategy, alloc, 0, out);
}

int c3_session_run_host(c3_session* s, int strategy, const c3_alloc* alloc, const void* host_a,
                        const void* host_send, void* host_out, int64_t out_bytes, c3_timing* out) {
    if (!s || !out) return set_error(C3_ERR_VALIDATION, "c3_session_run_host: null argument");
    if (out_bytes < 0 || out_bytes > s->d.m * s->d.n * s->elem || (out_bytes > 0 && !host_out))
        return set_error(C3_ERR_VALIDATION, "c3_session_run_host: out_bytes must be in [0, size of C] with a buffer");
    C3_CUDA(cudaSetDevice(s->w->device));
    HostIO io;
    io.a = host_a;
    io.send = host_send;
    io.out = host_out;
    io.out_bytes = out_bytes;
    return session_run_impl(s, strategy, alloc, 0, out, &io);
}

// Loopback parity helper: run every virtual rank's share of the collective.
int c3_session_run_all_ranks(c3_session* s, int strategy, const c3_alloc* alloc, c3_timing* out) {
    if (!s || !out) return set_error(C3_ERR_VALIDATION, "c3_session_run_all_ranks: null argument");
    C3_CUDA(cudaSetDevice(s->w->device));
    return session_run_impl(s, strategy, alloc, kRunAllRanks, out);
}

}  // extern "C"
