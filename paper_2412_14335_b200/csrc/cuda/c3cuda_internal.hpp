// Internal declarations shared by the CUDA translation units and the host
// runtime of libc3cuda.so. Nothing here crosses the C ABI.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "c3cuda.h"

namespace c3k {

// ------------------------------------------------------- driver entry points
// Resolved lazily via cudaGetDriverEntryPoint (driver.cpp); nullptr when the
// driver lacks the symbol. No link-time libcuda dependency.
struct Driver {
    PFN_cuGetErrorName_v6000 GetErrorName;
    PFN_cuInit_v2000 Init;
    PFN_cuDeviceGet_v2000 DeviceGet;
    PFN_cuDeviceGetDevResource_v12040 DeviceGetDevResource;
    PFN_cuDevSmResourceSplitByCount_v12040 DevSmResourceSplitByCount;
    PFN_cuDevResourceGenerateDesc_v12040 DevResourceGenerateDesc;
    PFN_cuGreenCtxCreate_v12040 GreenCtxCreate;
    PFN_cuGreenCtxDestroy_v12040 GreenCtxDestroy;
    PFN_cuGreenCtxStreamCreate_v12050 GreenCtxStreamCreate;
    PFN_cuStreamDestroy_v4000 StreamDestroy;
    PFN_cuStreamWriteValue32_v11070 StreamWriteValue32;
    PFN_cuStreamWaitValue32_v11070 StreamWaitValue32;
    PFN_cuTensorMapEncodeTiled_v12000 TensorMapEncodeTiled;
};
const Driver& drv();

// ----------------------------------------------------------------- errors
int set_error(int code, const std::string& msg);
const char* last_error_cstr();
int set_cuda_error(cudaError_t e, const char* what);
int set_driver_error(CUresult r, const char* what);

#define C3_TRY(expr)                   \
    do {                               \
        const int _rc = (expr);        \
        if (_rc != C3_OK) return _rc;  \
    } while (0)
#define C3_CUDA(expr)                                                   \
    do {                                                                \
        const cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::c3k::set_cuda_error(_e, #expr); \
    } while (0)
// Calls drv().fn(args...), failing cleanly when the entry point is missing.
#define C3_CU(fn, ...)                                                                  \
    do {                                                                                \
        if (!::c3k::drv().fn)                                                           \
            return ::c3k::set_error(C3_ERR_UNSUPPORTED, "driver entry point cu" #fn " missing"); \
        const CUresult _r = ::c3k::drv().fn(__VA_ARGS__);                               \
        if (_r != CUDA_SUCCESS) return ::c3k::set_driver_error(_r, "cu" #fn);           \
    } while (0)

// ------------------------------------------------------------------- GEMM
struct GemmPlan {
    enum Kind { kWide = 0, kNarrow = 1, kPair = 2, kPair512 = 3 };  // 128x256, 128x128, pair 256x256 / 256x512
    CUtensorMap map_a;     // 128-row boxes
    CUtensorMap map_b128;  // 128-row boxes (pair half tile, narrow kernel)
    CUtensorMap map_b256;  // 256-row boxes (wide kernel)
    CUtensorMap map_c;     // C stores: 32-row x 64-column boxes, 128B swizzle (pair kernels)
    // Workspace (gemm_workspace_bytes, zeroed once; the kernels leave their
    // arrival words at zero). fp32 (elem 4, gemm_f32.cu, map_a / map_b128 on the
    // raw operands): the split-K arrival words (and partials for > 2 parts).
    // bf16 single-CTA kinds: the stream-K tail's arrival words and partials for
    // up to sk_capacity tail tiles (nullptr: no stream-K).
    void* ws = nullptr;
    int sk_capacity = 0;
    int f32_splits = 1;
    void* c = nullptr;
    int* counters = nullptr;  // device [tile claims, CTA exits]; zero between launches
    int64_t m = 0, n = 0, k = 0;
    Kind kind = kWide;
    int elem = 2;  // 2: bf16 (kind::f16); 4: fp32 in/out, split-TF32 on the tensor cores
    int tiles_m = 0, tiles_n = 0, num_tiles = 0, k_blocks = 0;  // of the chosen kernel
};
// fp32 plans: split-K parts and workspace bytes
int gemm_f32_splits(int64_t m, int64_t n, int64_t k, int sm_count);
int64_t gemm_f32_workspace_bytes(int64_t m, int64_t n, int64_t k, int sm_count);
// a plan's kernel kind, and the workspace bytes its plan wants (0: none)
GemmPlan::Kind gemm_kind(int64_t m, int64_t n, int elem_bytes, int sm_count);
int64_t gemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int elem_bytes, int sm_count);
// the leading bytes of that workspace that must be zero before a plan's first
// launch (the arrival words; the partials need no initial value)
int64_t gemm_workspace_zero_bytes(int64_t m, int64_t n, int64_t k, int elem_bytes, int sm_count);
// stream-K arrival words (done, ready) for `cap` tail tiles, 256-byte aligned
inline int64_t gemm_sk_counter_bytes(int cap) { return (2 * static_cast<int64_t>(cap) * 4 + 255) / 256 * 256; }
// kernels one gemm_plan_launch issues
inline int gemm_launches(const GemmPlan&) { return 1; }
int gemm_plan_init(GemmPlan* plan, const void* A, const void* B, void* C, int64_t m, int64_t n,
                   int64_t k, int* counters, int sm_count, int elem_bytes = 2, void* ws = nullptr);
struct FusedComm;
// A rows that land while the GEMM runs (c3_session_run_host): flag[b] reaches
// `epoch` once rows [b * rows_per_flag, (b + 1) * rows_per_flag) of A are in
// device memory (a stream memop after each piece's copy). The CTA-pair GEMM's
// TMA producers wait on their tile's band before loading it.
struct RowGate {
    const uint32_t* flags = nullptr;
    uint32_t epoch = 0;
    int rows_per_flag = 0;
    uint32_t* timed_out = nullptr;  // error word: kWaitRowGate once a producer's bounded wait expired
};
int gemm_plan_launch(const GemmPlan* plan, int max_ctas, int sm_count, cudaStream_t stream,
                     const FusedComm* fc = nullptr, const RowGate* gate = nullptr);

// ------------------------------------------------------------ collectives
// Cross-process completion signalling. Every session owns a signal array of
// kSigWords u32 words; rank p's array is peer-mapped. A slot is C3_MAX_RANKS
// words, word [slot + g] is written by rank g only (st.release.sys, or a
// stream memop after a copy-engine batch) with the step's epoch; readers poll
// with ld.acquire.sys. Epochs only grow, so nothing is ever reset.
constexpr int kSigWords = 64;
constexpr int kSigPushExit = 0;    // all-gather / all-to-all push: my stores into you are done
constexpr int kSigRsEntry = 8;     // reduce-scatter pull: my input is ready
constexpr int kSigRsExit = 16;     // reduce-scatter pull: I finished reading your input
constexpr int kSigCeDone = 24;     // copy engines: my copies into your buffer have landed
constexpr int kSigPushEntry = 32;  // push / copy-engine entry: your previous result may be overwritten
constexpr int kFusedExitSlot = 40; // fused C3: my copy warps' stores into you are done
constexpr int kSigFusedEntry = 48; // fused C3 entry
// Error word codes (Signals::err, mapped host memory the host reads after a step)
constexpr uint32_t kWaitEntry = 1, kWaitExit = 2, kWaitCeDone = 3, kWaitFusedExit = 4,
                   kWaitFusedEntry = 5, kWaitRowGate = 6;
// Default bound of every device-side cross-rank wait (C3_WAIT_TIMEOUT_MS).
constexpr uint64_t kDefaultWaitNs = 2000000000ull;

// `mine` is this rank's flag array, `peers[p]` rank p's (peer-mapped). `done`
// is a device counter (one per launch site) used to elect the last CTA.
struct Signals {
    uint32_t* mine = nullptr;
    uint32_t* peers[C3_MAX_RANKS] = {};
    uint32_t* done = nullptr;
    uint32_t epoch = 0;        // exit / delivery epoch
    uint32_t entry_epoch = 0;  // entry barrier epoch
    bool enabled = false;
    int self = 0;  // this rank (the kernels' data-indexing `self` may differ: local reduce)
    // entry: wait until every peer wrote >= epoch into mine[entry_slot + p]
    // (entry_post: first post epoch into peers[p][entry_slot + self]; false =
    // wait only, for flags written by the peers' copy-engine streams).
    int entry_slot = -1;
    bool entry_post = true;
    int exit_slot = -1;  // last-CTA exit barrier slot (-1: none)
    uint32_t* err = nullptr;  // set to a kWait* code when a wait expires
    uint64_t timeout_ns = kDefaultWaitNs;
};

// Fused C3 (collective moved by the GEMM's own copy warp + TMA unit).
struct FusedComm {
    int enabled = 0;
    int kind = 0;                    // 0 all-gather, 1 all-to-all
    int n = 1;                       // ranks
    int self_begin = 0, self_end = 0;  // ranks whose share this launch moves
    int skip_self = 1;               // AG: own slot already in place
    int64_t chunk = 0;               // bytes per slot
    const uint8_t* src[C3_MAX_RANKS] = {};  // AG: rank v's own chunk; A2A: send base
    uint8_t* dst[C3_MAX_RANKS] = {};        // rank q's receive base
    float pace = 0.0f;               // finish copies by this share of the GEMM's loads (0 = unpaced)
    int64_t piece = 4096;            // bytes per bulk copy (<= 16 KiB buffer)
    int mode = 0;                    // 0: TMA bulk copies (lane 0), 1: LSU vectors (32 lanes)
    double link_bpns = 0.0;          // > 0: the launch's peer-traffic budget, bytes/ns (link emulation)
    float link_cta_bpns = 0.0f;      // per-CTA share, set by the launcher from the grid
    Signals sig;
};

struct PtrTable {
    const void* p[C3_MAX_RANKS];
};
struct MutPtrTable {
    void* p[C3_MAX_RANKS];
};

// link_bpns > 0: pace the launch's peer traffic to that many bytes/ns in total
// (= GB/s; NVLink emulation in loopback worlds, c3_session_set_link_rate).
// solo: the collective has the GPU to itself (no GEMM beside it), so an
// unpaced one on many CTAs may take the TMA bulk-copy kernel (collectives.cu).
int launch_allgather_push(int self, int n, const void* send, const MutPtrTable& recv,
                          int64_t chunk_bytes, int n_ctas, const Signals& sig,
                          cudaStream_t stream, double link_bpns = 0.0, bool solo = false);
int launch_alltoall_push(int self, int n, const void* send, const MutPtrTable& recv,
                         int64_t per_peer_bytes, int n_ctas, const Signals& sig, cudaStream_t stream,
                         double link_bpns = 0.0, int64_t stride_bytes = -1);  // stride: slot pitch (default = per_peer_bytes)
int launch_reduce_scatter_pull(int self, int n, const PtrTable& in, void* out, int64_t count,
                               int n_ctas, const Signals& sig, cudaStream_t stream,
                               double link_bpns = 0.0);
// One-thread kernel running only Signals' entry part (post and/or wait on
// entry_slot): the copy-engine path's entry barrier and its wait for the
// peers' delivery flags. Occupies one warp of one SM while it polls.
int launch_signal_wait(const Signals& sig, int n, cudaStream_t stream);
int launch_sm_hog(int sm_count, double ms, cudaStream_t stream);
// Fallback when stream memops are unavailable: store `value` into each of
// `count` (peer-mapped) words with st.release.sys, after the stream's prior work.
int launch_flag_store(uint32_t* const* words, int count, uint32_t value, cudaStream_t stream);
// fp32 buffer holding the same bf16 values widened (the fp32 GEMM's inputs)
int launch_fill_f32(void* dst, int64_t count, uint64_t seed, int rank, int tensor, cudaStream_t stream);
int launch_fill_bf16(void* dst, int64_t count, uint64_t seed, int rank, int tensor,
                     cudaStream_t stream);
int launch_fill_labels(void* dst, int64_t bytes, uint64_t seed, int rank, int tensor,
                       cudaStream_t stream);

}  // namespace c3k
