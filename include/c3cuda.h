/* c3cuda.h — C ABI of libc3cuda.so, the B200 execution layer of the C3 hot path:
 * a GEMM running concurrently with an all-gather / reduce-scatter across the
 * GPUs of one node, under the paper's strategies.
 *
 * Plain C: opaque handles, POD structs, int status codes, no exceptions and no
 * torch types across the boundary. Status codes mirror the reference error
 * taxonomy (/root/reference/proj/include/c3sim/errors.hpp:8-28): 0 ok,
 * 2 I/O, 3 unknown entity, 4 validation, 5 fit; >= 100 CUDA runtime / driver
 * failures, message in c3_last_error() (thread-local).
 *
 * Which reference interface each entry point stands in for (file:line under
 * /root/reference/proj) is given next to it. The reference never executes a
 * collective or a GEMM — it models them — so "replaces" means: this call
 * executes on B200 what that declaration describes/costs.
 *
 * Process model: one process per GPU (torchrun), or a LOOPBACK world in which
 * all n ranks are virtual and live on one device (parity tests, and the 1-GPU
 * bench, where the peers are stand-in HBM buffers and no NVLink is involved).
 * Peer memory is mapped with CUDA IPC: export a handle, exchange handles with
 * any host transport (the tests and bench use torch.distributed), import.
 */
#ifndef C3CUDA_H
#define C3CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define C3_OK 0
#define C3_ERR_IO 2
#define C3_ERR_UNKNOWN 3
#define C3_ERR_VALIDATION 4
#define C3_ERR_FIT 5
#define C3_ERR_CUDA 100
#define C3_ERR_DRIVER 101
#define C3_ERR_UNSUPPORTED 102
/* A bounded device-side cross-rank wait expired (C3_WAIT_TIMEOUT_MS, default
 * 2000): a peer process is dead or ran a mismatched step. The step's results
 * are undefined; destroy the session. */
#define C3_ERR_TIMEOUT 103

#define C3_MAX_RANKS 8
#define C3_IPC_HANDLE_BYTES 64

/* c3sim::CollectiveKind (workload.hpp:14) + the ReduceScatter extension. */
#define C3_ALL_GATHER 0
#define C3_ALL_TO_ALL 1
#define C3_REDUCE_SCATTER 2

/* c3sim::Strategy ordinals (sim.hpp:15). */
#define C3_SERIAL 0
#define C3_C3_BASE 1
#define C3_C3_SP 2
#define C3_C3_RP 3
#define C3_C3_SP_RP 4
#define C3_CONCCL 5
#define C3_CONCCL_RP 6
/* B200 extension of the DMA-offload idea (not a reference strategy): the
 * all-gather / all-to-all is moved INSIDE the CTA-pair GEMM kernel by its idle
 * warp 3 driving the SM's own TMA unit (cp.async.bulk global -> smem -> local
 * or NVLink-peer global), paced by the GEMM's load progress — no extra SMs,
 * kernels or copy-engine round trips. */
#define C3_FUSED 7
/* extra execution-only modes (not reference strategies): */
#define C3_GEMM_ONLY 100 /* isolated GEMM */
#define C3_COMM_ONLY_CU 101 /* isolated SM-driven collective */
#define C3_COMM_ONLY_DMA 102 /* isolated copy-engine collective */
/* serial kernels (GEMM, then the SM collective on the isolated run's CTAs)
 * with the host copies of c3_session_run_host overlapped as well as they can
 * be without overlapping the two kernels: A lands in row bands the GEMM waits
 * on, the collective's input crosses PCIe during the GEMM, C goes back while
 * the collective runs. The conservative serial baseline of the end-to-end
 * metric (a plain C3_SERIAL step does every copy and kernel in sequence). */
#define C3_SERIAL_OVERLAP_IO 103

/* c3sim::CommBackend (interference.hpp:14). */
#define C3_BACKEND_CU 0
#define C3_BACKEND_DMA 1
#define C3_BACKEND_TMA 2 /* C3_FUSED: the GEMM kernel's own TMA unit */

typedef struct c3_world c3_world;
typedef struct c3_session c3_session;

/* Mirror of c3sim::Transfer (conccl.hpp:15-23). */
typedef struct c3_transfer {
    int32_t src_gpu, dst_gpu;
    int64_t src_offset, dst_offset, length;
    int32_t engine_id, seq;
} c3_transfer;

typedef struct c3_world_info {
    int rank, n_ranks, device, loopback;
    int sm_count;            /* cus_per_gpu of the B200 machine descriptor */
    int async_engines;       /* dma_engines_per_gpu */
    int l2_bytes;            /* llc_capacity */
    int cc_major, cc_minor;
    int green_ctx;           /* 1 when SM partitioning via green contexts works */
    int sm_grain;            /* min_cu_grain: green-context SM split granularity */
    int stream_prio_lo, stream_prio_hi;
} c3_world_info;

/* One C3 scenario (c3sim::C3Scenario, workload.hpp:37-43), executable form:
 * GEMM C[m,n] = A[m,k] B[n,k]^T in bf16 with fp32 accumulation, plus one
 * collective of `payload_bytes` per rank (all-gather: gathered bytes;
 * all-to-all: send-buffer bytes; reduce-scatter: input bytes, bf16 elements)
 * over n_ranks. */
typedef struct c3_scenario_desc {
    int64_t m, n, k;
    int32_t collective;
    int32_t n_ranks;
    int64_t payload_bytes;
    /* GemmKernel::dtype_bytes (workload.hpp:18-25): 0 or 2 = bf16 in/out;
     * 4 = fp32 in/out on the TF32 tensor cores (configs[0]) */
    int32_t dtype_bytes;
} c3_scenario_desc;

/* c3sim::Allocation (sim.hpp:25-31), in SMs. */
typedef struct c3_alloc {
    int32_t cus_gemm, cus_comm, cus_idle;
    int32_t backend;
    int32_t comm_first;
    /* B200 extension: in a concurrent run, pace the SM (or fused) collective's
     * peer traffic to this rate in GB/s (the lower of it and the session's
     * link rate), spreading it over the GEMM instead of bursting it at link
     * speed (0 = unpaced). Isolated collective runs ignore it. */
    float comm_pace_gbps;
} c3_alloc;

/* Device-event timing of one C3 step on this rank, milliseconds from the
 * step's start event. partition: 0 none/CTA caps, 1 green contexts. */
typedef struct c3_timing {
    double gemm_start_ms, gemm_end_ms;
    double comm_start_ms, comm_end_ms;
    double total_ms;
    int32_t gemm_ctas, comm_ctas, partition, launches;
} c3_timing;

typedef struct c3_session_ptrs {
    void* a;          /* bf16 [m,k] */
    void* b;          /* bf16 [n,k] */
    void* c;          /* bf16 [m,n] */
    void* send;       /* AG: chunk bytes; RS: payload bytes (n slots) */
    void* recv;       /* AG: payload bytes (n slots); RS: payload/n bytes */
    void* staging;    /* RS copy-engine staging: payload bytes */
    int64_t a_bytes, b_bytes, c_bytes, send_bytes, recv_bytes, staging_bytes;
    int32_t virtual_ranks; /* loopback: n; else 1. ptrs above are rank 0's */
} c3_session_ptrs;

/* ---------------------------------------------------------------- errors */
const char* c3_last_error(void);
int c3_version(void);

/* ----------------------------------------------------------------- world
 * Replaces the reference's static machine model MachineDescriptor
 * (machine.hpp:13-28) with the live device: c3_world_get_info reports the
 * numbers a B200 machine file is generated from. */
int c3_world_create(int rank, int n_ranks, int device, int loopback, c3_world** out);
int c3_world_destroy(c3_world* w);
int c3_world_get_info(const c3_world* w, c3_world_info* out);
/* barrier-free device memory helpers (setup only; hot calls never allocate) */
int c3_malloc(c3_world* w, int64_t bytes, void** ptr);
int c3_free(c3_world* w, void* ptr);
int c3_memcpy(void* dst, const void* src, int64_t bytes, int kind /*cudaMemcpyKind*/, void* stream);
int c3_stream_sync(void* stream);
int c3_device_sync(void);
/* CUDA IPC mapping of a c3_malloc'ed buffer into peers. */
int c3_ipc_export(c3_world* w, void* ptr, void* handle_out);
int c3_ipc_import(c3_world* w, const void* handle, void** peer_ptr);
int c3_ipc_close(c3_world* w, void* peer_ptr);

/* --------------------------------------------------- synthetic inputs
 * Counter-hash data shared bit-for-bit with oracle/c3oracle.c. */
int c3_fill_bf16(void* dst, int64_t count, uint64_t seed, int rank, int tensor, void* stream);
int c3_fill_labels(void* dst, int64_t bytes, uint64_t seed, int rank, int tensor, void* stream);
/* fp32 buffer of the same values as c3_fill_bf16 (bf16 values widened, exact) */
int c3_fill_f32(void* dst, int64_t count, uint64_t seed, int rank, int tensor, void* stream);

/* ------------------------------------------------------------------ GEMM
 * Executes c3sim::GemmKernel (workload.hpp:18-25) whose cost
 * roofline_gemm_time (workload.hpp:62-63) models; max_ctas caps the
 * persistent grid = the GEMM's SM allocation (Allocation::cus_gemm). */
/* fp32 A, B, C on the TF32 tensor cores, split-TF32: each operand is split
 * into two TF32 numbers, x ~ hi + lo (hi = x as the tensor core reads it,
 * truncated to TF32; lo the rounded remainder), and tcgen05.mma kind::tf32
 * accumulates A_lo B_hi + A_hi B_lo + A_hi B_hi in fp32. The split happens in
 * shared memory inside the one GEMM kernel; split-K (two parts for 1024^3)
 * adds the parts in a fixed order, so results are bit-reproducible.
 * Operand error below 2^-20 |a b| per product (plain TF32: 2^-11); measured
 * GEMM error 2^-23 RMS of sum |a||b| against 2^-17 for plain TF32. A
 * stream-ordered workspace (cudaMallocAsync) holds the split-K arrival
 * words. Infinities and NaNs follow IEEE fp32 GEMM semantics (each product
 * formed once). K, N multiples of 4. */
int c3_gemm_f32(c3_world* w, const void* A, const void* B, void* C, int64_t m, int64_t n, int64_t k,
                int max_ctas, void* stream);
/* bf16 A, B, C. The result bits do not depend on max_ctas (a compute-bound
 * shape on the single-CTA kernels runs a stream-K tail decomposed by the SM
 * count, with a fixed-order fix-up); those shapes take a stream-ordered
 * workspace on `stream`. */
int c3_gemm_bf16(c3_world* w, const void* A, const void* B, void* C, int64_t m, int64_t n,
                 int64_t k, int max_ctas, void* stream);

/* ----------------------------------------------------------- collectives
 * SM-driven ("CU backend") direct algorithm over mapped peer memory.
 * recv[p] = rank p's receive base (peer-mapped, or local in loopback);
 * rank `self` writes its chunk to recv[p] + self*chunk for every p (its own
 * slot too, unless send already aliases it). n_ctas = the comm kernel's SM
 * allocation (Allocation::cus_comm). These standalone calls carry no
 * cross-rank completion signal: in a multi-process world pair them with a
 * host barrier (a c3_session's collectives signal through peer flags).
 * Replaces: CollectiveOp{AllGather} execution (workload.hpp:27-35) whose
 * wire time roofline_collective_time (workload.hpp:66-67) models. */
int c3_allgather_p2p(c3_world* w, int self, const void* send, void* const* recv,
                     int64_t chunk_bytes, int n_ctas, void* stream);
/* All-to-all, push form: slot p of `send` -> slot `self` of recv[p] (for every
 * p, including self). Executes CollectiveOp{AllToAll} (workload.hpp:27-35)
 * with plan_all_to_all's mapping (conccl.hpp:49-50). */
int c3_alltoall_p2p(c3_world* w, int self, const void* send, void* const* recv,
                    int64_t per_peer_bytes, int n_ctas, void* stream);
/* Direct reduce-scatter, pull form: out = sum_{g=0..n-1} in[g][self*count ..],
 * fp32 accumulation in rank order, one bf16 rounding. in[g] = rank g's
 * input (peer-mapped or local). Extension: no reference counterpart. */
int c3_reduce_scatter_p2p(c3_world* w, int self, const void* const* in, void* out,
                          int64_t count, int n_ctas, void* stream);
/* Local n-slot reduce (copy-engine reduce-scatter second phase). */
int c3_reduce_local_bf16(const void* const* slots, int n_slots, void* out, int64_t count,
                         int n_ctas, void* stream);
/* Copy-engine ("DMA backend", ConCCL) executor: each transfer with
 * src_gpu == src_filter (or every transfer when src_filter < 0) becomes one
 * cudaMemcpyAsync dst[t.dst_gpu]+dst_offset <- src[t.src_gpu]+src_offset on
 * the world's copy stream for t.engine_id; no SM runs a kernel for it.
 * Replaces: executing c3sim::TransferPlan (conccl.hpp:33-39) produced by
 * plan_all_gather / plan_all_to_all (conccl.hpp:44-50), whose cost plan_cost
 * (conccl.hpp:72-73) models. The plan must pass validate_plan first. */
int c3_ce_execute(c3_world* w, const c3_transfer* t, int n_transfers, const void* const* src,
                  void* const* dst, int src_filter, void* stream);

/* The ConCCL plan itself, from the product model layer (libc3sim): the
 * reference plan_all_gather / plan_all_to_all (conccl.hpp:44-50) plus the
 * reduce-scatter copy phase, validated with validate_plan (conccl.hpp:60)
 * before it is returned. out may be NULL to query *count. */
int c3_plan_transfers(int kind, int n_ranks, int64_t chunk_bytes, int dma_engines,
                      c3_transfer* out, int capacity, int* count);

/* One transformer layer as C3 scenarios, from the product model layer's
 * ingest_model (workload.hpp:80-94): the layer's forward GEMMs (qkv, attn
 * out, gate+up, down) each with the FSDP all-gather of its weight as payload
 * (0 when shards == 1). out may be NULL to query *count. */
int c3_ingest_model(int64_t hidden, int64_t ffn, int64_t tokens, int dtype_bytes, int shards,
                    c3_scenario_desc* out, int capacity, int* count);

/* ------------------------------------------------------------ C3 runtime
 * A session owns one scenario's operands and executes it under a strategy.
 * Replaces (executes) c3sim::simulate (sim.hpp:70-73) for the strategy the
 * reference's allocate_cus (sim.hpp:38-40) describes; alloc == NULL means
 * "use the model's own allocation for this machine". */
int c3_session_create(c3_world* w, const c3_scenario_desc* desc, c3_session** out);
int c3_session_destroy(c3_session* s);
int c3_session_pointers(const c3_session* s, int virtual_rank, c3_session_ptrs* out);
int c3_session_fill(c3_session* s, uint64_t seed);
/* multi-process: export this rank's recv/send/staging/signal handles
 * (C3_SESSION_HANDLE_BYTES), then import every rank's blob (rank order). */
#define C3_SESSION_HANDLE_BYTES (4 * C3_IPC_HANDLE_BYTES)
int c3_session_export(c3_session* s, void* blob_out);
int c3_session_import(c3_session* s, const void* all_blobs);
/* Host-staged copy-engine proxy (loopback worlds of >= 2 ranks; one-GPU
 * measurement of the ConCCL path): every peer's buffers of the DMA backend
 * become pinned host memory, so this GPU's share of the copy-engine
 * collective -- its n-1 outgoing transfers (D2H) and the n-1 incoming ones
 * (H2D, on a second bank of engine streams) -- runs on the copy engines over
 * PCIe instead of as same-device SM copies. Per-GPU HBM
 * traffic is the real node's; the rate is PCIe's, not NVLink's. Applies to the
 * plain c3_session_run (this rank's share), DMA strategies only; peer q's
 * host buffers (chunk bytes each: its own data, filled by c3_session_fill,
 * and what this rank sent it) are returned by c3_session_proxy_buffers. */
int c3_session_set_ce_proxy(c3_session* s, int on);
int c3_session_proxy_buffers(c3_session* s, int peer, void** host_send, void** host_recv);
/* Diagnostic: occupy every SM with one spinning CTA (most of its shared
 * memory, so nothing else fits beside it) for `ms` milliseconds on `stream`:
 * work that still completes meanwhile needs no SM (copy-engine proof). */
int c3_sm_hog(c3_world* w, double ms, void* stream);
/* One C3 step (synchronous on the host at the end; device-event timed). */
int c3_session_run(c3_session* s, int strategy, const c3_alloc* alloc, c3_timing* out);
/* One C3 step on HOST buffers (the end-to-end call): the step's inputs are
 * copied in from host memory (pinned for overlap) and the first `out_bytes`
 * of C copied back, all inside the step and its timing. `host_a` is A
 * (M x K bf16), `host_send` this rank's collective input (the `send` /
 * `send_bytes` of c3_session_pointers); either may be NULL to keep the device
 * contents. Concurrent strategies copy the first-launched kernel's input
 * first and overlap the second copy with that kernel; serial and fused copy
 * both before the GEMM. C (up to out_bytes) goes back once the GEMM ends: on
 * its own stream beside the collective for concurrent strategies and
 * C3_SERIAL_OVERLAP_IO, after everything for C3_SERIAL. */
int c3_session_run_host(c3_session* s, int strategy, const c3_alloc* alloc, const void* host_a,
                        const void* host_send, void* host_out, int64_t out_bytes, c3_timing* out);
/* Loopback parity form: every virtual rank's share of the collective runs (the
 * plain call runs rank 0's share only, the per-GPU load of a real world). */
int c3_session_run_all_ranks(c3_session* s, int strategy, const c3_alloc* alloc, c3_timing* out);
/* Cross-rank completion is device-side for every backend: the SM
 * collectives signal through peer flag words; the copy-engine collectives
 * (conccl / conccl_rp) write a delivery flag into each destination rank's
 * signal words from every engine stream after its copies (stream memop), and
 * the receiver waits on the device (a one-warp kernel, or the reduce-scatter's
 * local reduce) — nothing blocks the host, so the GEMM is launched at once.
 * All-gather / all-to-all (SM, fused or copy-engine) first pass an entry
 * barrier: no rank writes into a peer's receive buffer before that peer has
 * entered the same step. The copy-engine reduce-scatter stages into two
 * buffers by step parity. Every wait is bounded (c3_session_set_wait_timeout;
 * C3_ERR_TIMEOUT). c3_session_set_barrier is kept for source compatibility:
 * the callback is no longer called. */
typedef int (*c3_barrier_fn)(void* ctx);
/* C3_FUSED pacing: the copies of each CTA finish after this share of the
 * GEMM's operand loads (default 0 = as fast as possible); piece_bytes =
 * bytes per bulk copy (16..16384, multiple of 16, at most half the copy
 * ring: 64 KiB beside the 512-wide GEMM, 16 KiB beside the 256-wide one;
 * loads run ahead of stores). Default: 8 KiB for all-gather, 16 KiB for
 * all-to-all. piece_bytes = 0
 * selects the LSU mode instead: the copy warp's 32 lanes move 16-byte vectors
 * with plain loads/stores, leaving the TMA unit to the GEMM (pace unused). */
int c3_session_set_fused_pace(c3_session* s, float pace, int piece_bytes);
/* Link-rate emulation (for loopback worlds, where the "peers" are local HBM
 * buffers and no NVLink limits the collective): pace this rank's peer traffic
 * per step to `gbps` GB/s (per direction), e.g. 770 for one B200's measured
 * NVLink 5 peer bandwidth. Applies to the SM collectives (AG/A2A push bytes,
 * RS pulled bytes) and to C3_FUSED's copy warps; each CTA waits on the global
 * timer, so the collective's time does not depend on SM clocks or CTA count
 * (given enough CTAs to reach the rate). 0 = off (default). Copy-engine
 * transfers are not paced. */
int c3_session_set_link_rate(c3_session* s, double gbps);
int c3_session_set_barrier(c3_session* s, c3_barrier_fn fn, void* ctx);
/* Bound of every device-side cross-rank wait of this session, in ms
 * (default 2000, or C3_WAIT_TIMEOUT_MS). */
int c3_session_set_wait_timeout(c3_session* s, double ms);
/* Runtime heuristic (the paper's strategy choice, on the product model layer):
 * load measured interference tables (reference SlowdownTable CSV,
 * interference.hpp:57-61; data/b200-*-slowdown-tables.csv), then predict every
 * strategy with simulate() (sim.hpp:70-73) from this GPU's measured isolated
 * times and return the fastest (serial if nothing beats it) with its
 * allocation. allow_dma = 0 excludes conccl/conccl_rp (e.g. loopback worlds,
 * where same-device copies are SM copies). */
int c3_session_load_tables(c3_session* s, const char* csv_path);
/* Machine descriptor for the predictor from a reference-format machine JSON
 * (machine.hpp:13-41, load_machine_file), e.g. data/b200-node-n8.json written
 * by tools/make_machine.py from measured peaks and copy-engine overheads;
 * gpus_per_node must equal the session's ranks and cus_per_gpu the SM count.
 * Default: the same B200 figures built in. */
int c3_session_load_machine(c3_session* s, const char* machine_json_path);
/* Co-run penalties for the predictor from a params JSON (params_io.hpp:18-19),
 * e.g. data/b200-loopback-params.json fitted by `c3sim calibrate` on measured
 * B200 speedups (tools/calibrate_penalties.py). Default: unit penalties. */
int c3_session_load_params(c3_session* s, const char* params_json_path);
int c3_session_choose(c3_session* s, double t_gemm_ms, double t_comm_cu_ms, double t_comm_dma_ms,
                      int allow_dma, int* strategy, c3_alloc* alloc, double* predicted_ms);
/* The model's predicted makespan of one strategy (same inputs as choose). */
int c3_session_predict(c3_session* s, int strategy, double t_gemm_ms, double t_comm_cu_ms,
                       double t_comm_dma_ms, double* predicted_ms);
/* B200 extension: co-residency in the model (include/c3sim/coresident.hpp).
 * set_comm_curve: the collective's measured isolated time (ms) at each CTA
 * count (strictly increasing), under this world's real or emulated link rate;
 * it replaces the collective's slowdown table in every prediction (n = 0
 * restores the loaded table). load_coresident: co-residency penalties JSON
 * ({"gemm-compute-bound", "gemm-memory-bound", "comm"}; fitted by
 * tools/calibrate_coresident.py, e.g. data/b200-coresident.json); once loaded,
 * c3_session_choose also predicts the co-resident execution (GEMM on every SM,
 * the SM collective on c CTAs beside it) for c in {8,16,24,32,48,64} and the
 * curve's points, and returns it as C3_C3_BASE (GEMM launched first, the
 * collective's CTAs beside it) with cus_gemm = all SMs, cus_comm = c when it
 * is fastest and predicts at least 2% below serial (the co-residency model's
 * error; a smaller predicted gain keeps serial). NULL path disables. */
int c3_session_set_comm_curve(c3_session* s, const int* ctas, const double* ms, int n);
int c3_session_load_coresident(c3_session* s, const char* json_path);
/* Prediction for an explicit allocation: co-resident allocations (CU backend,
 * cus_gemm + cus_comm > SMs) use the co-resident model, others as
 * c3_session_predict. */
int c3_session_predict_alloc(c3_session* s, int strategy, const c3_alloc* alloc, double t_gemm_ms,
                             double t_comm_cu_ms, double t_comm_dma_ms, double* predicted_ms);
/* Measured refinement: run each (strategy, alloc) candidate `rounds` times in
 * round-robin order; medians[i] = candidate i's median step time, *best =
 * this rank's fastest. Multi-process: every rank must pass the same
 * candidates (the runs are collective) and must pick from the max over ranks
 * of `medians`, not from its local *best. */
int c3_session_autotune(c3_session* s, const int* strategies, const c3_alloc* allocs, int n,
                        int rounds, double* medians, int* best, double* best_ms);
/* The allocation c3_session_run uses for (strategy, alloc == NULL). */
int c3_session_default_alloc(c3_session* s, int strategy, c3_alloc* out);

#ifdef __cplusplus
}
#endif
#endif /* C3CUDA_H */
