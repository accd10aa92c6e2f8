/* c3oracle — CPU restatement of the C3 hot path's data semantics.
 *
 * TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or as the timed CPU baseline — never as a product code path.
 *
 * What it restates (reference file:line, paths relative to /root/reference):
 *   - byte labels and plan replay: the ByteOracle of proj/tests/test_conccl.cpp:18-70
 *     (label = f(rank, offset), pre-seeded resident slot, byte-written-twice check,
 *     post-state check against the collective definition);
 *   - all-gather / all-to-all transfer semantics: proj/src/conccl.cpp:24-84;
 *   - reduce-scatter (not in the reference): out_r = sum over
 *     g = 0..n-1 of in_g[slot r], fp32 accumulation in fixed rank order, one
 *     rounding to bf16 (round-to-nearest-even);
 *   - GEMM: C[i,j] = sum_k A[i,k] * B[j,k] with fp64 accumulation (B stored
 *     [N,K], K-major, the weight layout of y = x W^T), SURVEY.md §8(c) "GEMM
 *     numerics" — parity for the GEMM is against this definition (the reference
 *     has no GEMM execution, so GEMM parity is "unpinned" w.r.t. reference
 *     vectors; the data-movement semantics are pinned by the reference's own
 *     ByteOracle and validate_plan, see tests/test_oracle.py).
 *   - synthetic inputs: counter-based hash of (seed, rank, tensor, index) so the
 *     CUDA side regenerates bit-identical data (fill kernels in
 *     paper_2412_14335_b200/csrc/cuda/collectives.cu).
 */
#ifndef C3ORACLE_H
#define C3ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirror of c3sim::Transfer (proj/include/c3sim/conccl.hpp:15-23). */
typedef struct c3o_transfer {
    int32_t src_gpu, dst_gpu;
    int64_t src_offset, dst_offset, length;
    int32_t engine_id, seq;
} c3o_transfer;

/* Counter hash shared bit-for-bit with the CUDA fill kernels. */
uint64_t c3o_hash64(uint64_t x);
/* 8-byte label word for (seed, rank, tensor, word index). */
uint64_t c3o_label_word(uint64_t seed, int rank, int tensor, uint64_t word);
/* Fill `bytes` bytes (multiple of 8 not required) with labels. */
void c3o_fill_labels(void* buf, int64_t bytes, uint64_t seed, int rank, int tensor);
/* bf16 synthetic value U(-1,1)*2^-3 for element `idx`, as raw bits. */
uint16_t c3o_bf16_value(uint64_t seed, int rank, int tensor, uint64_t idx);
void c3o_fill_bf16(uint16_t* buf, int64_t count, uint64_t seed, int rank, int tensor);
float c3o_bf16_to_f32(uint16_t b);
uint16_t c3o_f32_to_bf16_rne(float f);

/* Execute a transfer plan with memcpy over n host "rank" buffers
 * (dst[t.dst_gpu] + dst_offset <- src[t.src_gpu] + src_offset).
 * Returns 0, or -1 on an out-of-range transfer. */
int c3o_replay_plan(const c3o_transfer* t, int n_transfers, int n_ranks,
                    void* const* src, int64_t src_bytes, void* const* dst, int64_t dst_bytes);

/* ByteOracle (test_conccl.cpp:18-70) on 64-bit labels: returns 0 when the plan
 * realises the collective (kind 0 = all-gather, 1 = all-to-all / reduce-scatter
 * copy phase), else a positive code and a message in `why` (may be NULL).
 * 1 rank out of range, 2 source out of range, 3 destination out of range,
 * 4 byte written twice, 5 wrong byte, 6 resident slot out of range, 7 empty byte. */
int c3o_byte_oracle(int kind, int n_ranks, int64_t chunk, int64_t src_bytes, int64_t dst_bytes,
                    const c3o_transfer* t, int n_transfers, char* why, size_t why_len);

/* Expected all-gather output of rank r's receive buffer given per-rank chunks
 * filled with c3o_fill_labels(seed, rank, tensor): slot g = rank g's chunk. */
void c3o_expected_allgather(void* out, int n_ranks, int64_t chunk, uint64_t seed, int tensor);

/* Expected all-to-all receive buffer of rank r when every rank g's send buffer
 * (n slots of `slot` bytes) holds c3o_fill_labels(seed, g, tensor): slot g of
 * rank r's receive = rank g's send slot r (test_conccl.cpp:63-64). */
void c3o_expected_alltoall(void* out, int n_ranks, int rank, int64_t slot, uint64_t seed, int tensor);

/* Reduce-scatter reference: inputs[g] is rank g's bf16 input of n*count
 * elements; out receives rank r's slot: sum_{g=0..n-1} inputs[g][r*count + i]
 * accumulated in fp32 in rank order, rounded once to bf16 (RNE). */
void c3o_reduce_scatter_bf16(const uint16_t* const* inputs, int n_ranks, int rank,
                             int64_t count, uint16_t* out);

/* fp64-accumulate reference for C = A * B^T at the given (i, j) pairs.
 * A: bf16 [M,K] row-major; B: bf16 [N,K] row-major; writes ref and
 * abs_dot = sum_k |A[i,k] * B[j,k]| per sample. */
void c3o_gemm_bf16_ref_samples(const uint16_t* A, const uint16_t* B, int64_t M, int64_t N,
                               int64_t K, const int64_t* rows, const int64_t* cols,
                               int64_t n_samples, double* ref, double* abs_dot);

/* Blocked fp32 GEMM C = A * B^T (A [M,K], B [N,K], C [M,N]) on `threads`
 * OpenMP threads: the CPU compute arm of the cfg1 C3 baseline. */
void c3o_gemm_f32(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                  int threads);

/* CPU C3 (cfg1 of BASELINE.json: fp32 GEMM concurrent with a plan-replayed
 * all-gather). Times, in seconds (medians over `iters` after `warmup`):
 * out[0] gemm alone, out[1] all-gather alone, out[2] concurrent (GEMM on
 * gemm_threads OpenMP threads, plan replay on one extra thread). */
int c3o_cpu_c3(int64_t M, int64_t N, int64_t K, int gemm_threads, const c3o_transfer* t,
               int n_transfers, int n_ranks, int64_t src_bytes, int64_t dst_bytes, int warmup,
               int iters, double* out);
/* The same for any collective kind (0 all-gather, 1 all-to-all, 2
 * reduce-scatter = the all-to-all plan into staging + a local fp32 reduce of
 * every rank's slots on the communication thread). */
int c3o_cpu_c3_kind(int64_t M, int64_t N, int64_t K, int gemm_threads, const c3o_transfer* t,
                    int n_transfers, int n_ranks, int64_t src_bytes, int64_t dst_bytes, int kind,
                    int warmup, int iters, double* out);

#ifdef __cplusplus
}
#endif
#endif
