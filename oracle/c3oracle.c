/* c3oracle.c — CPU restatement of the C3 data semantics. TEST INFRASTRUCTURE:
 * see c3oracle.h for scope, citations and who may call it. */
#define _GNU_SOURCE
#include "c3oracle.h"

#include <math.h>
#include <omp.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* splitmix64 finaliser; the CUDA fill kernel uses the same constants. */
uint64_t c3o_hash64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint64_t c3o_label_word(uint64_t seed, int rank, int tensor, uint64_t word) {
    const uint64_t key = seed ^ ((uint64_t)(uint32_t)rank << 56) ^ ((uint64_t)(uint32_t)tensor << 48);
    return c3o_hash64(key ^ word);
}

void c3o_fill_labels(void* buf, int64_t bytes, uint64_t seed, int rank, int tensor) {
    uint8_t* p = (uint8_t*)buf;
    const int64_t words = bytes / 8;
#pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < words; ++w) {
        const uint64_t v = c3o_label_word(seed, rank, tensor, (uint64_t)w);
        memcpy(p + w * 8, &v, 8);
    }
    if (bytes % 8) {
        const uint64_t v = c3o_label_word(seed, rank, tensor, (uint64_t)words);
        memcpy(p + words * 8, &v, (size_t)(bytes % 8));
    }
}

float c3o_bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

uint16_t c3o_f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

uint16_t c3o_bf16_value(uint64_t seed, int rank, int tensor, uint64_t idx) {
    const uint64_t h = c3o_label_word(seed, rank, tensor, idx);
    /* 24 random bits -> u in [-1, 1) exactly representable, times 2^-3. */
    const int32_t r24 = (int32_t)(h >> 40);              /* [0, 2^24) */
    const float u = (float)(r24 - (1 << 23)) * (1.0f / 8388608.0f);
    return c3o_f32_to_bf16_rne(u * 0.125f);
}

void c3o_fill_bf16(uint16_t* buf, int64_t count, uint64_t seed, int rank, int tensor) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) buf[i] = c3o_bf16_value(seed, rank, tensor, (uint64_t)i);
}

int c3o_replay_plan(const c3o_transfer* t, int n_transfers, int n_ranks, void* const* src,
                    int64_t src_bytes, void* const* dst, int64_t dst_bytes) {
    for (int i = 0; i < n_transfers; ++i) {
        const c3o_transfer* x = &t[i];
        if (x->src_gpu < 0 || x->src_gpu >= n_ranks || x->dst_gpu < 0 || x->dst_gpu >= n_ranks)
            return -1;
        if (x->src_offset < 0 || x->src_offset + x->length > src_bytes) return -1;
        if (x->dst_offset < 0 || x->dst_offset + x->length > dst_bytes) return -1;
        memcpy((uint8_t*)dst[x->dst_gpu] + x->dst_offset,
               (const uint8_t*)src[x->src_gpu] + x->src_offset, (size_t)x->length);
    }
    return 0;
}

/* test_conccl.cpp:21-23: label(rank, off) = (rank << 40) | off. */
static int64_t bo_label(int rank, int64_t off) { return ((int64_t)rank << 40) | off; }

int c3o_byte_oracle(int kind, int n, int64_t chunk, int64_t src_bytes, int64_t dst_bytes,
                    const c3o_transfer* t, int n_transfers, char* why, size_t why_len) {
#define BO_FAIL(code, ...)                                   \
    do {                                                     \
        if (why && why_len) snprintf(why, why_len, __VA_ARGS__); \
        rc = (code);                                         \
        goto done;                                           \
    } while (0)
    int rc = 0;
    const int64_t kEmpty = -1;
    int64_t** dst = (int64_t**)calloc((size_t)n, sizeof(int64_t*));
    for (int r = 0; r < n; ++r) {
        dst[r] = (int64_t*)malloc((size_t)(dst_bytes > 0 ? dst_bytes : 1) * sizeof(int64_t));
        for (int64_t j = 0; j < dst_bytes; ++j) dst[r][j] = kEmpty;
        for (int64_t j = 0; j < chunk; ++j) {
            const int64_t at = (int64_t)r * chunk + j;
            if (at >= dst_bytes) BO_FAIL(6, "resident slot out of range");
            dst[r][at] = kind == 0 ? bo_label(r, j) : bo_label(r, at);
        }
    }
    for (int i = 0; i < n_transfers; ++i) {
        const c3o_transfer* x = &t[i];
        if (x->src_gpu < 0 || x->src_gpu >= n || x->dst_gpu < 0 || x->dst_gpu >= n)
            BO_FAIL(1, "rank out of range");
        if (x->src_offset < 0 || x->src_offset + x->length > src_bytes)
            BO_FAIL(2, "source out of range");
        if (x->dst_offset < 0 || x->dst_offset + x->length > dst_bytes)
            BO_FAIL(3, "destination out of range");
        for (int64_t j = 0; j < x->length; ++j) {
            int64_t* cell = &dst[x->dst_gpu][x->dst_offset + j];
            if (*cell != kEmpty) BO_FAIL(4, "byte written twice");
            *cell = bo_label(x->src_gpu, x->src_offset + j);
        }
    }
    for (int r = 0; r < n; ++r)
        for (int s = 0; s < n; ++s)
            for (int64_t j = 0; j < chunk; ++j) {
                const int64_t got = dst[r][(int64_t)s * chunk + j];
                const int64_t want = kind == 0 ? bo_label(s, j) : bo_label(s, (int64_t)r * chunk + j);
                if (got == kEmpty) BO_FAIL(7, "empty byte at rank %d slot %d", r, s);
                if (got != want) BO_FAIL(5, "wrong byte at rank %d slot %d", r, s);
            }
done:
    for (int r = 0; r < n; ++r) free(dst[r]);
    free(dst);
    return rc;
#undef BO_FAIL
}

void c3o_expected_allgather(void* out, int n, int64_t chunk, uint64_t seed, int tensor) {
    for (int g = 0; g < n; ++g) c3o_fill_labels((uint8_t*)out + (int64_t)g * chunk, chunk, seed, g, tensor);
}

void c3o_expected_alltoall(void* out, int n, int rank, int64_t slot, uint64_t seed, int tensor) {
    uint8_t* buf = (uint8_t*)malloc((size_t)(n * slot) + 8);
    for (int g = 0; g < n; ++g) {
        c3o_fill_labels(buf, (int64_t)n * slot, seed, g, tensor);
        memcpy((uint8_t*)out + (int64_t)g * slot, buf + (int64_t)rank * slot, (size_t)slot);
    }
    free(buf);
}

void c3o_reduce_scatter_bf16(const uint16_t* const* inputs, int n, int rank, int64_t count,
                             uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        float acc = 0.0f;
        for (int g = 0; g < n; ++g) acc += c3o_bf16_to_f32(inputs[g][(int64_t)rank * count + i]);
        out[i] = c3o_f32_to_bf16_rne(acc);
    }
}

void c3o_gemm_bf16_ref_samples(const uint16_t* A, const uint16_t* B, int64_t M, int64_t N,
                               int64_t K, const int64_t* rows, const int64_t* cols,
                               int64_t n_samples, double* ref, double* abs_dot) {
    (void)M;
    (void)N;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < n_samples; ++s) {
        const uint16_t* a = A + rows[s] * K;
        const uint16_t* b = B + cols[s] * K;
        double acc = 0.0, mag = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            const double p = (double)c3o_bf16_to_f32(a[k]) * (double)c3o_bf16_to_f32(b[k]);
            acc += p;
            mag += fabs(p);
        }
        ref[s] = acc;
        if (abs_dot) abs_dot[s] = mag;
    }
}

void c3o_gemm_f32(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                  int threads) {
    /* C = A * B^T; both operands K-contiguous, so the inner loop is a dot
     * product over K blocked 64x64 in (i, j) for cache reuse. */
    const int64_t BI = 64, BJ = 64, BK = 256;
#pragma omp parallel for collapse(2) schedule(static) num_threads(threads)
    for (int64_t i0 = 0; i0 < M; i0 += BI)
        for (int64_t j0 = 0; j0 < N; j0 += BJ) {
            const int64_t i1 = i0 + BI < M ? i0 + BI : M;
            const int64_t j1 = j0 + BJ < N ? j0 + BJ : N;
            for (int64_t i = i0; i < i1; ++i)
                for (int64_t j = j0; j < j1; ++j) C[i * N + j] = 0.0f;
            for (int64_t k0 = 0; k0 < K; k0 += BK) {
                const int64_t k1 = k0 + BK < K ? k0 + BK : K;
                for (int64_t i = i0; i < i1; ++i) {
                    const float* a = A + i * K;
                    for (int64_t j = j0; j < j1; ++j) {
                        const float* b = B + j * K;
                        float acc = 0.0f;
#pragma omp simd reduction(+ : acc)
                        for (int64_t k = k0; k < k1; ++k) acc += a[k] * b[k];
                        C[i * N + j] += acc;
                    }
                }
            }
        }
}

/* ---- CPU C3 baseline ------------------------------------------------------ */

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : x > y;
}

static double median(double* v, int n) {
    qsort(v, (size_t)n, sizeof(double), cmp_double);
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

/* Reduce-scatter second phase on the host, every rank: out_r[i] = sum over g
 * of (g == r ? src_r[r slot] : dst_r[g slot])[i], fp32 in rank order, one
 * bf16 rounding (the same arithmetic as c3o_reduce_scatter_bf16). */
static void reduce_local_all(int n, int64_t slot_bytes, void* const* src, void* const* dst, uint16_t* out) {
    const int64_t count = slot_bytes / 2;
    for (int r = 0; r < n; ++r) {
        for (int64_t i = 0; i < count; ++i) {
            float acc = 0.0f;
            for (int g = 0; g < n; ++g) {
                /* own slot straight from the input, the others from staging */
                const uint16_t* sl = (const uint16_t*)(g == r ? src[r] : dst[r]) + (int64_t)g * count;
                acc += c3o_bf16_to_f32(sl[i]);
            }
            out[i] = c3o_f32_to_bf16_rne(acc); /* timing only: every rank reuses one buffer */
        }
    }
}

typedef struct {
    const c3o_transfer* t;
    int n_t, n, kind;
    void* const* src;
    int64_t src_bytes;
    void* const* dst;
    int64_t dst_bytes;
    uint16_t* rs_out;
} comm_job;

static void run_comm(const comm_job* j) {
    c3o_replay_plan(j->t, j->n_t, j->n, j->src, j->src_bytes, j->dst, j->dst_bytes);
    if (j->kind == 2) reduce_local_all(j->n, j->src_bytes / j->n, j->src, j->dst, j->rs_out);
}

static void* comm_thread(void* arg) {
    run_comm((const comm_job*)arg);
    return NULL;
}

int c3o_cpu_c3_kind(int64_t M, int64_t N, int64_t K, int gemm_threads, const c3o_transfer* t,
                    int n_transfers, int n_ranks, int64_t src_bytes, int64_t dst_bytes, int kind,
                    int warmup, int iters, double* out) {
    if (iters < 1 || n_ranks < 1 || kind < 0 || kind > 2) return -1;
    float* A = (float*)malloc((size_t)(M * K) * sizeof(float));
    float* B = (float*)malloc((size_t)(N * K) * sizeof(float));
    float* C = (float*)malloc((size_t)(M * N) * sizeof(float));
    void** src = (void**)calloc((size_t)n_ranks, sizeof(void*));
    void** dst = (void**)calloc((size_t)n_ranks, sizeof(void*));
    uint16_t* rs_out = kind == 2 ? (uint16_t*)malloc((size_t)(src_bytes / n_ranks)) : NULL;
    for (int64_t i = 0; i < M * K; ++i) A[i] = c3o_bf16_to_f32(c3o_bf16_value(20241217, 0, 0, (uint64_t)i));
    for (int64_t i = 0; i < N * K; ++i) B[i] = c3o_bf16_to_f32(c3o_bf16_value(20241217, 0, 1, (uint64_t)i));
    for (int r = 0; r < n_ranks; ++r) {
        src[r] = malloc((size_t)src_bytes);
        dst[r] = malloc((size_t)dst_bytes);
        if (kind == 2)
            c3o_fill_bf16((uint16_t*)src[r], src_bytes / 2, 20241217, r, 3);
        else
            c3o_fill_labels(src[r], src_bytes, 20241217, r, kind == 0 ? 2 : 4);
        memset(dst[r], 0, (size_t)dst_bytes);
    }
    double* tg = (double*)malloc(sizeof(double) * (size_t)iters);
    double* tc = (double*)malloc(sizeof(double) * (size_t)iters);
    double* tb = (double*)malloc(sizeof(double) * (size_t)iters);
    comm_job job = {t, n_transfers, n_ranks, kind, src, src_bytes, dst, dst_bytes, rs_out};
    for (int it = -warmup; it < iters; ++it) {
        double t0 = now_s();
        c3o_gemm_f32(A, B, C, M, N, K, gemm_threads);
        const double g = now_s() - t0;
        t0 = now_s();
        run_comm(&job);
        const double c = now_s() - t0;
        pthread_t th;
        t0 = now_s();
        pthread_create(&th, NULL, comm_thread, &job);
        c3o_gemm_f32(A, B, C, M, N, K, gemm_threads);
        pthread_join(th, NULL);
        const double b = now_s() - t0;
        if (it >= 0) {
            tg[it] = g;
            tc[it] = c;
            tb[it] = b;
        }
    }
    out[0] = median(tg, iters);
    out[1] = median(tc, iters);
    out[2] = median(tb, iters);
    for (int r = 0; r < n_ranks; ++r) {
        free(src[r]);
        free(dst[r]);
    }
    free(src);
    free(dst);
    free(rs_out);
    free(A);
    free(B);
    free(C);
    free(tg);
    free(tc);
    free(tb);
    return 0;
}

int c3o_cpu_c3(int64_t M, int64_t N, int64_t K, int gemm_threads, const c3o_transfer* t,
               int n_transfers, int n_ranks, int64_t src_bytes, int64_t dst_bytes, int warmup,
               int iters, double* out) {
    return c3o_cpu_c3_kind(M, N, K, gemm_threads, t, n_transfers, n_ranks, src_bytes, dst_bytes, 0, warmup,
                           iters, out);
}
