// SM-driven direct collectives over NVSwitch peer memory (the paper's "CU
// backend", executed instead of modeled) and the synthetic-input generators.
//
//  * all-gather, push form: rank `self` loads each 16-byte vector of its chunk
//    once and stores it into slot `self` of every rank's receive buffer — the
//    same (src, dst, offset) mapping as the reference's plan_all_gather
//    (/root/reference/proj/src/conccl.cpp:35-51), one step, no ring (every
//    peer is one NVSwitch hop away).
//  * reduce-scatter, pull form (extension): rank `self`
//    reads slot `self` of every rank's input, sums in fp32 in rank order
//    0..n-1 and rounds once to bf16 — bit-identical to the oracle
//    (oracle/c3oracle.c c3o_reduce_scatter_bf16). The same kernel, fed with
//    local staging slots, is the copy-engine path's local reduce.
//
// Multi-process completion uses per-rank flag words written with
// st.release.sys into peers' signal arrays (monotonic epochs; no reset).
//
// Link-rate emulation (loopback only, off by default): with cta_bpns > 0 each
// CTA paces its peer traffic to cta_bpns bytes/ns on the global timer
// (link_wait, ptx.cuh), so a loopback collective takes the time the node's
// NVLink would give it regardless of SM clocks or CTA count. The iteration
// loops are CTA-uniform so the pacing barrier is legal.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "c3cuda_internal.hpp"
#include "ptx.cuh"

namespace c3k {

namespace {

constexpr int kThreads = 512;  // byte-granular kernels (tiny parity cases)
// Vector collectives run 256-thread CTAs, two per unit of the caller's CTA
// budget (n_ctas counts 512-thread equivalents, the unit the slowdown tables
// and allocations were measured in). A 256-thread CTA fits beside the pair
// GEMM's CTA (256 x 152 registers) in one SM's 64K registers, where a
// 512-thread one (16 warps x 56 allocated) does not: the co-resident C3 mode.
constexpr int kVecThreads = 256;
constexpr int kCtasPerUnit = 2;
constexpr int kThreadsRs = kVecThreads;
// all-to-all moves one store per load (all-gather: n-1), so each thread keeps
// more vectors in flight: 16 (C3_A2A_UNROLL, build-time A/B): co-resident
// cfg2 all-to-all at 24-48 units 0.23-0.61 -> 0.82-0.88 of ideal
// (profiles/r01_a2a_unroll.txt)
#ifndef C3_A2A_UNROLL
#define C3_A2A_UNROLL 16
#endif
constexpr int kUnrollA2a = C3_A2A_UNROLL;
// all-gather: 8 vectors in flight per thread (64 registers: still co-resident
// beside the GEMM; 16 takes 112 and is not), profiles/r01_ag_unroll.txt
#ifndef C3_AG_UNROLL
#define C3_AG_UNROLL 8
#endif
constexpr int kUnrollAg = C3_AG_UNROLL;

// Bounded wait of one thread until every peer's word [slot + p] of this
// rank's signal array reached the epoch. A peer that never arrives (dead,
// or running a mismatched collective) trips the timeout: the thread records
// `code` in the session's error word and returns, so the step ends and the
// host fails it instead of the GPU hanging.
__device__ void wait_peers(const Signals& sig, int n, int slot, uint32_t epoch, uint32_t code) {
    wait_words_bounded(sig.mine, slot, sig.self, n, epoch, sig.timeout_ns, sig.err, code);
}

// Last-CTA election + cross-rank exit barrier. Called by every thread of every
// CTA after its stores; returns after this rank has seen `epoch` from all peers
// (only the elected CTA waits; the other CTAs exit).
__device__ void exit_barrier(const Signals& sig, int n) {
    __syncthreads();
    if (threadIdx.x != 0 || sig.exit_slot < 0) return;
    fence_sys();
    const uint32_t ticket = atomicAdd(sig.done, 1u);
    if (ticket != gridDim.x - 1) return;
    fence_sys();
    for (int p = 0; p < n; ++p)
        if (p != sig.self) st_release_sys(sig.peers[p] + sig.exit_slot + sig.self, sig.epoch);
    wait_peers(sig, n, sig.exit_slot, sig.epoch, kWaitExit);
    *sig.done = 0;  // next launch on this stream starts from zero
}

// Entry barrier: every peer has reached this collective (its inputs are
// ready, or its receive buffer may be overwritten). Block 0 posts; every
// CTA's thread 0 waits. With entry_post false it only waits (flags written
// by the peers' copy-engine streams after their copies into this rank).
__device__ void entry_barrier(const Signals& sig, int n) {
    if (sig.entry_slot < 0) return;
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0 && sig.entry_post) {
            fence_sys();
            for (int p = 0; p < n; ++p)
                if (p != sig.self) st_release_sys(sig.peers[p] + sig.entry_slot + sig.self, sig.entry_epoch);
        }
        wait_peers(sig, n, sig.entry_slot, sig.entry_epoch, sig.entry_post ? kWaitEntry : kWaitCeDone);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(32) signal_wait_kernel(Signals sig, int n) {
    entry_barrier(sig, n);
}

struct FlagWords {
    uint32_t* w[C3_MAX_RANKS];
};
__global__ void __launch_bounds__(32) flag_store_kernel(FlagWords f, int count, uint32_t value) {
    if (threadIdx.x != 0) return;
    fence_sys();
    for (int i = 0; i < count; ++i) st_release_sys(f.w[i], value);
}

// V: the access width (uint4 = 16 B, u256 = 32 B: LDG/STG .256), U: vectors
// in flight per thread; nvec / slot_vec count V-sized vectors.
template <typename V, int U>
__global__ void __launch_bounds__(kVecThreads)
ag_push_vec_kernel(const V* __restrict__ src, MutPtrTable recv, int self, int n,
                   int64_t nvec, int64_t slot_vec, int copy_self, int stream_l2, float cta_bpns,
                   Signals sig) {
    if (sig.enabled) entry_barrier(sig, n);  // peers' receive buffers are free
    const uint64_t pol = policy_evict_first();
    V* dst[C3_MAX_RANKS];
#pragma unroll
    for (int j = 0; j < C3_MAX_RANKS; ++j)
        dst[j] = j < n ? static_cast<V*>(recv.p[j]) + slot_vec * self : nullptr;
    const int64_t step = static_cast<int64_t>(gridDim.x) * kVecThreads * U;
    const uint64_t t0 = global_ns();
    double sent = 0.0;  // peer bytes this CTA has pushed (pacing)
    for (int64_t blk = static_cast<int64_t>(blockIdx.x) * kVecThreads * U; blk < nvec; blk += step) {
        if (cta_bpns > 0.f) {
            if (threadIdx.x == 0) link_wait(t0, sent, cta_bpns);
            __syncthreads();
            const int64_t left = nvec - blk;
            sent += static_cast<double>(sizeof(V)) * (n - 1) *
                    static_cast<double>(left < kVecThreads * U ? left : kVecThreads * U);
        }
        const int64_t base = blk + threadIdx.x;
        V v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * kVecThreads;
            if (i < nvec) v[u] = ld_vec(src + i, stream_l2 != 0, pol);
        }
        // peers in rotated order so the ranks do not all start on the same target
        for (int j = 1; j <= n; ++j) {
            const int p = (self + j) % n;
            if (p == self && !copy_self) continue;
            V* d = dst[p];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = base + static_cast<int64_t>(u) * kVecThreads;
                if (i < nvec) st_vec(d + i, v[u], stream_l2 != 0, pol);
            }
        }
    }
    if (cta_bpns > 0.f && threadIdx.x == 0) link_wait(t0, sent, cta_bpns);  // the last bytes' link time
    if (sig.enabled) exit_barrier(sig, n);
}

// All-gather, push form on the SM's TMA unit: one thread per CTA streams this
// CTA's pieces of the chunk global -> shared memory (nbuf buffers, loads
// issued nbuf-1 pieces ahead) -> slot `self` of every rank with bulk stores
// (cp.async.bulk), so a CTA moves `piece` bytes per instruction instead of 16.
constexpr int kBulkMaxBufs = 8;
__global__ void __launch_bounds__(32)
ag_push_bulk_kernel(const uint8_t* __restrict__ src, MutPtrTable recv, int self, int n, int64_t chunk,
                    int copy_self, int piece, int nbuf, int stream_l2, float cta_bpns, Signals sig) {
    if (sig.enabled) entry_barrier(sig, n);  // peers' receive buffers are free
    extern __shared__ __align__(128) uint8_t bulk_buf[];
    __shared__ __align__(8) uint64_t bar[kBulkMaxBufs];
    if (threadIdx.x == 0) {
        for (int b = 0; b < nbuf; ++b) mbar_init(&bar[b], 1);
        fence_mbar_init();
        const uint64_t pol = stream_l2 ? policy_evict_first() : policy_evict_normal();
        const int64_t G = gridDim.x;
        const int64_t pieces = (chunk + piece - 1) / piece;
        const int64_t mine = pieces > blockIdx.x ? (pieces - blockIdx.x + G - 1) / G : 0;
        const int targets = copy_self ? n : n - 1;
        auto piece_len = [&](int64_t k) {
            const int64_t left = chunk - (blockIdx.x + k * G) * piece;
            return static_cast<uint32_t>(left < piece ? left : piece);
        };
        auto issue_load = [&](int64_t k) {
            const int b = static_cast<int>(k % nbuf);
            const uint32_t len = piece_len(k);
            mbar_arrive_expect_tx(&bar[b], len);
            bulk_load(bulk_buf + static_cast<int64_t>(b) * piece, src + (blockIdx.x + k * G) * piece, len,
                      &bar[b], pol);
        };
        for (int64_t k = 0; k < nbuf - 1 && k < mine; ++k) issue_load(k);
        const uint64_t t0 = global_ns();
        double sent = 0.0;
        for (int64_t k = 0; k < mine; ++k) {
            const int b = static_cast<int>(k % nbuf);
            const uint32_t len = piece_len(k);
            mbar_wait(&bar[b], static_cast<uint32_t>((k / nbuf) & 1));
            if (cta_bpns > 0.f) link_wait(t0, sent, cta_bpns);
            sent += static_cast<double>(len) * (n - 1);
            const int64_t off = static_cast<int64_t>(self) * chunk + (blockIdx.x + k * G) * piece;
            for (int j = 1; j <= n; ++j) {  // rotated targets
                const int p = (self + j) % n;
                if (p == self && !copy_self) continue;
                bulk_store(static_cast<uint8_t*>(recv.p[p]) + off, bulk_buf + static_cast<int64_t>(b) * piece,
                           len, pol);
            }
            bulk_commit();
            // refill buffer (k-1) % nbuf (stores = group k-1) with piece k+nbuf-1
            if (k + nbuf - 1 < mine) {
                bulk_wait_read<1>();
                issue_load(k + nbuf - 1);
            }
        }
        bulk_wait_all();
        fence_proxy_async_global();
        if (cta_bpns > 0.f) link_wait(t0, sent, cta_bpns);
        (void)targets;
    }
    if (sig.enabled) exit_barrier(sig, n);
}

// Byte-granular fallback shape for chunks that are not 16-byte multiples or
// 16-byte aligned (tiny parity cases only; large runs always take the vector path).
__global__ void __launch_bounds__(kThreads)
ag_push_byte_kernel(const uint8_t* __restrict__ src, MutPtrTable recv, int self, int n,
                    int64_t chunk, int copy_self, Signals sig) {
    if (sig.enabled) entry_barrier(sig, n);  // peers' receive buffers are free
    const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < chunk; i += step) {
        const uint8_t v = src[i];
        for (int p = 0; p < n; ++p) {
            if (p == self && !copy_self) continue;
            static_cast<uint8_t*>(recv.p[p])[chunk * self + i] = v;
        }
    }
    if (sig.enabled) exit_barrier(sig, n);
}

// All-to-all, push form (plan_all_to_all's mapping, conccl.cpp:55-84): slot p
// of rank `self`'s send buffer goes to slot `self` of rank p's receive buffer.
template <typename V, int U>
__global__ void __launch_bounds__(kVecThreads)
a2a_push_vec_kernel(const V* __restrict__ send, MutPtrTable recv, int self, int n,
                    int64_t slot_vec, int64_t stride_vec, int stream_l2, float cta_bpns, Signals sig) {
    if (sig.enabled) entry_barrier(sig, n);  // peers' receive buffers are free
    const uint64_t pol = policy_evict_first();
    const int64_t step = static_cast<int64_t>(gridDim.x) * kVecThreads * U;
    const uint64_t t0 = global_ns();
    double sent = 0.0;
    for (int j = 0; j < n; ++j) {
        const int p = (self + 1 + j) % n;  // rotated: the ranks start on different targets
        const V* src = send + stride_vec * p;
        V* dst = static_cast<V*>(recv.p[p]) + stride_vec * self;
        for (int64_t blk = static_cast<int64_t>(blockIdx.x) * kVecThreads * U; blk < slot_vec; blk += step) {
            if (cta_bpns > 0.f && p != self) {
                if (threadIdx.x == 0) link_wait(t0, sent, cta_bpns);
                __syncthreads();
                const int64_t left = slot_vec - blk;
                sent += static_cast<double>(sizeof(V)) *
                        static_cast<double>(left < kVecThreads * U ? left : kVecThreads * U);
            }
            const int64_t base = blk + threadIdx.x;
            V v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = base + static_cast<int64_t>(u) * kVecThreads;
                if (i < slot_vec) v[u] = ld_vec(src + i, stream_l2 != 0, pol);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = base + static_cast<int64_t>(u) * kVecThreads;
                if (i < slot_vec) st_vec(dst + i, v[u], stream_l2 != 0, pol);
            }
        }
    }
    if (cta_bpns > 0.f && threadIdx.x == 0) link_wait(t0, sent, cta_bpns);
    if (sig.enabled) exit_barrier(sig, n);
}

__global__ void __launch_bounds__(kThreads)
a2a_push_byte_kernel(const uint8_t* __restrict__ send, MutPtrTable recv, int self, int n,
                     int64_t slot, Signals sig) {
    if (sig.enabled) entry_barrier(sig, n);  // peers' receive buffers are free
    const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int p = 0; p < n; ++p)
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < slot; i += step)
            static_cast<uint8_t*>(recv.p[p])[slot * self + i] = send[slot * p + i];
    if (sig.enabled) exit_barrier(sig, n);
}

__device__ __forceinline__ void acc_bf16x8(float (&acc)[8], const uint4& v) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        acc[2 * j] = __fadd_rn(acc[2 * j], f.x);
        acc[2 * j + 1] = __fadd_rn(acc[2 * j + 1], f.y);
    }
}

template <int N>
__global__ void __launch_bounds__(kThreadsRs)
rs_pull_vec_kernel(PtrTable in, uint4* __restrict__ out, int self, int64_t nvec,
                   int64_t slot_vec, int stream_l2, float cta_bpns, Signals sig) {
    const uint64_t pol = policy_evict_first();
    if (sig.enabled) entry_barrier(sig, N);
    const uint4* src[N];
#pragma unroll
    for (int g = 0; g < N; ++g) src[g] = static_cast<const uint4*>(in.p[g]) + slot_vec * self;
    const int64_t step = static_cast<int64_t>(gridDim.x) * kThreadsRs * 2;
    const uint64_t t0 = global_ns();
    double pulled = 0.0;  // peer bytes this CTA has read (pacing)
    for (int64_t blk = static_cast<int64_t>(blockIdx.x) * kThreadsRs * 2; blk < nvec; blk += step) {
        if (cta_bpns > 0.f) {
            if (threadIdx.x == 0) link_wait(t0, pulled, cta_bpns);
            __syncthreads();
            const int64_t left = nvec - blk;
            pulled += 16.0 * (N - 1) * static_cast<double>(left < kThreadsRs * 2 ? left : kThreadsRs * 2);
        }
        const int64_t base = blk + threadIdx.x;
        uint4 v[2][N];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * kThreadsRs;
            if (i < nvec)
#pragma unroll
                for (int g = 0; g < N; ++g)
                    v[u][g] = stream_l2 ? ld_stream_v4(src[g] + i, pol) : ld_v4(src[g] + i);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * kThreadsRs;
            if (i >= nvec) continue;
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int g = 0; g < N; ++g) acc_bf16x8(acc, v[u][g]);  // rank order 0..N-1
            uint4 o;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
            if (stream_l2)
                st_stream_v4(out + i, o, pol);
            else
                st_v4(out + i, o);
        }
    }
    if (cta_bpns > 0.f && threadIdx.x == 0) link_wait(t0, pulled, cta_bpns);
    if (sig.enabled) exit_barrier(sig, N);
}

__global__ void __launch_bounds__(kThreads)
rs_pull_scalar_kernel(PtrTable in, __nv_bfloat16* __restrict__ out, int self, int n, int64_t count,
                      Signals sig) {
    if (sig.enabled) entry_barrier(sig, n);
    const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < count; i += step) {
        float acc = 0.f;
        for (int g = 0; g < n; ++g)
            acc = __fadd_rn(acc, __bfloat162float(static_cast<const __nv_bfloat16*>(in.p[g])[count * self + i]));
        out[i] = __float2bfloat16_rn(acc);
    }
    if (sig.enabled) exit_barrier(sig, n);
}

// ------------------------------------------------------ synthetic inputs ---

__device__ __forceinline__ uint64_t hash64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t label_word(uint64_t key, uint64_t w) { return hash64(key ^ w); }

// T = __nv_bfloat16, or float: the same bf16 values widened (exact) for the
// fp32 GEMM's inputs
template <typename T>
__global__ void fill_bf16_kernel(T* dst, int64_t count, uint64_t key) {
    const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += step) {
        const uint64_t h = label_word(key, static_cast<uint64_t>(i));
        const int32_t r24 = static_cast<int32_t>(h >> 40);
        const float u = static_cast<float>(r24 - (1 << 23)) * (1.0f / 8388608.0f);
        const __nv_bfloat16 b = __float2bfloat16_rn(u * 0.125f);
        if constexpr (sizeof(T) == 4)
            dst[i] = __bfloat162float(b);
        else
            dst[i] = b;
    }
}

__global__ void fill_labels_kernel(uint8_t* dst, int64_t bytes, uint64_t key) {
    const int64_t words = bytes / 8;
    const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 7) == 0;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w <= words; w += step) {
        const uint64_t v = label_word(key, static_cast<uint64_t>(w));
        const int64_t at = w * 8;
        const int64_t nbytes = w < words ? 8 : bytes - at;
        if (nbytes == 8 && aligned) {
            *reinterpret_cast<uint64_t*>(dst + at) = v;
        } else {
            for (int64_t b = 0; b < nbytes; ++b) dst[at + b] = static_cast<uint8_t>(v >> (8 * b));
        }
    }
}

uint64_t label_key(uint64_t seed, int rank, int tensor) {
    return seed ^ (static_cast<uint64_t>(static_cast<uint32_t>(rank)) << 56) ^
           (static_cast<uint64_t>(static_cast<uint32_t>(tensor)) << 48);
}

// L2 evict-first streaming of collective payloads (default on; C3_COMM_L2=normal
// switches it off for A/B measurements).
int stream_l2_enabled() {
    static const int on = [] {
        const char* e = std::getenv("C3_COMM_L2");
        return (e != nullptr && std::string(e) == "normal") ? 0 : 1;
    }();
    return on;
}

// Bulk-copy (TMA) all-gather. Measured (profiles/r01_comm_impl_ab.txt): alone
// on the whole GPU it moves the loopback all-gather at 0.87 of the HBM peak
// against the LSU push's 0.72-0.75, but beside the GEMM its bulk copies starve
// behind the GEMM's TMA operand loads. So it is used when the collective runs
// alone, unpaced, on >= kBulkSoloUnits CTA units in a loopback world (the
// isolated collective and the serial step at full speed; the runtime's `solo`);
// C3_COMM_IMPL=bulk forces it everywhere and
// C3_COMM_IMPL=lsu never (dev A/B), C3_COMM_PIECE / C3_COMM_NBUF size its
// shared-memory ring.
constexpr int kBulkSoloUnits = 64;
struct BulkCfg {
    bool on, off;
    int piece, nbuf;
};
const BulkCfg& bulk_cfg() {
    static const BulkCfg c = [] {
        BulkCfg b{false, false, 16384, 4};
        const char* e = std::getenv("C3_COMM_IMPL");
        b.on = e != nullptr && std::string(e) == "bulk";
        b.off = e != nullptr && std::string(e) == "lsu";
        if (const char* p = std::getenv("C3_COMM_PIECE")) b.piece = std::max(16, std::atoi(p) / 16 * 16);
        if (const char* q = std::getenv("C3_COMM_NBUF")) b.nbuf = std::min(kBulkMaxBufs, std::max(2, std::atoi(q)));
        return b;
    }();
    return c;
}

// 32-byte (LDG/STG .256) vectors in the all-gather push when aligned: the
// same bytes in flight with half the instructions (co-resident cfg2 0.78-0.82
// -> 0.83-0.84 of ideal); C3_COMM_WIDE=0 keeps 16-byte vectors (dev A/B).
bool wide_vectors() {
    static const bool on = [] {
        const char* e = std::getenv("C3_COMM_WIDE");
        return !(e != nullptr && std::string(e) == "0");
    }();
    return on;
}

int grid_for(int64_t work_items, int threads, int cap) {
    const int64_t g = (work_items + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, cap)));
}

}  // namespace

int launch_allgather_push(int self, int n, const void* send, const MutPtrTable& recv,
                          int64_t chunk_bytes, int n_ctas, const Signals& sig,
                          cudaStream_t stream, double link_bpns, bool solo) {
    if (n < 1 || n > C3_MAX_RANKS || self < 0 || self >= n)
        return set_error(C3_ERR_VALIDATION, "allgather: bad rank/world");
    if (chunk_bytes < 0) return set_error(C3_ERR_VALIDATION, "allgather: negative chunk");
    if (n_ctas < 1) return set_error(C3_ERR_VALIDATION, "allgather: n_ctas must be >= 1");
    // send may alias slot `self` of recv[self] (in-place): then skip the self copy
    const bool in_place = send == static_cast<const uint8_t*>(recv.p[self]) + chunk_bytes * self;
    uintptr_t align = reinterpret_cast<uintptr_t>(send) | static_cast<uintptr_t>(chunk_bytes);
    for (int p = 0; p < n; ++p) align |= reinterpret_cast<uintptr_t>(recv.p[p]);
    if (chunk_bytes == 0 && !sig.enabled) return C3_OK;
    const bool bulk = bulk_cfg().on || (!bulk_cfg().off && solo && link_bpns <= 0.0 && n_ctas >= kBulkSoloUnits);
    if ((align & 15) == 0 && bulk) {
        const BulkCfg& bc = bulk_cfg();
        const size_t smem = static_cast<size_t>(bc.piece) * bc.nbuf;
        static bool attr = false;
        if (!attr) {
            C3_CUDA(cudaFuncSetAttribute(ag_push_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            attr = true;
        }
        const int grid = grid_for(std::max<int64_t>(chunk_bytes, 1), bc.piece, n_ctas);
        ag_push_bulk_kernel<<<grid, 32, smem, stream>>>(static_cast<const uint8_t*>(send), recv, self, n,
                                                        chunk_bytes, in_place ? 0 : 1, bc.piece, bc.nbuf,
                                                        stream_l2_enabled(),
                                                        static_cast<float>(link_bpns / grid), sig);
    } else if ((align & 31) == 0 && wide_vectors()) {
        // 32-byte vectors, half as many in flight per thread: the same bytes, half the instructions
        const int64_t nvec = chunk_bytes / 32;
        const int grid = grid_for(std::max<int64_t>(nvec, 1), kVecThreads * (kUnrollAg / 2), n_ctas * kCtasPerUnit);
        ag_push_vec_kernel<u256, kUnrollAg / 2><<<grid, kVecThreads, 0, stream>>>(
            static_cast<const u256*>(send), recv, self, n, nvec, nvec, in_place ? 0 : 1, stream_l2_enabled(),
            static_cast<float>(link_bpns / grid), sig);
    } else if ((align & 15) == 0) {
        const int64_t nvec = chunk_bytes / 16;
        const int grid = grid_for(std::max<int64_t>(nvec, 1), kVecThreads * kUnrollAg, n_ctas * kCtasPerUnit);
        ag_push_vec_kernel<uint4, kUnrollAg><<<grid, kVecThreads, 0, stream>>>(
            static_cast<const uint4*>(send), recv, self, n, nvec, nvec, in_place ? 0 : 1, stream_l2_enabled(),
            static_cast<float>(link_bpns / grid), sig);
    } else {
        const int grid = grid_for(std::max<int64_t>(chunk_bytes, 1), kThreads, n_ctas);
        ag_push_byte_kernel<<<grid, kThreads, 0, stream>>>(static_cast<const uint8_t*>(send), recv,
                                                          self, n, chunk_bytes, in_place ? 0 : 1, sig);
    }
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_alltoall_push(int self, int n, const void* send, const MutPtrTable& recv,
                         int64_t per_peer_bytes, int n_ctas, const Signals& sig, cudaStream_t stream,
                         double link_bpns, int64_t stride_bytes) {
    if (stride_bytes < 0) stride_bytes = per_peer_bytes;
    if (n < 1 || n > C3_MAX_RANKS || self < 0 || self >= n)
        return set_error(C3_ERR_VALIDATION, "alltoall: bad rank/world");
    if (per_peer_bytes < 0) return set_error(C3_ERR_VALIDATION, "alltoall: negative slot");
    if (n_ctas < 1) return set_error(C3_ERR_VALIDATION, "alltoall: n_ctas must be >= 1");
    if (per_peer_bytes == 0 && !sig.enabled) return C3_OK;
    if (stride_bytes < per_peer_bytes) return set_error(C3_ERR_VALIDATION, "alltoall: stride below the slot");
    uintptr_t align = reinterpret_cast<uintptr_t>(send) | static_cast<uintptr_t>(per_peer_bytes) |
                      static_cast<uintptr_t>(stride_bytes);
    for (int p = 0; p < n; ++p) align |= reinterpret_cast<uintptr_t>(recv.p[p]);
    if (stride_bytes != per_peer_bytes && (align & 15) != 0)
        return set_error(C3_ERR_VALIDATION, "alltoall: a strided slot range must be 16-byte aligned");
    // all-to-all keeps 16-byte vectors by default: 32-byte ones were faster
    // alone but slower beside the GEMM (0.72 vs 0.80 of ideal, profiles/r01_comm_wide.txt)
    static const bool wide_a2a = [] {
        const char* e = std::getenv("C3_COMM_WIDE_A2A");
        return e != nullptr && std::string(e) == "1";
    }();
    if ((align & 31) == 0 && wide_a2a && wide_vectors()) {
        const int64_t nvec = per_peer_bytes / 32;
        const int grid = grid_for(std::max<int64_t>(nvec, 1), kVecThreads * (kUnrollA2a / 2), n_ctas * kCtasPerUnit);
        a2a_push_vec_kernel<u256, kUnrollA2a / 2><<<grid, kVecThreads, 0, stream>>>(
            static_cast<const u256*>(send), recv, self, n, nvec, stride_bytes / 32, stream_l2_enabled(),
            static_cast<float>(link_bpns / grid), sig);
    } else if ((align & 15) == 0) {
        const int64_t nvec = per_peer_bytes / 16;
        const int grid = grid_for(std::max<int64_t>(nvec, 1), kVecThreads * kUnrollA2a, n_ctas * kCtasPerUnit);
        a2a_push_vec_kernel<uint4, kUnrollA2a><<<grid, kVecThreads, 0, stream>>>(
            static_cast<const uint4*>(send), recv, self, n, nvec, stride_bytes / 16, stream_l2_enabled(),
            static_cast<float>(link_bpns / grid), sig);
    } else {
        const int grid = grid_for(std::max<int64_t>(per_peer_bytes, 1), kThreads, n_ctas);
        a2a_push_byte_kernel<<<grid, kThreads, 0, stream>>>(static_cast<const uint8_t*>(send), recv,
                                                           self, n, per_peer_bytes, sig);
    }
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_reduce_scatter_pull(int self, int n, const PtrTable& in, void* out, int64_t count,
                               int n_ctas, const Signals& sig, cudaStream_t stream, double link_bpns) {
    if (n < 1 || n > C3_MAX_RANKS || self < 0 || self >= n)
        return set_error(C3_ERR_VALIDATION, "reduce_scatter: bad rank/world");
    if (count < 0) return set_error(C3_ERR_VALIDATION, "reduce_scatter: negative count");
    if (n_ctas < 1) return set_error(C3_ERR_VALIDATION, "reduce_scatter: n_ctas must be >= 1");
    if (count == 0 && !sig.enabled) return C3_OK;
    uintptr_t align = reinterpret_cast<uintptr_t>(out) | static_cast<uintptr_t>(count * 2);
    for (int g = 0; g < n; ++g) align |= reinterpret_cast<uintptr_t>(in.p[g]);
    if ((align & 15) == 0) {
        const int64_t nvec = count / 8;
        const int grid = grid_for(std::max<int64_t>(nvec, 1), kThreadsRs * 2, n_ctas * kCtasPerUnit);
        uint4* o = static_cast<uint4*>(out);
        switch (n) {
#define C3_RS_CASE(N)                                                                          \
    case N:                                                                                    \
        rs_pull_vec_kernel<N><<<grid, kThreadsRs, 0, stream>>>(                                \
            in, o, self, nvec, nvec, stream_l2_enabled(), static_cast<float>(link_bpns / grid), sig); \
        break;
            C3_RS_CASE(1) C3_RS_CASE(2) C3_RS_CASE(3) C3_RS_CASE(4)
            C3_RS_CASE(5) C3_RS_CASE(6) C3_RS_CASE(7) C3_RS_CASE(8)
#undef C3_RS_CASE
        }
    } else {
        const int grid = grid_for(std::max<int64_t>(count, 1), kThreads, n_ctas);
        rs_pull_scalar_kernel<<<grid, kThreads, 0, stream>>>(in, static_cast<__nv_bfloat16*>(out),
                                                             self, n, count, sig);
    }
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

// Diagnostic SM hog: every thread of every CTA spins on the global timer.
// 1024-thread CTAs with 100 KB of shared memory, two per SM, fill each SM's
// thread slots and most of its shared memory, so no other CTA can be resident.
__global__ void __launch_bounds__(1024) sm_hog_kernel(uint64_t ns) {
    extern __shared__ uint8_t hog_smem[];
    const uint64_t t0 = global_ns();
    while (global_ns() - t0 < ns) __nanosleep(1000);
    if (threadIdx.x == 0) hog_smem[0] = 0;
}

int launch_sm_hog(int sm_count, double ms, cudaStream_t stream) {
    constexpr int kSmem = 100 * 1024;
    static bool attr = false;
    if (!attr) {
        C3_CUDA(cudaFuncSetAttribute(sm_hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    sm_hog_kernel<<<2 * sm_count, 1024, kSmem, stream>>>(static_cast<uint64_t>(ms * 1e6));
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_signal_wait(const Signals& sig, int n, cudaStream_t stream) {
    if (!sig.enabled || sig.entry_slot < 0 || n < 2) return C3_OK;
    signal_wait_kernel<<<1, 32, 0, stream>>>(sig, n);
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_flag_store(uint32_t* const* words, int count, uint32_t value, cudaStream_t stream) {
    if (count <= 0) return C3_OK;
    if (count > C3_MAX_RANKS) return set_error(C3_ERR_VALIDATION, "flag_store: too many words");
    FlagWords f{};
    for (int i = 0; i < count; ++i) f.w[i] = words[i];
    flag_store_kernel<<<1, 32, 0, stream>>>(f, count, value);
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_fill_bf16(void* dst, int64_t count, uint64_t seed, int rank, int tensor,
                     cudaStream_t stream) {
    if (count <= 0) return C3_OK;
    fill_bf16_kernel<<<grid_for(count, 256, 148 * 16), 256, 0, stream>>>(
        static_cast<__nv_bfloat16*>(dst), count, label_key(seed, rank, tensor));
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_fill_f32(void* dst, int64_t count, uint64_t seed, int rank, int tensor, cudaStream_t stream) {
    if (count <= 0) return C3_OK;
    fill_bf16_kernel<<<grid_for(count, 256, 148 * 16), 256, 0, stream>>>(static_cast<float*>(dst), count,
                                                                         label_key(seed, rank, tensor));
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

int launch_fill_labels(void* dst, int64_t bytes, uint64_t seed, int rank, int tensor,
                       cudaStream_t stream) {
    if (bytes <= 0) return C3_OK;
    fill_labels_kernel<<<grid_for(bytes / 8 + 1, 256, 148 * 16), 256, 0, stream>>>(
        static_cast<uint8_t*>(dst), bytes, label_key(seed, rank, tensor));
    C3_CUDA(cudaGetLastError());
    return C3_OK;
}

}  // namespace c3k
