// fp32 GEMM on the TF32 tensor cores at fp32-level accuracy (configs[0]'s
// "fp32 GEMM 1024x1024x1024", BASELINE.json; the reference's GemmKernel with
// dtype_bytes 4, /root/reference/proj/include/c3sim/workload.hpp:18-25).
//
//   C[M,N] = A[M,K] * B[N,K]^T      (fp32 in, fp32 out; A, B K-major)
//
// Split-TF32 inside the SM: TMA brings the raw fp32 operand tiles into shared
// memory, converter warps split every element in place, x ~ hi + lo (hi the
// TF32 rounding of x, written over x; lo the TF32 rounding of x - hi, into a
// separate ring), and the MMA thread issues three tcgen05.mma kind::tf32 per
// 8-deep K step into one fp32 TMEM accumulator: A_lo B_hi + A_hi B_lo +
// A_hi B_hi (the dropped A_lo B_lo and the remainder lo misses are below
// 2^-21 |a b| per product; plain TF32 is 2^-11). Against the first version
// (a separate split pass over HBM, then three K segments each re-loading its
// operands) the operands cross L2 once instead of three times and there is
// one launch instead of two.
//
// Split-K: when the 128x128 tiles are fewer than the SMs (1024^3: 64 tiles),
// each tile's K range is cut into S parts (units = tiles x S, claimed like the
// bf16 kernels' tiles). A part's epilogue counts itself in the tile's arrival
// word. S = 2 (configs[0]): the part whose epilogue reaches the tile first
// zeroes the C tile while the main loops run, and both parts add into it with TMA reductions,
// in whichever order they finish: (0 + p0) + p1 = (0 + p1) + p0 (fp32 addition
// commutes), so the result is bit-reproducible and no part waits for the
// other's result. S > 2: every part but the
// last writes its fp32 partial to a workspace and counts it ready; the last
// sums the S parts in the fixed order 0..S-1, its own straight from TMEM. The
// waits cannot deadlock whatever the grid: the parts waited for are already
// in their epilogues, which wait on nothing.
//
// Infinities and NaNs: a stage holding any non-finite element takes a slow
// path (warp-vote, then a CTA-subset OR over the converter warps): the
// non-finite elements are 0 in hi and lo for the A_lo B_hi and A_hi B_lo
// MMAs, then written back whole into hi for the A_hi B_hi MMAs, so every
// product a*b is formed exactly once with IEEE semantics (inf * finite = inf,
// inf * 0 = NaN, inf * inf = inf), as in an fp32 GEMM. Finite inputs whose
// TF32 rounding would overflow are truncated instead (hi finite, exact lo).
//
// Warp roles (512 threads): warp 0 = tile claimer + TMA producer, warp 1 =
// MMA issuer, warp 2 = TMEM allocator, warps 4..7 = epilogue (TMEM lane
// quarter q = warp - 4), warps 8..15 = converters.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "c3cuda_internal.hpp"
#include "ptx.cuh"

namespace c3k {
namespace gemmf32 {

constexpr int BM = 128, BN = 128;
constexpr int BK = 32;            // fp32 elements per 128-byte swizzle row
constexpr int STAGES = 4;         // raw operand stages (converted to hi in place)
constexpr int LO_BUFS = 2;        // lo operand ring
constexpr int ACC_BUFS = 2;
constexpr int TILE_RING = 4;
constexpr int CONV_WARPS = 8;
constexpr int CONV_THREADS = 32 * CONV_WARPS;
constexpr int THREADS = 256 + CONV_THREADS;
constexpr int GROUP_M = 16;
constexpr uint32_t A_BYTES = BM * BK * 4;          // 16 KiB
constexpr uint32_t B_BYTES = BN * BK * 4;          // 16 KiB
constexpr uint32_t STAGE = A_BYTES + B_BYTES;      // [A | B], raw then hi
constexpr uint32_t VEC4 = STAGE / 16;              // float4 per stage
constexpr int VEC_PER_THREAD = VEC4 / CONV_THREADS;  // 8
constexpr uint32_t EPI_STG = 32 * 32 * 4;  // a warp's 32 rows x 32 fp32 columns (128B-swizzled rows)
constexpr int EPI_BUFS = 2;                 // per epilogue warp
constexpr uint32_t SMEM = STAGES * STAGE + LO_BUFS * STAGE + 4 * EPI_BUFS * EPI_STG + 1024 /*align*/ +
                          1024 /*barriers*/;
static_assert(VEC_PER_THREAD * 4 <= 32, "non-finite masks are 32 bits");
static_assert(SMEM <= 227 * 1024, "shared memory");
constexpr uint32_t kBarEpi = 1, kBarConv = 2;  // named barriers (0 = __syncthreads)

struct Params {
    int m, n, k;
    int tiles_m, tiles_n, num_tiles, k_blocks;
    int splits, num_units;  // split-K parts per tile; units = tiles x splits
    float* c;
    int ldc;
    float4* ws;       // splits > 2: partial tiles, [unit][BN / 4][BM] float4
    int* tile_done;   // splits > 1: per-tile arrivals (zero between launches)
    int* tile_ready;  // splits > 1: per-tile partials published (zero between launches)
    int* tile_counter;
    int* exit_counter;
    unsigned long long* dbg;  // dev timeline only (built with -DC3_F32_TIMELINE): per-CTA stamps [8]
    int dev;  // dev A/B only (C3_F32_DEV, results invalid when set): bit 0 converters skip the
              // split (arrive at once), bit 1 no MMAs (commits only)
};

struct Unit {
    int tile, part, tm, tn, kb0, kb1;
};

__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
    Unit x;
    x.part = u / p.num_tiles;
    x.tile = u - x.part * p.num_tiles;
    const int band = GROUP_M * p.tiles_n;
    const int first_m = (x.tile / band) * GROUP_M;
    const int rows = min(p.tiles_m - first_m, GROUP_M);
    const int in_band = x.tile % band;
    x.tm = first_m + in_band % rows;
    x.tn = in_band / rows;
    x.kb0 = static_cast<int>(static_cast<int64_t>(x.part) * p.k_blocks / p.splits);
    x.kb1 = static_cast<int>(static_cast<int64_t>(x.part + 1) * p.k_blocks / p.splits);
    return x;
}

// lo of x: the tensor core reads an fp32 operand as TF32 by truncation (the
// low 13 mantissa bits ignored; measured: tools/dev/f32_err.py), so hi is x
// itself as it sits in shared memory, hi = trunc(x), and lo is the nearest
// (ties away) TF32 of x - trunc(x), which is exact in fp32 and never overflows.
__device__ __forceinline__ uint32_t lo_of(uint32_t u) {
    return (__float_as_uint(__uint_as_float(u) - __uint_as_float(u & 0xFFFFE000u)) + 0x1000u) & 0xFFFFE000u;
}

__global__ void __launch_bounds__(THREADS, 1)
gemm_f32_split_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_c, const Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* stage_base = smem;                        // [STAGES][A | B]
    uint8_t* lo_base = smem + STAGES * STAGE;          // [LO_BUFS][A_lo | B_lo]
    uint8_t* epi_base = lo_base + LO_BUFS * STAGE;     // [4 warps][EPI_BUFS] C staging
    uint64_t* bars = reinterpret_cast<uint64_t*>(epi_base + 4 * EPI_BUFS * EPI_STG);
    uint64_t* full = bars;                    // [STAGES] TMA -> converters
    uint64_t* conv = full + STAGES;           // [STAGES] converters -> MMA
    uint64_t* empty = conv + STAGES;          // [STAGES] MMA -> TMA
    uint64_t* patch = empty + STAGES;         // [STAGES] slow path: A_lo B_hi, A_hi B_lo done -> converters
    uint64_t* conv2 = patch + STAGES;         // [STAGES] slow path: non-finite hi restored -> MMA
    uint64_t* lo_empty = conv2 + STAGES;      // [LO_BUFS] MMA -> converters
    uint64_t* acc_full = lo_empty + LO_BUFS;  // [ACC_BUFS]
    uint64_t* acc_empty = acc_full + ACC_BUFS;
    uint64_t* tile_full = acc_empty + ACC_BUFS;  // [TILE_RING]
    uint64_t* tile_empty = tile_full + TILE_RING;
    int* tile_ring = reinterpret_cast<int*>(tile_empty + TILE_RING);
    uint32_t* nf_flag = reinterpret_cast<uint32_t*>(tile_ring + TILE_RING);  // [STAGES]
    uint32_t* last_flag = nf_flag + STAGES;
    uint32_t* tmem_slot = last_flag + 1;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
#ifdef C3_F32_TIMELINE
    unsigned long long* dbg = p.dbg ? p.dbg + blockIdx.x * 8 : nullptr;
#define F32_STAMP(cond, slot) \
    if (dbg && (cond)) dbg[slot] = global_ns()
#else
#define F32_STAMP(cond, slot)
#endif
    F32_STAMP(threadIdx.x == 0, 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        tma_prefetch_desc(&map_c);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], CONV_WARPS);
            mbar_init(&empty[s], 1);
            mbar_init(&patch[s], 1);
            mbar_init(&conv2[s], CONV_WARPS);
        }
        for (int b = 0; b < LO_BUFS; ++b) mbar_init(&lo_empty[b], 1);
        for (int b = 0; b < ACC_BUFS; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        for (int r = 0; r < TILE_RING; ++r) {
            mbar_init(&tile_full[r], 1);
            mbar_init(&tile_empty[r], 1 + 4 + CONV_WARPS);  // MMA + epilogue warps + converter warps
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<ACC_BUFS * BN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    F32_STAMP(threadIdx.x == 0, 1);

    if (warp == 0 && lane == 0) {
        // ---------------- unit claimer + TMA producer ----------------
        // first unit = blockIdx.x, later ones claimed one ahead (gemm_tcgen05.cu)
        const uint64_t keep = policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        int u = static_cast<int>(blockIdx.x);
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            if (u >= p.num_units) u = -1;
            mbar_wait(&tile_empty[r], ((i / TILE_RING) & 1) ^ 1);
            tile_ring[r] = u;
            mbar_arrive(&tile_full[r]);
            if (u < 0) break;
            const int next = static_cast<int>(gridDim.x) + atomicAdd(p.tile_counter, 1);
            const Unit x = unit_of(p, u);
            for (int kb = x.kb0; kb < x.kb1; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_arrive_expect_tx(&full[stage], STAGE);
                uint8_t* dst = stage_base + stage * STAGE;
                tma_load_2d(dst, &map_a, &full[stage], kb * BK, x.tm * BM, keep);
                tma_load_2d(dst + A_BYTES, &map_b, &full[stage], kb * BK, x.tn * BN, keep);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            u = next;
        }
    } else if (warp >= 8) {
        // ---------------- converters: raw fp32 (= hi) -> lo ----------------
        const int ct = threadIdx.x - 256;
        int stage = 0, lo = 0;
        uint32_t phase = 0, lo_phase = 0, slow_par = 0;  // slow_par: patch/conv2 parity per stage (bit)
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            mbar_wait(&tile_full[r], (i / TILE_RING) & 1);
            const int u = tile_ring[r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&tile_empty[r]);
            if (u < 0) break;
            const Unit x = unit_of(p, u);
            for (int kb = x.kb0; kb < x.kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                mbar_wait(&lo_empty[lo], lo_phase ^ 1);
                uint8_t* hi = stage_base + stage * STAGE;
                uint8_t* lob = lo_base + lo * STAGE;
                uint32_t pinf = 0, ninf = 0, nan = 0;  // this thread's non-finite elements (bit 4j + c)
                if (!(p.dev & 1)) {
                    // all of this thread's loads in flight first, then the math and stores
                    uint4 v[VEC_PER_THREAD];
#pragma unroll
                    for (int j = 0; j < VEC_PER_THREAD; ++j)
                        v[j] = ld_shared_v4(hi + static_cast<uint32_t>(ct + j * CONV_THREADS) * 16);
#pragma unroll
                    for (int j = 0; j < VEC_PER_THREAD; ++j) {
                        const uint32_t off = static_cast<uint32_t>(ct + j * CONV_THREADS) * 16;
                        uint4 l = make_uint4(lo_of(v[j].x), lo_of(v[j].y), lo_of(v[j].z), lo_of(v[j].w));
                        const uint32_t mx = max(max(v[j].x & 0x7FFFFFFFu, v[j].y & 0x7FFFFFFFu),
                                                max(v[j].z & 0x7FFFFFFFu, v[j].w & 0x7FFFFFFFu));
                        if (mx >= 0x7F800000u) {  // rare: a non-finite element (the exact path)
                            const uint32_t in[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
                            uint32_t lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint32_t a = in[c] & 0x7FFFFFFFu;
                                if (a < 0x7F800000u) continue;
                                const uint32_t bit = 1u << (4 * j + c);
                                if (a == 0x7F800000u)
                                    (in[c] >> 31 ? ninf : pinf) |= bit;
                                else
                                    nan |= bit;
                                st_shared_u32(hi + off + 4 * c, 0u);  // 0 in the two mixed products; back below
                                lw[c] = 0u;
                            }
                            l = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                        }
                        st_shared_v4(lob + off, l);
                    }
                }
                fence_proxy_async_shared();  // generic-proxy writes -> the tensor core's reads
                const bool slow = named_bar_or(kBarConv, CONV_THREADS, (pinf | ninf | nan) != 0);
                if (ct == 0) st_shared_u32(&nf_flag[stage], slow ? 1u : 0u);
                __syncwarp();
                if (lane == 0) mbar_arrive(&conv[stage]);
                if (slow) {
                    // after the two mixed products: non-finite elements whole into hi
                    mbar_wait(&patch[stage], (slow_par >> stage) & 1);
                    const uint32_t any = pinf | ninf | nan;
                    if (any) {
#pragma unroll
                        for (int j = 0; j < VEC_PER_THREAD; ++j) {
                            const uint32_t off = static_cast<uint32_t>(ct + j * CONV_THREADS) * 16;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint32_t bit = 1u << (4 * j + c);
                                if (!(any & bit)) continue;
                                const uint32_t val = (pinf & bit) ? 0x7F800000u : (ninf & bit) ? 0xFF800000u : 0x7FC00000u;
                                st_shared_u32(hi + off + 4 * c, val);
                            }
                        }
                    }
                    fence_proxy_async_shared();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&conv2[stage]);
                    slow_par ^= 1u << stage;
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
                if (++lo == LO_BUFS) {
                    lo = 0;
                    lo_phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_tf32_f32(BM, BN);
        int stage = 0, lo = 0, acc = 0;
        uint32_t phase = 0, acc_phase = 0, slow_par = 0;
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            mbar_wait(&tile_full[r], (i / TILE_RING) & 1);
            const int u = tile_ring[r];
            mbar_arrive(&tile_empty[r]);
            if (u < 0) break;
            const Unit x = unit_of(p, u);
            mbar_wait(&acc_empty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kb = x.kb0; kb < x.kb1; ++kb) {
                mbar_wait(&conv[stage], phase);
                tc_fence_after();
                F32_STAMP(kb == x.kb0 && i == 0, 2);
                const bool slow = ld_volatile_shared(&nf_flag[stage]) != 0;
                const uint32_t a_hi = smem_u32(stage_base + stage * STAGE), b_hi = a_hi + A_BYTES;
                const uint32_t a_lo = smem_u32(lo_base + lo * STAGE), b_lo = a_lo + A_BYTES;
#pragma unroll
                for (int k = 0; k < ((p.dev & 2) ? 0 : 4); ++k) {  // +32 B = 8 TF32 of K per MMA, inside the swizzle atom
                    umma_tf32(d, smem_desc_k_sw128(a_lo + k * 32), smem_desc_k_sw128(b_hi + k * 32), idesc,
                              (kb != x.kb0 || k != 0) ? 1u : 0u);
                    umma_tf32(d, smem_desc_k_sw128(a_hi + k * 32), smem_desc_k_sw128(b_lo + k * 32), idesc, 1u);
                    if (!slow)
                        umma_tf32(d, smem_desc_k_sw128(a_hi + k * 32), smem_desc_k_sw128(b_hi + k * 32), idesc, 1u);
                }
                if (slow) {
                    umma_commit(&patch[stage]);
                    mbar_wait(&conv2[stage], (slow_par >> stage) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_tf32(d, smem_desc_k_sw128(a_hi + k * 32), smem_desc_k_sw128(b_hi + k * 32), idesc, 1u);
                    slow_par ^= 1u << stage;
                }
                umma_commit(&empty[stage]);
                umma_commit(&lo_empty[lo]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
                if (++lo == LO_BUFS) lo = 0;
            }
            umma_commit(&acc_full[acc]);
            F32_STAMP(i == 0, 3);
            if (++acc == ACC_BUFS) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- epilogue: TMEM -> C, or -> partial + last-arriver sum ----------------
        const int q = warp - 4;
        const int row_in_tile = q * 32 + lane;
        uint8_t* stg_base = epi_base + q * EPI_BUFS * EPI_STG;
        int stg_i = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            mbar_wait(&tile_full[r], (i / TILE_RING) & 1);
            const int u = tile_ring[r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&tile_empty[r]);
            if (u < 0) {
                if (lane == 0) bulk_wait_all();  // this warp's C stores complete
                break;
            }
            const Unit x = unit_of(p, u);
            // chunk c of this warp's rows (registers) -> swizzled staging -> one TMA
            // store, or a TMA fp32 add into C (OOB rows / columns clipped by the map)
            auto stage_out = [&](const uint32_t (&v)[32], int c, bool add) {
                uint8_t* stg = stg_base + stg_i * EPI_STG;
                if (lane == 0) bulk_wait_read<EPI_BUFS - 1>();  // this buffer's previous store has read it
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    st_shared_v4(stg + lane * 128 + ((j ^ (lane & 7)) << 4),
                                 make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
                fence_proxy_async_shared();
                __syncwarp();
                if (lane == 0) {
                    const int c0 = x.tn * BN + c, r0 = x.tm * BM + q * 32;
                    if (add)
                        tma_reduce_add_2d(&map_c, stg, c0, r0);
                    else
                        tma_store_2d(&map_c, stg, c0, r0);
                    bulk_commit();
                }
                if (++stg_i == EPI_BUFS) stg_i = 0;
            };
            if (p.splits == 2) {
                // the part whose epilogue reaches the tile first (the epilogue
                // warps are idle during the main loop) zeroes its C tile; both
                // parts then add into it (below). Nobody waits on a part that
                // has not started: the zeroing part is already here.
                named_bar_sync(kBarEpi, 128);  // every thread read the previous unit's last_flag
                if (threadIdx.x == 128)
                    st_shared_u32(last_flag, atomicCAS(p.tile_ready + x.tile, 0, 1) == 0 ? 1u : 0u);
                named_bar_sync(kBarEpi, 128);
                if (ld_volatile_shared(last_flag)) {
                    uint32_t zero[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) zero[j] = 0u;
                    for (int c = 0; c < BN; c += 32) stage_out(zero, c, false);
                    if (lane == 0) {
                        bulk_wait_all();  // the zeros are in C
                        fence_proxy_async_global();
                    }
                    __threadfence();
                    named_bar_sync(kBarEpi, 128);
                    if (threadIdx.x == 128) atomicExch(p.tile_ready + x.tile, 2);
                }
            }
            mbar_wait(&acc_full[acc], acc_phase);
            tc_fence_after();
            F32_STAMP(threadIdx.x == 128 && i == 0, 4);
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
            if (p.splits == 1) {
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(t_row + c, v);
                    tmem_ld_wait();
                    stage_out(v, c, false);
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[acc]);
            } else if (p.splits == 2) {
                // both parts add into the zeroed tile: C = (0 + p_a) + p_b = p0 + p1
                // whichever adds first (fp32 addition commutes), so no part waits
                // for the other's result, only for the zeroing
                if (threadIdx.x == 128)
                    wait_ge_gpu(p.tile_ready + x.tile, 2);
                named_bar_sync(kBarEpi, 128);
                if (lane == 0) fence_proxy_async_global();  // the acquire above orders this warp's TMA adds
                F32_STAMP(threadIdx.x == 128 && i == 0, 5);
#pragma unroll 1
                for (int c = 0; c < BN; c += 32) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(t_row + c, v);
                    tmem_ld_wait();
                    stage_out(v, c, true);
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[acc]);
                if (threadIdx.x == 128 && atomicAdd(p.tile_done + x.tile, 1) == 1) {
                    // the second part to finish: both passed their waits, reset for the next launch
                    p.tile_done[x.tile] = 0;
                    p.tile_ready[x.tile] = 0;
                    F32_STAMP(i == 0, 6);
                }
            } else {
                // split-K, S > 2: count in first (see the header)
                named_bar_sync(kBarEpi, 128);  // every thread read the previous unit's last_flag
                if (threadIdx.x == 128) {
                    const int before = atomicAdd(p.tile_done + x.tile, 1);
                    st_shared_u32(last_flag, before == p.splits - 1 ? 1u : 0u);
                }
                named_bar_sync(kBarEpi, 128);
                const size_t tile_f4 = static_cast<size_t>(BN / 4) * BM;  // float4 per partial tile
                const bool is_last = ld_volatile_shared(last_flag) != 0;
                if (!is_last) {
                    // partial tile, float4 (chunk, j) of row r at [(chunk * 8 + j) * BM + r]:
                    // a warp's 32 rows are 512 contiguous bytes per store
                    float4* mine = p.ws + static_cast<size_t>(u) * tile_f4;
#pragma unroll 1
                    for (int c = 0; c < BN; c += 32) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(t_row + c, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            mine[((c / 4) + j) * BM + row_in_tile] =
                                make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                    }
                    tc_fence_before();
                    mbar_arrive(&acc_empty[acc]);
                    __threadfence();  // the partial is visible before it is counted ready
                    named_bar_sync(kBarEpi, 128);
                    if (threadIdx.x == 128) atomicAdd(p.tile_ready + x.tile, 1);
                } else {
                    if (threadIdx.x == 128)
                        wait_ge_gpu(p.tile_ready + x.tile, p.splits - 1);
                    named_bar_sync(kBarEpi, 128);
                    __threadfence();
                    F32_STAMP(threadIdx.x == 128 && i == 0, 5);
#pragma unroll 1
                    for (int c = 0; c < BN; c += 32) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(t_row + c, v);
                        const size_t at = static_cast<size_t>(c / 4) * BM + row_in_tile;
                        float4 sum[8];
                        bool first = true;
                        for (int part = 0; part < p.splits; ++part) {
                            float4 t[8];
                            if (part == x.part) {
                                tmem_ld_wait();
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    t[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                       __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                            } else {
                                const float4* pp = p.ws + static_cast<size_t>(part * p.num_tiles + x.tile) * tile_f4 + at;
#pragma unroll
                                for (int j = 0; j < 8; ++j) t[j] = ld_cg_f4(pp + j * BM);
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                if (first) {
                                    sum[j] = t[j];
                                } else {
                                    sum[j].x += t[j].x;
                                    sum[j].y += t[j].y;
                                    sum[j].z += t[j].z;
                                    sum[j].w += t[j].w;
                                }
                            }
                            first = false;
                        }
                        uint32_t o[32];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            o[4 * j] = __float_as_uint(sum[j].x);
                            o[4 * j + 1] = __float_as_uint(sum[j].y);
                            o[4 * j + 2] = __float_as_uint(sum[j].z);
                            o[4 * j + 3] = __float_as_uint(sum[j].w);
                        }
                        stage_out(o, c, false);
                    }
                    tc_fence_before();
                    mbar_arrive(&acc_empty[acc]);
                    if (threadIdx.x == 128) {  // for the next launch (no one else touches them now)
                        p.tile_done[x.tile] = 0;
                        p.tile_ready[x.tile] = 0;
                    }
                    F32_STAMP(threadIdx.x == 128 && i == 0, 6);
                }
            }
            if (++acc == ACC_BUFS) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    F32_STAMP(threadIdx.x == 0, 7);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<ACC_BUFS * BN>(tmem_base);
    }
    if (threadIdx.x == 0) {  // the last CTA out resets the claim counter
        __threadfence();
        if (atomicAdd(p.exit_counter, 1) == static_cast<int>(gridDim.x) - 1) {
            *p.tile_counter = 0;
            *p.exit_counter = 0;
            __threadfence();
        }
    }
}

}  // namespace gemmf32

// ----------------------------------------------------------------- host ---

// split-K parts: enough units to fill the SMs when the tiles do not, at most
// 4 parts and at least 2 k-blocks each
int gemm_f32_splits(int64_t m, int64_t n, int64_t k, int sm_count) {
    const int64_t tiles = ((m + gemmf32::BM - 1) / gemmf32::BM) * ((n + gemmf32::BN - 1) / gemmf32::BN);
    const int64_t kb = (k + gemmf32::BK - 1) / gemmf32::BK;
    int64_t s = tiles > 0 ? sm_count / tiles : 1;
    s = std::min<int64_t>(std::min<int64_t>(s, 4), kb / 2);
    return static_cast<int>(std::max<int64_t>(s, 1));
}

int64_t gemm_f32_workspace_bytes(int64_t m, int64_t n, int64_t k, int sm_count) {
    const int64_t tiles = ((m + gemmf32::BM - 1) / gemmf32::BM) * ((n + gemmf32::BN - 1) / gemmf32::BN);
    const int s = gemm_f32_splits(m, n, k, sm_count);
    const int64_t counters = (2 * tiles * 4 + 255) / 256 * 256;  // tile_done, tile_ready
    return counters + (s > 2 ? tiles * s * gemmf32::BM * gemmf32::BN * 4 : 0);  // S = 2 adds into C
}

int gemm_f32_launch(const GemmPlan* plan, int grid, cudaStream_t stream) {
    using namespace gemmf32;
    static bool attr_done = false;
    if (!attr_done) {
        const cudaError_t e = cudaFuncSetAttribute(gemm_f32_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(SMEM));
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm f32)");
        attr_done = true;
    }
    Params p;
    p.m = static_cast<int>(plan->m);
    p.n = static_cast<int>(plan->n);
    p.k = static_cast<int>(plan->k);
    p.tiles_m = static_cast<int>((plan->m + BM - 1) / BM);
    p.tiles_n = static_cast<int>((plan->n + BN - 1) / BN);
    p.num_tiles = p.tiles_m * p.tiles_n;
    p.k_blocks = static_cast<int>((plan->k + BK - 1) / BK);
    p.splits = plan->f32_splits;
    p.num_units = p.num_tiles * p.splits;
    p.c = static_cast<float*>(plan->c);
    p.ldc = static_cast<int>(plan->n);
    p.tile_done = reinterpret_cast<int*>(plan->ws);
    p.tile_ready = p.tile_done + p.num_tiles;
    p.ws = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(plan->ws) +
                                     (2 * static_cast<int64_t>(p.num_tiles) * 4 + 255) / 256 * 256);
    p.tile_counter = plan->counters;
    p.exit_counter = plan->counters + 1;
    static const int dev = [] {
        const char* e = std::getenv("C3_F32_DEV");
        return e ? std::atoi(e) : 0;
    }();
    p.dev = dev;
    p.dbg = nullptr;
#ifdef C3_F32_TIMELINE
    // dev timeline builds only: stamps go to the device address in C3_F32_DBG
    const char* dbg = std::getenv("C3_F32_DBG");
    p.dbg = dbg ? reinterpret_cast<unsigned long long*>(std::strtoull(dbg, nullptr, 0)) : nullptr;
#endif
    grid = std::min(grid, p.num_units);
    gemm_f32_split_kernel<<<grid, THREADS, SMEM, stream>>>(plan->map_a, plan->map_b128, plan->map_c, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "gemm f32 launch");
    return C3_OK;
}

}  // namespace c3k
