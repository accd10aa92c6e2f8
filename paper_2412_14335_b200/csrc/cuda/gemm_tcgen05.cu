// Persistent GEMM for sm_100a: TMA -> shared memory (mbarrier ring) ->
// tcgen05.mma (single-thread issue, fp32 accumulators in TMEM, double
// buffered) -> tcgen05.ld epilogue -> global stores.
//
//   C[M,N] = A[M,K] * B[N,K]^T      (A, B K-major; C row-major)
//
// bf16 in / bf16 out (kind::f16). The fp32 GEMM (configs[0]) is
// gemm_f32.cu: split-TF32 inside the SM.
//
// This is the "compute" half of a C3 pair (reference GemmKernel,
// /root/reference/proj/include/c3sim/workload.hpp:18-25; its cost model
// roofline_gemm_time, src/workload.cpp:72-78). The grid is capped at
// `max_ctas` CTAs (one per SM): the B200 counterpart of the paper's CU
// allocation to the GEMM (allocate_cus cus_gemm, src/sim.cpp:40-100) and of
// ConCCL_rp's idle grain (src/strategy.cpp:96-113).
//
// Tiles are CLAIMED dynamically (global atomic counter, claimed by the TMA
// warp a few k-blocks before the MMA needs them, handed to the MMA and
// epilogue warps through a small shared-memory ring). Under C3 a co-running
// collective slows some SMs more than others (co-resident comm CTAs, HBM
// contention); with static round-robin tiles the slowest CTA sets the GEMM's
// end, with claiming the other SMs absorb the work (measured: profiles/
// r01_strategy_grid_*.json).
//
// Stream-K tail (compute-bound shapes whose last wave on the full GPU is
// partly empty): the claims after the whole tiles are equal k-block segments
// of the remaining tiles, one per SM; a tile cut into pieces is finished by
// the piece that arrives last (fixed-order fp32 fix-up, one bf16 rounding).
// See Params::full_units and the epilogue; profiles/r02g_streamk_ab.txt.
//
// Warp roles (256 threads): warp 0 = tile claimer + TMA producer (one
// thread), warp 1 = MMA issuer (one thread), warp 2 = TMEM allocator,
// warps 4..7 = epilogue (warp 4+q reads TMEM lanes 32q..32q+31 = tile rows).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "c3cuda_internal.hpp"
#include "ptx.cuh"

namespace c3k {

namespace gemm {

constexpr int BM = 128;          // UMMA M (one CTA)
constexpr int BK = 64;           // one 128-byte swizzle atom of bf16
constexpr int ACC_BUFS = 2;
constexpr int THREADS = 256;
constexpr int GROUP_M = 16;      // tile raster: 16 M-tiles per band for L2 reuse
constexpr int TILE_RING = 4;     // claimed-tile hand-off depth

template <int BN>
struct Cfg {
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr uint32_t A_STAGE = BM * BK * 2;
    static constexpr uint32_t B_STAGE = BN * BK * 2;
    static constexpr uint32_t STAGE = A_STAGE + B_STAGE;
    static constexpr uint32_t TMEM_COLS = ACC_BUFS * BN;  // 512 or 256
    static constexpr uint32_t SMEM = STAGES * STAGE + 1024 /*align*/ + 512 /*barriers, ring*/;
};

struct Params {
    int m, n, k;
    int tiles_m, tiles_n, num_tiles, k_blocks;
    void* c;  // bf16
    int ldc;
    int* tile_counter;  // claims; reset to 0 by the last CTA to exit
    int* exit_counter;
    // Stream-K tail (sk_segs > 0): claims u < full_units are whole tiles; the
    // k-blocks of the last num_tiles - full_units tiles are cut into sk_segs
    // equal segments (u = full_units + s) shorter than a tile, so a segment
    // is one or two pieces, and long enough that a tile is at most
    // kSkMaxPieces. The decomposition depends on the SM count only, not on
    // the launched grid, so a CTA cap changes no output bit. The piece
    // of a tile that arrives last finishes it: the others publish fp32
    // partials, it sums all in piece order (its own from TMEM) and rounds to
    // bf16 once.
    int full_units, num_units, sk_segs;
    int64_t sk_kb;      // k-blocks of the tail
    float4* sk_ws;      // [tail tile][kSkMaxPieces][BN / 4][BM] fp32 partials
    int* sk_done;       // [tail tile] pieces arrived  (zero between launches)
    int* sk_ready;      // [tail tile] partials published (zero between launches)
};
constexpr int kSkMaxPieces = 4;

struct Piece {
    int tile, kb0, kb1;
    int idx, count;  // this piece's index among its tile's pieces, and their number
};

// stream-K segment starts floor(s L / G), s = 1..G-1, at or below tail k-block x
__device__ __forceinline__ int64_t sk_cuts_le(const Params& p, int64_t x) {
    return min(static_cast<int64_t>(p.sk_segs - 1), ((x + 1) * p.sk_segs - 1) / p.sk_kb);
}

// the pieces of claim u (1 or 2)
__device__ __forceinline__ int unit_pieces(const Params& p, int u, Piece (&pc)[2]) {
    if (u < p.full_units) {
        pc[0] = {u, 0, p.k_blocks, 0, 1};
        return 1;
    }
    const int64_t s = u - p.full_units;
    int64_t pos = s * p.sk_kb / p.sk_segs;
    const int64_t end = (s + 1) * p.sk_kb / p.sk_segs;
    int n = 0;
    while (pos < end && n < 2) {
        const int t = static_cast<int>(pos / p.k_blocks);
        const int64_t base = static_cast<int64_t>(t) * p.k_blocks;
        const int64_t stop = min(end, base + p.k_blocks);
        const int64_t before = sk_cuts_le(p, base);  // cuts at or before the tile's start
        pc[n++] = {p.full_units + t, static_cast<int>(pos - base), static_cast<int>(stop - base),
                   static_cast<int>(sk_cuts_le(p, pos) - before),
                   static_cast<int>(1 + sk_cuts_le(p, base + p.k_blocks - 1) - before)};
        pos = stop;
    }
    return n;
}

__device__ __forceinline__ void tile_coords(const Params& p, int tile, int& tm, int& tn) {
    const int band = GROUP_M * p.tiles_n;
    const int first_m = (tile / band) * GROUP_M;
    const int rows = min(p.tiles_m - first_m, GROUP_M);
    const int in_band = tile % band;
    tm = first_m + in_band % rows;
    tn = in_band / rows;
}

// <= 136 registers per thread (as before the stream-K tail): a co-resident
// collective CTA still fits beside the GEMM's in the SM's register file (the
// memory-bound GEMM of configs[3])
#ifndef C3_NARROW_MAXNREG
#define C3_NARROW_MAXNREG 136
#endif
template <int BN>
__global__ void __maxnreg__(C3_NARROW_MAXNREG)
gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, const Params p) {
    using K = Cfg<BN>;
    constexpr int STAGES = K::STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + STAGES * K::A_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * K::STAGE);
    uint64_t* full = bars;                       // [STAGES]   TMA -> MMA
    uint64_t* empty = bars + STAGES;             // [STAGES]   MMA -> TMA
    uint64_t* acc_full = bars + 2 * STAGES;      // [ACC_BUFS] MMA -> epilogue
    uint64_t* acc_empty = acc_full + ACC_BUFS;   // [ACC_BUFS] epilogue -> MMA
    uint64_t* tile_full = acc_empty + ACC_BUFS;  // [TILE_RING] claimer -> MMA, epilogue
    uint64_t* tile_empty = tile_full + TILE_RING;
    int* tile_ring = reinterpret_cast<int*>(tile_empty + TILE_RING);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + TILE_RING);
    uint32_t* sk_flag = tmem_slot + 1;  // stream-K: this piece arrived first (epilogue warps)

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < ACC_BUFS; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        for (int r = 0; r < TILE_RING; ++r) {
            mbar_init(&tile_full[r], 1);
            mbar_init(&tile_empty[r], 1 + 4);  // MMA thread + one lane per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<K::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---------------- tile claimer + TMA producer ----------------
        const uint64_t keep = policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        // dynamic claiming, or static round-robin when no counter is given.
        // The first tile is the CTA's own (blockIdx.x) and only the later ones
        // are claimed: the claim runs one tile ahead, so with claimed first
        // tiles the CTAs that start first took two tiles each before the last
        // ones started (a collective launched beside the GEMM staggers the
        // starts): configs[0]'s 64-tile GEMM then took two tile times
        // (tools/dev/cfg1_probe.py: 49 -> 73 us beside the collective)
        const bool dyn = p.tile_counter != nullptr;
        int tile = static_cast<int>(blockIdx.x);
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            if (tile >= p.num_units) tile = -1;
            mbar_wait(&tile_empty[r], ((i / TILE_RING) & 1) ^ 1);
            tile_ring[r] = tile;
            mbar_arrive(&tile_full[r]);  // release: consumers read tile_ring[r] after their wait
            if (tile < 0) break;
            // claim the next unit now; its round trip overlaps this one's loads
            const int next = dyn ? static_cast<int>(gridDim.x) + atomicAdd(p.tile_counter, 1)
                                 : tile + static_cast<int>(gridDim.x);
            Piece pc[2];
            const int np = unit_pieces(p, tile, pc);
            for (int pi = 0; pi < np; ++pi) {
                int tm, tn;
                tile_coords(p, pc[pi].tile, tm, tn);
                for (int kb = pc[pi].kb0; kb < pc[pi].kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], K::STAGE);
                    tma_load_2d(smem_a + stage * K::A_STAGE, &map_a, &full[stage], kb * BK, tm * BM, keep);
                    tma_load_2d(smem_b + stage * K::B_STAGE, &map_b, &full[stage], kb * BK, tn * BN, keep);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            tile = next;
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
        const uint32_t a0 = smem_u32(smem_a), b0 = smem_u32(smem_b);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            mbar_wait(&tile_full[r], (i / TILE_RING) & 1);
            const int tile = tile_ring[r];
            mbar_arrive(&tile_empty[r]);
            if (tile < 0) break;
            Piece pc[2];
            const int np = unit_pieces(p, tile, pc);
            for (int pi = 0; pi < np; ++pi) {
                mbar_wait(&acc_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = pc[pi].kb0; kb < pc[pi].kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = a0 + stage * K::A_STAGE;
                    const uint32_t b_addr = b0 + stage * K::B_STAGE;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        // advancing K inside the 128-byte swizzle atom = +32 B (16 bf16, one UMMA K) per MMA
                        umma_bf16(d_tmem, smem_desc_k_sw128(a_addr + k * 32), smem_desc_k_sw128(b_addr + k * 32),
                                  idesc, (kb != pc[pi].kb0 || k != 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&acc_full[acc]);  // accumulator tile (piece) complete
                if (++acc == ACC_BUFS) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> bf16 -> global ----------------
        const int q = warp - 4;                 // TMEM lane quarter
        const int row_in_tile = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int r = i % TILE_RING;
            mbar_wait(&tile_full[r], (i / TILE_RING) & 1);
            const int tile = tile_ring[r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&tile_empty[r]);
            if (tile < 0) break;
            Piece pc[2];
            const int np = unit_pieces(p, tile, pc);
            for (int pi = 0; pi < np; ++pi) {
                int tm, tn;
                tile_coords(p, pc[pi].tile, tm, tn);
                mbar_wait(&acc_full[acc], acc_phase);
                tc_fence_after();
                const int row = tm * BM + row_in_tile;
                const bool row_ok = row < p.m;
                const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                       static_cast<uint32_t>(acc * BN);
                __nv_bfloat16* crow = static_cast<__nv_bfloat16*>(p.c) + static_cast<size_t>(row) * p.ldc;
                // 32 fp32 columns -> bf16 (one rounding) -> this row of C
                auto store32 = [&](const float (&f)[32], int col) {
                    if (!row_ok) return;
                    if (col + 32 <= p.n) {
                        uint4* dst = reinterpret_cast<uint4*>(crow + col);
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            dst[j] = make_uint4(pack_bf16x2(__float_as_uint(f[8 * j]), __float_as_uint(f[8 * j + 1])),
                                                pack_bf16x2(__float_as_uint(f[8 * j + 2]), __float_as_uint(f[8 * j + 3])),
                                                pack_bf16x2(__float_as_uint(f[8 * j + 4]), __float_as_uint(f[8 * j + 5])),
                                                pack_bf16x2(__float_as_uint(f[8 * j + 6]), __float_as_uint(f[8 * j + 7])));
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col + j < p.n) crow[col + j] = __float2bfloat16_rn(f[j]);
                    }
                };
                const bool whole = pc[pi].kb0 == 0 && pc[pi].kb1 == p.k_blocks;
                if (whole) {
#pragma unroll 1
                    for (int c = 0; c < BN; c += 32) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(t_row + c, v);
                        tmem_ld_wait();
                        float f[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                        store32(f, tn * BN + c);
                    }
                    tc_fence_before();
                    mbar_arrive(&acc_empty[acc]);
                } else {
                    // a stream-K tile in pieces: every piece but the last to arrive
                    // publishes its fp32 partial; the last waits for them (their
                    // epilogues already counted, and wait on nothing), sums all in
                    // piece order (its own from TMEM) and rounds once: the result
                    // does not depend on arrival order
                    const Piece& pce = pc[pi];
                    const int tt = pce.tile - p.full_units;
                    named_bar_sync(1, 128);  // every epilogue thread read the previous sk_flag
                    if (threadIdx.x == 128)
                        st_shared_u32(sk_flag, atomicAdd(p.sk_done + tt, 1) == pce.count - 1 ? 1u : 0u);
                    named_bar_sync(1, 128);
                    const size_t slot_f4 = static_cast<size_t>(BN / 4) * BM;
                    float4* slots = p.sk_ws + static_cast<size_t>(tt) * kSkMaxPieces * slot_f4 + row_in_tile;
                    if (!ld_volatile_shared(sk_flag)) {
                        float4* mine = slots + pce.idx * slot_f4;
#pragma unroll 1
                        for (int c = 0; c < BN; c += 32) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(t_row + c, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                mine[(c / 4 + j) * BM] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                                     __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                        }
                        tc_fence_before();
                        mbar_arrive(&acc_empty[acc]);
                        __threadfence();  // the partial is visible before it is counted ready
                        named_bar_sync(1, 128);
                        if (threadIdx.x == 128) atomicAdd(p.sk_ready + tt, 1);
                    } else {
                        if (threadIdx.x == 128)
                            wait_ge_gpu(p.sk_ready + tt, pce.count - 1);
                        named_bar_sync(1, 128);
                        __threadfence();
#pragma unroll 1
                        for (int c = 0; c < BN; c += 32) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(t_row + c, v);
                            tmem_ld_wait();
                            float f[32];
                            // fixed order: piece 0, 1, ... (own at its index); each
                            // other piece's 8 vectors as one batch of loads
#pragma unroll
                            for (int q_idx = 0; q_idx < kSkMaxPieces; ++q_idx) {
                                if (q_idx >= pce.count) continue;
                                float4 t[8];
                                if (q_idx == pce.idx) {
#pragma unroll
                                    for (int j = 0; j < 8; ++j)
                                        t[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                           __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                                } else {
#pragma unroll
                                    for (int j = 0; j < 8; ++j) t[j] = ld_cg_f4(slots + q_idx * slot_f4 + (c / 4 + j) * BM);
                                }
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    if (q_idx == 0) {
                                        f[4 * j] = t[j].x;
                                        f[4 * j + 1] = t[j].y;
                                        f[4 * j + 2] = t[j].z;
                                        f[4 * j + 3] = t[j].w;
                                    } else {
                                        f[4 * j] += t[j].x;
                                        f[4 * j + 1] += t[j].y;
                                        f[4 * j + 2] += t[j].z;
                                        f[4 * j + 3] += t[j].w;
                                    }
                                }
                            }
                            store32(f, tn * BN + c);
                        }
                        tc_fence_before();
                        mbar_arrive(&acc_empty[acc]);
                        if (threadIdx.x == 128) {  // for the next launch (no one else touches them now)
                            p.sk_done[tt] = 0;
                            p.sk_ready[tt] = 0;
                        }
                    }
                }
                if (++acc == ACC_BUFS) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<K::TMEM_COLS>(tmem_base);
    }
    // Last CTA out resets the claim counter for the next launch (every CTA's
    // claimer has drawn its terminal ticket before its CTA reaches here).
    if (threadIdx.x == 0 && p.tile_counter != nullptr) {
        __threadfence();
        if (atomicAdd(p.exit_counter, 1) == static_cast<int>(gridDim.x) - 1) {
            *p.tile_counter = 0;
            *p.exit_counter = 0;
            __threadfence();
        }
    }
}

}  // namespace gemm

// ----------------------------------------------------------------- host ---

namespace {

// K-major [rows, k] operand in boxes of one 128-byte swizzle row (64 bf16 or
// 32 fp32 elements) x box_rows
CUresult encode_kmajor_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t k,
                            uint32_t box_rows, int elem = 2) {
    const cuuint64_t dims[2] = {k, rows};
    const cuuint64_t strides[1] = {k * static_cast<uint64_t>(elem)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / elem), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    if (!drv().TensorMapEncodeTiled) return CUDA_ERROR_NOT_SUPPORTED;
    return drv().TensorMapEncodeTiled(map, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                      2, const_cast<void*>(ptr),
                                      dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <int BN>
int launch_bn(const GemmPlan* plan, const CUtensorMap& map_b, int grid, cudaStream_t stream) {
    using K = gemm::Cfg<BN>;
    static bool attr_done = false;
    if (!attr_done) {
        const cudaError_t e = cudaFuncSetAttribute(gemm::gemm_bf16_tn_kernel<BN>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(K::SMEM));
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm)");
        attr_done = true;
    }
    gemm::Params p;
    p.m = static_cast<int>(plan->m);
    p.n = static_cast<int>(plan->n);
    p.k = static_cast<int>(plan->k);
    p.tiles_m = static_cast<int>((plan->m + gemm::BM - 1) / gemm::BM);
    p.tiles_n = static_cast<int>((plan->n + BN - 1) / BN);
    p.num_tiles = p.tiles_m * p.tiles_n;
    p.k_blocks = plan->k_blocks;
    p.c = plan->c;
    p.ldc = static_cast<int>(plan->n);
    static const bool static_sched = [] {
        const char* e = std::getenv("C3_GEMM_SCHED");  // development A/B switch
        return e != nullptr && std::string(e) == "static";
    }();
    p.tile_counter = static_sched ? nullptr : plan->counters;
    p.exit_counter = plan->counters + 1;
    // Stream-K tail: when the tiles leave the last wave of the full GPU partly
    // empty, that wave's k-blocks are spread evenly over one segment per SM.
    // Decided from the SM count alone (not the grid), so the result bits do
    // not depend on the CTA cap. Segments of g >= (k - 1) / 3 k-blocks keep a
    // tile to at most kSkMaxPieces pieces (C3_GEMM_STREAMK=0: off, dev A/B).
    // Compute-bound GEMMs only (>= 200 FLOP per operand/output byte): a
    // memory-bound one's last wave already streams at the HBM rate with fewer
    // SMs, and the fix-up only adds traffic (measured, ncu: 256x4096x16384
    // 81.7 -> 56.4 us; 128x53248x16384 279.6 -> 284.3 us, so off there).
    static const bool streamk = [] {
        const char* e = std::getenv("C3_GEMM_STREAMK");
        return !(e != nullptr && std::string(e) == "0");
    }();
    const int segs = plan->sk_capacity;
    const int waves = p.num_tiles / segs, tail = p.num_tiles - waves * segs;
    const int64_t seg_kb = static_cast<int64_t>(tail) * p.k_blocks / segs;
    p.full_units = p.num_units = p.num_tiles;
    p.sk_segs = 0;
    p.sk_kb = 0;
    const double flops = 2.0 * static_cast<double>(plan->m) * plan->n * plan->k;
    const double bytes = 2.0 * (static_cast<double>(plan->m) * plan->k + static_cast<double>(plan->n) * plan->k +
                                static_cast<double>(plan->m) * plan->n);
    const bool compute_bound = flops >= 200.0 * bytes;
    if (streamk && compute_bound && plan->ws && tail > 0 && p.k_blocks >= 2 && seg_kb >= 1 &&
        p.k_blocks - 2 < 3 * seg_kb) {
        p.full_units = waves * segs;
        p.sk_segs = segs;
        p.num_units = p.full_units + segs;
        p.sk_kb = static_cast<int64_t>(tail) * p.k_blocks;
        p.sk_done = static_cast<int*>(plan->ws);
        p.sk_ready = p.sk_done + plan->sk_capacity;
        p.sk_ws = reinterpret_cast<float4*>(static_cast<uint8_t*>(plan->ws) + gemm_sk_counter_bytes(plan->sk_capacity));
    }
    grid = std::min(grid, p.num_units);
    gemm::gemm_bf16_tn_kernel<BN><<<grid, gemm::THREADS, K::SMEM, stream>>>(plan->map_a, map_b, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
    return C3_OK;
}

}  // namespace

int gemm_pair_launch(const GemmPlan* plan, int grid, cudaStream_t stream, const FusedComm* fc,
                     const RowGate* gate);
int gemm_f32_launch(const GemmPlan* plan, int grid, cudaStream_t stream);

// Kernel choice: CTA-pair 256x512, else 256x256 tiles when there is at least
// one pair tile per SM pair; else single-CTA 128x256 tiles, or 128x128 when
// that leaves fewer than two tiles per SM (e.g. M=128: 208 -> 416 tiles).
// 256x512 pair tiles when every SM pair gets one: 25% less L2->SM operand
// traffic than 256x256, which the 1 kW power cap turns into clock
// (sustained cfg2 / 8192^3 / cfg4: +3% / +4% / +7%, profiles/r01_gemm_pair512_ab.txt).
// fp32: 128 x 128 tiles of the split-TF32 kernel (gemm_f32.cu).
GemmPlan::Kind gemm_kind(int64_t m, int64_t n, int elem_bytes, int sm_count) {
    if (elem_bytes == 4) return GemmPlan::kNarrow;
    const int64_t sms = std::max(sm_count, 2);
    const int64_t tm1 = (m + 127) / 128;
    const int64_t pair_tiles = ((m + 255) / 256) * ((n + 255) / 256);
    const int64_t pair512_tiles = ((m + 255) / 256) * ((n + 511) / 512);
    GemmPlan::Kind kind = m >= 256 && pair512_tiles >= sms / 2 ? GemmPlan::kPair512
                          : m >= 256 && pair_tiles >= sms / 2 ? GemmPlan::kPair
                          : tm1 * ((n + 255) / 256) < 2 * sms ? GemmPlan::kNarrow
                                                              : GemmPlan::kWide;
    if (const char* f = std::getenv("C3_GEMM_KERNEL")) {  // tests force each variant
        const std::string v(f);
        if (v == "pair") kind = GemmPlan::kPair;
        if (v == "pair512") kind = GemmPlan::kPair512;
        if (v == "wide") kind = GemmPlan::kWide;
        if (v == "narrow") kind = GemmPlan::kNarrow;
    }
    return kind;
}

int64_t gemm_workspace_zero_bytes(int64_t m, int64_t n, int64_t k, int elem_bytes, int sm_count) {
    if (elem_bytes == 4) {
        const int64_t tiles = ((m + 127) / 128) * ((n + 127) / 128);  // the fp32 kernel's 128 x 128 tiles
        return std::min(gemm_f32_workspace_bytes(m, n, k, sm_count), (2 * tiles * 4 + 255) / 256 * 256);
    }
    return gemm_workspace_bytes(m, n, k, elem_bytes, sm_count) > 0 ? gemm_sk_counter_bytes(sm_count) : 0;
}

int64_t gemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int elem_bytes, int sm_count) {
    if (elem_bytes == 4) return gemm_f32_workspace_bytes(m, n, k, sm_count);
    const GemmPlan::Kind kind = gemm_kind(m, n, elem_bytes, sm_count);
    if (kind != GemmPlan::kNarrow && kind != GemmPlan::kWide) return 0;
    const int64_t bn = kind == GemmPlan::kNarrow ? 128 : 256;
    // stream-K: a partial per tail tile, fewer tail tiles than CTAs (<= SMs)
    return gemm_sk_counter_bytes(sm_count) + static_cast<int64_t>(sm_count) * gemm::kSkMaxPieces * gemm::BM * bn * 4;
}

int gemm_plan_init(GemmPlan* plan, const void* A, const void* B, void* C, int64_t m, int64_t n,
                   int64_t k, int* counters, int sm_count, int elem_bytes, void* ws) {
    if (elem_bytes != 2 && elem_bytes != 4)
        return set_error(C3_ERR_VALIDATION, "gemm: element size must be 2 (bf16) or 4 (fp32, split-TF32)");
    if (elem_bytes == 4 && !ws)
        return set_error(C3_ERR_VALIDATION, "gemm: an fp32 plan needs a workspace (gemm_workspace_bytes)");
    const int64_t row_elems = 16 / elem_bytes;
    if (m < 1 || n < 1 || k < 1) return set_error(C3_ERR_VALIDATION, "gemm: dimensions must be >= 1");
    if (k % row_elems != 0) return set_error(C3_ERR_VALIDATION, "gemm: K rows must be a multiple of 16 bytes");
    if (n % row_elems != 0) return set_error(C3_ERR_VALIDATION, "gemm: N rows must be a multiple of 16 bytes");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
        return set_error(C3_ERR_VALIDATION, "gemm: operands must be 16-byte aligned");
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX)
        return set_error(C3_ERR_VALIDATION, "gemm: dimension too large");
    if (!counters) return set_error(C3_ERR_VALIDATION, "gemm: missing tile-claim counters");
    plan->kind = gemm_kind(m, n, elem_bytes, sm_count);
    // fp32: the raw operands (the split happens in shared memory)
    plan->ws = ws;  // fp32: split-K words; bf16 single-CTA kinds: stream-K (nullptr: off)
    plan->sk_capacity = std::max(sm_count, 2);
    plan->f32_splits = elem_bytes == 4 ? gemm_f32_splits(m, n, k, sm_count) : 1;
    CUresult r = encode_kmajor_bf16(&plan->map_a, A, static_cast<uint64_t>(m), static_cast<uint64_t>(k), 128,
                                    elem_bytes);
    if (r == CUDA_SUCCESS)  // 128-row B boxes: the pair kernel's half tile and the narrow kernel
        r = encode_kmajor_bf16(&plan->map_b128, B, static_cast<uint64_t>(n), static_cast<uint64_t>(k), 128,
                               elem_bytes);
    if (r == CUDA_SUCCESS && elem_bytes == 2)
        r = encode_kmajor_bf16(&plan->map_b256, B, static_cast<uint64_t>(n), static_cast<uint64_t>(k), 256);
    // C [m, n] in 32-row boxes of one 128-byte swizzle row (64 bf16 / 32 fp32
    // columns): the TMA-store epilogues of the pair kernels and the fp32 kernel
    if (r == CUDA_SUCCESS)
        r = encode_kmajor_bf16(&plan->map_c, C, static_cast<uint64_t>(m), static_cast<uint64_t>(n), 32, elem_bytes);
    if (r != CUDA_SUCCESS) return set_driver_error(r, "cuTensorMapEncodeTiled");
    plan->m = m;
    plan->n = n;
    plan->k = k;
    plan->c = C;
    plan->counters = counters;
    plan->elem = elem_bytes;
    const int bke = elem_bytes == 4 ? 32 : gemm::BK;  // 128-byte K rows
    plan->k_blocks = static_cast<int>((k + bke - 1) / bke);
    const bool pair = plan->kind == GemmPlan::kPair || plan->kind == GemmPlan::kPair512;
    const int bm = pair ? 256 : 128;
    const int bn = plan->kind == GemmPlan::kNarrow ? 128 : plan->kind == GemmPlan::kPair512 ? 512 : 256;
    plan->tiles_m = static_cast<int>((m + bm - 1) / bm);
    plan->tiles_n = static_cast<int>((n + bn - 1) / bn);
    plan->num_tiles = plan->tiles_m * plan->tiles_n;
    return C3_OK;
}

int gemm_plan_launch(const GemmPlan* plan, int max_ctas, int sm_count, cudaStream_t stream,
                     const FusedComm* fc, const RowGate* gate) {
    int grid = max_ctas > 0 ? max_ctas : sm_count;
    grid = std::min(grid, sm_count);
    const bool pair = plan->kind == GemmPlan::kPair || plan->kind == GemmPlan::kPair512;
    if (fc && (!pair || grid < 2))
        return set_error(C3_ERR_UNSUPPORTED, "fused C3 needs the CTA-pair GEMM (M >= 256, enough tiles)");
    if (pair && grid >= 2) {
        // whole CTA pairs; a fused launch keeps every pair (its copy warps move data)
        grid = fc ? grid / 2 * 2 : std::min(grid / 2, plan->num_tiles) * 2;
        return gemm_pair_launch(plan, grid, stream, fc, gate);
    }
    if (plan->elem == 4) {
        if (gate && gate->flags) return set_error(C3_ERR_UNSUPPORTED, "row-gated GEMM needs the CTA-pair kernel");
        return gemm_f32_launch(plan, grid, stream);
    }
    if (gate && gate->flags) return set_error(C3_ERR_UNSUPPORTED, "row-gated GEMM needs the CTA-pair kernel");
    if (plan->kind == GemmPlan::kWide) return launch_bn<256>(plan, plan->map_b256, grid, stream);
    return launch_bn<128>(plan, plan->map_b128, grid, stream);  // narrow, or a 1-SM cap
}

}  // namespace c3k
