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
constexpr int UK = 16;           // UMMA K for 16-bit inputs
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
};

__device__ __forceinline__ void tile_coords(const Params& p, int tile, int& tm, int& tn) {
    const int band = GROUP_M * p.tiles_n;
    const int first_m = (tile / band) * GROUP_M;
    const int rows = min(p.tiles_m - first_m, GROUP_M);
    const int in_band = tile % band;
    tm = first_m + in_band % rows;
    tn = in_band / rows;
}

template <int BN>
__global__ void __launch_bounds__(THREADS, 1)
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
            if (tile >= p.num_tiles) tile = -1;
            mbar_wait(&tile_empty[r], ((i / TILE_RING) & 1) ^ 1);
            tile_ring[r] = tile;
            mbar_arrive(&tile_full[r]);  // release: consumers read tile_ring[r] after their wait
            if (tile < 0) break;
            // claim the next tile now; its round trip overlaps this tile's loads
            const int next = dyn ? static_cast<int>(gridDim.x) + atomicAdd(p.tile_counter, 1)
                                 : tile + static_cast<int>(gridDim.x);
            int tm, tn;
            tile_coords(p, tile, tm, tn);
            for (int kb = 0; kb < p.k_blocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_arrive_expect_tx(&full[stage], K::STAGE);
                tma_load_2d(smem_a + stage * K::A_STAGE, &map_a, &full[stage], kb * BK, tm * BM, keep);
                tma_load_2d(smem_b + stage * K::B_STAGE, &map_b, &full[stage], kb * BK, tn * BN, keep);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
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
            mbar_wait(&acc_empty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kb = 0; kb < p.k_blocks; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t a_addr = a0 + stage * K::A_STAGE;
                const uint32_t b_addr = b0 + stage * K::B_STAGE;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // advancing K inside the 128-byte swizzle atom = +32 B (16 bf16) per MMA
                    umma_bf16(d_tmem, smem_desc_k_sw128(a_addr + k * 32), smem_desc_k_sw128(b_addr + k * 32),
                              idesc, (kb | k) != 0);
                }
                umma_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            umma_commit(&acc_full[acc]);  // accumulator tile complete
            if (++acc == ACC_BUFS) {
                acc = 0;
                acc_phase ^= 1;
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
            int tm, tn;
            tile_coords(p, tile, tm, tn);
            mbar_wait(&acc_full[acc], acc_phase);
            tc_fence_after();
            const int row = tm * BM + row_in_tile;
            const bool row_ok = row < p.m;
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(t_row + c, v);
                tmem_ld_wait();
                const int col = tn * BN + c;
                if (!row_ok) continue;
                __nv_bfloat16* crow = static_cast<__nv_bfloat16*>(p.c) + static_cast<size_t>(row) * p.ldc;
                if (col + 32 <= p.n) {
                    uint4* dst = reinterpret_cast<uint4*>(crow + col);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint4 o;
                        __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
                        __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                        __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                        o.x = *reinterpret_cast<uint32_t*>(&h0);
                        o.y = *reinterpret_cast<uint32_t*>(&h1);
                        o.z = *reinterpret_cast<uint32_t*>(&h2);
                        o.w = *reinterpret_cast<uint32_t*>(&h3);
                        dst[j] = o;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (col + j < p.n) crow[col + j] = __float2bfloat16_rn(__uint_as_float(v[j]));
                }
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[acc]);
            if (++acc == ACC_BUFS) {
                acc = 0;
                acc_phase ^= 1;
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
    grid = std::min(grid, p.num_tiles);
    gemm::gemm_bf16_tn_kernel<BN><<<grid, gemm::THREADS, K::SMEM, stream>>>(plan->map_a, map_b, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
    return C3_OK;
}

}  // namespace

int gemm_pair_launch(const GemmPlan* plan, int grid, cudaStream_t stream, const FusedComm* fc,
                     const RowGate* gate);
int gemm_f32_launch(const GemmPlan* plan, int grid, cudaStream_t stream);

int gemm_plan_init(GemmPlan* plan, const void* A, const void* B, void* C, int64_t m, int64_t n,
                   int64_t k, int* counters, int sm_count, int elem_bytes, void* f32_ws) {
    if (elem_bytes != 2 && elem_bytes != 4)
        return set_error(C3_ERR_VALIDATION, "gemm: element size must be 2 (bf16) or 4 (fp32, split-TF32)");
    if (elem_bytes == 4 && !f32_ws)
        return set_error(C3_ERR_VALIDATION, "gemm: an fp32 plan needs a workspace (gemm_f32_workspace_bytes)");
    const int64_t row_elems = 16 / elem_bytes;
    if (m < 1 || n < 1 || k < 1) return set_error(C3_ERR_VALIDATION, "gemm: dimensions must be >= 1");
    if (k % row_elems != 0) return set_error(C3_ERR_VALIDATION, "gemm: K rows must be a multiple of 16 bytes");
    if (n % row_elems != 0) return set_error(C3_ERR_VALIDATION, "gemm: N rows must be a multiple of 16 bytes");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
        return set_error(C3_ERR_VALIDATION, "gemm: operands must be 16-byte aligned");
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX)
        return set_error(C3_ERR_VALIDATION, "gemm: dimension too large");
    if (!counters) return set_error(C3_ERR_VALIDATION, "gemm: missing tile-claim counters");
    // Kernel choice: CTA-pair 256x512, else 256x256 tiles when there is at
    // least one pair tile per SM pair; else single-CTA 128x256 tiles, or
    // 128x128 when that leaves fewer than two tiles per SM (e.g. M=128: 208 ->
    // 416 tiles).
    const int64_t sms = std::max(sm_count, 2);
    const int64_t tm1 = (m + 127) / 128;
    const int64_t pair_tiles = ((m + 255) / 256) * ((n + 255) / 256);
    const int64_t pair512_tiles = ((m + 255) / 256) * ((n + 511) / 512);
    // 256x512 pair tiles when every SM pair gets one: 25% less L2->SM operand
    // traffic than 256x256, which the 1 kW power cap turns into clock
    // (sustained cfg2 / 8192^3 / cfg4: +3% / +4% / +7%, profiles/r01_gemm_pair512_ab.txt)
    plan->kind = m >= 256 && pair512_tiles >= sms / 2 ? GemmPlan::kPair512
                 : m >= 256 && pair_tiles >= sms / 2 ? GemmPlan::kPair
                 : tm1 * ((n + 255) / 256) < 2 * sms ? GemmPlan::kNarrow
                                                     : GemmPlan::kWide;
    if (elem_bytes == 4)  // fp32: 128 x 128 tiles of the split-TF32 kernel (gemm_f32.cu)
        plan->kind = GemmPlan::kNarrow;
    if (const char* f = std::getenv("C3_GEMM_KERNEL"); f && elem_bytes == 2) {  // tests force each variant
        const std::string v(f);
        if (v == "pair") plan->kind = GemmPlan::kPair;
        if (v == "pair512") plan->kind = GemmPlan::kPair512;
        if (v == "wide") plan->kind = GemmPlan::kWide;
        if (v == "narrow") plan->kind = GemmPlan::kNarrow;
    }
    // fp32: the raw operands (the split happens in shared memory)
    plan->f32_ws = elem_bytes == 4 ? f32_ws : nullptr;
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
