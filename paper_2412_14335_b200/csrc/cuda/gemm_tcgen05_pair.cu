// CTA-pair variant of the persistent bf16 GEMM (tcgen05 cta_group::2).
//
// A cluster of two CTAs on one TPC computes a 256 x 256 output tile. Each CTA
// TMA-loads its own 128 rows of A and its half (128 rows) of the tile's B
// rows; the even ("leader") CTA issues tcgen05.mma.cta_group::2 with M = 256,
// which reads A and B from BOTH CTAs' shared memory (identical offsets) and
// accumulates each CTA's 128 rows x 256 columns into that CTA's own TMEM.
// Versus the single-CTA 128 x 256 tile this halves the B bytes each SM pulls
// from L2 per MMA (32 KiB instead of 48 KiB per 64-deep k-block): the
// single-CTA kernel's tensor pipe sat at 88% with ~2.9 GB of DRAM traffic
// per cfg2 launch (profiles/ncu_gemm_summary.json).
//
// Synchronisation (all mbarriers, no __syncthreads in the main loop):
//   full[s]     leader only; leader arms expect_tx(2 x stage bytes), both CTAs'
//               TMA loads complete_tx on it (peer bit of the address cleared)
//   empty[s]    both CTAs; the leader's tcgen05.commit multicasts to both
//   acc_full[b] both CTAs; multicast commit after a tile's last k-block
//   acc_h0      both CTAs (BN 512); multicast commit once half 0 of the tile is
//               final: with the tail lag, L k-blocks before half 1 is
//   acc_empty[b] leader; EPI_WARPS local + EPI_WARPS remote epilogue-warp arrivals
//               (BN 512: one barrier per 256-column half of the accumulator)
//   tile ring   leader claims tiles (global atomic, one tile ahead), writes
//               the id into both CTAs' rings (st.shared::cluster) and arrives
//               on both tile_full; consumers of both CTAs release the slot on
//               the leader's tile_empty (1 MMA + EPI_WARPS + 1 peer producer
//               + EPI_WARPS).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "c3cuda_internal.hpp"
#include "ptx.cuh"

namespace c3k {
namespace gemm2 {

constexpr int BM = 256;        // pair tile rows (128 per CTA)
constexpr int BK = 64;
constexpr int UK = 16;
// Pair-rows per raster band (C3_GEMM_BAND env overrides, dev A/B). Measured
// DRAM reads per cfg2 launch: band 8 -> 2.39 GB, 16 -> 3.85 GB, 32 -> 12.3 GB
// (profiles/r01_gemm_band_ab.txt): the L2 is split across the two dies, so a
// band's A slice must stay well under the nominal 126 MB.
constexpr int GROUP_M_DEFAULT = 8;
constexpr int RING = 4;
constexpr int kPreHalf = 4;  // BN 512: k-blocks issued into half 0 before half 1 is free (C3_GEMM_PREHALF; measured 1-4: 92.2 -> 93.1% tensor pipe)
// BN 512 tail lag (C3_GEMM_TAILLAG): the last L k-blocks of a tile run half 0
// first and half 1 after, so half 0 is final (and its drain starts) L k-blocks
// of MMA work before the tile ends. With the pre k-blocks at the next tile's
// start this hides the drain of both halves behind MMAs; without it the next
// tile waited for the whole half-0 drain (profiles/r02_gemm_drain_release_ab.txt:
// releasing the accumulator early is worth 0.8% burst / 2% sustained on cfg2).
constexpr int kTailLag = 4;
constexpr uint32_t A_STAGE = 128 * BK * 2;  // this CTA's 128 rows of A
constexpr uint32_t B_HALF = 128 * BK * 2;   // this CTA's 128 rows of one 256-column half of B
constexpr uint32_t TMEM_COLS = 512;
// fused C3: two 16 KiB copy buffers in the shared memory the GEMM leaves free
constexpr uint32_t PIECE = 8 * 1024;
// epilogue staging per warp: 32 rows x 64 bf16 columns
constexpr uint32_t kEpiWarpStage = 32 * 128;

// Pair tile 256 x BN. BN = 256: two TMEM accumulators (the epilogue of tile i
// overlaps the MMAs of tile i+1), 6 stages. BN = 512: one accumulator filling
// all 512 TMEM columns (the epilogue is exposed), 4 stages, but each k-block
// moves 48 KiB of operands per CTA for 2x the MMA work of a 256-wide tile
// (64 KiB per 256x256x64 -> 48 KiB): 25% less L2->SM traffic, which under
// the 1 kW power cap is clock (profiles/r01_ncu_gemm_vs_cublas.txt).
template <int BN_, bool FUSED_ = false>
struct PairCfg {
    static constexpr int BN = BN_;
    static constexpr int HALVES = BN / 256;  // N=256 MMAs per k-step
    // fused 512-wide: one operand stage fewer buys the copy warp a 64 KiB ring
    // (the fused all-to-all is latency-bound on its copy slots)
    static constexpr int STAGES = BN == 256 ? 6 : (FUSED_ ? 3 : 4);
    static constexpr int ACC_BUFS = BN == 256 ? 2 : 1;
    // epilogue warps (one per TMEM lane quadrant; 8 = two per quadrant, each
    // half the columns, measured no faster for 512-wide tiles)
    static constexpr int EPI_WARPS = 4;
    static constexpr int THREADS = 128 + 32 * EPI_WARPS;
    static constexpr uint32_t B_STAGE = HALVES * B_HALF;
    static constexpr uint32_t STAGE = A_STAGE + B_STAGE;
    // C staging: two tiles per epilogue warp (one when fused: the copy
    // buffers take the other's shared memory)
    static constexpr uint32_t EPI_SMEM = EPI_WARPS * kEpiWarpStage;
    static constexpr uint32_t SMEM = STAGES * STAGE + 1024 + 2 * EPI_SMEM + 512;
    // fused: the copy warp's slot ring after one staging tile per epilogue warp
    static constexpr uint32_t COPY_BYTES = BN == 512 && FUSED_ ? 64 * 1024 : 2 * PIECE;
    static constexpr uint32_t SMEM_FUSED = STAGES * STAGE + 1024 + EPI_SMEM + 512 + COPY_BYTES + 64;
    static_assert(SMEM <= 227 * 1024 && SMEM_FUSED <= 227 * 1024, "shared memory");
    static_assert(ACC_BUFS * BN <= static_cast<int>(TMEM_COLS), "TMEM");
    static_assert(BN / (EPI_WARPS / 4) % 128 == 0, "epilogue drains 128 columns per step");
};

struct Params {
    int m, n, k;
    int tiles_m, tiles_n, num_tiles, k_blocks;
    __nv_bfloat16* c;
    int ldc;
    int* tile_counter;
    int* exit_counter;
    int group_m;
    int pol_a, pol_b;  // L2 policy of the A / B operand loads (policy_by_kind)
    int pol_c;         // L2 policy hint of the C stores (0: none)
    int pre_half;      // BN 512: k-blocks into half 0 before waiting for half 1 (<= STAGES)
    int tail_lag;      // BN 512: last k-blocks whose half-1 MMAs follow the half-0 ones (<= STAGES)
    // BN 512 tail split: claims u < full_tiles are whole tiles; the last
    // num_tiles - full_tiles tiles are claimed as two 256-column halves each
    // (u in [full_tiles, num_units)), so an underfilled last wave takes half a
    // tile's time. full_tiles = num_units = num_tiles when not split.
    int full_tiles, num_units;
    RowGate gate;  // A rows landing during the launch (flags == nullptr: all resident)
    // dev A/B only (C3_GEMM_DEV, results invalid when set): bit 0 every tile
    // loads the operands of tile (0, 0) (L2-resident: the cost of DRAM traffic),
    // bit 1 the epilogue releases the accumulator without draining it (the
    // cost of the exposed TMEM drain), bit 2 / bit 3 (512-wide) it releases
    // half 0 / both halves as soon as the tile is done and drains after (the
    // gain a hidden drain would bring, with the drain's own work kept)
    int dev;
    FusedComm fc;  // only read by the FUSED instantiation
};

// Wait until A's row band `band` has landed (RowGate). Bounded: after 2 s the
// producer records the timeout and proceeds (the host then fails the step)
// rather than hang the GPU on a flag that never comes.
__device__ __forceinline__ void wait_row_band(const RowGate& g, int band) {
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(g.flags + band) < g.epoch) {
        if (global_ns() - t0 > 2000000000ull) {
            if (g.timed_out) st_release_sys(g.timed_out, kWaitRowGate);  // the host fails the step loudly
            break;
        }
        __nanosleep(500);
    }
    fence_proxy_async_global();  // the TMA loads that follow read what the flag published
}

// claim u -> tile and half (-1 = the whole tile, 0/1 = its 256-column half)
__device__ __forceinline__ void unit_tile(const Params& p, int u, int& tile, int& half) {
    if (u < p.full_tiles) {
        tile = u;
        half = -1;
    } else {
        tile = p.full_tiles + (u - p.full_tiles) / 2;
        half = (u - p.full_tiles) % 2;
    }
}

__device__ __forceinline__ void tile_coords(const Params& p, int tile, int& tm, int& tn) {
    const int band = p.group_m * p.tiles_n;
    const int first_m = (tile / band) * p.group_m;
    const int rows = min(p.tiles_m - first_m, p.group_m);
    const int in_band = tile % band;
    tm = first_m + in_band % rows;
    tn = in_band / rows;
}

// Fused C3 copy engine (warp 3, one thread, FUSED only): this rank's share of
// the collective moved by the SM's own TMA unit with bulk async copies —
// global -> shared ring -> every destination (local or NVLink peer). The
// 2 x PIECE bytes of copy buffer are cut into nb = 2 x PIECE / piece slots
// (<= kFusedSlots), and loads run nb-1 items ahead of the stores, so an
// all-to-all (one store per load) is not bound by one load round trip per
// piece. Item k of this CTA's `mine` items starts once the CTA's producer has
// issued k/mine * pace of its expected k-blocks (pace > 0). Work items are
// spread round-robin over the grid. AG: item = (rank v, piece j), one load,
// n-1 stores; A2A: item = (v, dest q, piece j), one load, one store.
constexpr int kFusedSlots = 8;
__device__ void fused_copy_loop(const Params& p, uint8_t* buf, uint32_t buf_bytes, uint64_t* lbar,
                                const uint32_t* progress, const volatile uint32_t* producer_done) {
    const FusedComm& fc = p.fc;
    const uint64_t pol = policy_evict_first();
    const int64_t piece = fc.piece;  // <= buf_bytes / 2
    const int nb = static_cast<int>(min(static_cast<int64_t>(kFusedSlots), static_cast<int64_t>(buf_bytes) / piece));
    const int64_t pieces = (fc.chunk + piece - 1) / piece;
    const int nv = fc.self_end - fc.self_begin;
    const int64_t per_v = fc.kind == 0 ? pieces : pieces * fc.n;
    const int64_t total = per_v * nv;
    const int64_t G = gridDim.x;
    const int64_t mine = total > blockIdx.x ? (total - blockIdx.x + G - 1) / G : 0;
    // expected producer k-blocks of this CTA over the GEMM (pair tiles / pairs)
    const double est_kb = static_cast<double>((p.num_tiles + G / 2 - 1) / (G / 2)) * p.k_blocks;
    const int targets = fc.kind == 0 ? (fc.skip_self ? fc.n - 1 : fc.n) : 1;
    struct Item {
        int v, q;
        int64_t off;
        uint32_t len;
    };
    // item k -> (rank, destination, offset): 32-bit division (item counts stay
    // far below 2^31; a 64-bit division per item was the copy thread's
    // bottleneck for all-to-all, which has n x the items of an all-gather)
    const bool small = total < (int64_t{1} << 31);
    auto item = [&](int64_t k) {
        const int64_t w = blockIdx.x + k * G;
        Item it;
        int64_t r, jj;
        if (small) {
            const uint32_t w32 = static_cast<uint32_t>(w), pv = static_cast<uint32_t>(per_v);
            const uint32_t pc = static_cast<uint32_t>(pieces);
            it.v = fc.self_begin + static_cast<int>(w32 / pv);
            const uint32_t r32 = w32 % pv;
            it.q = fc.kind == 0 ? -1 : static_cast<int>(r32 / pc);
            r = r32;
            jj = fc.kind == 0 ? r32 : r32 % pc;
        } else {
            it.v = fc.self_begin + static_cast<int>(w / per_v);
            r = w % per_v;
            it.q = fc.kind == 0 ? -1 : static_cast<int>(r / pieces);
            jj = fc.kind == 0 ? r : r % pieces;
        }
        it.off = jj * piece;
        const int64_t left = fc.chunk - it.off;
        it.len = static_cast<uint32_t>(left < piece ? left : piece);
        return it;
    };
    Item slot[kFusedSlots];  // the item in flight in each buffer slot
    auto issue_load = [&](int64_t k, int b) {
        const Item it = item(k);
        slot[b] = it;
        const uint8_t* src = fc.src[it.v] + (fc.kind == 0 ? 0 : static_cast<int64_t>(it.q) * fc.chunk) + it.off;
        mbar_arrive_expect_tx(&lbar[b], it.len);
        bulk_load(buf + b * piece, src, it.len, &lbar[b], pol);
    };
    for (int64_t k = 0; k < nb - 1 && k < mine; ++k) issue_load(k, static_cast<int>(k));
    const uint64_t t0 = global_ns();
    double sent = 0.0;  // peer bytes stored (link emulation)
    int b = 0, refill = nb - 1;  // slot of item k, slot of item k + nb - 1
    uint32_t par = 0;            // mbarrier parity of slot b's current use
    for (int64_t k = 0; k < mine; ++k) {
        const Item it = slot[b];
        if (fc.pace > 0.f) {
            const uint32_t target = static_cast<uint32_t>(est_kb * fc.pace * k / mine);
            while (ld_volatile_shared(progress) < target && !*producer_done) __nanosleep(256);
        }
        if (fc.link_cta_bpns > 0.f) link_wait(t0, sent, fc.link_cta_bpns);
        sent += static_cast<double>(it.len) * (fc.kind == 0 ? targets : (it.q == it.v ? 0 : 1));
        mbar_wait(&lbar[b], par);
        if (fc.kind == 0) {
            for (int t = 1; t <= fc.n; ++t) {
                const int d = (it.v + t) % fc.n;  // rotated targets
                if (d == it.v && fc.skip_self) continue;
                bulk_store(fc.dst[d] + static_cast<int64_t>(it.v) * fc.chunk + it.off, buf + b * piece, it.len, pol);
            }
        } else {
            bulk_store(fc.dst[it.q] + static_cast<int64_t>(it.v) * fc.chunk + it.off, buf + b * piece, it.len, pol);
        }
        bulk_commit();
        // refill slot (k-1) % nb (its stores = group k-1) with item k+nb-1
        if (k + nb - 1 < mine) {
            bulk_wait_read<1>();
            issue_load(k + nb - 1, refill);
        }
        if (++refill == nb) refill = 0;
        if (++b == nb) {
            b = 0;
            par ^= 1;
        }
    }
    bulk_wait_all();
    fence_proxy_async_global();
    if (fc.link_cta_bpns > 0.f) link_wait(t0, sent, fc.link_cta_bpns);  // the last pieces' link time
}

// Fused C3, LSU variant (all 32 lanes of warp 3): 16-byte vector loads and
// stores (L2 evict-first), AG: one load, n-1 stores per vector; A2A: one
// load, one store. Keeps the SM's TMA queue for the GEMM's operand loads.
__device__ void fused_copy_loop_lsu(const Params& p, int lane) {
    const FusedComm& fc = p.fc;
    const uint64_t pol = policy_evict_first();
    const int64_t vecs = fc.chunk / 16;
    const int nv = fc.self_end - fc.self_begin;
    const int64_t rows = fc.kind == 0 ? 1 : fc.n;  // (dest) sub-slots per rank
    const int64_t per_v = rows * vecs;
    const int64_t total = per_v * nv;
    constexpr int U = 4;
    const int64_t step = static_cast<int64_t>(gridDim.x) * 32 * U;
    const uint64_t t0 = global_ns();
    double sent = 0.0;  // peer bytes stored by this warp (link emulation)
    const double per_vec = 16.0 * (fc.kind == 0 ? (fc.skip_self ? fc.n - 1 : fc.n) : 1);
    for (int64_t blk = static_cast<int64_t>(blockIdx.x) * 32 * U; blk < total; blk += step) {
        if (fc.link_cta_bpns > 0.f) {
            if (lane == 0) link_wait(t0, sent, fc.link_cta_bpns);
            __syncwarp();
            const int64_t left = total - blk;
            sent += per_vec * static_cast<double>(left < 32 * U ? left : 32 * U);
        }
        const int64_t base = blk + lane;
        uint4 v[U];
        int vv[U], qq[U];
        int64_t ii[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t w = base + u * 32;
            if (w >= total) continue;
            vv[u] = fc.self_begin + static_cast<int>(w / per_v);
            const int64_t r = w % per_v;
            qq[u] = static_cast<int>(r / vecs);
            ii[u] = r % vecs;
            const uint4* src = reinterpret_cast<const uint4*>(fc.src[vv[u]]) + (fc.kind == 0 ? 0 : qq[u] * vecs);
            v[u] = ld_stream_v4(src + ii[u], pol);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * 32 >= total) continue;
            const int64_t off = static_cast<int64_t>(vv[u]) * vecs + ii[u];
            if (fc.kind == 0) {
                for (int t = 1; t <= fc.n; ++t) {
                    const int d = (vv[u] + t) % fc.n;
                    if (d == vv[u] && fc.skip_self) continue;
                    st_stream_v4(reinterpret_cast<uint4*>(fc.dst[d]) + off, v[u], pol);
                }
            } else {
                st_stream_v4(reinterpret_cast<uint4*>(fc.dst[qq[u]]) + off, v[u], pol);
            }
        }
    }
    __threadfence_system();
    if (fc.link_cta_bpns > 0.f && lane == 0) link_wait(t0, sent, fc.link_cta_bpns);
}

// <= 152 registers per thread: 256 x 152 = 38K of the SM's 64K leaves room
// for a collective CTA beside the GEMM's (all-gather / all-to-all: 512 x 50;
// reduce-scatter: 256 x 96), the B200 co-resident C3 mode.
// (setmaxnreg would not help: ptxas sizes every path for the launch count.)
#ifndef C3_PAIR_MAXNREG
#define C3_PAIR_MAXNREG 152
#endif
template <bool FUSED, int BN_>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(C3_PAIR_MAXNREG)
gemm_bf16_tn_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                         const __grid_constant__ CUtensorMap map_b,
                         const __grid_constant__ CUtensorMap map_c, const Params p) {
    using Cfg = PairCfg<BN_, FUSED>;
    constexpr int BN = Cfg::BN, STAGES = Cfg::STAGES, ACC_BUFS = Cfg::ACC_BUFS;
    constexpr uint32_t B_STAGE = Cfg::B_STAGE, STAGE = Cfg::STAGE;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + STAGES * A_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* acc_full = bars + 2 * STAGES;
    uint64_t* acc_empty = acc_full + ACC_BUFS;  // [2]: per accumulator (BN 256) / per 256-column half (BN 512)
    uint64_t* acc_h0 = acc_empty + 2;           // BN 512: half 0 of the tile final
    uint64_t* tile_full = acc_h0 + 1;
    uint64_t* tile_empty = tile_full + RING;
    int* tile_ring = reinterpret_cast<int*>(tile_empty + RING);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + RING);
    // fused C3 state (FUSED only): copy buffers after the ring, 1 KiB aligned
    uint64_t* lbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // [kFusedSlots] copy loads
    uint32_t* progress = reinterpret_cast<uint32_t*>(lbar + kFusedSlots);  // producer k-blocks issued
    uint32_t* producer_done = progress + 1;
    uint8_t* epi_stage = smem + STAGES * STAGE + 1024;
#ifndef C3_EPI_BUFS
#define C3_EPI_BUFS 2
#endif
    constexpr int EPI_BUFS = FUSED ? 1 : C3_EPI_BUFS;
    uint8_t* copy_buf = epi_stage + EPI_BUFS * Cfg::EPI_SMEM;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
        tma_prefetch_desc(&map_c);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < ACC_BUFS; ++b) {
            mbar_init(&acc_full[b], 1);
        }
        for (int b = 0; b < 2; ++b) mbar_init(&acc_empty[b], 2 * Cfg::EPI_WARPS);
        mbar_init(acc_h0, 1);
        for (int r = 0; r < RING; ++r) {
            mbar_init(&tile_full[r], 1);
            mbar_init(&tile_empty[r], 2 + 2 * Cfg::EPI_WARPS);
        }
        if (FUSED) {
            for (int b = 0; b < kFusedSlots; ++b) mbar_init(&lbar[b], 1);
            *progress = 0;
            *producer_done = 0;
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();  // barrier inits and TMEM allocation visible across the pair
    __syncthreads();  // CTA-scope order for the TMEM address slot (explicit for racecheck)
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ------------- tile claims (leader) + TMA producer (both CTAs) -------------
        const uint64_t pol_a = policy_by_kind(p.pol_a);
        const uint64_t pol_b = policy_by_kind(p.pol_b);
        int stage = 0;
        uint32_t phase = 0;
        int band_ready = -1;  // A row bands known resident (they land in order)
        // the pair's first unit is its own (blockIdx.x / 2), later ones are
        // claimed one ahead: claimed first units let the pairs that start first
        // take two each before the last ones started (gemm_tcgen05.cu)
        const int pairs = static_cast<int>(gridDim.x / 2);
        int tile = leader ? static_cast<int>(blockIdx.x / 2) : 0;
        for (int i = 0;; ++i) {
            const int r = i % RING;
            const uint32_t par = (i / RING) & 1;
            if (leader) {
                if (tile >= p.num_units) tile = -1;
                mbar_wait(&tile_empty[r], par ^ 1);
                tile_ring[r] = tile;
                st_cluster_u32(mapa(smem_u32(&tile_ring[r]), 1), static_cast<uint32_t>(tile));
                mbar_arrive(&tile_full[r]);
                mbar_arrive_cluster(mapa(smem_u32(&tile_full[r]), 1));
            } else {
                mbar_wait_cluster(&tile_full[r], par);
                tile = tile_ring[r];
                mbar_arrive_cluster(mapa(smem_u32(&tile_empty[r]), 0));
            }
            if (tile < 0) break;
            const int next = leader ? pairs + atomicAdd(p.tile_counter, 1) : 0;
            int tm, tn, t_idx, half;
            unit_tile(p, tile, t_idx, half);
            tile_coords(p, t_idx, tm, tn);
            if (p.dev & 1) tm = tn = 0;
            const int a_row = tm * BM + static_cast<int>(rank) * 128;
            if (p.gate.flags != nullptr) {
                const int band = a_row / p.gate.rows_per_flag;
                if (band > band_ready) {
                    wait_row_band(p.gate, band);
                    band_ready = band;
                }
            }
            // + 256 per half; a half tile loads only its own 256 B rows, into slot 0
            const int b_row = tn * BN + (half > 0 ? 256 : 0) + static_cast<int>(rank) * 128;
            const int halves = half < 0 ? Cfg::HALVES : 1;
            const uint32_t stage_tx = 2 * (A_STAGE + halves * B_HALF);
            for (int kb = 0; kb < p.k_blocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (leader) mbar_arrive_expect_tx(&full[stage], stage_tx);
                tma_load_2d_pair(smem_a + stage * A_STAGE, &map_a, &full[stage], kb * BK, a_row, pol_a);
                for (int h = 0; h < halves; ++h)
                    tma_load_2d_pair(smem_b + stage * B_STAGE + h * B_HALF, &map_b, &full[stage], kb * BK,
                                     b_row + h * 256, pol_b);
                if (FUSED) st_volatile_shared(progress, ld_volatile_shared(progress) + 1);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            tile = next;
        }
        if (FUSED) st_volatile_shared(producer_done, 1);
    } else if (FUSED && warp == 3) {
        if (p.fc.enabled) {
            // across processes: no copy warp stores into a peer's receive buffer
            // before that peer reached this step (its previous result is free)
            const Signals& sig = p.fc.sig;
            if (sig.enabled && lane == 0) {
                if (blockIdx.x == 0) {
                    fence_sys();
                    for (int q = 0; q < p.fc.n; ++q)
                        if (q != p.fc.self_begin)
                            st_release_sys(sig.peers[q] + kSigFusedEntry + p.fc.self_begin, sig.entry_epoch);
                }
                wait_words_bounded(sig.mine, kSigFusedEntry, p.fc.self_begin, p.fc.n, sig.entry_epoch, sig.timeout_ns,
                                   sig.err, kWaitFusedEntry);
            }
            __syncwarp();
            if (p.fc.mode == 1)
                fused_copy_loop_lsu(p, lane);
            else if (lane == 0)
                fused_copy_loop(p, copy_buf, Cfg::COPY_BYTES, lbar, progress, producer_done);
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // ------------- MMA issuer (leader only) -------------
        constexpr uint32_t idesc = idesc_bf16_f32(BM, 256);
        const uint32_t a0 = smem_u32(smem_a), b0 = smem_u32(smem_b);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int r = i % RING;
            mbar_wait(&tile_full[r], (i / RING) & 1);
            const int tile = tile_ring[r];
            mbar_arrive(&tile_empty[r]);
            if (tile < 0) break;
            int t_idx, half;
            unit_tile(p, tile, t_idx, half);
            const int halves = half < 0 ? Cfg::HALVES : 1;  // a half tile: one N=256 MMA per k-step
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
            int kb0 = 0;
            if (Cfg::HALVES == 2 && half >= 0) {
                mbar_wait(&acc_empty[0], acc_phase ^ 1);
                mbar_wait(&acc_empty[1], acc_phase ^ 1);
                tc_fence_after();
            } else if constexpr (Cfg::HALVES == 2) {
                // One 512-column accumulator, released by the epilogue in
                // 256-column halves: the first PRE k-blocks of the new tile
                // accumulate into half 0 while half 1 is still being drained.
                // at most the ring's stages: the half-1 MMAs of these k-blocks
                // release their stages, so more would wait on itself
                const int pre_cap = p.pre_half < STAGES ? p.pre_half : STAGES;
                const int pre = p.k_blocks < pre_cap ? p.k_blocks : pre_cap;
                mbar_wait(&acc_empty[0], acc_phase ^ 1);
                tc_fence_after();
                int st = stage;
                uint32_t ph = phase;
                for (int kb = 0; kb < pre; ++kb) {
                    mbar_wait(&full[st], ph);
                    tc_fence_after();
                    const uint32_t a_addr = a0 + st * A_STAGE, b_addr = b0 + st * B_STAGE;
#pragma unroll
                    for (int k = 0; k < BK / UK; ++k)
                        umma_bf16_pair(d_tmem, smem_desc_k_sw128(a_addr + k * UK * 2),
                                       smem_desc_k_sw128(b_addr + k * UK * 2), idesc, (kb | k) != 0);
                    if (++st == STAGES) {
                        st = 0;
                        ph ^= 1;
                    }
                }
                mbar_wait(&acc_empty[1], acc_phase ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < pre; ++kb) {  // the same stages, half 1, then release them
                    const uint32_t a_addr = a0 + stage * A_STAGE, b_addr = b0 + stage * B_STAGE;
#pragma unroll
                    for (int k = 0; k < BK / UK; ++k)
                        umma_bf16_pair(d_tmem + 256, smem_desc_k_sw128(a_addr + k * UK * 2),
                                       smem_desc_k_sw128(b_addr + B_HALF + k * UK * 2), idesc, (kb | k) != 0);
                    umma_commit_pair(&empty[stage], 0x3);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                kb0 = pre;
            } else {
                mbar_wait(&acc_empty[acc], acc_phase ^ 1);
                tc_fence_after();
            }
            // BN 512 whole tiles: the last `lag` k-blocks run half 0, then half 1
            int lag = 0;
            if constexpr (Cfg::HALVES == 2) {
                if (half < 0) lag = min(min(p.tail_lag, p.k_blocks - kb0), STAGES);
            }
            for (int kb = kb0; kb < p.k_blocks - lag; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t a_addr = a0 + stage * A_STAGE;
                const uint32_t b_addr = b0 + stage * B_STAGE;
#pragma unroll
                for (int k = 0; k < BK / UK; ++k)
                    for (int h = 0; h < halves; ++h)
                        umma_bf16_pair(d_tmem + h * 256, smem_desc_k_sw128(a_addr + k * UK * 2),
                                       smem_desc_k_sw128(b_addr + h * B_HALF + k * UK * 2), idesc,
                                       (kb | k) != 0);
                umma_commit_pair(&empty[stage], 0x3);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if constexpr (Cfg::HALVES == 2) {
                if (lag > 0) {
                    // half 0 of the last `lag` k-blocks (their stages stay held) ...
                    int st = stage;
                    uint32_t ph = phase;
                    for (int j = 0; j < lag; ++j) {
                        const int kb = p.k_blocks - lag + j;
                        mbar_wait(&full[st], ph);
                        tc_fence_after();
                        const uint32_t a_addr = a0 + st * A_STAGE, b_addr = b0 + st * B_STAGE;
#pragma unroll
                        for (int k = 0; k < BK / UK; ++k)
                            umma_bf16_pair(d_tmem, smem_desc_k_sw128(a_addr + k * UK * 2),
                                           smem_desc_k_sw128(b_addr + k * UK * 2), idesc, (kb | k) != 0);
                        if (++st == STAGES) {
                            st = 0;
                            ph ^= 1;
                        }
                    }
                    umma_commit_pair(acc_h0, 0x3);  // half 0 final: its drain overlaps what follows
                    // ... then half 1 of the same k-blocks, releasing the stages
                    for (int j = 0; j < lag; ++j) {
                        const int kb = p.k_blocks - lag + j;
                        const uint32_t a_addr = a0 + stage * A_STAGE, b_addr = b0 + stage * B_STAGE;
#pragma unroll
                        for (int k = 0; k < BK / UK; ++k)
                            umma_bf16_pair(d_tmem + 256, smem_desc_k_sw128(a_addr + k * UK * 2),
                                           smem_desc_k_sw128(b_addr + B_HALF + k * UK * 2), idesc,
                                           (kb | k) != 0);
                        umma_commit_pair(&empty[stage], 0x3);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                } else {
                    umma_commit_pair(acc_h0, 0x3);  // half 0 final with the whole tile
                }
            }
            umma_commit_pair(&acc_full[acc], 0x3);
            if (++acc == ACC_BUFS) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ------------- epilogue (both CTAs): own 128 rows x BN columns -------------
        const int q = warp % 4;  // TMEM lane quadrant this warp may access
        constexpr int COLS = BN / (Cfg::EPI_WARPS / 4);
        const int c_begin = (warp - 4) / 4 * COLS;
        uint8_t* stg_base = epi_stage + (warp - 4) * EPI_BUFS * kEpiWarpStage;
        int stg_i = 0;  // staging tile in use (ring of EPI_BUFS)
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            const int r = i % RING;
            if (leader)
                mbar_wait(&tile_full[r], (i / RING) & 1);
            else
                mbar_wait_cluster(&tile_full[r], (i / RING) & 1);
            const int tile = tile_ring[r];
            __syncwarp();
            if (lane == 0) {
                if (leader)
                    mbar_arrive(&tile_empty[r]);
                else
                    mbar_arrive_cluster(mapa(smem_u32(&tile_empty[r]), 0));
            }
            if (tile < 0) {
                if (lane == 0) bulk_wait_all();  // this warp's C stores complete
                break;
            }
            int tm, tn, t_idx, half;
            unit_tile(p, tile, t_idx, half);
            tile_coords(p, t_idx, tm, tn);
            const int cols = half < 0 ? COLS : 256;  // a half tile fills accumulator columns 0-255
            const int col_base = tn * BN + (half > 0 ? 256 : 0);
            // BN 512: half 0 may be final before half 1 (tail lag); the wait
            // for half 1 comes before its first TMEM load
            bool h1_ready = Cfg::HALVES != 2;
            if constexpr (Cfg::HALVES == 2)
                mbar_wait(acc_h0, acc_phase);
            else
                mbar_wait(&acc_full[acc], acc_phase);
            tc_fence_after();
            if (!h1_ready && (p.dev & 14)) {  // dev modes: the whole tile first
                mbar_wait(&acc_full[acc], acc_phase);
                tc_fence_after();
                h1_ready = true;
            }
            // dev bits 2 / 3 (BN 512): release half 0 / both halves before the
            // drain (the drain still runs): the time a hidden drain would save
            int early = 0;
            if constexpr (Cfg::HALVES == 2) {
                if (half < 0 && (p.dev & 12)) {
                    early = (p.dev & 8) ? 3 : 1;
                    __syncwarp();
                    if (lane == 0)
                        for (int h = 0; h < 2; ++h)
                            if (early >> h & 1) {
                                if (leader)
                                    mbar_arrive(&acc_empty[h]);
                                else
                                    mbar_arrive_cluster(mapa(smem_u32(&acc_empty[h]), 0));
                            }
                }
            }
            if (p.dev & 2) {  // dev: release without draining
                __syncwarp();
                if (lane == 0)
                    for (int h = 0; h < (Cfg::HALVES == 2 ? 2 : 1); ++h) {
                        const int rel = Cfg::HALVES == 2 ? h : acc;
                        if (leader)
                            mbar_arrive(&acc_empty[rel]);
                        else
                            mbar_arrive_cluster(mapa(smem_u32(&acc_empty[rel]), 0));
                    }
                if (++acc == ACC_BUFS) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                continue;
            }
            // TMEM row `lane` of this warp's quadrant -> packed bf16 -> the
            // warp's 32 x 64 staging tile in shared memory (16-byte chunks
            // XOR-swizzled by row: the TMA 128B swizzle) -> one TMA tensor
            // store per 64 columns (OOB rows/columns clipped by the map). The
            // TMEM loads of chunk c+64 are issued before chunk c's store, and
            // the accumulator is released right after the last TMEM load: with
            // one 512-column accumulator the next tile's MMAs wait for this.
            const int row0 = tm * BM + static_cast<int>(rank) * 128 + q * 32;  // warp's first row
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
            // chunk c in registers -> staging tile -> TMA store (lane 0)
            auto stage_store = [&](const uint32_t (&a)[32], const uint32_t (&b)[32], int c) {
                uint8_t* stg = stg_base + stg_i * kEpiWarpStage;
                if (lane == 0) bulk_wait_read<EPI_BUFS - 1>();  // this tile's previous store has read it
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t* v = j < 4 ? a + 8 * j : b + 8 * (j - 4);
                    uint4 o;
                    o.x = pack_bf16x2(v[0], v[1]);
                    o.y = pack_bf16x2(v[2], v[3]);
                    o.z = pack_bf16x2(v[4], v[5]);
                    o.w = pack_bf16x2(v[6], v[7]);
                    st_shared_v4(stg + lane * 128 + ((j ^ (lane & 7)) << 4), o);
                }
                fence_proxy_async_shared();
                __syncwarp();
                if (lane == 0) {
                    if (p.pol_c)
                        tma_store_2d_hint(&map_c, stg, col_base + c, row0, policy_by_kind(p.pol_c));
                    else
                        tma_store_2d(&map_c, stg, col_base + c, row0);
                    bulk_commit();
                }
                if (++stg_i == EPI_BUFS) stg_i = 0;
            };
            // two register sets: the TMEM loads of chunk c+64 are in flight
            // while chunk c is packed and stored; the accumulator is released
            // right after the last TMEM load completes
            uint32_t va0[32], va1[32], vb0[32], vb1[32];
            tmem_ld_32x32b_x32(t_row + c_begin, va0);
            tmem_ld_32x32b_x32(t_row + c_begin + 32, va1);
#pragma unroll 1
            for (int c = c_begin;; c += 128) {
                tmem_ld_wait();  // chunk c
                tmem_ld_32x32b_x32(t_row + c + 64, vb0);
                tmem_ld_32x32b_x32(t_row + c + 96, vb1);
                stage_store(va0, va1, c);
                tmem_ld_wait();  // chunk c + 64
                if constexpr (Cfg::HALVES == 2) {
                    if (c + 64 == 192 && !(early & 1)) {  // columns 0-255 read: release half 0
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (leader)
                                mbar_arrive(&acc_empty[0]);
                            else
                                mbar_arrive_cluster(mapa(smem_u32(&acc_empty[0]), 0));
                        }
                    }
                }
                const bool last = c + 128 >= c_begin + cols;
                if (!last) {
                    if (!h1_ready && c + 128 == 256) {  // half 1's first columns next
                        mbar_wait(&acc_full[acc], acc_phase);
                        tc_fence_after();
                        h1_ready = true;
                    }
                    tmem_ld_32x32b_x32(t_row + c + 128, va0);
                    tmem_ld_32x32b_x32(t_row + c + 160, va1);
                } else {
                    tc_fence_before();
                    __syncwarp();
                    const int rel = Cfg::HALVES == 2 ? 1 : acc;  // the last half / this accumulator
                    if (lane == 0 && !(early & 2)) {
                        if (leader)
                            mbar_arrive(&acc_empty[rel]);
                        else
                            mbar_arrive_cluster(mapa(smem_u32(&acc_empty[rel]), 0));
                    }
                }
                stage_store(vb0, vb1, c + 64);
                if (last) break;
            }
            if (++acc == ACC_BUFS) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    tc_fence_before();
    cluster_sync();  // no CTA leaves while its peer may still signal into it
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    }
    // fused C3 across processes: once every CTA's copies are complete, the
    // last CTA tells every peer and waits for all of them (peer flag words)
    if (FUSED && p.fc.enabled && p.fc.sig.enabled && threadIdx.x == 0) {
        const Signals& sig = p.fc.sig;
        fence_sys();
        if (atomicAdd(sig.done, 1u) == gridDim.x - 1) {
            fence_sys();
            for (int q = 0; q < p.fc.n; ++q)
                if (q != p.fc.self_begin) st_release_sys(sig.peers[q] + kFusedExitSlot + p.fc.self_begin, sig.epoch);
            wait_words_bounded(sig.mine, kFusedExitSlot, p.fc.self_begin, p.fc.n, sig.epoch, sig.timeout_ns,
                               sig.err, kWaitFusedExit);
            *sig.done = 0;
        }
    }
    if (threadIdx.x == 0 && leader) {
        __threadfence();
        if (atomicAdd(p.exit_counter, 1) == static_cast<int>(gridDim.x / 2) - 1) {
            *p.tile_counter = 0;
            *p.exit_counter = 0;
            __threadfence();
        }
    }
}

}  // namespace gemm2

namespace {

template <bool FUSED, int BN>
int launch_pair(const GemmPlan* plan, gemm2::Params p, int grid, cudaStream_t stream) {
    using Cfg = gemm2::PairCfg<BN, FUSED>;
    // fused: bytes per bulk copy, at most half the copy ring (>= 2 slots)
    if (FUSED) p.fc.piece = std::max<int64_t>(16, std::min<int64_t>(p.fc.piece, Cfg::COPY_BYTES / 2)) / 16 * 16;
    constexpr uint32_t smem = FUSED ? Cfg::SMEM_FUSED : Cfg::SMEM;
    static bool attr_done = false;
    if (!attr_done) {
        const cudaError_t e = cudaFuncSetAttribute(gemm2::gemm_bf16_tn_pair_kernel<FUSED, BN>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm pair)");
        attr_done = true;
    }
    gemm2::gemm_bf16_tn_pair_kernel<FUSED, BN><<<grid, Cfg::THREADS, smem, stream>>>(
        plan->map_a, plan->map_b128, plan->map_c, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "gemm pair launch");
    return C3_OK;
}

}  // namespace

int gemm_pair_launch(const GemmPlan* plan, int grid, cudaStream_t stream, const FusedComm* fc,
                     const RowGate* gate) {
    gemm2::Params p;
    p.gate = gate ? *gate : RowGate{};
    if (p.gate.flags && p.gate.rows_per_flag < 128)
        return set_error(C3_ERR_VALIDATION, "row gate: rows_per_flag must be >= 128");
    p.m = static_cast<int>(plan->m);
    p.n = static_cast<int>(plan->n);
    p.k = static_cast<int>(plan->k);
    p.tiles_m = plan->tiles_m;
    p.tiles_n = plan->tiles_n;
    p.num_tiles = plan->num_tiles;
    p.k_blocks = plan->k_blocks;
    p.c = static_cast<__nv_bfloat16*>(plan->c);
    p.ldc = static_cast<int>(plan->n);
    p.tile_counter = plan->counters;
    p.exit_counter = plan->counters + 1;
    static const int band = [] {
        const char* e = std::getenv("C3_GEMM_BAND");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? v : gemm2::GROUP_M_DEFAULT;
    }();
    p.group_m = band;
    // L2 policies of the operand loads, "<a><b>" digits (C3_GEMM_POL env, dev A/B;
    // profiles/r01_gemm_l2_policy_ab.txt)
    static const int pol = [] {
        const char* e = std::getenv("C3_GEMM_POL");
        if (!(e && e[0] && e[1])) return 110;
        return (e[0] - '0') * 100 + (e[1] - '0') * 10 + (e[2] ? e[2] - '0' : 0);
    }();
    p.pol_a = pol / 100;
    p.pol_b = pol / 10 % 10;
    p.pol_c = pol % 10;
    static const int pre_half = [] {
        const char* e = std::getenv("C3_GEMM_PREHALF");  // dev A/B
        const int v = e ? std::atoi(e) : gemm2::kPreHalf;
        return v < 1 ? 1 : v > gemm2::PairCfg<512>::STAGES ? gemm2::PairCfg<512>::STAGES : v;
    }();
    p.pre_half = pre_half;
    static const int tail_lag = [] {
        const char* e = std::getenv("C3_GEMM_TAILLAG");  // dev A/B: 0 = half 1 alongside half 0 to the end
        const int v = e ? std::atoi(e) : gemm2::kTailLag;
        return v < 0 ? 0 : v;
    }();
    p.tail_lag = tail_lag;
    static const int dev = [] {
        const char* e = std::getenv("C3_GEMM_DEV");  // dev A/B only: results invalid
        return e ? std::atoi(e) : 0;
    }();
    p.dev = dev;

    const bool wide = plan->kind == GemmPlan::kPair512;
    // tail split (512-wide): if the last wave is at most half full, its tiles
    // are claimed as 256-column halves (C3_GEMM_TAILSPLIT=0 turns it off, dev A/B)
    p.full_tiles = p.num_units = p.num_tiles;
    static const bool tail_split = [] {
        const char* e = std::getenv("C3_GEMM_TAILSPLIT");
        return !(e != nullptr && std::string(e) == "0");
    }();
    if (wide && tail_split) {
        const int pairs = grid / 2;
        const int rem = pairs > 0 ? p.num_tiles % pairs : 0;
        if (rem > 0 && 2 * rem <= pairs) {
            p.full_tiles = p.num_tiles - rem;
            p.num_units = p.num_tiles + rem;
        }
    }
    if (fc) {
        if (fc->chunk % 16 != 0) return set_error(C3_ERR_VALIDATION, "fused C3: slot bytes must be 16-byte multiples");
        p.fc = *fc;
        p.fc.link_cta_bpns = static_cast<float>(fc->link_bpns / grid);
        p.fc.piece = fc->piece;  // clamped to the variant's copy ring in launch_pair
        return wide ? launch_pair<true, 512>(plan, p, grid, stream) : launch_pair<true, 256>(plan, p, grid, stream);
    }
    p.fc = FusedComm{};
    return wide ? launch_pair<false, 512>(plan, p, grid, stream) : launch_pair<false, 256>(plan, p, grid, stream);
}

}  // namespace c3k
