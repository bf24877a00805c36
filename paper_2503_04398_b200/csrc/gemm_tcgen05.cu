// gemm_tcgen05.cu — K6: persistent, warp-specialised grouped GEMM for the
// expert FFN on sm_100a (TMA -> SMEM -> tcgen05.mma -> TMEM -> epilogue).
//
// The expert FFN is not in the reference; it is the
// one dense contraction of the layer.  One launch covers every (shard,
// expert) problem resident on this GPU: problem p multiplies rows
// [a_off_p, a_off_p + m_p) of the expert-input buffer by expert b_index_p's
// weight block.  Row counts live in device memory (written by the dispatch
// stage), so the launch needs no host synchronisation and is graph-capturable.
//
// CTA layout (256 threads, 1 CTA per SM, persistent over tiles):
//   warp 0 lane 0  TMA producer: A tile 128x64 + B tile 256x64 per k-block,
//                  4-stage mbarrier ring (full/empty)
//   warp 1 lane 0  MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//                  M=128 N=256 K=16, fp32 accumulator in TMEM; two
//                  accumulator buffers (2 x 256 columns) so the epilogue of
//                  tile t overlaps the MMAs of tile t+1
//   warp 2         TMEM allocator (512 columns)
//   warps 4..7     epilogue: tcgen05.ld 32x32b -> registers -> bf16 ->
//                  swizzled SMEM staging -> coalesced 16 B row stores
//                  (plain, SwiGLU-fused, or scattered to peer shards: the
//                  A2A combine is fused into the down-projection epilogue)
#include "common.cuh"
#include "gemm.h"
#include "tc_ptx.cuh"
#include <algorithm>
#include <cstdlib>

// Ring depth of the SM-pair variant (compile-time; profiles/r1_gemm_l2/
// cg2_ring_depth_scan.csv: 4 stages read ~algorithmic DRAM bytes at higher
// clocks but lower tensor-pipe occupancy, 6 the reverse; within +-2% in time).
#ifndef SMOE_CG2_STAGES
#define SMOE_CG2_STAGES 6
#endif
#ifndef SMOE_NARROW_STAGES
#define SMOE_NARROW_STAGES 5   // 6 measured slower (profiles/r1_narrow/narrow6_rejected_ab.jsonl)
#endif
namespace smoe {

constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kStagingBytes = 4 * 32 * 64;        // 4 epilogue warps x 32 rows x 64 B

// Problem table staged in shared memory (capacity CAP problems).
template <int CAP> struct SmemProblemsT {
  int64_t a_off[CAP];
  int64_t c_off[CAP];
  int32_t m[CAP];
  int32_t b_idx[CAP];
  int32_t tile_prefix[CAP + 1];
};

// Per cta_group: CG = 1 (one SM, tile 128 x 256) or CG = 2 (an SM pair, tile
// 256 x 256: each CTA stages 128 A rows and half of the 256 B rows, the
// leader issues tcgen05.mma.cta_group::2 over both CTAs' shared memory).
// NARROW (CG = 1 only, decode-sized batches): m-blocks of kGemmNarrowM rows.
// A stages shrink to 4 KiB, which buys a fifth stage — 160 instead of 128 KiB
// of weight tiles in flight per SM, the lever when the GEMM streams weights.
// The MMA stays M = 128: its A operand reads 16 KiB from the stage's address,
// i.e. the next stages' A rows (or the first B stage) as rows 32..127 — in
// bounds, and those accumulator rows are never stored (an MMA row of D only
// depends on the same row of A).
template <int CG, int NARROW = 0> struct GemmShape {
  static constexpr uint32_t kABytes = (NARROW ? kGemmNarrowM : kGemmBM) * kGemmBK * 2;
  static constexpr uint32_t kBBytes = (kGemmBN / CG) * kGemmBK * 2;   // B rows staged per CTA
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = NARROW ? SMOE_NARROW_STAGES : (CG == 1 ? 4 : SMOE_CG2_STAGES);
  static constexpr int kTileM = NARROW ? kGemmNarrowM : kGemmBM * CG;
  // narrow: only the first epilogue warp stores rows, and the problem table
  // holds kGemmNarrowMaxProblems entries — the room pays for the extra stage
  static constexpr uint32_t kStaging = NARROW ? 32 * 64 : kStagingBytes;
  static constexpr int kMaxProblems = NARROW ? kGemmNarrowMaxProblems : kGemmMaxProblems;
  using Problems = SmemProblemsT<kMaxProblems>;
  static constexpr size_t kSmem =
      1024 + kStages * kStageBytes + kStaging + 1024 + sizeof(Problems);
  // instruction descriptor: D f32, A/B bf16, K-major both, N = 256, M = 128 * CG
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                     (uint32_t(kGemmBN >> 3) << 17) |
                                     (uint32_t((kGemmBM * CG) >> 4) << 24);
};

// ---------------------------------------------------------------- tiles

struct TileCoord {
  int32_t p, m_blk, n_blk;
};

// Tiles are enumerated problem-major.  Inside a problem, m-blocks are taken
// in groups of `group_m` (sized on the host so a group's A rows stay in L2)
// and m varies fastest inside a group: the CTAs of one wave share a few weight
// tiles (n-blocks) and sweep the group's A rows, so A is read from DRAM once
// and B once per group.
template <int TILE_M, typename SmemProblems>
__device__ __forceinline__ TileCoord decode_tile(const SmemProblems& sp, int32_t np,
                                                 int32_t n_tiles_n, int32_t group_m, int32_t t,
                                                 int32_t& cursor) {
  while (cursor + 1 < np && sp.tile_prefix[cursor + 1] <= t) ++cursor;
  const int32_t local = t - sp.tile_prefix[cursor];
  const int32_t mt = (sp.m[cursor] + TILE_M - 1) / TILE_M;
  TileCoord c;
  c.p = cursor;
  if (group_m < 0) {
    // n-grouped order (group_m = -group_n): a group of n-blocks (a slice of the
    // weights that stays L2-resident) is swept for every m-block, n fastest
    const int32_t group_n = -group_m;
    const int32_t per_group = group_n * mt;
    const int32_t g = local / per_group;
    const int32_t first_n = g * group_n;
    const int32_t gn = min(group_n, n_tiles_n - first_n);
    const int32_t r = local - g * per_group;
    c.n_blk = first_n + r % gn;
    c.m_blk = r / gn;
    return c;
  }
  const int32_t per_group = group_m * n_tiles_n;
  const int32_t g = local / per_group;
  const int32_t first_m = g * group_m;
  const int32_t gm = min(group_m, mt - first_m);
  const int32_t r = local - g * per_group;
  c.m_blk = first_m + r % gm;
  c.n_blk = r / gm;
  return c;
}

template <int EPI, int CG, int NARROW>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                    const __grid_constant__ CUtensorMap tmap_b, const GemmArgs args) {
  static_assert(!NARROW || CG == 1, "narrow m-blocks are a one-SM variant");
  using S = GemmShape<CG, NARROW>;
  constexpr int kStages = S::kStages;
  constexpr uint32_t kABytes = S::kABytes;
  constexpr uint32_t kBBytes = S::kBBytes;
  constexpr int kTileM = S::kTileM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * kABytes;
  uint8_t* staging = smem + kStages * S::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + S::kStaging);
  // bars: full[kStages], empty[kStages], tfull[2], tempty[2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  // dynamic tiles: tile-index ring of 4 (full / empty mbarriers + the index)
  const uint32_t tile_full0 = smem_addr(bars + 2 * kStages + 8);
  const uint32_t tile_empty0 = smem_addr(bars + 2 * kStages + 12);
  volatile int32_t* s_tile = reinterpret_cast<volatile int32_t*>(bars + 2 * kStages + 16);
  typename S::Problems& sp = *reinterpret_cast<typename S::Problems*>(bars + 2 * kStages + 20);
  const bool dyn = CG == 1 && args.tile_counter != nullptr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t np = args.num_problems;
  constexpr int kTl = EPI == kEpiSwiGLU ? 5 : 6;
  SMOE_TL_ENTER(kTl);
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;     // CTA rank inside the SM pair
  // CTA -> tile assignment follows blockIdx: the launch order places
  // consecutive CTAs on the two SMs of a TPC, then round-robin over GPCs, so
  // the CTAs sharing a weight tile are spread over the chip.  Mapping by
  // %smid instead (or launching this kernel early via PDL, which scrambles
  // the placement) costs 5-10% (profiles/r1_pdl/).
  const int32_t unit = blockIdx.x / CG, n_units = gridDim.x / CG;

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_addr(&bars[s]), 1);
      mbar_init(smem_addr(&bars[kStages + s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_addr(&bars[2 * kStages + a]), 1);
      mbar_init(smem_addr(&bars[2 * kStages + 2 + a]), 4 * CG);   // one arrival per epilogue warp
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(tile_full0 + 8 * s, 1);            // the producer publishes a tile index
      mbar_init(tile_empty0 + 8 * s, 1 + 4);       // the MMA issuer + the 4 epilogue warps read it
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tmap_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tmap_b) : "memory");
  }
  if (warp == 2) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   :: "r"(smem_addr(tmem_holder)), "r"(kTmemCols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   :: "r"(smem_addr(tmem_holder)), "r"(kTmemCols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  // everything above touches constant data only (weights, tensor maps, smem,
  // TMEM); the problem table is written by the dispatch stage
  pdl_trigger();
  // role 2 (the decode down GEMM): no grid-wide wait on the up GEMM -- its
  // inputs written before the up GEMM started (problem table, row metadata)
  // are visible once this grid runs, and the up GEMM's hidden rows are
  // awaited per problem by the producer below
  if (args.ready_role != 2) pdl_wait();
  SMOE_TL_WAITED(kTl);
  // ---- problem table -> shared, tile prefix
  for (int p = threadIdx.x; p < np; p += kThreads) {
    const int64_t* q = args.problems + 4 * p;
    sp.a_off[p] = q[0];
    sp.m[p] = (int32_t)q[1];
    sp.b_idx[p] = (int32_t)q[2];
    sp.c_off[p] = q[3];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int p = 0; p < np; ++p) {
      sp.tile_prefix[p] = acc;
      const int32_t m = sp.m[p] > 0 ? sp.m[p] : 0;
      acc += ((m + kTileM - 1) / kTileM) * args.n_tiles_n;
    }
    sp.tile_prefix[np] = acc;
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int32_t total_tiles = sp.tile_prefix[np];
  const uint32_t full0 = smem_addr(&bars[0]);
  const uint32_t empty0 = smem_addr(&bars[kStages]);
  const uint32_t tfull0 = smem_addr(&bars[2 * kStages]);
  const uint32_t tempty0 = smem_addr(&bars[2 * kStages + 2]);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs of a pair; bytes land on the leader's barrier) =====
      int32_t stage = 0;
      uint32_t phase = 0;
      int32_t cursor = 0;
      // dynamic tiles: the next index is fetched once this tile's loads are
      // all issued (the ring's depth hides the atomic's round trip, and a CTA
      // never holds more than the tile it is about to load)
      int32_t next_t = dyn ? atomicAdd(args.tile_counter, 1) : 0;
      for (int32_t it = 0;; ++it) {
        int32_t t = unit + it * n_units;
        if (dyn) {
          const int slot = it & 3;
          t = next_t;
          if (it >= 4) mbar_wait(tile_empty0 + 8 * slot, ((it >> 2) - 1) & 1);
          s_tile[slot] = t;
          mbar_arrive(tile_full0 + 8 * slot);
        }
        if (t >= total_tiles) break;
        const TileCoord tc = decode_tile<kTileM>(sp, np, args.n_tiles_n, args.group_m, t, cursor);
        const int32_t a_row =
            (int32_t)(sp.a_off[tc.p] + (int64_t)tc.m_blk * kTileM + rank * kGemmBM);
        const int32_t b_row =
            sp.b_idx[tc.p] * args.n_b + tc.n_blk * kGemmBN + rank * (kGemmBN / CG);
        // tiled B: box (b_index, n-block, k-block) starts at row
        // ((b_index * n_tiles_n + n_blk) * num_k_blocks + kb) * 256 of a [*, 64] tensor
        const int32_t b_box0 =
            ((sp.b_idx[tc.p] * args.n_tiles_n + tc.n_blk) * args.num_k_blocks) * kGemmBN +
            rank * (kGemmBN / CG);
        if (args.ready_role == 2) {
          // every up tile of this problem must have stored its hidden rows
          const int32_t mp = sp.m[tc.p] > 0 ? sp.m[tc.p] : 0;
          const int32_t need =
              ((mp + args.ready_up_tile_m - 1) / args.ready_up_tile_m) * args.ready_up_n_tiles;
          const long long t0 = clock64();
          int32_t v;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v)
                         : "l"(args.ready + tc.p) : "memory");
            if (v < need && clock64() - t0 > 20000000ll) {   // ~10 ms: never hang
              if (args.err) atomicOr(args.err, SMOE_ERRBIT_TIMEOUT);
              break;
            }
          } while (v < need);
          // the rows were written through the generic proxy; TMA reads them
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int32_t kb = 0; kb < args.num_k_blocks; ++kb) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t fb = full0 + 8 * stage;
          const uint32_t sa = smem_addr(smem_a + stage * kABytes);
          const uint32_t sb = smem_addr(smem_b + stage * kBBytes);
          const int32_t bc0 = args.b_tiled ? 0 : kb * kGemmBK;
          const int32_t bc1 = args.b_tiled ? b_box0 + kb * kGemmBN : b_row;
          if (CG == 1) {
            mbar_expect_tx(fb, S::kStageBytes);
            tma_load_2d(sa, &tmap_a, fb, kb * kGemmBK, a_row);
            tma_load_2d(sb, &tmap_b, fb, bc0, bc1);
          } else {
            if (rank == 0) mbar_expect_tx(fb, 2 * S::kStageBytes);
            const uint32_t fb0 = map_to_rank(fb, 0);
            tma_load_2d_cg2(sa, &tmap_a, fb0, kb * kGemmBK, a_row);
            tma_load_2d_cg2(sb, &tmap_b, fb0, bc0, bc1);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (dyn) next_t = atomicAdd(args.tile_counter, 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (leader CTA only) =====
      int32_t stage = 0;
      uint32_t phase = 0;
      uint32_t acc = 0, acc_phase = 0;
      for (int32_t it = 0;; ++it) {
        int32_t t = unit + it * n_units;
        if (dyn) {
          const int slot = it & 3;
          mbar_wait(tile_full0 + 8 * slot, (it >> 2) & 1);
          t = s_tile[slot];
          mbar_arrive(tile_empty0 + 8 * slot);
        }
        if (t >= total_tiles) break;
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kGemmBN;
        for (int32_t kb = 0; kb < args.num_k_blocks; ++kb) {
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = sdesc(smem_addr(smem_a + stage * kABytes));
          const uint64_t bd = sdesc(smem_addr(smem_b + stage * kBBytes));
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {  // +32 B per K=16 step inside the swizzle atom
            if (CG == 1) tc_mma(d_tmem, ad + 2 * k, bd + 2 * k, S::kIdesc, (kb | k) != 0);
            else tc_mma_cg2(d_tmem, ad + 2 * k, bd + 2 * k, S::kIdesc, (kb | k) != 0);
          }
          if (CG == 1) tc_commit(empty0 + 8 * stage);
          else tc_commit_cg2_mc(empty0 + 8 * stage, 0x3);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (CG == 1) tc_commit(tfull0 + 8 * acc);
        else tc_commit_cg2_mc(tfull0 + 8 * acc, 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (both CTAs: each owns 128 rows of the tile) =====
    const int ew = warp - 4;                          // TMEM lane quarter
    uint8_t* stg = staging + ew * (32 * 64);
    uint32_t acc = 0, acc_phase = 0;
    int32_t cursor = 0;
    for (int32_t it = 0;; ++it) {
      int32_t t = unit + it * n_units;
      if (dyn) {
        const int slot = it & 3;
        mbar_wait(tile_full0 + 8 * slot, (it >> 2) & 1);
        t = s_tile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(tile_empty0 + 8 * slot);
      }
      if (t >= total_tiles) break;
      const TileCoord tc = decode_tile<kTileM>(sp, np, args.n_tiles_n, args.group_m, t, cursor);
      const int32_t m = sp.m[tc.p];
      const int32_t row0 = tc.m_blk * kTileM + rank * kGemmBM + ew * 32;   // first row of warp
      // narrow tiles: only the first warp's TMEM lanes hold rows of this tile
      if (NARROW && ew * 32 >= kTileM) {
        mbar_wait(tfull0 + 8 * acc, acc_phase);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      // per-lane destination row pointer (lane l <-> row row0 + l)
      char* my_row = nullptr;
      {
        const int32_t r = row0 + lane;
        if (r < m) {
          if (EPI == kEpiScatter) {
            const int64_t meta = __ldg(args.meta + sp.a_off[tc.p] + r);
            const int32_t shard = (int32_t)(meta >> 40);
            my_row = args.dst_base[shard] + ((meta & kMetaSlotMask) * args.ldd +
                                              (int64_t)tc.n_blk * kGemmBN) * 2;
          } else {
            const int64_t ncols = (EPI == kEpiSwiGLU) ? kGemmBN / 2 : kGemmBN;
            my_row = args.c + ((sp.c_off[tc.p] + r) * args.ldc + (int64_t)tc.n_blk * ncols) * 2;
          }
        }
      }
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * kGemmBN + ((uint32_t)(ew * 32) << 16);
      constexpr int kChunks = (EPI == kEpiSwiGLU) ? 4 : 8;   // 32 output columns per chunk
#pragma unroll 1
      for (int ch = 0; ch < kChunks; ++ch) {
        uint32_t packed[16];
        if (EPI == kEpiSwiGLU) {
          uint32_t g[32], u[32];
          SMOE_TMEM_LD32(tbase + ch * 32, g);
          SMOE_TMEM_LD32(tbase + 128 + ch * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float g0 = __uint_as_float(g[2 * j]), g1 = __uint_as_float(g[2 * j + 1]);
            const float u0 = __uint_as_float(u[2 * j]), u1 = __uint_as_float(u[2 * j + 1]);
            const float h0 = g0 / (1.0f + __expf(-g0)) * u0;
            const float h1 = g1 / (1.0f + __expf(-g1)) * u1;
            packed[j] = pack_bf16x2(h0, h1);
          }
        } else {
          uint32_t v[32];
          SMOE_TMEM_LD32(tbase + ch * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            packed[j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        }
        if (ch == kChunks - 1) {
          // this warp has read its accumulator lanes: release them to the MMA issuer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 1) mbar_arrive(tempty0 + 8 * acc);
            else mbar_arrive_cluster(map_to_rank(tempty0 + 8 * acc, 0));
          }
        }
        // stage row `lane` (64 B = 4 x 16 B chunks, XOR-swizzled against bank conflicts)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int pq = q ^ ((lane >> 1) & 3);
          *reinterpret_cast<uint4*>(stg + lane * 64 + pq * 16) =
              make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
        __syncwarp();
        // coalesced stores: 8 rows x 64 B per instruction
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int r = it * 8 + (lane >> 2);
          const int q = lane & 3;
          const unsigned long long rp =
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), r);
          if (rp) {
            const uint4 val =
                *reinterpret_cast<const uint4*>(stg + r * 64 + ((q ^ ((r >> 1) & 3)) * 16));
            st_v4(reinterpret_cast<char*>(rp) + ch * 64 + q * 16, val);
          }
        }
        __syncwarp();
      }
      if (args.ready_role == 1) {
        // publish this tile's hidden rows to the early-started down GEMM:
        // every epilogue thread fences its stores into the async proxy, the
        // four epilogue warps meet, one thread releases the count
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (ew == 0 && lane == 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" :: "l"(args.ready + tc.p)
                       : "memory");
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                   :: "r"(tmem_base), "r"(kTmemCols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;"
                   :: "r"(tmem_base), "r"(kTmemCols) : "memory");
  }
  SMOE_TL_EXIT(kTl);
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols,
                   int32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return SMOE_ERR_CUDA;
  if (rows <= 0 || cols <= 0 || (cols * 2) % 16 != 0 || ((uintptr_t)base % 16) != 0)
    return SMOE_ERR_INVALID_ARG;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)kGemmBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SMOE_OK : SMOE_ERR_CUDA;
}

template <int EPI, int CG, int NARROW = 0>
static int launch_impl(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args,
                       cudaStream_t st) {
  using S = GemmShape<CG, NARROW>;
  static_assert(S::kSmem <= 227 * 1024, "shared memory budget of one CTA per SM");
  static bool attr_set = false;
  if (!attr_set) {
    SMOE_CUDA_TRY(cudaFuncSetAttribute(grouped_gemm_kernel<EPI, CG, NARROW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)S::kSmem));
    attr_set = true;
  }
  GemmArgs g = args;
  if (g.group_m == 0) {
    // A-resident order: a group of m-blocks whose A rows fit ~40 MB of L2 is
    // swept for every n-block (B streams once per group).  When A tiles are
    // so large that fewer than 8 fit (the down projection, K = f), use the
    // B-resident order instead: all n-blocks of one m-block, then the next
    // (measured with tools/group_m_scan.sh: 9.8 GB vs 13.3 GB DRAM reads and
    // higher clocks under the power cap for Mixtral's down GEMM).
    const int64_t a_blk = (int64_t)S::kTileM * g.num_k_blocks * kGemmBK * 2;
    const int64_t fit = (40ll << 20) / a_blk;
    g.group_m = fit >= 8 ? (int32_t)fit : 1;
    const char* e = getenv(EPI == kEpiSwiGLU ? "SMOE_GROUP_M_UP" : "SMOE_GROUP_M_DOWN");
    if (e && atoi(e) != 0) g.group_m = atoi(e);     // tuning experiments (< 0: n-groups)
    const int opt = gemm_group_m(EPI == kEpiSwiGLU ? 0 : 1);   // SMOE_OPT_GEMM_GROUP_M_*
    if (opt != 0) g.group_m = opt;
  }
  const int grid = (num_sms() / CG) * CG;
  if (CG == 1) {
    SMOE_CUDA_TRY(
        launch_pdl(grouped_gemm_kernel<EPI, 1, NARROW>, grid, kThreads, S::kSmem, st, a, b, g));
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = S::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    SMOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<EPI, 2, 0>, a, b, g));
  }
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// cta_group per GEMM kind (SMOE_OPT_GEMM_CTA_GROUP_UP / _DOWN).  Measured on
// B200 (tools/gemm_ab.py, interleaved): the SM pair is ~10% faster for the
// down projection (K = f, scatter epilogue) and neutral for the SwiGLU up
// projection, so the defaults are up = 1, down = 2.
static int g_cta_group[2] = {1, 2};

int gemm_cta_group(int which) { return g_cta_group[which ? 1 : 0]; }
// -1: env SMOE_GEMM_PAIR_MIN_ROWS, else 1024.  The SM pair's 256-row tiles
// pad half a tile per expert on average (one SM: half of 128 rows); below
// ~1k routed rows per expert that padding outweighs the pair's ~10% MMA
// advantage (DeepSeek-V2 16K, 614 rows: down GEMM 1.48 -> 1.34 ms on one SM,
// profiles/r2/down_gemm/pair_min_rows_ab.jsonl; decode sizes: 5-16%)
static int g_pair_min_rows = -1;
int gemm_pair_min_rows() {
  if (g_pair_min_rows < 0) {
    const char* e = getenv("SMOE_GEMM_PAIR_MIN_ROWS");
    g_pair_min_rows = (e && atoi(e) >= 0) ? atoi(e) : 1024;
  }
  return g_pair_min_rows;
}
void set_gemm_pair_min_rows(int rows) { g_pair_min_rows = rows; }
void set_gemm_cta_group(int which, int cg) { g_cta_group[which ? 1 : 0] = (cg == 2) ? 2 : 1; }
int gemm_b_box_rows(int cg) { return kGemmBN / cg; }

// SMOE_OPT_GEMM_GROUP_M_UP / _DOWN: tile order override (0 = derived from K)
static int g_group_m[2] = {0, 0};
int gemm_group_m(int which) { return g_group_m[which ? 1 : 0]; }
void set_gemm_group_m(int which, int v) { g_group_m[which ? 1 : 0] = v; }

// SMOE_OPT_EARLY_DOWN (see GemmArgs::ready)
static int g_early_down = 1;
int gemm_early_down() { return g_early_down; }
void set_gemm_early_down(int on) { g_early_down = on ? 1 : 0; }

// -1: not set yet (env SMOE_GEMM_NARROW_MAX_ROWS, else 0 = off).  Off by
// default: the narrow variant wins only while the expert-input buffer's
// unused rows are zero (a fresh layer); in steady-state serving it measured
// neutral to 3% slower under the power cap (profiles/r1_narrow/).
static int g_narrow_max_rows = -1;
int gemm_narrow_max_rows() {
  if (g_narrow_max_rows < 0) {
    const char* e = getenv("SMOE_GEMM_NARROW_MAX_ROWS");
    g_narrow_max_rows = (e && atoi(e) >= 0) ? atoi(e) : 0;
  }
  return g_narrow_max_rows;
}
void set_gemm_narrow_max_rows(int rows) { g_narrow_max_rows = rows; }

int launch_grouped_gemm(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args,
                        int32_t epilogue, int cg, cudaStream_t st) {
  if (args.num_problems <= 0) return SMOE_OK;
  // readiness counters: one SM per 128-row tile on both sides (the epilogue
  // barrier counts four warps, the producer's target 128-row up tiles)
  if (args.ready_role != 0 && (cg != 1 || !args.ready)) return SMOE_ERR_INVALID_ARG;
  if (args.num_problems > kGemmMaxProblems) return SMOE_ERR_UNSUPPORTED;
  const bool pair = cg == 2;
  if (cg == 0) {   // narrow m-blocks (tmap_a has kGemmNarrowM-row boxes)
    if (args.num_problems > kGemmNarrowMaxProblems) return SMOE_ERR_UNSUPPORTED;
    switch (epilogue) {
      case kEpiStore: return launch_impl<kEpiStore, 1, 1>(a, b, args, st);
      case kEpiSwiGLU: return launch_impl<kEpiSwiGLU, 1, 1>(a, b, args, st);
      case kEpiScatter: return launch_impl<kEpiScatter, 1, 1>(a, b, args, st);
      default: return SMOE_ERR_INVALID_ARG;
    }
  }
  switch (epilogue) {
    case kEpiStore: return pair ? launch_impl<kEpiStore, 2>(a, b, args, st)
                                : launch_impl<kEpiStore, 1>(a, b, args, st);
    case kEpiSwiGLU: return pair ? launch_impl<kEpiSwiGLU, 2>(a, b, args, st)
                                 : launch_impl<kEpiSwiGLU, 1>(a, b, args, st);
    case kEpiScatter: return pair ? launch_impl<kEpiScatter, 2>(a, b, args, st)
                                  : launch_impl<kEpiScatter, 1>(a, b, args, st);
    default: return SMOE_ERR_INVALID_ARG;
  }
}

// w13[e, blk*256 + r]      = w1[e, blk*128 + r]        r < 128  (gate)
// w13[e, blk*256 + 128 + r] = w3[e, blk*128 + r]       r < 128  (up)
__global__ void pack_w13_kernel(const uint4* __restrict__ w1, const uint4* __restrict__ w3,
                                int64_t n_rows_out, int32_t ffn, int64_t row_vecs,
                                uint4* __restrict__ w13) {
  const int64_t total = n_rows_out * row_vecs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t orow = i / row_vecs, v = i - orow * row_vecs;
    const int64_t e = orow / (2 * ffn), r = orow - e * 2 * ffn;
    const int64_t blk = r / 256, rr = r - blk * 256;
    const int64_t src_row = e * ffn + blk * 128 + (rr & 127);
    w13[i] = (rr < 128 ? w1 : w3)[src_row * row_vecs + v];
  }
}

// dst box (rb, kb) = src rows [rb*256, +256) x cols [kb*64, +64), one 32 KiB run
__global__ void tile_weights_kernel(const uint4* __restrict__ src, int64_t rows, int64_t cols,
                                    uint4* __restrict__ dst) {
  const int64_t kbs = cols / kGemmBK;
  const int64_t total = rows * cols / 8;                  // 16-B vectors
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c8 = i & 7;                             // vector within a 64-element row
    const int64_t r = (i >> 3) & (kGemmBN - 1);           // row within the box
    const int64_t box = i >> 11;                          // 256 rows x 8 vectors per box
    const int64_t rb = box / kbs, kb = box - rb * kbs;
    dst[i] = src[((rb * kGemmBN + r) * cols + kb * kGemmBK) / 8 + c8];
  }
}

}  // namespace smoe

using namespace smoe;

extern "C" int smoe_tile_weights(const void* src, int64_t rows, int64_t cols, void* dst,
                                 void* stream) {
  if (!src || !dst || rows <= 0 || cols <= 0) return SMOE_ERR_INVALID_ARG;
  if (rows % kGemmBN || cols % kGemmBK) return SMOE_ERR_UNSUPPORTED;
  const int64_t vecs = rows * cols / 8;
  const int blocks = (int)std::min<int64_t>(ceil_div(vecs, 256), 148 * 32);
  tile_weights_kernel<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const uint4*>(src), rows,
                                                              cols, static_cast<uint4*>(dst));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_pack_w13(const void* w1, const void* w3, int32_t n_local_experts,
                             int32_t ffn, int32_t hidden, void* w13, void* stream) {
  if (n_local_experts <= 0 || ffn <= 0 || hidden <= 0 || !w1 || !w3 || !w13)
    return SMOE_ERR_INVALID_ARG;
  if (ffn % 128 != 0 || hidden % 8 != 0) return SMOE_ERR_UNSUPPORTED;
  const int64_t rows = (int64_t)n_local_experts * 2 * ffn;
  const int64_t vecs = hidden / 8;
  const int blocks = (int)std::min<int64_t>(ceil_div(rows * vecs, 256), 148 * 32);
  pack_w13_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      static_cast<const uint4*>(w1), static_cast<const uint4*>(w3), rows, ffn, vecs,
      static_cast<uint4*>(w13));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

extern "C" int smoe_grouped_gemm(const void* A, int64_t a_rows, int64_t K, const void* B,
                                 int64_t b_rows, int64_t n_b, const int64_t* problems,
                                 int32_t num_problems, int32_t epilogue, void* C, int64_t c_rows,
                                 int64_t ldc, void* stream) {
  (void)c_rows;
  if (!A || !B || !C || !problems || num_problems <= 0) return SMOE_ERR_INVALID_ARG;
  if (K % kGemmBK != 0 || n_b % kGemmBN != 0) return SMOE_ERR_UNSUPPORTED;
  if (epilogue != kEpiStore && epilogue != kEpiSwiGLU) return SMOE_ERR_INVALID_ARG;
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, A, a_rows, K, kGemmBM);
  if (rc) return rc;
  const int cg = gemm_cta_group(epilogue == kEpiSwiGLU ? 0 : 1);
  rc = make_tmap_bf16(&tb, B, b_rows, K, gemm_b_box_rows(cg));
  if (rc) return rc;
  GemmArgs args{};
  args.problems = problems;
  args.num_problems = num_problems;
  args.num_k_blocks = (int32_t)(K / kGemmBK);
  args.n_tiles_n = (int32_t)(n_b / kGemmBN);
  args.n_b = (int32_t)n_b;
  args.c = static_cast<char*>(C);
  args.ldc = ldc;
  return launch_grouped_gemm(ta, tb, args, epilogue, cg, as_stream(stream));
}

SMOE_TL_EXPORT(gemm)
