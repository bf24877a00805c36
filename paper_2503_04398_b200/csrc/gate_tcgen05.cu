// gate_tcgen05.cu — K4 on the 5th-generation tensor cores: router logits,
// softmax, top-k and the local/remote event count of every hidden row.
//
// The gate (semantics in DESIGN.md §2) multiplies each reduced
// hidden row h (bf16, d) by the N gate rows.  With N = 64 (DeepSeek-V2-Lite,
// Qwen2-MoE) the mma.sync kernel in layer_kernels.cu spends ~7x the HBM time
// of the rows it reads; here the contraction is one tcgen05 MMA chain per
// 128-row tile and the kernel streams h at HBM speed:
//
//   warp 0 lane 0  TMA producer: H tile 128 x 64 (from the resident shards'
//                  hs arena) + W tile N' x 64 per 64-wide k-block, 2 k-blocks
//                  per stage, 4-stage ring
//   warp 1 lane 0  tcgen05.mma.cta_group::1.kind::f16 M128 x N' x K16 into
//                  TMEM (fp32), two accumulators so the epilogue of tile t
//                  overlaps the MMAs of tile t + 1
//   warp 2         TMEM allocator
//   warps 4..7     epilogue, ONE THREAD PER ROW: tcgen05.ld 32x32b gives the
//                  thread its row's N' logits in registers; bias, max, softmax
//                  sum, top-k (larger logit first, lowest s-EG slot on ties) and
//                  the locality count need no shuffles or shared memory.  Each
//                  of the k selections is a max-TREE over the N' logits (depth
//                  log2 N', independent compares) instead of a linear scan:
//                  the scan was a 64-long dependent chain per pass and one
//                  warp per SMSP could not hide it (12 us of a 24 us decode
//                  gate at N = 64, k = 6).
//
// N' = N rounded up to 16 (the MMA's N granularity at M = 128); W rows past
// N are TMA out-of-bounds fills (zeros) and are masked to -inf.  Rows past a
// shard's token count are computed and discarded.
#include "common.cuh"
#include "gate_select.cuh"
#include "gemm.h"
#include "layer_kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstdlib>

namespace smoe {

// Timeline probe (build variant -DSMOE_GATE_PROBE only, tools/probe/gate_timeline.py):
// %globaltimer per CTA at fixed points of its first tile (16 slots; 8..12 and 14
// are inside the register epilogue / fused route, recorded by its first thread).
#ifdef SMOE_GATE_PROBE
__device__ unsigned long long g_gate_ts[2048][16];
#define GATE_TS(i)                                                                   \
  do {                                                                               \
    unsigned long long t_;                                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
    if (blockIdx.x < 2048) g_gate_ts[blockIdx.x][i] = t_;                            \
  } while (0)
#else
#define GATE_TS(i) \
  do {             \
  } while (0)
#endif

#ifndef SMOE_GATE_SPLIT
#define SMOE_GATE_SPLIT 1         // two epilogue threads per row at N' = 64 (0: one)
#endif
#ifndef SMOE_GATE_REG_MAX_NP
#define SMOE_GATE_REG_MAX_NP 64   // 32 (tournament for 48 / 64) measured: profiles/r2/gate/
#endif
#ifndef SMOE_GATE_WARP_ROWS
#define SMOE_GATE_WARP_ROWS 1     // a warp per row for tiles of <= 32 rows, N' >= 32 (0: off)
#endif

constexpr int kGtThreads = 256;
constexpr int kGtRows = 128;                               // MMA M: rows per tile
constexpr uint32_t kGtBoxBytes = kGtRows * kGemmBK * 2;   // one 128 x 64 H box: 16 KiB
constexpr int kGtMaxK = 8;

// NP = W rows (N rounded up to 16); SUB = 64-wide k-blocks per stage (one TMA
// box each, so a stage reads SUB * 128 contiguous bytes of every hidden row);
// ST = stages in the ring.
// Epilogue kind by N': up to kGtRegMaxNP every logit of a row lives in one
// thread's registers and each of the k selections is a max-tree over all of
// them; above it the row's logits are staged in shared memory and the
// selection is a two-level tournament over 16-column chunks.
constexpr int kGtRegMaxNP = SMOE_GATE_REG_MAX_NP;

template <int NP, int SUB, int ST> struct GtShape {
  static constexpr int kStages = ST;
  static constexpr bool kWide = NP > kGtRegMaxNP;
  // register path at N' = 64: two epilogue threads per row (warps 4..11, the
  // second four reading the upper 32 columns of the same TMEM lane quarters)
  // halve each thread's selection chain and give every SMSP two warps
  static constexpr int kSplit = (SMOE_GATE_SPLIT && !kWide && NP == 64) ? 2 : 1;
  static constexpr int kThreads = 128 + 128 * kSplit;
  static constexpr int kHalf = NP / kSplit;                // columns per epilogue thread
  static constexpr uint32_t kXchBytes = kSplit > 1 ? 128 * 80 : 0;   // per row: 8 keys,
                                                                      // 8 slots, max, sum
  static constexpr int kRows = kGtRows;
  static constexpr uint32_t kBox = kRows * kGemmBK * 2;    // one H box (TMA)
  static constexpr uint32_t kHBytes = SUB * kBox;
  static constexpr uint32_t kWBox = NP * kGemmBK * 2;     // NP rows of 128 B
  static constexpr uint32_t kWBytes = SUB * kWBox;
  static constexpr uint32_t kStageBytes = kHBytes + kWBytes;
  static constexpr uint32_t kTmemCols =
      2 * NP <= 32 ? 32 : 2 * NP <= 64 ? 64 : 2 * NP <= 128 ? 128 : 2 * NP <= 256 ? 256 : 512;
  static constexpr uint32_t kAccCols = kTmemCols / 2;      // column stride of the 2 accumulators
  // wide: each epilogue thread stages its row's logits in shared memory
  // (kWideRows rows at a time: 128, or 64 in two phases for N' > 192)
  static constexpr int kWideRows = NP > 192 ? 64 : 128;
  static constexpr int kWideLd = NP + 4;                   // floats per staged row (16 B pad)
  // + per staged row: each 16-column chunk's winner key / slot / taken mask
  // and the k selections (key, slot), stored field-major ([field][row]: the
  // lanes of a warp hit consecutive banks)
  static constexpr int kWideFields = 3 * (NP / 16) + 2 * kGtMaxK;
  static constexpr uint32_t kWideBytes =
      kWide ? kWideRows * kWideLd * 4 + kWideRows * kWideFields * 4 : 0;
  static constexpr size_t kSmem = 1024 + ST * kStageBytes + 128 + kWideBytes + kXchBytes;
  // register path, tiles of <= 32 valid rows: rows staged in shared memory,
  // a warp per row (static __shared__: plain LDS / STS)
  static constexpr bool kWarpRows = SMOE_GATE_WARP_ROWS && !kWide && NP >= 32;
  static constexpr int kWrLd = NP + 1;
  static constexpr int kWrFloats = kWarpRows ? 32 * kWrLd + 4 * kSplit * 64 : 1;
  // D f32, A/B bf16, both K-major, N = NP, M = 128
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                     (uint32_t(NP >> 3) << 17) | (uint32_t(kGtRows >> 4) << 24);
};

template <int NP, int SUB, int ST>
__global__ void __launch_bounds__(GtShape<NP, SUB, ST>::kThreads, 1)
gate_tc_kernel(const __grid_constant__ CUtensorMap tmap_h,
               const __grid_constant__ CUtensorMap tmap_w, const GateTcArgs a) {
  using S = GtShape<NP, SUB, ST>;
  constexpr int kGtStages = S::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_h = smem;
  uint8_t* smem_w = smem + kGtStages * S::kHBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_w + kGtStages * S::kWBytes);
  // bars: full[kGtStages], empty[kGtStages], tfull[2], tempty[2]
  float* wide = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 128);
  // split epilogue exchange: row r at xch + r * 20 words
  int32_t* xch = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(wide) + S::kWideBytes);
  __shared__ uint32_t tmem_holder;
  __shared__ int32_t s_cnt[SMOE_MAX_SHARDS];
  __shared__ int32_t s_prefix[SMOE_MAX_SHARDS + 1];
  __shared__ char* s_ids[SMOE_MAX_SHARDS];
  __shared__ char* s_wts[SMOE_MAX_SHARDS];
  __shared__ float s_bias[NP];
  __shared__ int32_t s_owner[NP];        // cluster of each expert slot (locality count)
  __shared__ float wr[S::kWrFloats];      // warp-per-row staging + scratch

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SMOE_TL_ENTER(2);
  if (threadIdx.x == 0) GATE_TS(0);
  if (threadIdx.x < NP) {
    s_bias[threadIdx.x] = (a.b_gate && threadIdx.x < a.n_experts) ? a.b_gate[threadIdx.x] : 0.f;
    // staged once: the epilogue's k owner lookups per row would otherwise be
    // dependent global loads (12 us of a 24 us decode gate at N = 64, k = 6)
    s_owner[threadIdx.x] = threadIdx.x < a.n_experts ? a.slot_owner[threadIdx.x] : -1;
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kGtStages; ++s) {
      mbar_init(smem_addr(&bars[s]), 1);
      mbar_init(smem_addr(&bars[kGtStages + s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_addr(&bars[2 * kGtStages + b]), 1);
      // one arrival per epilogue warp
      mbar_init(smem_addr(&bars[2 * kGtStages + 2 + b]), 4 * S::kSplit);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tmap_h) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tmap_w) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_addr(&tmem_holder)), "r"(S::kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // Everything above reads constant data only (weights, tensor maps).  The
  // shard row counts (plan) are read before the wait too: the SRS kernel this
  // gate follows triggers only after its own wait, i.e. after the plan
  // completed (profiles/r2/decode/prewait2/).  The dependents' early launch
  // is triggered at the END of this kernel: the dispatch kernel's CTAs,
  // resident and waiting from the start, slowed this gate (64-token forward
  // DSV2-Lite / Qwen2 -6.5 / -5.5 us, profiles/r2/decode/pdl_trigger/)
  if (threadIdx.x < 32) {
    // one lane per shard: the count loads are in flight together
    const int i = threadIdx.x;
    int32_t c = 0;
    if (i < a.shard_count)
      c = a.counts ? a.counts[a.shard_begin + i] : (i == 0 ? (int32_t)a.single_rows : 0);
    const int32_t tiles = (c + S::kRows - 1) / S::kRows;
    int32_t incl = tiles;                  // inclusive prefix of the tile counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (i >= o) incl += v;
    }
    if (i < a.shard_count) {
      s_cnt[i] = c;
      s_prefix[i] = incl - tiles;
    }
    if (i == a.shard_count - 1) s_prefix[a.shard_count] = incl;
    if (i == 0) {
#pragma unroll
      for (int j = 0; j < SMOE_MAX_SHARDS; ++j) {
        s_ids[j] = a.topk_ids.p[j];
        s_wts[j] = a.topk_w.p[j];
      }
    }
  }
  pdl_wait();
  SMOE_TL_WAITED(2);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_holder;
  const int32_t total = s_prefix[a.shard_count];
  if (threadIdx.x == 0) GATE_TS(1);
  const uint32_t full0 = smem_addr(&bars[0]);
  const uint32_t empty0 = smem_addr(&bars[kGtStages]);
  const uint32_t tfull0 = smem_addr(&bars[2 * kGtStages]);
  const uint32_t tempty0 = smem_addr(&bars[2 * kGtStages + 2]);

  auto decode = [&](int32_t t, int32_t& gl, int32_t& blk) {
    gl = 0;
    while (gl + 1 < a.shard_count && s_prefix[gl + 1] <= t) ++gl;
    blk = t - s_prefix[gl];
  };

  if (warp == 3) {
    // fused route: shards without rows have no tile -- CTA 0's idle warp
    // publishes their zero rows of the count matrix
    if (a.route && blockIdx.x == 0) {
      const int32_t Nn = a.n_experts;
      for (int gl = 0; gl < a.shard_count; ++gl) {
        if (s_cnt[gl] != 0) continue;
        const int64_t g = a.shard_begin + gl;
        for (int e = lane; e < Nn; e += 32)
          for (int i = 0; i < a.n_count_bufs; ++i)
            reinterpret_cast<int32_t*>(a.count_bufs.p[i])[g * Nn + e] = 0;
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int32_t stage = 0;
      uint32_t phase = 0;
      for (int32_t t = blockIdx.x; t < total; t += gridDim.x) {
        int32_t gl, blk;
        decode(t, gl, blk);
        const int32_t row = (int32_t)(gl * a.rows_per_shard + (int64_t)blk * S::kRows);
        for (int32_t kb = 0; kb < a.num_k_blocks; kb += SUB) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t fb = full0 + 8 * stage;
          mbar_expect_tx(fb, S::kStageBytes);
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
            tma_load_2d(smem_addr(smem_h + stage * S::kHBytes + u * S::kBox), &tmap_h, fb,
                        (kb + u) * kGemmBK, row);
            tma_load_2d(smem_addr(smem_w + stage * S::kWBytes + u * S::kWBox), &tmap_w, fb,
                        (kb + u) * kGemmBK, 0);
          }
          if (++stage == kGtStages) { stage = 0; phase ^= 1; }
        }
        if (t == (int32_t)blockIdx.x) GATE_TS(2);         // last TMA of the first tile issued
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      int32_t stage = 0;
      uint32_t phase = 0, acc = 0, acc_phase = 0;
      for (int32_t t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * S::kAccCols;
        for (int32_t kb = 0; kb < a.num_k_blocks; kb += SUB) {
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          if (kb == 0 && t == (int32_t)blockIdx.x) GATE_TS(3);   // first stage landed
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
            const uint64_t hd = sdesc(smem_addr(smem_h + stage * S::kHBytes + u * S::kBox));
            const uint64_t wd = sdesc(smem_addr(smem_w + stage * S::kWBytes + u * S::kWBox));
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k)
              tc_mma(d_tmem, hd + 2 * k, wd + 2 * k, S::kIdesc, (kb | u | k) != 0);
          }
          tc_commit(empty0 + 8 * stage);
          if (++stage == kGtStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(tfull0 + 8 * acc);
        if (t == (int32_t)blockIdx.x) GATE_TS(4);         // last MMA of the first tile issued
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: thread = row (kSplit threads per row at N' = 64) =====
    const int ew = (warp - 4) & 3;                 // TMEM lane quarter
    const int hf = (warp - 4) >> 2;                // column half (split epilogue)
    const int N = a.n_experts, K = a.k;
    uint32_t acc = 0, acc_phase = 0;
    unsigned long long my_local = 0, my_remote = 0, my_rrows = 0;
    // order-preserving int keys (+0 and -0 merged, -inf an ordinary
    // candidate); INT_MIN marks "not a candidate" (slots >= N, slots
    // already taken), so fewer than k finite logits still give k distinct
    // slots, as the stable argsort of the reference idiom does
    auto to_key = [](float x) {
      const int32_t b = __float_as_int(x + 0.0f);
      return b >= 0 ? b : b ^ 0x7fffffff;
    };
    auto key_to_f = [](int32_t k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); };
    for (int32_t t = blockIdx.x; t < total; t += gridDim.x) {
      int32_t gl, blk;
      decode(t, gl, blk);
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      if (ew == 0 && lane == 0 && t == (int32_t)blockIdx.x) GATE_TS(5);   // accumulator ready
      const uint32_t taddr = tmem_base + acc * S::kAccCols + ((uint32_t)(ew * 32) << 16);
      const int64_t j = (int64_t)blk * S::kRows + ew * 32 + lane;
      int sel_e[kGtMaxK];
      int32_t sel_k[kGtMaxK];
      float ex = 0.f;
      if constexpr (!S::kWide) {
        // every logit of the row in registers; the accumulator is released
        // before the selection so the MMAs of tile t + 2 can start
        constexpr int NH = S::kHalf;             // columns of this thread
        const int c0 = hf * NH;                  // first slot of this thread's columns
        uint32_t v[NH];
#pragma unroll
        for (int c = 0; c < NH / 16; ++c) SMOE_TMEM_LD16(taddr + c0 + c * 16, (v + c * 16));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty0 + 8 * acc);     // accumulator free for tile t + 2
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        if (threadIdx.x == 128) GATE_TS(8);                // logits in registers
        if constexpr (S::kWarpRows) {
          const int32_t rows_t = min(S::kRows, s_cnt[gl] - blk * S::kRows);
          if (rows_t <= 32) {
            // ===== warp per row (tile-uniform branch); arithmetic as below
            {
              const int r = ew * 32 + lane;
              if (r < rows_t) {
                float* dst = wr + r * S::kWrLd + c0;
#pragma unroll
                for (int e = 0; e < NH; ++e) dst[e] = __uint_as_float(v[e]) + s_bias[c0 + e];
              }
            }
            asm volatile("bar.sync 6, %0;" :: "n"(128 * S::kSplit) : "memory");
            const int we = warp - 4;
            float* sc = wr + 32 * S::kWrLd + we * 64;
            const bool v0 = lane < N, v1 = lane + 32 < N;
            for (int r = we; r < rows_t; r += 4 * S::kSplit) {
              const float* xr = wr + r * S::kWrLd;
              const float x0 = v0 ? xr[lane] : 0.f;
              const float x1 = v1 ? xr[lane + 32] : 0.f;
              int32_t k0 = v0 ? to_key(x0) : INT_MIN;
              int32_t k1 = v1 ? to_key(x1) : INT_MIN;
              const int32_t h0 = __reduce_max_sync(0xffffffffu, k0);
              const int32_t h1 = __reduce_max_sync(0xffffffffu, k1);
              int sel_e[kGtMaxK];
              int32_t sel_k[kGtMaxK];
#pragma unroll
              for (int s = 0; s < kGtMaxK; ++s) {
                sel_e[s] = 0;
                sel_k[s] = INT_MIN;
                if (s < K) {
                  // the max key, then the lowest slot holding it (the tree's order)
                  const int32_t mk = __reduce_max_sync(0xffffffffu, max(k0, k1));
                  const uint32_t b0 = __ballot_sync(0xffffffffu, k0 == mk);
                  const uint32_t b1 = __ballot_sync(0xffffffffu, k1 == mk);
                  const int bs = b0 ? __ffs(b0) - 1 : 31 + __ffs(b1);
                  sel_e[s] = bs;
                  sel_k[s] = mk;
                  if (bs == lane) k0 = INT_MIN;
                  if (bs == lane + 32) k1 = INT_MIN;
                }
              }
              // softmax denominator: terms in parallel, lane 0 sums them in
              // the thread paths' column order
              float ex_r = 0.f;
              if constexpr (S::kSplit == 1) {
                const float mx = key_to_f(sel_k[0]);
                if (v0) sc[lane] = __expf(x0 - mx);
                if (v1) sc[lane + 32] = __expf(x1 - mx);
                __syncwarp();
                if (lane == 0) {
                  for (int e = 0; e < NP; ++e)
                    if (e < N) ex_r += sc[e];
                }
              } else {
                const float mh = key_to_f(h0), m1 = key_to_f(h1);
                if (v0) sc[lane] = __expf(x0 - mh);
                if (v1) sc[lane + 32] = __expf(x1 - m1);
                __syncwarp();
                if (lane == 0) {
                  float sh = 0.f, s1 = 0.f;
                  if (mh > -INFINITY) {
                    for (int e = 0; e < 32; ++e)
                      if (e < N) sh += sc[e];
                  }
                  if (m1 > -INFINITY) {
                    for (int e = 0; e < 32; ++e)
                      if (32 + e < N) s1 += sc[32 + e];
                  }
                  const float mx = key_to_f(sel_k[0]);
                  ex_r = mx > -INFINITY ? sh * __expf(mh - mx) + s1 * __expf(m1 - mx)
                                        : __int_as_float(0x7fc00000);
                }
              }
              // weights / stores / locality, lane s = selection s (the tail's expressions)
              const float inv = __shfl_sync(0xffffffffu, 1.0f / ex_r, 0);
              const float mx = key_to_f(sel_k[0]);
              int my_e = 0;
              int32_t my_k = INT_MIN;
#pragma unroll
              for (int s = 0; s < kGtMaxK; ++s)
                if (lane == s) { my_e = sel_e[s]; my_k = sel_k[s]; }
              const float p_s = lane < K ? __expf(key_to_f(my_k) - mx) * inv : 0.f;
              float psum = 0.f;
#pragma unroll
              for (int s = 0; s < kGtMaxK; ++s) psum += __shfl_sync(0xffffffffu, p_s, s);
              const float scale = a.renorm ? 1.0f / psum : 1.0f;
              const int64_t jr = (int64_t)blk * S::kRows + r;
              const int32_t g = a.shard_begin + gl;
              const int32_t o = lane < K ? s_owner[my_e] : -1 - lane;
              if (lane < K) {
                reinterpret_cast<int32_t*>(s_ids[gl])[jr * K + lane] = my_e;
                reinterpret_cast<float*>(s_wts[gl])[jr * K + lane] = p_s * scale;
              }
              const uint32_t same = __match_any_sync(0xffffffffu, o);
              const uint32_t kmask = (1u << K) - 1u;
              const uint32_t loc = __ballot_sync(0xffffffffu, lane < K && o == g);
              const uint32_t first = __ballot_sync(0xffffffffu, (same & lanemask_lt()) == 0u);
              if (lane == 0) {
                const int nl = __popc(loc);
                my_local += nl;
                my_remote += K - nl;
                my_rrows += __popc(first & kmask & ~loc);
              }
              __syncwarp();
            }
            asm volatile("bar.sync 6, %0;" :: "n"(128 * S::kSplit) : "memory");
            continue;
          }
        }
        if (S::kSplit == 1 && j >= s_cnt[gl]) continue;
        constexpr int NT = NH <= 16 ? 16 : (NH <= 32 ? 32 : 64);   // tree leaves (power of 2)
        int32_t key[NT];
#pragma unroll
        for (int e = 0; e < NT; ++e)
          key[e] = (e < NH && c0 + e < N)
                       ? to_key(__uint_as_float(v[e < NH ? e : 0]) + s_bias[c0 + (e < NH ? e : 0)])
                       : INT_MIN;
        uint64_t taken = 0;      // a bit mask, not stores into key[]: a store at the
                                 // winner's index became local memory (STL)
#pragma unroll
        for (int s = 0; s < kGtMaxK; ++s) {
          sel_e[s] = 0;
          sel_k[s] = INT_MIN;
          if (s < K) {
            // max-tree: the right child wins only when strictly larger, so
            // equal logits resolve to the lower s-EG slot (test_acceptance.py:179-193)
            int32_t tv[NT / 2];
            int ti[NT / 2];
#pragma unroll
            for (int i = 0; i < NT / 2; ++i) {
              const int32_t k0 = ((taken >> (2 * i)) & 1) ? INT_MIN : key[2 * i];
              const int32_t k1 = ((taken >> (2 * i + 1)) & 1) ? INT_MIN : key[2 * i + 1];
              const bool r = k1 > k0;
              tv[i] = r ? k1 : k0;
              ti[i] = r ? 2 * i + 1 : 2 * i;
            }
#pragma unroll
            for (int w = NT / 4; w >= 1; w >>= 1) {
#pragma unroll
              for (int i = 0; i < w; ++i) {
                const bool r = tv[2 * i + 1] > tv[2 * i];
                tv[i] = r ? tv[2 * i + 1] : tv[2 * i];
                ti[i] = r ? ti[2 * i + 1] : ti[2 * i];
              }
            }
            sel_e[s] = c0 + ti[0];
            sel_k[s] = tv[0];
            taken |= 1ull << ti[0];
          }
        }
        if (threadIdx.x == 128) GATE_TS(9);                // k selections done
        if constexpr (S::kSplit == 1) {
          const float mx = key_to_f(sel_k[0]);
#pragma unroll
          for (int e = 0; e < NP; ++e)
            if (e < N) ex += __expf(__uint_as_float(v[e]) + s_bias[e] - mx);
        } else {
          // this half's softmax sum relative to its own max, then the upper
          // half hands (top-k, max, sum) to the lower one through shared
          // memory; the lower half merges the two sorted lists (its own
          // entries -- the lower slots -- first on equal keys) and rescales
          // the two sums to the row's max, in a fixed order
          const float mh = key_to_f(sel_k[0]);
          float sh = 0.f;                      // 0 when this half has no finite logit
          if (mh > -INFINITY) {
#pragma unroll
            for (int e = 0; e < NH; ++e)
              if (c0 + e < N) sh += __expf(__uint_as_float(v[e]) + s_bias[c0 + e] - mh);
          }
          int32_t* xr = xch + (ew * 32 + lane) * 20;
          if (hf == 1) {
#pragma unroll
            for (int s = 0; s < kGtMaxK; ++s) {
              xr[s] = sel_k[s];
              xr[8 + s] = sel_e[s];
            }
            xr[16] = __float_as_int(mh);
            xr[17] = __float_as_int(sh);
          }
          // the two warps of this lane quarter (barrier ids 1..4; 0 is
          // __syncthreads); both barriers are warp-uniform
          if (threadIdx.x == 128) GATE_TS(10);               // softmax sum, exchange written
          asm volatile("bar.sync %0, 64;" :: "r"(1 + ew) : "memory");
          const bool mine = hf == 0 && j < s_cnt[gl];
          float m1 = -INFINITY, s1 = 0.f;
          if (mine) {
            int32_t mk[kGtMaxK];
            int me[kGtMaxK];
            int ia = 0, ib = 0;
#pragma unroll
            for (int s = 0; s < kGtMaxK; ++s) {
              mk[s] = INT_MIN;
              me[s] = 0;
              if (s < K) {
                int32_t ka = INT_MIN;
                int ea = 0;
#pragma unroll
                for (int q = 0; q < kGtMaxK; ++q)
                  if (q == ia) { ka = sel_k[q]; ea = sel_e[q]; }
                const int32_t kb_ = xr[ib];
                if (ka >= kb_) { mk[s] = ka; me[s] = ea; ++ia; }
                else { mk[s] = kb_; me[s] = xr[8 + ib]; ++ib; }
              }
            }
#pragma unroll
            for (int s = 0; s < kGtMaxK; ++s) {
              sel_k[s] = mk[s];
              sel_e[s] = me[s];
            }
            m1 = __int_as_float(xr[16]);
            s1 = __int_as_float(xr[17]);
          }
          asm volatile("bar.sync %0, 64;" :: "r"(1 + ew) : "memory");     // xch reusable
          if (threadIdx.x == 128) GATE_TS(11);               // halves merged
          if (!mine) continue;
          const float mx = key_to_f(sel_k[0]);
          // all -inf rows: NaN, as the single-thread path gives
          ex = mx > -INFINITY ? sh * __expf(mh - mx) + s1 * __expf(m1 - mx) : __int_as_float(0x7fc00000);
        }
      } else {
        // N' > kGtRegMaxNP (e.g. DeepSeek-V2, 160 experts): too many logits
        // for one thread's registers.  A two-level tournament: one pass over
        // the row in 16-column TMEM chunks (warp-uniform loads) stages the
        // biased logits in shared memory with each chunk's winner (max-tree,
        // the lower slot winning ties) and an online softmax denominator;
        // each selection takes the best chunk winner (the lower chunk on
        // ties) and refills only that chunk from shared memory.  Every loop
        // over chunks and selections is ROLLED, with the per-chunk state in
        // the row's shared-memory record: fully unrolled, the N' = 160 epilogue
        // was ~6 900 straight-line instructions per warp that missed the
        // instruction cache on nearly every issue (34 us of an 82 us gate,
        // profiles/r2/gate/).  For N' > 192 the rows are staged 64 at a time.
        constexpr int NC = NP / 16;
        constexpr int kGroups = 128 / S::kWideRows;          // 1, or 2 for N' > 192
        constexpr int kWarpsPerGroup = 4 / kGroups;
        const int srow = (ew % kWarpsPerGroup) * 32 + lane;     // staging row of this thread
        float* myrow = wide + srow * S::kWideLd;
        constexpr int R = S::kWideRows;                          // field stride
        int32_t* fld = reinterpret_cast<int32_t*>(wide + R * S::kWideLd) + srow;
        int32_t* cwk = fld;                                      // [NC] chunk winner keys
        int32_t* cwi = fld + NC * R;                             // [NC] their slots
        int32_t* ctk = fld + 2 * NC * R;                         // [NC] taken masks
        int32_t* sk = fld + 3 * NC * R;                          // [kGtMaxK] selections
        int32_t* se = sk + kGtMaxK * R;
        // max-tree over the 16 staged keys of chunk c (taken / invalid -> INT_MIN)
        auto chunk_best = [&](int c, const float (&x)[16], uint32_t taken, int32_t& bk,
                              int& bi) {
          int32_t tv[8];
          int ti[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int e0 = c * 16 + 2 * i, e1 = e0 + 1;
            const int32_t k0 = (e0 < N && !((taken >> (2 * i)) & 1)) ? to_key(x[2 * i]) : INT_MIN;
            const int32_t k1 = (e1 < N && !((taken >> (2 * i + 1)) & 1)) ? to_key(x[2 * i + 1])
                                                                            : INT_MIN;
            const bool r = k1 > k0;
            tv[i] = r ? k1 : k0;
            ti[i] = r ? e1 : e0;
          }
#pragma unroll
          for (int w = 4; w >= 1; w >>= 1) {
#pragma unroll
            for (int i = 0; i < w; ++i) {
              const bool r = tv[2 * i + 1] > tv[2 * i];
              tv[i] = r ? tv[2 * i + 1] : tv[2 * i];
              ti[i] = r ? ti[2 * i + 1] : ti[2 * i];
            }
          }
          bk = tv[0];
          bi = ti[0];
        };
#pragma unroll 1
        for (int grp = 0; grp < kGroups; ++grp) {
          if (ew / kWarpsPerGroup == grp) {
            float m = -INFINITY;
#pragma unroll 1
            for (int c = 0; c < NC; ++c) {
              uint32_t v[16];
              SMOE_TMEM_LD16(taddr + c * 16, v);
              tmem_wait_ld();
              float x[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) x[i] = __uint_as_float(v[i]) + s_bias[c * 16 + i];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                *reinterpret_cast<float4*>(myrow + c * 16 + 4 * q) =
                    make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
              int32_t bk;
              int bi;
              chunk_best(c, x, 0u, bk, bi);
              cwk[c * R] = bk;
              cwi[c * R] = bi;
              ctk[c * R] = 0;
              float cm = -INFINITY;
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (c * 16 + i < N) cm = fmaxf(cm, x[i]);
              const float mn = fmaxf(m, cm);
              if (mn > -INFINITY) {
                ex = (m > -INFINITY ? ex * __expf(m - mn) : 0.f);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                  if (c * 16 + i < N) ex += __expf(x[i] - mn);
                m = mn;
              }
            }
            // every TMEM read of this warp is done: release its accumulator lanes
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
#pragma unroll 1
            for (int s = 0; s < K; ++s) {
              int32_t bk = cwk[0];
              int bc = 0;
#pragma unroll 1
              for (int c = 1; c < NC; ++c) {
                const int32_t ck = cwk[c * R];
                if (ck > bk) { bk = ck; bc = c; }
              }
              const int bi = cwi[bc * R];
              const uint32_t taken = (uint32_t)ctk[bc * R] | (1u << (bi & 15));
              ctk[bc * R] = (int32_t)taken;
              sk[s * R] = bk;
              se[s * R] = bi;
              if (s + 1 < K) {                   // refill the winning chunk (own row, smem)
                float x[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float4 f = *reinterpret_cast<const float4*>(myrow + bc * 16 + 4 * q);
                  x[4 * q] = f.x; x[4 * q + 1] = f.y; x[4 * q + 2] = f.z; x[4 * q + 3] = f.w;
                }
                int32_t nk;
                int ni;
                chunk_best(bc, x, taken, nk, ni);
                cwk[bc * R] = nk;
                cwi[bc * R] = ni;
              }
            }
#pragma unroll
            for (int s = 0; s < kGtMaxK; ++s) {
              sel_k[s] = s < K ? sk[s * R] : INT_MIN;
              sel_e[s] = s < K ? se[s * R] : 0;
            }
          }
          if constexpr (kGroups > 1) {
            // the next group's warps reuse the staging rows
            asm volatile("bar.sync 1, 128;" ::: "memory");
          }
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        if (j >= s_cnt[gl]) continue;
      }
      const float mx = key_to_f(sel_k[0]);
      const float inv = 1.0f / ex;
      float sel_p[kGtMaxK];
      float psum = 0.f;
#pragma unroll
      for (int s = 0; s < kGtMaxK; ++s) {
        sel_p[s] = s < K ? __expf(key_to_f(sel_k[s]) - mx) * inv : 0.f;
        psum += sel_p[s];
      }
      const int32_t g = a.shard_begin + gl;
      int32_t* ids = reinterpret_cast<int32_t*>(s_ids[gl]) + j * K;
      float* wts = reinterpret_cast<float*>(s_wts[gl]) + j * K;
      const float scale = a.renorm ? 1.0f / psum : 1.0f;
#pragma unroll
      for (int s = 0; s < kGtMaxK; ++s) {
        if (s < K) {
          ids[s] = sel_e[s];
          wts[s] = sel_p[s] * scale;
          const int32_t o = s_owner[sel_e[s]];
          if (o == g) {
            ++my_local;
          } else {
            ++my_remote;
            bool seen = false;                           // first pair to this shard?
#pragma unroll
            for (int s2 = 0; s2 < kGtMaxK; ++s2)
              if (s2 < s) seen |= s_owner[sel_e[s2]] == o;
            if (!seen) ++my_rrows;
          }
        }
      }
    }
    __syncwarp();
    if (ew == 0 && lane == 0 && hf == 0) GATE_TS(6);      // epilogue warp 4 done
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      my_local += __shfl_xor_sync(0xffffffffu, my_local, o);
      my_remote += __shfl_xor_sync(0xffffffffu, my_remote, o);
      my_rrows += __shfl_xor_sync(0xffffffffu, my_rrows, o);
    }
    if (lane == 0 && a.stats && (my_local | my_remote)) {
      atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + SMOE_STAT_LOCAL_PAIRS), my_local);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + SMOE_STAT_REMOTE_PAIRS),
                my_remote);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + SMOE_STAT_REMOTE_ROWS), my_rrows);
    }
    if (threadIdx.x == 128) GATE_TS(12);                  // + stats atomics
    if (a.route && (int32_t)blockIdx.x < total && hf == 0) {
      // ===== fused route (decode-sized batches: this CTA's one tile is all
      // of its shard's rows): stable rank of every pair among the shard's
      // pairs of its expert, in pair order p = row * k + s, 128 pairs per
      // round (match_any ranks inside a warp, per-warp counts in shared
      // memory) -- the route_rank_kernel result without its launch.  The
      // ring's shared memory is idle now (its only tile is consumed).
      int32_t gl, blk;
      decode(blockIdx.x, gl, blk);
      const int32_t Nn = a.n_experts;
      const int tid_e = ew * 32 + lane;
      int32_t* s_w = reinterpret_cast<int32_t*>(smem_h);    // [4][Nn] counts per warp
      int32_t* s_pre = s_w + 4 * Nn;                         // [Nn] earlier rounds' counts
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int e = tid_e; e < 5 * Nn; e += 128) s_w[e] = 0;
      asm volatile("bar.sync 5, 128;" ::: "memory");         // + this tile's ids stored
      const int64_t P = (int64_t)s_cnt[gl] * K;
      const int32_t* ids = reinterpret_cast<const int32_t*>(s_ids[gl]);
      int32_t* rank = reinterpret_cast<int32_t*>(a.pair_rank.p[gl]);
      for (int64_t c0 = 0; c0 < P; c0 += 128) {
        const int64_t p = c0 + tid_e;
        const int32_t e = p < P ? ids[p] : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, e);
        const int32_t rw = __popc(peers & lanemask_lt());
        if (e >= 0 && lane == __ffs(peers) - 1) s_w[ew * Nn + e] = __popc(peers);
        asm volatile("bar.sync 5, 128;" ::: "memory");
        if (e >= 0) {
          int32_t r = s_pre[e] + rw;
          for (int w = 0; w < ew; ++w) r += s_w[w * Nn + e];
          rank[p] = r;
        }
        asm volatile("bar.sync 5, 128;" ::: "memory");
        for (int ee = tid_e; ee < Nn; ee += 128) {
          int32_t sum = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) { sum += s_w[w * Nn + ee]; s_w[w * Nn + ee] = 0; }
          s_pre[ee] += sum;
        }
        asm volatile("bar.sync 5, 128;" ::: "memory");
      }
      // the shard's row of the [G, N] count matrix, to every process
      const int64_t g = a.shard_begin + gl;
      for (int ee = tid_e; ee < Nn; ee += 128)
        for (int i = 0; i < a.n_count_bufs; ++i)
          reinterpret_cast<int32_t*>(a.count_bufs.p[i])[g * Nn + ee] = s_pre[ee];
      if (threadIdx.x == 128) GATE_TS(14);                // fused route done
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) GATE_TS(7);
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 :: "r"(tmem_base), "r"(S::kTmemCols) : "memory");
  }
  pdl_trigger();
  SMOE_TL_EXIT(2);
}

template <int NP, int SUB, int ST>
static int launch_cfg(const CUtensorMap& mh, const CUtensorMap& mw, const GateTcArgs& a,
                      int64_t n_rows_bound, cudaStream_t st) {
  using S = GtShape<NP, SUB, ST>;
  static_assert(S::kSmem <= 227 * 1024, "shared memory budget of one CTA per SM");
  static bool attr = false;
  if (!attr) {
    SMOE_CUDA_TRY(cudaFuncSetAttribute(gate_tc_kernel<NP, SUB, ST>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::kSmem));
    attr = true;
  }
  const int64_t tiles = ceil_div(n_rows_bound, kGtRows) + a.shard_count;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms()));
  SMOE_CUDA_TRY(launch_pdl(gate_tc_kernel<NP, SUB, ST>, grid, S::kThreads, S::kSmem, st, mh, mw, a));
  SMOE_LAUNCH_CHECK();
  return SMOE_OK;
}

// Ring shape (SMOE_GATE_RING=<k-blocks per stage>x<stages>, tuning only):
// 1x8, 2x4 (default) or 4x2.
static int ring_sub() {
  static int sub = [] {
    const char* e = getenv("SMOE_GATE_RING");
    const int v = e ? atoi(e) : 2;
    return (v == 1 || v == 2 || v == 4) ? v : 2;
  }();
  return sub;
}

template <int NP>
static int launch_np(const CUtensorMap& mh, const CUtensorMap& mw, const GateTcArgs& a,
                     int64_t n_rows_bound, cudaStream_t st) {
  if constexpr (NP > 64) {
    // wide gates: one k-block per stage, and fewer stages to leave room for
    // the staged logits (NP <= 160: 3 stages, else 2)
    return launch_cfg<NP, 1, (NP <= 160 ? 3 : 2)>(mh, mw, a, n_rows_bound, st);
  } else if constexpr (GtShape<NP, 2, 3>::kWide) {
    // shared-memory tournament at N' <= 64: 3 stages of 2 k-blocks leave room
    // for the 128 staged rows
    return launch_cfg<NP, 2, 3>(mh, mw, a, n_rows_bound, st);
  } else {
    switch (ring_sub()) {
      case 1: return launch_cfg<NP, 1, 8>(mh, mw, a, n_rows_bound, st);
      case 4: return launch_cfg<NP, 4, 2>(mh, mw, a, n_rows_bound, st);
      default: return launch_cfg<NP, 2, 4>(mh, mw, a, n_rows_bound, st);
    }
  }
}

static int g_route_fused = 1;
int gate_route_fused() { return g_route_fused; }
void set_gate_route_fused(int on) { g_route_fused = on ? 1 : 0; }

static int g_gate_tc = 1;
int gate_tc_enabled() { return g_gate_tc; }
void set_gate_tc_enabled(int on) { g_gate_tc = on ? 1 : 0; }

// W box rows N': N rounded up to 16, and above 64 to 128 / 160 / 192 / 256
int gate_tc_rows(int32_t n_experts) {
  const int r = std::max(16, (n_experts + 15) / 16 * 16);
  if (r <= 64) return r;
  return r <= 128 ? 128 : r <= 160 ? 160 : r <= 192 ? 192 : 256;
}

bool gate_tc_supported(int32_t n_experts, int32_t top_k, int64_t d) {
  return n_experts >= 1 && n_experts <= kMaxExperts && top_k >= 1 && top_k <= kGtMaxK &&
         top_k <= n_experts && d % (4 * kGemmBK) == 0;
}

int launch_gate_tc(const CUtensorMap& map_h, const CUtensorMap& map_w, const GateTcArgs& a,
                   int64_t n_rows_bound, cudaStream_t st) {
  if (n_rows_bound <= 0) return SMOE_OK;
  switch (gate_tc_rows(a.n_experts)) {
    case 16: return launch_np<16>(map_h, map_w, a, n_rows_bound, st);
    case 32: return launch_np<32>(map_h, map_w, a, n_rows_bound, st);
    case 48: return launch_np<48>(map_h, map_w, a, n_rows_bound, st);
    case 64: return launch_np<64>(map_h, map_w, a, n_rows_bound, st);
    case 128: return launch_np<128>(map_h, map_w, a, n_rows_bound, st);
    case 160: return launch_np<160>(map_h, map_w, a, n_rows_bound, st);
    case 192: return launch_np<192>(map_h, map_w, a, n_rows_bound, st);
    case 256: return launch_np<256>(map_h, map_w, a, n_rows_bound, st);
    default: return SMOE_ERR_UNSUPPORTED;
  }
}

}  // namespace smoe

#ifdef SMOE_GATE_PROBE
extern "C" int smoe_probe_gate_ts(unsigned long long* host, int rows) {
  if (rows > 2048) rows = 2048;
  return cudaMemcpyFromSymbol(host, smoe::g_gate_ts, sizeof(unsigned long long) * 16 * rows) ==
                 cudaSuccess
             ? 0
             : -1;
}
extern "C" int smoe_probe_gate_reset() {
  static unsigned long long zero[2048 * 16];
  return cudaMemcpyToSymbol(smoe::g_gate_ts, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif

SMOE_TL_EXPORT(gate)
