// gemm.h — host interface of the tcgen05 grouped GEMM (K6).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/smoe.h"

namespace smoe {

enum GemmEpilogue : int32_t {
  kEpiStore = 0,    // C[c_off + i, n] = bf16(acc)
  kEpiSwiGLU = 1,   // C[c_off + i, n'] = bf16(silu(acc_gate) * acc_up), B packed by pack_w13
  kEpiScatter = 2,  // row i goes to dst_base[meta >> 40] + (meta & mask) * ldd  (A2A combine)
};

constexpr int kGemmBM = 128;
constexpr int kGemmBN = 256;
constexpr int kGemmBK = 64;
constexpr int kGemmNarrowM = 32;      // m-block rows of the narrow (decode) variant
constexpr int kGemmMaxProblems = 512;
constexpr int kGemmNarrowMaxProblems = 192;   // problem table of the narrow variant
constexpr int64_t kMetaSlotMask = (int64_t(1) << 40) - 1;

struct GemmArgs {
  const int64_t* problems;   // [P, 4] {a_off, m, b_index, c_off}
  int32_t num_problems;
  int32_t num_k_blocks;      // K / 64
  int32_t n_tiles_n;         // n_b / 256
  int32_t n_b;               // rows of B per problem (output columns before SwiGLU)
  int32_t group_m;           // > 0: m-blocks per rasterisation group; < 0: -(n-blocks per
                             // n-group); 0: derive from K
  char* c;                   // store / swiglu output
  int64_t ldc;               // elements
  int32_t b_tiled;           // B in smoe_tile_weights layout (one contiguous box per
                             // (problem b_index, n-block, k-block)); else row-major
  const int64_t* meta;       // scatter: per A row
  char* dst_base[SMOE_MAX_SHARDS];
  int64_t ldd;               // elements
  // Per-problem readiness between the two expert GEMMs of a decode-sized
  // forward (ready_role 0 = off).  Role 1 (up GEMM, one SM per 128-row tile):
  // after its epilogue has stored a tile's hidden rows, one thread adds 1 to
  // ready[p] (release, after a generic->async proxy fence).  Role 2 (down
  // GEMM, launched early under PDL): skips griddepcontrol.wait and its TMA
  // producer waits, per tile, until ready[p] counts every up tile of problem
  // p (ceil(m / ready_up_tile_m) * ready_up_n_tiles); a wait past ~10 ms sets
  // SMOE_ERRBIT_TIMEOUT in err and gives up instead of hanging.
  int32_t* ready;
  int32_t ready_role;
  int32_t ready_up_tile_m;
  int32_t ready_up_n_tiles;
  int32_t* err;
  // non-null (the decode down GEMM, whose CTAs start staggered as the up
  // GEMM's tiles finish): tiles are taken from this zeroed counter instead of
  // blockIdx-strided, so early-starting CTAs take more of them (cg == 1)
  int32_t* tile_counter;
};

// Encodes a 2D bf16 K-major tensor map (rows x cols, box 64 x box_rows, 128B swizzle).
int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols,
                   int32_t box_rows);

// cta_group of the up (which = 0) / down (which = 1) GEMM: 1 = one SM per
// 128x256 tile, 2 = SM pair per 256x256 tile (tcgen05 cta_group::2).
int gemm_cta_group(int which);
// The layer's down GEMM uses the SM pair only above this many routed rows per
// expert on average (SMOE_OPT_GEMM_PAIR_MIN_ROWS).
int gemm_pair_min_rows();
void set_gemm_pair_min_rows(int rows);
void set_gemm_cta_group(int which, int cg);
// Rows of B staged per CTA per k-block: the box height of B's tensor map.
int gemm_b_box_rows(int cg);

// Narrow m-blocks (cg = 0 in launch_grouped_gemm) while the batch has at most
// this many routed rows per expert on average (SMOE_OPT_GEMM_NARROW_MAX_ROWS).
int gemm_narrow_max_rows();
void set_gemm_narrow_max_rows(int rows);

// cg: 1 = one SM per 128x256 tile, 2 = SM pair per 256x256 tile, 0 = one SM
// per 32x256 tile (narrow; tmap_a must have kGemmNarrowM-row boxes).
// Tile order of the up (which = 0) / down (which = 1) GEMM: 0 = derived from
// K (A-resident groups of m-blocks that fit ~40 MB of L2, else B-resident);
// > 0: m-blocks per group; < 0: -(n-blocks per group).  SMOE_OPT_GEMM_GROUP_M_*.
int gemm_group_m(int which);
void set_gemm_group_m(int which, int v);

// SMOE_OPT_EARLY_DOWN (default 1)
int gemm_early_down();
void set_gemm_early_down(int on);

int launch_grouped_gemm(const CUtensorMap& tmap_a, const CUtensorMap& tmap_b,
                        const GemmArgs& args, int32_t epilogue, int cg, cudaStream_t stream);

}  // namespace smoe
