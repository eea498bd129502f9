// qfb_kernels.h — launch-level interface between the C-ABI host code
// (qfb_api.cpp) and the sm_100a kernels (qfb_fwd.cu, qfb_bwd.cu).
// Parameter tables are passed BY VALUE as __grid_constant__ kernel
// parameters (<= 32 KB), so every launch is self-contained and CUDA-graph
// capturable; nothing is staged through host-pinned memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qfb.h"

namespace qfb {

// Sets the thread-local qfb_last_error() message (qfb_api.cpp).
qfb_status set_error(qfb_status st, const char* msg);
// Context internals for the other TUs: a grow-only device scratch buffer
// per slot (0..3), the stream/device, launch accounting, CUDA error mapping.
qfb_status ctx_scratch(qfb_ctx* ctx, int slot, size_t bytes, void** p);
cudaStream_t ctx_stream(const qfb_ctx* ctx);
int ctx_device(const qfb_ctx* ctx);
void ctx_count_launches(qfb_ctx* ctx, int n);
qfb_status cuda_error(cudaError_t e, const char* where);

// Programmatic dependent launch for the main kernels (fwd TMA / ew, bwd,
// finisher): each of them executes griddepcontrol.wait before touching
// global memory and griddepcontrol.launch_dependents early, so the next
// kernel's CTAs are scheduled into SM slots as this grid's CTAs retire and
// its launch latency overlaps the tail. Stream order is unchanged: a
// dependent still observes every write of the grid before it.
// Which launches carry the attribute: bit 1 forward, 2 backward, 4
// finisher, 8 small forward launches (fewer than 4 chunks per CTA);
// QFB_PDL overrides the default mask (4).
constexpr int kPdlFwd = 1, kPdlBwd = 2, kPdlFin = 4, kPdlFwdSmall = 8;
bool pdl_enabled(int which);
// cudaLaunchKernelExC with the programmatic-serialization attribute when
// pdl_enabled(which).
cudaError_t launch_main(const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                        cudaStream_t st, int which);

struct FastDivHost {
  uint32_t d, m, s, pad;
};

inline FastDivHost make_fastdiv(uint32_t d) {
  FastDivHost f{d, 0u, 0u, 0u};
  if (d <= 1) {
    f.d = 1;
    return f;
  }
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;  // s = ceil(log2 d)
  const uint64_t m = ((1ull << 32) * ((1ull << s) - d)) / d + 1;
  f.m = (uint32_t)m;
  f.s = s;
  return f;
}

// ------------------------------------------------------ elementwise ----
constexpr int kEwThreads = 256;
constexpr int kEwUnroll = 4;
constexpr int kEwChunk = kEwThreads * kEwUnroll;  // units per chunk
constexpr int kMaxEwDesc = 96;

constexpr uint32_t kEwHalfGrid = 0x1u;   // == QFB_FLAG_HALF_GRID
constexpr uint32_t kEwStreaming = 0x2u;  // == QFB_FLAG_STREAMING
constexpr uint32_t kEwInt8Out = 0x4u;    // == QFB_FLAG_INT8_OUT: outputs are int8 codes
constexpr uint32_t kEwDemoteIn = 0x100u; // chain: demote v before FQ

// One fused elementwise job: v = act(a (+ b)) [demote]; preact = v;
// y[j] = FQ(v, s[j][ch]) [half]. Plain FQ forward: b = preact = NULL,
// act = none, no demote.
struct EwDesc {
  const void* a;
  const void* b;
  void* preact;
  void* y[2];
  const float* s[2];
  uint32_t nunits;  // vector units (vec elements each) or elements (vec 1)
  uint32_t vec;
  FastDivHost inner_u;  // units per [inner] row
  FastDivHost chans;    // channels
  int32_t n_out;
  int32_t act;
  uint32_t flags;
  float q;
};

struct EwBatch {
  int32_t n;
  uint32_t chunk_units;  // TMA path: units per chunk (<= kEwChunk); the register path uses kEwChunk
  uint32_t chunk_begin[kMaxEwDesc + 1];
  EwDesc d[kMaxEwDesc];
};

// dtype: 0 f32, 1 f16.
cudaError_t ew_occupancy(int dtype, bool chain, int* blocks_per_sm);
cudaError_t launch_ew(int dtype, bool chain, const EwBatch& b, uint32_t* status, int grid,
                      cudaStream_t st);
// TMA-staged plain forward: every descriptor must be on the vector path.
// chain = true: quant->act->quant descriptors (a and b staged); stages =
// TMA ring depth 2..4 (16 KB chunks per array).
constexpr int kTmaStagesMin = 2, kTmaStagesMax = 4;
cudaError_t ew_tma_occupancy(int dtype, bool chain, int stages, int* blocks_per_sm);
cudaError_t launch_ew_tma(int dtype, bool chain, int stages, const EwBatch& b, uint32_t* status,
                          int grid, cudaStream_t st,
                          bool small = false);

// int8 codes (vec path when aligned).
struct CodesDesc {
  const void* x;
  int8_t* codes;
  const float* s;
  uint32_t nunits;
  uint32_t vec;
  FastDivHost inner_u;
  FastDivHost chans;
  float q;
  uint32_t pad;
};
cudaError_t launch_codes(int dtype, const CodesDesc& d, int grid, cudaStream_t st);

// Per-operator sweeps (exec.hpp:276-342): op 0 divide, 1 clip, 2 round,
// 3 multiply. Elements are scalar; in/out float except op 0 input and
// op 3 output which use dtype.
struct PerOpDesc {
  const void* in;
  void* out;
  const float* s;
  uint64_t n;
  uint64_t inner;
  uint64_t chans;
  float q;
  uint32_t flags;
};
cudaError_t launch_perop(int dtype, int op, const PerOpDesc& d, uint32_t* status,
                         int grid, cudaStream_t st);

cudaError_t launch_fill_rng(int dtype, void* out, int64_t n, uint64_t seed, uint64_t stream,
                            uint64_t offset, int kind, double lo, double hi, int grid,
                            cudaStream_t st);

struct ResolveDesc {
  const double* log_s;
  float* s32;
  double* s64;
  double* chain;
  int64_t n;
  double lo, s_max, eps;
};
cudaError_t launch_resolve(const ResolveDesc& d, uint32_t* status, cudaStream_t st);

// --------------------------------------------------------- backward ----
constexpr int kBwdThreads = 256;
constexpr int kBwdGroupsLog = 8;  // leaf groups per full tile (= threads)
constexpr int kLeafMax = 16;      // leaf-group size bound (two <=8 folds)
constexpr int kBwdTileMax = kLeafMax << kBwdGroupsLog;  // 4096 elements
constexpr int kMaxBwdDesc = 64;

struct BwdDesc {
  const void* x;
  const void* up;
  void* dx;
  const double* s64;
  const double* chain;
  double* d_log_s;
  double* partials;  // [segments * tps] tile sums, reduced by bwd_finish
  uint64_t inner;    // row (segment) length n
  uint32_t outer;
  uint32_t chans;
  uint32_t tps_log;  // tiles per segment = 2^(depth - g)
  uint32_t part_log; // partials per segment (row) = 2^part_log, reduced by the finisher
  uint32_t depth;    // tree depth of the 16-bounded leaf groups
  uint32_t g;        // tile depth = min(depth, kBwdGroupsLog)
  int32_t accumulate;  // 0 fold, 1 fold into d_log_s, 2 (QFB_BWD_ROWS) one value per row
  double q;
  uint32_t vec;  // x/up/dx 16-byte aligned: TMA bulk staging
  uint32_t pad;
  uint64_t total_bytes;  // outer * chans * inner * sizeof(T)
  uint64_t row_stride;   // QFB_BWD_ROWS: d_log_s[o * row_stride + c]
  // streaming backward (sbwd_kernel) only: per-chunk block metadata of this
  // row shape (kSbMetaWords u32 per chunk of a row, built by the host) and
  // the chunks per row
  const uint32_t* sb_meta;
  uint32_t sb_nch;
  uint32_t pad3;
  FastDivHost sb_nch_div;
};

struct BwdBatch {
  int32_t n;
  int32_t nstages;       // TMA ring depth (2..4), sized from the max tile
  uint32_t stage_elems;  // elements per array per stage (16-byte multiple)
  uint32_t warp_part;    // tile kernel: consumer warps store the partials (tps_log = depth - 5)
  uint32_t layout;       // full-tile consumer layout: kBwdLayout* (warp_part batches only)
  uint32_t pad0;
  uint32_t tile_begin[kMaxBwdDesc + 1];
  BwdDesc d[kMaxBwdDesc];
};

// Consumer layouts of the full-tile kernel (BwdBatch::layout), bit flags:
// 8 warps x 1 leaf group per lane, or (kBwdLayoutQuad) 4 warps x 2 adjacent
// groups per lane (quad_sum); rint by FRND.F64 or (kBwdLayoutMagic) by the
// magic-number add (rint_small); the quotient by markstein2_div or
// (kBwdLayoutDD) markstein_dd. Every layout gives the same bits.
constexpr uint32_t kBwdLayout8 = 0;
constexpr uint32_t kBwdLayoutMagic = 1;
constexpr uint32_t kBwdLayoutQuad = 2;
constexpr uint32_t kBwdLayoutDD = 4;
constexpr uint32_t kBwdLayoutTwoCtas = 8;  // 2 CTAs per SM (up to 112 registers per thread)
constexpr uint32_t kBwdLayoutHalfF32 = 16; // binary16 storage: float32 terms (QFB_OPT_BWD_HALF_FP32)
constexpr uint32_t kBwdLayoutPrefetch = 32; // producer L2 prefetch one tile beyond the ring
constexpr uint32_t kBwdLayoutCU = 64;       // CTA-uniform main pass (bwd_cu_kernel)
// tiles visited last to first (runtime bit of the warp-specialized kernel,
// not a kernel instance): the step's backward starts on the quant points
// the forward touched last, whose inputs may still sit in L2
constexpr uint32_t kBwdLayoutReverse = 128;

cudaError_t bwd_occupancy(int dtype, int* blocks_per_sm);  // at the default ring size
cudaError_t bwd_occupancy_smem(int dtype, size_t smem, int* blocks_per_sm, bool warp_part = false,
                               uint32_t layout = kBwdLayout8);
// Ring sizing: stage_elems / nstages / dynamic smem for a batch whose
// largest tile has max_tile elements.
void bwd_ring_size(int dtype, uint32_t max_tile, uint32_t* stage_elems, int32_t* nstages,
                   size_t* smem_bytes);
// Main pass (tile partials) + finisher (segment trees, chain, outer fold);
// stream order replaces fences and tickets.
// fin_stream != nullptr: the finisher goes to fin_stream after `fork` (recorded
// on st after the main pass); the caller joins it later.
cudaError_t launch_bwd(int dtype, const BwdBatch& b, int grid, cudaStream_t st,
                       cudaEvent_t after_main = nullptr, cudaStream_t fin_stream = nullptr,
                       cudaEvent_t fork = nullptr);
// The finisher alone: per (descriptor, channel) the perfect tree over the
// 2^tps_log partials of each row, times chain, folded over the rows.
cudaError_t launch_bwd_finish(const BwdBatch& b, cudaStream_t st);

// ---------------------------------------------- streaming backward ----
// sbwd_kernel (qfb_sbwd.cu): fixed row-relative chunks of kSbChunk
// elements, TMA-staged with the overhang of the chunk's last tree block;
// element-parallel terms into shared memory, then one half-warp per block
// of 16 leaf groups (a tree node at depth D - 4) folds and reduces it; the
// block partials feed the same finisher (tps_log = D - 4).
constexpr int kSbThreads = 256;
constexpr int kSbChunk = 1024;        // elements of a row per chunk
constexpr int kSbBlockLog = 4;        // leaf groups per block = 16
constexpr int kSbMaxBlk = 256;        // block length bound (16 groups x 16)
constexpr int kSbWarpBlocks = 1;      // blocks per consumer warp (8 warps x 1 >= 1024 / 128)
constexpr int kSbMaxBlocks = 8 * kSbWarpBlocks;  // block starts per chunk bound (blocks >= 128 elements)
constexpr int kSbMetaWords = 24;      // {jb0, nblk, le, 0, lo[0..nblk]} padded to 96 bytes
constexpr int kSbWin = kSbChunk + kSbMaxBlk;  // staged elements per array per stage
size_t sbwd_smem(int dtype, int stages);
cudaError_t sbwd_occupancy(int dtype, int stages, int* blocks_per_sm);
cudaError_t launch_sbwd(int dtype, int stages, const BwdBatch& b, int grid, cudaStream_t st);

}  // namespace qfb
