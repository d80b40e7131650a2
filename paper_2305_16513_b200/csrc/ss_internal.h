// ss_internal.h -- host/device shared declarations of libss (not part of the ABI).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ss {

constexpr int kOpSum = 0;
constexpr int kOpMax = 1;
constexpr int kOpConv = 2;
constexpr int kOpMin = 3;
// padding modes of the window spec (ss.h ss_pad_mode_t)
constexpr int kPadZeros = 0, kPadReflect = 1, kPadCircular = 2, kPadReplicate = 3;
// max dynamic smem per CTA on sm_100a (227 KB) less room for the static
// ClcSmem work-claim block (ss_device.cuh)
constexpr int kSmemBudget = 227 * 1024 - 128;
constexpr int kConvTmaMaxK = 64;          // largest k served by the TMA conv kernel
constexpr int kPoolTmaMaxW = 1024;        // largest w served by the TMA pool kernel
constexpr int kSlideWarps = 15;           // consumer warps of the 1-D tile kernel
constexpr int kSlideTileRows = kSlideWarps * 16;  // output rows (of 32) per CTA tile

// Parameters of the TMA tile kernel (slide1d.cu).  x and y are viewed as 2-D
// arrays of 128-B rows starting at x_view / y_view (16-B aligned-down copies
// of the caller's pointers); shift_x / shift_y are the element offsets of the
// caller's x / y inside those views.
struct alignas(64) Slide1DParams {
  CUtensorMap tm_x_main;  // box {32, kSlideTileRows}, SWIZZLE_128B
  CUtensorMap tm_x_halo;  // box {32, 8},   SWIZZLE_128B
  CUtensorMap tm_y;       // box {32, 16},  SWIZZLE_128B (valid iff has_y_map)
  const void* x_view;
  void* y_view;
  int64_t N, L, batch;
  int64_t shift_x, shift_y;
  int64_t x_full_elems;   // elements covered by tm_x_* (32 * full rows)
  int64_t x_total_elems;  // shift_x + batch * N
  int64_t tiles_per_row, ntiles;
  int64_t y_rows;         // full 128-B rows of the y view
  int64_t y_pitch;        // y elements between consecutive batch rows (= L unless padded)
  int64_t y_off;          // offset of output 0 inside its y row (left zero padding)
  int64_t w;              // window (pool)
  uint32_t stage_bytes;
  int stages;
  int span;
  int has_y_map;
  int clc;  // 1: one CTA per work unit, units claimed by cluster launch control (ss_device.cuh); 0: static stride
  float taps[kConvTmaMaxK];  // conv taps, zero-padded to the kernel's KT
};

// Parameters of the generic (any stride / alignment / size) kernels.
struct GenericParams {
  const void* x;
  void* y;
  int64_t N, L, batch, w, stride;
  int64_t dilation, pad_left;  // window spec (NEXT #1): x index of tap j of output i = i*s + j*d - pl
  int64_t skip_lo, skip_hi;    // if skip_lo < skip_hi: outputs in [skip_lo, skip_hi) are not computed
  int pad_mode;                // kPadZeros / kPadReflect / kPadCircular / kPadReplicate
  float taps[1024];            // SS_K_MAX
};

struct Pool2DParams {
  const float* x;
  float* y;
  int64_t planes, H, W, OH, OW, kh, kw, sh, sw;
  int64_t bands;        // output-row bands per plane
  int64_t band_rows;    // output rows per band (last band may be shorter)
  int64_t ntiles;       // planes * bands
  uint32_t stage_bytes;
  int stages;
  int bulk;             // 1: rows are 16-B aligned -> cp.async.bulk staging
  int mode;             // 0 max, 1 avg
  float inv_area;       // 1 / (kh * kw) for avg
  int clc;  // 1: one CTA per work unit, units claimed by cluster launch control (ss_device.cuh); 0: static stride
};

void note_launch();
// Grid of a work-claiming kernel (ss_device.cuh ClcSmem): one CTA per unit
// when units are claimed by cluster launch control, else a persistent grid of
// `persistent` CTAs striding statically (clc is cleared if the unit count does
// not fit gridDim.x).
inline int64_t launch_grid(int64_t units, int64_t persistent, int& clc) {
  if (units < 1) units = 1;
  if (clc && units <= 0x7fffffffLL) return units;
  clc = 0;
  return units < persistent ? units : persistent;
}
// SS_DYNAMIC_TILES (read once, default 1): 0 selects the static stride (A/B only).
int dynamic_tiles();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize = kSmemBudget) once per kernel
// per device (thread-safe); returns the first call's status afterwards.
cudaError_t ensure_smem_attr(const void* kfn);
// 2-D [rows][32] view of 4-byte elements, 128-B swizzle, box {32, box_rows}.
bool encode_rows_map(CUtensorMap* m, const void* base, int64_t rows, int box_rows);
int num_sms(int device);

cudaError_t launch_conv_tma(Slide1DParams& p, int KT, cudaStream_t stream, int grid);
cudaError_t launch_pool_tma(Slide1DParams& p, int op, int dtype, int P, cudaStream_t stream,
                            int grid);
cudaError_t launch_pool_generic(const GenericParams& p, int op, int dtype, cudaStream_t stream,
                                int grid);
cudaError_t launch_conv_generic(const GenericParams& p, cudaStream_t stream, int grid);
cudaError_t launch_pool2d(Pool2DParams& p, cudaStream_t stream, int grid);

// Sliding window of gamma pairs (affine.cu).  u, v: [batch][N]; U, V:
// [batch][L]; U may be null.
struct AffineParams {
  const float* u;
  const float* v;
  float* U;
  float* V;
  int64_t N, L, batch, w, stride;
  int64_t tiles_per_row;  // set by launch_affine
  int q, nB;              // set by launch_affine
};
size_t affine_smem_bytes(int64_t w);
cudaError_t launch_affine(AffineParams& p, cudaStream_t stream, int num_sms);
cudaError_t launch_pool2d_direct(const Pool2DParams& p, cudaStream_t stream, int grid);

// Tensor-core conv1d (conv_tc.cu).  The input is viewed
// from x_view (x aligned down to 16 B; shift_x = x's element offset in it) as
// overlapping 128-element chunks: chunk m = view elements [128 m, 128 m + K).
// Output at view position P (window start) goes to
// y[b * y_pitch + y_off + i] with P - shift_x = b * N + i, if i < L_int.
constexpr int kConvTcMaxK = 64;  // K = 127 + k rounded to 8 must fit 2 x 192 TMEM columns
struct alignas(64) ConvTCParams {
  CUtensorMap tm_b;        // 3-D {32, m_ext, atoms}, strides {512 B, 128 B}, box {32, NC, group}, SW128
  const float* x_view;
  float* y;
  int64_t N, L_int, batch, shift_x, y_pitch, y_off;
  int64_t m_ext;           // chunks whose whole K span lies inside the view
  int64_t total_view;      // shift_x + batch * N
  int64_t ntiles;          // set by launch_conv_tc
  int k, K, atoms;         // filter length, MMA K (192), K-atoms (6)
  int hi_stages, lo_bufs;  // group slots (3 K-atoms) of the hi / lo rings (set by launch_conv_tc)
  int mixed;               // 1: TF32 xh*fh + one bf16 correction MMA; 0: 3xTF32
  int clc;  // 1: one CTA per work unit, units claimed by cluster launch control (ss_device.cuh); 0: static stride
  unsigned long long* trace;  // debug: per-tile role timestamps of CTA 0 (null = off)
  float taps[kConvTcMaxK];
};
bool encode_chunk_map(CUtensorMap* m, const void* base, int64_t m_ext, int atoms, int nc);
cudaError_t launch_conv_tc(ConvTCParams& p, int nc, cudaStream_t stream, int grid);

// Backward passes (backward.cu).  dy: [batch][L] (the
// forward output), dx: [batch][N]; x: the forward input (max / filter grad).
struct BackwardParams {
  const void* x;
  const void* dy;
  void* dx;
  int64_t N, L, batch, w, stride;
  float taps[1024];  // conv input gradient: the forward filter f (SS_K_MAX)
};
struct Pool2DBackwardParams {
  const float* x;
  const float* dy;
  float* dx;
  int64_t planes, H, W, OH, OW, kh, kw, sh, sw;
  int mode;  // 0 max, 1 avg
  float inv_area;
};
cudaError_t launch_transpose_window(const BackwardParams& p, int op, int dtype, cudaStream_t stream, int sms);
cudaError_t launch_pool_max_backward(const BackwardParams& p, cudaStream_t stream, int sms);
// Stride-1 max-pool gradient, TMA-staged tile kernel (maxbwd.cu) for the window lengths it is
// instantiated for (pool_max_backward_s1_supported); maps are 1-D over the flat x / dy arrays.
struct alignas(64) MaxBwdS1Params {
  CUtensorMap tm_x, tm_dy;  // fp32 [batch N] and [batch L], boxes of 256, OOB zero fill
  float* dx;
  int64_t N, L, batch, w;
  int64_t tiles_per_row, ntiles;  // set by the launcher
  int T;                          // stored positions per tile (2048 - w - 2)
};
bool pool_max_backward_s1_supported(int64_t w);
cudaError_t launch_pool_max_backward_s1(MaxBwdS1Params& p, cudaStream_t stream, int sms);
bool encode_flat_f32_map(CUtensorMap* m, const void* base, int64_t n);
bool encode_rows128_map(CUtensorMap* m, const void* base, int64_t rows);
int conv_filter_grad_ctas(int sms);
size_t conv_filter_grad_workspace(int64_t k, int ctas);
cudaError_t launch_conv_filter_grad(const BackwardParams& p, float* df, void* workspace, int ctas,
                                    cudaStream_t stream);
cudaError_t launch_pool2d_backward(const Pool2DBackwardParams& p, cudaStream_t stream, int sms);
cudaError_t launch_conv_filter_grad_finish(const double* part, int ctas, int64_t k, float* df, cudaStream_t stream);
// Tensor-core filter gradient (fgrad_tc.cu): stride 1, k <= 64, N % 4 == 0, 16-B aligned x.
struct alignas(64) FgradTcParams {
  CUtensorMap tm_x;              // x as 1-D fp32 [batch N], boxes of 256 (raw rows of a stage by TMA)
  const float* x;
  const float* dy;
  double* part;                  // caller's workspace: per-CTA fp64 partials, [ctas][64]
  int64_t N, L, batch, k;
  int64_t U, units_per_row, nunits;  // set by the launcher
  int64_t ctas;
};
bool tc_filter_grad_enabled();
bool conv_filter_grad_tc_supported(int64_t N, int64_t k, int64_t stride, const void* x);
cudaError_t launch_conv_filter_grad_tc(FgradTcParams& p, float* df, int ctas, int sms, cudaStream_t stream);

// Dilated stride-1 windows (dilated.cu): interior outputs
// i < L_int = N - (w-1) d of each row go to y[b * y_pitch + y_off + i].
struct DilatedParams {
  const void* x;
  void* y;
  int64_t N, L_int, batch, w, d, y_pitch, y_off;
  int stage_floats;  // set by launch_dilated
  float taps[32];    // conv (w <= 32), zero-padded
};
cudaError_t launch_dilated(DilatedParams& p, int op, cudaStream_t stream, int sms);

// 2-D single-channel sliding dot product (conv2d.cu).
struct Conv2DParams {
  const float* x;
  float* y;
  int64_t planes, H, W, OH, OW, kh, kw, sh, sw;
  uint32_t stage_bytes;  // set by launch_conv2d
  int stages;
  int clc;  // 1: one CTA per work unit, units claimed by cluster launch control (ss_device.cuh); 0: static stride
  float taps[1024];      // row-major [kh][kw], kh * kw <= SS_K_MAX
};
cudaError_t launch_conv2d(Conv2DParams& p, cudaStream_t stream, int grid);

// Stride-1 2-D correlation with virtual zero padding on FFMA2 (conv2d_tile.cu):
// ss_conv2d (pad 0) and the input gradient ss_conv2d_backward_input (pad
// KH-1 / KW-1, flipped filter) for 3x3, 5x5, 7x7 filters.
struct alignas(64) Conv2DTileParams {
  CUtensorMap tm_x;    // TMA mode: 3-D {IW, IH, planes}, box {P, TH, 1}, zero fill (encode_plane_map)
  const float* x;      // input planes [planes][IH][IW]
  float* y;            // output planes [planes][OH][OW], OH = IH + 2 pad_t - KH + 1
  int64_t planes;
  int IH, IW, OH, OW, KH, KW;
  int pad_t, pad_l;    // zero rows / columns in front of (and behind) the input
  int pad_c, shift;    // tile left padding pad_c = pad_l + shift, a multiple of 4 (set by the launcher)
  int P;               // shared-tile row pitch in floats (set by the launcher)
  int units, col_blocks;
  uint32_t tile_bytes, raw_bytes, tile_tx;
  int tile_stages, raw_stages;
  int tma;             // 1: each padded tile is one TMA tensor copy (16-B row pitch); 0: dense plane, lanes mask
  int clc;  // 1: one CTA per plane, planes claimed by cluster launch control; 0: static stride
  float taps[64];      // row-major [KH][KW]
};
bool conv2d_tile_supported(int kh, int kw, int64_t oh, int64_t ow);
bool encode_plane_map(CUtensorMap* m, const float* base, int64_t W, int64_t H, int64_t planes, int box_w, int box_h);
// Filter gradient on the same tiles (conv2d_tile.cu): x = p.x [planes][IH][IW], dy [planes][OH][OW];
// writes part[tap * grid + cta] (fp64) and returns grid, or -1 if the shape does not fit.
bool conv2d_df_tile_supported(int kh, int kw, int64_t H, int64_t W, int64_t OH, int64_t OW, const void* x,
                              const void* dy);
int launch_conv2d_df_tile(Conv2DTileParams& p, const float* dy, double* part, int sms, cudaStream_t stream);
cudaError_t launch_conv2d_tile(Conv2DTileParams& p, cudaStream_t stream, int sms);

// Gradients of the 2-D conv (conv2d_backward.cu, reading R21).
struct Conv2DBwdParams {
  const float* x;   // filter gradient
  const float* dy;
  float* dx;        // input gradient
  int64_t planes, H, W, OH, OW, kh, kw, sh, sw;
  int df_xr, df_xc;  // filter-gradient x region pitch (set by the launcher)
  int dx_r, dx_c;    // input-gradient dy region rows / pitch per buffer (set by the launcher)
  float taps[1024];  // input gradient: row-major [kh][kw]
};
cudaError_t launch_conv2d_backward_input(Conv2DBwdParams& p, cudaStream_t stream, int sms);
int conv2d_backward_filter_ctas(int sms);
size_t conv2d_backward_filter_workspace(int64_t taps, int ctas);
cudaError_t launch_conv2d_backward_filter(Conv2DBwdParams& p, float* df, void* workspace, int ctas,
                                          cudaStream_t stream);

// Multi-channel conv1d / conv2d, channels-last bf16 (conv_mc.cu; SURVEY 8f NEXT #4,
// readings R18, R22).  Positions are flat over batch x (H x) W; tap j reads the
// staged tile shifted by tap_off[j] positions (1-D: j; 2-D: a W + e).
constexpr int kMcMaxTaps = 64;
struct alignas(64) ConvMcParams {
  CUtensorMap tm_x;  // 3-D {64, positions, cin/64}, box {64, box_rows, 1}, SW128, bf16 (encode_mc_map)
  const void* x;     // [batch][N][cin] or [batch][H][W][cin] bf16
  const void* w;     // [cout][cin][k] or [cout][cin][kh][kw] bf16 (k = taps)
  float* y;          // [batch][L][cout] or [batch][OH][OW][cout] fp32
  int64_t batch, N, L, cin, cout, k;  // 1-D geometry (2-D: N = H * W, k = kh * kw)
  int64_t H, W, OH, OW;               // 2-D geometry (two_d)
  int two_d;
  int rows, box_rows, nbox, stages;   // staged positions per tile (multiple of 8), TMA boxes per atom, ring depth
  int batched;        // 1: tiles never cross batch rows; tm_x is 4-D {64, positions, atoms, batch} and a
                      //    tile's box starts `pad` positions early (zero-filled outside the row)
  int pad;            // left zero padding of each row (batched mode)
  int bwd_in;         // 1: weights staged transposed and flipped (input gradient: w'[ci][co][j] = w[co][ci][k-1-j])
  int64_t n_out, tiles_per_row;       // batched mode: outputs per row, tiles per row
  int mblk, nacc;  // 128-position M-blocks per tile (1, 2), TMEM accumulators (tiles in flight)
  uint32_t w_magic; int w_shift;     // 2-D: r = (umulhi(i, w_magic) + i) >> w_shift == i / W for i < 2^31
  int tap_off[kMcMaxTaps];
  // pad2d (2-D input gradient, reading R26): a tile is pd_R rows x pd_Cw columns of dx, staged as one
  // 5-D TMA box per atom of (pd_R + kh - 1) x pd_P dy positions (pitch pd_P = pd_Cw + kw - 1) starting
  // kh-1 rows / kw-1 columns early (zero-filled outside dy); tm_x is {64, OW, OH, atoms, batch}.
  // x = dy, y = dx, cin = dy channels, cout = dx channels, H x W = dx, OH x OW = dy.
  int pad2d, pd_kh, pd_kw, pd_P, pd_R, pd_Cw, pd_tx;
  int64_t pd_nrt, pd_nct;  // row / column tiles per image
  int64_t ntiles;    // set by launch_conv_mc
  int clc;  // 1: one CTA per work unit, units claimed by cluster launch control (ss_device.cuh); 0: static stride
};
bool encode_mc_map(CUtensorMap* m, const void* x, int64_t positions, int64_t cin, int box_rows);
bool encode_mc_map_batched(CUtensorMap* m, const void* x, int64_t batch, int64_t positions, int64_t cin,
                           int box_rows);
cudaError_t launch_conv_mc(ConvMcParams& p, bool tensor_path, cudaStream_t stream, int sms);
// pad2d tiling (sets pd_*, mblk, rows, tap_off); false: no tensor-core plan fits
bool conv_mc_plan_pad2d(ConvMcParams& p);
bool encode_mc_map_2d(CUtensorMap* m, const void* x, int64_t batch, int64_t OH, int64_t OW, int64_t c, int box_w,
                      int box_h);
// Multi-channel conv1d filter gradient (mc_fgrad.cu; reading R25): tensor cores for cin = 64,
// cout 64 (k <= 4) / 128 (k <= 2), else a direct kernel.  ws: per-CTA fp64 slices [sms][64 k][128].
struct alignas(64) McFgradParams {
  CUtensorMap tm_dy, tm_x;  // batched maps: dy {64, L, cout/64, batch} box 128 rows, x {64, N, 1, batch} box 136
  const uint16_t* dy;
  const uint16_t* x;
  float* dw;
  double* ws;
  int64_t batch, N, L, cin, cout, k;
  int64_t tiles_per_row, ntiles;  // set by the launcher
  int stages;                     // set by the launcher
  // 2-D (reading R27; k = kw, N = H * W): a tile is R dy rows staged with pitch W (dy box {64, W, R} of
  // the 5-D map {64, OW, OH, atoms, batch}: columns >= OW zero-filled) against x rows r0 + a .. r0 + a + R
  // (box {64, W, R + 1}); CTA c serves tap row a = c % kh.  Staged rows past the boxes are zeroed once.
  int two_d, kh, R, xrows, dy_rows, x_rows;  // xrows: x rows per stage (1-D: 136); rows the boxes fill
  uint32_t tx_dy, tx_x;                      // bytes one dy region / the x box deliver
  int64_t H, W, OH, OW, nrt;                 // 2-D geometry; row tiles per image
  // CTA groups (2-D: one per tap row, or per tap-row pair): pair = 1 (cout = 64) runs M = 128 MMAs whose
  // second dy region is the tile one image row down, accumulating tap rows a (rows 0-63) and a - 1
  // (rows 64-127) together; tiles then start one row early (shift).  mr: slice rows; dyreg: dy regions
  int groups, pair, shift, mr, dyreg;
  // dy staging: regions of dyrow_cap rows (the box fills dy_fill); ks K-steps of 16 positions; alo = the A
  // operand's M-atom stride (a region, or -- shifted mode, R W % 16 == 0 -- W rows: ONE region of R + 1
  // dy rows serves both halves of a paired accumulator)
  int dyrow_cap, dy_fill, ks;
  uint32_t alo;
};
bool mc_filter_grad_tc_supported(int64_t cin, int64_t cout, int64_t k);
bool mc_filter_grad_2d_plan(McFgradParams& p);  // 2-D tensor-core tiling (sets R, xrows, ...); false: direct
size_t mc_filter_grad_workspace(int64_t cin, int64_t cout, int64_t k, int sms, bool two_d = false);
cudaError_t launch_mc_filter_grad(McFgradParams& p, bool tc, cudaStream_t stream, int sms);
// Staged rows as the TMA boxes round them: multiple of 8, split into <= 256-row boxes of equal size
inline int mc_round_rows(int rows, int* nbox = nullptr, int* box_rows = nullptr) {
  rows = (rows + 7) / 8 * 8;
  const int nb = (rows + 255) / 256, br = ((rows + nb - 1) / nb + 7) / 8 * 8;
  if (nbox) *nbox = nb;
  if (box_rows) *box_rows = br;
  return br * nb;
}
// M-blocks per multi-channel tile: 2 (256 positions per tile, half the per-tile barrier round trips
// and a smaller halo share) when a 3-stage ring of rows1 + 128 staged positions fits next to the weights
// and the shape does not prefer one M-block (forward passes with k <= 4 and the 2-D forward: measured
// 2-3% faster with 128-position tiles, the 1-D k = 9 forward and the input gradients with 256)
int conv_mc_choose_mblk(int64_t cin, int64_t cout, int64_t k, int rows1, bool prefer_one = false);

}  // namespace ss
